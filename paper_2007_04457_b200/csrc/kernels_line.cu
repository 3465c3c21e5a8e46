// kernels_line.cu -- the fused level kernels of 1D grids (canonical extents
// (1, 1, n)): one thread per coarse node q reads the five fine values
// u[2q-2 .. 2q+2] (neighbouring threads share them through L1) and forms
//   * the mass-trans load K u at q (correction.hpp:141-154; in recompose mode
//     the coarse nodes are masked, correction.hpp:251),
//   * decompose: the coefficient of the refined cell 2q+1 (transforms.hpp:41-55)
//     and 0 at the coarse cell 2q (the assembly writes the pyramid there),
//   * recompose: the coarse node gathered into C_{l-1}.
// As in the 3D fused path, decompose applies K to U itself (K P = M_c), so the
// Thomas solve of the load gives the corrected coarse values directly.
// k_line_interp is GPK^-1 (refactor.hpp:77-87): coarse = C - Z, refined =
// coef + interp (or interp only). Both are HBM streams; the Thomas solve runs
// on k_thomas_long (kernels_thomas.cu).
#include "kernels.cuh"
#include "kernels_fused.cuh"
#include "launch.cuh"
#include "ptx.cuh"
#include "plan.hpp"

namespace hgrb {

namespace {

template <class T>
struct Pair;
template <>
struct Pair<float> { using type = float2; };
template <>
struct Pair<double> { using type = double2; };

template <class T, int MODE>
__global__ void __launch_bounds__(256)
    k_line_level(const T* __restrict__ U, T* __restrict__ coef, T* __restrict__ z,
                 T* __restrict__ gather, const T* __restrict__ taps, const T* __restrict__ wl,
                 const T* __restrict__ wr, int64_t n, int64_t nc, int* flag) {
  constexpr bool DEC = MODE == kFusedDecompose, REC = MODE == kFusedRecompose;
  ptx::pdl_trigger();
  ptx::pdl_wait();
  bool bad = false;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nc;
       q += int64_t(gridDim.x) * blockDim.x) {
    T u[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int64_t j = 2 * q - 2 + k;
      u[k] = (j >= 0 && j < n) ? U[j] : T(0);
    }
    T acc = T(0);
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int64_t j = 2 * q - 2 + k;
      if (j < 0 || j >= n) continue;
      if (REC && !(k & 1)) continue;  // masked coarse nodes (even j)
      acc += taps[q * 5 + k] * u[k];
    }
    z[q] = acc;
    if (DEC) {
      bad |= !isfinite(u[2]);
      if (q + 1 < nc) {
        bad |= !isfinite(u[3]);
        const T cv = u[3] - (wl[q] * u[2] + wr[q] * u[4]);
        using P2 = typename Pair<T>::type;
        *reinterpret_cast<P2*>(coef + 2 * q) = P2{T(0), cv};
      } else {
        coef[2 * q] = T(0);
      }
    }
    if (REC) gather[q] = u[2];
  }
  if (DEC && flag && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

template <class T, bool WITH, bool HASZ>
__global__ void __launch_bounds__(256)
    k_line_interp(const T* coef, T* out, const T* __restrict__ C, const T* __restrict__ Z,
                  const T* __restrict__ wl, const T* __restrict__ wr, int64_t nc) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nc;
       q += int64_t(gridDim.x) * blockDim.x) {
    const T c0 = HASZ ? C[q] - Z[q] : C[q];
    if (q + 1 < nc) {
      const T c1 = HASZ ? C[q + 1] - Z[q + 1] : C[q + 1];
      const T ip = wl[q] * c0 + wr[q] * c1;
      const T v = WITH ? coef[2 * q + 1] + ip : ip;  // read before the pair store (in place)
      using P2 = typename Pair<T>::type;
      *reinterpret_cast<P2*>(out + 2 * q) = P2{c0, v};
    } else {
      out[2 * q] = c0;
    }
  }
}

template <class T, int MODE>
void run_line(const T* U, T* coef, T* z, T* gather, const LevelArgs<T>& a, int* flag,
              cudaStream_t s) {
  const int64_t nc = a.c[2];
  launch_pdl(k_line_level<T, MODE>, dim3(grid_for(nc, 256)), dim3(256), 0, s, a.e[2], U, coef, z,
             gather,
             a.taps[2], a.wl[2], a.wr[2], a.e[2], nc, flag);
}

template <class T, bool WITH, bool HASZ>
void run_line_interp(const T* coef, T* out, const T* C, const T* Z, const LevelArgs<T>& a,
                     cudaStream_t s) {
  const int64_t nc = a.c[2];
  launch_pdl(k_line_interp<T, WITH, HASZ>, dim3(grid_for(nc, 256)), dim3(256), 0, s, a.e[2], coef,
             out, C, Z,
             a.wl[2], a.wr[2], nc);
}

}  // namespace

template <class T>
bool launch_line_level(const T* U, T* coef, T* z, T* gather, const LevelArgs<T>& a, int mode,
                       int* flag, cudaStream_t s) {
  const auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & (2 * sizeof(T) - 1)) == 0; };
  if (a.e[0] != 1 || a.e[1] != 1 || a.e[2] < 3) return false;
  if (mode == kFusedDecompose) {
    if (!al(coef)) return false;  // pair stores
    run_line<T, kFusedDecompose>(U, coef, z, gather, a, flag, s);
  } else if (mode == kFusedLoadOnly) {
    run_line<T, kFusedLoadOnly>(U, coef, z, gather, a, flag, s);
  } else {
    run_line<T, kFusedRecompose>(U, coef, z, gather, a, flag, s);
  }
  return true;
}

template <class T>
bool launch_line_interp(const T* coef, T* out, const T* C, const T* Z, const LevelArgs<T>& a,
                        bool with, cudaStream_t s) {
  const auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & (2 * sizeof(T) - 1)) == 0; };
  if (a.e[0] != 1 || a.e[1] != 1 || a.e[2] < 3 || !al(out)) return false;
  if (with && Z) run_line_interp<T, true, true>(coef, out, C, Z, a, s);
  else if (with) run_line_interp<T, true, false>(coef, out, C, Z, a, s);
  else if (Z) run_line_interp<T, false, true>(coef, out, C, Z, a, s);
  else run_line_interp<T, false, false>(coef, out, C, Z, a, s);
  return true;
}

template bool launch_line_level<float>(const float*, float*, float*, float*,
                                       const LevelArgs<float>&, int, int*, cudaStream_t);
template bool launch_line_level<double>(const double*, double*, double*, double*,
                                        const LevelArgs<double>&, int, int*, cudaStream_t);
template bool launch_line_interp<float>(const float*, float*, const float*, const float*,
                                        const LevelArgs<float>&, bool, cudaStream_t);
template bool launch_line_interp<double>(const double*, double*, const double*, const double*,
                                         const LevelArgs<double>&, bool, cudaStream_t);

}  // namespace hgrb
