// kernels_interp.cu -- recompose interpolation (GPK^-1, refactor.hpp:77-87).
//
// k_interp_rec: one thread per fine column, streaming down the fine rows of a
// (planes x rows) tile; the corrected coarse block (C - Z) sits in shared
// memory, the in-plane interpolant of odd rows is formed from the two even
// rows held in registers. out[coarse] = C - Z, out[refined] = coef + interp
// (or interp alone for classes above the recompose prefix). In-place safe.
#include <algorithm>

#include "kernels.cuh"
#include "kernels_fused.cuh"
#include "plan.hpp"

namespace hgrb {

namespace {

// ---- recompose interpolation -------------------------------------------------

template <class T, int B0, int B1, int B2>
__global__ void __launch_bounds__(2 * B2) k_interp_rec(const T* coef, T* out, const T* __restrict__ C,
                                                       const T* __restrict__ Z, LevelArgs<T> a,
                                                       bool with, int nb1, int nb2) {
  constexpr int NT = 2 * B2, S1 = B1 + 1, S2 = B2 + 2;
  extern __shared__ __align__(16) unsigned char smem_i[];
  T* cs = reinterpret_cast<T*>(smem_i);  // (B0+1) x S1 x S2 corrected coarse block
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int bid = blockIdx.x;
  const int b2 = bid % nb2;
  bid /= nb2;
  const int b1 = bid % nb1;
  const int b0 = bid / nb1;
  const int64_t c0 = a.c[0], c1 = a.c[1], c2 = a.c[2];
  const int64_t e0 = a.e[0], e1 = a.e[1], e2 = a.e[2];
  const int64_t qa0 = int64_t(b0) * B0, qa1 = int64_t(b1) * B1, qa2 = int64_t(b2) * B2;
  const int nb0 = int((c0 - 1 + B0 - 1) / B0) > 0 ? int((c0 - 1 + B0 - 1) / B0) : 1;
  const int tb0 = b0 == nb0 - 1 ? int(c0 - qa0) : B0;
  const int tb1 = b1 == nb1 - 1 ? int(c1 - qa1) : B1;
  const int tb2 = b2 == nb2 - 1 ? int(c2 - qa2) : B2;
  const int n0 = int(std::min<int64_t>(tb0 + 1, c0 - qa0));
  const int n1 = int(std::min<int64_t>(tb1 + 1, c1 - qa1));
  const int n2 = int(std::min<int64_t>(tb2 + 1, c2 - qa2));
  // corrected coarse block C - Z: rows (x0, x1) over warps, columns over lanes
  for (int row = warp; row < n0 * n1; row += NT / 32) {
    const int x0 = row / n1, x1 = row - x0 * n1;
    const int64_t q = ((qa0 + x0) * c1 + qa1 + x1) * c2 + qa2;
    T* dst = cs + (x0 * S1 + x1) * S2;
    for (int x2 = lane; x2 < n2; x2 += 32) dst[x2] = Z ? C[q + x2] - Z[q + x2] : C[q + x2];
  }
  __syncthreads();
  // owned fine ranges [2qa, min(2(qa+tb), e))
  const int f0 = int(std::min<int64_t>(2 * (qa0 + tb0), e0) - 2 * qa0);
  const int f1 = int(std::min<int64_t>(2 * (qa1 + tb1), e1) - 2 * qa1);
  const int f2 = int(std::min<int64_t>(2 * (qa2 + tb2), e2) - 2 * qa2);
  for (int x2 = tid; x2 < f2; x2 += NT) {
    const int b = x2 >> 1;
    const bool o2 = x2 & 1;
    const int64_t i2 = 2 * qa2 + x2;
    const T wl2 = o2 ? a.wl[2][i2 >> 1] : T(1), wr2 = o2 ? a.wr[2][i2 >> 1] : T(0);
    const int bn = o2 ? b + 1 : b;
    for (int x0 = 0; x0 < f0; ++x0) {
      const bool o0 = x0 & 1;
      const int64_t i0 = 2 * qa0 + x0;
      const T w0l = o0 ? a.wl[0][i0 >> 1] : T(1), w0r = o0 ? a.wr[0][i0 >> 1] : T(0);
      const T* pA = cs + (x0 >> 1) * S1 * S2;
      const T* pB = o0 ? pA + S1 * S2 : pA;
      // interpolant of the even fine row 2*q1 (dims 0 and 2)
      auto reven = [&](int q1) {
        const T vb = w0l * pA[q1 * S2 + b] + w0r * pB[q1 * S2 + b];
        const T vn = w0l * pA[q1 * S2 + bn] + w0r * pB[q1 * S2 + bn];
        return wl2 * vb + wr2 * vn;
      };
      const int64_t rowbase = (i0 * e1 + 2 * qa1) * e2 + i2;
      T rcur = reven(0);
#pragma unroll 4
      for (int x1 = 0; x1 < f1; x1 += 2) {
        const int64_t g0 = rowbase + int64_t(x1) * e2;
        const bool has_odd = x1 + 1 < f1;
        T cf0 = T(0), cf1 = T(0);
        if (with) {
          cf0 = coef[g0];
          if (has_odd) cf1 = coef[g0 + e2];
        }
        const bool coarse = !(o0 | o2);  // even row x1: coarse node iff x0, x2 even
        out[g0] = coarse ? rcur : cf0 + rcur;
        if (has_odd) {
          const int64_t i1 = 2 * qa1 + x1 + 1;
          const T rnext = reven((x1 >> 1) + 1);
          const T ip = a.wl[1][i1 >> 1] * rcur + a.wr[1][i1 >> 1] * rnext;
          out[g0 + e2] = cf1 + ip;
          rcur = rnext;
        }
      }
    }
  }
}

}  // namespace

template <class T>
bool launch_interp_rec(const T* coef, T* out, const T* C, const T* Z, const LevelArgs<T>& a,
                       bool with, cudaStream_t s) {
  constexpr int B0 = 2, B1 = 16, B2 = 128;
  const int64_t m0 = a.c[0] - 1, m1 = a.c[1] - 1, m2 = a.c[2] - 1;
  const int nb0 = int(std::max<int64_t>(1, (m0 + B0 - 1) / B0));
  const int nb1 = int(std::max<int64_t>(1, (m1 + B1 - 1) / B1));
  const int nb2 = int(std::max<int64_t>(1, (m2 + B2 - 1) / B2));
  const size_t smem = size_t(B0 + 1) * (B1 + 1) * (B2 + 2) * sizeof(T);
  static int attr_dev = -1;
  int dev = 0;
  HGR_CUDA_CHECK(cudaGetDevice(&dev));
  if (attr_dev != dev) {
    HGR_CUDA_CHECK(cudaFuncSetAttribute(k_interp_rec<T, B0, B1, B2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr_dev = dev;
  }
  k_interp_rec<T, B0, B1, B2><<<unsigned(int64_t(nb0) * nb1 * nb2), 2 * B2, smem, s>>>(
      coef, out, C, Z, a, with, nb1, nb2);
  HGR_CUDA_CHECK(cudaGetLastError());
  return true;
}

template bool launch_interp_rec<float>(const float*, float*, const float*, const float*,
                                       const LevelArgs<float>&, bool, cudaStream_t);
template bool launch_interp_rec<double>(const double*, double*, const double*, const double*,
                                        const LevelArgs<double>&, bool, cudaStream_t);

}  // namespace hgrb
