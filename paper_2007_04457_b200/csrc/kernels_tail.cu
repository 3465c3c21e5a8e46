// kernels_tail.cu -- the coarse tail of the hierarchy in one launch per direction.
//
// Levels below the fused-kernel threshold hold at most a few tens of thousands
// of nodes; run level by level as separate grids they cost a launch gap per
// step (about nine per level and direction). Here one CTA walks all of them,
// separating the steps with __syncthreads (global writes of a block are visible
// to the whole block after the barrier; the operands stay in L1 / L2):
//
//   decompose, levels lt .. 1 (refactor.hpp:41-54): coefficients of level l
//     (transforms.hpp:96-111, 0 at coarse nodes) and the coarse gather; the LPK
//     passes over the real dims in ascending order, masked on the first
//     (correction.hpp:238-260, :331); the Thomas passes (correction.hpp:202-208,
//     :262-278), the last one adding z to the coarse values (refactor.hpp:50-54).
//   recompose (refactor.hpp:63-90): levels min(m, lt) .. 1 compute their
//     correction from the stored coefficients and gather their coarse nodes;
//     then levels 1 .. lt interpolate in place (coarse -= z, refined = coef +
//     interp, or interp only above the prefix m).
//
// Every step is the one-thread-per-item formulation of kernels_basic.cu with a
// block-stride loop; the Thomas passes are the reference's sequential
// recurrence, one thread per line.
#include "kernels.cuh"
#include "kernels_fused.cuh"
#include "plan.hpp"

namespace hgrb {

namespace {

constexpr int kTailThreads = 512;

template <class T>
__device__ void tail_lpk(const T* __restrict__ in, const int (&e)[3], T* __restrict__ out,
                         int dim, int cd, const T* __restrict__ taps, bool mask) {
  int o[3] = {e[0], e[1], e[2]};
  o[dim] = cd;
  const int total = o[0] * o[1] * o[2];
  const int st[3] = {e[1] * e[2], e[2], 1};
  const int nd = e[dim];
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int x2 = idx % o[2], t = idx / o[2], x1 = t % o[1], x0 = t / o[1];
    const int x[3] = {x0, x1, x2};
    const int i = x[dim];
    bool other_even = true;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (d != dim && (x[d] & 1)) other_even = false;
    const bool zero_even = mask && other_even;
    int base = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (d != dim) base += x[d] * st[d];
    const int sd = st[dim];
    T acc = T(0);
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int j = 2 * i - 2 + k;
      if (j < 0 || j >= nd) continue;
      if (zero_even && (j & 1) == 0) continue;
      acc += taps[i * 5 + k] * in[base + j * sd];
    }
    out[idx] = acc;
  }
}

// one thread per line; apply != null: apply += sign * solution instead of storing it
template <class T>
__device__ void tail_thomas(T* z, const int (&e)[3], int dim, const T* __restrict__ mult,
                            const T* __restrict__ rpiv, const T* __restrict__ upper, T* apply,
                            int sign) {
  const int st[3] = {e[1] * e[2], e[2], 1};
  const int a = dim == 0 ? 1 : 0, b = dim == 2 ? 1 : 2;
  const int lines = e[a] * e[b];
  const int n = e[dim], sd = st[dim];
  for (int f = threadIdx.x; f < lines; f += blockDim.x) {
    const int ia = f / e[b], ib = f % e[b];
    T* x = z + ia * st[a] + ib * st[b];
    T prev = x[0];
    for (int i = 1; i < n; ++i) {
      prev = x[i * sd] - mult[i - 1] * prev;
      x[i * sd] = prev;
    }
    T next = prev * rpiv[n - 1];
    if (apply) {
      T* ap = apply + ia * st[a] + ib * st[b];
      ap[(n - 1) * sd] += sign > 0 ? next : -next;
      for (int i = n - 1; i-- > 0;) {
        next = (x[i * sd] - upper[i] * next) * rpiv[i];
        ap[i * sd] += sign > 0 ? next : -next;
      }
    } else {
      x[(n - 1) * sd] = next;
      for (int i = n - 1; i-- > 0;) {
        next = (x[i * sd] - upper[i] * next) * rpiv[i];
        x[i * sd] = next;
      }
    }
  }
}

// LPK passes (masked first) into z, then the Thomas passes (correction.hpp:295-340)
template <class T>
__device__ void tail_correction(const TailLevel<T>& L, int rank, const T* in, T* const (&stage)[2],
                                T* apply, int sign) {
  const LevelArgs<T>& a = L.a;
  int e[3] = {int(a.e[0]), int(a.e[1]), int(a.e[2])};
  const T* cur = in;
  int pass = 0;
  for (int k = 3 - rank; k < 3; ++k, ++pass) {
    T* dst = k == 2 ? L.z : stage[pass & 1];
    tail_lpk<T>(cur, e, dst, k, int(a.c[k]), a.taps[k], pass == 0);
    __syncthreads();
    e[k] = int(a.c[k]);
    cur = dst;
  }
  for (int k = 3 - rank; k < 3; ++k) {
    tail_thomas<T>(L.z, e, k, a.mult[k], a.rpiv[k], a.upper[k], k == 2 ? apply : nullptr, sign);
    __syncthreads();
  }
}

template <class T>
__global__ void __launch_bounds__(kTailThreads, 1)
    k_tail_decompose(const TailLevel<T>* __restrict__ levels, int lt, int rank, T* s0, T* s1) {
  T* const stage[2] = {s0, s1};
  for (int l = lt; l >= 1; --l) {
    const TailLevel<T>& L = levels[l];
    const LevelArgs<T>& a = L.a;
    const int e1 = int(a.e[1]), e2 = int(a.e[2]), n = int(a.e[0]) * e1 * e2;
    const int c1 = int(a.c[1]), c2 = int(a.c[2]);
    const T* U = L.src;
    auto coarse = [&](int64_t q0, int64_t q1, int64_t q2) {
      return U[((2 * q0) * e1 + 2 * q1) * e2 + 2 * q2];
    };
    for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
      const int i2 = idx % e2, t = idx / e2, i1 = t % e1, i0 = t / e1;
      if (((i0 | i1 | i2) & 1) == 0) {
        L.coarse[((i0 >> 1) * c1 + (i1 >> 1)) * c2 + (i2 >> 1)] = U[idx];
        L.coef[idx] = T(0);
      } else {
        L.coef[idx] = U[idx] - interp_node(a, i0, i1, i2, coarse);
      }
    }
    __syncthreads();
    tail_correction<T>(L, rank, L.coef, stage, L.coarse, +1);
  }
}

template <class T>
__global__ void __launch_bounds__(kTailThreads, 1)
    k_tail_recompose(const TailLevel<T>* __restrict__ levels, int lt, int m, int rank, T* s0,
                     T* s1) {
  T* const stage[2] = {s0, s1};
  for (int l = m < lt ? m : lt; l >= 1; --l) {
    const TailLevel<T>& L = levels[l];
    const LevelArgs<T>& a = L.a;
    // coarse nodes of the stored level into C_{l-1} (read only below, no barrier needed)
    const int c0 = int(a.c[0]), c1 = int(a.c[1]), c2 = int(a.c[2]);
    const int e1 = int(a.e[1]), e2 = int(a.e[2]);
    for (int q = threadIdx.x; q < c0 * c1 * c2; q += blockDim.x) {
      const int q2 = q % c2, t = q / c2, q1 = t % c1, q0 = t / c1;
      L.coarse[q] = L.src[((2 * q0) * e1 + 2 * q1) * e2 + 2 * q2];
    }
    tail_correction<T>(L, rank, L.src, stage, nullptr, 0);
  }
  for (int l = 1; l <= lt; ++l) {
    const TailLevel<T>& L = levels[l];
    const LevelArgs<T>& a = L.a;
    const bool with = l <= m;
    const T* Z = with ? L.z : nullptr;
    const int e1 = int(a.e[1]), e2 = int(a.e[2]), n = int(a.e[0]) * e1 * e2;
    const int c1 = int(a.c[1]), c2 = int(a.c[2]);
    const T* C = L.coarse;
    auto coarse = [&](int64_t q0, int64_t q1, int64_t q2) {
      const int64_t q = (q0 * c1 + q1) * c2 + q2;
      return Z ? C[q] - Z[q] : C[q];
    };
    T* out = L.src;  // in place: every cell reads only its own coefficient
    for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
      const int i2 = idx % e2, t = idx / e2, i1 = t % e1, i0 = t / e1;
      if (((i0 | i1 | i2) & 1) == 0) {
        out[idx] = coarse(i0 >> 1, i1 >> 1, i2 >> 1);
      } else {
        const T ip = interp_node(a, i0, i1, i2, coarse);
        out[idx] = with ? out[idx] + ip : ip;
      }
    }
    __syncthreads();
  }
}

}  // namespace

template <class T>
void launch_tail_decompose(const TailLevel<T>* d_levels, int lt, int rank, T* s0, T* s1,
                           cudaStream_t s) {
  k_tail_decompose<T><<<1, kTailThreads, 0, s>>>(d_levels, lt, rank, s0, s1);
  HGR_CUDA_CHECK(cudaGetLastError());
}

template <class T>
void launch_tail_recompose(const TailLevel<T>* d_levels, int lt, int m, int rank, T* s0, T* s1,
                           cudaStream_t s) {
  k_tail_recompose<T><<<1, kTailThreads, 0, s>>>(d_levels, lt, m, rank, s0, s1);
  HGR_CUDA_CHECK(cudaGetLastError());
}

template void launch_tail_decompose<float>(const TailLevel<float>*, int, int, float*, float*,
                                           cudaStream_t);
template void launch_tail_decompose<double>(const TailLevel<double>*, int, int, double*, double*,
                                            cudaStream_t);
template void launch_tail_recompose<float>(const TailLevel<float>*, int, int, int, float*, float*,
                                           cudaStream_t);
template void launch_tail_recompose<double>(const TailLevel<double>*, int, int, int, double*,
                                            double*, cudaStream_t);

}  // namespace hgrb
