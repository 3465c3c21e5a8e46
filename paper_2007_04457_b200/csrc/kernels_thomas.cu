// kernels_thomas.cu -- IPK: batched Thomas solves of the mass matrix
// (ThomasSolver::solve_fiber, correction.hpp:202-208; thomas_pass :262-278).
//
// Forward elimination f_i = x_i - m_{i-1} f_{i-1} and back substitution
// y_i = (f_i - u_i y_{i+1}) / p_i are first-order affine recurrences. A line is
// cut into chunks held in registers; each chunk computes its local result with
// a zero carry plus the product of its recurrence coefficients, the chunk
// carries are combined by an exact affine scan, and every chunk then re-runs
// the reference recurrence from its true carry. One HBM read and one write per
// element per dimension; no second pass over the forward-eliminated values.
//
//   dims 0/1 (strided lines): lanes = 32 consecutive lines along the contiguous
//     dim (coalesced rows), warps = chunks of the line; carries through smem.
//   dim 2 (contiguous rows): one warp per row, lanes = chunks; the row is staged
//     through shared memory for coalescing, carries by warp-shuffle scan.
#include "kernels_fused.cuh"
#include "plan.hpp"

namespace hgrb {

namespace {

template <class T, int CH, int W>
__global__ void __launch_bounds__(32 * W) k_thomas_strided(const T* in, T* out, int64_t e0,
                                                           int64_t e1, int64_t e2, int dim,
                                                           const T* __restrict__ mult,
                                                           const T* __restrict__ rpiv,
                                                           const T* __restrict__ upper) {
  __shared__ T s_g[W][32];
  __shared__ T s_a[W][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t n = dim == 0 ? e0 : e1;
  const int64_t sd = dim == 0 ? e1 * e2 : e2;
  const int64_t sa = dim == 0 ? e2 : e1 * e2;  // stride of the other strided dim
  const int64_t nblk2 = (e2 + 31) / 32;
  const int64_t ia = blockIdx.x / nblk2;
  const int64_t i2 = (blockIdx.x % nblk2) * 32 + lane;
  const bool live = i2 < e2;
  const int64_t base = ia * sa + i2;
  const int64_t s0 = int64_t(w) * CH;
  int cnt = int(n - s0);
  cnt = cnt < 0 ? 0 : (cnt > CH ? CH : cnt);

  T x[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k)
    if (k < cnt && live) x[k] = in[base + (s0 + k) * sd];

  // forward, local (zero carry): g and the carry coefficient A = prod(-m)
  T g = T(0), A = T(1);
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    if (k < cnt) {
      const int64_t i = s0 + k;
      if (i == 0) {
        g = x[k];
      } else {
        const T m = mult[i - 1];
        g = x[k] - m * g;
        A *= -m;
      }
    }
  }
  s_g[w][lane] = g;
  s_a[w][lane] = A;
  __syncthreads();
  T carry = T(0);
  for (int v = 0; v < w; ++v) carry = s_g[v][lane] + s_a[v][lane] * carry;
  T prev = carry;
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    if (k < cnt) {
      const int64_t i = s0 + k;
      if (i > 0) x[k] = x[k] - mult[i - 1] * prev;
      prev = x[k];
    }
  }
  // backward, local: h and B = prod(-u*rp)
  T h = T(0), B = T(1);
#pragma unroll
  for (int k = CH - 1; k >= 0; --k) {
    if (k < cnt) {
      const int64_t i = s0 + k;
      const T rp = rpiv[i];
      if (i == n - 1) {
        h = x[k] * rp;
      } else {
        const T u = upper[i];
        h = (x[k] - u * h) * rp;
        B *= -u * rp;
      }
    }
  }
  __syncthreads();
  s_g[w][lane] = h;
  s_a[w][lane] = B;
  __syncthreads();
  carry = T(0);
  for (int v = W - 1; v > w; --v) carry = s_g[v][lane] + s_a[v][lane] * carry;
  T next = carry;
#pragma unroll
  for (int k = CH - 1; k >= 0; --k) {
    if (k < cnt) {
      const int64_t i = s0 + k;
      x[k] = (i == n - 1) ? x[k] * rpiv[i] : (x[k] - upper[i] * next) * rpiv[i];
      next = x[k];
    }
  }
#pragma unroll
  for (int k = 0; k < CH; ++k)
    if (k < cnt && live) out[base + (s0 + k) * sd] = x[k];
}

template <class T>
__device__ __forceinline__ T shfl_up(T v, int d) {
  return __shfl_up_sync(0xffffffffu, v, d);
}
template <class T>
__device__ __forceinline__ T shfl_down(T v, int d) {
  return __shfl_down_sync(0xffffffffu, v, d);
}

template <class T, int CH>
__global__ void __launch_bounds__(256) k_thomas_rows(const T* in, T* out, int64_t rows,
                                                     int64_t n, const T* __restrict__ mult,
                                                     const T* __restrict__ rpiv,
                                                     const T* __restrict__ upper) {
  constexpr int PITCH = 32 * CH + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* buf = reinterpret_cast<T*>(smem_raw) + (threadIdx.x >> 5) * PITCH;
  const int lane = threadIdx.x & 31;
  const int64_t warps_total = int64_t(gridDim.x) * 8;
  const int s0 = lane * CH;
  int cnt = int(n) - s0;
  cnt = cnt < 0 ? 0 : (cnt > CH ? CH : cnt);
  for (int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5); row < rows; row += warps_total) {
    const T* src = in + row * n;
    for (int64_t i = lane; i < n; i += 32) buf[i] = src[i];
    __syncwarp();
    T x[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k)
      if (k < cnt) x[k] = buf[s0 + k];
    // forward local
    T g = T(0), A = T(1);
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      if (k < cnt) {
        const int i = s0 + k;
        if (i == 0) {
          g = x[k];
        } else {
          const T m = mult[i - 1];
          g = x[k] - m * g;
          A *= -m;
        }
      }
    }
    // inclusive affine scan over lanes: F_t = G_t + A_t F_{t-1}
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const T gp = shfl_up(g, d), ap = shfl_up(A, d);
      if (lane >= d) {
        g = g + A * gp;
        A = A * ap;
      }
    }
    T carry = shfl_up(g, 1);
    if (lane == 0) carry = T(0);
    T prev = carry;
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      if (k < cnt) {
        const int i = s0 + k;
        if (i > 0) x[k] = x[k] - mult[i - 1] * prev;
        prev = x[k];
      }
    }
    // backward local
    T h = T(0), B = T(1);
#pragma unroll
    for (int k = CH - 1; k >= 0; --k) {
      if (k < cnt) {
        const int i = s0 + k;
        const T rp = rpiv[i];
        if (i == n - 1) {
          h = x[k] * rp;
        } else {
          const T u = upper[i];
          h = (x[k] - u * h) * rp;
          B *= -u * rp;
        }
      }
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const T hn = shfl_down(h, d), bn = shfl_down(B, d);
      if (lane + d < 32) {
        h = h + B * hn;
        B = B * bn;
      }
    }
    T next = shfl_down(h, 1);
    if (lane == 31) next = T(0);
#pragma unroll
    for (int k = CH - 1; k >= 0; --k) {
      if (k < cnt) {
        const int i = s0 + k;
        x[k] = (i == n - 1) ? x[k] * rpiv[i] : (x[k] - upper[i] * next) * rpiv[i];
        next = x[k];
      }
    }
#pragma unroll
    for (int k = 0; k < CH; ++k)
      if (k < cnt) buf[s0 + k] = x[k];
    __syncwarp();
    T* dst = out + row * n;
    for (int64_t i = lane; i < n; i += 32) dst[i] = buf[i];
    __syncwarp();
  }
}

template <class T, int CH>
void run_rows(const T* in, T* out, int64_t rows, int64_t n, const T* mult, const T* rpiv,
              const T* upper, cudaStream_t s) {
  const size_t smem = size_t(8) * (32 * CH + 1) * sizeof(T);
  static bool attr = false;
  if (!attr) {
    HGR_CUDA_CHECK(cudaFuncSetAttribute(k_thomas_rows<T, CH>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  const int grid = grid_for(rows * 32, 256, 8);
  k_thomas_rows<T, CH><<<grid, 256, smem, s>>>(in, out, rows, n, mult, rpiv, upper);
  HGR_CUDA_CHECK(cudaGetLastError());
}

template <class T, int CH>
void run_strided(const T* in, T* out, const int64_t e[3], int dim, const T* mult,
                 const T* rpiv, const T* upper, cudaStream_t s) {
  constexpr int W = 16;
  const int64_t na = dim == 0 ? e[1] : e[0];
  const int64_t blocks = na * ((e[2] + 31) / 32);
  k_thomas_strided<T, CH, W><<<unsigned(blocks), 32 * W, 0, s>>>(in, out, e[0], e[1], e[2], dim,
                                                                  mult, rpiv, upper);
  HGR_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

template <class T>
bool launch_thomas_fast(const T* in, T* out, const int64_t e[3], int dim, const T* mult,
                        const T* rpiv, const T* upper, cudaStream_t s) {
  const int64_t n = e[dim];
  if (dim == 2) {
    const int64_t rows = e[0] * e[1];
    if (n <= 32 * 2) run_rows<T, 2>(in, out, rows, n, mult, rpiv, upper, s);
    else if (n <= 32 * 5) run_rows<T, 5>(in, out, rows, n, mult, rpiv, upper, s);
    else if (n <= 32 * 9) run_rows<T, 9>(in, out, rows, n, mult, rpiv, upper, s);
    else if (n <= 32 * 17) run_rows<T, 17>(in, out, rows, n, mult, rpiv, upper, s);
    else if (n <= 32 * 33) run_rows<T, 33>(in, out, rows, n, mult, rpiv, upper, s);
    else return false;
    return true;
  }
  if (n <= 16 * 2) run_strided<T, 2>(in, out, e, dim, mult, rpiv, upper, s);
  else if (n <= 16 * 5) run_strided<T, 5>(in, out, e, dim, mult, rpiv, upper, s);
  else if (n <= 16 * 9) run_strided<T, 9>(in, out, e, dim, mult, rpiv, upper, s);
  else if (n <= 16 * 17) run_strided<T, 17>(in, out, e, dim, mult, rpiv, upper, s);
  else if (n <= 16 * 33) run_strided<T, 33>(in, out, e, dim, mult, rpiv, upper, s);
  else return false;
  return true;
}

template bool launch_thomas_fast<float>(const float*, float*, const int64_t*, int, const float*,
                                        const float*, const float*, cudaStream_t);
template bool launch_thomas_fast<double>(const double*, double*, const int64_t*, int,
                                         const double*, const double*, const double*,
                                         cudaStream_t);

}  // namespace hgrb
