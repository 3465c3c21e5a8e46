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
// The factor tables (identical for every line of a (level, dim)) live in
// shared memory.
//
//   dims 0/1 (strided lines): persistent CTAs; a group = 32 consecutive lines
//     along the contiguous dim (lanes) x the whole line (warps own chunks).
//     The next group is prefetched by cp.async into shared memory while the
//     current one is solved; carries combine through shared memory.
//   dim 2 (contiguous rows): one warp per row, lanes own chunks; rows are
//     double-buffered in shared memory by cp.async; carries by warp shuffles.
#include "kernels_fused.cuh"
#include "plan.hpp"
#include "ptx.cuh"

namespace hgrb {

namespace {

template <class T>
__device__ __forceinline__ T shfl_up(T v, int d) {
  return __shfl_up_sync(0xffffffffu, v, d);
}
template <class T>
__device__ __forceinline__ T shfl_down(T v, int d) {
  return __shfl_down_sync(0xffffffffu, v, d);
}

// tables: tm[i] = mult[i] (i < n-1), tr[i] = 1/pivot[i], tu[i] = upper[i] (i < n-1)
template <class T>
__device__ __forceinline__ void load_tables(T* tm, T* tr, T* tu, const T* mult, const T* rpiv,
                                            const T* upper, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    tr[i] = rpiv[i];
    tm[i] = i + 1 < n ? mult[i] : T(0);
    tu[i] = i + 1 < n ? upper[i] : T(0);
  }
}

// forward pass of chunk [s0, s0+cnt): local result (zero carry) + carry coefficient
template <class T, int CH>
__device__ __forceinline__ void fwd_local(const T (&x)[CH], int s0, int cnt, const T* tm, T& g,
                                          T& A) {
  g = T(0);
  A = T(1);
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    if (k < cnt) {
      const int i = s0 + k;
      if (i == 0) {
        g = x[k];
      } else {
        const T m = tm[i - 1];
        g = x[k] - m * g;
        A *= -m;
      }
    }
  }
}

template <class T, int CH>
__device__ __forceinline__ void fwd_apply(T (&x)[CH], int s0, int cnt, const T* tm, T carry) {
  T prev = carry;
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    if (k < cnt) {
      const int i = s0 + k;
      if (i > 0) x[k] = x[k] - tm[i - 1] * prev;
      prev = x[k];
    }
  }
}

template <class T, int CH>
__device__ __forceinline__ void bwd_local(const T (&x)[CH], int s0, int cnt, int n, const T* tr,
                                          const T* tu, T& h, T& B) {
  h = T(0);
  B = T(1);
#pragma unroll
  for (int k = CH - 1; k >= 0; --k) {
    if (k < cnt) {
      const int i = s0 + k;
      const T rp = tr[i];
      if (i == n - 1) {
        h = x[k] * rp;
      } else {
        const T u = tu[i];
        h = (x[k] - u * h) * rp;
        B *= -u * rp;
      }
    }
  }
}

template <class T, int CH>
__device__ __forceinline__ void bwd_apply(T (&x)[CH], int s0, int cnt, int n, const T* tr,
                                          const T* tu, T carry) {
  T next = carry;
#pragma unroll
  for (int k = CH - 1; k >= 0; --k) {
    if (k < cnt) {
      const int i = s0 + k;
      x[k] = (i == n - 1) ? x[k] * tr[i] : (x[k] - tu[i] * next) * tr[i];
      next = x[k];
    }
  }
}

// ---- strided lines (dims 0 / 1) ---------------------------------------------------

template <class T, int CH, int W>
__global__ void __launch_bounds__(32 * W, 1)
    k_thomas_strided(const T* in, T* out, int64_t e0, int64_t e1, int64_t e2, int dim,
                     const T* __restrict__ mult, const T* __restrict__ rpiv,
                     const T* __restrict__ upper, int64_t ngroups) {
  constexpr int NT = 32 * W, NMAX = W * CH;
  extern __shared__ __align__(16) unsigned char smem_t[];
  T* buf = reinterpret_cast<T*>(smem_t);          // [NMAX][32]
  T* tm = buf + NMAX * 32;
  T* tr = tm + NMAX;
  T* tu = tr + NMAX;
  T* sg = tu + NMAX;                               // [W][32]
  T* sa = sg + W * 32;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int n = int(dim == 0 ? e0 : e1);
  const int64_t sd = dim == 0 ? e1 * e2 : e2;
  const int64_t so = dim == 0 ? e2 : e1 * e2;  // stride of the other strided dim
  const int64_t nblk2 = (e2 + 31) / 32;
  load_tables(tm, tr, tu, mult, rpiv, upper, n);
  const int s0 = w * CH;
  int cnt = n - s0;
  cnt = cnt < 0 ? 0 : (cnt > CH ? CH : cnt);

  auto group_base = [&](int64_t g, int& nl) {
    const int64_t ia = g / nblk2, i2 = (g % nblk2) * 32;
    nl = int(e2 - i2 < 32 ? e2 - i2 : 32);
    return ia * so + i2;
  };
  auto prefetch = [&](int64_t g) {
    int nl;
    const int64_t base = group_base(g, nl);
    for (int idx = tid; idx < n * 32; idx += NT) {
      const int i = idx >> 5, q = idx & 31;
      const bool ok = q < nl;
      ptx::cp_async_elem<int(sizeof(T))>(buf + idx, in + base + i * sd + (ok ? q : 0),
                                         ok ? int(sizeof(T)) : 0);
    }
    ptx::cp_async_commit();
  };

  int64_t g = blockIdx.x;
  if (g < ngroups) prefetch(g);
  for (; g < ngroups; g += gridDim.x) {
    ptx::cp_async_wait_all();
    __syncthreads();
    T x[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k)
      if (k < cnt) x[k] = buf[(s0 + k) * 32 + lane];
    __syncthreads();
    if (g + gridDim.x < ngroups) prefetch(g + gridDim.x);

    T gl, A;
    fwd_local<T, CH>(x, s0, cnt, tm, gl, A);
    sg[w * 32 + lane] = gl;
    sa[w * 32 + lane] = A;
    __syncthreads();
    T carry = T(0);
    for (int v = 0; v < w; ++v) carry = sg[v * 32 + lane] + sa[v * 32 + lane] * carry;
    fwd_apply<T, CH>(x, s0, cnt, tm, carry);
    T h, B;
    bwd_local<T, CH>(x, s0, cnt, n, tr, tu, h, B);
    __syncthreads();
    sg[w * 32 + lane] = h;
    sa[w * 32 + lane] = B;
    __syncthreads();
    carry = T(0);
    for (int v = W - 1; v > w; --v) carry = sg[v * 32 + lane] + sa[v * 32 + lane] * carry;
    bwd_apply<T, CH>(x, s0, cnt, n, tr, tu, carry);
    int nl;
    const int64_t base = group_base(g, nl);
    if (lane < nl) {
#pragma unroll
      for (int k = 0; k < CH; ++k)
        if (k < cnt) out[base + (s0 + k) * sd + lane] = x[k];
    }
  }
}

// ---- contiguous rows (dim 2) --------------------------------------------------------

template <class T, int CH>
__global__ void __launch_bounds__(256) k_thomas_rows(const T* in, T* out, int64_t rows, int n,
                                                     const T* __restrict__ mult,
                                                     const T* __restrict__ rpiv,
                                                     const T* __restrict__ upper) {
  constexpr int PITCH = 32 * CH + 1, NMAX = 32 * CH;
  extern __shared__ __align__(16) unsigned char smem_t[];
  T* tm = reinterpret_cast<T*>(smem_t);
  T* tr = tm + NMAX;
  T* tu = tr + NMAX;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T* bufs = tu + NMAX + warp * 2 * PITCH;
  load_tables(tm, tr, tu, mult, rpiv, upper, n);
  __syncthreads();
  const int s0 = lane * CH;
  int cnt = n - s0;
  cnt = cnt < 0 ? 0 : (cnt > CH ? CH : cnt);
  const int64_t stride = int64_t(gridDim.x) * 8;
  auto prefetch = [&](int64_t row, T* dst) {
    const T* src = in + row * n;
    for (int i = lane; i < n; i += 32)
      ptx::cp_async_elem<int(sizeof(T))>(dst + i, src + i, int(sizeof(T)));
  };
  int64_t row = int64_t(blockIdx.x) * 8 + warp;
  if (row < rows) prefetch(row, bufs);
  ptx::cp_async_commit();
  for (int it = 0; row < rows; row += stride, ++it) {
    T* cur = bufs + (it & 1) * PITCH;
    T* nxt = bufs + ((it + 1) & 1) * PITCH;
    if (row + stride < rows) prefetch(row + stride, nxt);
    ptx::cp_async_commit();
    ptx::cp_async_wait_group<1>();
    __syncwarp();
    T x[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k)
      if (k < cnt) x[k] = cur[s0 + k];
    T g, A;
    fwd_local<T, CH>(x, s0, cnt, tm, g, A);
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
    fwd_apply<T, CH>(x, s0, cnt, tm, carry);
    T h, B;
    bwd_local<T, CH>(x, s0, cnt, n, tr, tu, h, B);
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
    bwd_apply<T, CH>(x, s0, cnt, n, tr, tu, next);
#pragma unroll
    for (int k = 0; k < CH; ++k)
      if (k < cnt) cur[s0 + k] = x[k];
    __syncwarp();
    T* dst = out + row * n;
    for (int i = lane; i < n; i += 32) dst[i] = cur[i];
    __syncwarp();
  }
}

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

template <class T, int CH>
void run_rows(const T* in, T* out, int64_t rows, int64_t n, const T* mult, const T* rpiv,
              const T* upper, cudaStream_t s) {
  const size_t smem = size_t(3 * 32 * CH + 8 * 2 * (32 * CH + 1)) * sizeof(T);
  static int attr_dev = -1;
  int dev = 0;
  HGR_CUDA_CHECK(cudaGetDevice(&dev));
  if (attr_dev != dev) {
    HGR_CUDA_CHECK(cudaFuncSetAttribute(k_thomas_rows<T, CH>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr_dev = dev;
  }
  const int64_t want = (rows + 7) / 8;
  const int grid = int(want < int64_t(sm_count()) * 3 ? want : int64_t(sm_count()) * 3);
  k_thomas_rows<T, CH><<<grid, 256, smem, s>>>(in, out, rows, int(n), mult, rpiv, upper);
  HGR_CUDA_CHECK(cudaGetLastError());
}

template <class T, int CH>
void run_strided(const T* in, T* out, const int64_t e[3], int dim, const T* mult,
                 const T* rpiv, const T* upper, cudaStream_t s) {
  constexpr int W = 16;
  const size_t smem = size_t(W * CH * 32 + 3 * W * CH + 2 * W * 32) * sizeof(T);
  static int attr_dev = -1;
  int dev = 0;
  HGR_CUDA_CHECK(cudaGetDevice(&dev));
  if (attr_dev != dev) {
    HGR_CUDA_CHECK(cudaFuncSetAttribute(k_thomas_strided<T, CH, W>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr_dev = dev;
  }
  const int64_t na = dim == 0 ? e[1] : e[0];
  const int64_t groups = na * ((e[2] + 31) / 32);
  const int grid = int(groups < sm_count() ? groups : sm_count());
  k_thomas_strided<T, CH, W><<<grid, 32 * W, smem, s>>>(in, out, e[0], e[1], e[2], dim, mult,
                                                         rpiv, upper, groups);
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
