// kernels_basic.cu -- straightforward sm_100a kernels: one thread per node /
// output / line. They define the GPU semantics of every step of the hot path
// and serve the coarse levels and the single-level API; the fine levels use
// the fused kernels in kernels_fused.cu / kernels_thomas.cu.
#include <algorithm>
#include <cstdio>
#include <type_traits>
#include <mutex>
#include <vector>

#include "kernels.cuh"
#include "launch.cuh"
#include "ptx.cuh"
#include "plan.hpp"

namespace hgrb {

[[noreturn]] void throw_cuda(cudaError_t e, const char* expr, const char* file, int line) {
  cudaGetLastError();  // reported here; a non-sticky error must not resurface in a later check
  char buf[512];
  std::snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
                cudaGetErrorString(e), file, line, expr);
  throw Error(HGR_ERR_CUDA, buf);
}

void set_smem_attr(const void* fn, size_t bytes) {
  struct Set {
    int dev;
    const void* fn;
    size_t bytes;
  };
  static std::mutex mu;
  static std::vector<Set> done;
  int dev = 0;
  HGR_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  for (auto& d : done)
    if (d.dev == dev && d.fn == fn) {
      if (d.bytes >= bytes) return;
      HGR_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
      d.bytes = bytes;
      return;
    }
  HGR_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
  done.push_back(Set{dev, fn, bytes});
}

[[noreturn]] void launch_failed(cudaError_t e, const void* kern, dim3 grid, dim3 block, size_t smem) {
  cudaGetLastError();  // a failed launch is not sticky: do not let it leak into later checks
  const char* name = nullptr;
  if (cudaFuncGetName(&name, kern) != cudaSuccess || !name) name = "?";
  char buf[768];
  std::snprintf(buf, sizeof buf, "CUDA error %s (%s) launching %s grid (%u,%u,%u) block (%u,%u,%u) smem %zu",
                cudaGetErrorName(e), cudaGetErrorString(e), name, grid.x, grid.y, grid.z, block.x,
                block.y, block.z, smem);
  throw Error(HGR_ERR_CUDA, buf);
}

int grid_for(int64_t work, int threads, int blocks_per_sm) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  int64_t need = ceil_div(work, threads);
  int64_t cap = int64_t(sms) * blocks_per_sm;
  if (need < 1) need = 1;
  return int(need < cap ? need : cap);
}

#define GRID_STRIDE(i, n) \
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < (n); i += int64_t(gridDim.x) * blockDim.x)

// ---- GPK ---------------------------------------------------------------------

template <class T>
__global__ void __launch_bounds__(256) k_gpk_dec(T* __restrict__ U, T* __restrict__ C,
                                                 LevelArgs<T> a, int* flag, bool check) {
  const int64_t e1 = a.e[1], e2 = a.e[2], n = a.e[0] * e1 * e2;
  const int64_t c1 = a.c[1], c2 = a.c[2];
  auto coarse = [&](int64_t q0, int64_t q1, int64_t q2) {
    return U[((2 * q0) * e1 + 2 * q1) * e2 + 2 * q2];
  };
  bool bad = false;
  GRID_STRIDE(idx, n) {
    const int64_t i2 = idx % e2, t = idx / e2, i1 = t % e1, i0 = t / e1;
    const T u = U[idx];
    if (check && !isfinite(u)) bad = true;
    if (((i0 | i1 | i2) & 1) == 0) {
      C[((i0 >> 1) * c1 + (i1 >> 1)) * c2 + (i2 >> 1)] = u;
    } else {
      U[idx] = u - interp_node(a, i0, i1, i2, coarse);
    }
  }
  if (check && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

template <class T>
__global__ void __launch_bounds__(256) k_gpk_rec(const T* __restrict__ coef, T* out,
                                                 const T* __restrict__ C,
                                                 const T* __restrict__ Z, LevelArgs<T> a,
                                                 bool with) {
  const int64_t e1 = a.e[1], e2 = a.e[2], n = a.e[0] * e1 * e2;
  const int64_t c1 = a.c[1], c2 = a.c[2];
  auto coarse = [&](int64_t q0, int64_t q1, int64_t q2) {
    const int64_t q = (q0 * c1 + q1) * c2 + q2;
    return Z ? C[q] - Z[q] : C[q];
  };
  GRID_STRIDE(idx, n) {
    const int64_t i2 = idx % e2, t = idx / e2, i1 = t % e1, i0 = t / e1;
    if (((i0 | i1 | i2) & 1) == 0) {
      out[idx] = coarse(i0 >> 1, i1 >> 1, i2 >> 1);
    } else {
      const T ip = interp_node(a, i0, i1, i2, coarse);
      out[idx] = with ? coef[idx] + ip : ip;
    }
  }
}

template <class T>
__global__ void k_coefficients(const T* __restrict__ fine, T* __restrict__ out, LevelArgs<T> a) {
  const int64_t e1 = a.e[1], e2 = a.e[2], n = a.e[0] * e1 * e2;
  auto coarse = [&](int64_t q0, int64_t q1, int64_t q2) {
    return fine[((2 * q0) * e1 + 2 * q1) * e2 + 2 * q2];
  };
  GRID_STRIDE(idx, n) {
    const int64_t i2 = idx % e2, t = idx / e2, i1 = t % e1, i0 = t / e1;
    out[idx] = (((i0 | i1 | i2) & 1) == 0) ? T(0) : fine[idx] - interp_node(a, i0, i1, i2, coarse);
  }
}

template <class T>
__global__ void k_interpolate(const T* __restrict__ C, T* __restrict__ out, LevelArgs<T> a) {
  const int64_t e1 = a.e[1], e2 = a.e[2], n = a.e[0] * e1 * e2;
  const int64_t c1 = a.c[1], c2 = a.c[2];
  auto coarse = [&](int64_t q0, int64_t q1, int64_t q2) { return C[(q0 * c1 + q1) * c2 + q2]; };
  GRID_STRIDE(idx, n) {
    const int64_t i2 = idx % e2, t = idx / e2, i1 = t % e1, i0 = t / e1;
    out[idx] = (((i0 | i1 | i2) & 1) == 0) ? coarse(i0 >> 1, i1 >> 1, i2 >> 1)
                                           : interp_node(a, i0, i1, i2, coarse);
  }
}

template <class T>
__global__ void k_check_coarse_zero(const T* __restrict__ v, LevelArgs<T> a, int* flag) {
  const int64_t c1 = a.c[1], c2 = a.c[2], n = a.c[0] * c1 * c2;
  const int64_t e1 = a.e[1], e2 = a.e[2];
  GRID_STRIDE(q, n) {
    const int64_t q2 = q % c2, t = q / c2, q1 = t % c1, q0 = t / c1;
    if (v[((2 * q0) * e1 + 2 * q1) * e2 + 2 * q2] != T(0)) atomicOr(flag, 1);
  }
}

template <class T>
__global__ void k_check_finite(const T* __restrict__ v, int64_t n, int* flag) {
  bool bad = false;
  GRID_STRIDE(i, n) if (!isfinite(v[i])) bad = true;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// ---- LPK: one thread per output (correction.hpp:141-154, :238-260) -------------

template <class T>
__global__ void __launch_bounds__(256) k_lpk(const T* __restrict__ in, T* __restrict__ out,
                                             int64_t n0, int64_t n1, int64_t n2, int dim,
                                             int64_t cd, const T* __restrict__ taps, bool mask) {
  int64_t o[3] = {n0, n1, n2};
  o[dim] = cd;
  const int64_t total = o[0] * o[1] * o[2];
  const int64_t st[3] = {n1 * n2, n2, 1};
  const int64_t nd = dim == 0 ? n0 : (dim == 1 ? n1 : n2);
  GRID_STRIDE(idx, total) {
    const int64_t x2 = idx % o[2], t = idx / o[2], x1 = t % o[1], x0 = t / o[1];
    const int64_t x[3] = {x0, x1, x2};
    const int64_t i = x[dim];
    bool other_even = true;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (d != dim && (x[d] & 1)) other_even = false;
    const bool zero_even = mask && other_even;
    int64_t base = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      if (d != dim) base += x[d] * st[d];
    const int64_t sd = st[dim];
    T acc = T(0);
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const int64_t j = 2 * i - 2 + k;
      if (j < 0 || j >= nd) continue;
      if (zero_even && (j & 1) == 0) continue;
      acc += taps[i * 5 + k] * in[base + j * sd];
    }
    out[idx] = acc;
  }
}

// ---- IPK: one thread per line (correction.hpp:202-208, :262-278) ---------------

template <class T>
__global__ void __launch_bounds__(128) k_thomas(T* z, int64_t n0, int64_t n1, int64_t n2,
                                                int dim, const T* __restrict__ mult,
                                                const T* __restrict__ rpiv,
                                                const T* __restrict__ upper, T* apply,
                                                int sign) {
  const int64_t ext[3] = {n0, n1, n2};
  const int64_t st[3] = {n1 * n2, n2, 1};
  const int a = dim == 0 ? 1 : 0, b = dim == 2 ? 1 : 2;
  const int64_t lines = ext[a] * ext[b];
  const int64_t n = ext[dim], sd = st[dim];
  GRID_STRIDE(f, lines) {
    const int64_t ia = f / ext[b], ib = f % ext[b];
    T* x = z + ia * st[a] + ib * st[b];
    T prev = x[0];
    for (int64_t i = 1; i < n; ++i) {
      prev = x[i * sd] - mult[i - 1] * prev;
      x[i * sd] = prev;
    }
    T next = prev * rpiv[n - 1];
    if (apply) {
      T* ap = apply + ia * st[a] + ib * st[b];
      ap[(n - 1) * sd] += sign > 0 ? next : -next;
      for (int64_t i = n - 1; i-- > 0;) {
        next = (x[i * sd] - upper[i] * next) * rpiv[i];
        ap[i * sd] += sign > 0 ? next : -next;
      }
    } else {
      x[(n - 1) * sd] = next;
      for (int64_t i = n - 1; i-- > 0;) {
        next = (x[i * sd] - upper[i] * next) * rpiv[i];
        x[i * sd] = next;
      }
    }
  }
}

// ---- gathers / scatters ------------------------------------------------------

// Row-wise gathers / scatters: a warp per segment of up to kRowSeg elements of a
// row of the compact array (one index division per segment, consecutive lanes
// on consecutive elements; long rows -- 1D grids -- spread over many warps).
constexpr int64_t kRowSeg = 1024;

template <class T>
__global__ void __launch_bounds__(256) k_gather(const T* __restrict__ src, int64_t s1, int64_t s2,
                                                int64_t stride, T* __restrict__ dst, int64_t d0,
                                                int64_t d1, int64_t d2) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int64_t nseg = (d2 + kRowSeg - 1) / kRowSeg, items = d0 * d1 * nseg;
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t it = int64_t(blockIdx.x) * wpb + (threadIdx.x >> 5); it < items;
       it += int64_t(gridDim.x) * wpb) {
    const int64_t row = it / nseg, seg = it - row * nseg;
    const int64_t q0 = row / d1, q1 = row - q0 * d1;
    const T* sr = src + ((q0 * stride) * s1 + q1 * stride) * s2;
    T* dr = dst + row * d2;
    const int64_t hi = (seg + 1) * kRowSeg < d2 ? (seg + 1) * kRowSeg : d2;
    for (int64_t q2 = seg * kRowSeg + lane; q2 < hi; q2 += 32) dr[q2] = sr[q2 * stride];
  }
}

template <class T>
__global__ void __launch_bounds__(256) k_scatter_even(const T* __restrict__ src, T* __restrict__ dst,
                                                      LevelArgs<T> a) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int64_t c1 = a.c[1], c2 = a.c[2];
  const int64_t nseg = (c2 + kRowSeg - 1) / kRowSeg, items = a.c[0] * c1 * nseg;
  const int64_t e1 = a.e[1], e2 = a.e[2];
  const int lane = threadIdx.x & 31;
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t it = int64_t(blockIdx.x) * wpb + (threadIdx.x >> 5); it < items;
       it += int64_t(gridDim.x) * wpb) {
    const int64_t row = it / nseg, seg = it - row * nseg;
    const int64_t q0 = row / c1, q1 = row - q0 * c1;
    const T* sr = src + row * c2;
    T* dr = dst + ((2 * q0) * e1 + 2 * q1) * e2;
    const int64_t hi = (seg + 1) * kRowSeg < c2 ? (seg + 1) * kRowSeg : c2;
    for (int64_t q2 = seg * kRowSeg + lane; q2 < hi; q2 += 32) dr[2 * q2] = sr[q2];
  }
}

// Even rows of even planes of a level decomposed with side rows, written whole:
// even columns from the compact coarser pyramid, odd columns from the side rows.
// Persistent CTAs stream rows through an NST-stage ring: the coarse row and the
// side row arrive as bulk copies (their 16-byte aligned supersets), every thread
// assembles one aligned 16-byte output vector from shared memory and stores it
// -- full-sector writes instead of the strided scatter's read-modify-writes.
constexpr int kMergeStages = 3, kMergeRows = 4;  // ring stages x rows per stage
template <class T>
struct MergeCfg {
  static constexpr int V = 16 / int(sizeof(T));
  static __host__ __device__ int64_t row_elems(int64_t c2) { return (c2 + 2 * V - 1) / V * V; }  // superset + slack
  static size_t smem(int64_t c2) {
    return size_t(kMergeStages) * kMergeRows * 2 * size_t(row_elems(c2)) * sizeof(T) +
           2 * kMergeStages * 8;
  }
};

// One producer warp (the last) streams groups of R coarse rows + side rows into a
// ring of stages (full[st]: bytes landed); the consumer threads write the output
// rows whole and hand a stage back (empty[st]: every consumer arrived) -- no CTA
// barrier between groups.
template <class T>
__global__ void __launch_bounds__(1024) k_merge_even(const T* __restrict__ coarse,
                                                     const T* __restrict__ side, T* __restrict__ out,
                                                     LevelArgs<T> a) {
  ptx::pdl_trigger();
  constexpr int V = MergeCfg<T>::V;
  using VT = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
  const int64_t c1 = a.c[1], c2 = a.c[2], e1 = a.e[1], e2 = a.e[2];
  const int64_t rows = a.c[0] * c1, RE = MergeCfg<T>::row_elems(c2);
  extern __shared__ __align__(16) unsigned char smem_m[];
  constexpr int R = kMergeRows, S = kMergeStages;
  T* ring = reinterpret_cast<T*>(smem_m);  // [stage][row][coarse row | side row]
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + S * R * 2 * RE);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x;
  const int nc = int(blockDim.x) - 32;  // consumer threads
  if (tid == 0) {
    for (int k = 0; k < S; ++k) {
      ptx::mbar_init(&full[k], 1);
      ptx::mbar_init(&empty[k], nc);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int64_t groups = (rows + R - 1) / R;  // a group = R consecutive rows
  const int64_t G = gridDim.x;
  ptx::pdl_wait();
  if (tid >= nc) {
    // ---- producer warp (lane 0)
    if (tid != nc) return;
    int it = 0;
    for (int64_t grp = blockIdx.x; grp < groups; grp += G, ++it) {
      const int st = it % S;
      if (it >= S) ptx::mbar_wait(&empty[st], uint32_t(((it / S) - 1) & 1));
      uint32_t total = 0;
      for (int r = 0; r < R; ++r) {
        const int64_t rr = grp * R + r;
        if (rr >= rows) break;
        const int64_t cb = rr * c2, sb = rr * (c2 - 1);
        const int pc = int(cb & (V - 1)), ps = int(sb & (V - 1));
        total += uint32_t((pc + c2 + V - 1) / V * V * sizeof(T)) +
                 uint32_t((ps + c2 - 1 + V - 1) / V * V * sizeof(T));
      }
      ptx::mbar_arrive_expect_tx(&full[st], total);
      for (int r = 0; r < R; ++r) {
        const int64_t rr = grp * R + r;
        if (rr >= rows) break;
        const int64_t cb = rr * c2, sb = rr * (c2 - 1);
        const int pc = int(cb & (V - 1)), ps = int(sb & (V - 1));
        T* dst = ring + (int64_t(st) * R + r) * 2 * RE;
        ptx::bulk_g2s(dst, coarse + (cb - pc), uint32_t((pc + c2 + V - 1) / V * V * sizeof(T)),
                      &full[st]);
        ptx::bulk_g2s(dst + RE, side + (sb - ps), uint32_t((ps + c2 - 1 + V - 1) / V * V * sizeof(T)),
                      &full[st]);
      }
    }
    return;
  }
  // ---- consumers
  int it = 0;
  for (int64_t grp = blockIdx.x; grp < groups; grp += G, ++it) {
    const int st = it % S;
    ptx::mbar_wait(&full[st], uint32_t((it / S) & 1));
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t rr = grp * R + r;
      if (rr >= rows) break;
      const T* base = ring + (int64_t(st) * R + r) * 2 * RE;
      const T* cr = base + int((rr * c2) & (V - 1));
      const T* sr = base + RE + int((rr * (c2 - 1)) & (V - 1));
      const int q0 = int(rr) / int(c1), q1 = int(rr) - q0 * int(c1);  // rows < 2^31
      const int64_t g = ((2 * int64_t(q0)) * e1 + 2 * q1) * e2;
      const int ph = int(g & (V - 1));
      const int nvec = int((ph + e2 + V - 1) / V);
      T* orow = out + (g - ph);
      VT* ov = reinterpret_cast<VT*>(orow);
      // output position p = u*V + k - ph: even p from the coarse row, odd from the
      // side row. Interior vectors are whole: no range checks, parity fixed by ph.
      auto edge = [&](int u) {
#pragma unroll
        for (int k = 0; k < V; ++k) {
          const int p = u * V + k - ph;
          if (p >= 0 && p < e2) orow[u * V + k] = (p & 1) ? sr[p >> 1] : cr[p >> 1];
        }
      };
      if (tid == 0) edge(0);
      if (tid == 1 && nvec > 1) edge(nvec - 1);
      if (!(ph & 1)) {
        for (int u = 1 + tid; u < nvec - 1; u += nc) {
          const int a0 = (u * V - ph) >> 1;
          VT w;
          if constexpr (V == 4) {
            w.x = cr[a0]; w.y = sr[a0]; w.z = cr[a0 + 1]; w.w = sr[a0 + 1];
          } else {
            w.x = cr[a0]; w.y = sr[a0];
          }
          ov[u] = w;
        }
      } else {
        for (int u = 1 + tid; u < nvec - 1; u += nc) {
          const int a0 = (u * V - ph) >> 1;
          VT w;
          if constexpr (V == 4) {
            w.x = sr[a0]; w.y = cr[a0 + 1]; w.z = sr[a0 + 1]; w.w = cr[a0 + 2];
          } else {
            w.x = sr[a0]; w.y = cr[a0 + 1];
          }
          ov[u] = w;
        }
      }
    }
    ptx::mbar_arrive(&empty[st]);  // this thread is done with the stage
  }
}

// Rank of level-cls node (i0,i1,i2) among the class-cls nodes in row-major
// order, skipping all-even indices (refactor.hpp:134-145).
__device__ __forceinline__ int64_t class_rank(int64_t i0, int64_t i1, int64_t i2, int64_t e1,
                                              int64_t e2) {
  const int64_t c1 = (e1 + 1) / 2, c2 = (e2 + 1) / 2;
  const int64_t flat = (i0 * e1 + i1) * e2 + i2;
  int64_t evens = ((i0 + 1) / 2) * c1 * c2;  // all-even nodes in planes < i0
  if ((i0 & 1) == 0) {
    evens += ((i1 + 1) / 2) * c2;
    if ((i1 & 1) == 0) evens += (i2 + 1) / 2;
  }
  return flat - evens;
}

template <class T>
__global__ void k_class_copy(T* data, int64_t n1, int64_t n2, int64_t stride, int64_t e0,
                             int64_t e1, int64_t e2, bool cls0, T* vals, bool extract) {
  const int64_t n = e0 * e1 * e2;
  GRID_STRIDE(idx, n) {
    const int64_t i2 = idx % e2, t = idx / e2, i1 = t % e1, i0 = t / e1;
    int64_t k;
    if (cls0) {
      k = idx;
    } else {
      if (((i0 | i1 | i2) & 1) == 0) continue;
      k = class_rank(i0, i1, i2, e1, e2);
    }
    T* p = data + ((i0 * stride) * n1 + i1 * stride) * n2 + i2 * stride;
    if (extract) vals[k] = *p;
    else *p = vals[k];
  }
}

// ---- fiber operators (tests / single-fiber API) ------------------------------

template <class T>
__global__ void k_fiber_mass(const T* __restrict__ v, T* __restrict__ out, int64_t n,
                             int64_t count, const T* __restrict__ h) {
  GRID_STRIDE(idx, n * count) {
    const int64_t i = idx % n;
    const T* f = v + (idx - i);
    const T left = i > 0 ? h[i - 1] : T(0), right = i + 1 < n ? h[i] : T(0);
    T acc = T(2) * (left + right) * f[i];
    if (i > 0) acc += left * f[i - 1];
    if (i + 1 < n) acc += right * f[i + 1];
    out[idx] = acc;
  }
}

// apply_fiber (correction.hpp:141-154); zero_even: even fine inputs read as 0
template <class T>
__global__ void k_fiber_masstrans(const T* __restrict__ v, T* __restrict__ out, int64_t n,
                                  int64_t count, const T* __restrict__ taps, bool zero_even) {
  const int64_t nc = (n - 1) / 2 + 1;
  GRID_STRIDE(idx, nc * count) {
    const int64_t i = idx % nc, f = idx / nc;
    T acc = T(0);
    for (int k = 0; k < 5; ++k) {
      const int64_t j = 2 * i - 2 + k;
      if (j < 0 || j >= n || (zero_even && !(j & 1))) continue;
      acc += taps[i * 5 + k] * v[f * n + j];
    }
    out[idx] = acc;
  }
}

// transfer_apply (correction.hpp:67-88): coarse i gathers fine 2i with the
// refined neighbours 2i-1 / 2i+1 at their interpolation weights toward i
template <class T>
__global__ void k_fiber_transfer(const T* __restrict__ v, T* __restrict__ out, int64_t n,
                                 int64_t count, const T* __restrict__ trl,
                                 const T* __restrict__ trr) {
  const int64_t nc = (n - 1) / 2 + 1;
  GRID_STRIDE(idx, nc * count) {
    const int64_t i = idx % nc;
    const T* f = v + (idx / nc) * n;
    T acc = T(0);
    if (i > 0) acc += trl[i] * f[2 * i - 1];
    acc += f[2 * i];
    if (i + 1 < nc) acc += trr[i] * f[2 * i + 1];
    out[idx] = acc;
  }
}

template <class T>
__global__ void k_fiber_thomas(const T* __restrict__ v, T* __restrict__ out, int64_t n,
                               int64_t count, const T* mult, const T* rpiv, const T* upper) {
  GRID_STRIDE(f, count) {
    const T* x = v + f * n;
    T* y = out + f * n;
    T prev = x[0];
    y[0] = prev;
    for (int64_t i = 1; i < n; ++i) {
      prev = x[i] - mult[i - 1] * prev;
      y[i] = prev;
    }
    T next = prev * rpiv[n - 1];
    y[n - 1] = next;
    for (int64_t i = n - 1; i-- > 0;) {
      next = (y[i] - upper[i] * next) * rpiv[i];
      y[i] = next;
    }
  }
}

// y[i] += sign * x[i] (coarse += / -= correction after a register-tiled Thomas pass)
template <class T>
__global__ void k_axpy(T* y, const T* x, int64_t n, int sign) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    y[i] = sign > 0 ? y[i] + x[i] : y[i] - x[i];
}

// ---- launchers -----------------------------------------------------------------

#define LAUNCH(kernel, work, threads, s, ...)                                   \
  do {                                                                          \
    kernel<<<grid_for((work), (threads)), (threads), 0, (s)>>>(__VA_ARGS__);    \
    HGR_CUDA_CHECK(cudaGetLastError());                                         \
  } while (0)

template <class T>
void launch_gpk_dec(T* U, T* C, const LevelArgs<T>& a, int* flag, bool check, cudaStream_t s) {
  LAUNCH(k_gpk_dec<T>, a.e[0] * a.e[1] * a.e[2], 256, s, U, C, a, flag, check);
}
template <class T>
void launch_gpk_rec(const T* coef, T* out, const T* C, const T* Z, const LevelArgs<T>& a,
                    bool with, cudaStream_t s) {
  LAUNCH(k_gpk_rec<T>, a.e[0] * a.e[1] * a.e[2], 256, s, coef, out, C, Z, a, with);
}
template <class T>
void launch_lpk(const T* in, const int64_t e[3], T* out, int dim, int64_t cd, const T* taps,
                bool mask, cudaStream_t s) {
  int64_t o = e[0] * e[1] * e[2] / e[dim] * cd;
  LAUNCH(k_lpk<T>, o, 256, s, in, out, e[0], e[1], e[2], dim, cd, taps, mask);
}
template <class T>
void launch_thomas(T* z, const int64_t e[3], int dim, const T* mult, const T* rpiv,
                   const T* upper, T* apply, int sign, cudaStream_t s) {
  int64_t lines = e[0] * e[1] * e[2] / e[dim];
  LAUNCH(k_thomas<T>, lines, 128, s, z, e[0], e[1], e[2], dim, mult, rpiv, upper, apply, sign);
}
template <class T>
void launch_axpy(T* y, const T* x, int64_t n, int sign, cudaStream_t s) {
  LAUNCH(k_axpy<T>, n, 256, s, y, x, n, sign);
}
template <class T>
void launch_gather(const T* src, const int64_t se[3], int64_t stride, T* dst,
                   const int64_t de[3], cudaStream_t s) {
  // a warp per destination row
  const int64_t items = de[0] * de[1] * ((de[2] + kRowSeg - 1) / kRowSeg);  // a warp each
  launch_pdl(k_gather<T>, dim3(grid_for(items * 32, 256)), dim3(256), 0, s, 8 * de[0] * de[1] * de[2],
             src, se[1], se[2], stride,
             dst, de[0], de[1], de[2]);
}
template <class T>
bool merge_even_fits(int64_t c2) {
  return MergeCfg<T>::smem(c2) <= 200 * 1024;
}
template <class T>
void launch_merge_even(const T* coarse, const T* side, T* out, const LevelArgs<T>& a,
                       cudaStream_t s) {
  constexpr int64_t V = MergeCfg<T>::V;
  const int64_t nvec = (a.e[2] + 2 * V - 2) / V;
  // consumer threads cover a row's vectors once, plus the producer warp
  const int threads = int(std::min<int64_t>(992, (nvec + 31) / 32 * 32)) + 32;
  const size_t smem = MergeCfg<T>::smem(a.c[2]);
  require(merge_even_fits<T>(a.c[2]), "merge_even: rows too long for the shared-memory ring");
  set_smem_attr(reinterpret_cast<const void*>(k_merge_even<T>), smem);
  int per_sm = 0;
  HGR_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_merge_even<T>, threads, smem));
  const int64_t groups = (a.c[0] * a.c[1] + kMergeRows - 1) / kMergeRows;
  const int64_t grid = grid_for(groups * threads, threads, std::max(1, per_sm));
  launch_pdl(k_merge_even<T>, dim3(unsigned(grid)), dim3(threads), smem, s, a.e[0] * a.e[1] * a.e[2],
             coarse, side, out, a);
}
template <class T>
void launch_scatter_even(const T* src, T* dst, const LevelArgs<T>& a, cudaStream_t s) {
  const int64_t items = a.c[0] * a.c[1] * ((a.c[2] + kRowSeg - 1) / kRowSeg);  // a warp each
  launch_pdl(k_scatter_even<T>, dim3(grid_for(items * 32, 256)), dim3(256), 0, s,
             a.e[0] * a.e[1] * a.e[2], src, dst, a);
}
template <class T>
void launch_coefficients(const T* fine, T* coeffs, const LevelArgs<T>& a, cudaStream_t s) {
  LAUNCH(k_coefficients<T>, a.e[0] * a.e[1] * a.e[2], 256, s, fine, coeffs, a);
}
template <class T>
void launch_interpolate(const T* coarse, T* fine, const LevelArgs<T>& a, cudaStream_t s) {
  LAUNCH(k_interpolate<T>, a.e[0] * a.e[1] * a.e[2], 256, s, coarse, fine, a);
}
template <class T>
void launch_check_coarse_zero(const T* v, const LevelArgs<T>& a, int* flag, cudaStream_t s) {
  LAUNCH(k_check_coarse_zero<T>, a.c[0] * a.c[1] * a.c[2], 256, s, v, a, flag);
}
template <class T>
void launch_class_copy(T* data, const int64_t fe[3], int64_t stride, const int64_t ce[3],
                       bool cls0, T* vals, bool extract, cudaStream_t s) {
  LAUNCH(k_class_copy<T>, ce[0] * ce[1] * ce[2], 256, s, data, fe[1], fe[2], stride, ce[0],
         ce[1], ce[2], cls0, vals, extract);
}
template <class T>
void check_finite(const T* v, int64_t n, int* flag, cudaStream_t s) {
  LAUNCH(k_check_finite<T>, n, 256, s, v, n, flag);
}
template <class T>
void launch_fiber_mass(const T* v, T* out, int64_t n, int64_t count, const T* h, cudaStream_t s) {
  LAUNCH(k_fiber_mass<T>, n * count, 256, s, v, out, n, count, h);
}
template <class T>
void launch_fiber_masstrans(const T* v, T* out, int64_t n, int64_t count, const T* taps,
                            bool zero_even, cudaStream_t s) {
  LAUNCH(k_fiber_masstrans<T>, ((n - 1) / 2 + 1) * count, 256, s, v, out, n, count, taps,
         zero_even);
}
template <class T>
void launch_fiber_transfer(const T* v, T* out, int64_t n, int64_t count, const T* trl,
                           const T* trr, cudaStream_t s) {
  LAUNCH(k_fiber_transfer<T>, ((n - 1) / 2 + 1) * count, 256, s, v, out, n, count, trl, trr);
}
template <class T>
void launch_fiber_thomas(const T* v, T* out, int64_t n, int64_t count, const T* mult,
                         const T* rpiv, const T* upper, cudaStream_t s) {
  LAUNCH(k_fiber_thomas<T>, count, 128, s, v, out, n, count, mult, rpiv, upper);
}

#define INSTANTIATE(T)                                                                       \
  template void launch_gpk_dec<T>(T*, T*, const LevelArgs<T>&, int*, bool, cudaStream_t);    \
  template void launch_gpk_rec<T>(const T*, T*, const T*, const T*, const LevelArgs<T>&, bool, \
                                  cudaStream_t);                                             \
  template void launch_lpk<T>(const T*, const int64_t*, T*, int, int64_t, const T*, bool,    \
                              cudaStream_t);                                                 \
  template void launch_thomas<T>(T*, const int64_t*, int, const T*, const T*, const T*, T*,  \
                                 int, cudaStream_t);                                         \
  template void launch_axpy<T>(T*, const T*, int64_t, int, cudaStream_t);                    \
  template void launch_gather<T>(const T*, const int64_t*, int64_t, T*, const int64_t*,      \
                                 cudaStream_t);                                              \
  template void launch_scatter_even<T>(const T*, T*, const LevelArgs<T>&, cudaStream_t);     \
  template void launch_merge_even<T>(const T*, const T*, T*, const LevelArgs<T>&, cudaStream_t); \
  template bool merge_even_fits<T>(int64_t);                                                 \
  template void launch_coefficients<T>(const T*, T*, const LevelArgs<T>&, cudaStream_t);     \
  template void launch_interpolate<T>(const T*, T*, const LevelArgs<T>&, cudaStream_t);      \
  template void launch_check_coarse_zero<T>(const T*, const LevelArgs<T>&, int*, cudaStream_t); \
  template void launch_class_copy<T>(T*, const int64_t*, int64_t, const int64_t*, bool, T*,  \
                                     bool, cudaStream_t);                                    \
  template void check_finite<T>(const T*, int64_t, int*, cudaStream_t);                     \
  template void launch_fiber_mass<T>(const T*, T*, int64_t, int64_t, const T*, cudaStream_t); \
  template void launch_fiber_masstrans<T>(const T*, T*, int64_t, int64_t, const T*, bool,    \
                                          cudaStream_t);                                     \
  template void launch_fiber_transfer<T>(const T*, T*, int64_t, int64_t, const T*, const T*, \
                                         cudaStream_t);                                      \
  template void launch_fiber_thomas<T>(const T*, T*, int64_t, int64_t, const T*, const T*,   \
                                       const T*, cudaStream_t);

INSTANTIATE(float)
INSTANTIATE(double)

}  // namespace hgrb
