// report.cu -- error_report (refactor.hpp:100-120) on the device: L2 and Linf
// absolute / relative errors accumulated in double. A fixed grid of
// kRepBlocks CTAs reduces grid-stride slices into per-CTA partials and one CTA
// folds them in index order, so the result does not depend on scheduling (no
// atomics) and is identical run to run. Bandwidth bound: reads 2nS bytes.
#include "plan.hpp"

namespace hgrb {

namespace {

constexpr int kRepThreads = 512;
constexpr int kRepBlocks = 148 * 4;

struct Acc {
  double sq_diff, sq_orig, max_diff, max_orig;
};

__device__ inline Acc combine(Acc a, const Acc& b) {
  a.sq_diff += b.sq_diff;
  a.sq_orig += b.sq_orig;
  a.max_diff = fmax(a.max_diff, b.max_diff);
  a.max_orig = fmax(a.max_orig, b.max_orig);
  return a;
}

__device__ inline Acc block_reduce(Acc v) {
  __shared__ Acc sh[kRepThreads / 32];
  for (int o = 16; o > 0; o >>= 1) {
    Acc w;
    w.sq_diff = __shfl_down_sync(0xffffffffu, v.sq_diff, o);
    w.sq_orig = __shfl_down_sync(0xffffffffu, v.sq_orig, o);
    w.max_diff = __shfl_down_sync(0xffffffffu, v.max_diff, o);
    w.max_orig = __shfl_down_sync(0xffffffffu, v.max_orig, o);
    v = combine(v, w);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < kRepThreads / 32 ? sh[lane] : Acc{0, 0, 0, 0};
    for (int o = 8; o > 0; o >>= 1) {
      Acc w;
      w.sq_diff = __shfl_down_sync(0xffffffffu, v.sq_diff, o);
      w.sq_orig = __shfl_down_sync(0xffffffffu, v.sq_orig, o);
      w.max_diff = __shfl_down_sync(0xffffffffu, v.max_diff, o);
      w.max_orig = __shfl_down_sync(0xffffffffu, v.max_orig, o);
      v = combine(v, w);
    }
  }
  return v;
}

template <class T>
__global__ void __launch_bounds__(kRepThreads) k_report_partial(const T* __restrict__ a,
                                                                 const T* __restrict__ b,
                                                                 int64_t n, Acc* partial) {
  Acc v{0, 0, 0, 0};
  const int64_t stride = int64_t(gridDim.x) * kRepThreads;
  for (int64_t i = int64_t(blockIdx.x) * kRepThreads + threadIdx.x; i < n; i += stride) {
    const double x = double(a[i]);
    const double d = x - double(b[i]);
    v.sq_diff += d * d;
    v.sq_orig += x * x;
    v.max_diff = fmax(v.max_diff, fabs(d));
    v.max_orig = fmax(v.max_orig, fabs(x));
  }
  v = block_reduce(v);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
}

__global__ void __launch_bounds__(kRepThreads) k_report_final(const Acc* partial, int count,
                                                              double* out) {
  Acc v{0, 0, 0, 0};
  for (int i = threadIdx.x; i < count; i += kRepThreads) v = combine(v, partial[i]);
  v = block_reduce(v);
  if (threadIdx.x == 0) {
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    const double l2 = sqrt(v.sq_diff);
    out[0] = l2;
    out[1] = v.sq_orig > 0 ? l2 / sqrt(v.sq_orig) : (l2 > 0 ? inf : 0.0);
    out[2] = v.max_diff;
    out[3] = v.max_orig > 0 ? v.max_diff / v.max_orig : (v.max_diff > 0 ? inf : 0.0);
  }
}

}  // namespace

template <class T>
void error_report(const T* a, const T* b, int64_t n, double out[4], cudaStream_t s) {
  Acc* partial = nullptr;
  double* d_out = nullptr;
  HGR_CUDA_CHECK(cudaMallocAsync(&partial, sizeof(Acc) * kRepBlocks + 4 * sizeof(double), s));
  d_out = reinterpret_cast<double*>(partial + kRepBlocks);
  const int blocks = int(std::min<int64_t>(kRepBlocks, std::max<int64_t>(1, ceil_div(n, kRepThreads))));
  k_report_partial<T><<<blocks, kRepThreads, 0, s>>>(a, b, n, partial);
  HGR_CUDA_CHECK(cudaGetLastError());
  k_report_final<<<1, kRepThreads, 0, s>>>(partial, blocks, d_out);
  HGR_CUDA_CHECK(cudaGetLastError());
  HGR_CUDA_CHECK(cudaMemcpyAsync(out, d_out, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
  HGR_CUDA_CHECK(cudaFreeAsync(partial, s));
  HGR_CUDA_CHECK(cudaStreamSynchronize(s));
}

template void error_report<float>(const float*, const float*, int64_t, double*, cudaStream_t);
template void error_report<double>(const double*, const double*, int64_t, double*, cudaStream_t);

}  // namespace hgrb
