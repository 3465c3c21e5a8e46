// synth.cu -- deterministic synthetic fields for benchmarks and tests
// (SURVEY.md §8d), bitwise identical to tests/synthetic.py.
#include <vector>

#include "../../include/hgr_cuda.h"
#include "plan.hpp"

namespace hgrb {

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <class T>
__global__ void k_synth(T* out, int64_t e1, int64_t e2, int64_t n, uint64_t seed,
                        const double* __restrict__ fa, const double* __restrict__ fb,
                        const double* __restrict__ fc) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = i % e2, t = i / e2, j = t % e1, p = t / e1;
    const double base = __dadd_rn(__dmul_rn(fa[p], fb[j]), fc[k]);
    const uint64_t z = splitmix64(seed + uint64_t(i));
    const double eta = __dadd_rn(__dmul_rn(__dmul_rn(double(z >> 11), 0x1.0p-53), 2.0), -1.0);
    out[i] = T(__dadd_rn(base, __dmul_rn(1e-3, eta)));
  }
}

}  // namespace

template <class T>
void synthetic_field(const hgr_grid_desc* g, T* out, uint64_t seed, const double* ha,
                     const double* hb, const double* hc, cudaStream_t s) {
  require(g && g->rank >= 1 && g->rank <= 3, "grid must have 1 to 3 dimensions");
  int64_t e[3] = {1, 1, 1};
  for (int d = 0; d < g->rank; ++d) e[d] = int64_t(g->extents[d]);
  const int64_t n = e[0] * e[1] * e[2];
  double* dt = nullptr;
  HGR_CUDA_CHECK(cudaMalloc(&dt, size_t(e[0] + e[1] + e[2]) * sizeof(double)));
  HGR_CUDA_CHECK(cudaMemcpyAsync(dt, ha, size_t(e[0]) * sizeof(double), cudaMemcpyHostToDevice, s));
  HGR_CUDA_CHECK(cudaMemcpyAsync(dt + e[0], hb, size_t(e[1]) * sizeof(double), cudaMemcpyHostToDevice, s));
  HGR_CUDA_CHECK(cudaMemcpyAsync(dt + e[0] + e[1], hc, size_t(e[2]) * sizeof(double),
                                 cudaMemcpyHostToDevice, s));
  k_synth<T><<<grid_for(n, 256, 16), 256, 0, s>>>(out, e[1], e[2], n, seed, dt, dt + e[0],
                                                   dt + e[0] + e[1]);
  HGR_CUDA_CHECK(cudaGetLastError());
  HGR_CUDA_CHECK(cudaStreamSynchronize(s));
  HGR_CUDA_CHECK(cudaFree(dt));
}

template void synthetic_field<float>(const hgr_grid_desc*, float*, uint64_t, const double*,
                                     const double*, const double*, cudaStream_t);
template void synthetic_field<double>(const hgr_grid_desc*, double*, uint64_t, const double*,
                                      const double*, const double*, cudaStream_t);

}  // namespace hgrb
