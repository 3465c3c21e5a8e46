// tma_probe.cu -- which 1D/2D tensor-map copies are legal on sm_100a (dev aid)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__global__ void k1(const __grid_constant__ CUtensorMap map, int x, int y, int rank, double* out, int n, int doff) {
  __shared__ __align__(1024) double buf[1024];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(n * 8));
    if (rank == 1)
      asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                   ::"r"(sa(buf + doff)), "l"(&map), "r"(x), "r"(sa(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(sa(buf)), "l"(&map), "r"(x), "r"(y), "r"(sa(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(sa(&bar)) : "memory");
    for (int i = 0; i < n; ++i) out[i] = buf[i + doff];
  }
}
int main(int argc, char** argv) {
  int which = atoi(argv[1]);
  long N = atol(argv[2]); int box = atoi(argv[3]); int x = atoi(argv[4]);
  double* U; cudaMalloc(&U, (N + 64) * 8);
  double* h = (double*)malloc((N + 64) * 8); for (long i = 0; i < N + 64; ++i) h[i] = double(i);
  cudaMemcpy(U, h, (N + 64) * 8, cudaMemcpyHostToDevice);
  double* out; cudaMalloc(&out, 4096 * 8);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap map; CUresult r;
  int n = box;
  if (which == 1) {
    cuuint64_t gdim[1] = {cuuint64_t(N)}, gstr[1] = {8};
    cuuint32_t bx[1] = {cuuint32_t(box)}, es[1] = {1};
    r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, U, gdim, gstr, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t gdim[2] = {1024, cuuint64_t(N / 1024)}, gstr[1] = {8192};
    cuuint32_t bx[2] = {cuuint32_t(box), 1}, es[2] = {1, 1};
    r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, U, gdim, gstr, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  printf("rank %d N %ld box %d x %d: encode %d ", which, N, box, x, int(r));
  k1<<<1, 32>>>(map, x, 0, which, out, n, argc > 5 ? atoi(argv[5]) : 0);
  cudaError_t e = cudaDeviceSynchronize();
  double o[4096]; cudaMemcpy(o, out, n * 8, cudaMemcpyDeviceToHost);
  printf("-> %s  out[0]=%g out[n-1]=%g\n", cudaGetErrorString(e), o[0], o[n - 1]);
  return 0;
}
