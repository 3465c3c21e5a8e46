// stream_mb.cu -- microbenchmark (dev aid, not product): how fast can a CTA
// stream halo'd plane windows of a 1025^3 array through shared memory?
//   A: 1D TMA tensor copies (one per window row), one issuing thread
//   A4: same, issued by one lane per warp
//   B: 16-byte cp.async by all threads (the v6 level-kernel scheme)
//   C: direct coalesced LDG, no shared memory
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 stream_mb.cu -o stream_mb -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

using T = double;
#define NT ((int)blockDim.x)

__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void arrive_tx(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(sa(b)), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) { while (!try_wait(b, ph)) {} }
__device__ __forceinline__ void tma1d(void* dst, const CUtensorMap* m, int x, uint64_t* b) {
  asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
               ::"r"(sa(dst)), "l"(m), "r"(x), "r"(sa(b)) : "memory");
}
__device__ __forceinline__ void cpa16(void* d, const void* s) { asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(d)), "l"(s) : "memory"); }
__device__ __forceinline__ void cpa_arrive(uint64_t* b) { asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(b)) : "memory"); }

struct Geo { int64_t e; int RW, CW, step_r, step_c, S; int nt1, nt2, nseg; int P; int B; };

template <int MODE, int NS>
__global__ void __launch_bounds__(512, 1) k_stream(const T* U, const __grid_constant__ CUtensorMap map, Geo g, T* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int SLOT = g.RW * g.P;
  T* raw = reinterpret_cast<T*>(smem);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + size_t(NS) * SLOT * sizeof(T));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int bid = blockIdx.x;
  const int t2 = bid % g.nt2; bid /= g.nt2;
  const int t1 = bid % g.nt1; const int seg = bid / g.nt1;
  const int64_t e = g.e, plane = e * e;
  const int64_t r0 = int64_t(t1) * g.step_r, c0 = int64_t(t2) * g.step_c;
  const int64_t j0 = int64_t(seg) * g.S;
  int np = g.S; if (j0 + np > e) np = int(e - j0);
  T acc = 0;
  if (MODE == 2) {  // direct LDG
    for (int p = 0; p < np; ++p) {
      const T* base = U + (j0 + p) * plane;
      for (int i = tid; i < SLOT; i += NT) {
        const int r = i / g.CW, c = i - r * g.CW;
        const int64_t gr = r0 + r, gc = c0 + c;
        if (gr < e && gc < e) acc += __ldg(base + gr * e + gc);
      }
    }
    sink[blockIdx.x * NT + tid] = acc;
    return;
  }
  if (tid == 0) { for (int s = 0; s < NS; ++s) mbar_init(&bar[s], MODE == 1 ? NT : 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  auto issue = [&](int p) {
    const int sl = p % NS;
    T* dst = raw + sl * SLOT;
    const int64_t pb = (j0 + p) * plane;
    if (MODE == 0) {
      if (tid == 0) {
        arrive_tx(&bar[sl], uint32_t(g.RW * g.B * sizeof(T)));
        for (int r = 0; r < g.RW; ++r) tma1d(dst + r * g.P, &map, int((pb + (r0 + r) * e + c0) & ~int64_t(1)), &bar[sl]);
      }
    } else if (MODE == 3) {
      if (tid == 0) arrive_tx(&bar[sl], uint32_t(g.RW * g.B * sizeof(T)));
      __syncwarp();
      if (lane == 0)
        for (int r = warp; r < g.RW; r += NT / 32) tma1d(dst + r * g.P, &map, int((pb + (r0 + r) * e + c0) & ~int64_t(1)), &bar[sl]);
    } else {
      // 16-byte chunks of the aligned superset of each row
      for (int r = warp; r < g.RW; r += NT / 32) {
        const int64_t f = pb + (r0 + r) * e + c0;
        const int64_t alo = f & ~int64_t(1);
        const int nch = int((f - alo + g.CW + 1) >> 1);
        for (int ch = lane; ch < nch; ch += 32)
          if (alo + 2 * ch + 2 <= e * e * e) cpa16(dst + r * g.P + 2 * ch, U + alo + 2 * ch);
      }
      cpa_arrive(&bar[sl]);
    }
  };
  for (int p = 0; p < NS && p < np; ++p) issue(p);
  for (int p = 0; p < np; ++p) {
    const int sl = p % NS;
    wait(&bar[sl], (p / NS) & 1);
    const T* S = raw + sl * SLOT;
    for (int i = tid; i < SLOT; i += NT) acc += S[i];
    __syncthreads();
    if (p + NS < np) issue(p + NS);
  }
  sink[blockIdx.x * NT + tid] = acc;
}

int main(int argc, char** argv) {
  const int64_t e = 1025, N = e * e * e;
  T* U; CK(cudaMalloc(&U, (N + 64) * sizeof(T)));
  CK(cudaMemset(U, 0, (N + 64) * sizeof(T)));
  T* sink; CK(cudaMalloc(&sink, sizeof(T) * 4096 * 2048));
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  struct Case { int mode; int RW, CW, step_r, step_c; const char* name; };
  std::vector<Case> cases;
  int nthr = 512;
  if (argc >= 7) {
    cases.push_back({atoi(argv[1]), atoi(argv[2]), atoi(argv[3]), atoi(argv[4]), atoi(argv[5]), "custom"});
    nthr = atoi(argv[6]);
  } else {
    cases = {{3, 61, 62, 58, 58, "TMA1d warp issuers, 61x62"}, {1, 61, 62, 58, 58, "cp.async16, 61x62"}};
  }
  for (auto& cs : cases) {
    CUtensorMap map;
    cuuint64_t gdim[1] = {cuuint64_t(N)}, gstr[1] = {0};
    cuuint32_t box[1] = {cuuint32_t((cs.CW + 2) & ~1)}, es[1] = {1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, U, gdim, gstr, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", int(r)); continue; }
    for (int S : {64, 128}) {
      Geo g{e, cs.RW, cs.CW, cs.step_r, cs.step_c, S, 0, 0, 0, (cs.CW + 2 + 15) / 16 * 16, (cs.CW + 2) & ~1};
      g.nt1 = int((e - 3 + cs.step_r - 1) / cs.step_r);
      g.nt2 = int((e - 3 + cs.step_c - 1) / cs.step_c);
      g.nseg = int((e + S - 1) / S);
      const int grid = g.nt1 * g.nt2 * g.nseg;
      constexpr int NS = 5;
      size_t smem = size_t(NS) * cs.RW * g.P * sizeof(T) + 64;
      if (smem > 227 * 1024) { printf("%s: smem too big\n", cs.name); continue; }
      auto run = [&]() {
        switch (cs.mode) {
          case 0: CK(cudaFuncSetAttribute(k_stream<0, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))); k_stream<0, NS><<<grid, nthr, smem>>>(U, map, g, sink); break;
          case 1: CK(cudaFuncSetAttribute(k_stream<1, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))); k_stream<1, NS><<<grid, nthr, smem>>>(U, map, g, sink); break;
          case 2: k_stream<2, NS><<<grid, nthr, 0>>>(U, map, g, sink); break;
          case 3: CK(cudaFuncSetAttribute(k_stream<3, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))); k_stream<3, NS><<<grid, nthr, smem>>>(U, map, g, sink); break;
        }
      };
      run(); CK(cudaDeviceSynchronize());
      cudaEventRecord(a);
      const int it = 5;
      for (int i = 0; i < it; ++i) run();
      cudaEventRecord(b); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b); ms /= it;
      const double moved = double(grid) / g.nseg * cs.RW * cs.CW * double(e) * sizeof(T);
      printf("%-30s S=%3d grid=%6d  %7.3f ms  unique %6.0f GB/s  moved %6.0f GB/s\n", cs.name, S, grid, ms,
             N * sizeof(T) / ms / 1e6, moved / ms / 1e6);
    }
  }
  return 0;
}
