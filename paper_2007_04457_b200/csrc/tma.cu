// tma.cu -- see tma.hpp.
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <mutex>
#include <string>

#include "plan.hpp"
#include "tma.hpp"

namespace hgrb {

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}
}  // namespace

void make_tma_1d(CUtensorMap* map, const void* base, uint64_t n, int elem_bytes, int box) {
  auto fn = encode_fn();
  require(fn != nullptr, "cuTensorMapEncodeTiled is unavailable (driver too old?)");
  require((reinterpret_cast<uintptr_t>(base) & 15) == 0, "TMA base must be 16-byte aligned");
  require(box > 0 && box <= 256 && (box * elem_bytes) % 16 == 0, "TMA box size");
  // a 1D map's extent must stay below 2^31 elements (larger extents are an illegal
  // instruction at copy time, measured on B200); callers keep every box of a
  // launch inside the first 2^31 - 1 elements from the base (run_fused / run_interp)
  const uint64_t nmax = (uint64_t(1) << 31) - 1;
  const cuuint64_t gdim[1] = {cuuint64_t(n < nmax ? n : nmax)};
  const cuuint64_t gstride[1] = {cuuint64_t(elem_bytes)};  // unused for rank 1
  const cuuint32_t bdim[1] = {cuuint32_t(box)};
  const cuuint32_t estr[1] = {1};
  const CUresult r = fn(map, elem_bytes == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                             : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                        1, const_cast<void*>(base), gdim, gstride, bdim, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

}  // namespace hgrb
