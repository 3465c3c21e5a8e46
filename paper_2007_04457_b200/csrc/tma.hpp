// tma.hpp -- host-side encoding of 1D TMA tensor maps (cuTensorMapEncodeTiled
// through the runtime's driver entry point, so the library needs no -lcuda).
#pragma once

#include <cuda.h>
#include <cstdint>

namespace hgrb {

// 1D map over `n` elements of `elem_bytes` (4 or 8) starting at `base` (16-byte
// aligned), box of `box` elements (box*elem_bytes a multiple of 16, <= 256
// elements). Elements outside [0, min(n, 2^31 - 1)) read as zero. Throws on failure.
void make_tma_1d(CUtensorMap* map, const void* base, uint64_t n, int elem_bytes, int box);

}  // namespace hgrb
