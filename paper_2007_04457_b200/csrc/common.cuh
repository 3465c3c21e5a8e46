// common.cuh -- shared device-side types for the hierarchical refactoring kernels.
//
// Canonical layout: every level array is a compact row-major 3D array with
// extents (e0, e1, e2), dimension 2 contiguous. Rank-r reference arrays are
// padded on the LEFT (rank 1: (1,1,n); rank 2: (1,n0,n1)) so the contiguous
// dimension is always dim 2 and the reference's ascending dimension order
// (correction.hpp:322, :335) is preserved on the real dimensions. The
// reference pads on the right (ndarray.hpp:90-94); the flat memory layout is
// identical.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hgrb {

// Per-level, per-dimension device tables (built on the host in plan.cu):
//  wl/wr  : refined-node weights toward coarse q / q+1 (grid_hierarchy.hpp:27-31,
//           built in double, cast to T as transforms.hpp:46-51 does), c_d-1 entries
//  taps   : mass-trans stencil K = R*M, 5 per coarse row (correction.hpp:96-133), in T
//  mult/pivot/upper/rpiv : Thomas factors of the level-(l-1) mass matrix
//           (correction.hpp:188-198), in T; rpiv = 1/pivot
//  h      : level-l spacings in T (spacings_as<T>, correction.hpp:227-231), e_d-1
//  trl/trr: transfer weights in T (correction.hpp:67-88): weight of fine node
//           2q-1 (trl) / 2q+1 (trr) into coarse node q, 0 at the ends; c_d entries
template <class T>
struct LevelArgs {
  int64_t e[3];  // level-l (fine) extents
  int64_t c[3];  // level-(l-1) (coarse) extents
  const T* wl[3];
  const T* wr[3];
  const T* taps[3];
  const T* h[3];
  const T* trl[3];
  const T* trr[3];
  const T* mult[3];
  const T* pivot[3];
  const T* upper[3];
  const T* rpiv[3];
};

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

#define HGR_CUDA_CHECK(expr)                                                   \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) ::hgrb::throw_cuda(_e, #expr, __FILE__, __LINE__);  \
  } while (0)

[[noreturn]] void throw_cuda(cudaError_t e, const char* expr, const char* file, int line);

// Grid size for grid-stride kernels: a multiple of the SM count.
int grid_for(int64_t work, int threads, int blocks_per_sm = 8);

}  // namespace hgrb
