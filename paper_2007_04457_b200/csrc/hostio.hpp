// hostio.hpp -- host <-> device movement of the host-pointer entry points
// (hostio.cu): pinned buffers by direct DMA, pageable ones through the plan's
// pinned staging ring with a multi-threaded host copy beside the DMA.
#pragma once

#include <cstddef>

#include "plan.hpp"

namespace hgrb {

// the plan's finest-size device buffer `which` (0 or 1), allocated on first use
void* host_device_buffer(Plan& p, int which, std::size_t bytes);
// the plan's private stream for the synchronous host-pointer calls
cudaStream_t host_stream(Plan& p);
// enqueue h -> d on s (pageable sources are staged; returns once h may be reused)
void host_to_device(Plan& p, void* d, const void* h, std::size_t bytes, cudaStream_t s);
// d -> h after the work already on s; returns when h holds the data
void device_to_host(Plan& p, void* h, const void* d, std::size_t bytes, cudaStream_t s);

// grid-key helpers of the one-shot plan cache (capi.cu), chunked over the copy
// pool: 1D grids carry as many coordinates as data values
// c[i] == i for every i (null: the uniform grid)
bool host_coords_iota(const double* c, std::size_t n);
// bitwise equality of two coordinate arrays
bool host_coords_equal(const double* x, const double* y, std::size_t n);

}  // namespace hgrb
