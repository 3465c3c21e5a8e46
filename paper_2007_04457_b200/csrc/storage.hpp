// storage.hpp -- the .hg container (reference storage.hpp:17-218) on the GPU path.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace hgrb {

class Plan;

// HgFileHeader (storage.hpp:36-55)
struct HgInfo {
  uint16_t version = 1;
  uint8_t precision_bytes = 0;
  uint8_t rank = 0;
  std::vector<uint64_t> extents;
  std::vector<std::vector<double>> coords;
  std::vector<uint64_t> offsets, bytes;  // per class, coarse first
  uint64_t header_bytes = 0, file_bytes = 0;
};

uint64_t hg_header_bytes(int rank, const uint64_t* extents, int classes);
HgInfo hg_read_info(const std::string& path);
// returns the file size; byte-identical to hgr::write_file
uint64_t hg_write(const std::string& path, Plan& plan, const void* d_pyramid, cudaStream_t s);
// returns bytes_read (header + classes 0..upto); synchronous
uint64_t hg_read_prefix(const std::string& path, const HgInfo& info, Plan& plan, int upto,
                        void* d_pyramid, cudaStream_t s);

}  // namespace hgrb
