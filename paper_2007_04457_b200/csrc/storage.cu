// storage.cu -- the progressive ".hg" container of the reference
// (storage.hpp:17-218) on the GPU path: classes are packed / unpacked on the
// device (the class order of extract_class / scatter_class, refactor.hpp:134-170)
// and move between host and device as one contiguous payload through a pinned
// staging buffer. Files are byte-identical to hgr::write_file's; error texts
// keep storage.hpp's substrings.
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "plan.hpp"
#include "storage.hpp"

namespace hgrb {

namespace {

constexpr char kMagic[4] = {'H', 'G', 'R', 'F'};
constexpr uint16_t kVersion = 1;
constexpr std::size_t kStage = std::size_t(256) << 20;  // pinned staging chunk

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

struct Pinned {
  void* p = nullptr;
  explicit Pinned(std::size_t bytes) { HGR_CUDA_CHECK(cudaMallocHost(&p, bytes)); }
  ~Pinned() { cudaFreeHost(p); }
};

struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(std::size_t bytes) { HGR_CUDA_CHECK(cudaMalloc(&p, bytes ? bytes : 16)); }
  ~DevBuf() { cudaFree(p); }
};

template <class U>
void get(FILE* f, U& v, const std::string& path) {
  require(std::fread(&v, sizeof v, 1, f) == 1, path + ": truncated file");
}

bool pow2_plus_1(uint64_t n) { return n >= 2 && ((n - 1) & (n - 2)) == 0; }

}  // namespace

uint64_t hg_header_bytes(int rank, const uint64_t* extents, int classes) {
  uint64_t coords = 0;
  for (int d = 0; d < rank; ++d) coords += 8 * extents[d];
  return 4 + 2 + 1 + 1 + 8 * uint64_t(rank) + coords + 2 + 16 * uint64_t(classes);
}

// read_info (storage.hpp:129-177)
HgInfo hg_read_info(const std::string& path) {
  File file;
  file.f = std::fopen(path.c_str(), "rb");
  require(file.f != nullptr, path + ": cannot open");
  char magic[4] = {0, 0, 0, 0};
  require(std::fread(magic, 1, 4, file.f) == 4 && std::memcmp(magic, kMagic, 4) == 0,
          path + ": not an HGRF file (bad magic)");
  HgInfo h;
  get(file.f, h.version, path);
  require(h.version == kVersion, path + ": unsupported format version " + std::to_string(h.version));
  get(file.f, h.precision_bytes, path);
  require(h.precision_bytes == 4 || h.precision_bytes == 8, path + ": invalid precision code");
  get(file.f, h.rank, path);
  require(h.rank >= 1 && h.rank <= 3, path + ": invalid dimension count");
  h.extents.resize(h.rank);
  for (auto& e : h.extents) {
    get(file.f, e, path);
    require(pow2_plus_1(e), path + ": dimension size must be 2^k+1");
  }
  h.coords.resize(h.rank);
  for (int d = 0; d < h.rank; ++d) {
    auto& c = h.coords[std::size_t(d)];
    c.resize(h.extents[std::size_t(d)]);
    require(std::fread(c.data(), 8, c.size(), file.f) == c.size(),
            path + ": truncated coordinate table");
  }
  uint16_t classes = 0;
  get(file.f, classes, path);
  require(classes >= 1, path + ": empty class table");
  h.offsets.resize(classes);
  h.bytes.resize(classes);
  for (int c = 0; c < classes; ++c) {
    get(file.f, h.offsets[std::size_t(c)], path);
    get(file.f, h.bytes[std::size_t(c)], path);
  }
  h.header_bytes = hg_header_bytes(h.rank, h.extents.data(), classes);
  require(h.offsets.front() == h.header_bytes, path + ": corrupt class table");
  uint64_t expect = h.header_bytes, elements = 0, total = 1;
  for (auto e : h.extents) total *= e;
  for (int c = 0; c < classes; ++c) {
    require(h.offsets[std::size_t(c)] == expect,
            path + ": class offsets must be contiguous and increasing");
    require(h.bytes[std::size_t(c)] % h.precision_bytes == 0,
            path + ": class byte length misaligned");
    expect = h.offsets[std::size_t(c)] + h.bytes[std::size_t(c)];
    elements += h.bytes[std::size_t(c)] / h.precision_bytes;
  }
  require(elements == total, path + ": class sizes do not cover the array");
  h.file_bytes = expect;
  return h;
}

// write_file (storage.hpp:86-126): header, then classes 0..L packed on the
// device into one payload, copied out in pinned chunks.
uint64_t hg_write(const std::string& path, Plan& plan, const void* d_pyramid, cudaStream_t s) {
  const Hierarchy& h = plan.h;
  const std::size_t S = plan.dtype == HGR_F64 ? 8 : 4;
  const int classes = h.L + 1;
  std::vector<uint64_t> ext(std::size_t(h.rank));
  for (int d = 0; d < h.rank; ++d) ext[std::size_t(d)] = h.coords[std::size_t(d)].size();
  const uint64_t header = hg_header_bytes(h.rank, ext.data(), classes);
  std::vector<uint64_t> off(static_cast<std::size_t>(classes)), bytes(off.size());
  uint64_t o = header;
  for (int c = 0; c < classes; ++c) {
    off[std::size_t(c)] = o;
    bytes[std::size_t(c)] = h.class_node_count(c) * S;
    o += bytes[std::size_t(c)];
  }
  const uint64_t payload = o - header;

  DevBuf dev(payload);
  for (int c = 0; c < classes; ++c)
    plan.class_copy(const_cast<void*>(d_pyramid), c,
                    static_cast<char*>(dev.p) + (off[std::size_t(c)] - header), true, s);

  File file;
  file.f = std::fopen(path.c_str(), "wb");
  require(file.f != nullptr, path + ": cannot open for writing");
  std::vector<char> hb;
  auto put = [&](const void* p, std::size_t n) {
    hb.insert(hb.end(), static_cast<const char*>(p), static_cast<const char*>(p) + n);
  };
  put(kMagic, 4);
  put(&kVersion, 2);
  const uint8_t prec = uint8_t(S), rank = uint8_t(h.rank);
  put(&prec, 1);
  put(&rank, 1);
  for (auto e : ext) put(&e, 8);
  for (int d = 0; d < h.rank; ++d) put(h.coords[std::size_t(d)].data(), 8 * ext[std::size_t(d)]);
  const uint16_t nc = uint16_t(classes);
  put(&nc, 2);
  for (int c = 0; c < classes; ++c) {
    put(&off[std::size_t(c)], 8);
    put(&bytes[std::size_t(c)], 8);
  }
  require(std::fwrite(hb.data(), 1, hb.size(), file.f) == hb.size(), path + ": write failed");
  Pinned stage(std::min<std::size_t>(payload ? payload : 16, kStage));
  for (uint64_t pos = 0; pos < payload; pos += kStage) {
    const std::size_t n = std::size_t(std::min<uint64_t>(kStage, payload - pos));
    HGR_CUDA_CHECK(cudaMemcpyAsync(stage.p, static_cast<char*>(dev.p) + pos, n,
                                   cudaMemcpyDeviceToHost, s));
    HGR_CUDA_CHECK(cudaStreamSynchronize(s));
    require(std::fwrite(stage.p, 1, n, file.f) == n, path + ": write failed");
  }
  require(std::fflush(file.f) == 0, path + ": write failed");
  return o;
}

// read_prefix (storage.hpp:187-216): the pyramid is zero-filled, classes
// 0..upto (one contiguous byte range after the header) are staged to the
// device and scattered there.
uint64_t hg_read_prefix(const std::string& path, const HgInfo& info, Plan& plan, int upto,
                        void* d_pyramid, cudaStream_t s) {
  const std::size_t S = plan.dtype == HGR_F64 ? 8 : 4;
  require(info.precision_bytes == S, path + ": file precision is " +
                                         std::to_string(info.precision_bytes) +
                                         " bytes per element, reader expects " + std::to_string(S));
  require(upto >= 0 && upto < int(info.offsets.size()), path + ": class index out of range");
  require(plan.h.L + 1 == int(info.offsets.size()), path + ": class count mismatch");
  const uint64_t n = plan.h.node_count(plan.h.L);
  HGR_CUDA_CHECK(cudaMemsetAsync(d_pyramid, 0, n * S, s));
  const uint64_t prefix = info.offsets[std::size_t(upto)] + info.bytes[std::size_t(upto)] -
                          info.header_bytes;
  DevBuf dev(prefix);
  File file;
  file.f = std::fopen(path.c_str(), "rb");
  require(file.f != nullptr, path + ": cannot open");
  require(std::fseek(file.f, long(info.header_bytes), SEEK_SET) == 0, path + ": truncated payload");
  Pinned stage(std::min<std::size_t>(prefix ? prefix : 16, kStage));
  for (uint64_t pos = 0; pos < prefix; pos += kStage) {
    const std::size_t m = std::size_t(std::min<uint64_t>(kStage, prefix - pos));
    HGR_CUDA_CHECK(cudaStreamSynchronize(s));  // the staging buffer is free again
    require(std::fread(stage.p, 1, m, file.f) == m, path + ": truncated payload");
    HGR_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(dev.p) + pos, stage.p, m,
                                   cudaMemcpyHostToDevice, s));
  }
  for (int c = 0; c <= upto; ++c)
    plan.class_copy(d_pyramid, c,
                    static_cast<char*>(dev.p) + (info.offsets[std::size_t(c)] - info.header_bytes),
                    false, s);
  HGR_CUDA_CHECK(cudaStreamSynchronize(s));
  return info.offsets[std::size_t(upto)] + info.bytes[std::size_t(upto)];
}

}  // namespace hgrb
