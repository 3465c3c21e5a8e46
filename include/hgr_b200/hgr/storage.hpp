// hgr_b200/hgr/storage.hpp -- drop-in for hgr/storage.hpp (storage.hpp:13-218):
// the progressive ".hg" container. Classes are packed and scattered on the GPU
// (csrc/storage.cu) and move as one contiguous payload; files are
// byte-identical to the reference's write_file. Header parsing and its error
// texts are the library's (hgr_hg_read_info: "bad magic", "truncated", ...).
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "error.hpp"
#include "refactor.hpp"

namespace HGR_B200_NAMESPACE {

inline constexpr std::array<char, 4> hg_magic{'H', 'G', 'R', 'F'};
inline constexpr std::uint16_t hg_format_version = 1;

struct HgClassRange {
  std::uint64_t offset = 0;
  std::uint64_t bytes = 0;
};

struct HgFileHeader {
  std::uint16_t version = hg_format_version;
  std::uint8_t precision_bytes = 0;
  std::uint8_t rank = 0;
  std::vector<std::uint64_t> extents;
  std::vector<std::vector<double>> coords;
  std::vector<HgClassRange> classes;  // coarse first
  std::uint64_t header_bytes = 0;
  std::uint64_t file_bytes = 0;

  int class_count() const { return static_cast<int>(classes.size()); }
  std::uint64_t class_elements(int cls) const {
    return classes[static_cast<std::size_t>(cls)].bytes / precision_bytes;
  }
  std::uint64_t total_elements() const {
    std::uint64_t n = 1;
    for (auto e : extents) n *= e;
    return n;
  }
};

namespace detail {

// magic, version, precision, rank, extents, coordinates, class count, class table
inline std::uint64_t hg_header_bytes(int rank, const std::vector<std::uint64_t>& extents,
                                     int class_count) {
  std::uint64_t b = 4 + 2 + 1 + 1 + 2 + 8 * std::uint64_t(rank) + 16 * std::uint64_t(class_count);
  for (auto e : extents) b += 8 * e;
  return b;
}

}  // namespace detail

/// Writes the pyramid (classes packed on the GPU); returns the file size.
template <class T>
std::uint64_t write_file(const RefactoredArray<T>& r, const std::string& path) {
  const hgr_grid_desc d = r.hierarchy.desc();
  std::uint64_t n = 0;
  if constexpr (detail::is_f64<T>()) detail::check(hgr_write_hg_host_f64(path.c_str(), &d, r.data.data(), &n));
  else detail::check(hgr_write_hg_host_f32(path.c_str(), &d, r.data.data(), &n));
  return n;
}

/// Header and class table only; payloads are not read.
inline HgFileHeader read_info(const std::string& path) {
  hgr_hg_info info{};
  detail::check(hgr_hg_read_info(path.c_str(), &info));
  HgFileHeader h;
  h.version = static_cast<std::uint16_t>(info.version);
  h.precision_bytes = static_cast<std::uint8_t>(info.precision_bytes);
  h.rank = static_cast<std::uint8_t>(info.rank);
  for (int d = 0; d < info.rank; ++d) {
    h.extents.push_back(info.extents[d]);
    h.coords.emplace_back(info.extents[d]);
    detail::check(hgr_hg_read_coords(path.c_str(), d, h.coords.back().data()));
  }
  std::vector<std::uint64_t> off(std::size_t(info.class_count)), len(off.size());
  detail::check(hgr_hg_read_class_table(path.c_str(), off.data(), len.data(), info.class_count));
  for (std::size_t c = 0; c < off.size(); ++c) h.classes.push_back({off[c], len[c]});
  h.header_bytes = info.header_bytes;
  h.file_bytes = info.file_bytes;
  return h;
}

template <class T>
struct PrefixRead {
  RefactoredArray<T> array;
  std::uint64_t bytes_read = 0;
};

/// Header plus classes 0..upto_class, scattered on the GPU into a zero-filled
/// pyramid; bytes_read counts the header and the classes read.
template <class T>
PrefixRead<T> read_prefix(const std::string& path, int upto_class) {
  const HgFileHeader h = read_info(path);
  detail::require(h.precision_bytes == sizeof(T),
                  path + ": file precision is " + std::to_string(h.precision_bytes) +
                      " bytes per element, reader expects " + std::to_string(sizeof(T)));
  detail::require(upto_class >= 0 && upto_class < h.class_count(), path + ": class index out of range");
  GridHierarchy g(h.coords);
  PrefixRead<T> out{{ndarray<T>(g.finest_extents()), g}, 0};
  if constexpr (detail::is_f64<T>())
    detail::check(hgr_read_hg_prefix_host_f64(path.c_str(), upto_class, out.array.data.data(), &out.bytes_read));
  else
    detail::check(hgr_read_hg_prefix_host_f32(path.c_str(), upto_class, out.array.data.data(), &out.bytes_read));
  return out;
}

}  // namespace HGR_B200_NAMESPACE
