// hgr_b200/hgr/error.hpp -- drop-in for the reference's hgr/error.hpp
// (error.hpp:9-17): the one exception type of the library and the argument
// check that raises it. Every other drop-in header includes this one, so the
// namespace switch and the C ABI live here.
//
// The drop-in tree mirrors /root/reference/proj/include/hgr file by file; put
// include/hgr_b200 on the include path (-I include/hgr_b200) and reference
// callers' `#include "hgr/hgr.hpp"` / `"hgr/refactor.hpp"` / ... resolve here.
// Link with -lhgr_b200 (paper_2007_04457_b200/lib). No CUDA headers needed.
#pragma once

#include <stdexcept>
#include <string>
#include <type_traits>

#include "../../hgr_cuda.h"

// The namespace can be renamed (-DHGR_B200_NAMESPACE=...) when a program also
// includes the reference headers (the oracle does so in its own TU).
#ifndef HGR_B200_NAMESPACE
#define HGR_B200_NAMESPACE hgr
#endif

namespace HGR_B200_NAMESPACE {

/// Thrown for all domain, format and I/O failures (error.hpp:9-11).
struct error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {

inline void require(bool ok, const std::string& what) {
  if (!ok) throw error(what);
}

// C ABI status -> hgr::error carrying the library's (reference-worded) message
inline void check(int status) {
  if (status != HGR_OK) throw error(hgr_cuda_last_error());
}

template <class T>
constexpr bool is_f64() {
  static_assert(std::is_same_v<T, double> || std::is_same_v<T, float>,
                "the GPU library is instantiated for float and double");
  return std::is_same_v<T, double>;
}

}  // namespace detail
}  // namespace HGR_B200_NAMESPACE
