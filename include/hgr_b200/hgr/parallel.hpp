// hgr_b200/hgr/parallel.hpp -- drop-in for hgr/parallel.hpp (parallel.hpp:14-77).
// The reference spreads its fiber and node loops over std::threads; on the GPU
// path those loops are kernels, so the worker controls only keep their
// contract (HGR_THREADS / set_worker_count are honoured as numbers and
// results never depend on them) and parallel_for runs its chunks on the
// calling thread. Nothing on the decompose / recompose path uses them.
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <thread>

#include "error.hpp"

namespace HGR_B200_NAMESPACE {

namespace detail {

inline std::size_t& worker_override() {
  static std::size_t n = 0;  // 0: automatic
  return n;
}

inline std::size_t env_worker_count() {
  if (const char* v = std::getenv("HGR_THREADS")) {
    char* end = nullptr;
    const long n = std::strtol(v, &end, 10);
    if (end != v && n > 0) return static_cast<std::size_t>(n);
  }
  const unsigned hw = std::thread::hardware_concurrency();
  return hw ? hw : 1;
}

}  // namespace detail

/// Worker count the reference would use (override, HGR_THREADS, or the
/// hardware thread count).
inline std::size_t worker_count() {
  if (const std::size_t n = detail::worker_override()) return n;
  static const std::size_t env = detail::env_worker_count();
  return env;
}

/// Override the worker count (0 restores the automatic choice).
inline void set_worker_count(std::size_t n) { detail::worker_override() = n; }

namespace detail {

// fn(begin, end) over [0, count) in grain-sized chunks, in order, on this thread
template <class Fn>
void parallel_for(std::size_t count, std::size_t grain, Fn&& fn) {
  grain = std::max<std::size_t>(grain, 1);
  for (std::size_t b = 0; b < count; b += grain) fn(b, std::min(count, b + grain));
}

}  // namespace detail
}  // namespace HGR_B200_NAMESPACE
