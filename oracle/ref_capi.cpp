// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Thin extern "C" wrapper that compiles the UNMODIFIED reference library
// (header-only, /root/reference/proj/include/hgr/*.hpp, included in place via
// -I, never copied) into oracle/_ref/libhgr_ref.so. It is the "reference"
// oracle / CPU baseline: tests use it to pin the C restatement
// (oracle/hgr_oracle.c) and bench.py --impl reference times it.
//
// Build recipe: oracle/Makefile (target `ref`), only when /root/reference is
// present. The reference's own CMake is not used.
#include <hgr/hgr.hpp>

#include <cstring>
#include <exception>
#include <random>
#include <string>
#include <vector>

#include "hgr_oracle.h"

namespace {

thread_local std::string g_err;

hgr::GridHierarchy make_grid(const hgro_grid* g) {
  std::vector<std::vector<double>> coords(static_cast<std::size_t>(g->rank));
  for (int d = 0; d < g->rank; ++d) {
    coords[d].resize(g->n[d]);
    for (std::size_t i = 0; i < g->n[d]; ++i)
      coords[d][i] = g->coords[d] ? g->coords[d][i] : static_cast<double>(i);
  }
  return hgr::GridHierarchy(std::move(coords));
}

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

template <class T>
hgr::ndarray<T> wrap(const std::vector<std::size_t>& ext, const T* p) {
  std::size_t n = 1;
  for (auto e : ext) n *= e;
  return hgr::ndarray<T>(ext, std::vector<T>(p, p + n));
}

template <class T>
int decompose(const hgro_grid* g, T* data) {
  return guarded([&] {
    auto grid = make_grid(g);
    auto r = hgr::decompose(wrap(grid.finest_extents(), data), grid);
    std::memcpy(data, r.data.data(), r.data.size() * sizeof(T));
  });
}

template <class T>
int recompose(const hgro_grid* g, const T* in, T* out, int upto) {
  return guarded([&] {
    auto grid = make_grid(g);
    hgr::RefactoredArray<T> r{wrap(grid.finest_extents(), in), grid};
    auto back = hgr::recompose(r, upto);
    std::memcpy(out, back.data(), back.size() * sizeof(T));
  });
}

template <class T>
int interp(const hgro_grid* g, int level, const T* coarse, T* fine) {
  return guarded([&] {
    auto grid = make_grid(g);
    hgr::detail::require(level >= 1 && level <= grid.levels(), "level out of range");
    auto out = hgr::interpolate_to_fine(wrap(grid.level_extents(level - 1), coarse), grid, level);
    std::memcpy(fine, out.data(), out.size() * sizeof(T));
  });
}

template <class T>
int coeffs(const hgro_grid* g, int level, const T* fine, T* out) {
  return guarded([&] {
    auto grid = make_grid(g);
    hgr::detail::require(level >= 0 && level <= grid.levels(), "level out of range");
    auto c = hgr::compute_coefficients(wrap(grid.level_extents(level), fine), grid, level);
    std::memcpy(out, c.data(), c.size() * sizeof(T));
  });
}

template <class T>
int correction(const hgro_grid* g, int level, const T* c, T* z) {
  return guarded([&] {
    auto grid = make_grid(g);
    hgr::detail::require(level >= 0 && level <= grid.levels(), "level out of range");
    auto r = hgr::compute_correction(wrap(grid.level_extents(level), c), grid, level);
    std::memcpy(z, r.data(), r.size() * sizeof(T));
  });
}

template <class T, class Op>
int fiber(std::size_t n, const T* v, const T* h, T* out, Op op) {
  return guarded([&] {
    std::vector<T> vv(v, v + n), hh(h, h + (n ? n - 1 : 0));
    auto r = op(std::span<const T>(vv), std::span<const T>(hh));
    std::memcpy(out, r.data(), r.size() * sizeof(T));
  });
}

template <class T>
int extract(const hgro_grid* g, const T* data, int cls, T* out) {
  return guarded([&] {
    auto grid = make_grid(g);
    hgr::RefactoredArray<T> r{wrap(grid.finest_extents(), data), grid};
    auto c = hgr::extract_class(r, cls);
    std::memcpy(out, c.values.data(), c.values.size() * sizeof(T));
  });
}

template <class T>
int scatter(const hgro_grid* g, T* data, int cls, const T* vals) {
  return guarded([&] {
    auto grid = make_grid(g);
    hgr::RefactoredArray<T> r{wrap(grid.finest_extents(), data), grid};
    std::vector<T> v(vals, vals + grid.class_node_count(cls));
    hgr::scatter_class(r, cls, v);
    std::memcpy(data, r.data.data(), r.data.size() * sizeof(T));
  });
}

template <class T>
int write_file_(const hgro_grid* g, const T* data, const char* path, unsigned long long* bytes) {
  return guarded([&] {
    auto grid = make_grid(g);
    hgr::RefactoredArray<T> r{wrap(grid.finest_extents(), data), grid};
    *bytes = hgr::write_file(r, path);
  });
}

template <class T>
int read_prefix_(const char* path, int upto, T* out, unsigned long long* bytes) {
  return guarded([&] {
    auto pr = hgr::read_prefix<T>(path, upto);
    std::memcpy(out, pr.array.data.data(), pr.array.data.size() * sizeof(T));
    *bytes = pr.bytes_read;
  });
}

}  // namespace

extern "C" {

const char* hgrref_last_error(void) { return g_err.c_str(); }

int hgrref_levels(const hgro_grid* g) {
  int L = -1;
  if (guarded([&] { L = make_grid(g).levels(); })) return -1;
  return L;
}

void hgrref_set_worker_count(std::size_t n) { hgr::set_worker_count(n); }
std::size_t hgrref_worker_count(void) { return hgr::worker_count(); }

#define REF_EXPORTS(T, S)                                                                      \
  int hgrref_decompose_##S(const hgro_grid* g, T* d) { return decompose<T>(g, d); }            \
  int hgrref_recompose_##S(const hgro_grid* g, const T* in, T* out, int m) {                   \
    return recompose<T>(g, in, out, m);                                                        \
  }                                                                                            \
  int hgrref_interpolate_to_fine_##S(const hgro_grid* g, int l, const T* c, T* f) {           \
    return interp<T>(g, l, c, f);                                                              \
  }                                                                                            \
  int hgrref_compute_coefficients_##S(const hgro_grid* g, int l, const T* f, T* c) {          \
    return coeffs<T>(g, l, f, c);                                                              \
  }                                                                                            \
  int hgrref_compute_correction_##S(const hgro_grid* g, int l, const T* c, T* z) {            \
    return correction<T>(g, l, c, z);                                                          \
  }                                                                                            \
  int hgrref_mass_apply_##S(std::size_t n, const T* v, const T* h, T* o) {                     \
    return fiber<T>(n, v, h, o, [](auto a, auto b) { return hgr::mass_apply<T>(a, b); });      \
  }                                                                                            \
  int hgrref_transfer_apply_##S(std::size_t n, const T* v, const T* h, T* o) {                 \
    return fiber<T>(n, v, h, o, [](auto a, auto b) { return hgr::transfer_apply<T>(a, b); });  \
  }                                                                                            \
  int hgrref_masstrans_apply_##S(std::size_t n, const T* v, const T* h, T* o) {                \
    return fiber<T>(n, v, h, o, [](auto a, auto b) { return hgr::masstrans_apply<T>(a, b); }); \
  }                                                                                            \
  int hgrref_thomas_solve_##S(std::size_t n, const T* v, const T* h, T* o) {                   \
    return fiber<T>(n, v, h, o, [](auto a, auto b) { return hgr::thomas_solve<T>(a, b); });    \
  }                                                                                            \
  int hgrref_extract_class_##S(const hgro_grid* g, const T* d, int c, T* o) {                  \
    return extract<T>(g, d, c, o);                                                             \
  }                                                                                            \
  int hgrref_scatter_class_##S(const hgro_grid* g, T* d, int c, const T* v) {                  \
    return scatter<T>(g, d, c, v);                                                             \
  }                                                                                            \
  int hgrref_write_file_##S(const hgro_grid* g, const T* d, const char* p,                     \
                            unsigned long long* b) {                                           \
    return write_file_<T>(g, d, p, b);                                                         \
  }                                                                                            \
  int hgrref_read_prefix_##S(const char* p, int m, T* o, unsigned long long* b) {             \
    return read_prefix_<T>(p, m, o, b);                                                        \
  }

REF_EXPORTS(double, f64)
REF_EXPORTS(float, f32)

// perf_model.hpp:71-98 (the CLI's rank-configs)
double hgrref_estimate_time(int kind, unsigned long long bx, unsigned long long by,
                            unsigned long long bz, unsigned long long n, unsigned long long S,
                            unsigned long long L, unsigned long long G, double bw) {
  hgr::PerfParams p;
  p.n = n;
  p.transaction_bytes = S;
  p.element_bytes = L;
  p.ghost_elements = G;
  p.peak_bandwidth = bw;
  const hgr::KernelKind k = kind == 0 ? hgr::KernelKind::gpk
                            : kind == 1 ? hgr::KernelKind::lpk : hgr::KernelKind::ipk;
  double t = -1;
  guarded([&] { t = hgr::estimate_time(k, hgr::KernelConfig{bx, by, bz}, p); });
  return t;
}

// Seeded fixtures exactly as the reference's tests draw them
// (tests/oracle_helpers.hpp:230-246): libstdc++ mt19937 + uniform_real.
void hgrref_random_coords(std::size_t n, unsigned seed, double* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> gap(0.2, 1.8);
  out[0] = 0.0;
  for (std::size_t i = 1; i < n; ++i) out[i] = out[i - 1] + gap(rng);
}

void hgrref_random_values(std::size_t n, unsigned seed, double* out) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (std::size_t i = 0; i < n; ++i) out[i] = dist(rng);
}

}  // extern "C"
