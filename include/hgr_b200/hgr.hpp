// hgr_b200/hgr.hpp -- C++ drop-in for the reference's public API (hgr,
// /root/reference/proj/include/hgr/hgr.hpp), running decompose / recompose and
// the single-level operators on B200 through the C ABI (include/hgr_cuda.h,
// libhgr_b200.so). Same namespace, types, signatures and error behaviour, so
// reference callers (tools/hgr_main.cpp, storage.hpp, the tests) recompile
// against this header unchanged:
//
//   ndarray<T>, ndview<T>, full_view, level_view      (ndarray.hpp, grid_hierarchy.hpp)
//   GridHierarchy, build_hierarchy, node_weights      (grid_hierarchy.hpp:15-199)
//   RefactoredArray<T>, decompose, recompose          (refactor.hpp:20-90)
//   ErrorReport, error_report                         (refactor.hpp:93-120)
//   CoefficientClass, extract_class, scatter_class    (refactor.hpp:124-170)
//   interpolate_to_fine, compute_coefficients, apply_coefficients (transforms.hpp:76-124)
//   compute_correction, mass_apply, masstrans_apply, thomas_solve (correction.hpp)
//   error, worker_count, set_worker_count             (error.hpp, parallel.hpp)
//
// The namespace can be renamed with -DHGR_B200_NAMESPACE=... when a program
// also includes the reference headers (the oracle build does so in its own TU).
// Link: -Lpaper_2007_04457_b200/lib -lhgr_b200 (no CUDA headers needed).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstddef>
#include <limits>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../hgr_cuda.h"

#ifndef HGR_B200_NAMESPACE
#define HGR_B200_NAMESPACE hgr
#endif

namespace HGR_B200_NAMESPACE {

inline constexpr int max_rank = 3;

/// Thrown for all domain failures (error.hpp:9-11).
struct error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void require(bool ok, const std::string& what) {
  if (!ok) throw error(what);
}
inline void check(int status) {
  if (status != HGR_OK) throw error(hgr_cuda_last_error());
}
template <class T>
constexpr bool is_f64() {
  static_assert(std::is_same_v<T, double> || std::is_same_v<T, float>, "float or double only");
  return std::is_same_v<T, double>;
}
}  // namespace detail

/// CPU worker controls of the reference (parallel.hpp:35-42): kept for source
/// compatibility; the GPU path has no host workers.
inline std::size_t worker_count() { return 1; }
inline void set_worker_count(std::size_t) {}

/// Dense row-major array of rank 1..3 (ndarray.hpp:15-57).
template <class T>
class ndarray {
 public:
  ndarray() = default;
  explicit ndarray(std::vector<std::size_t> extents)
      : extents_(std::move(extents)), data_(count_of(extents_)) {}
  ndarray(std::vector<std::size_t> extents, std::vector<T> values)
      : extents_(std::move(extents)), data_(std::move(values)) {
    detail::require(data_.size() == count_of(extents_),
                    "ndarray: value count does not match extents");
  }
  int rank() const { return static_cast<int>(extents_.size()); }
  const std::vector<std::size_t>& extents() const { return extents_; }
  std::size_t extent(int d) const { return extents_[static_cast<std::size_t>(d)]; }
  std::size_t size() const { return data_.size(); }
  T* data() { return data_.data(); }
  const T* data() const { return data_.data(); }
  std::vector<T>& values() { return data_; }
  const std::vector<T>& values() const { return data_; }
  T& operator[](std::size_t i) { return data_[i]; }
  const T& operator[](std::size_t i) const { return data_[i]; }
  friend bool operator==(const ndarray& a, const ndarray& b) {
    return a.extents_ == b.extents_ && a.data_ == b.data_;
  }
  static std::size_t count_of(const std::vector<std::size_t>& extents) {
    detail::require(!extents.empty() && extents.size() <= max_rank,
                    "ndarray: rank must be between 1 and 3");
    std::size_t n = 1;
    for (std::size_t e : extents) n *= e;
    return n;
  }

 private:
  std::vector<std::size_t> extents_;
  std::vector<T> data_;
};

/// Strided rank-3 window (ndarray.hpp:61-70).
template <class T>
struct ndview {
  T* ptr = nullptr;
  std::array<std::size_t, 3> shape{1, 1, 1};
  std::array<std::size_t, 3> stride{0, 0, 0};
  T& operator()(std::size_t i, std::size_t j, std::size_t k) const {
    return ptr[i * stride[0] + j * stride[1] + k * stride[2]];
  }
};

namespace detail {
inline std::array<std::size_t, 3> natural_strides(const std::vector<std::size_t>& e) {
  std::array<std::size_t, 3> s{0, 0, 0};
  std::size_t acc = 1;
  for (int d = static_cast<int>(e.size()) - 1; d >= 0; --d) {
    s[static_cast<std::size_t>(d)] = acc;
    acc *= e[static_cast<std::size_t>(d)];
  }
  return s;
}
inline std::array<std::size_t, 3> padded_extents(const std::vector<std::size_t>& e) {
  std::array<std::size_t, 3> p{1, 1, 1};
  for (std::size_t d = 0; d < e.size(); ++d) p[d] = e[d];
  return p;
}
}  // namespace detail

template <class T>
ndview<T> full_view(ndarray<T>& a) {
  return {a.data(), detail::padded_extents(a.extents()), detail::natural_strides(a.extents())};
}
template <class T>
ndview<const T> full_view(const ndarray<T>& a) {
  return {a.data(), detail::padded_extents(a.extents()), detail::natural_strides(a.extents())};
}

template <class Real>
struct node_weights {
  Real to_left;
  Real to_right;
};

/// Dyadic level structure (grid_hierarchy.hpp:47-194). Validation runs through
/// the library so the messages are the reference's.
class GridHierarchy {
 public:
  GridHierarchy() = default;
  explicit GridHierarchy(std::vector<std::vector<double>> coords_per_dim)
      : coords_(std::move(coords_per_dim)) {
    detail::require(!coords_.empty() && coords_.size() <= max_rank,
                    "grid must have 1 to 3 dimensions");
    const hgr_grid_desc g = desc();
    levels_ = hgr_levels(&g);
    if (levels_ < 0) throw error(hgr_cuda_last_error());
  }
  static GridHierarchy uniform(const std::vector<std::size_t>& sizes) {
    std::vector<std::vector<double>> c(sizes.size());
    for (std::size_t d = 0; d < sizes.size(); ++d) {
      c[d].resize(sizes[d]);
      for (std::size_t i = 0; i < sizes[d]; ++i) c[d][i] = static_cast<double>(i);
    }
    return GridHierarchy(std::move(c));
  }
  int rank() const { return static_cast<int>(coords_.size()); }
  int levels() const { return levels_; }
  int class_count() const { return levels_ + 1; }
  const std::vector<double>& coords(int d) const { return coords_[check_dim(d)]; }
  std::size_t finest_extent(int d) const { return coords_[check_dim(d)].size(); }
  std::vector<std::size_t> finest_extents() const {
    std::vector<std::size_t> e(coords_.size());
    for (std::size_t d = 0; d < coords_.size(); ++d) e[d] = coords_[d].size();
    return e;
  }
  std::size_t level_stride(int level) const {
    return std::size_t{1} << static_cast<unsigned>(levels_ - check_level(level));
  }
  std::size_t level_extent(int level, int d) const {
    return (finest_extent(d) - 1) / level_stride(level) + 1;
  }
  std::vector<std::size_t> level_extents(int level) const {
    std::vector<std::size_t> e(coords_.size());
    for (int d = 0; d < rank(); ++d) e[static_cast<std::size_t>(d)] = level_extent(level, d);
    return e;
  }
  std::size_t level_node_count(int level) const {
    std::size_t n = 1;
    for (int d = 0; d < rank(); ++d) n *= level_extent(level, d);
    return n;
  }
  /// Spacings between consecutive level-l nodes along d (grid_hierarchy.hpp:163-177).
  std::vector<double> spacings(int level, int d) const {
    const std::size_t s = level_stride(level);
    const auto& c = coords(d);
    std::vector<double> h((c.size() - 1) / s);
    for (std::size_t i = 0; i < h.size(); ++i) h[i] = c[(i + 1) * s] - c[i * s];
    return h;
  }
  /// Refined-node weights (grid_hierarchy.hpp:27-31, :178-187).
  std::vector<node_weights<double>> refined_weights(int level, int d) const {
    detail::require(level >= 1 && level <= levels_, "level out of range");
    const auto h = spacings(level, d);
    std::vector<node_weights<double>> w(h.size() / 2);
    for (std::size_t q = 0; q < w.size(); ++q) {
      const double span = h[2 * q] + h[2 * q + 1];
      w[q] = {h[2 * q + 1] / span, h[2 * q] / span};
    }
    return w;
  }
  int node_class(std::span<const std::size_t> finest_index) const {
    int cls = 0;
    for (int d = 0; d < rank(); ++d) {
      const std::size_t i = finest_index[static_cast<std::size_t>(d)];
      if (i == 0) continue;
      int tz = 0;
      for (std::size_t v = i; !(v & 1u); v >>= 1) ++tz;
      if (levels_ - tz > cls) cls = levels_ - tz;
    }
    return cls;
  }
  std::size_t class_node_count(int cls) const {
    check_level(cls);
    if (cls == 0) return level_node_count(0);
    return level_node_count(cls) - level_node_count(cls - 1);
  }
  /// C-ABI view of this hierarchy (coordinates stay owned here).
  hgr_grid_desc desc() const {
    hgr_grid_desc g{};
    g.rank = rank();
    for (int d = 0; d < g.rank; ++d) {
      g.extents[d] = coords_[static_cast<std::size_t>(d)].size();
      g.coords[d] = coords_[static_cast<std::size_t>(d)].data();
    }
    return g;
  }

 private:
  std::size_t check_dim(int d) const {
    detail::require(d >= 0 && d < rank(), "dimension index out of range");
    return static_cast<std::size_t>(d);
  }
  int check_level(int level) const {
    detail::require(level >= 0 && level <= levels_, "level out of range");
    return level;
  }
  std::vector<std::vector<double>> coords_;
  int levels_ = 0;
};

inline GridHierarchy build_hierarchy(std::vector<std::vector<double>> coords_per_dim) {
  return GridHierarchy(std::move(coords_per_dim));
}

template <class T>
ndview<T> level_view(ndarray<T>& a, const GridHierarchy& g, int level) {
  detail::require(a.extents() == g.finest_extents(), "array shape does not match the finest grid");
  auto s = detail::natural_strides(a.extents());
  for (auto& x : s) x *= g.level_stride(level);
  return {a.data(), detail::padded_extents(g.level_extents(level)), s};
}
template <class T>
ndview<const T> level_view(const ndarray<T>& a, const GridHierarchy& g, int level) {
  detail::require(a.extents() == g.finest_extents(), "array shape does not match the finest grid");
  auto s = detail::natural_strides(a.extents());
  for (auto& x : s) x *= g.level_stride(level);
  return {a.data(), detail::padded_extents(g.level_extents(level)), s};
}

/// In-place coefficient pyramid (refactor.hpp:20-26).
template <class T>
struct RefactoredArray {
  ndarray<T> data;
  GridHierarchy hierarchy;
  static constexpr std::size_t precision_bytes = sizeof(T);
};

/// hgr::decompose (refactor.hpp:32-57) on the GPU: H2D, fused level kernels,
/// D2H. Finiteness is checked before the input is modified.
template <class T>
RefactoredArray<T> decompose(ndarray<T> data, const GridHierarchy& g) {
  detail::require(data.extents() == g.finest_extents(), "decompose: array shape does not match grid");
  const hgr_grid_desc d = g.desc();
  if constexpr (detail::is_f64<T>()) detail::check(hgr_decompose_host_f64(&d, data.data()));
  else detail::check(hgr_decompose_host_f32(&d, data.data()));
  return {std::move(data), g};
}

/// hgr::recompose (refactor.hpp:63-90).
template <class T>
ndarray<T> recompose(const RefactoredArray<T>& r, int upto_class) {
  const GridHierarchy& g = r.hierarchy;
  detail::require(upto_class >= 0 && upto_class <= g.levels(), "recompose: class index out of range");
  ndarray<T> out(r.data.extents());
  const hgr_grid_desc d = g.desc();
  if constexpr (detail::is_f64<T>())
    detail::check(hgr_recompose_host_f64(&d, r.data.data(), out.data(), upto_class));
  else
    detail::check(hgr_recompose_host_f32(&d, r.data.data(), out.data(), upto_class));
  return out;
}

struct ErrorReport {
  double l2_abs = 0, l2_rel = 0, linf_abs = 0, linf_rel = 0;
};

/// error_report (refactor.hpp:100-120), accumulated in double.
template <class T>
ErrorReport error_report(const ndarray<T>& original, const ndarray<T>& reconstruction) {
  detail::require(original.extents() == reconstruction.extents(), "error_report: shape mismatch");
  double sq_diff = 0, sq_orig = 0, max_diff = 0, max_orig = 0;
  for (std::size_t i = 0; i < original.size(); ++i) {
    const double a = static_cast<double>(original[i]);
    const double dd = a - static_cast<double>(reconstruction[i]);
    sq_diff += dd * dd;
    sq_orig += a * a;
    max_diff = std::max(max_diff, std::abs(dd));
    max_orig = std::max(max_orig, std::abs(a));
  }
  ErrorReport rep;
  rep.l2_abs = std::sqrt(sq_diff);
  rep.linf_abs = max_diff;
  const double inf = std::numeric_limits<double>::infinity();
  rep.l2_rel = sq_orig > 0 ? rep.l2_abs / std::sqrt(sq_orig) : (rep.l2_abs > 0 ? inf : 0.0);
  rep.linf_rel = max_orig > 0 ? rep.linf_abs / max_orig : (rep.linf_abs > 0 ? inf : 0.0);
  return rep;
}

template <class T>
struct CoefficientClass {
  int level = 0;
  std::vector<T> values;
};

namespace detail {
// refactor.hpp:134-145 class walk (row-major, all-even indices skipped for cls > 0)
template <class Array, class Fn>
void for_each_class_node(Array& data, const GridHierarchy& g, int cls, Fn&& fn) {
  auto view = level_view(data, g, cls);
  const auto ext = padded_extents(g.level_extents(cls));
  for (std::size_t i0 = 0; i0 < ext[0]; ++i0)
    for (std::size_t i1 = 0; i1 < ext[1]; ++i1)
      for (std::size_t i2 = 0; i2 < ext[2]; ++i2) {
        if (cls > 0 && (i0 & 1) == 0 && (i1 & 1) == 0 && (i2 & 1) == 0) continue;
        fn(view(i0, i1, i2));
      }
}
}  // namespace detail

template <class T>
CoefficientClass<T> extract_class(const RefactoredArray<T>& r, int cls) {
  CoefficientClass<T> out;
  out.level = cls;
  out.values.reserve(r.hierarchy.class_node_count(cls));
  detail::for_each_class_node(r.data, r.hierarchy, cls, [&](const T& v) { out.values.push_back(v); });
  return out;
}

template <class T>
void scatter_class(RefactoredArray<T>& r, int cls, std::span<const T> values) {
  detail::require(values.size() == r.hierarchy.class_node_count(cls),
                  "scatter_class: value count does not match class size");
  std::size_t k = 0;
  detail::for_each_class_node(r.data, r.hierarchy, cls, [&](T& v) { v = values[k++]; });
}
template <class T>
void scatter_class(RefactoredArray<T>& r, int cls, const std::vector<T>& values) {
  scatter_class(r, cls, std::span<const T>(values));
}

namespace detail {
template <class T>
ndarray<T> level_op(int op, const ndarray<T>& in, const GridHierarchy& g, int level,
                    int out_level) {
  ndarray<T> out(g.level_extents(out_level));
  const hgr_grid_desc d = g.desc();
  if constexpr (is_f64<T>()) check(hgr_host_level_op_f64(&d, op, level, in.data(), out.data()));
  else check(hgr_host_level_op_f32(&d, op, level, in.data(), out.data()));
  return out;
}
template <class T>
void check_level_shape(const ndarray<T>& a, const GridHierarchy& g, int level, const char* what) {
  require(a.extents() == g.level_extents(level), std::string(what) + ": shape mismatch");
}
template <class T>
std::vector<T> fiber_op(int op, std::span<const T> v, std::span<const T> h, std::size_t nout) {
  std::vector<T> out(nout);
  if constexpr (is_f64<T>()) check(hgr_host_fiber_op_f64(op, v.size(), 1, v.data(), h.data(), out.data()));
  else check(hgr_host_fiber_op_f32(op, v.size(), 1, v.data(), h.data(), out.data()));
  return out;
}
}  // namespace detail

/// interpolate_to_fine (transforms.hpp:76-92)
template <class T>
ndarray<T> interpolate_to_fine(const ndarray<T>& coarse, const GridHierarchy& g, int level) {
  detail::require(level >= 1 && level <= g.levels(), "level out of range");
  detail::check_level_shape(coarse, g, level - 1, "interpolate_to_fine");
  return detail::level_op(0, coarse, g, level, level);
}

/// compute_coefficients (transforms.hpp:96-111)
template <class T>
ndarray<T> compute_coefficients(const ndarray<T>& fine, const GridHierarchy& g, int level) {
  detail::require(level >= 1 && level <= g.levels(), "level out of range");
  detail::check_level_shape(fine, g, level, "compute_coefficients");
  return detail::level_op(1, fine, g, level, level);
}

/// apply_coefficients (transforms.hpp:115-124)
template <class T>
ndarray<T> apply_coefficients(const ndarray<T>& coarse, const ndarray<T>& coeffs,
                              const GridHierarchy& g, int level) {
  detail::require(level >= 1 && level <= g.levels(), "level out of range");
  detail::check_level_shape(coarse, g, level - 1, "apply_coefficients");
  detail::check_level_shape(coeffs, g, level, "apply_coefficients");
  ndarray<T> fine = interpolate_to_fine(coarse, g, level);
  for (std::size_t i = 0; i < fine.size(); ++i) fine[i] += coeffs[i];
  return fine;
}

/// compute_correction (correction.hpp:348-365)
template <class T>
ndarray<T> compute_correction(const ndarray<T>& coeffs, const GridHierarchy& g, int level) {
  detail::require(level >= 1 && level <= g.levels(), "level out of range");
  detail::require(coeffs.extents() == g.level_extents(level), "compute_correction: shape mismatch");
  return detail::level_op(2, coeffs, g, level, level - 1);
}

/// mass_apply / masstrans_apply / thomas_solve (correction.hpp:58-223)
template <class T>
std::vector<T> mass_apply(std::span<const T> v, std::span<const T> h) {
  detail::require(v.size() == h.size() + 1, "mass_apply: |v| must equal |h|+1");
  return detail::fiber_op<T>(0, v, h, v.size());
}
template <class T>
std::vector<T> masstrans_apply(std::span<const T> v, std::span<const T> h) {
  detail::require(v.size() == h.size() + 1, "masstrans_apply: |v| must equal |h|+1");
  return detail::fiber_op<T>(1, v, h, (v.size() - 1) / 2 + 1);
}
template <class T>
std::vector<T> thomas_solve(std::span<const T> rhs, std::span<const T> h) {
  detail::require(rhs.size() == h.size() + 1, "thomas_solve: |rhs| must equal |h|+1");
  return detail::fiber_op<T>(2, rhs, h, rhs.size());
}

}  // namespace HGR_B200_NAMESPACE
