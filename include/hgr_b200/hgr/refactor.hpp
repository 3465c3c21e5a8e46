// hgr_b200/hgr/refactor.hpp -- drop-in for hgr/refactor.hpp (refactor.hpp:14-172):
// the full multilevel decompose / recompose on the GPU (the library's fused
// level kernels, Thomas passes and pyramid assembly; host arrays move through
// the plan's cached device buffers -- pinned staging for pageable memory), the
// error report as a device reduction, and the class packing walk.
#pragma once

#include <cstddef>
#include <span>
#include <utility>
#include <vector>

#include "correction.hpp"
#include "error.hpp"
#include "grid_hierarchy.hpp"
#include "ndarray.hpp"
#include "transforms.hpp"

namespace HGR_B200_NAMESPACE {

/// In-place coefficient pyramid over the finest-shape array: class-l
/// coefficients at the nodes level l adds, corrected nodal values at the
/// coarsest nodes (class 0).
template <class T>
struct RefactoredArray {
  ndarray<T> data;
  GridHierarchy hierarchy;
  static constexpr std::size_t precision_bytes = sizeof(T);
};

/// Decompose (consumes `data`, like the reference's by-value parameter).
/// Finiteness is checked on the device before the array is overwritten.
template <class T>
RefactoredArray<T> decompose(ndarray<T> data, const GridHierarchy& g) {
  detail::require(data.extents() == g.finest_extents(), "decompose: array shape does not match grid");
  const hgr_grid_desc d = g.desc();
  if constexpr (detail::is_f64<T>()) detail::check(hgr_decompose_host_f64(&d, data.data()));
  else detail::check(hgr_decompose_host_f32(&d, data.data()));
  return {std::move(data), g};
}

/// Recompose classes 0..upto_class (absent classes read as zero).
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
  double l2_abs = 0;
  double l2_rel = 0;
  double linf_abs = 0;
  double linf_rel = 0;
};

/// L2 / Linf errors in double (refactor.hpp:100-120), reduced on the device.
template <class T>
ErrorReport error_report(const ndarray<T>& original, const ndarray<T>& reconstruction) {
  detail::require(original.extents() == reconstruction.extents(), "error_report: shape mismatch");
  double v[4] = {0, 0, 0, 0};
  if constexpr (detail::is_f64<T>())
    detail::check(hgr_error_report_host_f64(original.size(), original.data(), reconstruction.data(), v));
  else
    detail::check(hgr_error_report_host_f32(original.size(), original.data(), reconstruction.data(), v));
  return {v[0], v[1], v[2], v[3]};
}

/// One class's values in row-major order of its finest-grid indices.
template <class T>
struct CoefficientClass {
  int level = 0;
  std::vector<T> values;
};

namespace detail {

// The class order (refactor.hpp:134-145): row-major over the level-cls
// indices, skipping the all-even ones (already on level cls-1) for cls > 0.
template <class Array, class Fn>
void for_each_class_node(Array& data, const GridHierarchy& g, int cls, Fn&& fn) {
  const auto v = level_view(data, g, cls);
  for (std::size_t i0 = 0; i0 < v.shape[0]; ++i0)
    for (std::size_t i1 = 0; i1 < v.shape[1]; ++i1)
      for (std::size_t i2 = 0; i2 < v.shape[2]; ++i2)
        if (cls == 0 || ((i0 | i1 | i2) & 1u)) fn(v(i0, i1, i2));
}

}  // namespace detail

/// Host arrays are walked in place (a device pyramid uses
/// hgr_cuda_extract_class_* / _scatter_class_*).
template <class T>
CoefficientClass<T> extract_class(const RefactoredArray<T>& r, int cls) {
  CoefficientClass<T> out{cls, {}};
  out.values.reserve(r.hierarchy.class_node_count(cls));
  detail::for_each_class_node(r.data, r.hierarchy, cls, [&](const T& x) { out.values.push_back(x); });
  return out;
}

template <class T>
void scatter_class(RefactoredArray<T>& r, int cls, std::span<const T> values) {
  detail::require(values.size() == r.hierarchy.class_node_count(cls),
                  "scatter_class: value count does not match class size");
  std::size_t k = 0;
  detail::for_each_class_node(r.data, r.hierarchy, cls, [&](T& x) { x = values[k++]; });
}

template <class T>
void scatter_class(RefactoredArray<T>& r, int cls, const std::vector<T>& values) {
  scatter_class(r, cls, std::span<const T>(values));
}

}  // namespace HGR_B200_NAMESPACE
