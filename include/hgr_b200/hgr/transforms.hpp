// hgr_b200/hgr/transforms.hpp -- drop-in for hgr/transforms.hpp
// (transforms.hpp:76-124): the single-level grid processing operators (GPK) on
// compact level arrays, run by the GPU library (host arrays are staged through
// the plan's device buffers; hgr_host_level_op_*, hgr_host_apply_coefficients_*).
#pragma once

#include <cstddef>
#include <string>
#include <vector>

#include "error.hpp"
#include "grid_hierarchy.hpp"
#include "ndarray.hpp"

namespace HGR_B200_NAMESPACE {
namespace detail {

template <class T>
void check_level_shape(const ndarray<T>& a, const GridHierarchy& g, int level, const char* what) {
  require(a.extents() == g.level_extents(level), std::string(what) + ": shape mismatch");
}

// op 0 interpolate_to_fine, 1 compute_coefficients, 2 compute_correction
template <class T>
ndarray<T> level_op(int op, const ndarray<T>& in, const GridHierarchy& g, int level, int out_level) {
  ndarray<T> out(g.level_extents(out_level));
  const hgr_grid_desc d = g.desc();
  if constexpr (is_f64<T>()) check(hgr_host_level_op_f64(&d, op, level, in.data(), out.data()));
  else check(hgr_host_level_op_f32(&d, op, level, in.data(), out.data()));
  return out;
}

}  // namespace detail

/// Coarse values copied through; refined nodes get the multilinear blend.
template <class T>
ndarray<T> interpolate_to_fine(const ndarray<T>& coarse, const GridHierarchy& g, int level) {
  detail::require(level >= 1 && level <= g.levels(), "level out of range");
  detail::check_level_shape(coarse, g, level - 1, "interpolate_to_fine");
  return detail::level_op(0, coarse, g, level, level);
}

/// Level-l data minus the interpolation of its own coarse restriction.
template <class T>
ndarray<T> compute_coefficients(const ndarray<T>& fine, const GridHierarchy& g, int level) {
  detail::require(level >= 1 && level <= g.levels(), "level out of range");
  detail::check_level_shape(fine, g, level, "compute_coefficients");
  return detail::level_op(1, fine, g, level, level);
}

/// Inverse of compute_coefficients: interpolation plus the coefficients.
template <class T>
ndarray<T> apply_coefficients(const ndarray<T>& coarse, const ndarray<T>& coeffs,
                              const GridHierarchy& g, int level) {
  detail::require(level >= 1 && level <= g.levels(), "level out of range");
  detail::check_level_shape(coarse, g, level - 1, "apply_coefficients");
  detail::check_level_shape(coeffs, g, level, "apply_coefficients");
  ndarray<T> fine(g.level_extents(level));
  const hgr_grid_desc d = g.desc();
  if constexpr (detail::is_f64<T>())
    detail::check(hgr_host_apply_coefficients_f64(&d, level, coarse.data(), coeffs.data(), fine.data()));
  else
    detail::check(hgr_host_apply_coefficients_f32(&d, level, coarse.data(), coeffs.data(), fine.data()));
  return fine;
}

}  // namespace HGR_B200_NAMESPACE
