// hgr_b200/hgr/correction.hpp -- drop-in for hgr/correction.hpp
// (correction.hpp:13-365): the linear processing (mass-trans, LPK) and
// iterative processing (Thomas, IPK) operators and the per-level correction.
// Operator tables come from the GPU library's own builders (hgr_masstrans_taps_*,
// hgr_thomas_factors_*, the ones its plans upload); applying an operator to
// fibers runs on the GPU (hgr_host_fiber_op_*: one batched launch per call, the
// fibers of a pass gathered into one contiguous batch). compute_correction runs
// the plan's level path.
#pragma once

#include <algorithm>
#include <array>
#include <cstddef>
#include <span>
#include <vector>

#include "error.hpp"
#include "grid_hierarchy.hpp"
#include "ndarray.hpp"
#include "parallel.hpp"

namespace HGR_B200_NAMESPACE {

namespace detail {

// fiber op codes of hgr_host_fiber_op_* (include/hgr_cuda.h)
enum FiberOp : int { kMass = 0, kMassTrans = 1, kThomas = 2, kTransfer = 3, kMassTransMasked = 4 };

template <class T>
void fiber_op(int op, std::size_t n, std::size_t count, const T* v, const T* h, T* out) {
  if constexpr (is_f64<T>()) check(hgr_host_fiber_op_f64(op, n, count, v, h, out));
  else check(hgr_host_fiber_op_f32(op, n, count, v, h, out));
}

template <class T>
std::vector<T> fiber_op(int op, std::span<const T> v, std::span<const T> h, std::size_t nout) {
  std::vector<T> out(nout);
  fiber_op<T>(op, v.size(), 1, v.data(), h.data(), out.data());
  return out;
}

}  // namespace detail

/// Tridiagonal operator of one grid line (lower[i-1], main[i], upper[i] of row
/// i). mass_matrix builds the reference's mass form (h_{i-1}, 2(h_{i-1}+h_i), h_i).
/// apply() is a host utility (the reference uses it in tests only); the device
/// operator is mass_apply.
template <class T>
struct TridiagonalOperator {
  std::vector<T> lower;
  std::vector<T> main;
  std::vector<T> upper;

  std::size_t size() const { return main.size(); }

  static TridiagonalOperator mass_matrix(std::span<const T> spacings) {
    detail::require(!spacings.empty(), "mass matrix needs at least one interval");
    const std::size_t n = spacings.size() + 1;
    TridiagonalOperator op;
    op.main.assign(n, T(0));
    op.lower.assign(spacings.begin(), spacings.end());
    op.upper.assign(spacings.begin(), spacings.end());
    for (std::size_t i = 0; i < n; ++i)
      op.main[i] = T(2) * ((i > 0 ? spacings[i - 1] : T(0)) + (i + 1 < n ? spacings[i] : T(0)));
    return op;
  }

  std::vector<T> apply(std::span<const T> v) const {
    detail::require(v.size() == size(), "tridiagonal apply: length mismatch");
    std::vector<T> out(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) {
      T acc = main[i] * v[i];
      if (i > 0) acc += lower[i - 1] * v[i - 1];
      if (i + 1 < v.size()) acc += upper[i] * v[i + 1];
      out[i] = acc;
    }
    return out;
  }
};

/// (Mv)_i with the mass matrix of spacings h, on the GPU.
template <class T>
std::vector<T> mass_apply(std::span<const T> v, std::span<const T> h) {
  detail::require(v.size() == h.size() + 1, "mass_apply: |v| must equal |h|+1");
  return detail::fiber_op<T>(detail::kMass, v, h, v.size());
}

/// Transpose of prolongation (R = P^T) on one fiber, on the GPU.
template <class T>
std::vector<T> transfer_apply(std::span<const T> v, std::span<const T> h) {
  detail::require(v.size() == h.size() + 1, "transfer_apply: |v| must equal |h|+1");
  detail::require(v.size() >= 3 && v.size() % 2 == 1, "transfer_apply: fine fiber length must be odd");
  return detail::fiber_op<T>(detail::kTransfer, v, h, (v.size() - 1) / 2 + 1);
}

/// K = R*M as a five-tap coarse-by-fine stencil (taps over fine 2i-2..2i+2),
/// built in T by the library's table builder.
template <class T>
class MassTransOperator {
 public:
  explicit MassTransOperator(std::span<const T> fine_spacings)
      : h_(fine_spacings.begin(), fine_spacings.end()) {
    detail::require(fine_spacings.size() >= 2 && fine_spacings.size() % 2 == 0,
                    "mass-trans: fine fiber length must be odd");
    nf_ = h_.size() + 1;
    nc_ = (nf_ - 1) / 2 + 1;
    taps_.resize(5 * nc_);
    if constexpr (detail::is_f64<T>()) detail::check(hgr_masstrans_taps_f64(nf_, h_.data(), taps_.data()));
    else detail::check(hgr_masstrans_taps_f32(nf_, h_.data(), taps_.data()));
  }

  std::size_t fine_size() const { return nf_; }
  std::size_t coarse_size() const { return nc_; }

  /// out_i = sum_k taps[i][k] * in_{2i-2+k} over one strided fiber; with
  /// zero_even_inputs, even fine indices read as zero.
  void apply_fiber(const T* in, std::size_t in_stride, bool zero_even_inputs, T* out,
                   std::size_t out_stride) const {
    std::vector<T> f(nf_), r(nc_);
    for (std::size_t j = 0; j < nf_; ++j) f[j] = in[j * in_stride];
    detail::fiber_op<T>(zero_even_inputs ? detail::kMassTransMasked : detail::kMassTrans, nf_, 1,
                        f.data(), h_.data(), r.data());
    for (std::size_t i = 0; i < nc_; ++i) out[i * out_stride] = r[i];
  }

  /// Dense row i over the fine fiber.
  std::vector<T> row(std::size_t i) const {
    std::vector<T> r(nf_, T(0));
    for (std::size_t k = 0; k < 5; ++k) {
      const std::ptrdiff_t j = std::ptrdiff_t(2 * i) - 2 + std::ptrdiff_t(k);
      if (j >= 0 && j < std::ptrdiff_t(nf_)) r[std::size_t(j)] = taps_[5 * i + k];
    }
    return r;
  }

  const std::vector<T>& spacings() const { return h_; }

 private:
  std::vector<T> h_;
  std::vector<T> taps_;  // 5 per coarse row
  std::size_t nf_ = 0;
  std::size_t nc_ = 0;
};

template <class T>
std::vector<T> masstrans_apply(std::span<const T> v, std::span<const T> h) {
  detail::require(v.size() == h.size() + 1, "masstrans_apply: |v| must equal |h|+1");
  detail::require(v.size() >= 3 && v.size() % 2 == 1, "mass-trans: fine fiber length must be odd");
  return detail::fiber_op<T>(detail::kMassTrans, v, h, (v.size() - 1) / 2 + 1);
}

/// Tridiagonal solve with the mass matrix of one line: forward elimination and
/// back substitution with the factors of correction.hpp:188-198, on the GPU.
template <class T>
class ThomasSolver {
 public:
  explicit ThomasSolver(std::span<const T> spacings) : h_(spacings.begin(), spacings.end()) {
    detail::require(!spacings.empty(), "mass matrix needs at least one interval");
    const std::size_t n = h_.size() + 1;
    mult_.resize(n - 1);
    pivot_.resize(n);
    upper_.resize(n - 1);
    if constexpr (detail::is_f64<T>())
      detail::check(hgr_thomas_factors_f64(n, h_.data(), mult_.data(), pivot_.data(), upper_.data()));
    else
      detail::check(hgr_thomas_factors_f32(n, h_.data(), mult_.data(), pivot_.data(), upper_.data()));
  }

  std::size_t size() const { return pivot_.size(); }

  void solve_fiber(T* x, std::size_t stride) const {
    const std::size_t n = size();
    std::vector<T> f(n), r(n);
    for (std::size_t i = 0; i < n; ++i) f[i] = x[i * stride];
    detail::fiber_op<T>(detail::kThomas, n, 1, f.data(), h_.data(), r.data());
    for (std::size_t i = 0; i < n; ++i) x[i * stride] = r[i];
  }

  const std::vector<T>& spacings() const { return h_; }
  const std::vector<T>& pivots() const { return pivot_; }
  const std::vector<T>& multipliers() const { return mult_; }

 private:
  std::vector<T> h_;
  std::vector<T> mult_, pivot_, upper_;
};

/// Solves mass(h) z = rhs.
template <class T>
std::vector<T> thomas_solve(std::span<const T> rhs, std::span<const T> h) {
  detail::require(rhs.size() == h.size() + 1, "thomas_solve: |rhs| must equal |h|+1");
  return detail::fiber_op<T>(detail::kThomas, rhs, h, rhs.size());
}

namespace detail {

template <class T>
std::vector<T> spacings_as(const GridHierarchy& g, int level, int d) {
  const auto& h = g.spacings(level, d);
  return std::vector<T>(h.begin(), h.end());
}

// the two fiber axes of a pass along `dim` (the reference's a/b, correction.hpp:241-242)
inline void fiber_axes(int dim, int& a, int& b) {
  a = dim == 0 ? 1 : 0;
  b = dim == 2 ? 1 : 2;
}

// Mass-trans pass along `dim` (correction.hpp:238-260): every fiber of `in`
// gathered into one batch, one GPU launch, results scattered into `out`. With
// `mask`, fibers whose other two indices are even read their even entries as 0.
template <class T>
void masstrans_pass(const MassTransOperator<T>& op, ndview<const T> in, ndview<T> out, int dim,
                    bool mask) {
  int a, b;
  fiber_axes(dim, a, b);
  const std::size_t na = in.shape[std::size_t(a)], nb = in.shape[std::size_t(b)];
  const std::size_t nf = op.fine_size(), nc = op.coarse_size(), fibers = na * nb;
  require(in.shape[std::size_t(dim)] == nf && out.shape[std::size_t(dim)] == nc,
          "mass-trans pass: fiber length mismatch");
  std::vector<T> batch(fibers * nf), res(fibers * nc);
  for (std::size_t f = 0; f < fibers; ++f) {
    const std::size_t ia = f / nb, ib = f % nb;
    const bool zero_even = mask && ia % 2 == 0 && ib % 2 == 0;
    const T* src = in.ptr + ia * in.stride[std::size_t(a)] + ib * in.stride[std::size_t(b)];
    for (std::size_t j = 0; j < nf; ++j)
      batch[f * nf + j] = (zero_even && j % 2 == 0) ? T(0) : src[j * in.stride[std::size_t(dim)]];
  }
  fiber_op<T>(kMassTrans, nf, fibers, batch.data(), op.spacings().data(), res.data());
  for (std::size_t f = 0; f < fibers; ++f) {
    const std::size_t ia = f / nb, ib = f % nb;
    T* dst = out.ptr + ia * out.stride[std::size_t(a)] + ib * out.stride[std::size_t(b)];
    for (std::size_t i = 0; i < nc; ++i) dst[i * out.stride[std::size_t(dim)]] = res[f * nc + i];
  }
}

// Thomas pass along `dim` (correction.hpp:262-278), batched the same way.
template <class T>
void thomas_pass(const ThomasSolver<T>& solver, ndview<T> data, int dim) {
  int a, b;
  fiber_axes(dim, a, b);
  const std::size_t na = data.shape[std::size_t(a)], nb = data.shape[std::size_t(b)];
  const std::size_t n = solver.size(), fibers = na * nb;
  require(data.shape[std::size_t(dim)] == n, "thomas pass: line length mismatch");
  std::vector<T> batch(fibers * n), res(fibers * n);
  auto base = [&](std::size_t f) {
    return data.ptr + (f / nb) * data.stride[std::size_t(a)] + (f % nb) * data.stride[std::size_t(b)];
  };
  for (std::size_t f = 0; f < fibers; ++f)
    for (std::size_t i = 0; i < n; ++i) batch[f * n + i] = base(f)[i * data.stride[std::size_t(dim)]];
  fiber_op<T>(kThomas, n, fibers, batch.data(), solver.spacings().data(), res.data());
  for (std::size_t f = 0; f < fibers; ++f)
    for (std::size_t i = 0; i < n; ++i) base(f)[i * data.stride[std::size_t(dim)]] = res[f * n + i];
}

/// Scratch elements correction_level needs beyond its output (correction.hpp:281-289):
/// the stages after the first (and, in 3D, second) mass-trans pass.
inline std::size_t correction_workspace_elements(const GridHierarchy& g, int level) {
  if (g.rank() == 1) return 0;
  const auto f = padded_extents(g.level_extents(level));
  const auto c = padded_extents(g.level_extents(level - 1));
  return c[0] * f[1] * f[2] + (g.rank() == 3 ? c[0] * c[1] * f[2] : 0);
}

// correction_level (correction.hpp:295-340): mass-trans passes in ascending
// dimension order (mask on the first), the last one into `out`, then Thomas
// passes in ascending order on `out`; each pass one batched GPU launch.
template <class T>
void correction_level(ndview<const T> fine, bool mask, const GridHierarchy& g, int level,
                      ndarray<T>& out, std::vector<T>& workspace) {
  const int rank = g.rank();
  require(out.extents() == g.level_extents(level - 1), "correction output shape mismatch");
  workspace.resize(std::max(workspace.size(), correction_workspace_elements(g, level)));
  std::vector<std::size_t> ext = g.level_extents(level);
  const std::vector<std::size_t> cext = g.level_extents(level - 1);
  ndview<const T> cur = fine;
  std::size_t used = 0;
  for (int d = 0; d < rank; ++d) {
    ext[std::size_t(d)] = cext[std::size_t(d)];
    ndview<T> dst = d == rank - 1 ? full_view(out)
                                  : ndview<T>{workspace.data() + used, padded_extents(ext),
                                              natural_strides(ext)};
    if (d < rank - 1) used += ndarray<T>::count_of(ext);
    const auto h = spacings_as<T>(g, level, d);
    masstrans_pass(MassTransOperator<T>(std::span<const T>(h)), cur, dst, d, mask && d == 0);
    cur = as_const(dst);
  }
  for (int d = 0; d < rank; ++d) {
    const auto h = spacings_as<T>(g, level - 1, d);
    thomas_pass(ThomasSolver<T>(std::span<const T>(h)), full_view(out), d);
  }
}

}  // namespace detail

/// L2 projection of the level-l coefficients onto level l-1 (the plan's fused
/// level path). Coefficients at coarse positions must be zero.
template <class T>
ndarray<T> compute_correction(const ndarray<T>& coeffs, const GridHierarchy& g, int level) {
  detail::require(level >= 1 && level <= g.levels(), "level out of range");
  detail::require(coeffs.extents() == g.level_extents(level), "compute_correction: shape mismatch");
  ndarray<T> z(g.level_extents(level - 1));
  const hgr_grid_desc d = g.desc();
  if constexpr (detail::is_f64<T>()) detail::check(hgr_host_level_op_f64(&d, 2, level, coeffs.data(), z.data()));
  else detail::check(hgr_host_level_op_f32(&d, 2, level, coeffs.data(), z.data()));
  return z;
}

}  // namespace HGR_B200_NAMESPACE
