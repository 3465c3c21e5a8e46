// tables.hpp -- host construction of the per-(level, dimension) operator
// tables, in the reference's precisions and arithmetic order. Shared by the
// plan (plan.cu) and the fiber-operator entry points (capi.cu), so the
// known-answer tests exercise the same builders as the hot path.
#pragma once

#include <cstddef>
#include <cmath>
#include <vector>

namespace hgrb {

// MassTransOperator<T> taps (correction.hpp:96-133), computed in T exactly as
// the reference does (spacings cast to T, refined_node_weights in T).
template <class T>
inline std::vector<T> masstrans_taps(const std::vector<T>& h) {
  const std::size_t nf = h.size() + 1, nc = (nf - 1) / 2 + 1;
  auto main_ = [&](std::size_t i) {
    const T left = i > 0 ? h[i - 1] : T(0);
    const T right = i + 1 < nf ? h[i] : T(0);
    return T(2) * (left + right);
  };
  auto mass_entry = [&](std::size_t t, std::size_t j) -> T {
    if (j == t) return main_(t);
    if (j + 1 == t) return h[t - 1];
    if (j == t + 1) return h[t];
    return T(0);
  };
  std::vector<T> taps(nc * 5, T(0));
  for (std::size_t i = 0; i < nc; ++i) {
    std::size_t rj[3];
    T rw[3];
    std::size_t rn = 0;
    if (i > 0) {
      const T span = h[2 * i - 2] + h[2 * i - 1];
      rj[rn] = 2 * i - 1;
      rw[rn++] = h[2 * i - 2] / span;  // to_right
    }
    rj[rn] = 2 * i;
    rw[rn++] = T(1);
    if (i + 1 < nc) {
      const T span = h[2 * i] + h[2 * i + 1];
      rj[rn] = 2 * i + 1;
      rw[rn++] = h[2 * i + 1] / span;  // to_left
    }
    for (std::size_t k = 0; k < 5; ++k) {
      const long j = long(2 * i) - 2 + long(k);
      if (j < 0 || j >= long(nf)) continue;
      T sum = T(0);
      for (std::size_t r = 0; r < rn; ++r) sum += rw[r] * mass_entry(rj[r], std::size_t(j));
      taps[i * 5 + k] = sum;
    }
  }
  return taps;
}

// ThomasSolver<T> factors (correction.hpp:188-198)
template <class T>
inline void thomas_factors(const std::vector<T>& h, std::vector<T>& mult, std::vector<T>& pivot,
                    std::vector<T>& upper, std::vector<T>& rpiv) {
  const std::size_t n = h.size() + 1;
  auto main_ = [&](std::size_t i) {
    const T left = i > 0 ? h[i - 1] : T(0);
    const T right = i + 1 < n ? h[i] : T(0);
    return T(2) * (left + right);
  };
  pivot.assign(n, T(0));
  mult.assign(n > 1 ? n - 1 : 1, T(0));
  upper.assign(n > 1 ? n - 1 : 1, T(0));
  rpiv.assign(n, T(0));
  for (std::size_t i = 0; i < n; ++i) pivot[i] = main_(i);
  for (std::size_t i = 0; i + 1 < n; ++i) upper[i] = h[i];
  for (std::size_t i = 1; i < n; ++i) {
    mult[i - 1] = h[i - 1] / pivot[i - 1];
    pivot[i] = main_(i) - mult[i - 1] * upper[i - 1];
  }
  for (std::size_t i = 0; i < n; ++i) rpiv[i] = T(1) / pivot[i];
}

// Lookahead bands of the streaming IPK passes (kernels_stream.cu, bands of
// kStreamBand positions): the smallest K such that the backward carry through
// any K consecutive bands -- the product of the factors u_i / p_i over their
// positions -- is below 2^-bits (56 fp64, 26 fp32), i.e. below rounding. The
// bound 1/2 per factor gives K = ceil(bits / 16); the actual factors of a grid
// (about 0.27 on uniform spacings) usually give less. Returns at least 1.
constexpr int kStreamBand = 16;
template <class T>
inline int stream_lookahead(const std::vector<T>& upper, const std::vector<T>& rpiv) {
  const double bits = sizeof(T) == 8 ? 56.0 : 26.0;
  const std::size_t n = rpiv.size();
  const std::size_t nb = (n + kStreamBand - 1) / kStreamBand;
  std::vector<double> d(nb, 0.0);  // -log2 of each band's carry factor
  for (std::size_t i = 0; i < n; ++i) {
    const double f = i + 1 < n ? std::fabs(double(upper[i]) * double(rpiv[i])) : 0.0;
    d[i / kStreamBand] += f > 0.0 ? -std::log2(f) : 1e300;
  }
  for (std::size_t K = 1; K + 1 < nb; ++K) {
    bool ok = true;
    for (std::size_t b = 1; b + K <= nb && ok; ++b) {  // bands b .. b+K-1 after a finished one
      double s = 0.0;
      for (std::size_t t = 0; t < K; ++t) s += d[b + t];
      ok = s >= bits;
    }
    if (ok) return int(K);
  }
  return int(nb > 1 ? nb - 1 : 1);
}

// Transfer weights in T (refined_node_weights<T>, correction.hpp:67-88): the
// weight of fine node 2q-1 (trl) / 2q+1 (trr) into coarse node q; 0 at the ends.
template <class T>
inline void transfer_weights(const std::vector<T>& h, std::vector<T>& trl, std::vector<T>& trr) {
  const std::size_t nc = h.size() / 2 + 1;
  trl.assign(nc, T(0));
  trr.assign(nc, T(0));
  for (std::size_t q = 0; q < nc; ++q) {
    if (q > 0) trl[q] = h[2 * q - 2] / (h[2 * q - 2] + h[2 * q - 1]);
    if (q + 1 < nc) trr[q] = h[2 * q + 1] / (h[2 * q] + h[2 * q + 1]);
  }
}

}  // namespace hgrb
