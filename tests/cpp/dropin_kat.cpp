// dropin_kat.cpp -- the reference's known-answer and property checks, written
// against the C++ drop-in (include/hgr_b200/hgr.hpp) exactly as a reference
// caller would use the API (namespace hgr, same types and signatures). Built
// and run by tests/test_dropin_cpp.py; prints one PASS/FAIL line per check.
#include <hgr_b200/hgr.hpp>

#include <cmath>
#include <cstdio>
#include <cstdint>
#include <functional>
#include <limits>
#include <string>
#include <thread>
#include <vector>

using hgr::GridHierarchy;
using hgr::ndarray;

static int failures = 0;

static void check(const char* name, const std::function<bool()>& body) {
  bool ok = false;
  std::string note;
  try {
    ok = body();
  } catch (const std::exception& e) {
    note = e.what();
  }
  std::printf("%s  %s%s%s\n", ok ? "PASS" : "FAIL", name, note.empty() ? "" : " -- ", note.c_str());
  if (!ok) ++failures;
}

template <class Fn>
static bool throws_with(Fn&& fn, const char* substr) {
  try {
    fn();
  } catch (const hgr::error& e) {
    return std::string(e.what()).find(substr) != std::string::npos;
  }
  return false;
}

// deterministic values in [-1, 1)
template <class T>
static std::vector<T> values(std::size_t n, std::uint64_t seed) {
  std::vector<T> v(n);
  std::uint64_t s = seed * 0x9E3779B97F4A7C15ull + 1;
  for (auto& x : v) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    x = static_cast<T>(double(s >> 11) * 0x1.0p-53 * 2.0 - 1.0);
  }
  return v;
}

template <class T>
static double rel_linf(const ndarray<T>& a, const ndarray<T>& b) {
  double d = 0, s = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    d = std::max(d, std::abs(double(a[i]) - double(b[i])));
    s = std::max(s, std::abs(double(a[i])));
  }
  return s > 0 ? d / s : d;
}

int main() {
  // test_refactor.cpp:31-46
  check("decompose sampled quadratic [6,2,0,0,2] -> [3.5,-1,-4,-1,-0.5]", [] {
    auto g = GridHierarchy::uniform({5});
    auto r = hgr::decompose(ndarray<double>({5}, {6, 2, 0, 0, 2}), g);
    const double want[5] = {3.5, -1, -4, -1, -0.5};
    for (int i = 0; i < 5; ++i)
      if (std::abs(r.data[i] - want[i]) > 1e-14 * 4) return false;
    auto c2 = hgr::extract_class(r, 2);
    if (c2.values != std::vector<double>{-1, -1}) return false;
    auto back = hgr::recompose(r, 2);
    return rel_linf(ndarray<double>({5}, {6, 2, 0, 0, 2}), back) <= 1e-12;
  });
  // test_transforms.cpp:30-59, 78-111
  check("interpolate [6,0,2] -> [6,3,0,1,2]", [] {
    GridHierarchy g({{0, 1, 2, 3, 4}});
    return hgr::interpolate_to_fine(ndarray<double>({3}, {6, 0, 2}), g, 2).values() ==
           std::vector<double>{6, 3, 0, 1, 2};
  });
  check("nonuniform weight -> 1", [] {
    GridHierarchy g({{0, 1, 3}});
    return std::abs(hgr::interpolate_to_fine(ndarray<double>({2}, {0, 3}), g, 1)[1] - 1.0) <= 1e-15;
  });
  check("coefficients of the quadratic [0,-1,0,-1,0]", [] {
    GridHierarchy g({{0, 1, 2, 3, 4}});
    return hgr::compute_coefficients(ndarray<double>({5}, {6, 2, 0, 0, 2}), g, 2).values() ==
           std::vector<double>{0, -1, 0, -1, 0};
  });
  check("2D bump coefficient", [] {
    auto g = GridHierarchy::uniform({3, 3});
    ndarray<double> d({3, 3}, {0, 0, 0, 0, 1, 0, 0, 0, 0});
    return hgr::compute_coefficients(d, g, 1).values() == d.values();
  });
  check("apply_coefficients inverts compute_coefficients", [] {
    GridHierarchy g({{0, 1, 2, 3, 4}});
    auto f = hgr::apply_coefficients(ndarray<double>({3}, {6, 0, 2}),
                                     ndarray<double>({5}, {0, -1, 0, -1, 0}), g, 2);
    return f.values() == std::vector<double>{6, 2, 0, 0, 2};
  });
  // test_correction.cpp:35-68, 109-175
  check("mass / mass-trans / Thomas known answers", [] {
    std::vector<double> h{1, 1, 1, 1}, c{0, -1, 0, -1, 0}, ones{1, 1, 1, 1, 1};
    if (hgr::mass_apply<double>(ones, h) != std::vector<double>{3, 6, 6, 6, 3}) return false;
    if (hgr::masstrans_apply<double>(c, h) != std::vector<double>{-3, -6, -3}) return false;
    std::vector<double> h2{2, 2}, rhs{-3, -6, -3};
    auto z = hgr::thomas_solve<double>(rhs, h2);
    for (double v : z)
      if (std::abs(v + 0.5) > 1e-14) return false;
    return true;
  });
  check("correction of the quadratic = -0.5 ; 2D separable = 0.25", [] {
    auto g = GridHierarchy::uniform({5});
    auto z = hgr::compute_correction(ndarray<double>({5}, {0, -1, 0, -1, 0}), g, 2);
    for (std::size_t i = 0; i < 3; ++i)
      if (std::abs(z[i] + 0.5) > 1e-14) return false;
    auto g2 = GridHierarchy::uniform({5, 5});
    ndarray<double> c2({5, 5});
    const double c1[5] = {0, -1, 0, -1, 0};
    for (int i = 0; i < 5; ++i)
      for (int j = 0; j < 5; ++j) c2[i * 5 + j] = c1[i] * c1[j];
    auto z2 = hgr::compute_correction(c2, g2, 2);
    for (std::size_t i = 0; i < 9; ++i)
      if (std::abs(z2[i] - 0.25) > 1e-13) return false;
    return true;
  });
  check("nonzero coarse entries rejected ('zero at coarse')", [] {
    auto g = GridHierarchy::uniform({5});
    return throws_with([&] { hgr::compute_correction(ndarray<double>({5}, {1, -1, 0, -1, 0}), g, 2); },
                       "zero at coarse");
  });
  // test_refactor.cpp:101-126 round trips
  check("round trip double 17^3 <= 1e-12", [] {
    auto g = GridHierarchy::uniform({17, 17, 17});
    ndarray<double> d(g.finest_extents(), values<double>(17 * 17 * 17, 1));
    return rel_linf(d, hgr::recompose(hgr::decompose(d, g), g.levels())) <= 1e-12;
  });
  check("round trip float 65^3 <= 1e-5", [] {
    auto g = GridHierarchy::uniform({65, 65, 65});
    ndarray<float> d(g.finest_extents(), values<float>(65 * 65 * 65, 2));
    return rel_linf(d, hgr::recompose(hgr::decompose(d, g), g.levels())) <= 1e-5;
  });
  check("round trip double nonuniform 33x17 <= 1e-12", [] {
    std::vector<double> a(33), b(17);
    for (std::size_t i = 0; i < 33; ++i) a[i] = std::expm1(2.0 * i / 32) / std::expm1(2.0);
    for (std::size_t i = 0; i < 17; ++i) b[i] = i * i + i;
    GridHierarchy g({a, b});
    ndarray<double> d(g.finest_extents(), values<double>(33 * 17, 3));
    return rel_linf(d, hgr::recompose(hgr::decompose(d, g), g.levels())) <= 1e-12;
  });
  // test_refactor.cpp:159-172 prefix bit identity
  check("reconstruction depends only on the class prefix (bitwise)", [] {
    auto g = GridHierarchy::uniform({17, 17});
    auto r = hgr::decompose(ndarray<double>(g.finest_extents(), values<double>(289, 4)), g);
    for (int m = 0; m <= g.levels(); ++m) {
      auto direct = hgr::recompose(r, m);
      auto zeroed = r;
      for (int cls = m + 1; cls <= g.levels(); ++cls)
        hgr::scatter_class(zeroed, cls, std::vector<double>(g.class_node_count(cls), 0.0));
      if (!(direct.values() == hgr::recompose(zeroed, m).values())) return false;
    }
    return true;
  });
  check("class counts follow the dyadic ladder", [] {
    return GridHierarchy::uniform({513}).class_count() == 10 &&
           GridHierarchy::uniform({513, 513, 513}).class_count() == 10 &&
           GridHierarchy::uniform({33, 33, 33}).class_count() == 6;
  });
  check("two-node passthrough", [] {
    GridHierarchy g({{0.0, 1.0}});
    auto r = hgr::decompose(ndarray<double>({2}, {3.5, -1.25}), g);
    return r.data.values() == std::vector<double>{3.5, -1.25} &&
           hgr::recompose(r, 0).values() == std::vector<double>{3.5, -1.25};
  });
  // test_refactor.cpp:250-259, test_grid_hierarchy.cpp:27-35
  check("validation messages", [] {
    auto g = GridHierarchy::uniform({5});
    const double nan = std::numeric_limits<double>::quiet_NaN();
    bool ok = throws_with([&] { hgr::decompose(ndarray<double>({5}, {0, 1, nan, 3, 4}), g); },
                          "non-finite");
    ok = ok && throws_with([&] { GridHierarchy::uniform({6}); }, "2^k+1");
    auto r = hgr::decompose(ndarray<double>({5}, {1, 2, 3, 4, 5}), g);
    ok = ok && throws_with([&] { hgr::recompose(r, 3); }, "class index out of range");
    ok = ok && throws_with([&] { hgr::decompose(ndarray<double>({4}), g); }, "shape");
    return ok;
  });
  check("error report norms", [] {
    ndarray<double> a({2}, {1, 1}), b({2}, {1, 0});
    auto rep = hgr::error_report(a, b);
    return rep.linf_abs == 1.0 && rep.l2_abs == 1.0 && std::abs(rep.l2_rel - 1 / std::sqrt(2.0)) < 1e-15;
  });
  // test_correction.cpp:35-107: the operator classes of the drop-in
  check("TridiagonalOperator::mass_matrix apply [1,1,1,1,1] -> [3,6,6,6,3]", [] {
    std::vector<double> h{1, 1, 1, 1};
    auto m = hgr::TridiagonalOperator<double>::mass_matrix(h);
    return m.size() == 5 && m.apply(std::vector<double>{1, 1, 1, 1, 1}) == std::vector<double>{3, 6, 6, 6, 3} &&
           m.apply(std::vector<double>{0, -1, 0, -1, 0}) == std::vector<double>{-1, -4, -2, -4, -1};
  });
  check("mass_apply float [0,-1,0,-1,0] -> [-1,-4,-2,-4,-1]", [] {
    std::vector<float> h{1, 1, 1, 1}, c{0, -1, 0, -1, 0};
    return hgr::mass_apply<float>(c, h) == std::vector<float>{-1, -4, -2, -4, -1};
  });
  check("transfer_apply -> [-0.5,-1,-0.5]; h=[1,2] [0,3,0] -> [2,1]", [] {
    std::vector<double> h{1, 1, 1, 1}, c{0, -1, 0, -1, 0};
    if (hgr::transfer_apply<double>(c, h) != std::vector<double>{-0.5, -1, -0.5}) return false;
    std::vector<double> h2{1, 2}, v{0, 3, 0};
    auto t = hgr::transfer_apply<double>(v, h2);
    return std::abs(t[0] - 2) < 1e-15 && std::abs(t[1] - 1) < 1e-15 &&
           hgr::transfer_apply<float>(std::vector<float>{0, -1, 0, -1, 0}, std::vector<float>{1, 1, 1, 1}) ==
               std::vector<float>{-0.5f, -1, -0.5f};
  });
  check("transfer_apply rejects even fibers", [] {
    std::vector<double> h{1, 1, 1}, v{1, 2, 3, 4};
    return throws_with([&] { hgr::transfer_apply<double>(v, h); }, "odd");
  });
  check("MassTransOperator row 0 = [2.5,3,0.5,0,0]; apply_fiber masked/strided", [] {
    std::vector<double> h{1, 1, 1, 1};
    hgr::MassTransOperator<double> op{std::span<const double>(h)};
    if (op.fine_size() != 5 || op.coarse_size() != 3) return false;
    if (op.row(0) != std::vector<double>{2.5, 3, 0.5, 0, 0}) return false;
    // strided fiber (stride 2) with the even entries masked == the coefficient-only product
    std::vector<double> in{7, 0, -1, 0, 9, 0, -1, 0, 5, 0}, out(6, 0.0);
    op.apply_fiber(in.data(), 2, true, out.data(), 2);
    return out[0] == -3 && out[2] == -6 && out[4] == -3 && out[1] == 0;
  });
  check("ThomasSolver solve_fiber h=[2,2] [-3,-6,-3] -> -0.5 (strided)", [] {
    std::vector<double> h{2, 2};
    hgr::ThomasSolver<double> t{std::span<const double>(h)};
    std::vector<double> x{-3, 1, -6, 1, -3, 1};
    t.solve_fiber(x.data(), 2);
    return t.size() == 3 && std::abs(x[0] + 0.5) < 1e-15 && std::abs(x[2] + 0.5) < 1e-15 &&
           std::abs(x[4] + 0.5) < 1e-15 && x[1] == 1;
  });
  check("correction_workspace_elements (test_correction.cpp:297)", [] {
    using hgr::detail::correction_workspace_elements;
    auto g3 = GridHierarchy::uniform({9, 17, 33});
    auto g1 = GridHierarchy::uniform({33});
    return correction_workspace_elements(g3, 3) == 5u * 17 * 33 + 5u * 9 * 33 &&
           correction_workspace_elements(g1, 2) == 0;
  });
  check("detail::correction_level (batched fiber passes) == compute_correction", [] {
    std::vector<double> a(17), b(9), c(17);
    for (std::size_t i = 0; i < 17; ++i) a[i] = i + 0.01 * i * i, c[i] = 2.0 * i + std::sin(double(i));
    for (std::size_t i = 0; i < 9; ++i) b[i] = i * i + i;
    GridHierarchy g({a, b, c});
    const int l = g.levels();
    auto d = ndarray<double>(g.finest_extents(), values<double>(17 * 9 * 17, 5));
    auto coef = hgr::compute_coefficients(d, g, l);
    auto z1 = hgr::compute_correction(coef, g, l);
    ndarray<double> z2(g.level_extents(l - 1));
    std::vector<double> ws;
    hgr::detail::correction_level(hgr::as_const(hgr::full_view(coef)), true, g, l, z2, ws);
    double diff = 0, sc = 0;
    for (std::size_t i = 0; i < z1.size(); ++i)
      diff = std::max(diff, std::abs(z1[i] - z2[i])), sc = std::max(sc, std::abs(z1[i]));
    return ws.size() >= hgr::detail::correction_workspace_elements(g, l) && diff <= 1e-13 * sc;
  });
  check("concurrent decompose of distinct arrays on one grid == serial (bitwise)", [] {
    auto g = GridHierarchy::uniform({33, 33, 65});
    std::vector<ndarray<double>> in;
    for (int t = 0; t < 4; ++t) in.emplace_back(g.finest_extents(), values<double>(33 * 33 * 65, 10 + t));
    std::vector<ndarray<double>> serial, par(4);
    for (int t = 0; t < 4; ++t) serial.push_back(hgr::decompose(in[std::size_t(t)], g).data);
    for (int rep = 0; rep < 3; ++rep) {
      std::vector<std::thread> th;
      for (int t = 0; t < 4; ++t)
        th.emplace_back([&, t] { par[std::size_t(t)] = hgr::decompose(in[std::size_t(t)], g).data; });
      for (auto& x : th) x.join();
      for (int t = 0; t < 4; ++t)
        if (!(par[std::size_t(t)] == serial[std::size_t(t)])) return false;
    }
    return true;
  });
  check("device error_report (float) matches the definition", [] {
    ndarray<float> a({4}, {1, -2, 3, 4}), b({4}, {1, -2, 2.5f, 4});
    auto rep = hgr::error_report(a, b);
    return rep.linf_abs == 0.5 && rep.linf_rel == 0.125 && std::abs(rep.l2_abs - 0.5) < 1e-15;
  });
  std::printf("%d failure(s)\n", failures);
  return failures == 0 ? 0 : 1;
}
