// ref_storage_on_dropin.cpp -- an unmodified reference translation unit on top
// of the drop-in. The reference's own storage.hpp (passed in as HGR_REF_STORAGE,
// /root/reference/proj/include/hgr/storage.hpp) is compiled against the drop-in
// headers (-I include/hgr_b200): its `#include "hgr/refactor.hpp"` resolves to
// the drop-in, so its write_file / read_prefix run on pyramids produced by the
// GPU decompose. Checks (one PASS/FAIL line each):
//  * the reference writer's file is byte-identical to the GPU writer's
//    (hgr_write_hg_host_f64, C ABI) for the same pyramid;
//  * read_prefix of every class count + GPU recompose reproduces the input
//    (full prefix) and matches the GPU recompose of the in-memory prefix;
//  * read_info accounting (header + class bytes = file size).
// Built by __graft_entry__.build() while /root/reference exists (the binary
// travels to the GPU box); run by tests/test_dropin_cpp.py.
#include "hgr/refactor.hpp"
#include HGR_REF_STORAGE

#include <cmath>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

static int failures = 0;

static void report(const char* name, bool ok, const std::string& note = "") {
  std::printf("%s  %s%s%s\n", ok ? "PASS" : "FAIL", name, note.empty() ? "" : " -- ", note.c_str());
  if (!ok) ++failures;
}

static std::vector<char> slurp(const std::string& p) {
  std::ifstream is(p, std::ios::binary);
  return {std::istreambuf_iterator<char>(is), {}};
}

template <class T>
static void run(const std::vector<std::size_t>& shape, bool nonuniform, const std::string& dir,
                double tol) {
  std::vector<std::vector<double>> coords(shape.size());
  for (std::size_t d = 0; d < shape.size(); ++d) {
    double x = 0;
    for (std::size_t i = 0; i < shape[d]; ++i) {
      coords[d].push_back(x);
      x += nonuniform ? 0.2 + 1.6 * std::fmod(0.6180339887 * double(i * (d + 3) + 1), 1.0) : 1.0;
    }
  }
  hgr::GridHierarchy g(coords);
  hgr::ndarray<T> u(shape);
  for (std::size_t i = 0; i < u.size(); ++i)
    u[i] = T(std::sin(0.013 * double(i)) + 0.25 * std::cos(0.0007 * double(i * i % 10007)));
  const std::string tag = std::to_string(shape.size()) + "d_" + (sizeof(T) == 8 ? "f64" : "f32") +
                          (nonuniform ? "_nu" : "");
  auto r = hgr::decompose(u, g);  // GPU

  const std::string ref_path = dir + "/ref_" + tag + ".hg", gpu_path = dir + "/gpu_" + tag + ".hg";
  const std::uint64_t nref = hgr::write_file(r, ref_path);  // the reference's writer
  std::uint64_t ngpu = 0;
  const hgr_grid_desc d = g.desc();
  int rc = sizeof(T) == 8
               ? hgr_write_hg_host_f64(gpu_path.c_str(), &d, reinterpret_cast<const double*>(r.data.data()), &ngpu)
               : hgr_write_hg_host_f32(gpu_path.c_str(), &d, reinterpret_cast<const float*>(r.data.data()), &ngpu);
  report(("write_file byte-identical " + tag).c_str(),
         rc == 0 && nref == ngpu && slurp(ref_path) == slurp(gpu_path),
         rc ? hgr_cuda_last_error() : "");

  const auto info = hgr::read_info(ref_path);
  std::uint64_t total = info.header_bytes;
  for (const auto& c : info.classes) total += c.bytes;
  report(("read_info accounting " + tag).c_str(), total == nref && info.file_bytes == nref &&
                                                       info.class_count() == g.class_count());

  for (int m = 0; m <= g.levels(); ++m) {
    auto pr = hgr::read_prefix<T>(ref_path, m);  // the reference's reader
    std::uint64_t expect = info.header_bytes;
    for (int c = 0; c <= m; ++c) expect += info.classes[std::size_t(c)].bytes;
    const auto back = hgr::recompose(pr.array, m);  // GPU
    const auto direct = hgr::recompose(r, m);
    double diff = 0, scale = 0;
    for (std::size_t i = 0; i < back.size(); ++i) {
      diff = std::fmax(diff, std::fabs(double(back[i]) - double(direct[i])));
      scale = std::fmax(scale, std::fabs(double(u[i])));
    }
    const bool exact = diff == 0.0;
    report(("read_prefix+recompose " + tag + " m=" + std::to_string(m)).c_str(),
           pr.bytes_read == expect && exact, "max diff " + std::to_string(diff));
    if (m == g.levels()) {
      const auto rep = hgr::error_report(u, back);
      report(("round trip " + tag).c_str(), rep.linf_rel <= tol,
             "linf_rel " + std::to_string(rep.linf_rel));
    }
  }
}

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : "/tmp";
  run<double>({65, 33, 129}, false, dir, 1e-12);
  run<double>({129, 65}, true, dir, 1e-12);
  run<float>({33, 65, 65}, true, dir, 1e-5);
  run<double>({1025}, false, dir, 1e-12);
  std::printf("%d failure(s)\n", failures);
  return failures ? 1 : 0;
}
