// hgr_b200_cli.cpp -- command-line front end on the GPU path, mirroring the
// reference CLI (tools/hgr_main.cpp:290-378): the same subcommands, flags,
// human and --json reports (compact, sorted keys, like nlohmann::json::dump)
// and exit codes (0 ok, 1 usage error, 2 data or format error). Refactoring
// runs on the B200 through the C ABI (include/hgr_cuda.h); the .hg files are
// byte-identical to the reference's.
//
//   hgr-b200 decompose --input RAW --dims n0[,n1[,n2]] [--precision f32|f64]
//                      [--coords-file F ...] [--uniform] --output HG [--json]
//   hgr-b200 recompose --input HG --classes K --output RAW [--json]
//   hgr-b200 info --input HG [--json]
//   hgr-b200 error --original RAW --reconstruction RAW [--precision f32|f64] [--json]
//   hgr-b200 rank-configs [--n N] [--bytes-per-element B] [--transaction-bytes S]
//                         [--ghost G] [--peak-bw BW] [--kernel gpk|lpk|ipk|all]
//                         [--configs FILE] [--top K] [--json]
//     (the paper's analytical launch-configuration cost model, perf_model.hpp:71-162;
//      host arithmetic, kept so the reference's CLI surface is complete)
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iostream>
#include <iterator>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hgr_cuda.h"

namespace {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void require(bool ok, const std::string& what) {
  if (!ok) throw DataError(what);
}
void check(int rc) {
  if (rc != HGR_OK) throw DataError(hgr_cuda_last_error());
}
void cuda(cudaError_t e) {
  if (e != cudaSuccess) throw DataError(std::string("CUDA error: ") + cudaGetErrorString(e));
}

// ---- JSON (nlohmann::json::dump formatting: sorted keys, no spaces) --------------
std::string jnum(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".e") == std::string::npos) s += ".0";
  return s;
}
std::string jstr(const std::string& v) {
  std::string o = "\"";
  for (char c : v) {
    if (c == '"' || c == '\\') {
      o += '\\';
      o += c;
    } else if (static_cast<unsigned char>(c) < 0x20) {
      char b[8];
      std::snprintf(b, sizeof b, "\\u%04x", c);
      o += b;
    } else {
      o += c;
    }
  }
  return o + "\"";
}
struct Json {
  std::map<std::string, std::string> kv;
  void set(const std::string& k, const std::string& raw) { kv[k] = raw; }
  void str(const std::string& k, const std::string& v) { kv[k] = jstr(v); }
  void u64(const std::string& k, uint64_t v) { kv[k] = std::to_string(v); }
  void i64(const std::string& k, long long v) { kv[k] = std::to_string(v); }
  void dbl(const std::string& k, double v) { kv[k] = jnum(v); }
  void arr(const std::string& k, const std::vector<uint64_t>& v) {
    std::string s = "[";
    for (std::size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
    kv[k] = s + "]";
  }
  std::string dump() const {
    std::string s = "{";
    bool first = true;
    for (const auto& [k, v] : kv) {
      s += (first ? "" : ",") + jstr(k) + ":" + v;
      first = false;
    }
    return s + "}";
  }
};

// ---- argument parsing --------------------------------------------------------------
struct Args {
  std::map<std::string, std::vector<std::string>> opt;
  std::map<std::string, bool> flag;
};

Args parse(int argc, char** argv, int first, const std::vector<std::string>& options,
           const std::vector<std::string>& flags) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string t = argv[i];
    std::string val;
    bool has_val = false;
    if (auto eq = t.find('='); t.rfind("--", 0) == 0 && eq != std::string::npos) {
      val = t.substr(eq + 1);
      t = t.substr(0, eq);
      has_val = true;
    }
    bool is_opt = false, is_flag = false;
    for (const auto& o : options) is_opt |= t == o;
    for (const auto& f : flags) is_flag |= t == f;
    if (is_flag && !has_val) {
      a.flag[t] = true;
    } else if (is_opt) {
      if (!has_val) {
        if (i + 1 >= argc) throw UsageError(t + " requires an argument");
        val = argv[++i];
      }
      a.opt[t].push_back(val);
    } else {
      throw UsageError("the following argument was not expected: " + t);
    }
  }
  return a;
}

std::string one(const Args& a, const std::string& k, const std::string& dflt = "",
                bool required = true) {
  auto it = a.opt.find(k);
  if (it == a.opt.end()) {
    if (required) throw UsageError(k + " is required");
    return dflt;
  }
  if (it->second.size() != 1) throw UsageError(k + " given more than once");
  return it->second.front();
}

std::vector<char> read_bytes(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  require(bool(is), path + ": cannot open");
  return {std::istreambuf_iterator<char>(is), std::istreambuf_iterator<char>()};
}

std::vector<double> read_coords_file(const std::string& path) {
  std::ifstream is(path);
  require(bool(is), path + ": cannot open");
  std::vector<double> c;
  std::string line;
  while (std::getline(is, line)) {
    if (line.empty()) continue;
    c.push_back(std::stod(line));
  }
  return c;
}

template <class T>
struct Dev {
  T* p = nullptr;
  explicit Dev(std::size_t n) { cuda(cudaMalloc(&p, (n ? n : 1) * sizeof(T))); }
  ~Dev() { cudaFree(p); }
};

// ---- decompose (hgr_main.cpp:86-114) --------------------------------------------
template <class T>
int run_decompose(const std::string& input, const std::string& output,
                  const std::vector<std::size_t>& dims, const std::vector<std::string>& cfiles,
                  bool as_json) {
  require(!dims.empty() && dims.size() <= 3, "dims must have 1 to 3 components");
  hgr_grid_desc g{};
  g.rank = int(dims.size());
  std::vector<std::vector<double>> coords;
  if (!cfiles.empty()) {
    require(cfiles.size() == dims.size(), "need one --coords-file per dimension");
    for (const auto& f : cfiles) coords.push_back(read_coords_file(f));
  }
  for (int d = 0; d < g.rank; ++d) {
    g.extents[d] = coords.empty() ? dims[std::size_t(d)] : coords[std::size_t(d)].size();
    g.coords[d] = coords.empty() ? nullptr : coords[std::size_t(d)].data();
  }
  if (hgr_levels(&g) < 0) throw DataError(hgr_cuda_last_error());  // make_hierarchy validation
  for (std::size_t d = 0; d < coords.size(); ++d)
    require(coords[d].size() == dims[d], cfiles[d] + ": coordinate count does not match --dims");
  std::size_t total = 1;
  for (auto d : dims) total *= d;
  const auto bytes = read_bytes(input);
  require(bytes.size() == total * sizeof(T),
          input + ": file holds " + std::to_string(bytes.size()) +
              " bytes but the given dims need " + std::to_string(total * sizeof(T)));
  Dev<T> in(total), out(total);
  cuda(cudaMemcpy(in.p, bytes.data(), bytes.size(), cudaMemcpyHostToDevice));
  if constexpr (sizeof(T) == 8) check(hgr_cuda_decompose_to_f64(&g, in.p, out.p, nullptr));
  else check(hgr_cuda_decompose_to_f32(&g, in.p, out.p, nullptr));
  uint64_t written = 0;
  if constexpr (sizeof(T) == 8) check(hgr_cuda_write_hg_f64(output.c_str(), &g, out.p, &written, nullptr));
  else check(hgr_cuda_write_hg_f32(output.c_str(), &g, out.p, &written, nullptr));
  hgr_hg_info info{};
  check(hgr_hg_read_info(output.c_str(), &info));
  std::vector<uint64_t> off(std::size_t(info.class_count)), cb(off.size()), ce(off.size());
  check(hgr_hg_read_class_table(output.c_str(), off.data(), cb.data(), info.class_count));
  for (std::size_t c = 0; c < cb.size(); ++c) ce[c] = cb[c] / info.precision_bytes;
  if (as_json) {
    Json j;
    j.str("command", "decompose");
    j.str("input", input);
    j.str("output", output);
    j.u64("bytes", written);
    j.i64("classes", info.class_count);
    j.arr("class_bytes", cb);
    j.arr("class_elements", ce);
    std::cout << j.dump() << "\n";
  } else {
    std::cout << "wrote " << output << " (" << written << " bytes)\n";
    std::cout << "classes: " << info.class_count << "\n";
    for (std::size_t c = 0; c < cb.size(); ++c)
      std::cout << "  class " << c << ": " << ce[c] << " elements, " << cb[c] << " bytes\n";
  }
  return 0;
}

// ---- recompose (hgr_main.cpp:122-138) -------------------------------------------
template <class T>
int run_recompose(const std::string& input, const std::string& output, int classes,
                  const hgr_hg_info& info, bool as_json) {
  std::size_t total = 1;
  hgr_grid_desc g{};
  g.rank = info.rank;
  std::vector<std::vector<double>> coords(std::size_t(info.rank));
  for (int d = 0; d < info.rank; ++d) {
    total *= info.extents[d];
    coords[std::size_t(d)].resize(info.extents[d]);
    check(hgr_hg_read_coords(input.c_str(), d, coords[std::size_t(d)].data()));
    g.extents[d] = info.extents[d];
    g.coords[d] = coords[std::size_t(d)].data();
  }
  Dev<T> pyr(total), out(total);
  uint64_t bytes_read = 0;
  if constexpr (sizeof(T) == 8) check(hgr_cuda_read_hg_prefix_f64(input.c_str(), classes, pyr.p, &bytes_read, nullptr));
  else check(hgr_cuda_read_hg_prefix_f32(input.c_str(), classes, pyr.p, &bytes_read, nullptr));
  if constexpr (sizeof(T) == 8) check(hgr_cuda_recompose_f64(&g, pyr.p, out.p, classes, nullptr));
  else check(hgr_cuda_recompose_f32(&g, pyr.p, out.p, classes, nullptr));
  std::vector<T> host(total);
  cuda(cudaMemcpy(host.data(), out.p, total * sizeof(T), cudaMemcpyDeviceToHost));
  std::ofstream os(output, std::ios::binary | std::ios::trunc);
  require(bool(os), output + ": cannot open for writing");
  os.write(reinterpret_cast<const char*>(host.data()), std::streamsize(total * sizeof(T)));
  os.flush();
  require(bool(os), output + ": write failed");
  if (as_json) {
    Json j;
    j.str("command", "recompose");
    j.str("input", input);
    j.str("output", output);
    j.i64("classes_used", classes);
    j.u64("bytes_read", bytes_read);
    j.u64("file_bytes", info.file_bytes);
    std::cout << j.dump() << "\n";
  } else {
    std::cout << "reconstructed " << output << " from classes 0.." << classes << "\n";
    std::cout << "bytes read: " << bytes_read << " of " << info.file_bytes << " ("
              << 100.0 * double(bytes_read) / double(info.file_bytes) << "%)\n";
  }
  return 0;
}

// ---- info (hgr_main.cpp:140-169) ------------------------------------------------
int run_info(const std::string& input, bool as_json) {
  hgr_hg_info h{};
  check(hgr_hg_read_info(input.c_str(), &h));
  std::vector<uint64_t> off(std::size_t(h.class_count)), cb(off.size()), ce(off.size());
  check(hgr_hg_read_class_table(input.c_str(), off.data(), cb.data(), h.class_count));
  for (std::size_t c = 0; c < cb.size(); ++c) ce[c] = cb[c] / h.precision_bytes;
  std::vector<uint64_t> dims(h.extents, h.extents + h.rank);
  if (as_json) {
    Json j;
    j.str("command", "info");
    j.str("input", input);
    j.u64("version", h.version);
    j.u64("precision_bytes", h.precision_bytes);
    j.arr("dims", dims);
    j.i64("classes", h.class_count);
    j.u64("header_bytes", h.header_bytes);
    j.u64("file_bytes", h.file_bytes);
    j.arr("class_bytes", cb);
    j.arr("class_elements", ce);
    std::cout << j.dump() << "\n";
    return 0;
  }
  std::cout << input << ":\n  version " << h.version << ", "
            << (h.precision_bytes == 4 ? "f32" : "f64") << ", dims";
  double total = 1;
  for (auto e : dims) {
    std::cout << " " << e;
    total *= double(e);
  }
  std::cout << "\n  " << h.class_count << " classes, " << h.file_bytes << " bytes ("
            << h.header_bytes << " header)\n";
  for (std::size_t c = 0; c < cb.size(); ++c)
    std::cout << "  class " << c << ": " << ce[c] << " elements ("
              << 100.0 * double(ce[c]) / total << "% of volume), " << cb[c] << " bytes\n";
  return 0;
}

// ---- error (hgr_main.cpp:171-198; error_report refactor.hpp:100-120) --------------
template <class T>
int run_error(const std::string& original, const std::string& recon, bool as_json) {
  const auto a = read_bytes(original), b = read_bytes(recon);
  require(a.size() == b.size(), "error: input files differ in size");
  require(a.size() % sizeof(T) == 0, "error: file size is not a whole number of elements");
  const std::size_t n = a.size() / sizeof(T);
  const T* x = reinterpret_cast<const T*>(a.data());
  const T* y = reinterpret_cast<const T*>(b.data());
  double sq_diff = 0, sq_orig = 0, max_diff = 0, max_orig = 0;
  for (std::size_t i = 0; i < n; ++i) {
    T xa, yb;
    std::memcpy(&xa, x + i, sizeof(T));
    std::memcpy(&yb, y + i, sizeof(T));
    const double av = double(xa), d = av - double(yb);
    sq_diff += d * d;
    sq_orig += av * av;
    max_diff = std::max(max_diff, std::abs(d));
    max_orig = std::max(max_orig, std::abs(av));
  }
  const double inf = std::numeric_limits<double>::infinity();
  const double l2_abs = std::sqrt(sq_diff), linf_abs = max_diff;
  const double l2_rel = sq_orig > 0 ? l2_abs / std::sqrt(sq_orig) : (l2_abs > 0 ? inf : 0.0);
  const double linf_rel = max_orig > 0 ? linf_abs / max_orig : (linf_abs > 0 ? inf : 0.0);
  if (as_json) {
    Json j;
    j.str("command", "error");
    j.str("original", original);
    j.str("reconstruction", recon);
    j.dbl("l2_abs", l2_abs);
    j.dbl("l2_rel", l2_rel);
    j.dbl("linf_abs", linf_abs);
    j.dbl("linf_rel", linf_rel);
    std::cout << j.dump() << "\n";
  } else {
    std::cout << "l2_abs   " << l2_abs << "\n"
              << "l2_rel   " << l2_rel << "\n"
              << "linf_abs " << linf_abs << "\n"
              << "linf_rel " << linf_rel << "\n";
  }
  return 0;
}


// ---- rank-configs (hgr_main.cpp:230-286; perf_model.hpp:71-162) ------------------
struct KCfg {
  uint64_t bx = 1, by = 1, bz = 1;
};

double estimate_time(int kind, const KCfg& c, uint64_t n, uint64_t S, uint64_t L, uint64_t G,
                     double bw) {
  require(c.bx >= 1 && c.by >= 1 && c.bz >= 1, "thread-block dimensions must be positive");
  require(n >= 1, "problem size must be positive");
  require(S >= 1 && L >= 1, "byte sizes must be positive");
  require(S % L == 0, "transaction size must be a multiple of the element size");
  require(bw > 0, "peak bandwidth must be positive");
  auto cdiv = [](uint64_t a, uint64_t b) { return (a + b - 1) / b; };
  auto pad = [&](uint64_t e, uint64_t per) { return cdiv(e, per) * per; };
  const uint64_t spl = S / L, ghost = G ? G : spl;
  const uint64_t bxn = cdiv(n, c.bx), byn = cdiv(n, c.by), bzn = cdiv(n, c.bz);
  uint64_t touched = 0;
  if (kind == 0)
    touched = pad(c.bx + 1, spl) * (c.by + 1) * (c.bz + 1) * bxn * byn * bzn;
  else if (kind == 1)
    touched = (pad(c.bx, spl) + 2 * spl) * c.by * c.bz * bxn * byn * bzn;
  else
    touched = (pad(ghost, spl) + pad(c.bx, spl) * bxn) * c.by * c.bz * byn * bzn;
  return double(touched) * 2.0 * double(L) / bw;
}

int run_rank_configs(const Args& a, int& stage) {
  auto u64 = [&](const std::string& k, uint64_t d) {
    const std::string v = one(a, k, "", false);
    if (v.empty()) return d;
    try {
      std::size_t pos = 0;
      const unsigned long long x = std::stoull(v, &pos);
      if (pos != v.size()) throw std::invalid_argument(v);
      return uint64_t(x);
    } catch (const std::exception&) {
      throw UsageError(k + ": not a non-negative integer");
    }
  };
  const uint64_t n = u64("--n", 513), L = u64("--bytes-per-element", 8);
  const uint64_t S = u64("--transaction-bytes", 32), G = u64("--ghost", 0);
  const uint64_t top = u64("--top", 0);
  double bw = 1.0;
  if (a.opt.count("--peak-bw")) {
    try {
      bw = std::stod(one(a, "--peak-bw"));
    } catch (const std::exception&) {
      throw UsageError("--peak-bw: not a number");
    }
  }
  const std::string kernel = one(a, "--kernel", "all", false);
  std::vector<int> kinds;
  if (kernel == "all") kinds = {0, 1, 2};
  else if (kernel == "gpk") kinds = {0};
  else if (kernel == "lpk") kinds = {1};
  else if (kernel == "ipk") kinds = {2};
  else throw UsageError("--kernel must be gpk, lpk, ipk, or all");
  stage = 2;  // parsing done: the rest are data errors
  std::vector<KCfg> cfgs = {{2, 2, 2}, {4, 4, 4}, {8, 4, 4}, {16, 4, 4},
                            {32, 4, 4}, {64, 2, 2}, {128, 2, 2}};  // default_block_configs
  const std::string file = one(a, "--configs", "", false);
  if (!file.empty()) {
    std::ifstream is(file);
    require(bool(is), file + ": cannot open");
    cfgs.clear();
    std::string line;
    while (std::getline(is, line)) {
      if (auto h = line.find('#'); h != std::string::npos) line.erase(h);
      for (auto& c : line)
        if (c == ',') c = ' ';
      std::istringstream ss(line);
      KCfg c;
      if (ss >> c.bx >> c.by >> c.bz) cfgs.push_back(c);
    }
    require(!cfgs.empty(), file + ": no configurations found");
  }
  static const char* names[3] = {"GPK", "LPK", "IPK"};
  Json out;
  out.str("command", "rank-configs");
  out.u64("n", n);
  for (int kind : kinds) {
    std::vector<std::pair<double, std::size_t>> order;
    for (std::size_t i = 0; i < cfgs.size(); ++i)
      order.emplace_back(estimate_time(kind, cfgs[i], n, S, L, G, bw), i);
    std::stable_sort(order.begin(), order.end(),
                     [](const auto& x, const auto& y) { return x.first < y.first; });
    if (top > 0) {
      require(top <= order.size(), "--top exceeds the configuration count");
      order.resize(top);
    }
    if (a.flag.count("--json") && a.flag.at("--json")) {
      std::string list = "[";
      for (std::size_t r = 0; r < order.size(); ++r) {
        const KCfg& c = cfgs[order[r].second];
        Json e;
        e.u64("bx", c.bx);
        e.u64("by", c.by);
        e.u64("bz", c.bz);
        e.i64("rank", static_cast<long long>(r + 1));
        e.dbl("seconds", order[r].first);
        list += (r ? "," : "") + e.dump();
      }
      out.set(names[kind], list + "]");
    } else {
      std::cout << names[kind] << " (n=" << n << ", S=" << S << ", L=" << L
                << ", G=" << (G ? G : S / L) << ", bw=" << bw << "):\n";
      std::cout << "  rank    bx    by    bz        est. seconds\n";
      for (std::size_t r = 0; r < order.size(); ++r) {
        const KCfg& c = cfgs[order[r].second];
        std::ostringstream row;
        row.setf(std::ios::scientific);
        row.precision(6);
        row << "  " << r + 1 << "\t" << c.bx << "\t" << c.by << "\t" << c.bz << "\t"
            << order[r].first;
        std::cout << row.str() << "\n";
      }
    }
  }
  if (a.flag.count("--json") && a.flag.at("--json")) std::cout << out.dump() << "\n";
  return 0;
}

const char* kUsage =
    "hierarchical grid refactoring for structured scientific data (B200 path)\n"
    "usage: hgr-b200 {decompose,recompose,info,error,rank-configs} [options]\n";

std::vector<std::size_t> parse_dims(const std::string& s) {
  std::vector<std::size_t> dims;
  std::stringstream ss(s);
  std::string part;
  while (std::getline(ss, part, ',')) {
    std::size_t pos = 0;
    unsigned long long v = 0;
    try {
      v = std::stoull(part, &pos);
    } catch (const std::exception&) {
      throw UsageError("--dims: not an integer list: " + s);
    }
    if (pos != part.size()) throw UsageError("--dims: not an integer list: " + s);
    dims.push_back(std::size_t(v));
  }
  return dims;
}

std::string precision_of(const Args& a) {
  const std::string p = one(a, "--precision", "f64", false);
  if (p != "f32" && p != "f64") throw UsageError("--precision: f32 or f64");
  return p;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << kUsage << "A subcommand is required\n";
    return 1;
  }
  const std::string cmd = argv[1];
  if (cmd == "-h" || cmd == "--help") {
    std::cout << kUsage;
    return 0;
  }
  int stage = 1;  // 1 = parsing (usage errors), 2 = running (data errors)
  try {
    if (cmd == "decompose") {
      Args a = parse(argc, argv, 2, {"--input", "--dims", "--precision", "--coords-file", "--output"},
                     {"--uniform", "--json"});
      const auto input = one(a, "--input"), output = one(a, "--output");
      const auto dims = parse_dims(one(a, "--dims"));
      const auto prec = precision_of(a);
      const auto cf = a.opt.count("--coords-file") ? a.opt["--coords-file"] : std::vector<std::string>{};
      if (a.flag["--uniform"] && !cf.empty())
        throw UsageError("--uniform excludes --coords-file");
      stage = 2;
      return prec == "f32" ? run_decompose<float>(input, output, dims, cf, a.flag["--json"])
                           : run_decompose<double>(input, output, dims, cf, a.flag["--json"]);
    }
    if (cmd == "recompose") {
      Args a = parse(argc, argv, 2, {"--input", "--classes", "--output"}, {"--json"});
      const auto input = one(a, "--input"), output = one(a, "--output");
      int classes = 0;
      try {
        classes = std::stoi(one(a, "--classes"));
      } catch (const UsageError&) {
        throw;
      } catch (const std::exception&) {
        throw UsageError("--classes: not an integer");
      }
      stage = 2;
      hgr_hg_info info{};
      check(hgr_hg_read_info(input.c_str(), &info));
      return info.precision_bytes == 4 ? run_recompose<float>(input, output, classes, info, a.flag["--json"])
                                       : run_recompose<double>(input, output, classes, info, a.flag["--json"]);
    }
    if (cmd == "info") {
      Args a = parse(argc, argv, 2, {"--input"}, {"--json"});
      const auto input = one(a, "--input");
      stage = 2;
      return run_info(input, a.flag["--json"]);
    }
    if (cmd == "error") {
      Args a = parse(argc, argv, 2, {"--original", "--reconstruction", "--precision"}, {"--json"});
      const auto o = one(a, "--original"), r = one(a, "--reconstruction");
      const auto prec = precision_of(a);
      stage = 2;
      return prec == "f32" ? run_error<float>(o, r, a.flag["--json"])
                           : run_error<double>(o, r, a.flag["--json"]);
    }
    if (cmd == "rank-configs") {
      Args a = parse(argc, argv, 2,
                     {"--n", "--bytes-per-element", "--transaction-bytes", "--ghost", "--peak-bw",
                      "--kernel", "--configs", "--top"},
                     {"--json"});
      return run_rank_configs(a, stage);
    }
    throw UsageError("unknown subcommand: " + cmd);
  } catch (const UsageError& e) {
    std::cerr << kUsage << e.what() << "\n";
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return stage == 1 ? 1 : 2;
  }
}
