// plan.cu -- host orchestration: hierarchy, device tables, workspace, and the
// per-level launch schedule of decompose / recompose.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "kernels.cuh"
#include "kernels_fused.cuh"
#include "plan.hpp"
#include "tables.hpp"

namespace hgrb {

namespace {
// NVTX ranges per level and phase for nsys / ncu timelines (knob HGR_NVTX=1;
// header-only NVTX v3: no cost unless a tool is attached and the knob is set)
bool nvtx_on() {
  static const bool v = [] {
    const char* e = std::getenv("HGR_NVTX");
    return e && e[0] == '1';
  }();
  return v;
}
struct NvtxScope {
  bool on;
  NvtxScope(const char* what, int l) : on(nvtx_on()) {
    if (!on) return;
    char b[64];
    std::snprintf(b, sizeof b, "%s %d", what, l);
    nvtxRangePushA(b);
  }
  ~NvtxScope() {
    if (on) nvtxRangePop();
  }
};
}  // namespace


// ---- Hierarchy (grid_hierarchy.hpp:51-188) ------------------------------------

Hierarchy Hierarchy::from_desc(const hgr_grid_desc* g) {
  require(g != nullptr, "grid descriptor is null");
  require(g->rank >= 1 && g->rank <= 3, "grid must have 1 to 3 dimensions");
  Hierarchy h;
  h.rank = g->rank;
  h.coords.resize(std::size_t(g->rank));
  int min_depth = -1;
  for (int d = 0; d < g->rank; ++d) {
    const std::size_t n = g->extents[d];
    require(n >= 2 && ((n - 1) & (n - 2)) == 0,
            "dimension size must be 2^k+1 (dimension " + std::to_string(d) + " has " +
                std::to_string(n) + " nodes)");
    auto& c = h.coords[std::size_t(d)];
    c.resize(n);
    for (std::size_t i = 0; i < n; ++i) c[i] = g->coords[d] ? g->coords[d][i] : double(i);
    for (std::size_t i = 0; i + 1 < n; ++i)
      require(c[i] < c[i + 1],
              "coordinates must be strictly increasing (dimension " + std::to_string(d) + ")");
    int depth = 0;
    for (std::size_t v = n - 1; !(v & 1); v >>= 1) ++depth;
    if (min_depth < 0 || depth < min_depth) min_depth = depth;
  }
  h.L = min_depth;
  return h;
}

std::size_t Hierarchy::node_count(int l) const {
  std::size_t n = 1;
  for (int d = 0; d < rank; ++d) n *= extent(l, d);
  return n;
}

std::size_t Hierarchy::class_node_count(int cls) const {
  require(cls >= 0 && cls <= L, "level out of range");
  return cls == 0 ? node_count(0) : node_count(cls) - node_count(cls - 1);
}

std::vector<double> Hierarchy::spacings(int l, int d) const {
  const std::size_t s = stride(l);
  const auto& c = coords[std::size_t(d)];
  std::vector<double> h((c.size() - 1) / s);
  for (std::size_t i = 0; i < h.size(); ++i) h[i] = c[(i + 1) * s] - c[i * s];
  return h;
}

void Hierarchy::canon_extents(int l, int64_t e[3]) const {
  e[0] = e[1] = e[2] = 1;
  for (int d = 0; d < rank; ++d) e[d + 3 - rank] = int64_t(extent(l, d));
}

int Plan::sync_status(cudaStream_t s) {
  HGR_CUDA_CHECK(cudaMemcpyAsync(h_flag_, d_flag_, sizeof(int), cudaMemcpyDeviceToHost, s));
  HGR_CUDA_CHECK(cudaStreamSynchronize(s));
  return *h_flag_ ? HGR_ERR_NONFINITE : HGR_OK;
}

void Plan::begin_use(cudaStream_t s) {
  if (!use_ev_) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  HGR_CUDA_CHECK(cudaStreamIsCapturing(s, &cs));
  if (cs == cudaStreamCaptureStatusNone) HGR_CUDA_CHECK(cudaStreamWaitEvent(s, use_ev_, 0));
}

void Plan::end_use(cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
  if (!use_ev_ && cudaEventCreateWithFlags(&use_ev_, cudaEventDisableTiming) != cudaSuccess) {
    use_ev_ = nullptr;
    return;
  }
  cudaEventRecord(use_ev_, s);
}

Plan::~Plan() {
  if (use_ev_) cudaEventDestroy(use_ev_);
  for (void* p : host_dev_) cudaFree(p);
  for (void* p : host_pin_) cudaFreeHost(p);
  for (cudaStream_t st : host_streams_)
    if (st) cudaStreamDestroy(st);
  for (cudaEvent_t e : host_ev_)
    if (e) cudaEventDestroy(e);
  for (auto& g : graphs_)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (gstream_) cudaStreamDestroy(gstream_);
  for (cudaEvent_t e : gev_)
    if (e) cudaEventDestroy(e);
  for (auto& r : prof_pending_) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (cudaEvent_t e : ev_free_) cudaEventDestroy(e);
}

cudaEvent_t Plan::take_event() {
  if (!ev_free_.empty()) {
    cudaEvent_t e = ev_free_.back();
    ev_free_.pop_back();
    return e;
  }
  cudaEvent_t e;
  HGR_CUDA_CHECK(cudaEventCreate(&e));
  return e;
}

void Plan::set_profiling(bool on) {
  KindStats drop[kKindCount];
  read_profile(drop);  // recycles pending events
  for (auto& k : prof_acc_) k = KindStats{};
  profiling_ = on;
}

void Plan::prof_begin(int kind, double bytes, cudaStream_t s) {
  if (!profiling_) return;
  ProfRec r{kind, bytes, take_event(), take_event()};
  HGR_CUDA_CHECK(cudaEventRecord(r.a, s));
  prof_pending_.push_back(r);
}

void Plan::prof_end(cudaStream_t s) {
  if (!profiling_) return;
  HGR_CUDA_CHECK(cudaEventRecord(prof_pending_.back().b, s));
}

void Plan::read_profile(KindStats out[kKindCount]) {
  for (auto& r : prof_pending_) {
    HGR_CUDA_CHECK(cudaEventSynchronize(r.b));
    float ms = 0;
    HGR_CUDA_CHECK(cudaEventElapsedTime(&ms, r.a, r.b));
    KindStats& k = prof_acc_[r.kind];
    k.ms += ms;
    k.bytes += r.bytes;
    k.launches += 1;
    ev_free_.push_back(r.a);
    ev_free_.push_back(r.b);
  }
  prof_pending_.clear();
  for (int i = 0; i < kKindCount; ++i) out[i] = prof_acc_[i];
}

void Plan::clear_graphs() {
  for (auto& g : graphs_)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  graphs_.clear();
}

void Plan::run_graphed(int dir, const void* in, const void* out, int m, cudaStream_t s,
                       const std::function<void(cudaStream_t)>& direct) {
  if (profiling_ || !use_graphs) {
    direct(s);
    return;
  }
  ++graph_clock_;
  GraphEntry* e = nullptr;
  for (auto& g : graphs_)
    if (g.dir == dir && g.in == in && g.out == out && g.m == m) e = &g;
  if (!e) {  // first sighting: run directly, capture next time
    if (graphs_.size() >= 8) {
      auto lru = std::min_element(graphs_.begin(), graphs_.end(), [](const GraphEntry& a,
                                                                     const GraphEntry& b) {
        return a.last_use < b.last_use;
      });
      if (lru->exec) cudaGraphExecDestroy(lru->exec);
      graphs_.erase(lru);
    }
    graphs_.push_back(GraphEntry{dir, in, out, m, nullptr, graph_clock_});
    direct(s);
    return;
  }
  e->last_use = graph_clock_;
  if (!gstream_) {
    HGR_CUDA_CHECK(cudaStreamCreateWithFlags(&gstream_, cudaStreamNonBlocking));
    HGR_CUDA_CHECK(cudaEventCreateWithFlags(&gev_[0], cudaEventDisableTiming));
    HGR_CUDA_CHECK(cudaEventCreateWithFlags(&gev_[1], cudaEventDisableTiming));
  }
  if (!e->exec) {
    HGR_CUDA_CHECK(cudaStreamBeginCapture(gstream_, cudaStreamCaptureModeThreadLocal));
    try {
      direct(gstream_);
    } catch (...) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(gstream_, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    cudaGraph_t g = nullptr;
    HGR_CUDA_CHECK(cudaStreamEndCapture(gstream_, &g));
    const cudaError_t ie = cudaGraphInstantiate(&e->exec, g, 0);
    cudaGraphDestroy(g);
    HGR_CUDA_CHECK(ie);
  }
  HGR_CUDA_CHECK(cudaEventRecord(gev_[0], s));
  HGR_CUDA_CHECK(cudaStreamWaitEvent(gstream_, gev_[0], 0));
  HGR_CUDA_CHECK(cudaGraphLaunch(e->exec, gstream_));
  HGR_CUDA_CHECK(cudaEventRecord(gev_[1], gstream_));
  HGR_CUDA_CHECK(cudaStreamWaitEvent(s, gev_[1], 0));
}

// ---- precision-specific plan ----------------------------------------------------

namespace {

template <class T>
class PlanT final : public Plan {
 public:
  explicit PlanT(const Hierarchy& hier);
  ~PlanT() override;

  void decompose(void* d_data, cudaStream_t s) override;
  void recompose(const void* d_in, void* d_out, int upto, cudaStream_t s) override;
  int launches(int direction, int upto) override;
  std::string autotune(const void* d_in, void* d_out, cudaStream_t s) override;
  void reset_tuning() override;
  std::size_t workspace_bytes() const override { return ws_bytes_; }
  void interpolate_to_fine(int level, const void* coarse, void* fine, cudaStream_t s) override;
  void compute_coefficients(int level, const void* fine, void* coeffs, cudaStream_t s) override;
  void compute_correction(int level, const void* coeffs, void* z, cudaStream_t s) override;
  void apply_coefficients(int level, const void* coarse, const void* coeffs, void* fine,
                          cudaStream_t s) override;
  void class_copy(void* data, int cls, void* values, bool extract, cudaStream_t s) override;

  void decompose_to(const void* d_in, void* d_out, cudaStream_t s) override;
  void decompose_to_direct(const void* d_in, void* d_out, cudaStream_t s);
  void decompose_direct(void* d_data, cudaStream_t s);
  void recompose_direct(const void* d_in, void* d_out, int upto, cudaStream_t s);

 private:
  void correction(int l, const T* in, T* z, T* apply, int sign, cudaStream_t s);
  void thomas_all(int l, T* src, T* last_out, cudaStream_t s);
  bool thomas_route(int l, const T* src, const T* last_out) const;
  T* thomas_src(int l, T* last_out) const;
  void assemble(T* out, cudaStream_t s);
  // SURVEY §8(d) reference-step bytes of levels 1..lt (one direction)
  double tail_model_bytes() const {
    double total = 0;
    for (int l = 1; l <= tail_lt_; ++l) {
      const auto& e = ext_[std::size_t(l)];
      const auto& c = ext_[std::size_t(l) - 1];
      const int D = h.rank, k0 = 3 - D;
      const double n = double(e[0] * e[1] * e[2]), cn = double(c[0] * c[1] * c[2]), r = n - cn;
      std::vector<double> st(std::size_t(D) + 1);
      for (int k = 0; k <= D; ++k) {  // s_k: the first k real dims coarse
        double v = 1;
        for (int d = 0; d < D; ++d) v *= double(d < k ? c[std::size_t(k0 + d)] : e[std::size_t(k0 + d)]);
        st[std::size_t(k)] = v;
      }
      double b = (n + r) + (r + st[1]);
      for (int k = 1; k < D; ++k) b += st[std::size_t(k)] + st[std::size_t(k) + 1];
      total += sz() * (b + 2.0 * D * cn + 3.0 * cn);
    }
    return total;
  }
  void tail_decompose(cudaStream_t s) {
    if (tail_lt_ <= 0) return;
    prof_begin(kKindSmall, tail_model_bytes(), s);
    launch_tail_decompose<T>(tail_dev_, tail_lt_, h.rank, stage_[0], stage_[1], s);
    prof_end(s);
    ++launch_count_;
  }
  static constexpr double sz() { return double(sizeof(T)); }
  void decompose_level(int l, const T* src, T* coef_dst, bool in_place, cudaStream_t s);
  // levels with at least big_nodes_ nodes run the fused / TMA kernels, smaller
  // ones the one-thread-per-item kernels (tuning knob: HGR_BIG_LEVEL_NODES)
  bool big(int l) const { return h.node_count(l) >= big_nodes_; }
  std::size_t big_nodes_ = 4096;
  int L() const { return h.L; }

  std::vector<LevelArgs<T>> args_;     // index l = 1..L (0 unused)
  std::vector<std::array<int64_t, 3>> ext_;  // canonical extents per level 0..L
  // lookahead bands of the streaming IPK passes per (level, canonical dim)
  std::vector<std::array<int, 3>> stream_k_;
  std::vector<T*> C_;                  // compact level arrays 0..L-1
  std::vector<T*> D_;                  // compact coefficient arrays 1..L-1 (decompose)
  std::vector<T*> Z_;                  // corrections 1..L
  T* stage_[2] = {nullptr, nullptr};
  // LPK stage buffers of a fused-size level that had to take the reference
  // path (an operand the TMA kernels reject, e.g. a user pointer that is not
  // 16-byte aligned): allocated on first use, sized for that level
  T* stage_fb_[2] = {nullptr, nullptr};
  T* const* stages_for(int l);
  T* W_ = nullptr;                     // scratch of the windowed (out-of-place) Thomas passes
  // side rows of the top level (2D / 3D, fused): odd-column coefficients of its
  // even rows of even planes, merged into the output with the coarser pyramid by
  // k_merge_even (knob HGR_SIDE_ROWS=0: strided scatter instead)
  T* E_ = nullptr;
  // face scratch of the fused level kernels (two-phase faces, kernels_level.cu);
  // knob HGR_FACE2=0: the one-kernel faces instead
  T* F_ = nullptr;
  bool side_used_ = false;
  // coarse tail: levels 1..tail_lt_ (all below the fused threshold, under the
  // top) run as one single-CTA launch per direction (kernels_tail.cu)
  int tail_lt_ = 0;
  bool auto_tune_pending_ = false;  // HGR_AUTOTUNE=1
  // 3D IPK as dim 0 + fused dims 1+2 (kernels_band.cu); knob HGR_THOMAS_BAND:
  // 0 three passes, 1 strided-line dim 0 + cluster planes, 2 cluster passes for
  // both. Default: 1 for fp32, 0 for fp64 (its 135 KB plane tiles leave one
  // single-buffered CTA per SM; measured slower than three passes)
  int band_thomas_ = sizeof(T) == 4 ? 1 : 0;
  // 3D IPK as streaming column passes (kernels_stream.cu), ahead of the band
  // kernels; knob HGR_THOMAS_STREAM=0 disables
  bool stream_thomas_ = true;
  // smallest level (coarse nodes) for the streaming passes: fp64 levels below
  // 2^20 run the three-pass kernels (257x513x1025 fp64: 2.083 -> 2.062 ms per
  // round trip; 1025^3 fp64 unchanged); fp32 streams every level (the plane
  // pass wins at every size). Knob HGR_STREAM_MIN.
  std::size_t tune_top_ = 3;  // autotune: candidates measured per kernel (knob HGR_TUNE_TOP)
  int64_t stream_min_ = sizeof(T) == 8 ? int64_t(1) << 20 : 0;
  TailLevel<T>* tail_dev_ = nullptr;
  // tuned segment lengths per level (0: heuristic): decompose, recompose, interp
  std::vector<int> s0_dec_, s0_rec_, s0_int_;
  char* tables_ = nullptr;
  char* ws_ = nullptr;
  std::size_t ws_bytes_ = 0;
  int launch_count_ = 0;
  int last_launches_[2] = {0, 0};
};

template <class T>
PlanT<T>::PlanT(const Hierarchy& hier) {
  h = hier;
  // 1D/2D levels are a few rows of fused tiles: the fused path wins from 4096
  // nodes (with programmatic launches), 3D levels from 2^15 (measured)
  // 4096 nodes for every rank (3D: 513^3 fp32 1.250 -> 1.242 ms, 1025^3 fp32
  // 6.693 -> 6.685 ms against 2^15; 257x513x1025 fp64 unchanged)
  big_nodes_ = std::size_t(4096);
  if (const char* v = std::getenv("HGR_BIG_LEVEL_NODES")) big_nodes_ = std::size_t(std::atoll(v));
  if (const char* v = std::getenv("HGR_AUTOTUNE")) auto_tune_pending_ = v[0] == '1';
  if (const char* v = std::getenv("HGR_THOMAS_BAND")) band_thomas_ = std::atoi(v);
  if (const char* v = std::getenv("HGR_THOMAS_STREAM")) stream_thomas_ = v[0] != '0';
  if (const char* v = std::getenv("HGR_STREAM_MIN")) stream_min_ = std::atoll(v);
  if (const char* v = std::getenv("HGR_TUNE_TOP")) tune_top_ = std::size_t(std::max(1, std::atoi(v)));
  dtype = sizeof(T) == 8 ? HGR_F64 : HGR_F32;
  s0_dec_.assign(std::size_t(h.L) + 1, 0);
  s0_rec_.assign(std::size_t(h.L) + 1, 0);
  s0_int_.assign(std::size_t(h.L) + 1, 0);
  HGR_CUDA_CHECK(cudaGetDevice(&device));
  const int rank = h.rank, Lv = h.L;
  ext_.resize(std::size_t(Lv) + 1);
  for (int l = 0; l <= Lv; ++l) h.canon_extents(l, ext_[std::size_t(l)].data());

  // -- host tables, packed into one device allocation
  std::vector<char> blob;
  auto push = [&](const std::vector<T>& v) {
    std::size_t off = (blob.size() + 255) & ~std::size_t(255);
    blob.resize(off + v.size() * sizeof(T));
    std::memcpy(blob.data() + off, v.data(), v.size() * sizeof(T));
    return off;
  };
  struct Off {
    std::size_t wl, wr, taps, mult, pivot, upper, rpiv, h, trl, trr;
  };
  std::vector<std::array<Off, 3>> offs(std::size_t(Lv) + 1);
  stream_k_.assign(std::size_t(Lv) + 1, std::array<int, 3>{0, 0, 0});
  for (int l = 1; l <= Lv; ++l) {
    for (int d = 0; d < rank; ++d) {
      const int k = d + 3 - rank;
      Off o{};
      const auto hf = h.spacings(l, d);
      std::vector<T> wl(hf.size() / 2), wr(hf.size() / 2);
      for (std::size_t q = 0; q < hf.size() / 2; ++q) {
        const double span = hf[2 * q] + hf[2 * q + 1];
        wl[q] = T(hf[2 * q + 1] / span);
        wr[q] = T(hf[2 * q] / span);
      }
      o.wl = push(wl);
      o.wr = push(wr);
      std::vector<T> hT(hf.begin(), hf.end());
      o.taps = push(masstrans_taps<T>(hT));
      o.h = push(hT);
      {
        std::vector<T> trl, trr;
        transfer_weights<T>(hT, trl, trr);
        o.trl = push(trl);
        o.trr = push(trr);
      }
      const auto hc = h.spacings(l - 1, d);
      std::vector<T> hcT(hc.begin(), hc.end()), mult, pivot, upper, rpiv;
      thomas_factors<T>(hcT, mult, pivot, upper, rpiv);
      o.mult = push(mult);
      o.pivot = push(pivot);
      o.upper = push(upper);
      o.rpiv = push(rpiv);
      stream_k_[std::size_t(l)][std::size_t(k)] = stream_lookahead<T>(upper, rpiv);
      if (const char* v = std::getenv("HGR_STREAM_K"))  // test knob: at least this many
        stream_k_[std::size_t(l)][std::size_t(k)] =
            std::max(stream_k_[std::size_t(l)][std::size_t(k)], std::atoi(v));
      offs[std::size_t(l)][std::size_t(k)] = o;
    }
  }
  if (!blob.empty()) {
    HGR_CUDA_CHECK(cudaMalloc(&tables_, blob.size()));
    HGR_CUDA_CHECK(cudaMemcpy(tables_, blob.data(), blob.size(), cudaMemcpyHostToDevice));
  }
  args_.resize(std::size_t(Lv) + 1);
  for (int l = 1; l <= Lv; ++l) {
    LevelArgs<T>& a = args_[std::size_t(l)];
    std::memset(&a, 0, sizeof a);
    for (int k = 0; k < 3; ++k) {
      a.e[k] = ext_[std::size_t(l)][std::size_t(k)];
      a.c[k] = ext_[std::size_t(l) - 1][std::size_t(k)];
      if (k < 3 - rank) continue;
      const Off& o = offs[std::size_t(l)][std::size_t(k)];
      auto P = [&](std::size_t off) { return reinterpret_cast<const T*>(tables_ + off); };
      a.wl[k] = P(o.wl);
      a.wr[k] = P(o.wr);
      a.taps[k] = P(o.taps);
      a.mult[k] = P(o.mult);
      a.pivot[k] = P(o.pivot);
      a.upper[k] = P(o.upper);
      a.rpiv[k] = P(o.rpiv);
      a.h[k] = P(o.h);
      a.trl[k] = P(o.trl);
      a.trr[k] = P(o.trr);
    }
  }

  // -- workspace: compact level arrays C_0..C_{L-1}, corrections Z_1..Z_L, LPK stages
  auto nelem = [&](int l) {
    const auto& e = ext_[std::size_t(l)];
    return std::size_t(e[0] * e[1] * e[2]);
  };
  std::size_t stage_n[2] = {0, 0};
  for (int l = 1; l <= Lv; ++l) {
    if (big(l)) continue;  // fused levels need no LPK stage buffers
    std::array<int64_t, 3> e = ext_[std::size_t(l)];
    int pass = 0;
    for (int k = 3 - rank; k < 2; ++k, ++pass) {  // all but the last pass write a stage
      e[std::size_t(k)] = ext_[std::size_t(l) - 1][std::size_t(k)];
      stage_n[pass & 1] = std::max(stage_n[pass & 1], std::size_t(e[0] * e[1] * e[2]));
    }
  }
  std::vector<std::size_t> off_c(static_cast<std::size_t>(Lv)),
      off_z(static_cast<std::size_t>(Lv) + 1), off_d(static_cast<std::size_t>(Lv) + 1);
  std::size_t total = 0;
  const std::size_t esz = sizeof(T);
  // +256 B slack per buffer: bulk copies of the last row may round up to 16 B
  for (int l = 0; l < Lv; ++l) {
    off_c[std::size_t(l)] = total;
    total += (nelem(l) * esz + 511) & ~std::size_t(255);
  }
  for (int l = 1; l < Lv; ++l) {
    off_d[std::size_t(l)] = total;
    total += (nelem(l) * esz + 511) & ~std::size_t(255);
  }
  for (int l = 1; l <= Lv; ++l) {
    off_z[std::size_t(l)] = total;
    total += (nelem(l - 1) * esz + 511) & ~std::size_t(255);
  }
  std::size_t w_n = 0;
  for (int l = 1; l <= Lv; ++l) {
    for (int k = 3 - rank; k < 3; ++k)
      if (thomas_needs_out_of_place<T>(ext_[std::size_t(l) - 1].data(), k))
        w_n = std::max(w_n, nelem(l - 1));
  }
  const std::size_t off_w = total;
  total += (w_n * esz + 511) & ~std::size_t(255);
  std::size_t e_n = 0;
  {
    // rows longer than the merge kernel's shared-memory ring keep the scatter
    bool side = rank >= 2 && Lv >= 1 && big(Lv) && merge_even_fits<T>(ext_[std::size_t(Lv) - 1][2]);
    if (const char* v = std::getenv("HGR_SIDE_ROWS")) side = side && v[0] != '0';
    if (side) {
      const auto& c = ext_[std::size_t(Lv) - 1];
      e_n = std::size_t(c[0] * c[1] * (c[2] - 1));
    }
  }
  const std::size_t off_e = total;
  total += (e_n * esz + 511) & ~std::size_t(255);
  std::size_t f_n = 0;
  {
    bool face2 = true;
    if (const char* v = std::getenv("HGR_FACE2")) face2 = v[0] != '0';
    for (int l = 1; l <= Lv && face2; ++l)
      if (big(l))
        f_n = std::max(f_n, std::size_t(level_face_ws_elems<T>(ext_[std::size_t(l)].data(),
                                                                ext_[std::size_t(l) - 1].data())));
  }
  const std::size_t off_f = total;
  total += (f_n * esz + 511) & ~std::size_t(255);
  const std::size_t off_s0 = total;
  total += (stage_n[0] * esz + 511) & ~std::size_t(255);
  const std::size_t off_s1 = total;
  total += (stage_n[1] * esz + 511) & ~std::size_t(255);
  ws_bytes_ = total;
  if (total) HGR_CUDA_CHECK(cudaMalloc(&ws_, total));
  // debug / test knob: NaN-fill the workspace so a read-before-write shows up
  if (const char* v = std::getenv("HGR_POISON_WORKSPACE"))
    if (total && v[0] == '1') HGR_CUDA_CHECK(cudaMemset(ws_, 0xFF, total));
  C_.resize(std::size_t(Lv));
  Z_.assign(std::size_t(Lv) + 1, nullptr);
  for (int l = 0; l < Lv; ++l) C_[std::size_t(l)] = reinterpret_cast<T*>(ws_ + off_c[std::size_t(l)]);
  D_.assign(std::size_t(Lv) + 1, nullptr);
  for (int l = 1; l < Lv; ++l) D_[std::size_t(l)] = reinterpret_cast<T*>(ws_ + off_d[std::size_t(l)]);
  for (int l = 1; l <= Lv; ++l) Z_[std::size_t(l)] = reinterpret_cast<T*>(ws_ + off_z[std::size_t(l)]);
  if (w_n) W_ = reinterpret_cast<T*>(ws_ + off_w);
  if (e_n) E_ = reinterpret_cast<T*>(ws_ + off_e);
  if (f_n) F_ = reinterpret_cast<T*>(ws_ + off_f);
  stage_[0] = reinterpret_cast<T*>(ws_ + off_s0);
  {
    // one CTA is the better engine only while a level is a few thousand nodes
    // (tuning knob HGR_TAIL_NODES, 0 disables the tail)
    // 1D: the tail solves its one line sequentially in one thread, so only short
    // levels go there (2^26+1 fp64: 5.09 -> 4.83 ms with 64 instead of 1200)
    std::size_t tail_nodes = h.rank == 1 ? 64 : 1200;
    if (const char* v = std::getenv("HGR_TAIL_NODES")) tail_nodes = std::size_t(std::atoll(v));
    for (int l = Lv - 1; l >= 1; --l)
      if (!big(l) && h.node_count(l) <= tail_nodes) { tail_lt_ = l; break; }
  }
  stage_[1] = reinterpret_cast<T*>(ws_ + off_s1);
  if (tail_lt_ > 0) {
    std::vector<TailLevel<T>> tl(std::size_t(tail_lt_) + 1);
    for (int l = 1; l <= tail_lt_; ++l)
      tl[std::size_t(l)] = TailLevel<T>{args_[std::size_t(l)], C_[std::size_t(l)],
                                        D_[std::size_t(l)], C_[std::size_t(l) - 1],
                                        Z_[std::size_t(l)]};
    HGR_CUDA_CHECK(cudaMalloc(&tail_dev_, tl.size() * sizeof(TailLevel<T>)));
    HGR_CUDA_CHECK(cudaMemcpy(tail_dev_, tl.data(), tl.size() * sizeof(TailLevel<T>),
                              cudaMemcpyHostToDevice));
  }
  HGR_CUDA_CHECK(cudaMalloc(&d_flag_, sizeof(int)));
  HGR_CUDA_CHECK(cudaMemset(d_flag_, 0, sizeof(int)));
  HGR_CUDA_CHECK(cudaMallocHost(&h_flag_, sizeof(int)));
}

template <class T>
PlanT<T>::~PlanT() {
  cudaFree(stage_fb_[0]);
  cudaFree(stage_fb_[1]);
  cudaFree(tables_);
  cudaFree(ws_);
  cudaFree(tail_dev_);
  cudaFree(d_flag_);
  cudaFreeHost(h_flag_);
}

// LPK stage buffers for the reference path of level l: the shared ones for
// small levels, lazily grown fallback buffers for fused-size levels
template <class T>
T* const* PlanT<T>::stages_for(int l) {
  if (!big(l)) return stage_;
  if (!stage_fb_[0]) {  // sized once for every fused-size level (the top one dominates)
    std::size_t need[2] = {1, 1};
    for (int lv = 1; lv <= L(); ++lv) {
      if (!big(lv)) continue;
      std::array<int64_t, 3> e = ext_[std::size_t(lv)];
      int pass = 0;
      for (int k = 3 - h.rank; k < 2; ++k, ++pass) {
        e[std::size_t(k)] = ext_[std::size_t(lv) - 1][std::size_t(k)];
        need[pass & 1] = std::max(need[pass & 1], std::size_t(e[0] * e[1] * e[2]));
      }
    }
    HGR_CUDA_CHECK(cudaMalloc(&stage_fb_[0], need[0] * sizeof(T)));
    HGR_CUDA_CHECK(cudaMalloc(&stage_fb_[1], need[1] * sizeof(T)));
  }
  return stage_fb_;
}

// correction_level (correction.hpp:295-340): LPK passes over the real dims in
// ascending order (mask on the first), then Thomas passes in ascending order;
// the last Thomas pass optionally applies apply += sign*z instead of storing z.
template <class T>
void PlanT<T>::correction(int l, const T* in, T* z, T* apply, int sign, cudaStream_t s) {
  const LevelArgs<T>& a = args_[std::size_t(l)];
  const int rank = h.rank;
  int64_t e[3] = {a.e[0], a.e[1], a.e[2]};
  const T* cur = in;
  T* const* stage = stages_for(l);
  int pass = 0;
  for (int k = 3 - rank; k < 3; ++k, ++pass) {
    T* dst = (k == 2) ? z : stage[pass & 1];
    const double n_in = double(e[0] * e[1] * e[2]);
    prof_begin(kKindSmall, sz() * (n_in + n_in / double(e[k]) * double(a.c[k])), s);
    launch_lpk<T>(cur, e, dst, k, a.c[k], a.taps[k], pass == 0, s);
    prof_end(s);
    ++launch_count_;
    e[k] = a.c[k];
    cur = dst;
  }
  // Thomas passes: register-tiled kernels where the line fits them (windowed
  // passes ping-pong between z and W_), else one thread per line
  T* zc = z;
  const int64_t n = e[0] * e[1] * e[2];
  bool applied = false;
  for (int k = 3 - rank; k < 3; ++k) {
    const bool last = k == 2;
    prof_begin(kKindThomas, sz() * 2.0 * double(n), s);
    T* dst = thomas_needs_out_of_place<T>(e, k) ? (zc == W_ ? z : W_) : zc;
    if (launch_thomas_fast<T>(zc, dst, e, k, a.mult[k], a.rpiv[k], a.upper[k], s)) {
      zc = dst;
    } else {
      launch_thomas<T>(zc, e, k, a.mult[k], a.rpiv[k], a.upper[k], last ? apply : nullptr, sign, s);
      applied = last && apply;
    }
    prof_end(s);
    ++launch_count_;
  }
  if (apply && !applied) {
    launch_axpy<T>(apply, zc, n, sign, s);
    ++launch_count_;
  } else if (!apply && zc != z) {
    HGR_CUDA_CHECK(cudaMemcpyAsync(z, zc, std::size_t(n) * sizeof(T), cudaMemcpyDeviceToDevice, s));
  }
}

// Thomas passes (thomas_pass, correction.hpp:335-339) over the real dims in
// ascending order, starting from `src` (the load vector, clobbered); the last
// pass writes last_out. Passes that cut lines into overlapping windows run out
// of place between z and the scratch W_, the others in place.
template <class T>
bool PlanT<T>::thomas_route(int l, const T* src, const T* last_out) const {
  const LevelArgs<T>& a = args_[std::size_t(l)];
  const int64_t c[3] = {a.c[0], a.c[1], a.c[2]};
  const T* cur = src;
  for (int k = 3 - h.rank; k < 3; ++k) {
    const bool win = thomas_needs_out_of_place<T>(c, k);
    if (k == 2) return !(win && cur == last_out);
    if (win) cur = cur == W_ ? Z_[std::size_t(l)] : W_;
  }
  return true;
}

template <class T>
T* PlanT<T>::thomas_src(int l, T* last_out) const {
  T* z = Z_[std::size_t(l)];
  return thomas_route(l, z, last_out) ? z : W_;
}

template <class T>
void PlanT<T>::thomas_all(int l, T* src, T* last_out, cudaStream_t s) {
  const LevelArgs<T>& a = args_[std::size_t(l)];
  const int64_t c[3] = {a.c[0], a.c[1], a.c[2]};
  if (h.rank == 3 && stream_thomas_ && c[0] * c[1] * c[2] >= stream_min_) {
    // dim 0 strips in place, then dims 1+2 (fp32 planes; fp64 strips + rows) into last_out
    prof_begin(kKindThomas, sz() * (sizeof(T) == 8 ? 6.0 : 4.0) * double(c[0] * c[1] * c[2]), s);
    const int nl = launch_thomas_stream<T>(src, last_out, c, a.mult, a.rpiv, a.upper,
                                           stream_k_[std::size_t(l)].data(),
                                           int64_t(h.node_count(l)), s);
    prof_end(s);
    if (nl > 0) {
      launch_count_ += nl;
      return;
    }
  }
  if (h.rank == 3 && band_thomas_) {
    // two cluster passes: dim 0 in place, dims 1 + 2 fused into last_out
    prof_begin(kKindThomas, sz() * 4.0 * double(c[0] * c[1] * c[2]), s);
    const bool ok = launch_thomas_planes<T>(src, last_out, c, a.mult, a.rpiv, a.upper,
                                            int64_t(h.node_count(l)), band_thomas_ == 2, s);
    prof_end(s);
    if (ok) {
      launch_count_ += 2;
      return;
    }
  }
  T* cur = src;
  for (int k = 3 - h.rank; k < 3; ++k) {
    T* dst = cur;
    if (k == 2) dst = last_out;
    else if (thomas_needs_out_of_place<T>(c, k)) dst = cur == W_ ? Z_[std::size_t(l)] : W_;
    ++launch_count_;
    prof_begin(kKindThomas, sz() * 2.0 * double(c[0] * c[1] * c[2]), s);
    const bool fast = launch_thomas_fast<T>(cur, dst, c, k, a.mult[k], a.rpiv[k], a.upper[k], s);
    if (!fast) {
      launch_thomas<T>(cur, c, k, a.mult[k], a.rpiv[k], a.upper[k], nullptr, 0, s);
      if (dst != cur)
        HGR_CUDA_CHECK(cudaMemcpyAsync(dst, cur, std::size_t(c[0] * c[1] * c[2]) * sizeof(T),
                                       cudaMemcpyDeviceToDevice, s));
    }
    prof_end(s);
    cur = dst;
  }
}

// One decompose level (refactor.hpp:41-54): coefficients of level l into
// coef_dst and the corrected level-(l-1) nodal values into C_{l-1}.
template <class T>
void PlanT<T>::decompose_level(int l, const T* src, T* coef_dst, bool in_place, cudaStream_t s) {
  NvtxScope nv("decompose level", l);
  const LevelArgs<T>& a = args_[std::size_t(l)];
  T* Cn = C_[std::size_t(l) - 1];
  T* z = Z_[std::size_t(l)];
  const bool top = l == L();
  const double n = double(h.node_count(l)), c = double(h.node_count(l - 1));
  if (big(l)) {
    if (!in_place) {
      // read the level once, write the coefficients and the load vector once
      prof_begin(kKindFusedDec, sz() * (n + (n - c) + c), s);
      T* side = top ? E_ : nullptr;
      const bool ok = launch_level_fused<T>(src, coef_dst, z, nullptr, a, kFusedDecompose,
                                            top ? d_flag_ : nullptr, s, s0_dec_[std::size_t(l)], side,
                                            F_);
      prof_end(s);
      if (top) side_used_ = ok && side != nullptr;
      if (ok) {
        ++launch_count_;
        thomas_all(l, z, Cn, s);  // C_{l-1} = M_c^-1 K U = coarse + z
        return;
      }
    } else {
      // in place: the load vector and the coarse gather in one read of the level,
      // then the coefficients in place by the interpolation march in subtract mode
      prof_begin(kKindFusedDec, sz() * (n + 2 * c), s);
      const bool ok = launch_level_fused<T>(src, nullptr, z, Cn, a, kFusedLoadOnly, nullptr, s,
                                            s0_dec_[std::size_t(l)], nullptr, F_);
      prof_end(s);
      if (ok) {
        prof_begin(kKindInterp, sz() * (n + (n - c) + c), s);
        const bool sub = launch_coef_inplace<T>(coef_dst, Cn, a, top ? d_flag_ : nullptr, s,
                                                s0_int_[std::size_t(l)]);
        if (!sub) launch_gpk_dec<T>(coef_dst, Cn, a, d_flag_, top, s);  // coefficients in place
        prof_end(s);
        launch_count_ += 2;
        thomas_all(l, z, Cn, s);
        return;
      }
    }
  }
  // reference-faithful small-level path: GPK, gather, correction of the
  // coefficients, coarse += z (fused into the last Thomas pass)
  prof_begin(kKindSmall, sz() * (2 * n + c), s);
  if (in_place) {
    launch_gpk_dec<T>(coef_dst, Cn, a, d_flag_, top, s);
    ++launch_count_;
  } else {
    if (top) {
      check_finite<T>(src, a.e[0] * a.e[1] * a.e[2], d_flag_, s);
      ++launch_count_;
    }
    launch_coefficients<T>(src, coef_dst, a, s);
    launch_gather<T>(src, a.e, 2, Cn, a.c, s);
    launch_count_ += 2;
  }
  prof_end(s);
  correction(l, coef_dst, z, Cn, +1, s);
}

// pyramid assembly: each finished level-(l-1) pyramid into the even positions
// of level l (C_0 -> D_1 -> ... -> D_{L-1} -> out)
template <class T>
void PlanT<T>::assemble(T* out, cudaStream_t s) {
  NvtxScope nv("assemble pyramid levels", L());
  const int Lv = L();
  for (int l = 1; l <= Lv; ++l) {
    const T* src = l == 1 ? C_[0] : D_[std::size_t(l) - 1];
    prof_begin(kKindAssembly, sz() * 2.0 * double(h.node_count(l - 1)), s);
    if (l == Lv && side_used_)
      launch_merge_even<T>(src, E_, out, args_[std::size_t(l)], s);
    else
      launch_scatter_even<T>(src, l == Lv ? out : D_[std::size_t(l)], args_[std::size_t(l)], s);
    prof_end(s);
    ++launch_count_;
  }
}

// decompose (refactor.hpp:32-57) on compact level arrays: levels L..1 write the
// level-l coefficients (level L into the output, coarser ones into D_l) and the
// corrected coarse values C_{l-1}; the pyramid is then assembled bottom-up by
// writing each finished level-(l-1) pyramid into the even positions of level l.
template <class T>
void PlanT<T>::decompose_to(const void* d_in, void* d_out, cudaStream_t s) {
  if (d_in == d_out) return decompose(d_out, s);
  // HGR_AUTOTUNE=1: tune on the first out-of-place decompose (its output is
  // about to be overwritten anyway), for callers that never call autotune()
  if (auto_tune_pending_) {
    auto_tune_pending_ = false;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    HGR_CUDA_CHECK(cudaStreamIsCapturing(s, &cs));
    if (!profiling_ && cs == cudaStreamCaptureStatusNone) {
      try {
        autotune(d_in, d_out, s);
      } catch (const Error&) {
        reset_tuning();  // tuning is an optimisation: keep the heuristics
      }
    }
  }
  run_graphed(0, d_in, d_out, 0, s, [&](cudaStream_t st) { decompose_to_direct(d_in, d_out, st); });
}

template <class T>
void PlanT<T>::decompose_to_direct(const void* d_in, void* d_out, cudaStream_t s) {
  const T* in = static_cast<const T*>(d_in);
  T* out = static_cast<T*>(d_out);
  launch_count_ = 0;
  side_used_ = false;
  HGR_CUDA_CHECK(cudaMemsetAsync(d_flag_, 0, sizeof(int), s));
  const int Lv = L();
  if (Lv == 0) {
    check_finite<T>(in, h.node_count(0), d_flag_, s);
    HGR_CUDA_CHECK(cudaMemcpyAsync(out, in, h.node_count(0) * sizeof(T), cudaMemcpyDeviceToDevice, s));
    launch_count_ = 1;
    last_launches_[0] = launch_count_;
    return;
  }
  for (int l = Lv; l > tail_lt_; --l)
    decompose_level(l, l == Lv ? in : C_[std::size_t(l)], l == Lv ? out : D_[std::size_t(l)], false, s);
  tail_decompose(s);
  assemble(out, s);
  last_launches_[0] = launch_count_;
}

template <class T>
void PlanT<T>::decompose(void* d_data, cudaStream_t s) {
  run_graphed(2, d_data, d_data, 0, s, [&](cudaStream_t st) { decompose_direct(d_data, st); });
}

template <class T>
void PlanT<T>::decompose_direct(void* d_data, cudaStream_t s) {
  T* data = static_cast<T*>(d_data);
  launch_count_ = 0;
  HGR_CUDA_CHECK(cudaMemsetAsync(d_flag_, 0, sizeof(int), s));
  const int Lv = L();
  if (Lv == 0) {
    check_finite<T>(data, h.node_count(0), d_flag_, s);
    launch_count_ = 1;
    last_launches_[0] = launch_count_;
    return;
  }
  side_used_ = false;
  decompose_level(Lv, data, data, true, s);
  for (int l = Lv - 1; l > tail_lt_; --l)
    decompose_level(l, C_[std::size_t(l)], D_[std::size_t(l)], false, s);
  tail_decompose(s);
  assemble(data, s);
  last_launches_[0] = launch_count_;
}

// recompose (refactor.hpp:63-90): top-down, each level's correction z_l is
// computed from its coefficients (masked LPK + Thomas) while its coarse nodes
// (the coarser pyramid) are gathered into C_{l-1}; bottom-up, each level
// applies coarse -= z_l and the interpolation (refined = coef + interp).
template <class T>
void PlanT<T>::recompose(const void* d_in, void* d_out, int m, cudaStream_t s) {
  require(m >= 0 && m <= L(), "recompose: class index out of range");
  run_graphed(1, d_in, d_out, m, s, [&](cudaStream_t st) { recompose_direct(d_in, d_out, m, st); });
}

template <class T>
void PlanT<T>::recompose_direct(const void* d_in, void* d_out, int m, cudaStream_t s) {
  const T* in = static_cast<const T*>(d_in);
  T* out = static_cast<T*>(d_out);
  launch_count_ = 0;
  const int Lv = L();
  require(m >= 0 && m <= Lv, "recompose: class index out of range");
  if (Lv == 0) {
    if (out != in)
      HGR_CUDA_CHECK(cudaMemcpyAsync(out, in, h.node_count(0) * sizeof(T),
                                     cudaMemcpyDeviceToDevice, s));
    last_launches_[1] = 0;
    return;
  }
  const auto& fe = ext_[std::size_t(Lv)];
  if (m < Lv) {
    prof_begin(kKindAssembly, sz() * 2.0 * double(h.node_count(m)), s);
    launch_gather<T>(in, fe.data(), int64_t(1) << (Lv - m), C_[std::size_t(m)],
                     ext_[std::size_t(m)].data(), s);
    prof_end(s);
    ++launch_count_;
  }
  for (int l = m; l > tail_lt_; --l) {
    NvtxScope nv("recompose correction level", l);
    const T* src = l == Lv ? in : C_[std::size_t(l)];
    const LevelArgs<T>& a = args_[std::size_t(l)];
    const double n = double(h.node_count(l)), c = double(h.node_count(l - 1));
    if (big(l)) {
      // read the level once, write the load vector and the gathered coarse nodes
      T* zl = thomas_src(l, Z_[std::size_t(l)]);
      prof_begin(kKindFusedRec, sz() * (n + 2 * c), s);
      const bool ok = launch_level_fused<T>(src, nullptr, zl, C_[std::size_t(l) - 1], a,
                                            kFusedRecompose, nullptr, s, s0_rec_[std::size_t(l)],
                                            nullptr, F_);
      prof_end(s);
      if (ok) {
        ++launch_count_;
        thomas_all(l, zl, Z_[std::size_t(l)], s);
        continue;
      }
    }
    correction(l, src, Z_[std::size_t(l)], nullptr, 0, s);
    prof_begin(kKindSmall, sz() * 2.0 * c, s);
    launch_gather<T>(src, ext_[std::size_t(l)].data(), 2, C_[std::size_t(l) - 1],
                     ext_[std::size_t(l) - 1].data(), s);
    prof_end(s);
    ++launch_count_;
  }
  if (tail_lt_ > 0) {
    prof_begin(kKindSmall, tail_model_bytes(), s);
    launch_tail_recompose<T>(tail_dev_, tail_lt_, m, h.rank, stage_[0], stage_[1], s);
    prof_end(s);
    ++launch_count_;
  }
  for (int l = tail_lt_ + 1; l <= Lv; ++l) {
    NvtxScope nv("recompose interpolation level", l);
    const bool with = l <= m;
    const T* coef = l == Lv ? in : C_[std::size_t(l)];
    T* dst = l == Lv ? out : C_[std::size_t(l)];
    const T* Z = with ? Z_[std::size_t(l)] : nullptr;
    const double n = double(h.node_count(l)), c = double(h.node_count(l - 1));
    ++launch_count_;
    // read the coefficients (if any) and the coarse block (C, Z), write the level
    const double bytes = sz() * ((with ? (n - c) + 2 * c : c) + n);
    if (big(l)) {
      prof_begin(kKindInterp, bytes, s);
      const bool ok = launch_interp_rec<T>(coef, dst, C_[std::size_t(l) - 1], Z,
                                           args_[std::size_t(l)], with, s, s0_int_[std::size_t(l)]);
      prof_end(s);
      if (ok) continue;
    }
    prof_begin(kKindSmall, bytes, s);
    launch_gpk_rec<T>(coef, dst, C_[std::size_t(l) - 1], Z, args_[std::size_t(l)], with, s);
    prof_end(s);
  }
  last_launches_[1] = launch_count_;
}

template <class T>
int PlanT<T>::launches(int direction, int) {
  return last_launches_[direction ? 1 : 0];
}

template <class T>
void PlanT<T>::interpolate_to_fine(int level, const void* coarse, void* fine, cudaStream_t s) {
  require(level >= 1 && level <= L(), "level out of range");
  launch_interpolate<T>(static_cast<const T*>(coarse), static_cast<T*>(fine),
                        args_[std::size_t(level)], s);
}

template <class T>
void PlanT<T>::apply_coefficients(int level, const void* coarse, const void* coeffs, void* fine,
                                  cudaStream_t s) {
  require(level >= 1 && level <= L(), "level out of range");
  launch_interpolate<T>(static_cast<const T*>(coarse), static_cast<T*>(fine),
                        args_[std::size_t(level)], s);
  launch_axpy<T>(static_cast<T*>(fine), static_cast<const T*>(coeffs),
                 int64_t(h.node_count(level)), +1, s);
}

template <class T>
void PlanT<T>::compute_coefficients(int level, const void* fine, void* coeffs, cudaStream_t s) {
  require(level >= 1 && level <= L(), "level out of range");
  launch_coefficients<T>(static_cast<const T*>(fine), static_cast<T*>(coeffs),
                         args_[std::size_t(level)], s);
}

template <class T>
void PlanT<T>::compute_correction(int level, const void* coeffs, void* z, cudaStream_t s) {
  require(level >= 1 && level <= L(), "level out of range");
  HGR_CUDA_CHECK(cudaMemsetAsync(d_flag_, 0, sizeof(int), s));
  launch_check_coarse_zero<T>(static_cast<const T*>(coeffs), args_[std::size_t(level)], d_flag_,
                              s);
  HGR_CUDA_CHECK(cudaMemcpyAsync(h_flag_, d_flag_, sizeof(int), cudaMemcpyDeviceToHost, s));
  HGR_CUDA_CHECK(cudaStreamSynchronize(s));
  require(*h_flag_ == 0,
          "compute_correction: coefficients must be zero at coarse-grid positions");
  correction(level, static_cast<const T*>(coeffs), static_cast<T*>(z), nullptr, 0, s);
}

template <class T>
void PlanT<T>::reset_tuning() {
  std::fill(s0_dec_.begin(), s0_dec_.end(), 0);
  std::fill(s0_rec_.begin(), s0_rec_.end(), 0);
  std::fill(s0_int_.begin(), s0_int_.end(), 0);
  clear_graphs();
}

template <class T>
std::string PlanT<T>::autotune(const void* d_in, void* d_out, cudaStream_t s) {
  require(!profiling_, "autotune: disable profiling first");
  auto_tune_pending_ = false;  // an explicit tuning is not redone implicitly
  const int Lv = L();
  const T* in = static_cast<const T*>(d_in);
  T* out = static_cast<T*>(d_out);
  double bw = 6540.0;  // GB/s; only the ranking depends on it
  if (const char* v = std::getenv("HGR_MODEL_HBM_GBS")) bw = std::atof(v);
  cudaEvent_t e0, e1;
  HGR_CUDA_CHECK(cudaEventCreate(&e0));
  HGR_CUDA_CHECK(cudaEventCreate(&e1));
  // time one launch sequence: one warm run, then the mean of two
  auto time_us = [&](const std::function<void()>& run) {
    run();
    HGR_CUDA_CHECK(cudaEventRecord(e0, s));
    run();
    run();
    HGR_CUDA_CHECK(cudaEventRecord(e1, s));
    HGR_CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0.f;
    HGR_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    return 1e3 * double(ms) / 2.0;
  };
  std::string rep = "{\"hbm_model_gbs\": " + std::to_string(bw) + ", \"kernels\": [";
  bool first = true;
  auto tune = [&](int l, const char* name, std::vector<SegChoice> cands, int dflt,
                  const std::function<void(int)>& run, int& slot) {
    const std::size_t k = std::min<std::size_t>(tune_top_, cands.size());
    double best = 0;
    int best_s0 = 0;
    std::string cj;
    for (std::size_t i = 0; i < cands.size(); ++i) {
      double us = -1;
      if (i < k) {
        us = time_us([&] { run(cands[i].s0); });
        if (best_s0 == 0 || us < best) best = us, best_s0 = cands[i].s0;
      }
      cj += std::string(i ? ", " : "") + "{\"s0\": " + std::to_string(cands[i].s0) +
            ", \"blocks\": " + std::to_string(cands[i].blocks) +
            ", \"model_us\": " + std::to_string(cands[i].model_us) +
            ", \"measured_us\": " + (us < 0 ? std::string("null") : std::to_string(us)) + "}";
    }
    slot = best_s0;
    rep += std::string(first ? "" : ", ") + "{\"level\": " + std::to_string(l) +
           ", \"kernel\": \"" + name + "\", \"heuristic_s0\": " + std::to_string(dflt) +
           ", \"chosen_s0\": " + std::to_string(best_s0) + ", \"candidates\": [" + cj + "]}";
    first = false;
  };
  for (int l = Lv; l >= 1; --l) {
    if (!big(l) || h.rank < 3) continue;  // rank < 3: one plane, nothing to segment
    const LevelArgs<T>& a = args_[std::size_t(l)];
    const T* src = l == Lv ? in : C_[std::size_t(l)];
    T* coef = l == Lv ? out : D_[std::size_t(l)];
    T* z = Z_[std::size_t(l)];
    T* gat = C_[std::size_t(l) - 1];
    // operands the fused kernels accept (16-byte aligned); else the level is not fused
    if (!launch_level_fused<T>(src, coef, z, nullptr, a, kFusedDecompose, nullptr, s, 0, nullptr, F_))
      continue;
    tune(l, "decompose_level", level_fused_candidates<T>(a, kFusedDecompose, bw),
         level_fused_default_s0<T>(a),
         [&](int v) {
           launch_level_fused<T>(src, coef, z, nullptr, a, kFusedDecompose, nullptr, s, v, nullptr, F_);
         },
         s0_dec_[std::size_t(l)]);
    tune(l, "recompose_level", level_fused_candidates<T>(a, kFusedRecompose, bw),
         level_fused_default_s0<T>(a),
         [&](int v) {
           launch_level_fused<T>(src, nullptr, z, gat, a, kFusedRecompose, nullptr, s, v, nullptr, F_);
         },
         s0_rec_[std::size_t(l)]);
    T* dst = l == Lv ? out : C_[std::size_t(l)];
    const T* cf = l == Lv ? in : C_[std::size_t(l)];
    tune(l, "recompose_interp", interp_candidates<T>(a, true, true, bw), interp_default_s0<T>(a),
         [&](int v) { launch_interp_rec<T>(cf, dst, gat, z, a, true, s, v); },
         s0_int_[std::size_t(l)]);
  }
  rep += "]}";
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  clear_graphs();
  return rep;
}

template <class T>
void PlanT<T>::class_copy(void* data, int cls, void* values, bool extract, cudaStream_t s) {
  require(cls >= 0 && cls <= L(), "level out of range");
  launch_class_copy<T>(static_cast<T*>(data), ext_[std::size_t(L())].data(),
                       int64_t(1) << (L() - cls), ext_[std::size_t(cls)].data(), cls == 0,
                       static_cast<T*>(values), extract, s);
}

}  // namespace

std::unique_ptr<Plan> make_plan(const hgr_grid_desc* g, int dtype) {
  Hierarchy h = Hierarchy::from_desc(g);
  if (dtype == HGR_F64) return std::make_unique<PlanT<double>>(h);
  require(dtype == HGR_F32, "dtype must be HGR_F32 or HGR_F64");
  return std::make_unique<PlanT<float>>(h);
}

}  // namespace hgrb
