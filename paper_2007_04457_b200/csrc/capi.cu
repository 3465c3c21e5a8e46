// capi.cu -- extern "C" boundary (include/hgr_cuda.h). Every entry point maps
// hgrb::Error (and CUDA failures) to an hgr_status + thread-local message.
#include <algorithm>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hgr_cuda.h"
#include "kernels.cuh"
#include "plan.hpp"
#include "storage.hpp"

using hgrb::Error;
using hgrb::Plan;

struct hgr_plan_s {
  std::unique_ptr<Plan> plan;
};

namespace {

thread_local std::string g_last_error;

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return HGR_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return HGR_ERR_NOMEM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return HGR_ERR_INVALID;
  }
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// ---- plan cache for the one-shot entry points ------------------------------
struct CacheKey {
  int dtype, device, rank;
  std::size_t n[3];
  std::vector<double> coords;
  bool operator==(const CacheKey& o) const {
    return dtype == o.dtype && device == o.device && rank == o.rank && n[0] == o.n[0] &&
           n[1] == o.n[1] && n[2] == o.n[2] && coords == o.coords;
  }
};

CacheKey make_key(const hgr_grid_desc* g, int dtype) {
  hgrb::require(g != nullptr, "grid descriptor is null");
  hgrb::require(g->rank >= 1 && g->rank <= 3, "grid must have 1 to 3 dimensions");
  CacheKey k{};
  k.dtype = dtype;
  cudaGetDevice(&k.device);
  k.rank = g->rank;
  for (int d = 0; d < 3; ++d) k.n[d] = d < g->rank ? g->extents[d] : 1;
  for (int d = 0; d < g->rank; ++d) {
    k.coords.push_back(g->coords[d] ? 1.0 : 0.0);
    if (g->coords[d]) k.coords.insert(k.coords.end(), g->coords[d], g->coords[d] + g->extents[d]);
  }
  return k;
}

std::mutex g_cache_mu;
std::list<std::pair<CacheKey, std::shared_ptr<Plan>>> g_cache;  // MRU first
constexpr std::size_t kCacheCap = 8;

std::shared_ptr<Plan> cached_plan(const hgr_grid_desc* g, int dtype) {
  CacheKey key = make_key(g, dtype);
  std::lock_guard<std::mutex> lock(g_cache_mu);
  for (auto it = g_cache.begin(); it != g_cache.end(); ++it)
    if (it->first == key) {
      g_cache.splice(g_cache.begin(), g_cache, it);
      return g_cache.front().second;
    }
  std::shared_ptr<Plan> p(hgrb::make_plan(g, dtype).release());
  g_cache.emplace_front(std::move(key), p);
  if (g_cache.size() > kCacheCap) g_cache.pop_back();
  return p;
}

std::size_t finest_count(const Plan& p) { return p.h.node_count(p.h.L); }

template <class T>
int decompose_dev(const hgr_grid_desc* g, T* d, void* stream) {
  return guarded([&] {
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32);
    p->decompose(d, as_stream(stream));
    int st = p->sync_status(as_stream(stream));
    if (st != HGR_OK) throw Error(st, "decompose: input contains non-finite values");
  });
}

template <class T>
int decompose_to_dev(const hgr_grid_desc* g, const T* in, T* out, void* stream) {
  return guarded([&] {
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32);
    p->decompose_to(in, out, as_stream(stream));
    int st = p->sync_status(as_stream(stream));
    if (st != HGR_OK) throw Error(st, "decompose: input contains non-finite values");
  });
}

template <class T>
int recompose_dev(const hgr_grid_desc* g, const T* in, T* out, int m, void* stream) {
  return guarded([&] {
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32);
    p->recompose(in, out, m, as_stream(stream));
  });
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(std::size_t n) { HGR_CUDA_CHECK(cudaMalloc(&p, (n ? n : 1) * sizeof(T))); }
  ~DevBuf() { cudaFree(p); }
};

template <class T>
int decompose_host(const hgr_grid_desc* g, T* h) {
  return guarded([&] {
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32);
    const std::size_t n = finest_count(*p);
    DevBuf<T> d(n), o(n);
    cudaStream_t s = nullptr;
    HGR_CUDA_CHECK(cudaMemcpy(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice));
    // finiteness is validated before h is modified (refactor.hpp:36-38)
    p->decompose_to(d.p, o.p, s);
    int st = p->sync_status(s);
    if (st != HGR_OK) throw Error(st, "decompose: input contains non-finite values");
    HGR_CUDA_CHECK(cudaMemcpy(h, o.p, n * sizeof(T), cudaMemcpyDeviceToHost));
  });
}

template <class T>
int recompose_host(const hgr_grid_desc* g, const T* in, T* out, int m) {
  return guarded([&] {
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32);
    const std::size_t n = finest_count(*p);
    DevBuf<T> d(n);
    HGR_CUDA_CHECK(cudaMemcpy(d.p, in, n * sizeof(T), cudaMemcpyHostToDevice));
    p->recompose(d.p, d.p, m, nullptr);
    HGR_CUDA_CHECK(cudaMemcpy(out, d.p, n * sizeof(T), cudaMemcpyDeviceToHost));
  });
}

template <class T>
int single_level(const hgr_grid_desc* g, int op, int level, const T* in, T* out, void* stream) {
  return guarded([&] {
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32);
    cudaStream_t s = as_stream(stream);
    if (op == 0) p->interpolate_to_fine(level, in, out, s);
    else if (op == 1) p->compute_coefficients(level, in, out, s);
    else p->compute_correction(level, in, out, s);
    HGR_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

template <class T>
int class_copy(const hgr_grid_desc* g, T* data, int cls, T* vals, bool extract, void* stream) {
  return guarded([&] {
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32);
    p->class_copy(data, cls, vals, extract, as_stream(stream));
    HGR_CUDA_CHECK(cudaStreamSynchronize(as_stream(stream)));
  });
}

// ---- fiber operators ------------------------------------------------------------

template <class T>
std::vector<T> fiber_taps(std::size_t n, const T* h) {
  hgrb::require(n >= 3 && (n - 1) % 2 == 0, "mass-trans: fine fiber length must be odd");
  const std::size_t nf = n, nc = (nf - 1) / 2 + 1;
  std::vector<T> taps(nc * 5, T(0));
  auto main_ = [&](std::size_t i) {
    const T left = i > 0 ? h[i - 1] : T(0);
    const T right = i + 1 < nf ? h[i] : T(0);
    return T(2) * (left + right);
  };
  for (std::size_t i = 0; i < nc; ++i) {
    std::size_t rj[3];
    T rw[3];
    std::size_t rn = 0;
    if (i > 0) {
      rj[rn] = 2 * i - 1;
      rw[rn++] = h[2 * i - 2] / (h[2 * i - 2] + h[2 * i - 1]);
    }
    rj[rn] = 2 * i;
    rw[rn++] = T(1);
    if (i + 1 < nc) {
      rj[rn] = 2 * i + 1;
      rw[rn++] = h[2 * i + 1] / (h[2 * i] + h[2 * i + 1]);
    }
    for (std::size_t k = 0; k < 5; ++k) {
      const long j = long(2 * i) - 2 + long(k);
      if (j < 0 || j >= long(nf)) continue;
      T sum = T(0);
      for (std::size_t r = 0; r < rn; ++r) {
        const std::size_t t = rj[r], jj = std::size_t(j);
        const T me = jj == t ? main_(t) : (jj + 1 == t ? h[t - 1] : (jj == t + 1 ? h[t] : T(0)));
        sum += rw[r] * me;
      }
      taps[i * 5 + k] = sum;
    }
  }
  return taps;
}

template <class T>
T* upload(const std::vector<T>& v, std::vector<void*>& owned) {
  T* d = nullptr;
  HGR_CUDA_CHECK(cudaMalloc(&d, std::max<std::size_t>(v.size(), 1) * sizeof(T)));
  owned.push_back(d);
  HGR_CUDA_CHECK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

struct Owned {
  std::vector<void*> p;
  ~Owned() {
    for (void* x : p) cudaFree(x);
  }
};

template <class T>
int fiber_op(int op, std::size_t n, std::size_t count, const T* v, const T* h, T* out,
             void* stream) {
  return guarded([&] {
    hgrb::require(n >= 2, "mass matrix needs at least one interval");
    cudaStream_t s = as_stream(stream);
    Owned own;
    std::vector<T> hv(h, h + n - 1);
    if (op == 0) {
      hgrb::launch_fiber_mass<T>(v, out, int64_t(n), int64_t(count), upload(hv, own.p), s);
    } else if (op == 1) {
      hgrb::launch_fiber_masstrans<T>(v, out, int64_t(n), int64_t(count),
                                      upload(fiber_taps<T>(n, h), own.p), s);
    } else {
      std::vector<T> mult(n - 1), pivot(n), upper(n - 1), rpiv(n);
      auto main_ = [&](std::size_t i) {
        const T left = i > 0 ? h[i - 1] : T(0);
        const T right = i + 1 < n ? h[i] : T(0);
        return T(2) * (left + right);
      };
      for (std::size_t i = 0; i < n; ++i) pivot[i] = main_(i);
      for (std::size_t i = 0; i + 1 < n; ++i) upper[i] = h[i];
      for (std::size_t i = 1; i < n; ++i) {
        mult[i - 1] = h[i - 1] / pivot[i - 1];
        pivot[i] = main_(i) - mult[i - 1] * upper[i - 1];
      }
      for (std::size_t i = 0; i < n; ++i) rpiv[i] = T(1) / pivot[i];
      hgrb::launch_fiber_thomas<T>(v, out, int64_t(n), int64_t(count), upload(mult, own.p),
                                   upload(rpiv, own.p), upload(upper, own.p), s);
    }
    HGR_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

template <class T>
int host_level_op(const hgr_grid_desc* g, int op, int level, const T* h_in, T* h_out) {
  return guarded([&] {
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32);
    hgrb::require(level >= 1 && level <= p->h.L, "level out of range");
    const std::size_t nf = p->h.node_count(level), nc = p->h.node_count(level - 1);
    const std::size_t nin = op == 0 ? nc : nf, nout = op == 2 ? nc : nf;
    DevBuf<T> din(nin), dout(nout);
    HGR_CUDA_CHECK(cudaMemcpy(din.p, h_in, nin * sizeof(T), cudaMemcpyHostToDevice));
    cudaStream_t s = nullptr;
    if (op == 0) p->interpolate_to_fine(level, din.p, dout.p, s);
    else if (op == 1) p->compute_coefficients(level, din.p, dout.p, s);
    else p->compute_correction(level, din.p, dout.p, s);
    HGR_CUDA_CHECK(cudaMemcpy(h_out, dout.p, nout * sizeof(T), cudaMemcpyDeviceToHost));
  });
}

template <class T>
int host_fiber_op(int op, std::size_t n, std::size_t count, const T* h_v, const T* h_h, T* h_out) {
  const std::size_t nout = op == 1 ? (n - 1) / 2 + 1 : n;
  int rc = HGR_OK;
  rc = guarded([&] {
    hgrb::require(n >= 2, "mass matrix needs at least one interval");
    DevBuf<T> dv(n * count), dout(nout * count);
    HGR_CUDA_CHECK(cudaMemcpy(dv.p, h_v, n * count * sizeof(T), cudaMemcpyHostToDevice));
    int r = fiber_op<T>(op, n, count, dv.p, h_h, dout.p, nullptr);
    if (r != HGR_OK) throw Error(r, g_last_error);
    HGR_CUDA_CHECK(cudaMemcpy(h_out, dout.p, nout * count * sizeof(T), cudaMemcpyDeviceToHost));
  });
  return rc;
}

}  // namespace

extern "C" {

int hgr_host_level_op_f64(const hgr_grid_desc* g, int op, int level, const double* i, double* o) {
  return host_level_op(g, op, level, i, o);
}
int hgr_host_level_op_f32(const hgr_grid_desc* g, int op, int level, const float* i, float* o) {
  return host_level_op(g, op, level, i, o);
}
int hgr_host_fiber_op_f64(int op, size_t n, size_t c, const double* v, const double* h, double* o) {
  return host_fiber_op(op, n, c, v, h, o);
}
int hgr_host_fiber_op_f32(int op, size_t n, size_t c, const float* v, const float* h, float* o) {
  return host_fiber_op(op, n, c, v, h, o);
}

const char* hgr_cuda_last_error(void) { return g_last_error.c_str(); }
int hgr_cuda_abi_version(void) { return HGR_CUDA_ABI_VERSION; }

int hgr_cuda_plan_create(const hgr_grid_desc* grid, int dtype, hgr_plan* out) {
  return guarded([&] {
    hgrb::require(out != nullptr, "plan output pointer is null");
    auto* p = new hgr_plan_s;
    try {
      p->plan = hgrb::make_plan(grid, dtype);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

void hgr_cuda_plan_destroy(hgr_plan plan) { delete plan; }

int hgr_cuda_plan_levels(hgr_plan plan) { return plan ? plan->plan->h.L : -1; }

size_t hgr_cuda_plan_workspace_bytes(hgr_plan plan) {
  return plan ? plan->plan->workspace_bytes() : 0;
}

int hgr_cuda_plan_launches(hgr_plan plan, int direction, int upto_class) {
  return plan ? plan->plan->launches(direction, upto_class) : -1;
}

int hgr_cuda_plan_decompose(hgr_plan plan, void* d_data, void* stream) {
  return guarded([&] {
    hgrb::require(plan != nullptr, "plan is null");
    plan->plan->decompose(d_data, as_stream(stream));
  });
}

int hgr_cuda_plan_decompose_to(hgr_plan plan, const void* d_in, void* d_out, void* stream) {
  return guarded([&] {
    hgrb::require(plan != nullptr, "plan is null");
    plan->plan->decompose_to(d_in, d_out, as_stream(stream));
  });
}

int hgr_cuda_plan_recompose(hgr_plan plan, const void* d_in, void* d_out, int upto_class,
                            void* stream) {
  return guarded([&] {
    hgrb::require(plan != nullptr, "plan is null");
    plan->plan->recompose(d_in, d_out, upto_class, as_stream(stream));
  });
}

int hgr_cuda_plan_sync_status(hgr_plan plan, void* stream) {
  int st = HGR_OK;
  int rc = guarded([&] {
    hgrb::require(plan != nullptr, "plan is null");
    st = plan->plan->sync_status(as_stream(stream));
    if (st != HGR_OK) throw Error(st, "decompose: input contains non-finite values");
  });
  return rc;
}

int hgr_cuda_plan_autotune(hgr_plan plan, const void* d_in, void* d_out, void* stream,
                           char* report, size_t report_bytes, size_t* report_len) {
  return guarded([&] {
    hgrb::require(plan != nullptr, "plan is null");
    hgrb::require(d_in != nullptr && d_out != nullptr, "autotune: null operand");
    const std::string rep = plan->plan->autotune(d_in, d_out, as_stream(stream));
    if (report_len) *report_len = rep.size();
    if (report && report_bytes) {
      const size_t n = std::min(rep.size(), report_bytes - 1);
      std::memcpy(report, rep.data(), n);
      report[n] = 0;
    }
  });
}

int hgr_cuda_plan_reset_tuning(hgr_plan plan) {
  return guarded([&] {
    hgrb::require(plan != nullptr, "plan is null");
    plan->plan->reset_tuning();
  });
}

int hgr_cuda_plan_set_profiling(hgr_plan plan, int enable) {
  return guarded([&] {
    hgrb::require(plan != nullptr, "plan is null");
    plan->plan->set_profiling(enable != 0);
  });
}

int hgr_cuda_plan_read_profile(hgr_plan plan, double* ms, double* bytes, long* launches) {
  return guarded([&] {
    hgrb::require(plan != nullptr, "plan is null");
    hgrb::KindStats st[hgrb::kKindCount];
    plan->plan->read_profile(st);
    for (int i = 0; i < hgrb::kKindCount; ++i) {
      if (ms) ms[i] = st[i].ms;
      if (bytes) bytes[i] = st[i].bytes;
      if (launches) launches[i] = st[i].launches;
    }
  });
}

int hgr_cuda_synthetic_field_f64(const hgr_grid_desc* g, double* d, unsigned long long seed,
                                 const double* a, const double* b, const double* c, void* s) {
  return guarded([&] { hgrb::synthetic_field<double>(g, d, seed, a, b, c, as_stream(s)); });
}
int hgr_cuda_synthetic_field_f32(const hgr_grid_desc* g, float* d, unsigned long long seed,
                                 const double* a, const double* b, const double* c, void* s) {
  return guarded([&] { hgrb::synthetic_field<float>(g, d, seed, a, b, c, as_stream(s)); });
}

int hgr_cuda_decompose_f64(const hgr_grid_desc* g, double* d, void* s) { return decompose_dev(g, d, s); }
int hgr_cuda_decompose_f32(const hgr_grid_desc* g, float* d, void* s) { return decompose_dev(g, d, s); }
int hgr_cuda_decompose_to_f64(const hgr_grid_desc* g, const double* i, double* o, void* s) {
  return decompose_to_dev(g, i, o, s);
}
int hgr_cuda_decompose_to_f32(const hgr_grid_desc* g, const float* i, float* o, void* s) {
  return decompose_to_dev(g, i, o, s);
}
int hgr_cuda_recompose_f64(const hgr_grid_desc* g, const double* i, double* o, int m, void* s) {
  return recompose_dev(g, i, o, m, s);
}
int hgr_cuda_recompose_f32(const hgr_grid_desc* g, const float* i, float* o, int m, void* s) {
  return recompose_dev(g, i, o, m, s);
}

int hgr_decompose_host_f64(const hgr_grid_desc* g, double* h) { return decompose_host(g, h); }
int hgr_decompose_host_f32(const hgr_grid_desc* g, float* h) { return decompose_host(g, h); }
int hgr_recompose_host_f64(const hgr_grid_desc* g, const double* i, double* o, int m) {
  return recompose_host(g, i, o, m);
}
int hgr_recompose_host_f32(const hgr_grid_desc* g, const float* i, float* o, int m) {
  return recompose_host(g, i, o, m);
}

int hgr_cuda_interpolate_to_fine_f64(const hgr_grid_desc* g, int l, const double* c, double* f, void* s) {
  return single_level(g, 0, l, c, f, s);
}
int hgr_cuda_interpolate_to_fine_f32(const hgr_grid_desc* g, int l, const float* c, float* f, void* s) {
  return single_level(g, 0, l, c, f, s);
}
int hgr_cuda_compute_coefficients_f64(const hgr_grid_desc* g, int l, const double* f, double* c, void* s) {
  return single_level(g, 1, l, f, c, s);
}
int hgr_cuda_compute_coefficients_f32(const hgr_grid_desc* g, int l, const float* f, float* c, void* s) {
  return single_level(g, 1, l, f, c, s);
}
int hgr_cuda_compute_correction_f64(const hgr_grid_desc* g, int l, const double* c, double* z, void* s) {
  return single_level(g, 2, l, c, z, s);
}
int hgr_cuda_compute_correction_f32(const hgr_grid_desc* g, int l, const float* c, float* z, void* s) {
  return single_level(g, 2, l, c, z, s);
}

int hgr_cuda_extract_class_f64(const hgr_grid_desc* g, const double* d, int cls, double* v, void* s) {
  return class_copy(g, const_cast<double*>(d), cls, v, true, s);
}
int hgr_cuda_extract_class_f32(const hgr_grid_desc* g, const float* d, int cls, float* v, void* s) {
  return class_copy(g, const_cast<float*>(d), cls, v, true, s);
}
int hgr_cuda_scatter_class_f64(const hgr_grid_desc* g, double* d, int cls, const double* v, void* s) {
  return class_copy(g, d, cls, const_cast<double*>(v), false, s);
}
int hgr_cuda_scatter_class_f32(const hgr_grid_desc* g, float* d, int cls, const float* v, void* s) {
  return class_copy(g, d, cls, const_cast<float*>(v), false, s);
}

size_t hgr_class_node_count(const hgr_grid_desc* g, int cls) {
  std::size_t n = 0;
  if (guarded([&] { n = hgrb::Hierarchy::from_desc(g).class_node_count(cls); }) != HGR_OK) return 0;
  return n;
}

int hgr_levels(const hgr_grid_desc* g) {
  int L = -1;
  if (guarded([&] { L = hgrb::Hierarchy::from_desc(g).L; }) != HGR_OK) return -1;
  return L;
}

int hgr_cuda_mass_apply_f64(size_t n, size_t c, const double* v, const double* h, double* o, void* s) {
  return fiber_op(0, n, c, v, h, o, s);
}
int hgr_cuda_masstrans_apply_f64(size_t n, size_t c, const double* v, const double* h, double* o, void* s) {
  return fiber_op(1, n, c, v, h, o, s);
}
int hgr_cuda_thomas_solve_f64(size_t n, size_t c, const double* v, const double* h, double* o, void* s) {
  return fiber_op(2, n, c, v, h, o, s);
}
int hgr_cuda_masstrans_apply_f32(size_t n, size_t c, const float* v, const float* h, float* o, void* s) {
  return fiber_op(1, n, c, v, h, o, s);
}
int hgr_cuda_thomas_solve_f32(size_t n, size_t c, const float* v, const float* h, float* o, void* s) {
  return fiber_op(2, n, c, v, h, o, s);
}

}  // extern "C"

// ---- .hg container (storage.hpp:17-218) ---------------------------------------

namespace {

template <class T>
int write_hg(const char* path, const hgr_grid_desc* g, const T* d, uint64_t* bytes, void* s) {
  return guarded([&] {
    hgrb::require(path != nullptr, "path is null");
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32);
    const uint64_t n = hgrb::hg_write(path, *p, d, as_stream(s));
    if (bytes) *bytes = n;
  });
}

template <class T>
int read_hg_prefix(const char* path, int upto, T* d, uint64_t* bytes, void* s) {
  return guarded([&] {
    hgrb::require(path != nullptr, "path is null");
    const hgrb::HgInfo info = hgrb::hg_read_info(path);
    hgr_grid_desc g{};
    g.rank = info.rank;
    for (int k = 0; k < info.rank; ++k) {
      g.extents[k] = info.extents[std::size_t(k)];
      g.coords[k] = info.coords[std::size_t(k)].data();
    }
    auto p = cached_plan(&g, sizeof(T) == 8 ? HGR_F64 : HGR_F32);
    const uint64_t n = hgrb::hg_read_prefix(path, info, *p, upto, d, as_stream(s));
    if (bytes) *bytes = n;
  });
}

}  // namespace

extern "C" {

int hgr_hg_read_info(const char* path, hgr_hg_info* out) {
  return guarded([&] {
    hgrb::require(path != nullptr && out != nullptr, "null argument");
    const hgrb::HgInfo h = hgrb::hg_read_info(path);
    *out = hgr_hg_info{};
    out->version = h.version;
    out->precision_bytes = h.precision_bytes;
    out->rank = h.rank;
    for (int k = 0; k < h.rank; ++k) out->extents[k] = h.extents[std::size_t(k)];
    out->class_count = int(h.offsets.size());
    out->header_bytes = h.header_bytes;
    out->file_bytes = h.file_bytes;
  });
}

int hgr_hg_read_coords(const char* path, int dim, double* h_out) {
  return guarded([&] {
    const hgrb::HgInfo h = hgrb::hg_read_info(path);
    hgrb::require(dim >= 0 && dim < h.rank, "dimension out of range");
    const auto& c = h.coords[std::size_t(dim)];
    std::memcpy(h_out, c.data(), c.size() * sizeof(double));
  });
}

int hgr_hg_read_class_table(const char* path, uint64_t* offsets, uint64_t* bytes, int max_classes) {
  return guarded([&] {
    const hgrb::HgInfo h = hgrb::hg_read_info(path);
    for (std::size_t c = 0; c < h.offsets.size() && int(c) < max_classes; ++c) {
      if (offsets) offsets[c] = h.offsets[c];
      if (bytes) bytes[c] = h.bytes[c];
    }
  });
}

int hgr_cuda_write_hg_f64(const char* path, const hgr_grid_desc* g, const double* d, uint64_t* b,
                          void* s) {
  return write_hg(path, g, d, b, s);
}
int hgr_cuda_write_hg_f32(const char* path, const hgr_grid_desc* g, const float* d, uint64_t* b,
                          void* s) {
  return write_hg(path, g, d, b, s);
}
int hgr_cuda_read_hg_prefix_f64(const char* path, int upto, double* d, uint64_t* b, void* s) {
  return read_hg_prefix(path, upto, d, b, s);
}
int hgr_cuda_read_hg_prefix_f32(const char* path, int upto, float* d, uint64_t* b, void* s) {
  return read_hg_prefix(path, upto, d, b, s);
}

}  // extern "C"
