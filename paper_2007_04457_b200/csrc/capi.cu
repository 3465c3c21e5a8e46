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
#include "hostio.hpp"
#include "tables.hpp"
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
// A grid key stores the coordinates only where they are not the uniform 0..n-1
// (the null-coordinate grid): 1D grids carry as many coordinates as data
// values, so a lookup compares the caller's arrays in place (chunked over the
// host copy pool, hostio.cu) instead of copying them into a fresh key per call.
struct CacheKey {
  int dtype, device, rank;
  std::size_t n[3];
  std::vector<double> coords[3];  // empty: uniform (0..n-1)
};

struct GridView {  // the caller's grid as a lookup key (no copies)
  int dtype, device, rank;
  std::size_t n[3];
  const double* coords[3];  // nullptr: uniform
};

GridView view_of(const hgr_grid_desc* g, int dtype) {
  hgrb::require(g != nullptr, "grid descriptor is null");
  hgrb::require(g->rank >= 1 && g->rank <= 3, "grid must have 1 to 3 dimensions");
  GridView v{};
  v.dtype = dtype;
  cudaGetDevice(&v.device);
  v.rank = g->rank;
  for (int d = 0; d < 3; ++d) {
    v.n[d] = d < g->rank ? g->extents[d] : 1;
    v.coords[d] = d < g->rank && g->coords[d] && !hgrb::host_coords_iota(g->coords[d], g->extents[d])
                      ? g->coords[d]
                      : nullptr;
  }
  return v;
}

bool matches(const CacheKey& k, const GridView& v) {
  if (k.dtype != v.dtype || k.device != v.device || k.rank != v.rank) return false;
  for (int d = 0; d < 3; ++d) {
    if (k.n[d] != v.n[d]) return false;
    if (k.coords[d].empty() != (v.coords[d] == nullptr)) return false;
  }
  for (int d = 0; d < 3; ++d)
    if (v.coords[d] && !hgrb::host_coords_equal(k.coords[d].data(), v.coords[d], v.n[d]))
      return false;
  return true;
}

CacheKey key_of(const GridView& v) {
  CacheKey k{};
  k.dtype = v.dtype;
  k.device = v.device;
  k.rank = v.rank;
  for (int d = 0; d < 3; ++d) {
    k.n[d] = v.n[d];
    if (v.coords[d]) k.coords[d].assign(v.coords[d], v.coords[d] + v.n[d]);
  }
  return k;
}

// Each grid key holds a small pool of plans: a call leases one that no other
// host thread is using (a second plan is built when all are busy, up to
// kPoolCap), so distinct arrays of the same grid are processed concurrently
// (SPEC.md:287); a lease also orders the call's stream after the previous
// user of that plan (Plan::begin_use / end_use).
struct CacheEntry {
  CacheKey key;
  std::vector<std::shared_ptr<Plan>> pool;
};
std::mutex g_cache_mu;
std::list<CacheEntry> g_cache;  // MRU first
constexpr std::size_t kCacheCap = 8;
constexpr std::size_t kPoolCap = 4;

// kHostCall: the caller orders its work on the plan's private host stream itself
const cudaStream_t kHostCall = reinterpret_cast<cudaStream_t>(~uintptr_t(0));

struct Lease {
  std::shared_ptr<Plan> plan;
  std::unique_lock<std::recursive_mutex> lock;
  cudaStream_t s;
  Lease(std::shared_ptr<Plan> p, std::unique_lock<std::recursive_mutex> l, cudaStream_t st)
      : plan(std::move(p)), lock(std::move(l)), s(st) {
    if (s != kHostCall) plan->begin_use(s);
  }
  Lease(Lease&&) = default;
  ~Lease() {
    if (plan && lock.owns_lock() && s != kHostCall) plan->end_use(s);
  }
  Plan* operator->() const { return plan.get(); }
  Plan& operator*() const { return *plan; }
};

Lease cached_plan(const hgr_grid_desc* g, int dtype, cudaStream_t s = nullptr) {
  const GridView view = view_of(g, dtype);
  std::shared_ptr<Plan> busy;
  {
    std::lock_guard<std::mutex> lock(g_cache_mu);
    auto it = g_cache.begin();
    for (; it != g_cache.end(); ++it)
      if (matches(it->key, view)) break;
    if (it != g_cache.end()) {
      g_cache.splice(g_cache.begin(), g_cache, it);
      for (auto& p : g_cache.front().pool) {
        std::unique_lock<std::recursive_mutex> l(p->use_mu, std::try_to_lock);
        if (l.owns_lock()) return Lease(p, std::move(l), s);
      }
      if (g_cache.front().pool.size() >= kPoolCap) busy = g_cache.front().pool.front();
    }
  }
  if (busy) {  // every plan of the pool is in use: wait for the first
    std::unique_lock<std::recursive_mutex> l(busy->use_mu);
    return Lease(busy, std::move(l), s);
  }
  // build outside the cache lock (uploads tables, allocates the workspace)
  std::shared_ptr<Plan> p(hgrb::make_plan(g, dtype).release());
  std::unique_lock<std::recursive_mutex> l(p->use_mu);
  {
    std::lock_guard<std::mutex> lock(g_cache_mu);
    auto it = g_cache.begin();
    for (; it != g_cache.end(); ++it)
      if (matches(it->key, view)) break;
    if (it == g_cache.end()) {
      g_cache.push_front(CacheEntry{key_of(view), {}});
      it = g_cache.begin();
      if (g_cache.size() > kCacheCap) g_cache.pop_back();
    }
    if (it->pool.size() < kPoolCap) it->pool.push_back(p);
  }
  return Lease(p, std::move(l), s);
}

// an explicit plan handle: same serialisation, no pool
struct PlanUse {
  Plan& p;
  cudaStream_t s;
  std::lock_guard<std::recursive_mutex> lock;
  PlanUse(Plan& pl, cudaStream_t st) : p(pl), s(st), lock(pl.use_mu) { p.begin_use(s); }
  ~PlanUse() { p.end_use(s); }
};

std::size_t finest_count(const Plan& p) { return p.h.node_count(p.h.L); }

template <class T>
int decompose_dev(const hgr_grid_desc* g, T* d, void* stream) {
  return guarded([&] {
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32, as_stream(stream));
    p->decompose(d, as_stream(stream));
    int st = p->sync_status(as_stream(stream));
    if (st != HGR_OK) throw Error(st, "decompose: input contains non-finite values");
  });
}

template <class T>
int decompose_to_dev(const hgr_grid_desc* g, const T* in, T* out, void* stream) {
  return guarded([&] {
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32, as_stream(stream));
    p->decompose_to(in, out, as_stream(stream));
    int st = p->sync_status(as_stream(stream));
    if (st != HGR_OK) throw Error(st, "decompose: input contains non-finite values");
  });
}

template <class T>
int recompose_dev(const hgr_grid_desc* g, const T* in, T* out, int m, void* stream) {
  return guarded([&] {
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32, as_stream(stream));
    p->recompose(in, out, m, as_stream(stream));
  });
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(std::size_t n) { HGR_CUDA_CHECK(cudaMalloc(&p, (n ? n : 1) * sizeof(T))); }
  ~DevBuf() { cudaFree(p); }
};

// Host-pointer decompose / recompose (the reference's ndarray calls,
// refactor.hpp:32-33, :63-68): the plan's cached device buffers and private
// stream, pinned sources by direct DMA, pageable ones through the staging ring
// (hostio.cu). Synchronous like the reference.
template <class T>
int decompose_host(const hgr_grid_desc* g, T* h) {
  return guarded([&] {
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32, kHostCall);
    cudaStream_t s = hgrb::host_stream(*p);
    p->begin_use(s);
    const std::size_t bytes = finest_count(*p) * sizeof(T);
    void* din = hgrb::host_device_buffer(*p, 0, bytes);
    void* dout = hgrb::host_device_buffer(*p, 1, bytes);
    hgrb::host_to_device(*p, din, h, bytes, s);
    p->decompose_to(din, dout, s);
    // finiteness is validated before h is modified (refactor.hpp:36-38)
    const int st = p->sync_status(s);
    if (st != HGR_OK) throw Error(st, "decompose: input contains non-finite values");
    hgrb::device_to_host(*p, h, dout, bytes, s);
    p->end_use(s);
  });
}

template <class T>
int recompose_host(const hgr_grid_desc* g, const T* in, T* out, int m) {
  return guarded([&] {
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32, kHostCall);
    cudaStream_t s = hgrb::host_stream(*p);
    p->begin_use(s);
    const std::size_t bytes = finest_count(*p) * sizeof(T);
    void* din = hgrb::host_device_buffer(*p, 0, bytes);
    void* dout = hgrb::host_device_buffer(*p, 1, bytes);
    hgrb::host_to_device(*p, din, in, bytes, s);
    p->recompose(din, dout, m, s);
    hgrb::device_to_host(*p, out, dout, bytes, s);
    p->end_use(s);
  });
}

template <class T>
int single_level(const hgr_grid_desc* g, int op, int level, const T* in, T* out, void* stream) {
  return guarded([&] {
    cudaStream_t s = as_stream(stream);
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32, s);
    if (op == 0) p->interpolate_to_fine(level, in, out, s);
    else if (op == 1) p->compute_coefficients(level, in, out, s);
    else p->compute_correction(level, in, out, s);
    HGR_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

template <class T>
int class_copy(const hgr_grid_desc* g, T* data, int cls, T* vals, bool extract, void* stream) {
  return guarded([&] {
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32, as_stream(stream));
    p->class_copy(data, cls, vals, extract, as_stream(stream));
    HGR_CUDA_CHECK(cudaStreamSynchronize(as_stream(stream)));
  });
}

// ---- fiber operators ------------------------------------------------------------

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

// op: 0 mass_apply, 1 masstrans_apply, 2 thomas_solve, 3 transfer_apply,
// 4 masstrans with even inputs masked (MassTransOperator::apply_fiber's
// zero_even_inputs). Tables come from the plan's builders (tables.hpp).
template <class T>
int fiber_op(int op, std::size_t n, std::size_t count, const T* v, const T* h, T* out,
             void* stream) {
  return guarded([&] {
    hgrb::require(n >= 2, "mass matrix needs at least one interval");
    if (op == 1 || op == 3 || op == 4)
      hgrb::require(n >= 3 && (n - 1) % 2 == 0,
                    op == 3 ? "transfer_apply: fine fiber length must be odd"
                            : "mass-trans: fine fiber length must be odd");
    cudaStream_t s = as_stream(stream);
    Owned own;
    std::vector<T> hv(h, h + n - 1);
    if (op == 0) {
      hgrb::launch_fiber_mass<T>(v, out, int64_t(n), int64_t(count), upload(hv, own.p), s);
    } else if (op == 1 || op == 4) {
      hgrb::launch_fiber_masstrans<T>(v, out, int64_t(n), int64_t(count),
                                      upload(hgrb::masstrans_taps<T>(hv), own.p), op == 4, s);
    } else if (op == 3) {
      std::vector<T> trl, trr;
      hgrb::transfer_weights<T>(hv, trl, trr);
      hgrb::launch_fiber_transfer<T>(v, out, int64_t(n), int64_t(count), upload(trl, own.p),
                                     upload(trr, own.p), s);
    } else {
      std::vector<T> mult, pivot, upper, rpiv;
      hgrb::thomas_factors<T>(hv, mult, pivot, upper, rpiv);
      hgrb::launch_fiber_thomas<T>(v, out, int64_t(n), int64_t(count), upload(mult, own.p),
                                   upload(rpiv, own.p), upload(upper, own.p), s);
    }
    HGR_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

template <class T>
int host_level_op(const hgr_grid_desc* g, int op, int level, const T* h_in, T* h_out) {
  return guarded([&] {
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32, kHostCall);
    hgrb::require(level >= 1 && level <= p->h.L, "level out of range");
    const std::size_t nf = p->h.node_count(level), nc = p->h.node_count(level - 1);
    const std::size_t nin = op == 0 ? nc : nf, nout = op == 2 ? nc : nf;
    cudaStream_t s = hgrb::host_stream(*p);
    p->begin_use(s);
    void* din = hgrb::host_device_buffer(*p, 0, nin * sizeof(T));
    void* dout = hgrb::host_device_buffer(*p, 1, nout * sizeof(T));
    hgrb::host_to_device(*p, din, h_in, nin * sizeof(T), s);
    if (op == 0) p->interpolate_to_fine(level, din, dout, s);
    else if (op == 1) p->compute_coefficients(level, din, dout, s);
    else p->compute_correction(level, din, dout, s);
    hgrb::device_to_host(*p, h_out, dout, nout * sizeof(T), s);
    p->end_use(s);
  });
}

template <class T>
int apply_coefficients_dev(const hgr_grid_desc* g, int level, const T* coarse, const T* coeffs,
                           T* fine, void* stream) {
  return guarded([&] {
    cudaStream_t s = as_stream(stream);
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32, s);
    p->apply_coefficients(level, coarse, coeffs, fine, s);
    HGR_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

template <class T>
int apply_coefficients_host(const hgr_grid_desc* g, int level, const T* h_coarse,
                            const T* h_coeffs, T* h_fine) {
  return guarded([&] {
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32, kHostCall);
    hgrb::require(level >= 1 && level <= p->h.L, "level out of range");
    const std::size_t nf = p->h.node_count(level), nc = p->h.node_count(level - 1);
    cudaStream_t s = hgrb::host_stream(*p);
    p->begin_use(s);
    DevBuf<T> dc(nc), dcoef(nf);
    T* df = static_cast<T*>(hgrb::host_device_buffer(*p, 1, nf * sizeof(T)));
    hgrb::host_to_device(*p, dc.p, h_coarse, nc * sizeof(T), s);
    hgrb::host_to_device(*p, dcoef.p, h_coeffs, nf * sizeof(T), s);
    p->apply_coefficients(level, dc.p, dcoef.p, df, s);
    hgrb::device_to_host(*p, h_fine, df, nf * sizeof(T), s);
    p->end_use(s);
  });
}

template <class T>
int error_report_host(size_t n, const T* a, const T* b, double* out) {
  return guarded([&] {
    cudaStream_t s = nullptr;
    HGR_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct S {
      cudaStream_t s;
      ~S() { cudaStreamDestroy(s); }
    } guard{s};
    DevBuf<T> da(n), db(n);
    HGR_CUDA_CHECK(cudaMemcpyAsync(da.p, a, n * sizeof(T), cudaMemcpyHostToDevice, s));
    HGR_CUDA_CHECK(cudaMemcpyAsync(db.p, b, n * sizeof(T), cudaMemcpyHostToDevice, s));
    hgrb::error_report<T>(da.p, db.p, int64_t(n), out, s);
  });
}

template <class T>
int write_hg_host(const char* path, const hgr_grid_desc* g, const T* h, uint64_t* bytes) {
  return guarded([&] {
    hgrb::require(path != nullptr, "path is null");
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32, kHostCall);
    cudaStream_t s = hgrb::host_stream(*p);
    p->begin_use(s);
    const std::size_t nb = finest_count(*p) * sizeof(T);
    void* d = hgrb::host_device_buffer(*p, 0, nb);
    hgrb::host_to_device(*p, d, h, nb, s);
    const uint64_t n = hgrb::hg_write(path, *p, d, s);
    if (bytes) *bytes = n;
    p->end_use(s);
  });
}

template <class T>
int read_hg_prefix_host(const char* path, int upto, T* h, uint64_t* bytes) {
  return guarded([&] {
    hgrb::require(path != nullptr, "path is null");
    const hgrb::HgInfo info = hgrb::hg_read_info(path);
    hgr_grid_desc g{};
    g.rank = info.rank;
    for (int k = 0; k < info.rank; ++k) {
      g.extents[k] = info.extents[std::size_t(k)];
      g.coords[k] = info.coords[std::size_t(k)].data();
    }
    auto p = cached_plan(&g, sizeof(T) == 8 ? HGR_F64 : HGR_F32, kHostCall);
    cudaStream_t s = hgrb::host_stream(*p);
    p->begin_use(s);
    const std::size_t nb = finest_count(*p) * sizeof(T);
    void* d = hgrb::host_device_buffer(*p, 0, nb);
    const uint64_t n = hgrb::hg_read_prefix(path, info, *p, upto, d, s);
    hgrb::device_to_host(*p, h, d, nb, s);
    if (bytes) *bytes = n;
    p->end_use(s);
  });
}

template <class T>
int host_fiber_op(int op, std::size_t n, std::size_t count, const T* h_v, const T* h_h, T* h_out) {
  const std::size_t nout = (op == 1 || op == 3 || op == 4) ? (n - 1) / 2 + 1 : n;
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

template <class T>
int masstrans_taps_host(size_t n, const T* h, T* taps) {
  return guarded([&] {
    hgrb::require(h && taps, "null argument");
    hgrb::require(n >= 3 && (n - 1) % 2 == 0, "mass-trans: fine fiber length must be odd");
    const auto t = hgrb::masstrans_taps<T>(std::vector<T>(h, h + n - 1));
    std::copy(t.begin(), t.end(), taps);
  });
}
template <class T>
int thomas_factors_host(size_t n, const T* h, T* mult, T* pivot, T* upper) {
  return guarded([&] {
    hgrb::require(n >= 2, "mass matrix needs at least one interval");
    std::vector<T> m, p, u, r;
    hgrb::thomas_factors<T>(std::vector<T>(h, h + n - 1), m, p, u, r);
    if (mult) std::copy(m.begin(), m.begin() + std::ptrdiff_t(n - 1), mult);
    if (pivot) std::copy(p.begin(), p.end(), pivot);
    if (upper) std::copy(u.begin(), u.begin() + std::ptrdiff_t(n - 1), upper);
  });
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
    PlanUse use(*plan->plan, as_stream(stream));
    plan->plan->decompose(d_data, as_stream(stream));
  });
}

int hgr_cuda_plan_decompose_to(hgr_plan plan, const void* d_in, void* d_out, void* stream) {
  return guarded([&] {
    hgrb::require(plan != nullptr, "plan is null");
    PlanUse use(*plan->plan, as_stream(stream));
    plan->plan->decompose_to(d_in, d_out, as_stream(stream));
  });
}

int hgr_cuda_plan_recompose(hgr_plan plan, const void* d_in, void* d_out, int upto_class,
                            void* stream) {
  return guarded([&] {
    hgrb::require(plan != nullptr, "plan is null");
    PlanUse use(*plan->plan, as_stream(stream));
    plan->plan->recompose(d_in, d_out, upto_class, as_stream(stream));
  });
}

int hgr_cuda_plan_sync_status(hgr_plan plan, void* stream) {
  int st = HGR_OK;
  int rc = guarded([&] {
    hgrb::require(plan != nullptr, "plan is null");
    PlanUse use(*plan->plan, as_stream(stream));
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
    PlanUse use(*plan->plan, as_stream(stream));
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
int hgr_cuda_mass_apply_f32(size_t n, size_t c, const float* v, const float* h, float* o, void* s) {
  return fiber_op(0, n, c, v, h, o, s);
}
int hgr_cuda_transfer_apply_f64(size_t n, size_t c, const double* v, const double* h, double* o, void* s) {
  return fiber_op(3, n, c, v, h, o, s);
}
int hgr_cuda_transfer_apply_f32(size_t n, size_t c, const float* v, const float* h, float* o, void* s) {
  return fiber_op(3, n, c, v, h, o, s);
}
int hgr_cuda_masstrans_apply_f32(size_t n, size_t c, const float* v, const float* h, float* o, void* s) {
  return fiber_op(1, n, c, v, h, o, s);
}
int hgr_cuda_thomas_solve_f32(size_t n, size_t c, const float* v, const float* h, float* o, void* s) {
  return fiber_op(2, n, c, v, h, o, s);
}

int hgr_masstrans_taps_f64(size_t n, const double* h, double* t) { return masstrans_taps_host(n, h, t); }
int hgr_masstrans_taps_f32(size_t n, const float* h, float* t) { return masstrans_taps_host(n, h, t); }
int hgr_thomas_factors_f64(size_t n, const double* h, double* m, double* p, double* u) {
  return thomas_factors_host(n, h, m, p, u);
}
int hgr_thomas_factors_f32(size_t n, const float* h, float* m, float* p, float* u) {
  return thomas_factors_host(n, h, m, p, u);
}

int hgr_cuda_apply_coefficients_f64(const hgr_grid_desc* g, int l, const double* c, const double* k,
                                    double* f, void* s) {
  return apply_coefficients_dev(g, l, c, k, f, s);
}
int hgr_cuda_apply_coefficients_f32(const hgr_grid_desc* g, int l, const float* c, const float* k,
                                    float* f, void* s) {
  return apply_coefficients_dev(g, l, c, k, f, s);
}
int hgr_host_apply_coefficients_f64(const hgr_grid_desc* g, int l, const double* c, const double* k,
                                    double* f) {
  return apply_coefficients_host(g, l, c, k, f);
}
int hgr_host_apply_coefficients_f32(const hgr_grid_desc* g, int l, const float* c, const float* k,
                                    float* f) {
  return apply_coefficients_host(g, l, c, k, f);
}
int hgr_error_report_host_f64(size_t n, const double* a, const double* b, double* o) {
  return error_report_host(n, a, b, o);
}
int hgr_error_report_host_f32(size_t n, const float* a, const float* b, double* o) {
  return error_report_host(n, a, b, o);
}
int hgr_write_hg_host_f64(const char* path, const hgr_grid_desc* g, const double* h, uint64_t* b) {
  return write_hg_host(path, g, h, b);
}
int hgr_write_hg_host_f32(const char* path, const hgr_grid_desc* g, const float* h, uint64_t* b) {
  return write_hg_host(path, g, h, b);
}
int hgr_read_hg_prefix_host_f64(const char* path, int upto, double* h, uint64_t* b) {
  return read_hg_prefix_host(path, upto, h, b);
}
int hgr_read_hg_prefix_host_f32(const char* path, int upto, float* h, uint64_t* b) {
  return read_hg_prefix_host(path, upto, h, b);
}

int hgr_cuda_error_report_f64(size_t n, const double* a, const double* b, double* o, void* s) {
  return guarded([&] { hgrb::error_report<double>(a, b, int64_t(n), o, as_stream(s)); });
}
int hgr_cuda_error_report_f32(size_t n, const float* a, const float* b, double* o, void* s) {
  return guarded([&] { hgrb::error_report<float>(a, b, int64_t(n), o, as_stream(s)); });
}

}  // extern "C"

// ---- .hg container (storage.hpp:17-218) ---------------------------------------

namespace {

template <class T>
int write_hg(const char* path, const hgr_grid_desc* g, const T* d, uint64_t* bytes, void* s) {
  return guarded([&] {
    hgrb::require(path != nullptr, "path is null");
    auto p = cached_plan(g, sizeof(T) == 8 ? HGR_F64 : HGR_F32, as_stream(s));
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
    auto p = cached_plan(&g, sizeof(T) == 8 ? HGR_F64 : HGR_F32, as_stream(s));
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
