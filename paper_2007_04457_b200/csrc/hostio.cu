// hostio.cu -- host <-> device movement for the host-pointer entry points
// (hgr_decompose_host_*, hgr_recompose_host_*, the C++ drop-in templates).
//
// The reference's decompose / recompose take host ndarrays (refactor.hpp:32-33,
// :63-68), so a drop-in user's data crosses PCIe twice per call. Pinned host
// buffers are moved by DMA directly. Pageable buffers go through a ring of
// pinned staging slots owned by the plan: host threads copy chunk i+1 into a
// free slot while the copy engine moves chunk i, so the pageable path runs at
// close to the DMA rate instead of the driver's synchronous bounce buffer.
// Device buffers are allocated once per plan and reused (no per-call cudaMalloc).
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "hostio.hpp"

namespace hgrb {

namespace {

constexpr std::size_t kSlot = std::size_t(32) << 20;  // bytes per staging slot
constexpr int kSlots = 3;

// Persistent workers for large host memcpys (one pageable chunk is split over
// all of them). Started on first use, joined at exit.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }
  std::size_t threads() const { return workers_.size() + 1; }
  void copy(void* dst, const void* src, std::size_t bytes) {
    const std::size_t parts = std::min<std::size_t>(workers_.size() + 1, (bytes + (1 << 20) - 1) >> 20);
    if (parts <= 1) {
      std::memcpy(dst, src, bytes);
      return;
    }
    const std::size_t per = (bytes / parts + 63) & ~std::size_t(63);
    run_parts(parts, [=](std::size_t k) {
      const std::size_t a = std::min(bytes, k * per), b = std::min(bytes, a + per);
      if (b > a) std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
    });
  }
  // part(k) for k in [0, parts) on the workers and the calling thread
  void run_parts(std::size_t parts, const std::function<void(std::size_t)>& part) {
    if (parts <= 1) {
      if (parts == 1) part(0);
      return;
    }
    std::lock_guard<std::mutex> one(call_mu_);  // one pooled job at a time
    std::unique_lock<std::mutex> lk(mu_);
    {
      job_ = part;
      next_ = 1;
      parts_ = parts;
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    lk.unlock();
    part(0);
    lk.lock();
    // help with the remaining parts, then wait for the workers' ones
    while (next_ < parts_) {
      const std::size_t k = next_++;
      lk.unlock();
      part(k);
      lk.lock();
      ++done_;
    }
    done_cv_.wait(lk, [&] { return done_ + 1 >= parts_; });
    job_ = nullptr;
  }

 private:
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned n = std::min(8u, std::max(1u, hw / 2)) - 1;
    for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this] { run(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void run() {
    unsigned long seen = 0;
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      cv_.wait(lk, [&] { return stop_ || (gen_ != seen && job_ && next_ < parts_); });
      if (stop_) return;
      seen = gen_;
      while (job_ && next_ < parts_) {
        const std::size_t k = next_++;
        auto job = job_;
        lk.unlock();
        job(k);
        lk.lock();
        ++done_;
        done_cv_.notify_all();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  std::function<void(std::size_t)> job_;
  std::size_t next_ = 0, parts_ = 0, done_ = 0;
  unsigned long gen_ = 0;
  bool stop_ = false;
};

// a predicate over [0, n) evaluated in chunks on the copy pool (large n only)
bool all_chunks(std::size_t n, const std::function<bool(std::size_t, std::size_t)>& ok) {
  constexpr std::size_t kMin = std::size_t(1) << 20;
  auto& pool = CopyPool::get();
  const std::size_t parts = std::min<std::size_t>(pool.threads(), (n + kMin - 1) / kMin);
  if (parts <= 1) return ok(0, n);
  const std::size_t per = (n + parts - 1) / parts;
  std::vector<char> res(parts, 1);
  pool.run_parts(parts, [&](std::size_t k) {
    const std::size_t a = std::min(n, k * per), b = std::min(n, a + per);
    res[k] = ok(a, b) ? 1 : 0;
  });
  return std::all_of(res.begin(), res.end(), [](char r) { return r != 0; });
}

bool is_pinned(const void* h) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

void ensure_staging(Plan& p) {
  if (!p.host_pin_[0]) {
    HGR_CUDA_CHECK(cudaMallocHost(&p.host_pin_[0], kSlot * kSlots));
    p.host_pin_bytes_ = kSlot * kSlots;
  }
  for (int i = 0; i < kSlots; ++i)
    if (!p.host_ev_[i]) HGR_CUDA_CHECK(cudaEventCreateWithFlags(&p.host_ev_[i], cudaEventDisableTiming));
}

char* slot(Plan& p, int i) { return static_cast<char*>(p.host_pin_[0]) + std::size_t(i) * kSlot; }

}  // namespace

void* host_device_buffer(Plan& p, int which, std::size_t bytes) {
  if (!p.host_dev_[which]) {
    const std::size_t n = p.h.node_count(p.h.L);
    const std::size_t esz = p.dtype == HGR_F64 ? 8 : 4;
    HGR_CUDA_CHECK(cudaMalloc(&p.host_dev_[which], std::max<std::size_t>(n * esz, 16)));
  }
  (void)bytes;
  return p.host_dev_[which];
}

cudaStream_t host_stream(Plan& p) {
  if (!p.host_streams_[0]) HGR_CUDA_CHECK(cudaStreamCreateWithFlags(&p.host_streams_[0], cudaStreamNonBlocking));
  return p.host_streams_[0];
}

void host_to_device(Plan& p, void* d, const void* h, std::size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  if (is_pinned(h)) {
    HGR_CUDA_CHECK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  ensure_staging(p);
  CopyPool& pool = CopyPool::get();
  std::size_t off = 0;
  for (int i = 0; off < bytes; ++i, off += kSlot) {
    const int k = i % kSlots;
    const std::size_t len = std::min(kSlot, bytes - off);
    if (i >= kSlots) HGR_CUDA_CHECK(cudaEventSynchronize(p.host_ev_[k]));  // slot drained
    pool.copy(slot(p, k), static_cast<const char*>(h) + off, len);
    HGR_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(d) + off, slot(p, k), len,
                                   cudaMemcpyHostToDevice, s));
    HGR_CUDA_CHECK(cudaEventRecord(p.host_ev_[k], s));
  }
}

void device_to_host(Plan& p, void* h, const void* d, std::size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  if (is_pinned(h)) {
    HGR_CUDA_CHECK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s));
    HGR_CUDA_CHECK(cudaStreamSynchronize(s));
    return;
  }
  ensure_staging(p);
  CopyPool& pool = CopyPool::get();
  const std::size_t chunks = (bytes + kSlot - 1) / kSlot;
  auto issue = [&](std::size_t i) {
    const std::size_t off = i * kSlot, len = std::min(kSlot, bytes - off);
    const int k = int(i % kSlots);
    HGR_CUDA_CHECK(cudaMemcpyAsync(slot(p, k), static_cast<const char*>(d) + off, len,
                                   cudaMemcpyDeviceToHost, s));
    HGR_CUDA_CHECK(cudaEventRecord(p.host_ev_[k], s));
  };
  // keep kSlots - 1 DMAs ahead of the host copy-out
  const std::size_t ahead = std::min<std::size_t>(chunks, kSlots - 1);
  for (std::size_t i = 0; i < ahead; ++i) issue(i);
  for (std::size_t i = 0; i < chunks; ++i) {
    if (i + ahead < chunks) issue(i + ahead);
    const int k = int(i % kSlots);
    HGR_CUDA_CHECK(cudaEventSynchronize(p.host_ev_[k]));
    const std::size_t off = i * kSlot, len = std::min(kSlot, bytes - off);
    pool.copy(static_cast<char*>(h) + off, slot(p, k), len);
  }
}

bool host_coords_iota(const double* c, std::size_t n) {
  if (c == nullptr) return true;
  return all_chunks(n, [c](std::size_t a, std::size_t b) {
    for (std::size_t i = a; i < b; ++i)
      if (c[i] != double(i)) return false;
    return true;
  });
}

bool host_coords_equal(const double* x, const double* y, std::size_t n) {
  return all_chunks(n, [x, y](std::size_t a, std::size_t b) {
    return std::memcmp(x + a, y + a, (b - a) * sizeof(double)) == 0;
  });
}

}  // namespace hgrb
