// plan.hpp -- host-side orchestration (C++): grid hierarchy, per-level device
// tables, device workspace and the per-level launch schedule.
//
// Mirrors the reference's host structures:
//   Hierarchy            <- GridHierarchy (grid_hierarchy.hpp:47-194)
//   PlanT<T>::decompose  <- hgr::decompose (refactor.hpp:32-57)
//   PlanT<T>::recompose  <- hgr::recompose (refactor.hpp:63-90)
//   PlanT<T>::correction <- detail::correction_level (correction.hpp:295-340)
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hgr_cuda.h"
#include "common.cuh"

namespace hgrb {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

inline void require(bool ok, const std::string& what, int code = HGR_ERR_INVALID) {
  if (!ok) throw Error(code, what);
}

// GridHierarchy (grid_hierarchy.hpp:47-194) in reference dimension order.
struct Hierarchy {
  int rank = 0;
  int L = 0;
  std::vector<std::vector<double>> coords;

  static Hierarchy from_desc(const hgr_grid_desc* g);
  std::size_t stride(int l) const { return std::size_t{1} << unsigned(L - l); }
  std::size_t extent(int l, int d) const { return (coords[d].size() - 1) / stride(l) + 1; }
  std::size_t node_count(int l) const;
  std::size_t class_node_count(int cls) const;
  // spacings (grid_hierarchy.hpp:163-177)
  std::vector<double> spacings(int l, int d) const;
  // canonical (left-padded) extents of level l
  void canon_extents(int l, int64_t e[3]) const;
};

// Kernel classes for the optional per-launch CUDA-event profile (bench.py's
// roofline of the dominant kernel). Order matches HGR_KIND_* in hgr_cuda.h.
enum KernelKind : int {
  kKindFusedDec = 0,   // k_level_fused, decompose (GPK + LPK)
  kKindFusedRec = 1,   // k_level_fused, recompose (masked LPK + gather)
  kKindThomas = 2,     // IPK passes
  kKindInterp = 3,     // recompose interpolation (GPK^-1)
  kKindAssembly = 4,   // pyramid assembly / gathers
  kKindSmall = 5,      // one-thread-per-item kernels of the small levels
  kKindCount = 6
};

struct KindStats {
  double ms = 0, bytes = 0;
  long launches = 0;
};

class Plan {
 public:
  virtual ~Plan();
  Hierarchy h;
  int dtype = HGR_F64;
  int device = 0;

  // profiling: when enabled, every launch is bracketed by CUDA events on its
  // stream and charged to its kernel class with its algorithmic bytes
  void set_profiling(bool on);
  void read_profile(KindStats out[kKindCount]);  // synchronizes; clears the window
  virtual void decompose(void* d_data, cudaStream_t s) = 0;
  virtual void decompose_to(const void* d_in, void* d_out, cudaStream_t s) = 0;
  virtual void recompose(const void* d_in, void* d_out, int upto, cudaStream_t s) = 0;
  virtual int launches(int direction, int upto) = 0;
  virtual std::size_t workspace_bytes() const = 0;
  int sync_status(cudaStream_t s);

  // single-level / packing entry points (compact level arrays)
  virtual void interpolate_to_fine(int level, const void* coarse, void* fine, cudaStream_t s) = 0;
  virtual void compute_coefficients(int level, const void* fine, void* coeffs, cudaStream_t s) = 0;
  virtual void compute_correction(int level, const void* coeffs, void* z, cudaStream_t s) = 0;
  // apply_coefficients (transforms.hpp:115-124): fine = interp(coarse) + coeffs
  virtual void apply_coefficients(int level, const void* coarse, const void* coeffs, void* fine,
                                  cudaStream_t s) = 0;
  virtual void class_copy(void* data, int cls, void* values, bool extract, cudaStream_t s) = 0;

  // Tile-segment autotuning (perf_model.hpp:71-137): for every
  // level on the fused kernels, rank the segment lengths of the decompose,
  // recompose and interpolation kernels with the sector model, time the top
  // three on this device with d_in / d_out / the workspace as operands (d_out
  // and the workspace are overwritten) and keep the fastest. Returns a JSON
  // report; later calls replay with the tuned launches (graphs are rebuilt).
  virtual std::string autotune(const void* d_in, void* d_out, cudaStream_t s) = 0;
  // drop the tuning (back to the built-in heuristics)
  virtual void reset_tuning() = 0;

  // Exclusive use of the plan (workspace, flag, graphs) for one call, the
  // reference's "distinct arrays may be processed concurrently" contract
  // (SPEC.md:287): host threads are serialised by `use_mu`, and a call's work
  // on its stream is ordered after the previous call's by an event recorded
  // at the end of every call, so two streams never share the workspace at the
  // same time. Skipped while the caller's stream is being captured.
  std::recursive_mutex use_mu;
  void begin_use(cudaStream_t s);
  void end_use(cudaStream_t s);
  // device staging of the host-pointer entry points (allocated on first use)
  void* host_dev_[2] = {nullptr, nullptr};
  void* host_pin_[2] = {nullptr, nullptr};
  std::size_t host_pin_bytes_ = 0;
  cudaStream_t host_streams_[2] = {nullptr, nullptr};
  cudaEvent_t host_ev_[4] = {nullptr, nullptr, nullptr, nullptr};

 protected:
  cudaEvent_t use_ev_ = nullptr;
  int* d_flag_ = nullptr;   // non-finite flag set by the level-L decompose kernel
  int* h_flag_ = nullptr;   // pinned mirror

  // profiling helpers (no-ops unless enabled)
  void prof_begin(int kind, double bytes, cudaStream_t s);
  void prof_end(cudaStream_t s);
  struct ProfRec {
    int kind;
    double bytes;
    cudaEvent_t a, b;
  };
  bool profiling_ = false;
  std::vector<ProfRec> prof_pending_;
  std::vector<cudaEvent_t> ev_free_;
  KindStats prof_acc_[kKindCount];
  cudaEvent_t take_event();

  // CUDA-graph replay of whole decompose / recompose launch sequences, keyed by
  // (direction, input, output, prefix): the first call runs directly (it also
  // sets kernel attributes), the second captures the sequence on a private
  // stream and every call from then on replays it, ordered after / before the
  // caller's stream by events. Disabled while profiling (per-launch events).
  void run_graphed(int dir, const void* in, const void* out, int m, cudaStream_t s,
                   const std::function<void(cudaStream_t)>& direct);
  struct GraphEntry {
    int dir;
    const void* in;
    const void* out;
    int m;
    cudaGraphExec_t exec;
    unsigned long last_use;
  };
  std::vector<GraphEntry> graphs_;
  void clear_graphs();
  unsigned long graph_clock_ = 0;
  cudaStream_t gstream_ = nullptr;
  cudaEvent_t gev_[2] = {nullptr, nullptr};

 public:
  bool use_graphs = true;
};

std::unique_ptr<Plan> make_plan(const hgr_grid_desc* g, int dtype);

// report.cu: error_report (refactor.hpp:100-120) of b against a; synchronizes s
template <class T>
void error_report(const T* a, const T* b, int64_t n, double out[4], cudaStream_t s);

// synth.cu
template <class T>
void synthetic_field(const hgr_grid_desc* g, T* out, uint64_t seed, const double* ha,
                     const double* hb, const double* hc, cudaStream_t s);

}  // namespace hgrb
