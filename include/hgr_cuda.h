/*
 * hgr_cuda.h -- C ABI of the B200-native hierarchical refactoring library
 * (libhgr_b200.so, sources in paper_2007_04457_b200/csrc/).
 *
 * Drop-in boundary for the reference's hot path. The reference (`hgr`,
 * header-only C++20, /root/reference/proj/include/hgr) has no FFI of its own;
 * its public entry points are C++ templates. Each function below states the
 * reference interface it replaces (file:line, relative to proj/include/hgr/).
 * The C++ template drop-in that re-declares the reference API on top of this
 * ABI is include/hgr_b200/hgr.hpp; the Python mirror is
 * paper_2007_04457_b200/__init__.py.
 *
 * Conventions
 *  - Arrays are row-major, last dimension contiguous (ndarray.hpp:15-57), rank 1..3.
 *  - "d_" pointers are device pointers (cudaMalloc'd or torch tensors) on the
 *    current CUDA device; "h_" pointers are host pointers.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Device-pointer calls are stream-ordered and asynchronous unless noted.
 *  - Every call returns an hgr_status; on failure hgr_cuda_last_error() (thread
 *    local) holds a message whose substrings match the reference's hgr::error
 *    texts ("2^k+1", "non-finite", "zero at coarse", "level out of range",
 *    "class index out of range", "shape").
 */
#ifndef HGR_CUDA_H
#define HGR_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HGR_CUDA_ABI_VERSION 1

typedef enum hgr_status {
  HGR_OK = 0,
  HGR_ERR_INVALID = 1,   /* argument/shape/level validation (reference: detail::require) */
  HGR_ERR_CUDA = 2,      /* CUDA runtime failure */
  HGR_ERR_NONFINITE = 3, /* decompose input held NaN/Inf (refactor.hpp:36-38) */
  HGR_ERR_NOMEM = 4
} hgr_status;

typedef enum hgr_dtype { HGR_F32 = 0, HGR_F64 = 1 } hgr_dtype;

/* Grid description = the arguments of GridHierarchy(coords_per_dim)
 * (grid_hierarchy.hpp:51-70) / GridHierarchy::uniform (:73-80).
 * coords[d] may be NULL for uniform integer coordinates 0..n-1. */
typedef struct hgr_grid_desc {
  int rank;
  size_t extents[3];
  const double* coords[3];
} hgr_grid_desc;

typedef struct hgr_plan_s* hgr_plan;

const char* hgr_cuda_last_error(void);
int hgr_cuda_abi_version(void);

/* ---- plans: GridHierarchy + device tables + workspace ---------------------
 * Replaces GridHierarchy construction (grid_hierarchy.hpp:51-70, build_caches
 * :163-188) and the per-call workspace of correction_level (correction.hpp:301).
 * A plan may be shared by host threads and streams: calls on one plan are
 * serialised (a per-plan lock while a call enqueues, and each call's work is
 * ordered after the previous call's by an event), so results never depend on
 * interleaving. For concurrent execution create one plan per stream; the
 * one-shot entry points below do this themselves (a small pool of plans per
 * grid, "distinct arrays may be processed concurrently"). */
int hgr_cuda_plan_create(const hgr_grid_desc* grid, int dtype, hgr_plan* out);
void hgr_cuda_plan_destroy(hgr_plan plan);
/* GridHierarchy::levels() (grid_hierarchy.hpp:85) */
int hgr_cuda_plan_levels(hgr_plan plan);
/* bytes of device workspace held by the plan */
size_t hgr_cuda_plan_workspace_bytes(hgr_plan plan);
/* number of kernel launches one decompose/recompose enqueues */
int hgr_cuda_plan_launches(hgr_plan plan, int direction /*0 dec, 1 rec*/, int upto_class);

/* decompose (refactor.hpp:32-57): in place on the finest-shape device array.
 * Non-finite inputs are detected inside the first kernel; the outcome is
 * reported by hgr_cuda_plan_sync_status (d_data is then unspecified, the
 * reference's by-value input is preserved by the host/C++ layers). */
int hgr_cuda_plan_decompose(hgr_plan plan, void* d_data, void* stream);
/* decompose out of place: d_in is left untouched (the reference's by-value
 * `decompose(ndarray<T> data, ...)`, refactor.hpp:32-33); fastest path. */
int hgr_cuda_plan_decompose_to(hgr_plan plan, const void* d_in, void* d_out, void* stream);
/* recompose (refactor.hpp:63-90): classes 0..upto_class; d_out may equal d_in. */
int hgr_cuda_plan_recompose(hgr_plan plan, const void* d_in, void* d_out, int upto_class,
                            void* stream);
/* synchronizes `stream`; returns HGR_ERR_NONFINITE if the last decompose saw NaN/Inf */
int hgr_cuda_plan_sync_status(hgr_plan plan, void* stream);

/* Per-launch profile (no reference counterpart; bench/roofline support). When
 * enabled, every launch of the plan is bracketed by CUDA events on its stream
 * and charged to a kernel class with its algorithmic bytes. Classes:
 * 0 fused decompose level, 1 fused recompose level, 2 Thomas passes,
 * 3 recompose interpolation, 4 assembly/gathers, 5 small-level kernels.
 * read_profile synchronizes and returns the totals since set_profiling. */
#define HGR_KIND_COUNT 6
int hgr_cuda_plan_set_profiling(hgr_plan plan, int enable);
int hgr_cuda_plan_read_profile(hgr_plan plan, double* ms, double* bytes, long* launches);

/* Tile-segment autotuning (the reference ranks launch
 * configurations with its sector model, perf_model.hpp:71-137 rank_configs /
 * top_k, and leaves the measuring to its caller). For every level on the
 * fused kernels the segment lengths of the decompose, recompose and
 * interpolation kernels are ranked by the same kind of model and the top three
 * are timed on this device; the fastest is kept by the plan. d_in is read,
 * d_out and the workspace are overwritten. Synchronizes `stream`. The JSON
 * report (per level and kernel: candidates with model and measured times, the
 * heuristic's and the chosen segment) is copied to `report` (truncated to
 * report_bytes - 1 characters; may be NULL); *report_len (may be NULL) gets its
 * full length. */
int hgr_cuda_plan_autotune(hgr_plan plan, const void* d_in, void* d_out, void* stream,
                           char* report, size_t report_bytes, size_t* report_len);
/* back to the built-in segment heuristics */
int hgr_cuda_plan_reset_tuning(hgr_plan plan);

/* Synthetic input (bench/test data): u = a[i]*b[j] + c[k] +
 * 1e-3*eta(seed + flat) with eta from splitmix64 in [-1, 1), computed in
 * double with IEEE-exact mul/add and rounded once to the dtype. The factor
 * tables (host, lengths = extents padded to rank 3 on the right) are supplied
 * by the caller so host and device fields are bitwise identical. */
int hgr_cuda_synthetic_field_f64(const hgr_grid_desc* g, double* d_out, unsigned long long seed,
                                 const double* h_a, const double* h_b, const double* h_c,
                                 void* stream);
int hgr_cuda_synthetic_field_f32(const hgr_grid_desc* g, float* d_out, unsigned long long seed,
                                 const double* h_a, const double* h_b, const double* h_c,
                                 void* stream);

/* ---- one-shot entry points (plan cached by grid + dtype) --------------------
 * C-ABI twins of hgr::decompose<T> / hgr::recompose<T> (refactor.hpp:32-33, :63-64). */
int hgr_cuda_decompose_f64(const hgr_grid_desc* grid, double* d_data, void* stream);
int hgr_cuda_decompose_f32(const hgr_grid_desc* grid, float* d_data, void* stream);
int hgr_cuda_decompose_to_f64(const hgr_grid_desc* grid, const double* d_in, double* d_out,
                              void* stream);
int hgr_cuda_decompose_to_f32(const hgr_grid_desc* grid, const float* d_in, float* d_out,
                              void* stream);
int hgr_cuda_recompose_f64(const hgr_grid_desc* grid, const double* d_in, double* d_out,
                           int upto_class, void* stream);
int hgr_cuda_recompose_f32(const hgr_grid_desc* grid, const float* d_in, float* d_out,
                           int upto_class, void* stream);

/* Host-pointer convenience (synchronous: H2D, run, D2H). This is what the
 * C++ template drop-in (include/hgr_b200/hgr.hpp) calls. decompose checks
 * finiteness before touching h_data (refactor.hpp:36-38). Device buffers are
 * cached per plan; pinned host buffers move by direct DMA, pageable ones
 * through a pinned staging ring with a multi-threaded host copy overlapping
 * the DMA. Thread-safe (plan pool, as above). */
int hgr_decompose_host_f64(const hgr_grid_desc* grid, double* h_data);
int hgr_decompose_host_f32(const hgr_grid_desc* grid, float* h_data);
int hgr_recompose_host_f64(const hgr_grid_desc* grid, const double* h_in, double* h_out,
                           int upto_class);
int hgr_recompose_host_f32(const hgr_grid_desc* grid, const float* h_in, float* h_out,
                           int upto_class);

/* ---- single-level entry points (known-answer-test surface) -----------------
 * Compact level arrays (extents of level `level` / `level-1`), device pointers,
 * synchronous. */
/* interpolate_to_fine (transforms.hpp:76-92) */
int hgr_cuda_interpolate_to_fine_f64(const hgr_grid_desc* g, int level, const double* d_coarse,
                                     double* d_fine, void* stream);
int hgr_cuda_interpolate_to_fine_f32(const hgr_grid_desc* g, int level, const float* d_coarse,
                                     float* d_fine, void* stream);
/* compute_coefficients (transforms.hpp:96-111) */
int hgr_cuda_compute_coefficients_f64(const hgr_grid_desc* g, int level, const double* d_fine,
                                      double* d_coeffs, void* stream);
int hgr_cuda_compute_coefficients_f32(const hgr_grid_desc* g, int level, const float* d_fine,
                                      float* d_coeffs, void* stream);
/* compute_correction (correction.hpp:348-365); rejects nonzero coarse entries */
int hgr_cuda_compute_correction_f64(const hgr_grid_desc* g, int level, const double* d_coeffs,
                                    double* d_z, void* stream);
int hgr_cuda_compute_correction_f32(const hgr_grid_desc* g, int level, const float* d_coeffs,
                                    float* d_z, void* stream);

/* apply_coefficients (transforms.hpp:115-124): fine = interpolate_to_fine(coarse) + coeffs */
int hgr_cuda_apply_coefficients_f64(const hgr_grid_desc* g, int level, const double* d_coarse,
                                    const double* d_coeffs, double* d_fine, void* stream);
int hgr_cuda_apply_coefficients_f32(const hgr_grid_desc* g, int level, const float* d_coarse,
                                    const float* d_coeffs, float* d_fine, void* stream);
int hgr_host_apply_coefficients_f64(const hgr_grid_desc* g, int level, const double* h_coarse,
                                    const double* h_coeffs, double* h_fine);
int hgr_host_apply_coefficients_f32(const hgr_grid_desc* g, int level, const float* h_coarse,
                                    const float* h_coeffs, float* h_fine);

/* Host-pointer twins of the single-level entry points (synchronous), used by
 * the C++ drop-in: op 0 = interpolate_to_fine, 1 = compute_coefficients,
 * 2 = compute_correction. h_in / h_out are compact level arrays. */
int hgr_host_level_op_f64(const hgr_grid_desc* g, int op, int level, const double* h_in,
                          double* h_out);
int hgr_host_level_op_f32(const hgr_grid_desc* g, int op, int level, const float* h_in,
                          float* h_out);
/* Host-pointer fiber operators (correction.hpp:58-223); count fibers of
 * length n: op 0 = mass_apply, 1 = masstrans_apply, 2 = thomas_solve,
 * 3 = transfer_apply, 4 = MassTransOperator::apply_fiber with
 * zero_even_inputs (even fine inputs read as 0, correction.hpp:147-150). */
int hgr_host_fiber_op_f64(int op, size_t n, size_t count, const double* h_v, const double* h_h,
                          double* h_out);
int hgr_host_fiber_op_f32(int op, size_t n, size_t count, const float* h_v, const float* h_h,
                          float* h_out);

/* ---- class packing (refactor.hpp:134-170) ----------------------------------
 * extract_class / scatter_class on the finest-shape pyramid, device pointers.
 * d_values holds class_node_count(cls) values in the reference's row-major order. */
int hgr_cuda_extract_class_f64(const hgr_grid_desc* g, const double* d_data, int cls,
                               double* d_values, void* stream);
int hgr_cuda_extract_class_f32(const hgr_grid_desc* g, const float* d_data, int cls,
                               float* d_values, void* stream);
int hgr_cuda_scatter_class_f64(const hgr_grid_desc* g, double* d_data, int cls,
                               const double* d_values, void* stream);
int hgr_cuda_scatter_class_f32(const hgr_grid_desc* g, float* d_data, int cls,
                               const float* d_values, void* stream);
/* GridHierarchy::class_node_count (grid_hierarchy.hpp:146-150); 0 on error */
size_t hgr_class_node_count(const hgr_grid_desc* g, int cls);
/* GridHierarchy levels (grid_hierarchy.hpp:51-70); -1 on error */
int hgr_levels(const hgr_grid_desc* g);

/* ---- fiber operators (correction.hpp:58-223), batched over `count` fibers --
 * d_v: count fibers of length n (contiguous, fiber-major); d_h: n-1 spacings
 * shared by all fibers. Outputs: mass n, transfer/masstrans (n-1)/2+1, thomas n. */
int hgr_cuda_mass_apply_f64(size_t n, size_t count, const double* d_v, const double* h_h,
                            double* d_out, void* stream);
int hgr_cuda_mass_apply_f32(size_t n, size_t count, const float* d_v, const float* h_h,
                            float* d_out, void* stream);
/* transfer_apply (correction.hpp:67-88): R = P^T, weights refined_node_weights<T> */
int hgr_cuda_transfer_apply_f64(size_t n, size_t count, const double* d_v, const double* h_h,
                                double* d_out, void* stream);
int hgr_cuda_transfer_apply_f32(size_t n, size_t count, const float* d_v, const float* h_h,
                                float* d_out, void* stream);
int hgr_cuda_masstrans_apply_f64(size_t n, size_t count, const double* d_v, const double* h_h,
                                 double* d_out, void* stream);
int hgr_cuda_thomas_solve_f64(size_t n, size_t count, const double* d_rhs, const double* h_h,
                              double* d_out, void* stream);
int hgr_cuda_masstrans_apply_f32(size_t n, size_t count, const float* d_v, const float* h_h,
                                 float* d_out, void* stream);
int hgr_cuda_thomas_solve_f32(size_t n, size_t count, const float* d_rhs, const float* h_h,
                              float* d_out, void* stream);

/* ---- operator tables (host) -------------------------------------------------
 * The builders the plans use, in T and in the reference's arithmetic order:
 * MassTransOperator<T> taps (correction.hpp:96-133), 5 per coarse row over fine
 * 2i-2..2i+2, (n-1)/2+1 rows for n fine nodes; ThomasSolver<T> factors
 * (correction.hpp:188-198): mult n-1, pivot n, upper n-1. h holds n-1 spacings. */
int hgr_masstrans_taps_f64(size_t n, const double* h_h, double* h_taps);
int hgr_masstrans_taps_f32(size_t n, const float* h_h, float* h_taps);
int hgr_thomas_factors_f64(size_t n, const double* h_h, double* h_mult, double* h_pivot,
                           double* h_upper);
int hgr_thomas_factors_f32(size_t n, const float* h_h, float* h_mult, float* h_pivot,
                           float* h_upper);

/* ---- error_report (refactor.hpp:100-120) on the device ------------------------
 * L2 / Linf absolute and relative errors of d_b against d_a (n values each),
 * accumulated in double by a deterministic two-level reduction (no atomics, so
 * run-to-run identical). out[4] = {l2_abs, l2_rel, linf_abs, linf_rel};
 * synchronizes `stream`. */
int hgr_cuda_error_report_f64(size_t n, const double* d_a, const double* d_b, double* h_out,
                              void* stream);
int hgr_cuda_error_report_f32(size_t n, const float* d_a, const float* d_b, double* h_out,
                              void* stream);
/* host-pointer twins (the C++ drop-in's error_report on host ndarrays) */
int hgr_error_report_host_f64(size_t n, const double* h_a, const double* h_b, double* h_out);
int hgr_error_report_host_f32(size_t n, const float* h_a, const float* h_b, double* h_out);

/* ---- the progressive .hg container (storage.hpp:17-218) ----------------------
 * Files are byte-identical to hgr::write_file's. Classes are packed / unpacked
 * on the device (extract_class / scatter_class order) and move as one
 * contiguous payload through pinned staging buffers. Synchronous. */
typedef struct hgr_hg_info {
  unsigned version;          /* HgFileHeader (storage.hpp:36-55) */
  unsigned precision_bytes;  /* 4 or 8 */
  int rank;
  size_t extents[3];
  int class_count;
  uint64_t header_bytes;
  uint64_t file_bytes;
} hgr_hg_info;
/* read_info (storage.hpp:129-177): header and class table only */
int hgr_hg_read_info(const char* path, hgr_hg_info* info);
/* the coordinate table of dimension dim (extents[dim] values) */
int hgr_hg_read_coords(const char* path, int dim, double* h_out);
/* per-class (offset, byte length), coarse first; max_classes entries at most */
int hgr_hg_read_class_table(const char* path, uint64_t* offsets, uint64_t* bytes, int max_classes);
/* write_file (storage.hpp:86-126) of a device pyramid; *bytes_written = file size */
int hgr_cuda_write_hg_f64(const char* path, const hgr_grid_desc* g, const double* d_pyramid,
                          uint64_t* bytes_written, void* stream);
int hgr_cuda_write_hg_f32(const char* path, const hgr_grid_desc* g, const float* d_pyramid,
                          uint64_t* bytes_written, void* stream);
/* read_prefix (storage.hpp:187-216): classes 0..upto_class into a zero-filled
 * device pyramid of the file's extents (hgr_hg_read_info); *bytes_read = header
 * plus the classes read */
int hgr_cuda_read_hg_prefix_f64(const char* path, int upto_class, double* d_pyramid,
                                uint64_t* bytes_read, void* stream);
int hgr_cuda_read_hg_prefix_f32(const char* path, int upto_class, float* d_pyramid,
                                uint64_t* bytes_read, void* stream);
/* host-pointer twins (the C++ drop-in's write_file / read_prefix): the pyramid
 * is staged through the plan's device buffer and packed / scattered there */
int hgr_write_hg_host_f64(const char* path, const hgr_grid_desc* g, const double* h_pyramid,
                          uint64_t* bytes_written);
int hgr_write_hg_host_f32(const char* path, const hgr_grid_desc* g, const float* h_pyramid,
                          uint64_t* bytes_written);
int hgr_read_hg_prefix_host_f64(const char* path, int upto_class, double* h_pyramid,
                                uint64_t* bytes_read);
int hgr_read_hg_prefix_host_f32(const char* path, int upto_class, float* h_pyramid,
                                uint64_t* bytes_read);

#ifdef __cplusplus
}
#endif
#endif /* HGR_CUDA_H */
