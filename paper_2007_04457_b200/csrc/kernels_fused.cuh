// kernels_fused.cuh -- launchers of the bandwidth-optimised sm_100a kernels.
#pragma once

#include <vector>

#include "common.cuh"

namespace hgrb {

// Batched Thomas solve of the level-(l-1) mass matrix along `dim` (IPK,
// correction.hpp:202-208 / :262-278), out-of-place allowed (in may equal out).
// Lines are split into chunks held in registers; the chunks are stitched with
// an exact affine carry scan (the forward/backward recurrences are first-order
// affine), then each chunk re-runs the reference recurrence from its true
// carry. Returns false if the line length exceeds the register tiling (the
// caller then uses the one-thread-per-line kernel).
template <class T>
bool launch_thomas_fast(const T* in, T* out, const int64_t ext[3], int dim, const T* mult,
                        const T* rpiv, const T* upper, cudaStream_t s);

// True if the pass along `dim` cuts lines into overlapping windows; such a
// pass must run out of place (in != out).
template <class T>
bool thomas_needs_out_of_place(const int64_t ext[3], int dim);

// IPK of a 3D level in two passes (kernels_band.cu): dim 0 in place on src (the
// strided-line kernel, or a cluster band pass when band_dim0), then dims 1 + 2
// fused per dim-0 plane by thread-block clusters from src into dst (src is
// clobbered; dst may equal src). Returns false (nothing launched) when the
// coarse extents or operands do not fit.
// Streaming IPK of a 3D level (kernels_stream.cu): dim 0 as column strips in
// place on src, then (fp32) dims 1+2 on whole planes src -> dst, or (fp64) dim 1
// strips in place and the dim-2 row kernel src -> dst. Returns the launches
// (0: nothing launched).
template <class T>
bool thomas_stream_supported(const int64_t c[3]);
template <class T>
int launch_thomas_stream(T* src, T* dst, const int64_t c[3], const T* const mult[3],
                         const T* const rpiv[3], const T* const upper[3], const int K[3],
                         int64_t level_nodes, cudaStream_t s);
template <class T>
bool thomas_band_supported(const int64_t c[3]);
template <class T>
bool launch_thomas_planes(T* src, T* dst, const int64_t c[3], const T* const mult[3],
                          const T* const rpiv[3], const T* const upper[3], int64_t level_nodes,
                          bool band_dim0, cudaStream_t s);

// The coarse tail (kernels_tail.cu): levels 1..lt of a plan in one CTA per
// direction. Per level: its arguments and compact buffers.
template <class T>
struct TailLevel {
  LevelArgs<T> a;
  T* src;     // compact level-l array C_l (decompose input; recompose coefficients, in place)
  T* coef;    // D_l: decompose coefficients
  T* coarse;  // C_{l-1}
  T* z;       // Z_l
};
template <class T>
void launch_tail_decompose(const TailLevel<T>* d_levels, int lt, int rank, T* s0, T* s1,
                           cudaStream_t s);
// prefix m: levels <= m use their stored coefficients
template <class T>
void launch_tail_recompose(const TailLevel<T>* d_levels, int lt, int m, int rank, T* s0, T* s1,
                           cudaStream_t s);

enum FusedMode : int {
  kFusedDecompose = 0,  // coefficients -> coef_out, K*U -> zload
  kFusedLoadOnly = 1,   // K*U -> zload only
  kFusedRecompose = 2   // K*(U masked at coarse nodes) -> zload, coarse nodes -> gather
};

// Fused level kernel (GPK + LPK on all dimensions): marches along dim 0 over
// (dim1, dim2) tiles of the level-l array U; fine planes arrive in shared
// memory through cp.async.bulk (TMA bulk-copy engine) into an mbarrier ring.
// Returns false if the level is not supported (caller falls back).
// flag (decompose mode, may be null): set to 1 if any input value is NaN/Inf.
// s0: coarse planes per CTA segment along dim 0 (0 = built-in heuristic).
// side (decompose mode, 2D / 3D, may be null): the coefficients on even rows of
// even planes (odd columns only) go to the compact side rows
// side[((j/2)*c1 + r/2)*(c2-1) + (c-1)/2] instead of coef_out, and those output
// rows are left for launch_merge_even.
template <class T>
bool launch_level_fused(const T* U, T* coef_out, T* zload, T* gather, const LevelArgs<T>& a,
                        int mode, int* flag, cudaStream_t s, int s0 = 0, T* side = nullptr,
                        T* face_ws = nullptr);
// face scratch of launch_level_fused's two-phase faces: e0*e1 + 3*e0*c2 elements
template <class T>
inline int64_t level_face_ws_elems(const int64_t e[3], const int64_t c[3]) {
  return e[0] * e[1] + 3 * e[0] * c[2];
}

// Pyramid assembly of a level decomposed with side rows: every even row of an
// even plane of `out` (level-l extents e) is written whole, its even columns
// from the finished level-(l-1) pyramid `coarse` (compact c) and its odd
// columns from the side rows -- full-sector writes instead of a strided scatter.
// whether k_merge_even's shared-memory ring holds rows of c2 coarse columns
template <class T>
bool merge_even_fits(int64_t c2);
template <class T>
void launch_merge_even(const T* coarse, const T* side, T* out, const LevelArgs<T>& a,
                       cudaStream_t s);

// Recompose interpolation (GPK^-1, refactor.hpp:77-87): coarse = C - Z (Z may be
// null), out[coarse] = coarse, out[refined] = (with ? coef : 0) + interp(coarse).
// 3D tiles with the coarse block staged in shared memory. in-place safe.
// In-place coefficients of a fused level (the in-place decompose): U becomes
// U - interp(C) at refined nodes, C = the gathered coarse nodes; the
// interpolation march in subtract mode; flag: non-finite input seen.
template <class T>
bool launch_coef_inplace(T* U, const T* C, const LevelArgs<T>& a, int* flag, cudaStream_t s,
                         int s0 = 0);
template <class T>
bool launch_interp_rec(const T* coef, T* out, const T* C, const T* Z, const LevelArgs<T>& a,
                       bool with_coeffs, cudaStream_t s, int s0 = 0);

// 1D grids (canonical (1, 1, n)): the fused level / interpolation steps as
// per-coarse-node streams (kernels_line.cu). Return false if not 1D.
template <class T>
bool launch_line_level(const T* U, T* coef, T* z, T* gather, const LevelArgs<T>& a, int mode,
                       int* flag, cudaStream_t s);
template <class T>
bool launch_line_interp(const T* coef, T* out, const T* C, const T* Z, const LevelArgs<T>& a,
                        bool with_coeffs, cudaStream_t s);

// Tile-segment candidates of the level / interpolation kernels ranked by a
// sector-traffic model (the reference's perf_model.hpp:71-100 estimate_time
// restated for these tiles: every row a CTA moves padded to 32-byte sectors,
// reads + writes, times the blocks covering the level, over the bandwidth,
// times the wave-quantisation loss of 148 SMs x resident CTAs). Sorted by
// model time, ties in candidate order. s0 = 0 marks the heuristic's choice.
struct SegChoice {
  int s0;           // coarse planes per CTA segment
  int blocks;       // CTAs launched
  double model_us;  // model time
};
template <class T>
std::vector<SegChoice> level_fused_candidates(const LevelArgs<T>& a, int mode, double bw_gbs);
template <class T>
std::vector<SegChoice> interp_candidates(const LevelArgs<T>& a, bool with_coeffs, bool has_z,
                                         double bw_gbs);
template <class T>
int level_fused_default_s0(const LevelArgs<T>& a);
template <class T>
int interp_default_s0(const LevelArgs<T>& a);

}  // namespace hgrb
