// kernels_thomas.cu -- IPK: batched Thomas solves of the mass matrix
// (ThomasSolver::solve_fiber, correction.hpp:202-208; thomas_pass :262-278).
//
// Forward elimination y_i = x_i - m_{i-1} y_{i-1} and back substitution
// z_i = (y_i - u_i z_{i+1}) / p_i are first-order affine recurrences whose
// coefficients are the same for every line of a (level, dimension). A line is
// cut into NC chunks held in registers, one chunk per thread:
//   g = local forward result with zero carry;  y = g + P * c_f
//   h = local backward result of y with zero carry;  z = h + Q * c_b
// where P_i = prod_{k=s..i} (-m_{k-1}) and Q_i = prod_{k=i..e-1} (-u_k / p_k)
// are line-independent tables built once per CTA, and the chunk carries c_f
// (= y at the position before the chunk) and c_b (= z after it) come from an
// exact affine scan over the chunk summaries in shared memory. One HBM read
// and one write per element per dimension, five flops per element.
//
//   k_thomas_lines (dims 0 / 1, strided lines): a group = 32 consecutive
//     lines along the contiguous dimension (lanes) x the whole line (16 warps,
//     one chunk each). Every thread streams its own chunk of the next group
//     into a private shared-memory landing zone with cp.async while it solves
//     the current group from registers; stores are coalesced rows.
//   k_thomas_rows (dim 2, contiguous rows): a group = R consecutive rows, a
//     contiguous block moved by one bulk copy (TMA engine) into a double-buffered
//     shared-memory tile; each row is cut into 16*32/R chunks spread over the
//     lanes; results go back through the tile and one bulk store.
#include <type_traits>

#include "kernels_fused.cuh"
#include "launch.cuh"
#include "plan.hpp"
#include "ptx.cuh"
#include "thomas_chunk.cuh"

namespace hgrb {

namespace {

using namespace thomas;

// ---- strided lines (dims 0 / 1) ---------------------------------------------------

constexpr int kLW = 16;  // warps (= chunks per line) of k_thomas_lines

// Groups: "full" groups (ia, ib) cover lines ib*W .. ib*W+W-1 (W = 32*LPT; lane
// L owns the LPT adjacent lines W*ib + LPT*L + u) along dim 2 of row ia of the
// other strided dim; the c2 % W remaining columns form "tail" groups whose
// threads take W consecutive ia at one column. All offsets are 32-bit (the
// launcher requires < 2^31 elements).
// WIN (lines longer than one group's NP positions): a line is cut into windows
// of NP positions overlapping by 2*H (see k_thomas_long below); groups are
// (window, line group) pairs, window-major, and the tables are rebuilt when a
// CTA moves to another window. The window start ws shifts every position.

template <class T, int CH, int LPT, bool RP, bool WIN>
__global__ void __launch_bounds__(32 * kLW, 1)
    k_thomas_lines(const T* in, T* out, int n, int sd, int so, int na, int c2, int nfull,
                   int ntail, int nlg, int S, int J, const T* __restrict__ mult,
                   const T* __restrict__ rpiv, const T* __restrict__ upper) {
  ptx::pdl_trigger();
  constexpr int NT = 32 * kLW, NC = kLW, GW = 32 * LPT;
  constexpr int CHP = chunk_pitch<T, CH>(), NTB = NC * CHP;
  constexpr int H = window_halo<T>();
  extern __shared__ __align__(16) unsigned char smem_t[];
  T* tm = reinterpret_cast<T*>(smem_t);
  T* tP = tm + NTB;
  T* tp = tP + NTB;
  T* tu = tp + NTB;
  T* tQ = tu + NTB;
  T* sf = tQ + NTB;        // [NC][GW] forward chunk summaries
  T* sb = sf + NC * GW;    // [NC][GW] backward chunk summaries
  T* land = sb + NC * GW;  // [CH][NT][LPT] per-thread landing zone
  if (!WIN) build_tables(tm, tP, tp, tu, tQ, n, NC, CH, CHP, mult, rpiv, upper);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int s0 = w * CH, ts = w * CHP;  // chunk start position, table offset
  const int kmax = n - s0 < CH ? n - s0 : CH;  // valid positions of this warp's chunk (!WIN)
  const int nfull_groups = na * nfull;
  const int ngroups = WIN ? nlg * J : nlg;
  // window of group g (WIN): start position, owned positions [lo, hi)
  auto wstart = [&](int g) { return WIN && J > 1 ? (g / nlg) * S - H : 0; };

  // offset of position 0 of line u of this thread in line group lg (-1: no
  // line); full groups: lines adjacent (offset + u), tail groups: offset + u*so
  auto line_base = [&](int lg, int u) {
    if (lg < nfull_groups) {
      const int ia = int(unsigned(lg) / unsigned(nfull)), ib = lg - ia * nfull;
      return ia * so + ib * GW + LPT * lane + u;
    }
    const int t = lg - nfull_groups;  // tail: GW rows ia at column c2 - ntail + (t % ntail)
    const int ia = (t / ntail) * GW + LPT * lane + u, col = c2 - ntail + t % ntail;
    return ia < na ? ia * so + col : -1;
  };
  // offset of position s0 of line u in group g (!WIN)
  auto line_off = [&](int g, int u) {
    const int b = line_base(g, u);
    return b < 0 ? -1 : b + s0 * sd;
  };
  auto prefetch = [&](int g) {
    T* ld = land + tid * LPT;
    if constexpr (WIN) {
      const int lg = g % nlg, p0 = wstart(g) + s0;
#pragma unroll
      for (int u = 0; u < LPT; ++u) {
        const int off = line_base(lg, u);
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          const int p = p0 + k;
          const bool ok = off >= 0 && p >= 0 && p < n;
          ptx::cp_async_elem<int(sizeof(T))>(ld + k * NT * LPT + u, in + (ok ? off + p * sd : 0),
                                             ok ? int(sizeof(T)) : 0);
        }
      }
    } else if (g < nfull_groups && kmax == CH) {
      const int off = line_off(g, 0);
#pragma unroll
      for (int k = 0; k < CH; ++k) {
#pragma unroll
        for (int u = 0; u < LPT; ++u)
          ptx::cp_async_elem<int(sizeof(T))>(ld + k * NT * LPT + u, in + (off + k * sd + u),
                                             int(sizeof(T)));
      }
    } else if (g < nfull_groups) {
      const T* src = in + line_off(g, 0);
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const int by = k < kmax ? int(sizeof(T)) : 0;
#pragma unroll
        for (int u = 0; u < LPT; ++u)
          ptx::cp_async_elem<int(sizeof(T))>(ld + k * NT * LPT + u, src + u, by);
        if (k + 1 < kmax) src += sd;
      }
    } else {
#pragma unroll
      for (int u = 0; u < LPT; ++u) {
        const int off = line_off(g, u);
        const T* src = in + (off < 0 ? 0 : off);
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          const bool ok = off >= 0 && k < kmax;
          ptx::cp_async_elem<int(sizeof(T))>(ld + k * NT * LPT + u, src, ok ? int(sizeof(T)) : 0);
          if (k + 1 < kmax) src += sd;
        }
      }
    }
    ptx::cp_async_commit();
  };

  // RP (register prefetch, LPT == 1): the next group's chunk is loaded straight
  // into a second register set instead of the shared-memory landing zone
  T nx[RP ? CH : 1];
  auto prefetch_regs = [&](int g) {
    if constexpr (WIN) {
      const int off = line_base(g % nlg, 0), p0 = wstart(g) + s0;
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const int p = p0 + k;
        nx[k] = (off >= 0 && p >= 0 && p < n) ? __ldg(in + off + p * sd) : T(0);
      }
    } else {
      const int off = line_off(g, 0);
      if (off >= 0 && kmax == CH) {  // full chunk: no per-element predicates
#pragma unroll
        for (int k = 0; k < CH; ++k) nx[k] = __ldg(in + (off + k * sd));
      } else {
        const T* src = in + (off < 0 ? 0 : off);
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          nx[k] = (off >= 0 && k < kmax) ? __ldg(src) : T(0);
          if (k + 1 < kmax) src += sd;
        }
      }
    }
  };
  int g = blockIdx.x;
  ptx::pdl_wait();  // the lines are the previous launches' output
  if (g < ngroups) {
    if constexpr (RP) prefetch_regs(g);
    else prefetch(g);
  }
  int cur_w = -1;
  for (; g < ngroups; g += gridDim.x) {
    if constexpr (WIN) {
      const int wi = g / nlg;
      if (wi != cur_w) {  // every thread is past the previous group's table reads
        cur_w = wi;
        __syncthreads();
        build_tables(tm, tP, tp, tu, tQ, n, NC, CH, CHP, mult, rpiv, upper, wstart(g));
      }
    }
    T x[LPT][CH];
    if constexpr (RP) {
#pragma unroll
      for (int k = 0; k < CH; ++k) x[0][k] = nx[k];
      if (g + int(gridDim.x) < ngroups) prefetch_regs(g + gridDim.x);
    } else {
      ptx::cp_async_wait_all();
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        if constexpr (LPT == 2) {
          using T2 = typename std::conditional<sizeof(T) == 8, double2, float2>::type;
          const T2 v = *reinterpret_cast<const T2*>(land + (k * NT + tid) * 2);
          x[0][k] = v.x;
          x[1][k] = v.y;
        } else {
          x[0][k] = land[k * NT + tid];
        }
      }
      if (g + int(gridDim.x) < ngroups) prefetch(g + gridDim.x);
    }

    // forward: local solve, exact carry scan over the chunks before this one
    T e[LPT], c[LPT];
    ChunkSolveV<T, CH, LPT>::fwd_local(x, tm + ts, e);
#pragma unroll
    for (int u = 0; u < LPT; ++u) sf[w * GW + LPT * lane + u] = e[u];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < LPT; ++u) c[u] = T(0);
    for (int v = w > scan_depth<T, CH>() ? w - scan_depth<T, CH>() : 0; v < w; ++v) {
      const T pe = tP[v * CHP + CH - 1];
#pragma unroll
      for (int u = 0; u < LPT; ++u) c[u] = sf[v * GW + LPT * lane + u] + pe * c[u];
    }
    ChunkSolveV<T, CH, LPT>::apply(x, tP + ts, c);
    // backward: local solve, carry scan over the chunks after this one
    ChunkSolveV<T, CH, LPT>::bwd_local(x, tu + ts, tp + ts, e);
#pragma unroll
    for (int u = 0; u < LPT; ++u) sb[w * GW + LPT * lane + u] = e[u];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < LPT; ++u) c[u] = T(0);
    for (int v = w + scan_depth<T, CH>() < NC - 1 ? w + scan_depth<T, CH>() : NC - 1; v > w; --v) {
      const T qs = tQ[v * CHP];
#pragma unroll
      for (int u = 0; u < LPT; ++u) c[u] = sb[v * GW + LPT * lane + u] + qs * c[u];
    }
    ChunkSolveV<T, CH, LPT>::apply(x, tQ + ts, c);

    if constexpr (WIN) {
      const int wi = g / nlg, ws = wstart(g), p0 = ws + s0;
      const int lo = J > 1 ? wi * S : 0, hi = J > 1 && wi * S + S < n ? wi * S + S : n;
#pragma unroll
      for (int u = 0; u < LPT; ++u) {
        const int off = line_base(g % nlg, u);
        if (off < 0) continue;
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          const int p = p0 + k;
          if (p >= lo && p < hi) out[off + p * sd] = x[u][k];
        }
      }
    } else if (g < nfull_groups && kmax == CH) {
      const int off = line_off(g, 0);
#pragma unroll
      for (int k = 0; k < CH; ++k) {
#pragma unroll
        for (int u = 0; u < LPT; ++u) out[off + k * sd + u] = x[u][k];
      }
    } else if (g < nfull_groups) {
      T* dst = out + line_off(g, 0);
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        if (k < kmax) {
#pragma unroll
          for (int u = 0; u < LPT; ++u) dst[u] = x[u][k];
        }
        dst += sd;
      }
    } else {
#pragma unroll
      for (int u = 0; u < LPT; ++u) {
        const int off = line_off(g, u);
        if (off < 0) continue;
        T* dst = out + off;
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          if (k < kmax) *dst = x[u][k];
          dst += sd;
        }
      }
    }
  }
}

// ---- contiguous rows (dim 2) --------------------------------------------------------

template <class T, int CH, int R, bool STAGE>
struct RowsCfg {
  static constexpr int NT = 512, NW = NT / 32;
  static constexpr int CPW = 32 / R;         // chunks per warp
  static constexpr int NC = NW * CPW;        // chunks per row
  static constexpr int NP = NC * CH;
  static constexpr int CHP = chunk_pitch<T, CH>(), NTB = NC * CHP;  // table entries
  // byte offset of the first tile (16-byte aligned)
  static constexpr size_t tiles_off = (size_t(5) * NTB + size_t(2) * NC * R) * sizeof(T) / 16 * 16 + 16;
  // a tile holds R rows of n; the last row's padded chunk positions read up to NP past its start
  static __host__ __device__ size_t buf_elems(int n) {
    return (size_t(R - 1) * n + (NP > n ? NP : n) + 15) / 16 * 16;
  }
  // two input tiles (loads double-buffered) and, with STAGE, one output staging tile
  static size_t smem(int n) {
    return tiles_off + (STAGE ? 3 : 2) * buf_elems(n) * sizeof(T) + 2 * 8;
  }
};

// STAGE: results go to a separate staging tile, so an input tile is refilled as
// soon as its rows are in registers; otherwise results go back into the input
// tile, which is refilled once the bulk store has read it (less shared memory).
template <class T, int CH, int R, bool STAGE>
__global__ void __launch_bounds__(512, 1)
    k_thomas_rows(const T* in, T* out, int64_t rows, int n, const T* __restrict__ mult,
                  const T* __restrict__ rpiv, const T* __restrict__ upper) {
  using C = RowsCfg<T, CH, R, STAGE>;
  ptx::pdl_trigger();
  constexpr int NC = C::NC, CPW = C::CPW, CHP = C::CHP, NTB = C::NTB;
  extern __shared__ __align__(16) unsigned char smem_t[];
  T* tm = reinterpret_cast<T*>(smem_t);
  T* tP = tm + NTB;
  T* tp = tP + NTB;
  T* tu = tp + NTB;
  T* tQ = tu + NTB;
  T* sf = tQ + NTB;      // [NC][R]
  T* sb = sf + NC * R;   // [NC][R]
  const size_t BE = C::buf_elems(n);
  T* buf0 = reinterpret_cast<T*>(smem_t + C::tiles_off);
  T* ot = buf0 + 2 * BE;  // output staging tile (STAGE)
  uint64_t* bar = reinterpret_cast<uint64_t*>(buf0 + (STAGE ? 3 : 2) * BE);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int r = lane % R, q = w * CPW + lane / R, s0 = q * CH, ts = q * CHP;
  const int64_t ngroups = (rows + R - 1) / R;

  // zero the tiles once: positions past a row's end then read finite data
  for (size_t i = tid; i < (STAGE ? 3 : 2) * BE; i += blockDim.x) buf0[i] = T(0);
  build_tables(tm, tP, tp, tu, tQ, n, NC, CH, CHP, mult, rpiv, upper);
  if (tid == 0) {
    ptx::mbar_init(&bar[0], 1);
    ptx::mbar_init(&bar[1], 1);
    ptx::fence_mbar_init();
  }
  ptx::fence_proxy_async_smem();
  __syncthreads();

  auto gbytes = [&](int64_t g) {
    const int64_t nr = (rows - g * R) < R ? (rows - g * R) : R;
    return uint32_t((uint64_t(nr) * n * sizeof(T) + 15) & ~uint64_t(15));
  };
  auto load = [&](int64_t g, int b) {  // tid 0 only
    const uint32_t by = gbytes(g);
    ptx::mbar_arrive_expect_tx(&bar[b], by);
    ptx::bulk_g2s(buf0 + b * BE, in + g * R * int64_t(n), by, &bar[b]);
  };
  int64_t g = blockIdx.x;
  const int64_t G = gridDim.x;
  ptx::pdl_wait();
  if (tid == 0) {
    if (g < ngroups) load(g, 0);
    if (g + G < ngroups) load(g + G, 1);
  }
  for (int it = 0; g < ngroups; g += G, ++it) {
    const int b = it & 1;
    ptx::mbar_wait(&bar[b], uint32_t((it >> 1) & 1));
    const T* mine = buf0 + b * BE + r * n + s0;
    T x[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) x[k] = s0 + k < n ? mine[k] : T(0);  // padding: 0, whatever the tile holds

    sf[q * R + r] = ChunkSolveV<T, CH>::fwd_local(x, tm + ts);
    __syncthreads();
    // every thread has read its chunk: the input tile takes group g + 2G
    if (STAGE && tid == 0 && g + 2 * G < ngroups) load(g + 2 * G, b);
    T c = T(0);
    for (int v = q > scan_depth<T, CH>() ? q - scan_depth<T, CH>() : 0; v < q; ++v)
      c = sf[v * R + r] + tP[v * CHP + CH - 1] * c;
    ChunkSolveV<T, CH>::apply(x, tP + ts, c);
    sb[q * R + r] = ChunkSolveV<T, CH>::bwd_local(x, tu + ts, tp + ts);
    if (STAGE && tid == 0) ptx::bulk_wait_read0();  // the previous store has read `ot`
    __syncthreads();
    c = T(0);
    for (int v = q + scan_depth<T, CH>() < NC - 1 ? q + scan_depth<T, CH>() : NC - 1; v > q; --v)
      c = sb[v * R + r] + tQ[v * CHP] * c;
    ChunkSolveV<T, CH>::apply(x, tQ + ts, c);

    T* dst = (STAGE ? ot : buf0 + b * BE) + r * n + s0;
#pragma unroll
    for (int k = 0; k < CH; ++k)
      if (s0 + k < n) dst[k] = x[k];
    ptx::fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      ptx::bulk_s2g(out + g * R * int64_t(n), STAGE ? ot : buf0 + b * BE, gbytes(g));
      ptx::bulk_commit();
      if (!STAGE && g + 2 * G < ngroups) {
        ptx::bulk_wait_read0();  // the store has read the tile; refill it
        load(g + 2 * G, b);
      }
    }
  }
  if (tid == 0) ptx::bulk_wait0();
}

// ---- long contiguous rows (dim 2, rows beyond the row tiles) ------------------------
//
// A row is cut into windows of NP = 512*CH positions that overlap by 2*H: the
// carry into a window from outside it is dropped, which the damping bound above
// makes invisible (< 2^-B) once H >= B positions away from the window's edges,
// so only the window's middle [H, NP-H) is stored (the whole row when it fits
// one window). Groups = (window, row) pairs, window-major, so a CTA keeps one
// window's per-position factors in registers across consecutive rows.

template <class T, int CH>
struct LongCfg {
  static constexpr int NT = 512, NC = NT, NP = NC * CH;
  static constexpr int TILE = NP + NC;  // one pad element per chunk: conflict-free chunk reads
  // two data tiles, the chunk summaries / products, and one window's three factor
  // tables (same padded layout), prefetched with the data
  static size_t smem() { return (size_t(5) * TILE + size_t(4) * NC) * sizeof(T); }
};

template <class T, int CH>
__global__ void __launch_bounds__(512, 1)
    k_thomas_long(const T* in, T* out, int64_t rows, int64_t n, int64_t S, int64_t J,
                  const T* __restrict__ mult, const T* __restrict__ rpiv,
                  const T* __restrict__ upper) {
  using C = LongCfg<T, CH>;
  ptx::pdl_trigger();
  constexpr int NT = C::NT, NC = C::NC, TILE = C::TILE;
  constexpr int H = window_halo<T>();
  extern __shared__ __align__(16) unsigned char smem_t[];
  T* tile = reinterpret_cast<T*>(smem_t);  // [2][TILE]
  T* sf = tile + 2 * TILE;                 // [NC] forward chunk summaries
  T* sb = sf + NC;                         // [NC] backward chunk summaries
  T* sP = sb + NC;                         // [NC] forward chunk products
  T* sQ = sP + NC;                         // [NC] backward chunk products
  T* fm = sQ + NC;                         // [3][TILE] next window's mult, rpiv, upper
  T* fp = fm + TILE;
  T* fu = fp + TILE;
  const int tid = threadIdx.x, q = tid, s0 = q * CH;
  const int64_t ngroups = rows * J;
  auto wstart = [&](int64_t j) { return J == 1 ? int64_t(0) : j * S - H; };
  auto prefetch = [&](int64_t g, int b) {
    const int64_t j = g / rows, r = g - j * rows, ws = wstart(j);
    const T* row = in + r * n;
    T* t = tile + b * TILE;
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const int i = k * NT + tid;
      const int64_t pos = ws + i;
      const bool ok = pos >= 0 && pos < n;
      ptx::cp_async_elem<int(sizeof(T))>(t + i + i / CH, row + (ok ? pos : 0),
                                         ok ? int(sizeof(T)) : 0);
    }
    ptx::cp_async_commit();
  };
  // window j's factors (zero past the line: padding positions never feed back),
  // issued with a data prefetch so that their latency hides under the current
  // group's solve (1D grids change window on every group)
  auto prefetch_tab = [&](int64_t j) {
    const int64_t ws = wstart(j);
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const int i = k * NT + tid, pi = i + i / CH;
      const int64_t pos = ws + i;
      const bool om = pos >= 1 && pos < n, op = pos >= 0 && pos < n, ou = pos >= 0 && pos < n - 1;
      ptx::cp_async_elem<int(sizeof(T))>(fm + pi, mult + (om ? pos - 1 : 0), om ? int(sizeof(T)) : 0);
      ptx::cp_async_elem<int(sizeof(T))>(fp + pi, rpiv + (op ? pos : 0), op ? int(sizeof(T)) : 0);
      ptx::cp_async_elem<int(sizeof(T))>(fu + pi, upper + (ou ? pos : 0), ou ? int(sizeof(T)) : 0);
    }
  };

  T tm[CH], tp[CH], tu[CH];
  int64_t cur_j = -1;
  int64_t g = blockIdx.x;
  ptx::pdl_wait();
  if (g < ngroups) {
    prefetch_tab(g / rows);
    prefetch(g, 0);
  }
  for (int it = 0; g < ngroups; g += gridDim.x, ++it) {
    const int b = it & 1;
    const int64_t j = g / rows, r = g - j * rows, ws = wstart(j);
    ptx::cp_async_wait_all();
    __syncthreads();  // tile b (and window j's tables) complete; the previous group's store has read tile b^1
    if (j != cur_j) {  // this window's factors, from the prefetched tables
      cur_j = j;
      T a = T(1), c = T(1);
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        tm[k] = fm[s0 + q + k];  // padded index i + i / CH
        tp[k] = fp[s0 + q + k];
        tu[k] = fu[s0 + q + k];
        a *= -tm[k];
        c *= -(tu[k] * tp[k]);
      }
      sP[q] = a;  // read by the scans after the barrier below
      sQ[q] = c;
    }
    if (g + int64_t(gridDim.x) < ngroups) {
      const int64_t jn = (g + int64_t(gridDim.x)) / rows;
      if (jn != j) {  // the tables are overwritten: every thread has its factors
        __syncthreads();
        prefetch_tab(jn);
      }
      prefetch(g + gridDim.x, b ^ 1);
    }
    T* t = tile + b * TILE;
    T x[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) x[k] = t[s0 + q + k];  // padded index i + i / CH

    // forward: local solve, truncated exact carry scan, running-product apply
    sf[q] = ChunkSolve<T, CH>::fwd_local(x, tm);
    __syncthreads();
    T c = T(0);
    for (int v = q > scan_depth<T, CH>() ? q - scan_depth<T, CH>() : 0; v < q; ++v)
      c = sf[v] + sP[v] * c;
    {
      T p = T(1);
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        p *= -tm[k];
        x[k] += p * c;
      }
    }
    // backward
    sb[q] = ChunkSolve<T, CH>::bwd_local(x, tu, tp);
    __syncthreads();
    c = T(0);
    for (int v = q + scan_depth<T, CH>() < NC - 1 ? q + scan_depth<T, CH>() : NC - 1; v > q; --v)
      c = sb[v] + sQ[v] * c;
    {
      T p = T(1);
#pragma unroll
      for (int k = CH - 1; k >= 0; --k) {
        p *= -(tu[k] * tp[k]);
        x[k] += p * c;
      }
    }
#pragma unroll
    for (int k = 0; k < CH; ++k) t[s0 + q + k] = x[k];
    __syncthreads();
    // coalesced store of the window's owned positions
    const int lo = J == 1 ? 0 : H;
    const int64_t hi64 = J == 1 ? n : (j * S + S < n ? j * S + S : n) - ws;
    const int hi = int(hi64);
    T* orow = out + r * n + ws;
    for (int i = lo + tid; i < hi; i += NT) orow[i] = t[i + i / CH];
  }
}

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

template <class T, int CH, int R>
void run_rows(const T* in, T* out, int64_t rows, int64_t n, const T* mult, const T* rpiv,
              const T* upper, cudaStream_t s) {
  constexpr bool STAGE = sizeof(T) == 4;  // fp64's 16-row tiles leave no room for a third
  using C = RowsCfg<T, CH, R, STAGE>;
  const size_t smem = C::smem(int(n));
  auto kern = k_thomas_rows<T, CH, R, STAGE>;
  set_smem_attr(reinterpret_cast<const void*>(kern), smem);
  const int64_t groups = (rows + R - 1) / R;
  const int grid = int(groups < sm_count() ? groups : sm_count());
  launch_pdl(kern, dim3(grid), dim3(C::NT), smem, s, 8 * rows * n, in, out, rows, int(n), mult, rpiv,
             upper);
}

template <class T, int CH, bool WIN>
void run_lines(const T* in, T* out, const int64_t e[3], int dim, const T* mult, const T* rpiv,
               const T* upper, cudaStream_t s) {
  // fp32: the next group's chunk is prefetched into registers (fp64 chunks are
  // too large for a second register set and go through the cp.async landing zone)
  constexpr int LPT = 1;
  constexpr bool RP = sizeof(T) == 4;
  constexpr int NT = 32 * kLW, NP = kLW * CH, GW = 32 * LPT;
  constexpr int NTB = kLW * chunk_pitch<T, CH>();
  const size_t smem =
      (size_t(5) * NTB + 2 * kLW * GW + (RP ? 0 : size_t(CH) * NT * LPT)) * sizeof(T);
  auto kern = k_thomas_lines<T, CH, LPT, RP, WIN>;
  set_smem_attr(reinterpret_cast<const void*>(kern), smem);
  const int n = int(e[dim]);
  const int sd = int(dim == 0 ? e[1] * e[2] : e[2]);
  const int so = int(dim == 0 ? e[2] : e[1] * e[2]);  // stride of the other strided dim
  const int na = int(dim == 0 ? e[1] : e[0]);
  const int c2 = int(e[2]);
  const int nfull = c2 / GW, ntail = c2 % GW;
  const int nlg = na * nfull + ((na + GW - 1) / GW) * ntail;
  const int S = n <= NP ? n : NP - 2 * window_halo<T>();
  const int J = (n + S - 1) / S;
  const int64_t groups = int64_t(nlg) * J;
  const int grid = int(groups < sm_count() ? groups : sm_count());
  launch_pdl(kern, dim3(grid), dim3(NT), smem, s, 8 * e[0] * e[1] * e[2], in, out, n, sd, so, na, c2,
             nfull, ntail, nlg, S,
             J, mult, rpiv, upper);
}

template <class T, int CH>
void run_long(const T* in, T* out, int64_t rows, int64_t n, const T* mult, const T* rpiv,
              const T* upper, cudaStream_t s) {
  using C = LongCfg<T, CH>;
  const int64_t S = n <= C::NP ? n : C::NP - 2 * window_halo<T>();
  const int64_t J = (n + S - 1) / S;
  auto kern = k_thomas_long<T, CH>;
  set_smem_attr(reinterpret_cast<const void*>(kern), C::smem());
  const int64_t groups = rows * J;
  const int grid = int(groups < sm_count() ? groups : sm_count());
  launch_pdl(kern, dim3(grid), dim3(C::NT), C::smem(), s, 8 * rows * n, in, out, rows, n, S, J, mult,
             rpiv,
             upper);
}

// longest rows of the register-tiled row kernels; longer rows take k_thomas_long
template <class T>
constexpr int64_t rows_max() {
  return sizeof(T) == 8 ? 64 * 17 : 32 * 33;
}
constexpr int kLinesMaxCH = 33;
// long rows: fp64 chunks of 8, fp32 chunks of 16 (512 chunks per window)
template <class T>
constexpr int long_ch() {
  return sizeof(T) == 8 ? 8 : 16;
}

}  // namespace

template <class T>
bool thomas_needs_out_of_place(const int64_t e[3], int dim) {
  const int64_t n = e[dim];
  if (dim == 2) return n > rows_max<T>() && n > int64_t(512) * long_ch<T>();
  return n > int64_t(kLW) * kLinesMaxCH;
}

template <class T>
bool launch_thomas_fast(const T* in, T* out, const int64_t e[3], int dim, const T* mult,
                        const T* rpiv, const T* upper, cudaStream_t s) {
  const int64_t n = e[dim];
  if (n < 2) return false;
  if (dim == 2) {
    const int64_t rows = e[0] * e[1];
    if (n > rows_max<T>()) {
      require(in != out || !thomas_needs_out_of_place<T>(e, dim),
              "windowed Thomas pass must run out of place");
      run_long<T, long_ch<T>()>(in, out, rows, n, mult, rpiv, upper, s);
      return true;
    }
    // bulk copies need 16-byte aligned group blocks
    if ((reinterpret_cast<uintptr_t>(in) & 15) || (reinterpret_cast<uintptr_t>(out) & 15))
      return false;
    if constexpr (sizeof(T) == 8) {
      if (n <= 32 * 2) run_rows<T, 2, 16>(in, out, rows, n, mult, rpiv, upper, s);
      else if (n <= 32 * 5) run_rows<T, 5, 16>(in, out, rows, n, mult, rpiv, upper, s);
      else if (n <= 32 * 9) run_rows<T, 9, 16>(in, out, rows, n, mult, rpiv, upper, s);
      else if (n <= 32 * 17) run_rows<T, 17, 16>(in, out, rows, n, mult, rpiv, upper, s);
      else run_rows<T, 17, 8>(in, out, rows, n, mult, rpiv, upper, s);
    } else {
      if (n <= 32 * 2) run_rows<T, 2, 16>(in, out, rows, n, mult, rpiv, upper, s);
      else if (n <= 32 * 5) run_rows<T, 5, 16>(in, out, rows, n, mult, rpiv, upper, s);
      else if (n <= 32 * 9) run_rows<T, 9, 16>(in, out, rows, n, mult, rpiv, upper, s);
      else if (n <= 32 * 17) run_rows<T, 17, 16>(in, out, rows, n, mult, rpiv, upper, s);
      else run_rows<T, 33, 16>(in, out, rows, n, mult, rpiv, upper, s);
    }
    return true;
  }
  if (e[0] * e[1] * e[2] >= (int64_t(1) << 31)) return false;  // 32-bit offsets
  if (n <= kLW * 2) run_lines<T, 2, false>(in, out, e, dim, mult, rpiv, upper, s);
  else if (n <= kLW * 5) run_lines<T, 5, false>(in, out, e, dim, mult, rpiv, upper, s);
  else if (n <= kLW * 9) run_lines<T, 9, false>(in, out, e, dim, mult, rpiv, upper, s);
  else if (n <= kLW * 17) run_lines<T, 17, false>(in, out, e, dim, mult, rpiv, upper, s);
  else if (n <= kLW * kLinesMaxCH) run_lines<T, kLinesMaxCH, false>(in, out, e, dim, mult, rpiv, upper, s);
  else {
    require(in != out, "windowed Thomas pass must run out of place");
    run_lines<T, kLinesMaxCH, true>(in, out, e, dim, mult, rpiv, upper, s);
  }
  return true;
}

template bool thomas_needs_out_of_place<float>(const int64_t*, int);
template bool thomas_needs_out_of_place<double>(const int64_t*, int);
template bool launch_thomas_fast<float>(const float*, float*, const int64_t*, int, const float*,
                                        const float*, const float*, cudaStream_t);
template bool launch_thomas_fast<double>(const double*, double*, const int64_t*, int,
                                         const double*, const double*, const double*,
                                         cudaStream_t);

}  // namespace hgrb
