// kernels_level.cu -- fused level kernel for the fine levels: one pass over a
// level-l array U does the GPK and the three LPK passes (paper kernel classes
// 1 and 2; transforms.hpp:20-65, correction.hpp:141-154 / :238-260).
//
//   A CTA (16 warps) owns a (dim1, dim2) tile of TW1 x 64 coarse outputs and
//   marches along dim 0 over a segment of coarse planes. Each fine plane's halo
//   window (2*TW1+3 rows x 131 columns) arrives in shared memory through 1D TMA
//   tensor copies, one per window row, issued by lane 0 of every warp into an
//   NS-slot mbarrier ring. A TMA box must start 16-byte aligned and 2^k+1 row
//   pitches give every row its own phase, so each row lands as its aligned
//   superset and readers offset by the row's phase. (Streaming probe
//   tools/mb/stream_mb.cu on B200: warp-issued 1D TMA rows of this geometry move
//   7.0 TB/s of unique data; 16-byte cp.async by all threads 3.4 TB/s.)
//
//   Row stage (every window row of a plane): the two warp groups own coarse
//   columns [0, 32) and [32, 64); lane L of group G owns coarse column
//   t = 32G + L, window columns 2t..2t+4 and fine cells 2t+2, 2t+3 (loads of
//   consecutive lanes are consecutive, so shared-memory reads are conflict
//   free). From the five values it forms
//     * P2 = K2 u at its coarse column (the fused mass-trans stencil K = R*M of
//       correction.hpp:96-133 applied directly, 5 taps; in recompose mode the
//       coarse nodes of even rows of even planes are masked, correction.hpp:251)
//       -> shared P2 row;
//     * decompose: the interpolant of its two cells (dim-2 blend on even rows;
//       on odd rows the blend of the even rows above / below: the warps of a
//       group own bands of four rows starting on an even row and look one row
//       ahead), the coefficients u - interp of even planes and -- deferred by
//       one plane -- of the odd plane behind it, whose interpolant blends the
//       previous even plane's (kept in registers) with the current one
//       (transforms.hpp:41-55 evaluated as a separable product);
//     * recompose: the coarse nodes of even rows of even planes gathered into
//       the compact level-(l-1) array.
//   Column stage (the previous plane): thread (s, 2 columns) applies K1 (5
//   taps over the P2 rows) and accumulates K0 across planes in registers; a
//   completed coarse plane is stored to the load vector zload.
//   Decompose applies K to U itself: K*P = M_c exactly for nested hat spaces,
//   so M_c^-1 K U = RU + M_c^-1 K (U - P R U) = coarse + z and the three Thomas
//   passes on zload give the corrected coarse values (refactor.hpp:48-54).
//   The last coarse row and column of a level (and the fine row / column on
//   them) are the faces of k_level_face, so every tile is a full TW1 x 64 block
//   or a clipped one.
#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstdlib>

#include "kernels.cuh"
#include "kernels_fused.cuh"
#include "plan.hpp"
#include "ptx.cuh"
#include "launch.cuh"
#include "tma.hpp"

namespace hgrb {

namespace {

constexpr int kMaxSeg = 64;  // coarse planes per dim-0 segment (S0 <= kMaxSeg)

template <class T>
struct LCfg {
  // fp64: lane = 1 coarse column, tile 16 x 32, 8 warps, two CTAs per SM;
  // fp32: lane = 2 coarse columns (16-byte loads), tile 16 x 64, 8 warps, two CTAs per SM
  static constexpr int CPL = sizeof(T) == 8 ? 1 : 2;           // coarse columns per lane
  static constexpr int NG = 1;                                 // column groups
  static constexpr int NT = 256, NW = NT / 32, WG = NW / NG;
  static constexpr int MINB = 2;                               // CTAs per SM
  static constexpr int TW2 = 32 * CPL * NG;                    // coarse columns
  static constexpr int TW1 = 16;                               // coarse rows
  static constexpr int NS = 4;                                 // ring slots
  static constexpr int V = 16 / int(sizeof(T));                // elements per 16 bytes
  static constexpr int RW = 2 * TW1 + 3, CW = 2 * TW2 + 3;     // window rows / columns
  static constexpr int NB = TW1 / 2;                           // bands of 4 owned rows
  static_assert(NB <= WG, "one band per warp of a group");
  static constexpr int NCELL = 2 * CPL, NV = 2 * CPL + 3;      // cells / window values per lane
  static constexpr int BOX = (CW + V - 1 + V - 1) / V * V;     // aligned superset of a row
  static constexpr int ALN = 128 / int(sizeof(T));             // TMA smem alignment (128 B)
  static constexpr int PITCH = (BOX + ALN - 1) / ALN * ALN;
  static_assert(PITCH >= CW + 2 * V, "vector reads stay inside the row");
  static constexpr int SLOT = RW * PITCH;
  static constexpr int P2W = TW2;
  static constexpr int CQ = V;                                 // column-stage columns per item
  static constexpr int NQ = TW1 * (TW2 / CQ);                  // column-stage work items
  static_assert(NQ <= NT, "one column-stage item per thread");
  static constexpr int K0N = kMaxSeg + 6;                      // K0 tap rows ka-2 .. kb+1
  static constexpr int W0N = kMaxSeg + 4;                      // dim-0 weights ka-1 .. kb+2
  static constexpr size_t raw_bytes = size_t(NS) * SLOT * sizeof(T);
  static constexpr size_t p2_off = raw_bytes;
  static constexpr size_t k0_off = p2_off + size_t(2) * RW * P2W * sizeof(T);
  static constexpr size_t w0_off = k0_off + size_t(K0N) * 5 * sizeof(T);
  static constexpr size_t bar_off = (w0_off + size_t(2) * W0N * sizeof(T) + 15) / 16 * 16;
  static constexpr size_t total = bar_off + NS * sizeof(uint64_t);
  static_assert(total * MINB <= 227 * 1024, "shared memory budget");
};

template <class T>
struct Vec2;
template <>
struct Vec2<double> { using type = double2; };
template <>
struct Vec2<float> { using type = float2; };

// v[k] = row[pos + k], k < 5, pos = ph + (even base): pairs by 2-element vector loads
template <class T>
__device__ __forceinline__ void load5(const T* row, int pos, T (&v)[5]) {
  using T2 = typename Vec2<T>::type;
  if (!(pos & 1)) {
    const T2 x = *reinterpret_cast<const T2*>(row + pos);
    const T2 y = *reinterpret_cast<const T2*>(row + pos + 2);
    v[0] = x.x; v[1] = x.y; v[2] = y.x; v[3] = y.y; v[4] = row[pos + 4];
  } else {
    const T2 x = *reinterpret_cast<const T2*>(row + pos + 1);
    const T2 y = *reinterpret_cast<const T2*>(row + pos + 3);
    v[0] = row[pos]; v[1] = x.x; v[2] = x.y; v[3] = y.x; v[4] = y.y;
  }
}
// fp32: v[k] = row[base + ph + k], k < 7, base a multiple of 4 (16-byte float4 loads)
template <int PH>
__device__ __forceinline__ void load7f(const float* row, int base, float (&v)[7]) {
  const float4* p = reinterpret_cast<const float4*>(row + base);
  const float4 a = p[0], b = p[1];
  float w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, 0.f, 0.f, 0.f, 0.f};
  if constexpr (PH >= 2) {
    const float4 c = p[2];
    w[8] = c.x; w[9] = c.y; w[10] = c.z; w[11] = c.w;
  }
#pragma unroll
  for (int k = 0; k < 7; ++k) v[k] = w[k + PH];
}
// fp64 with a compile-time parity of pos = base + PH (base even)
template <class T, int PH>
__device__ __forceinline__ void load5c(const T* row, int base, T (&v)[5]) {
  using T2 = typename Vec2<T>::type;
  const int pos = base + PH;
  if constexpr (PH == 0) {
    const T2 x = *reinterpret_cast<const T2*>(row + pos);
    const T2 y = *reinterpret_cast<const T2*>(row + pos + 2);
    v[0] = x.x; v[1] = x.y; v[2] = y.x; v[3] = y.y; v[4] = row[pos + 4];
  } else {
    const T2 x = *reinterpret_cast<const T2*>(row + pos + 1);
    const T2 y = *reinterpret_cast<const T2*>(row + pos + 3);
    v[0] = row[pos]; v[1] = x.x; v[2] = x.y; v[3] = y.x; v[4] = y.y;
  }
}
// loadV with the row phase known at compile time (no per-row dispatch)
template <class T, int NV, int PH>
__device__ __forceinline__ void loadVc(const T* row, int base, T (&v)[NV]) {
  if constexpr (NV == 5) load5c<T, PH>(row, base, v);
  else load7f<PH>(row, base, v);
}
template <int N>
using IC = std::integral_constant<int, N>;

// the lane's window values: NV = 2*CPL+3 values starting at window column base
template <class T, int NV>
__device__ __forceinline__ void loadV(const T* row, int ph, int base, T (&v)[NV]) {
  if constexpr (NV == 5) {
    load5<T>(row, ph + base, v);
  } else {
    static_assert(NV == 7 && sizeof(T) == 4, "fp32 lanes own two coarse columns");
    switch (ph) {
      case 0: load7f<0>(row, base, v); break;
      case 1: load7f<1>(row, base, v); break;
      case 2: load7f<2>(row, base, v); break;
      default: load7f<3>(row, base, v); break;
    }
  }
}

// E1C, E2C: the extents of dims 1 and 2 at compile time (the 2^k+1 shapes of the
// large levels; 0 = run time), so the address arithmetic folds
template <class T, int MODE, int E1C = 0, int E2C = 0>
__global__ void __launch_bounds__(LCfg<T>::NT, LCfg<T>::MINB)
    k_level_fused(const __grid_constant__ CUtensorMap map, int64_t map_off, T* __restrict__ coef_out,
                  T* __restrict__ zload, T* __restrict__ gather, T* __restrict__ side, LevelArgs<T> a,
                  int S0, int nt1, int nt2, int nseg, int seg_base, int* flag) {
  using C = LCfg<T>;
  using T2 = typename Vec2<T>::type;
  ptx::pdl_trigger();
  constexpr int V = C::V, PITCH = C::PITCH, SLOT = C::SLOT, NS = C::NS, NT = C::NT;
  constexpr int TW1 = C::TW1, TW2 = C::TW2, P2W = C::P2W, NW = C::NW, NB = C::NB, WG = C::WG;
  constexpr int CPL = C::CPL, NCELL = C::NCELL, NV = C::NV, CQ = C::CQ;
  constexpr bool DEC = MODE == kFusedDecompose, REC = MODE == kFusedRecompose;
  extern __shared__ __align__(128) unsigned char smem[];
  T* raw = reinterpret_cast<T*>(smem);
  T* p2 = reinterpret_cast<T*>(smem + C::p2_off);
  T* k0t = reinterpret_cast<T*>(smem + C::k0_off);
  T* w0t = reinterpret_cast<T*>(smem + C::w0_off);  // [2][W0N]: wl, wr of dim-0 intervals
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::bar_off);

  const int tid = threadIdx.x, lane = tid & 31, warp = ptx::warp_id_uniform();
  const int64_t e0 = a.e[0], e1 = E1C ? E1C : a.e[1], e2 = E2C ? E2C : a.e[2];
  const int64_t c0 = a.c[0], c1 = E1C ? (E1C + 1) / 2 : a.c[1], c2 = E2C ? (E2C + 1) / 2 : a.c[2];
  const int64_t plane_sz = e1 * e2;
  int bid = blockIdx.x;
  const int t2i = bid % nt2;
  bid /= nt2;
  const int t1i = bid % nt1;
  const int seg = seg_base + bid / nt1;
  const bool lastseg = seg == nseg - 1;
  // tiles cover coarse rows / columns [0, c-1); the last coarse row and column
  // (and the fine row / column on them) are the faces of k_level_face
  const int64_t q1a = int64_t(t1i) * TW1, q2a = int64_t(t2i) * TW2;
  const int tw1 = int(c1 - 1 - q1a < TW1 ? c1 - 1 - q1a : TW1);
  const int tw2 = int(c2 - 1 - q2a < TW2 ? c2 - 1 - q2a : TW2);
  const int64_t ka = int64_t(seg) * S0;
  const int64_t kb = lastseg ? c0 : ka + S0;
  const int64_t wr0 = 2 * q1a - 2, wc0 = 2 * q2a - 2;
  const int RWn = 2 * tw1 + 3;
  const int64_t j0 = (2 * ka - 2) > 0 ? (2 * ka - 2) : 0;
  const int64_t jend = (2 * kb) < (e0 - 1) ? (2 * kb) : (e0 - 1);
  const int orows = 2 * tw1;  // owned fine rows: window rows [2, 2 + orows)

  // ---- per-lane columns: coarse t0..t0+CPL-1 (tile-local), window columns 2t0.. -------
  const int grp = warp / WG, wg = warp % WG;
  const int t0 = CPL * (32 * grp + lane);
  const int wb = 2 * t0;  // first window column of the lane
  T k2[CPL][5];
  T hl[CPL], hr[CPL];  // interpolation weights of the odd cells 2t+3
  bool cvalid[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int64_t tg = q2a + t0 + c;
    cvalid[c] = t0 + c < tw2;
#pragma unroll
    for (int k = 0; k < 5; ++k) k2[c][k] = cvalid[c] ? a.taps[2][tg * 5 + k] : T(0);
    hl[c] = (DEC && cvalid[c]) ? a.wl[2][tg] : T(0);
    hr[c] = (DEC && cvalid[c]) ? a.wr[2][tg] : T(0);
  }

  // ---- per-warp row band: owned rows [b, b+4), lookahead row b+4 ---------------------
  const bool has_band = wg < NB;
  const int b = 2 + 4 * wg;
  bool rown[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) rown[i] = has_band && b + i - 2 < orows;
  T w1l[2] = {T(0), T(0)}, w1r[2] = {T(0), T(0)};  // odd rows b+1, b+3
  if (DEC && has_band) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int64_t gr = wr0 + b + 1 + 2 * i;
      if (gr < e1 - 1) { w1l[i] = a.wl[1][gr >> 1]; w1r[i] = a.wr[1][gr >> 1]; }
    }
  }
  // K-only rows outside the bands: window rows 0, 1 (the last window row is the
  // lookahead row of the last band)
  const int xr0 = (wg == WG - 1) ? 0 : -1;
  const int xr1 = (NB < WG) ? ((wg == WG - 1) ? 1 : -1) : ((wg == WG - 2) ? 1 : -1);
  const bool krow_look = wg == NB - 1;

  // ---- column stage item: coarse row s, columns cq..cq+CQ-1 ---------------------------
  const bool qv = tid < C::NQ;
  const int s = tid / (TW2 / CQ), cq = CQ * (tid % (TW2 / CQ));
  T k1[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) k1[k] = (qv && s < tw1) ? a.taps[1][(q1a + s) * 5 + k] : T(0);

  // ---- TMA issue: window row r of plane jj lands as its aligned box at slot row r
  int nrows_in = 0;
  for (int r = 0; r < RWn; ++r) nrows_in += (wr0 + r >= 0 && wr0 + r < e1) ? 1 : 0;
  const uint32_t tx_bytes = uint32_t(nrows_in) * C::BOX * uint32_t(sizeof(T));
  // per issuing lane (lane 0 of warp w: rows w, w+NW, ...): 32-bit TMA coordinate of
  // window column 0 of the row in plane 0 relative to the map base (arithmetic
  // modulo 2^32: the true coordinates of a launch lie in [-2, 2^31))
  constexpr int RPW = (C::RW + NW - 1) / NW;
  uint32_t rc[RPW];
  unsigned rvalid = 0;
#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    const int r = warp + NW * i;
    const int64_t gr = wr0 + r;
    rc[i] = uint32_t(uint64_t(gr * e2 + wc0 - map_off));
    if (r < RWn && gr >= 0 && gr < e1) rvalid |= 1u << i;
  }
  const uint32_t raw_s = ptx::smem_addr(raw) + uint32_t(warp * PITCH * sizeof(T));
  const uint32_t bar_s = ptx::smem_addr(bar);
  auto issue = [&](int64_t jj) {
    const int sl = int(jj - j0) % NS;
    if (tid == 0) ptx::mbar_arrive_expect_tx(&bar[sl], tx_bytes);
    if (ptx::elect_one()) {
      const uint32_t dst = raw_s + uint32_t(sl * SLOT * sizeof(T));
      const uint32_t bs = bar_s + uint32_t(sl * sizeof(uint64_t));
      const uint32_t pb = uint32_t(uint64_t(jj * plane_sz));
#pragma unroll
      for (int i = 0; i < RPW; ++i)
        if (rvalid & (1u << i))
          ptx::tma_load_1d_s(dst + uint32_t(i * NW * PITCH * sizeof(T)), &map,
                             int((pb + rc[i]) & ~uint32_t(V - 1)), bs);
    }
  };

  // zero the ring once (rows outside the domain are never copied and stay 0)
  for (int i = tid; i < int(C::k0_off / sizeof(T)); i += NT) raw[i] = T(0);
  ptx::fence_proxy_async_smem();
  for (int i = tid; i < C::K0N * 5; i += NT) {
    const int64_t ci = ka - 2 + i / 5;
    const int k = i % 5;
    T v = T(0);
    if (e0 == 1) v = (ci == 0 && k == 2) ? T(1) : T(0);
    else if (ci >= 0 && ci < c0 && ci <= kb + 1) v = a.taps[0][ci * 5 + k];
    k0t[i] = v;
  }
  for (int i = tid; i < C::W0N; i += NT) {
    const int64_t q = ka - 1 + i;  // dim-0 interval of odd plane 2q+1
    const bool ok = DEC && e0 > 1 && q >= 0 && q < c0 - 1;
    w0t[i] = ok ? a.wl[0][q] : T(0);
    w0t[C::W0N + i] = ok ? a.wr[0][q] : T(0);
  }
  if (tid == 0) {
    for (int q = 0; q < NS; ++q) ptx::mbar_init(&bar[q], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int nplanes = int(jend - j0 + 1);
  ptx::pdl_wait();  // U is the previous launches' output
  for (int p = 0; p < nplanes && p < NS; ++p) issue(j0 + p);

  const int e2m = int(e2 & (V - 1));
  // rows and planes advance the phase by one (every 2^k+1 extent with k >= 2)
  const bool ph_regular = e2m == 1 && (plane_sz & (V - 1)) == 1;
  // vector coefficient stores: whole tile row owned, and coef_out and U on the
  // same 16-byte phase (both 16-byte aligned), so a cell's global phase is its
  // window phase; lanes start their cells on a 16-byte window boundary + 2
  const bool vstore = DEC && tw2 == TW2 &&
                      ((reinterpret_cast<uintptr_t>(coef_out) & 15) == 0) && (wb % V) == 0 &&
                      ((map_off & (V - 1)) == 0);
  const int ph00 = int((wr0 * e2 + wc0) & (V - 1));
  // phase (shared-memory position of window column 0) of row r in a plane of phase phj
  auto plane_ph = [&](int64_t jj) { return int((jj * plane_sz + ph00) & (V - 1)); };
  auto rph = [&](int phj, int r) { return (phj + r * e2m) & (V - 1); };

  T acc0[CQ], acc1[CQ], acc2[CQ];
#pragma unroll
  for (int k = 0; k < CQ; ++k) acc0[k] = acc1[k] = acc2[k] = T(0);
  T A1p[4][NCELL];  // interpolant of the previous even plane at this lane's band cells
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int k = 0; k < NCELL; ++k) A1p[i][k] = T(0);
  T bad = T(0);

  // K2 of one row at the lane's coarse columns -> P2 row
  auto k2row = [&](const T (&v)[NV], bool masked, T* P2row) {
    T pv[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const T* u = v + 2 * c;
      if (REC && masked)
        pv[c] = k2[c][1] * u[1] + k2[c][3] * u[3];
      else
        pv[c] = (k2[c][0] * u[0] + k2[c][1] * u[1] + k2[c][2] * u[2]) +
                (k2[c][3] * u[3] + k2[c][4] * u[4]);
    }
    if constexpr (CPL == 1) {
      P2row[t0] = pv[0];
    } else {
      T2 w;
      w.x = pv[0];
      w.y = pv[1];
      *reinterpret_cast<T2*>(P2row + t0) = w;
    }
  };

  // column stage for plane jj: K1 over the P2 rows, K0 into the accumulators
  auto column_stage = [&](int64_t jj) {
    if (!qv) return;
    const T* P2 = p2 + (jj & 1) * (C::RW * P2W) + 2 * s * P2W + cq;
    T P[CQ];
#pragma unroll
    for (int k = 0; k < CQ; ++k) P[k] = T(0);
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      if constexpr (CQ == 2) {
        const T2 x = *reinterpret_cast<const T2*>(P2 + k * P2W);
        P[0] += k1[k] * x.x;
        P[1] += k1[k] * x.y;
      } else {
        const float4 x = *reinterpret_cast<const float4*>(P2 + k * P2W);
        P[0] += k1[k] * x.x;
        P[1] += k1[k] * x.y;
        P[2] += k1[k] * x.z;
        P[3] += k1[k] * x.w;
      }
    }
    const int64_t E = (jj & 1) ? jj + 1 : jj;
    const int ib0 = int(E / 2 - 1 - (ka - 2));  // K0 table row of coarse plane E/2 - 1
    T kA, kB, kC;
    if (!(jj & 1)) {
      kA = k0t[ib0 * 5 + 4];
      kB = k0t[(ib0 + 1) * 5 + 2];
      kC = k0t[(ib0 + 2) * 5 + 0];
    } else {
      kA = k0t[ib0 * 5 + 3];
      kB = k0t[(ib0 + 1) * 5 + 1];
      kC = T(0);
    }
#pragma unroll
    for (int k = 0; k < CQ; ++k) {
      acc0[k] += kA * P[k];
      acc1[k] += kB * P[k];
      acc2[k] += kC * P[k];
    }
  };
  // store coarse plane i (acc0) if this segment owns it, then rotate
  auto flush = [&](int64_t i) {
    if (qv && i >= ka && i < kb && s < tw1) {
      T* zr = zload + (i * c1 + q1a + s) * c2 + q2a + cq;
#pragma unroll
      for (int k = 0; k < CQ; ++k)
        if (cq + k < tw2) zr[k] = acc0[k];
    }
#pragma unroll
    for (int k = 0; k < CQ; ++k) {
      acc0[k] = acc1[k];
      acc1[k] = acc2[k];
      acc2[k] = T(0);
    }
  };

  for (int64_t j = j0; j <= jend; ++j) {
    const int p = int(j - j0);
    const int sl = p % NS;
    ptx::mbar_wait(&bar[sl], uint32_t((p / NS) & 1));
    const T* S = raw + sl * SLOT;
    T* P2 = p2 + (j & 1) * (C::RW * P2W);
    const bool jodd = j & 1;
    const int phj = plane_ph(j);

    // ---- row stage ----
#pragma unroll
    for (int xi = 0; xi < 2; ++xi) {  // K-only rows 0, 1
      const int xr = xi ? xr1 : xr0;
      if (xr >= 0) {
        T v[NV];
        loadV<T, NV>(S + xr * PITCH, rph(phj, xr), wb, v);
        k2row(v, !jodd && !(xr & 1), P2 + xr * P2W);
      }
    }
    if (has_band) {
      if (jodd || !DEC) {
        // K path only (odd planes; recompose / load-only modes); PH: the row's
        // phase, or -1 to dispatch at run time
        auto krow = [&](auto i_c, auto ph_c) {
          constexpr int i = decltype(i_c)::value, PH = decltype(ph_c)::value;
          const int r = b + i;
          if (i == 4 && !krow_look) return;
          T v[NV];
          if constexpr (PH >= 0) loadVc<T, NV, PH>(S + r * PITCH, wb, v);
          else loadV<T, NV>(S + r * PITCH, rph(phj, r), wb, v);
          const bool masked = !jodd && !(r & 1);
          k2row(v, masked, P2 + r * P2W);
          if ((REC || (MODE == kFusedLoadOnly && gather != nullptr)) && masked && i < 4 &&
              rown[i] && j >= 2 * ka && j < 2 * kb) {
            // gather the coarse nodes of this row into C_{l-1}
            T* gd = gather + ((j >> 1) * c1 + ((wr0 + r) >> 1)) * c2 + q2a + t0;
#pragma unroll
            for (int c = 0; c < CPL; ++c)
              if (cvalid[c]) gd[c] = v[2 + 2 * c];
          }
        };
        auto krows = [&](auto phb_c) {
          constexpr int P = decltype(phb_c)::value;
          auto ph = [](auto ic) { return IC<P < 0 ? -1 : (P + decltype(ic)::value) & (V - 1)>{}; };
          krow(IC<0>{}, ph(IC<0>{}));
          krow(IC<1>{}, ph(IC<1>{}));
          krow(IC<2>{}, ph(IC<2>{}));
          krow(IC<3>{}, ph(IC<3>{}));
          krow(IC<4>{}, ph(IC<4>{}));
        };
        if (ph_regular) {
          const int phb = (phj + b * e2m) & (V - 1);
          if constexpr (V == 2) {
            if (phb == 0) krows(IC<0>{});
            else krows(IC<1>{});
          } else {
            switch (phb) {
              case 0: krows(IC<0>{}); break;
              case 1: krows(IC<1>{}); break;
              case 2: krows(IC<2>{}); break;
              default: krows(IC<3>{}); break;
            }
          }
        } else {
          krows(IC<-1>{});
        }
      } else {
        // decompose, even plane j: K path, coefficients of j and of the odd
        // plane j-1 behind it (deferred), interpolants kept for plane j+1
        const bool own_e = j >= 2 * ka && j < 2 * kb;
        const bool own_o = j > j0 && j - 1 >= 2 * ka && j - 1 < 2 * kb;
        const int iw = int(((j - 1) >> 1) - (ka - 1));
        const T w0l = own_o ? w0t[iw] : T(0), w0r = own_o ? w0t[C::W0N + iw] : T(0);
        const T* So = raw + ((p + NS - 1) % NS) * SLOT;  // slot of plane j-1
        const int phm = plane_ph(j - 1);
        T* orow_e = coef_out + (j * e1 + wr0 + b) * e2 + wc0 + wb + 2;
        T* orow_o = orow_e - plane_sz;
        T A2e[3][NCELL];  // dim-2 interpolants of the even rows b, b+2, b+4
        // row order b, b+2, b+1, b+4, b+3: odd rows see both even neighbours.
        // One step per row; PH / PHO: the row's phase in plane j / j-1, or -1 to
        // dispatch at run time.
        auto step_row = [&](auto step_c, auto ph_c, auto pho_c) {
          constexpr int step = decltype(step_c)::value;
          constexpr int i = step == 0 ? 0 : step == 1 ? 2 : step == 2 ? 1 : step == 3 ? 4 : 3;
          constexpr int PH = decltype(ph_c)::value, PHO = decltype(pho_c)::value;
          const int r = b + i;
          T v[NV];
          if constexpr (PH >= 0) loadVc<T, NV, PH>(S + r * PITCH, wb, v);
          else loadV<T, NV>(S + r * PITCH, rph(phj, r), wb, v);
          if (i < 4 || krow_look) k2row(v, false, P2 + r * P2W);
          if constexpr (!(i & 1)) {
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
              A2e[i >> 1][2 * c] = v[2 + 2 * c];
              A2e[i >> 1][2 * c + 1] = hl[c] * v[2 + 2 * c] + hr[c] * v[4 + 2 * c];
            }
          }
          if constexpr (i != 4) {
            T A1[NCELL];
#pragma unroll
            for (int k = 0; k < NCELL; ++k)
              A1[k] = (i & 1) ? w1l[i >> 1] * A2e[i >> 1][k] + w1r[i >> 1] * A2e[(i >> 1) + 1][k]
                              : A2e[i >> 1][k];
            if (rown[i]) {
              if (own_e) {
                T* o = orow_e + int64_t(i) * e2;
                T cv[NCELL];
#pragma unroll
                for (int k = 0; k < NCELL; ++k) {
                  cv[k] = v[2 + k] - A1[k];
                  bad = cv[k] * T(0) + bad;
                }
                if (!(i & 1) && side != nullptr) {
                  // even row of an even plane: its odd cells go to the compact side
                  // rows; the output row is written whole by k_merge_even
                  T* sr = side + ((j >> 1) * c1 + ((wr0 + r) >> 1)) * (c2 - 1) + q2a + t0;
                  if constexpr (CPL == 2) {
                    if (cvalid[0] && cvalid[1]) {
                      T2 w;
                      w.x = cv[1];
                      w.y = cv[3];
                      *reinterpret_cast<T2*>(sr) = w;
                    } else if (cvalid[0]) {
                      sr[0] = cv[1];
                    }
                  } else {
                    if (cvalid[0]) sr[0] = cv[1];
                  }
                } else
                // the cells' global phase equals the input's: window phase + 2
                if constexpr (PH >= 0) {
                  if (vstore) {
                    store_cells<T, NCELL, (PH + 2) & (V - 1)>(o, cv);
                  } else {
#pragma unroll
                    for (int k = 0; k < NCELL; ++k)
                      if (cvalid[k >> 1]) o[k] = cv[k];
                  }
                } else {
#pragma unroll
                  for (int k = 0; k < NCELL; ++k)
                    if (cvalid[k >> 1]) o[k] = cv[k];
                }
              }
              if (own_o) {
                T u[NV];
                if constexpr (PHO >= 0) loadVc<T, NV, PHO>(So + r * PITCH, wb, u);
                else loadV<T, NV>(So + r * PITCH, rph(phm, r), wb, u);
                T* o = orow_o + int64_t(i) * e2;
                T cv[NCELL];
#pragma unroll
                for (int k = 0; k < NCELL; ++k) {
                  cv[k] = u[2 + k] - (w0l * A1p[i][k] + w0r * A1[k]);
                  bad = cv[k] * T(0) + bad;
                }
                if constexpr (PHO >= 0) {
                  if (vstore) {
                    store_cells<T, NCELL, (PHO + 2) & (V - 1)>(o, cv);
                  } else {
#pragma unroll
                    for (int k = 0; k < NCELL; ++k)
                      if (cvalid[k >> 1]) o[k] = cv[k];
                  }
                } else {
#pragma unroll
                  for (int k = 0; k < NCELL; ++k)
                    if (cvalid[k >> 1]) o[k] = cv[k];
                }
              }
            }
#pragma unroll
            for (int k = 0; k < NCELL; ++k) A1p[i][k] = A1[k];
          }
        };
        // 2^k+1 extents: rows and planes advance the phase by one, bands start on
        // multiples of four rows, so the five rows' phases follow from plane j's
        auto steps = [&](auto phb_c) {
          constexpr int P = decltype(phb_c)::value;
          auto ph = [](auto ic) { return IC<P < 0 ? -1 : (P + decltype(ic)::value) & (V - 1)>{}; };
          auto pho = [](auto ic) {
            return IC<P < 0 ? -1 : (P + V - 1 + decltype(ic)::value) & (V - 1)>{};
          };
          step_row(IC<0>{}, ph(IC<0>{}), pho(IC<0>{}));
          step_row(IC<1>{}, ph(IC<2>{}), pho(IC<2>{}));
          step_row(IC<2>{}, ph(IC<1>{}), pho(IC<1>{}));
          step_row(IC<3>{}, ph(IC<4>{}), pho(IC<4>{}));
          step_row(IC<4>{}, ph(IC<3>{}), pho(IC<3>{}));
        };
        if (ph_regular) {
          const int phb = (phj + b * e2m) & (V - 1);
          if constexpr (V == 2) {
            if (phb == 0) steps(IC<0>{});
            else steps(IC<1>{});
          } else {
            switch (phb) {
              case 0: steps(IC<0>{}); break;
              case 1: steps(IC<1>{}); break;
              case 2: steps(IC<2>{}); break;
              default: steps(IC<3>{}); break;
            }
          }
        } else {
          steps(IC<-1>{});
        }
      }
    }
    // ---- column stage of the previous plane ----
    if (j > j0) {
      column_stage(j - 1);
      if (!((j - 1) & 1)) flush((j - 1) / 2 - 1);
    }
    __syncthreads();
    // the slot of plane j-1 is free now (its last reader ran in this phase)
    if (j > j0 && j - 1 + NS <= jend) issue(j - 1 + NS);
  }
  column_stage(jend);
  flush(jend / 2 - 1);
  flush(jend / 2);
  if (DEC && flag) {
    const bool nf = !(bad == T(0));
    if (__syncthreads_or(nf) && tid == 0) atomicOr(flag, 1);
  }
}

// Faces outside the tiles of k_level_fused. blockIdx.y selects the face:
//   0: zload on the last coarse column (c2-1) of coarse plane i0 = blockIdx.x,
//   1: zload on the last coarse row (c1-1, i2 < c2-1) of coarse plane i0,
//   2: (decompose) coefficients of the fine cells on the last fine column of
//      fine plane blockIdx.x, 3: ... on the last fine row (columns < e2-1).
// Recompose mode masks the coarse nodes (correction.hpp:251) and gathers the
// coarse nodes of faces 0/1. K0 (x) K1 (x) K2 is applied separably: the CTA
// first reduces the 3 fine columns (rows) next to the face with K2 (K1) for the
// 5 fine planes of its coarse plane into shared memory, then every thread forms
// its output from 25 of those sums.
// Face CTAs are small (latency-bound strided reads): faces 0/1 take kFaceSeg
// coarse outputs per CTA, faces 2/3 kFaceCells fine cells (one per thread).
constexpr int kFaceSeg = 64, kFaceCells = 256;

template <class T, int MODE>
__global__ void __launch_bounds__(256)
    k_level_face(const T* __restrict__ U, T* __restrict__ coef_out, T* __restrict__ zload,
                 T* __restrict__ gather, T* __restrict__ side, LevelArgs<T> a, int* flag) {
  constexpr bool DEC = MODE == kFusedDecompose, REC = MODE == kFusedRecompose;
  ptx::pdl_trigger();
  ptx::pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_f[];
  T* Rs = reinterpret_cast<T*>(smem_f);  // [5][e] partial sums
  const int e0 = int(a.e[0]), e1 = int(a.e[1]), e2 = int(a.e[2]);
  const int c0 = int(a.c[0]), c1 = int(a.c[1]), c2 = int(a.c[2]);
  const int face = blockIdx.y, tid = threadIdx.x, nt = blockDim.x;
  const int64_t plane = int64_t(e1) * e2;
  if (face <= 1) {
    const int i0 = blockIdx.x;
    if (i0 >= c0) return;
    const int ne = face == 0 ? e1 : e2;  // fine extent along the free dimension
    // this CTA's outputs q0 .. q1-1 along the free dimension and their fine span
    const int nout = face == 0 ? c1 : c2 - 1;
    const int q0 = int(blockIdx.z) * kFaceSeg;
    if (q0 >= nout) return;
    const int q1 = min(nout, q0 + kFaceSeg);
    const int f_lo = max(0, 2 * q0 - 2), W = min(ne, 2 * q1 + 1) - f_lo;
    // R[a][f] = sum over the 3 fine cells next to the face (K2 or K1 boundary row)
#pragma unroll 3
    for (int idx = tid; idx < 5 * W; idx += nt) {
      const int x = idx / W, f = f_lo + idx - x * W;
      const int f0 = 2 * i0 - 2 + x;
      T r = T(0);
      if (f0 >= 0 && f0 < e0) {
        for (int c = 0; c < 3; ++c) {
          int f1, f2;
          T w;
          if (face == 0) {
            f1 = f; f2 = e2 - 3 + c; w = a.taps[2][int64_t(c2 - 1) * 5 + c];
          } else {
            f1 = e1 - 3 + c; f2 = f; w = a.taps[1][int64_t(c1 - 1) * 5 + c];
          }
          const bool masked = REC && !((f0 | f1 | f2) & 1);
          r += w * (masked ? T(0) : U[f0 * plane + int64_t(f1) * e2 + f2]);
        }
      }
      Rs[idx] = r;
    }
    __syncthreads();
    for (int q = q0 + tid; q < q1; q += nt) {
      T acc = T(0);
      for (int x = 0; x < 5; ++x) {
        const int f0 = 2 * i0 - 2 + x;
        if (f0 < 0 || f0 >= e0) continue;
        const T w0 = e0 == 1 ? T(1) : a.taps[0][int64_t(i0) * 5 + x];
        T acc1 = T(0);
        for (int y = 0; y < 5; ++y) {
          const int f = 2 * q - 2 + y;
          if (f < 0 || f >= ne) continue;
          const T w = face == 0 ? a.taps[1][int64_t(q) * 5 + y] : a.taps[2][int64_t(q) * 5 + y];
          acc1 += w * Rs[x * W + f - f_lo];
        }
        acc += w0 * acc1;
      }
      const int i1 = face == 0 ? q : c1 - 1, i2 = face == 0 ? c2 - 1 : q;
      const int64_t o = (int64_t(i0) * c1 + i1) * c2 + i2;
      zload[o] = acc;
      if (REC || (MODE == kFusedLoadOnly && gather != nullptr))
        gather[o] = U[(2 * int64_t(i0)) * plane + int64_t(2 * i1) * e2 + 2 * i2];
    }
    return;
  }
  if (!DEC) return;
  const int j = blockIdx.x;
  if (j >= e0) return;
  auto coarse = [&](int64_t b0, int64_t b1, int64_t b2) {
    return U[(2 * b0) * plane + (2 * b1) * e2 + 2 * b2];
  };
  const int n = face == 2 ? e1 : e2 - 1;
  const int q0 = int(blockIdx.z) * kFaceCells;
  if (q0 >= n) return;
  const int q1 = min(n, q0 + kFaceCells);
  bool bad = false;
  for (int q = q0 + tid; q < q1; q += nt) {
    const int r = face == 2 ? q : e1 - 1, c = face == 2 ? e2 - 1 : q;
    const int64_t idx = j * plane + int64_t(r) * e2 + c;
    const T u = U[idx];
    bad |= !isfinite(u);
    if ((j | r | c) & 1) {
      const T cv = u - interp_node(a, j, r, c, coarse);
      if (side != nullptr && !((j | r) & 1))  // even row of an even plane (c odd)
        side[((j >> 1) * int64_t(c1) + (r >> 1)) * (c2 - 1) + (c >> 1)] = cv;
      else
        coef_out[idx] = cv;
    }
  }
  if (flag && __syncthreads_or(bad) && tid == 0) atomicOr(flag, 1);
}

// Two-phase faces (default; the scratch comes from the plan). Phase 1 reads each
// face slab of the fine level once:
//   blockIdx.y = 0: R2[j][r] = K2 of the last coarse column at fine row r of fine
//       plane j (the last three fine columns; strided, one sector per row), and
//       (decompose) the checks and coefficients of the cells on the last fine column;
//   blockIdx.y = 1: P2f[j][y][q2] = K2 of coarse column q2 at fine row e1-3+y
//       (contiguous rows), and (decompose) the cells on the last fine row
//       (columns < e2-1; side rows for the odd columns of even planes).
// Phase 2 forms the load vector on the faces from those compact arrays, K1 and K0
// over coalesced rows (recompose: plus the gather of the face coarse nodes).
// Recompose masks the coarse nodes (correction.hpp:251) in phase 1.
constexpr int kFaceItems = 1024;  // phase-1 items per CTA (4 per thread)

template <class T, int MODE>
__global__ void __launch_bounds__(256)
    k_face_slab(const T* __restrict__ U, T* __restrict__ coef_out, T* __restrict__ side,
                T* __restrict__ gather, T* __restrict__ R2, T* __restrict__ P2f, LevelArgs<T> a,
                int* flag) {
  constexpr bool DEC = MODE == kFusedDecompose, REC = MODE == kFusedRecompose;
  constexpr bool GATHER = MODE != kFusedDecompose;  // recompose; load-only when asked
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int e1 = int(a.e[1]), e2 = int(a.e[2]);
  const int c1 = int(a.c[1]), c2 = int(a.c[2]);
  const int j = blockIdx.x;
  const int64_t plane = int64_t(e1) * e2;
  const T* Up = U + j * plane;
  auto coarse = [&](int64_t b0, int64_t b1, int64_t b2) {
    return U[(2 * b0) * plane + (2 * b1) * e2 + 2 * b2];
  };
  bool bad = false;
  const int i0 = int(blockIdx.z) * kFaceItems;
  if (blockIdx.y == 0) {
    const T t0 = a.taps[2][int64_t(c2 - 1) * 5 + 0], t1 = a.taps[2][int64_t(c2 - 1) * 5 + 1],
            t2 = a.taps[2][int64_t(c2 - 1) * 5 + 2];
    const int i1 = min(e1, i0 + kFaceItems);
    for (int r = i0 + int(threadIdx.x); r < i1; r += blockDim.x) {
      const T* row = Up + int64_t(r) * e2 + (e2 - 3);
      const T u0 = row[0], u1 = row[1], u2 = row[2];
      const bool masked = REC && !((j | r) & 1);  // e2-3 and e2-1 are even columns
      R2[int64_t(j) * e1 + r] = masked ? t1 * u1 : t0 * u0 + t1 * u1 + t2 * u2;
      if (GATHER && gather != nullptr && !((j | r) & 1))  // a coarse node of the last coarse column
        gather[((int64_t(j) >> 1) * c1 + (r >> 1)) * c2 + (c2 - 1)] = u2;
      if (DEC) {
        bad |= !isfinite(u2);
        if ((j | r) & 1)  // never a side cell: the column is even
          coef_out[j * plane + int64_t(r) * e2 + (e2 - 1)] = u2 - interp_node(a, j, r, e2 - 1, coarse);
      }
    }
  } else {
    // P2f: 3 rows x (c2 - 1) coarse columns
    const int n = 3 * (c2 - 1);
    const int i1 = min(n, i0 + kFaceItems);
    for (int it = i0 + int(threadIdx.x); it < i1; it += blockDim.x) {
      const int y = it / (c2 - 1), q2 = it - y * (c2 - 1);
      const int r = e1 - 3 + y;
      const T* row = Up + int64_t(r) * e2;
      const bool maskrow = REC && !((j | r) & 1);
      T acc = T(0);
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int f = 2 * q2 - 2 + k;
        if (f < 0 || f >= e2) continue;
        const bool masked = maskrow && !(f & 1);
        acc += a.taps[2][int64_t(q2) * 5 + k] * (masked ? T(0) : row[f]);
      }
      P2f[(int64_t(j) * 3 + y) * c2 + q2] = acc;
      if (GATHER && gather != nullptr && y == 2 && !(j & 1))  // a coarse node of the last coarse row
        gather[((int64_t(j) >> 1) * c1 + (c1 - 1)) * c2 + q2] = row[2 * q2];
    }
    if (DEC) {  // the last fine row, columns < e2-1 (contiguous)
      const int r = e1 - 1;
      const int ic1 = min(e2 - 1, i0 + kFaceItems);
      for (int c = i0 + int(threadIdx.x); c < ic1; c += blockDim.x) {
        const int64_t idx = j * plane + int64_t(r) * e2 + c;
        const T u = U[idx];
        bad |= !isfinite(u);
        if ((j | c) & 1) {  // r = e1-1 is even
          const T cv = u - interp_node(a, j, r, c, coarse);
          if (side != nullptr && !(j & 1))  // even row of an even plane (c odd)
            side[((j >> 1) * int64_t(c1) + (r >> 1)) * (c2 - 1) + (c >> 1)] = cv;
          else
            coef_out[idx] = cv;
        }
      }
    }
  }
  if (DEC && flag && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

template <class T, int MODE>
__global__ void __launch_bounds__(256)
    k_face_zload(T* __restrict__ zload, const T* __restrict__ R2, const T* __restrict__ P2f,
                 LevelArgs<T> a) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int e0 = int(a.e[0]), e1 = int(a.e[1]), e2 = int(a.e[2]);
  const int c0 = int(a.c[0]), c1 = int(a.c[1]), c2 = int(a.c[2]);
  const int i0 = blockIdx.x;
  if (i0 >= c0) return;
  T w0[5];
  int f0[5];
#pragma unroll
  for (int x = 0; x < 5; ++x) {
    f0[x] = 2 * i0 - 2 + x;
    w0[x] = (f0[x] < 0 || f0[x] >= e0) ? T(0) : e0 == 1 ? T(1) : a.taps[0][int64_t(i0) * 5 + x];
    if (f0[x] < 0 || f0[x] >= e0) f0[x] = 0;
  }
  const int q = int(blockIdx.z) * blockDim.x + threadIdx.x;
  if (blockIdx.y == 0) {  // last coarse column, every coarse row
    if (q >= c1) return;
    T acc = T(0);
#pragma unroll
    for (int x = 0; x < 5; ++x) {
      const T* R = R2 + int64_t(f0[x]) * e1;
      T s = T(0);
#pragma unroll
      for (int y = 0; y < 5; ++y) {
        const int f = 2 * q - 2 + y;
        if (f >= 0 && f < e1) s += a.taps[1][int64_t(q) * 5 + y] * R[f];
      }
      acc += w0[x] * s;
    }
    const int64_t o = (int64_t(i0) * c1 + q) * c2 + (c2 - 1);
    zload[o] = acc;
  } else {  // last coarse row, columns < c2-1
    if (q >= c2 - 1) return;
    T k1[3];
#pragma unroll
    for (int y = 0; y < 3; ++y) k1[y] = a.taps[1][int64_t(c1 - 1) * 5 + y];
    T acc = T(0);
#pragma unroll
    for (int x = 0; x < 5; ++x) {
      const T* Pp = P2f + int64_t(f0[x]) * 3 * c2 + q;
      acc += w0[x] * (k1[0] * Pp[0] + k1[1] * Pp[c2] + k1[2] * Pp[2 * c2]);
    }
    const int64_t o = (int64_t(i0) * c1 + (c1 - 1)) * c2 + q;
    zload[o] = acc;
  }
}

template <class T, int MODE>
void set_level_face_smem(size_t bytes) {
  if (bytes > 48 * 1024) set_smem_attr(reinterpret_cast<const void*>(k_level_face<T, MODE>), bytes);
}

template <class T>
int fused_tiles(const LevelArgs<T>& a) {
  using C = LCfg<T>;
  const int64_t nt1 = (a.c[1] - 1 + C::TW1 - 1) / C::TW1;
  const int64_t nt2 = (a.c[2] - 1 + C::TW2 - 1) / C::TW2;
  return int(nt1 * nt2);
}

template <class T>
int fused_heuristic_s0(const LevelArgs<T>& a) {
  const int64_t tiles = fused_tiles(a);
  int S0 = kMaxSeg;
  while (S0 > 8 && tiles * std::max<int64_t>(1, (a.c[0] - 1) / S0) < 1200) S0 /= 2;
  return S0;
}

template <class T, int MODE>
void run_fused(const T* U, T* coef, T* z, T* gather, T* side, const LevelArgs<T>& a, int* flag,
               cudaStream_t s, int s0, T* face_ws) {
  using C = LCfg<T>;
  auto kern = k_level_fused<T, MODE>;
  if (a.e[1] == 1025 && a.e[2] == 1025) kern = k_level_fused<T, MODE, 1025, 1025>;
  else if (a.e[1] == 513 && a.e[2] == 513) kern = k_level_fused<T, MODE, 513, 513>;
  else if (a.e[1] == 513 && a.e[2] == 1025) kern = k_level_fused<T, MODE, 513, 1025>;
  else if (a.e[1] == 257 && a.e[2] == 513) kern = k_level_fused<T, MODE, 257, 513>;
  set_smem_attr(reinterpret_cast<const void*>(kern), C::total);
  const int nt1 = int((a.c[1] - 1 + C::TW1 - 1) / C::TW1);
  const int nt2 = int((a.c[2] - 1 + C::TW2 - 1) / C::TW2);
  const int64_t tiles = int64_t(nt1) * nt2;
  const int S0 = s0 > 0 ? std::min(s0, kMaxSeg) : fused_heuristic_s0(a);
  const int nseg = int(std::max<int64_t>(1, (a.c[0] - 1) / S0));
  // 1D TMA coordinates are 32-bit: split the segments into launches whose planes
  // fit below 2^31 elements from the launch's own (16-byte aligned) map base.
  constexpr int V = C::V;
  const int64_t plane_sz = a.e[1] * a.e[2], N = a.e[0] * plane_sz;
  const int64_t lim = (int64_t(1) << 31) - 4 * int64_t(C::BOX);
  int sa = 0;
  while (sa < nseg) {
    const int64_t p_lo = std::max<int64_t>(0, 2 * int64_t(sa) * S0 - 2);
    auto p_hi = [&](int sg) {
      return std::min<int64_t>(a.e[0] - 1, 2 * int64_t(sg) * S0 + 2 * S0);
    };
    int sb = sa + 1;
    while (sb < nseg && (p_hi(sb) + 1 - p_lo) * plane_sz < lim) ++sb;
    require((p_hi(sb - 1) + 1 - p_lo) * plane_sz < lim, "level too large for the 1D TMA path");
    const int64_t map_off = std::max<int64_t>(0, p_lo * plane_sz - 2 * V) & ~int64_t(V - 1);
    CUtensorMap map;
    make_tma_1d(&map, U + map_off, uint64_t(N - map_off), int(sizeof(T)), C::BOX);
    const int64_t blocks = tiles * (sb - sa);
    launch_pdl(kern, dim3(unsigned(blocks)), dim3(C::NT), C::total, s, N, map, map_off, coef, z,
               gather, side, a, S0, nt1, nt2, nseg, sa, flag);
    sa = sb;
  }
  // two-phase faces for levels with large faces (one launch each below: the
  // small levels are launch-latency bound)
  // knob HGR_FACE2_MIN: smallest e0*e1 for two phases (2^16: 257x513x1025 fp64
  // 2.093 -> 2.083 ms, 2^18 before; smaller thresholds change nothing measurable)
  static const int64_t face2_min = [] {
    const char* v = std::getenv("HGR_FACE2_MIN");
    return v ? int64_t(std::atoll(v)) : int64_t(1) << 16;
  }();
  if (face_ws != nullptr && a.e[0] * a.e[1] >= face2_min) {
    T* R2 = face_ws;
    T* P2f = face_ws + a.e[0] * a.e[1];
    const int64_t n1 = std::max({a.e[1], 3 * (a.c[2] - 1), a.e[2] - 1});
    launch_pdl(k_face_slab<T, MODE>,
               dim3(unsigned(a.e[0]), 2, unsigned((n1 + kFaceItems - 1) / kFaceItems)), dim3(256), 0, s,
               a.e[0] * a.e[1] * a.e[2], U, coef, side, gather, R2, P2f, a, flag);
    const int64_t n2 = std::max(a.c[1], a.c[2]);
    launch_pdl(k_face_zload<T, MODE>, dim3(unsigned(a.c[0]), 2, unsigned((n2 + 255) / 256)), dim3(256),
               0, s, a.e[0] * a.e[1] * a.e[2], z, R2, P2f, a);
    return;
  }
  const int64_t fseg =
      std::max((std::max(a.c[1], a.c[2]) + kFaceSeg - 1) / kFaceSeg,
               MODE == kFusedDecompose ? (std::max(a.e[1], a.e[2]) + kFaceCells - 1) / kFaceCells : 0);
  const dim3 fgrid(unsigned(std::max(a.c[0], a.e[0])), MODE == kFusedDecompose ? 4 : 2,
                   unsigned(fseg));
  const size_t fsmem = size_t(5) * size_t(2 * kFaceSeg + 3) * sizeof(T);
  set_level_face_smem<T, MODE>(fsmem);
  launch_pdl(k_level_face<T, MODE>, fgrid, dim3(256), fsmem, s, a.e[0] * a.e[1] * a.e[2], U, coef,
             z, gather, side, a, flag);
}

}  // namespace

template <class T>
bool launch_level_fused(const T* U, T* coef_out, T* zload, T* gather, const LevelArgs<T>& a,
                        int mode, int* flag, cudaStream_t s, int s0, T* side, T* face_ws) {
  // TMA needs a 16-byte aligned base; dim 0 segments need c0-1 = 2^k
  if (a.e[0] == 1 && a.e[1] == 1) {
    require(side == nullptr, "side rows are a 2D / 3D decompose option");
    return launch_line_level<T>(U, coef_out, zload, gather, a, mode, flag, s);
  }
  if ((reinterpret_cast<uintptr_t>(U) & 15) != 0) return false;
  if (a.e[1] < 3 || a.e[2] < 3 || a.h[2] == nullptr) return false;
  if (a.c[0] > 1 && ((a.c[0] - 1) & (a.c[0] - 2)) != 0) return false;
  require(side == nullptr || mode == kFusedDecompose, "side rows are a decompose option");
  if (mode == kFusedDecompose)
    run_fused<T, kFusedDecompose>(U, coef_out, zload, gather, side, a, flag, s, s0, face_ws);
  else if (mode == kFusedLoadOnly)
    run_fused<T, kFusedLoadOnly>(U, coef_out, zload, gather, nullptr, a, flag, s, s0, face_ws);
  else
    run_fused<T, kFusedRecompose>(U, coef_out, zload, gather, nullptr, a, flag, s, s0, face_ws);
  return true;
}

template <class T>
int level_fused_default_s0(const LevelArgs<T>& a) {
  return fused_heuristic_s0(a);
}

template <class T>
std::vector<SegChoice> level_fused_candidates(const LevelArgs<T>& a, int mode, double bw_gbs) {
  using C = LCfg<T>;
  const double S = double(sizeof(T));
  const int64_t tiles = fused_tiles(a);
  const double slots = 148.0 * C::MINB;
  auto sectors = [&](double elems) { return std::ceil(elems * S / 32.0) * 32.0 / S; };
  std::vector<SegChoice> out;
  int last_nseg = -1;
  for (int S0 = kMaxSeg; S0 >= 1; S0 /= 2) {
    const int nseg = int(std::max<int64_t>(1, (a.c[0] - 1) / S0));
    if (nseg == last_nseg) continue;
    last_nseg = nseg;
    const double planes = std::min<double>(double(a.e[0]), 2.0 * S0 + 3);   // fine planes read
    const double outp = std::min<double>(double(a.e[0]), 2.0 * S0);         // fine planes owned
    double elems = planes * C::RW * sectors(C::BOX);                         // TMA rows read
    if (mode == kFusedDecompose) elems += outp * 2 * C::TW1 * sectors(2 * C::TW2);  // coefficients
    elems += std::min<double>(double(a.c[0]), S0) * C::TW1 * sectors(C::TW2);       // load vector
    if (mode == kFusedRecompose) elems += std::min<double>(double(a.c[0]), S0) * C::TW1 * sectors(C::TW2);
    const double blocks = double(tiles) * nseg;
    const double waves = std::ceil(blocks / slots) / (blocks / slots);
    out.push_back({S0, int(blocks), blocks * elems * S / (bw_gbs * 1e3) * waves});
  }
  std::stable_sort(out.begin(), out.end(),
                   [](const SegChoice& x, const SegChoice& y) { return x.model_us < y.model_us; });
  return out;
}

template int level_fused_default_s0<float>(const LevelArgs<float>&);
template int level_fused_default_s0<double>(const LevelArgs<double>&);
template std::vector<SegChoice> level_fused_candidates<float>(const LevelArgs<float>&, int, double);
template std::vector<SegChoice> level_fused_candidates<double>(const LevelArgs<double>&, int,
                                                                double);

template bool launch_level_fused<float>(const float*, float*, float*, float*,
                                        const LevelArgs<float>&, int, int*, cudaStream_t, int, float*,
                                        float*);
template bool launch_level_fused<double>(const double*, double*, double*, double*,
                                         const LevelArgs<double>&, int, int*, cudaStream_t, int,
                                         double*, double*);

}  // namespace hgrb
