// kernels_level.cu -- fused level kernel for the fine levels: one pass over a
// level-l array U does the GPK and the three LPK passes.
//
//   A CTA (16 warps) owns a (dim1, dim2) tile of coarse outputs and marches
//   along dim 0 over a segment of coarse planes. Each fine plane's halo window
//   arrives in shared memory through 1D TMA tensor copies (one per window row,
//   issued by lane 0 of every warp) into an NS-slot mbarrier ring, two planes
//   ahead. A TMA box must start 16-byte aligned, and 2^k+1 row pitches make
//   every row's phase differ, so each row lands as its aligned superset and the
//   consumer offsets by the row's phase. (Measured on B200 with a streaming
//   probe, tools/mb/stream_mb.cu: warp-issued 1D TMA rows move 6.9 TB/s of
//   unique data, 16-byte cp.async by all threads 3.4 TB/s, one issuing thread
//   1.8 TB/s.)
//   Each warp owns a band of 4 window rows, lanes own window columns; what a
//   lane needs about its columns (mass stencil row, interpolation weights,
//   ownership) is computed once per CTA and kept in registers. Slots are zeroed
//   once and cells outside the domain carry zero weights, so the per-element
//   work is branch- and predicate-free. One CTA barrier per plane.
//   Per plane and row (warp-local):
//     m = M2 u (tridiagonal mass row along dim 2 from the three neighbours each
//       lane loads); decompose also forms the interpolant of the coarse nodes
//       (in-plane for even planes; for odd planes the blend of the two
//       neighbouring even planes' interpolants, which each thread keeps in
//       registers for its own cells) and writes the coefficients U - interp of
//       the owned nodes out of place; recompose masks the coarse nodes and
//       gathers them into the compact level-(l-1) array;
//     P2 = R2 m (transfer along dim 2; K2 = R2 M2 is the fused mass-trans
//       stencil of correction.hpp:90-133).
//   After the barrier: K1 along dim 1 (5 taps) on P2 and K0 along dim 0
//   accumulated in registers over the rolling window of coarse planes;
//   completed coarse planes are stored to the load vector zload.
//   Decompose applies K to U itself: K*P = M_c exactly for nested hat spaces,
//   so M_c^-1 K U = RU + M_c^-1 K (U - P R U) = coarse + z and the three Thomas
//   passes on zload give the corrected coarse values (refactor.hpp:48-54)
//   directly. Recompose applies K to U with the coarse nodes masked
//   (correction.hpp:251, the pass-0 mask).
#include <algorithm>

#include "kernels.cuh"
#include "kernels_fused.cuh"
#include "plan.hpp"
#include "ptx.cuh"
#include "tma.hpp"

namespace hgrb {

namespace {

// Tile shapes: 4 window rows per warp; 64 (fp64) or 128 (fp32) window columns,
// except fp32 decompose, whose per-lane interpolant registers need the
// narrower tile to stay spill-free. fp32 recompose uses 57 coarse columns so
// the TMA box (the row's 16-byte aligned superset) fits a 128-float pitch.
template <class T, int MODE>
struct FCfg {
  static constexpr int TW1 = 29, TW2 = (sizeof(T) == 4 && MODE != kFusedDecompose) ? 57 : 29;
  static constexpr int NS = 5;
};

constexpr int kMaxSeg = 64;  // coarse planes per dim-0 segment (S0 <= kMaxSeg)

template <class T, int TW1, int TW2, int NS>
struct FLayout {
  static constexpr int NT = 512, NW = NT / 32;
  static constexpr int V = 16 / int(sizeof(T));
  static constexpr int RW = 2 * (TW1 + 1) + 3;        // max window rows
  static constexpr int CW = 2 * (TW2 + 1) + 3;        // max window cols
  static constexpr int KC = (CW + 31) / 32;           // column iterations per lane
  static constexpr int KT = (TW2 + 1 + 31) / 32;      // output-column iterations
  static constexpr int RB = 4;                        // band rows per warp
  static_assert(RW <= RB * NW, "window rows must fit the warp bands");
  static constexpr int RC = (RW + NW - 1) / NW;       // rows a warp copies
  static constexpr int SQ = (TW1 + 1 + NW - 1) / NW;  // output rows per warp
  static constexpr int MW = KC * 32;                  // row pitch of the m buffer
  // TMA box: the 16-byte aligned superset of a window row
  static constexpr int BOX = (CW + V - 1 + V - 1) / V * V;
  static constexpr int ALN = 128 / int(sizeof(T));    // 128-byte granule in elements
  static constexpr int PITCH = (BOX + ALN - 1) / ALN * ALN;
  // slot: front pad (reads of window col -1) + band rows; rows beyond RW stay zero.
  // Reads reach row_off + MW + 1 <= PITCH + V + 1: a few elements into the next
  // row (finite data with zero weights), never past the slot region's end.
  static constexpr int SLOT = ALN + RB * NW * PITCH;
  static constexpr int P2W = KT * 32;
  static constexpr int K0N = kMaxSeg + 6;             // K0 tap rows: coarse planes ka-2 .. kb+1
  static constexpr size_t raw_bytes = size_t(NS) * SLOT * sizeof(T);
  static constexpr size_t m_off = raw_bytes;                              // per-warp m row
  static constexpr size_t p2_off = m_off + size_t(NW) * (MW + 8) * sizeof(T);
  static constexpr size_t k0_off = p2_off + size_t(2) * RB * NW * P2W * sizeof(T);
  static constexpr size_t bar_off = (k0_off + size_t(K0N) * 5 * sizeof(T) + 15) / 16 * 16;
  static constexpr size_t total = bar_off + NS * sizeof(uint64_t);
};

template <class T, int TW1, int TW2, int NS, int MODE>
__global__ void __launch_bounds__(512, 1)
    k_level_fused(const __grid_constant__ CUtensorMap map, int64_t map_off, T* __restrict__ coef_out,
                  T* __restrict__ zload, T* __restrict__ gather, LevelArgs<T> a, int S0, int nt1,
                  int nt2, int nseg, int seg_base, int* flag) {
  using Lay = FLayout<T, TW1, TW2, NS>;
  constexpr int V = Lay::V, PITCH = Lay::PITCH, SLOT = Lay::SLOT;
  constexpr int MW = Lay::MW, P2W = Lay::P2W, NT = Lay::NT, NW = Lay::NW, KC = Lay::KC;
  constexpr int KT = Lay::KT, RB = Lay::RB, RC = Lay::RC, SQ = Lay::SQ;
  constexpr bool DEC = MODE == kFusedDecompose, REC = MODE == kFusedRecompose;
  extern __shared__ __align__(128) unsigned char smem[];
  T* raw = reinterpret_cast<T*>(smem);
  T* p2 = reinterpret_cast<T*>(smem + Lay::p2_off);
  T* k0t = reinterpret_cast<T*>(smem + Lay::k0_off);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Lay::bar_off);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  T* mrow = reinterpret_cast<T*>(smem + Lay::m_off) + warp * (MW + 8);
  const int64_t e0 = a.e[0], e1 = a.e[1], e2 = a.e[2];
  const int64_t c0 = a.c[0], c1 = a.c[1], c2 = a.c[2];
  const int64_t plane_sz = e1 * e2;
  int bid = blockIdx.x;
  const int t2i = bid % nt2;
  bid /= nt2;
  const int t1i = bid % nt1;
  const int seg = seg_base + bid / nt1;
  const bool last1 = t1i == nt1 - 1, last2 = t2i == nt2 - 1, lastseg = seg == nseg - 1;
  const int64_t q1a = int64_t(t1i) * TW1, q2a = int64_t(t2i) * TW2;
  const int tw1 = last1 ? int(c1 - q1a) : TW1;
  const int tw2 = last2 ? int(c2 - q2a) : TW2;
  const int64_t ka = int64_t(seg) * S0;
  const int64_t kb = lastseg ? c0 : ka + S0;
  const int64_t wr0 = 2 * q1a - 2, wc0 = 2 * q2a - 2;
  const int RWn = 2 * tw1 + 3, CWn = 2 * tw2 + 3;
  const int64_t j0 = (2 * ka - 2) > 0 ? (2 * ka - 2) : 0;
  const int64_t jend = (2 * kb) < (e0 - 1) ? (2 * kb) : (e0 - 1);
  const int e2m = int(e2 & (V - 1));
  const bool pad0 = e0 == 1, pad1 = e1 == 1;
  // owned fine range [2qa, min(2(qa+tw), e)) in window coordinates [2, 2 + own)
  const int orows = 2 * tw1 - (last1 ? 1 : 0);
  const int ocols = 2 * tw2 - (last2 ? 1 : 0);
  const int rs = RB * warp;  // this warp's band of window rows [rs, rs + RB)
  const bool co = lane & 1;  // parity of every column this lane owns

  // ---- per-lane column constants (zero weights outside the domain) ----------------
  T cml[KC], cmm[KC], cmr[KC];  // mass row (masked variant for recompose coarse rows)
  T xml[KC], xmm[KC], xmr[KC];
  T hl[KC], hr[KC];             // interpolation weights of odd columns
  bool cown[KC];
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    const int c = lane + 32 * k;
    const int64_t g = wc0 + c;
    const bool in = c < CWn && g >= 0 && g < e2;
    cown[k] = c >= 2 && c < 2 + ocols;
    cml[k] = (in && g >= 1) ? a.h[2][g - 1] : T(0);
    cmr[k] = (in && g + 1 < e2) ? a.h[2][g] : T(0);
    cmm[k] = in ? T(2) * (cml[k] + cmr[k]) : T(0);
    xml[k] = co ? T(0) : cml[k];
    xmr[k] = co ? T(0) : cmr[k];
    xmm[k] = co ? cmm[k] : T(0);
    hl[k] = hr[k] = T(0);
    if (DEC && in && co) {
      hl[k] = a.wl[2][g >> 1];
      hr[k] = a.wr[2][g >> 1];
    }
  }
  T trl[KT], trr[KT];
#pragma unroll
  for (int k = 0; k < KT; ++k) {
    const int t = lane + 32 * k;
    trl[k] = trr[k] = T(0);
    if (t < tw2) {
      trl[k] = a.trl[2][q2a + t];
      trr[k] = a.trr[2][q2a + t];
    }
  }
  // output rows s = warp + NW*q: K1 taps in registers
  T k1[SQ][5];
#pragma unroll
  for (int q = 0; q < SQ; ++q) {
    const int s = warp + NW * q;
    const bool sv = s < tw1 && !pad1;
#pragma unroll
    for (int k = 0; k < 5; ++k) k1[q][k] = sv ? a.taps[1][(q1a + s) * 5 + k] : T(0);
  }
  // rows this warp copies: r = warp + NW*i, element offset of window col 0 in a plane
  int64_t roff[RC];
  bool cval[RC];
  int nvalid = 0;  // window rows inside the domain (every warp counts them all)
#pragma unroll
  for (int i = 0; i < RC; ++i) {
    const int r = warp + NW * i;
    const int64_t g = wr0 + r;
    cval[i] = r < RWn && g >= 0 && g < e1;
    roff[i] = g * e2 + wc0 - map_off;
  }
  for (int r = 0; r < RWn; ++r) nvalid += (wr0 + r >= 0 && wr0 + r < e1) ? 1 : 0;
  const uint32_t tx_bytes = uint32_t(nvalid) * Lay::BOX * uint32_t(sizeof(T));

  // smem element offset of window col 0 in window row r of plane jj (the row's phase)
  auto plane_phase = [&](int64_t jj) { return int((jj * plane_sz + wr0 * e2 + wc0) & (V - 1)); };
  auto row_off = [&](int ph, int r) { return (ph + r * e2m) & (V - 1); };

  // Window row r of plane jj lands as the aligned box [alo, alo + BOX) at slot
  // row r (cells before the domain start are zero-filled by the TMA; rows outside
  // the domain are never copied and stay zero). Completion: one mbarrier per slot
  // with one arrival (tid 0, expect_tx of the whole plane) plus the copies' bytes.
  auto issue = [&](int64_t jj) {
    const int sl = int(jj - j0) % NS;
    T* dst = raw + sl * SLOT + Lay::ALN;
    if (tid == 0) ptx::mbar_arrive_expect_tx(&bar[sl], tx_bytes);
    if (lane == 0) {
      const int64_t pbase = jj * plane_sz;
#pragma unroll
      for (int i = 0; i < RC; ++i) {
        if (!cval[i]) continue;
        const int64_t f = pbase + roff[i];
        ptx::tma_load_1d(dst + (warp + NW * i) * PITCH, &map, int(f & ~int64_t(V - 1)), &bar[sl]);
      }
    }
  };

  // zero all buffers once: slot cells never copied (outside the domain, band
  // rows beyond the window) stay 0; K0 taps of this segment into shared memory
  for (int i = tid; i < int(Lay::k0_off / sizeof(T)); i += NT) raw[i] = T(0);
  ptx::fence_proxy_async_smem();  // the zeros (generic proxy) before TMA writes (async proxy)
  for (int i = tid; i < Lay::K0N * 5; i += NT) {
    const int64_t ci = ka - 2 + i / 5;
    k0t[i] = (!pad0 && ci >= 0 && ci < c0 && ci <= kb + 1) ? a.taps[0][ci * 5 + i % 5] : T(0);
  }
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) ptx::mbar_init(&bar[s], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int nplanes = int(jend - j0 + 1);
  for (int p = 0; p < nplanes && p < NS; ++p) issue(j0 + p);

  T accA[SQ][KT], accB[SQ][KT], accC[SQ][KT];
#pragma unroll
  for (int q = 0; q < SQ; ++q)
#pragma unroll
    for (int k = 0; k < KT; ++k) accA[q][k] = accB[q][k] = accC[q][k] = T(0);
  // interpolant of the last two even planes at this thread's (row, column)
  // cells (decompose): odd planes blend them. A thread keeps the same cells
  // for every plane, so they stay in registers.
  T ipA[RB][KC], ipB[RB][KC];
#pragma unroll
  for (int ib = 0; ib < RB; ++ib)
#pragma unroll
    for (int k = 0; k < KC; ++k) ipA[ib][k] = ipB[ib][k] = T(0);
  bool bad = false;
  int pb = 0;

  auto load3 = [&](const T* rp, T (&u)[KC], T (&ul)[KC], T (&ur)[KC]) {
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      const int c = lane + 32 * k;
      u[k] = rp[c];
      ul[k] = rp[c - 1];
      ur[k] = rp[c + 1];
    }
  };

  auto process = [&](int64_t j) {
    const int p = int(j - j0);
    const int sl = p % NS;
    ptx::mbar_wait(&bar[sl], uint32_t((p / NS) & 1));
    const T* S = raw + sl * SLOT + Lay::ALN;
    const bool jodd = j & 1;
    const int ph = plane_phase(j);
    const bool own = j >= 2 * ka && j < 2 * kb;
    // even planes whose interpolant an owned odd plane needs (incl. plane 2kb)
    const bool needip = DEC && !jodd && j >= 2 * ka && j <= 2 * kb;
    T w0l = T(0), w0r = T(0);
    if (DEC && jodd && own) {
      w0l = a.wl[0][j >> 1];
      w0r = a.wr[0][j >> 1];
    }
    T* P2 = p2 + pb * (RB * NW * P2W);
    T u[KC], ul[KC], ur[KC], hprev[KC];
    load3(S + rs * PITCH + row_off(ph, rs), u, ul, ur);

#pragma unroll
    for (int ib = 0; ib < RB; ++ib) {
      const int r = rs + ib;
      const int64_t gr = wr0 + r;
      const bool ro = r & 1;  // window and global row parities agree (wr0 even)
      const bool rown = own && r >= 2 && r < 2 + orows;
      if (REC && !jodd && !ro) {  // coarse nodes of this row read as zero
#pragma unroll
        for (int k = 0; k < KC; ++k)
          mrow[lane + 32 * k] = xmm[k] * u[k] + xml[k] * ul[k] + xmr[k] * ur[k];
        if (rown) {  // gather the coarse nodes of this row into C_{l-1}
          const T* rp = S + r * PITCH + row_off(ph, r);
          T* gdst = gather + ((j >> 1) * c1 + (gr >> 1)) * c2 + q2a;
          for (int t = lane; t < tw2; t += 32) gdst[t] = rp[2 + 2 * t];
        }
      } else {
#pragma unroll
        for (int k = 0; k < KC; ++k)
          mrow[lane + 32 * k] = cmm[k] * u[k] + cml[k] * ul[k] + cmr[k] * ur[k];
      }
      // next row's values (also the even row below an odd row, for its interpolant)
      T nu[KC], nl[KC], nr[KC];
      load3(S + (r + 1) * PITCH + row_off(ph, r + 1), nu, nl, nr);
      if (DEC) {
        T* orow = coef_out + (j * e1 + gr) * e2 + wc0;
        const bool ripr = needip && r >= 2 && r <= 2 + orows && gr < e1;
        if (ripr) {
#pragma unroll
          for (int k = 0; k < KC; ++k) {
            T ip;
            if (!ro) {  // even row: interp along dim 2
              ip = co ? hl[k] * ul[k] + hr[k] * ur[k] : u[k];
              hprev[k] = ip;
            } else {    // odd row: from the even rows above / below
              const T hn = co ? hl[k] * nl[k] + hr[k] * nr[k] : nu[k];
              ip = a.wl[1][gr >> 1] * hprev[k] + a.wr[1][gr >> 1] * hn;
            }
            ipB[ib][k] = ip;
            if (rown && cown[k]) {
              orow[lane + 32 * k] = u[k] - ip;
              bad |= !isfinite(u[k]);
            }
          }
        } else if (jodd && rown) {  // odd plane: blend of the neighbouring even planes
#pragma unroll
          for (int k = 0; k < KC; ++k) {
            const T ip = w0l * ipA[ib][k] + w0r * ipB[ib][k];
            if (cown[k]) {
              orow[lane + 32 * k] = u[k] - ip;
              bad |= !isfinite(u[k]);
            }
          }
        }
      }
      __syncwarp();
      // P2 = R2 m for this row
#pragma unroll
      for (int k = 0; k < KT; ++k) {
        const int t = lane + 32 * k;
        P2[r * P2W + t] = mrow[2 * t + 2] + trl[k] * mrow[2 * t + 1] + trr[k] * mrow[2 * t + 3];
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < KC; ++k) {
        u[k] = nu[k];
        ul[k] = nl[k];
        ur[k] = nr[k];
      }
    }
    __syncthreads();

    // ---- K1 along dim 1 (5 taps), K0 accumulated across planes
    const int64_t E = jodd ? j + 1 : j;
    const int ib0 = int(E / 2 - 1 - (ka - 2));  // K0 table row of coarse plane E/2 - 1
    T kA, kB, kC;
    if (pad0) {
      kA = T(0); kB = T(1); kC = T(0);
    } else if (!jodd) {
      kA = k0t[ib0 * 5 + 4];
      kB = k0t[(ib0 + 1) * 5 + 2];
      kC = k0t[(ib0 + 2) * 5 + 0];
    } else {
      kA = k0t[ib0 * 5 + 3];
      kB = k0t[(ib0 + 1) * 5 + 1];
      kC = T(0);
    }
#pragma unroll
    for (int q = 0; q < SQ; ++q) {
      const int s = warp + NW * q;
      if (s < tw1) {
#pragma unroll
        for (int k = 0; k < KT; ++k) {
          const int t = lane + 32 * k;
          T P;
          if (pad1) {
            P = P2[2 * P2W + t];
          } else {
            const T* pc = P2 + (2 * s) * P2W + t;
            P = k1[q][0] * pc[0] + k1[q][1] * pc[P2W] + k1[q][2] * pc[2 * P2W] +
                k1[q][3] * pc[3 * P2W] + k1[q][4] * pc[4 * P2W];
          }
          accA[q][k] += kA * P;
          accB[q][k] += kB * P;
          accC[q][k] += kC * P;
        }
      }
    }
    pb ^= 1;
  };

  auto flush = [&](int64_t i) {
    if (i < ka || i >= kb) return;
#pragma unroll
    for (int q = 0; q < SQ; ++q) {
      const int s = warp + NW * q;
      if (s >= tw1) continue;
      T* zr = zload + (i * c1 + q1a + s) * c2 + q2a;
#pragma unroll
      for (int k = 0; k < KT; ++k) {
        const int t = lane + 32 * k;
        if (t < tw2) zr[t] = accA[q][k];
      }
    }
  };

  for (int64_t E = j0; E <= jend; E += 2) {
    process(E);
    if (E > j0) process(E - 1);
    flush(E / 2 - 1);
    if (DEC) {
#pragma unroll
      for (int ib = 0; ib < RB; ++ib)
#pragma unroll
        for (int k = 0; k < KC; ++k) ipA[ib][k] = ipB[ib][k];
    }
#pragma unroll
    for (int q = 0; q < SQ; ++q)
#pragma unroll
      for (int k = 0; k < KT; ++k) {
        accA[q][k] = accB[q][k];
        accB[q][k] = accC[q][k];
        accC[q][k] = T(0);
      }
    if (E > j0) {  // slots of planes E-2, E-1 are free (barrier inside process(E-1))
      if (E - 2 + NS <= jend) issue(E - 2 + NS);
      if (E - 1 + NS <= jend) issue(E - 1 + NS);
    }
  }
  flush(jend / 2);
  if (DEC && flag && __syncthreads_or(bad) && tid == 0) atomicOr(flag, 1);
}

template <class T, int MODE>
void run_fused(const T* U, T* coef, T* z, T* gather, const LevelArgs<T>& a, int* flag,
               cudaStream_t s) {
  using Cfg = FCfg<T, MODE>;
  constexpr int TW1 = Cfg::TW1, TW2 = Cfg::TW2, NS = Cfg::NS;
  using Lay = FLayout<T, TW1, TW2, NS>;
  auto kern = k_level_fused<T, TW1, TW2, NS, MODE>;
  static int attr_dev = -1;
  int dev = 0;
  HGR_CUDA_CHECK(cudaGetDevice(&dev));
  if (attr_dev != dev) {
    HGR_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(Lay::total)));
    attr_dev = dev;
  }
  const int nt1 = int(std::max<int64_t>(1, (a.c[1] - 1 + TW1 - 1) / TW1));
  const int nt2 = int(std::max<int64_t>(1, (a.c[2] - 1 + TW2 - 1) / TW2));
  const int64_t tiles = int64_t(nt1) * nt2;
  int S0 = kMaxSeg;
  while (S0 > 8 && tiles * std::max<int64_t>(1, (a.c[0] - 1) / S0) < 1200) S0 /= 2;
  const int nseg = int(std::max<int64_t>(1, (a.c[0] - 1) / S0));
  // 1D TMA coordinates are 32-bit: split the segments into launches whose planes
  // fit below 2^31 elements from the launch's own (16-byte aligned) map base.
  constexpr int V = Lay::V;
  const int64_t plane_sz = a.e[1] * a.e[2], N = a.e[0] * plane_sz;
  const int64_t lim = (int64_t(1) << 31) - 4 * int64_t(Lay::BOX);
  int sa = 0;
  while (sa < nseg) {
    const int64_t p_lo = std::max<int64_t>(0, 2 * int64_t(sa) * S0 - 2);
    int sb = sa + 1;
    auto p_hi = [&](int sg) { return std::min<int64_t>(a.e[0] - 1, 2 * int64_t(sg) * S0 + 2 * S0); };
    while (sb < nseg && (p_hi(sb) + 1 - p_lo) * plane_sz < lim) ++sb;
    require((p_hi(sb - 1) + 1 - p_lo) * plane_sz < lim, "level too large for the 1D TMA path");
    const int64_t map_off = std::max<int64_t>(0, p_lo * plane_sz - 2 * V) & ~int64_t(V - 1);
    CUtensorMap map;
    make_tma_1d(&map, U + map_off, uint64_t(N - map_off), int(sizeof(T)), Lay::BOX);
    const int64_t blocks = tiles * (sb - sa);
    kern<<<unsigned(blocks), Lay::NT, Lay::total, s>>>(map, map_off, coef, z, gather, a, S0, nt1,
                                                       nt2, nseg, sa, flag);
    HGR_CUDA_CHECK(cudaGetLastError());
    sa = sb;
  }
}

}  // namespace

template <class T>
bool launch_level_fused(const T* U, T* coef_out, T* zload, T* gather, const LevelArgs<T>& a,
                        int mode, int* flag, cudaStream_t s) {
  // TMA needs a 16-byte aligned base; dim 0 segments need c0-1 = 2^k
  if ((reinterpret_cast<uintptr_t>(U) & 15) != 0) return false;
  if (a.e[2] < 3 || a.h[2] == nullptr) return false;
  if (a.c[0] > 1 && ((a.c[0] - 1) & (a.c[0] - 2)) != 0) return false;
  if (mode == kFusedDecompose)
    run_fused<T, kFusedDecompose>(U, coef_out, zload, gather, a, flag, s);
  else if (mode == kFusedLoadOnly)
    run_fused<T, kFusedLoadOnly>(U, coef_out, zload, gather, a, flag, s);
  else
    run_fused<T, kFusedRecompose>(U, coef_out, zload, gather, a, flag, s);
  return true;
}

template bool launch_level_fused<float>(const float*, float*, float*, float*,
                                        const LevelArgs<float>&, int, int*, cudaStream_t);
template bool launch_level_fused<double>(const double*, double*, double*, double*,
                                         const LevelArgs<double>&, int, int*, cudaStream_t);

}  // namespace hgrb
