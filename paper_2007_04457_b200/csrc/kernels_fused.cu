// kernels_fused.cu -- fused level kernels for the fine levels.
//
// k_level_fused: one pass over a level-l array U (GPK + the three LPK passes).
//   A CTA (16 warps) owns a (dim1, dim2) tile of coarse outputs and marches
//   along dim 0 over a segment of coarse planes. Each fine plane's halo window
//   arrives in shared memory via 16-byte cp.async (LDGSTS) issued by all warps
//   into an NS-slot mbarrier ring, two planes ahead. (Row copies through the
//   TMA bulk engine were tried first: with ~500-byte rows the per-copy cost
//   capped reads near 0.9 TB/s; tensor maps are unusable because 2^k+1 row
//   pitches are not 16-byte multiples.)
//   Each warp owns a contiguous band of window rows, lanes own window columns;
//   what a lane needs about its columns (mass stencil row, interpolation
//   weights, ownership) is computed once per CTA and kept in registers. The
//   slots are zeroed once, cells outside the domain carry zero weights, so the
//   per-element work is branch- and predicate-free. One CTA barrier per plane.
//   Per plane and row (warp-local):
//     m = M2 u (tridiagonal mass row along dim 2 from the three neighbours each
//       lane loads); decompose also forms the interpolant of the coarse nodes
//       (in-plane for even planes, from the two neighbouring even planes for
//       odd planes) and writes the coefficients U - interp of the owned nodes
//       out of place; recompose masks the coarse nodes and gathers them into
//       the compact level-(l-1) array;
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
//
// k_interp_rec: recompose interpolation (GPK^-1). One thread per fine column,
//   streaming down the fine rows of a (planes x rows) tile; the corrected
//   coarse block (C - Z) sits in shared memory, the in-plane interpolant of
//   odd rows is formed from the two even rows held in registers.
#include <algorithm>

#include "kernels.cuh"
#include "kernels_fused.cuh"
#include "plan.hpp"
#include "ptx.cuh"

namespace hgrb {

namespace {

template <class T>
struct FCfg;
template <>
struct FCfg<double> {
  static constexpr int TW1 = 14, TW2 = 29, NS = 5;
};
template <>
struct FCfg<float> {
  static constexpr int TW1 = 14, TW2 = 61, NS = 5;
};

template <class T, int TW1, int TW2, int NS>
struct FLayout {
  static constexpr int NT = 512, NW = NT / 32;
  static constexpr int V = 16 / int(sizeof(T));
  static constexpr int LOGV = V == 2 ? 1 : 2;
  static constexpr int RW = 2 * (TW1 + 1) + 3;        // max window rows
  static constexpr int CW = 2 * (TW2 + 1) + 3;        // max window cols
  static constexpr int KC = (CW + 31) / 32;           // column iterations per lane
  static constexpr int KT = (TW2 + 1 + 31) / 32;      // output-column iterations
  static constexpr int RB = RW - 2 * (NW - 1) > 2 ? RW - 2 * (NW - 1) : 2;  // max band rows
  static constexpr int RC = (RW + NW - 1) / NW;       // rows a warp copies
  static constexpr int MW = KC * 32;                  // row pitch of the m / interp buffers
  // copies land at position 2V (room for the c-1 neighbour of window col 0 and
  // the alignment shift); reads reach position row_off + MW <= 3V + MW
  static constexpr int PITCH =
      ((CW + 4 * V > MW + 3 * V + 1 ? CW + 4 * V : MW + 3 * V + 1) + V - 1) / V * V;
  static constexpr int SLOT = RW * PITCH;
  static constexpr int P2W = KT * 32;
  static constexpr size_t raw_bytes = size_t(NS) * SLOT * sizeof(T);
  static constexpr size_t m_off = raw_bytes;                              // per-warp m row
  static constexpr size_t ip_off = m_off + size_t(NW) * (MW + 8) * sizeof(T);
  static constexpr size_t p2_off = ip_off + size_t(2) * RW * MW * sizeof(T);
  static constexpr size_t bar_off = (p2_off + size_t(2) * RW * P2W * sizeof(T) + 15) / 16 * 16;
  static constexpr size_t total = bar_off + NS * sizeof(uint64_t);
};

template <class T, int TW1, int TW2, int NS, int MODE>
__global__ void __launch_bounds__(512, 1)
    k_level_fused(const T* __restrict__ U, T* __restrict__ coef_out, T* __restrict__ zload,
                  T* __restrict__ gather, LevelArgs<T> a, int S0, int nt1, int nt2, int nseg,
                  int* flag) {
  using Lay = FLayout<T, TW1, TW2, NS>;
  constexpr int V = Lay::V, LOGV = Lay::LOGV, PITCH = Lay::PITCH, SLOT = Lay::SLOT;
  constexpr int MW = Lay::MW, P2W = Lay::P2W, NT = Lay::NT, NW = Lay::NW, KC = Lay::KC;
  constexpr int KT = Lay::KT, RW = Lay::RW, RB = Lay::RB, RC = Lay::RC;
  constexpr bool DEC = MODE == kFusedDecompose, REC = MODE == kFusedRecompose;
  extern __shared__ __align__(128) unsigned char smem[];
  T* raw = reinterpret_cast<T*>(smem);
  T* ipb = reinterpret_cast<T*>(smem + Lay::ip_off);
  T* p2 = reinterpret_cast<T*>(smem + Lay::p2_off);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Lay::bar_off);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  T* mrow = reinterpret_cast<T*>(smem + Lay::m_off) + warp * (MW + 8);
  const int64_t e0 = a.e[0], e1 = a.e[1], e2 = a.e[2];
  const int64_t c0 = a.c[0], c1 = a.c[1], c2 = a.c[2];
  const int64_t Ntot = e0 * e1 * e2, plane_sz = e1 * e2;
  int bid = blockIdx.x;
  const int t2i = bid % nt2;
  bid /= nt2;
  const int t1i = bid % nt1;
  const int seg = bid / nt1;
  const bool last1 = t1i == nt1 - 1, last2 = t2i == nt2 - 1, lastseg = seg == nseg - 1;
  const int64_t q1a = int64_t(t1i) * TW1, q2a = int64_t(t2i) * TW2;
  const int tw1 = last1 ? int(c1 - q1a) : TW1;
  const int tw2 = last2 ? int(c2 - q2a) : TW2;
  const int64_t ka = int64_t(seg) * S0;
  const int64_t kb = lastseg ? c0 : ka + S0;
  const int64_t wr0 = 2 * q1a - 2, wc0 = 2 * q2a - 2;
  const int RWn = 2 * tw1 + 3, CWn = 2 * tw2 + 3;
  const int64_t col_lo = wc0 > 0 ? wc0 : 0;
  const int64_t col_hi = (wc0 + CWn) < e2 ? (wc0 + CWn) : e2;
  const int ncols = int(col_hi - col_lo);
  const int64_t j0 = (2 * ka - 2) > 0 ? (2 * ka - 2) : 0;
  const int64_t jend = (2 * kb) < (e0 - 1) ? (2 * kb) : (e0 - 1);
  const int dcol = int(col_lo - wc0);
  const int e2m = int(e2 & (V - 1));
  const bool pad0 = e0 == 1, pad1 = e1 == 1;
  // owned fine range [2qa, min(2(qa+tw), e)) in window coordinates [2, 2 + own)
  const int orows = 2 * tw1 - (last1 ? 1 : 0);
  const int ocols = 2 * tw2 - (last2 ? 1 : 0);
  // this warp's band of window rows [rs, rs + nrb)
  const int rs = 2 * warp;
  const int nrb = warp == NW - 1 ? (RWn - rs > 0 ? RWn - rs : 0)
                                 : (RWn - rs >= 2 ? 2 : (RWn - rs > 0 ? RWn - rs : 0));

  // ---- per-lane column constants (zero weights outside the domain) ----------------
  T cml[KC], cmm[KC], cmr[KC];   // mass row
  T hl[KC], hu[KC], hr[KC];      // in-row interpolant: odd col -> (wl, 0, wr), even -> (0, 1, 0)
  T xml[KC], xmm[KC], xmr[KC];   // mass row with the coarse (even) columns masked
  bool cown[KC];
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    const int c = lane + 32 * k;
    const int64_t g = wc0 + c;
    const bool in = c < CWn && g >= 0 && g < e2;
    const bool co = c & 1;
    cown[k] = c >= 2 && c < 2 + ocols;
    cml[k] = (in && g >= 1) ? a.h[2][g - 1] : T(0);
    cmr[k] = (in && g + 1 < e2) ? a.h[2][g] : T(0);
    cmm[k] = in ? T(2) * (cml[k] + cmr[k]) : T(0);
    xml[k] = co ? T(0) : cml[k];
    xmr[k] = co ? T(0) : cmr[k];
    xmm[k] = co ? cmm[k] : T(0);
    hl[k] = hr[k] = T(0);
    hu[k] = (in && !co) ? T(1) : T(0);
    if (in && co) {
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
  // per-warp output row s = warp: K1 taps in registers
  T k1[5];
  {
    const bool sv = warp < tw1 && !pad1;
#pragma unroll
    for (int k = 0; k < 5; ++k) k1[k] = sv ? a.taps[1][(q1a + warp) * 5 + k] : T(0);
  }
  // rows this warp copies: r = warp + NW*i, element offset of col_lo within a plane
  int64_t coff[RC];
  bool cval[RC];
#pragma unroll
  for (int i = 0; i < RC; ++i) {
    const int r = warp + NW * i;
    const int64_t g = wr0 + r;
    cval[i] = r < RWn && g >= 0 && g < e1;
    coff[i] = g * e2 + col_lo;
  }

  // smem element offset of window col 0 in window row r of plane jj
  auto plane_phase = [&](int64_t jj) {
    return int((jj * plane_sz + wr0 * e2 + col_lo) & (V - 1));
  };
  auto row_off = [&](int ph, int r) { return ((ph + r * e2m) & (V - 1)) - dcol + 2 * V; };

  // Plane window rows arrive by 16-byte cp.async (LDGSTS) from every warp. Each
  // row copies the 16-byte aligned superset of its segment, so window col c of
  // row r sits at smem position row_off(ph, r) + c; a chunk reaching past the
  // array end is zero-filled (src-size < 16), nothing beyond it is read.
  // Completion: one mbarrier per slot, every thread arrives (.noinc).
  auto issue = [&](int64_t jj) {
    const int sl = int(jj - j0) % NS;
    T* dst = raw + sl * SLOT;
    const int64_t pbase = jj * plane_sz;
#pragma unroll
    for (int i = 0; i < RC; ++i) {
      if (!cval[i]) continue;
      const int64_t f = pbase + coff[i];
      const int64_t alo = f & ~int64_t(V - 1);
      const int nch = int((f - alo + ncols + V - 1) >> LOGV);
      T* d = dst + (warp + NW * i) * PITCH + 2 * V;
      const T* s = U + alo;
      if (alo + int64_t(nch) * V <= Ntot) {
        for (int ch = lane; ch < nch; ch += 32) ptx::cp_async16(d + ch * V, s + ch * V, 16);
      } else {
        for (int ch = lane; ch < nch; ch += 32) {
          const int64_t rem = Ntot - (alo + int64_t(ch) * V);
          ptx::cp_async16(d + ch * V, s + ch * V, rem >= V ? 16 : int(rem * int64_t(sizeof(T))));
        }
      }
    }
    ptx::cp_async_mbar_arrive(&bar[sl]);
  };

  // zero all buffers once: slot cells never copied (outside the domain) stay 0
  for (int i = tid; i < int(Lay::bar_off / sizeof(T)); i += NT) raw[i] = T(0);
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) ptx::mbar_init(&bar[s], NT);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int nplanes = int(jend - j0 + 1);
  for (int p = 0; p < nplanes && p < NS; ++p) issue(j0 + p);

  T accA[KT], accB[KT], accC[KT];
#pragma unroll
  for (int k = 0; k < KT; ++k) accA[k] = accB[k] = accC[k] = T(0);
  bool bad = false;
  int pb = 0;

  auto process = [&](int64_t j) {
    const int p = int(j - j0);
    const int sl = p % NS;
    ptx::mbar_wait(&bar[sl], uint32_t((p / NS) & 1));
    const T* S = raw + sl * SLOT;
    const bool jodd = j & 1;
    const int ph = plane_phase(j);
    const bool own = j >= 2 * ka && j < 2 * kb;
    // even planes whose interpolant an owned odd plane needs (incl. plane 2kb)
    const bool needip = DEC && !jodd && j >= 2 * ka && j <= 2 * kb;
    // even plane E writes interp buffer (E/2)&1; odd plane j reads both neighbours
    T* ipc = ipb + int((j >> 1) & 1) * (RW * MW);
    const T* ipn = ipb + int(((j + 1) >> 1) & 1) * (RW * MW);
    T* P2 = p2 + pb * (RW * P2W);
    T hprev[KC];
#pragma unroll
    for (int k = 0; k < KC; ++k) hprev[k] = T(0);

#pragma unroll
    for (int ib = 0; ib < RB; ++ib) {
      if (ib >= nrb) break;
      const int r = rs + ib;
      const int64_t gr = wr0 + r;
      if (gr < 0 || gr >= e1) continue;
      const T* rp = S + r * PITCH + row_off(ph, r);
      const bool ro = r & 1;
      const bool rown = own && r >= 2 && r < 2 + orows;
      T u[KC], ul[KC], ur[KC];
#pragma unroll
      for (int k = 0; k < KC; ++k) {
        const int c = lane + 32 * k;
        u[k] = rp[c];
        ul[k] = rp[c - 1];
        ur[k] = rp[c + 1];
      }
      if (REC && !jodd && !ro) {  // coarse nodes of this row read as zero
#pragma unroll
        for (int k = 0; k < KC; ++k)
          mrow[lane + 32 * k] = xmm[k] * u[k] + xml[k] * ul[k] + xmr[k] * ur[k];
        if (rown) {  // gather the coarse nodes of this row into C_{l-1}
          T* gdst = gather + ((j >> 1) * c1 + (gr >> 1)) * c2 + q2a;
          for (int t = lane; t < tw2; t += 32) gdst[t] = rp[2 + 2 * t];
        }
      } else {
#pragma unroll
        for (int k = 0; k < KC; ++k)
          mrow[lane + 32 * k] = cmm[k] * u[k] + cml[k] * ul[k] + cmr[k] * ur[k];
      }
      if (DEC) {
        T* orow = coef_out + (j * e1 + gr) * e2 + wc0;
        const bool ripr = needip && r >= 2 && r <= 2 + orows;
        if (ripr && !ro) {  // even row of an even plane: interp along dim 2
#pragma unroll
          for (int k = 0; k < KC; ++k) {
            const int c = lane + 32 * k;
            const T ip = hl[k] * ul[k] + hu[k] * u[k] + hr[k] * ur[k];
            hprev[k] = ip;
            if (cown[k]) {
              ipc[r * MW + c] = ip;
              if (rown) {
                orow[c] = u[k] - ip;
                bad |= !isfinite(u[k]);
              }
            }
          }
        } else if (ripr) {  // odd row of an even plane: from the even rows above/below
          const T w1l = a.wl[1][gr >> 1], w1r = a.wr[1][gr >> 1];
          const T* rq = S + (r + 1) * PITCH + row_off(ph, r + 1);
#pragma unroll
          for (int k = 0; k < KC; ++k) {
            const int c = lane + 32 * k;
            const T hn = hl[k] * rq[c - 1] + hu[k] * rq[c] + hr[k] * rq[c + 1];
            const T ip = w1l * hprev[k] + w1r * hn;
            if (cown[k]) {
              ipc[r * MW + c] = ip;
              if (rown) {
                orow[c] = u[k] - ip;
                bad |= !isfinite(u[k]);
              }
            }
          }
        } else if (jodd && rown) {  // odd plane: from the two neighbouring even planes
          const T w0l = a.wl[0][j >> 1], w0r = a.wr[0][j >> 1];
#pragma unroll
          for (int k = 0; k < KC; ++k) {
            const int c = lane + 32 * k;
            const T ip = w0l * ipc[r * MW + c] + w0r * ipn[r * MW + c];
            if (cown[k]) {
              orow[c] = u[k] - ip;
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
        if (t < tw2) P2[r * P2W + t] = mrow[2 * t + 2] + trl[k] * mrow[2 * t + 1] + trr[k] * mrow[2 * t + 3];
      }
      __syncwarp();
    }
    __syncthreads();

    // ---- K1 along dim 1 (5 taps), K0 accumulated across planes
    const int64_t E = jodd ? j + 1 : j;
    const int64_t iA = E / 2 - 1, iB = E / 2, iC = E / 2 + 1;
    T kA, kB, kC;
    if (pad0) {
      kA = T(0); kB = T(1); kC = T(0);
    } else if (!jodd) {
      kA = (iA >= 0) ? a.taps[0][iA * 5 + 4] : T(0);
      kB = a.taps[0][iB * 5 + 2];
      kC = (iC < c0) ? a.taps[0][iC * 5 + 0] : T(0);
    } else {
      kA = a.taps[0][iA * 5 + 3];
      kB = (iB < c0) ? a.taps[0][iB * 5 + 1] : T(0);
      kC = T(0);
    }
    if (warp < tw1) {
      const int s = warp;
#pragma unroll
      for (int k = 0; k < KT; ++k) {
        const int t = lane + 32 * k;
        if (t < tw2) {
          T P;
          if (pad1) {
            P = P2[2 * P2W + t];
          } else {
            const T* pc = P2 + (2 * s) * P2W + t;
            P = k1[0] * pc[0] + k1[1] * pc[P2W] + k1[2] * pc[2 * P2W] + k1[3] * pc[3 * P2W] +
                k1[4] * pc[4 * P2W];
          }
          accA[k] += kA * P;
          accB[k] += kB * P;
          accC[k] += kC * P;
        }
      }
    }
    pb ^= 1;
  };

  auto flush = [&](int64_t i) {
    if (i < ka || i >= kb || warp >= tw1) return;
    T* zr = zload + (i * c1 + q1a + warp) * c2 + q2a;
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      const int t = lane + 32 * k;
      if (t < tw2) zr[t] = accA[k];
    }
  };

  for (int64_t E = j0; E <= jend; E += 2) {
    process(E);
    if (E > j0) process(E - 1);
    flush(E / 2 - 1);
#pragma unroll
    for (int k = 0; k < KT; ++k) {
      accA[k] = accB[k];
      accB[k] = accC[k];
      accC[k] = T(0);
    }
    if (E > j0) {  // slots of planes E-2, E-1 are free (barrier inside process(E-1))
      if (E - 2 + NS <= jend) issue(E - 2 + NS);
      if (E - 1 + NS <= jend) issue(E - 1 + NS);
    }
  }
  flush(jend / 2);
  if (DEC && flag && __syncthreads_or(bad) && tid == 0) atomicOr(flag, 1);
}

// ---- recompose interpolation -------------------------------------------------

template <class T, int B0, int B1, int B2>
__global__ void __launch_bounds__(2 * B2) k_interp_rec(const T* coef, T* out, const T* __restrict__ C,
                                                       const T* __restrict__ Z, LevelArgs<T> a,
                                                       bool with, int nb1, int nb2) {
  constexpr int NT = 2 * B2, S1 = B1 + 1, S2 = B2 + 2;
  extern __shared__ __align__(16) unsigned char smem_i[];
  T* cs = reinterpret_cast<T*>(smem_i);  // (B0+1) x S1 x S2 corrected coarse block
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int bid = blockIdx.x;
  const int b2 = bid % nb2;
  bid /= nb2;
  const int b1 = bid % nb1;
  const int b0 = bid / nb1;
  const int64_t c0 = a.c[0], c1 = a.c[1], c2 = a.c[2];
  const int64_t e0 = a.e[0], e1 = a.e[1], e2 = a.e[2];
  const int64_t qa0 = int64_t(b0) * B0, qa1 = int64_t(b1) * B1, qa2 = int64_t(b2) * B2;
  const int nb0 = int((c0 - 1 + B0 - 1) / B0) > 0 ? int((c0 - 1 + B0 - 1) / B0) : 1;
  const int tb0 = b0 == nb0 - 1 ? int(c0 - qa0) : B0;
  const int tb1 = b1 == nb1 - 1 ? int(c1 - qa1) : B1;
  const int tb2 = b2 == nb2 - 1 ? int(c2 - qa2) : B2;
  const int n0 = int(std::min<int64_t>(tb0 + 1, c0 - qa0));
  const int n1 = int(std::min<int64_t>(tb1 + 1, c1 - qa1));
  const int n2 = int(std::min<int64_t>(tb2 + 1, c2 - qa2));
  // corrected coarse block C - Z: rows (x0, x1) over warps, columns over lanes
  for (int row = warp; row < n0 * n1; row += NT / 32) {
    const int x0 = row / n1, x1 = row - x0 * n1;
    const int64_t q = ((qa0 + x0) * c1 + qa1 + x1) * c2 + qa2;
    T* dst = cs + (x0 * S1 + x1) * S2;
    for (int x2 = lane; x2 < n2; x2 += 32) dst[x2] = Z ? C[q + x2] - Z[q + x2] : C[q + x2];
  }
  __syncthreads();
  // owned fine ranges [2qa, min(2(qa+tb), e))
  const int f0 = int(std::min<int64_t>(2 * (qa0 + tb0), e0) - 2 * qa0);
  const int f1 = int(std::min<int64_t>(2 * (qa1 + tb1), e1) - 2 * qa1);
  const int f2 = int(std::min<int64_t>(2 * (qa2 + tb2), e2) - 2 * qa2);
  for (int x2 = tid; x2 < f2; x2 += NT) {
    const int b = x2 >> 1;
    const bool o2 = x2 & 1;
    const int64_t i2 = 2 * qa2 + x2;
    const T wl2 = o2 ? a.wl[2][i2 >> 1] : T(1), wr2 = o2 ? a.wr[2][i2 >> 1] : T(0);
    const int bn = o2 ? b + 1 : b;
    for (int x0 = 0; x0 < f0; ++x0) {
      const bool o0 = x0 & 1;
      const int64_t i0 = 2 * qa0 + x0;
      const T w0l = o0 ? a.wl[0][i0 >> 1] : T(1), w0r = o0 ? a.wr[0][i0 >> 1] : T(0);
      const T* pA = cs + (x0 >> 1) * S1 * S2;
      const T* pB = o0 ? pA + S1 * S2 : pA;
      // interpolant of the even fine row 2*q1 (dims 0 and 2)
      auto reven = [&](int q1) {
        const T vb = w0l * pA[q1 * S2 + b] + w0r * pB[q1 * S2 + b];
        const T vn = w0l * pA[q1 * S2 + bn] + w0r * pB[q1 * S2 + bn];
        return wl2 * vb + wr2 * vn;
      };
      const int64_t rowbase = (i0 * e1 + 2 * qa1) * e2 + i2;
      T rcur = reven(0);
#pragma unroll 4
      for (int x1 = 0; x1 < f1; x1 += 2) {
        const int64_t g0 = rowbase + int64_t(x1) * e2;
        const bool has_odd = x1 + 1 < f1;
        T cf0 = T(0), cf1 = T(0);
        if (with) {
          cf0 = coef[g0];
          if (has_odd) cf1 = coef[g0 + e2];
        }
        const bool coarse = !(o0 | o2);  // even row x1: coarse node iff x0, x2 even
        out[g0] = coarse ? rcur : cf0 + rcur;
        if (has_odd) {
          const int64_t i1 = 2 * qa1 + x1 + 1;
          const T rnext = reven((x1 >> 1) + 1);
          const T ip = a.wl[1][i1 >> 1] * rcur + a.wr[1][i1 >> 1] * rnext;
          out[g0 + e2] = cf1 + ip;
          rcur = rnext;
        }
      }
    }
  }
}

template <class T, int MODE>
void run_fused(const T* U, T* coef, T* z, T* gather, const LevelArgs<T>& a, int* flag,
               cudaStream_t s) {
  constexpr int TW1 = FCfg<T>::TW1, TW2 = FCfg<T>::TW2, NS = FCfg<T>::NS;
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
  int S0 = 64;
  while (S0 > 8 && tiles * std::max<int64_t>(1, (a.c[0] - 1) / S0) < 1200) S0 /= 2;
  const int nseg = int(std::max<int64_t>(1, (a.c[0] - 1) / S0));
  kern<<<unsigned(tiles * nseg), Lay::NT, Lay::total, s>>>(U, coef, z, gather, a, S0, nt1, nt2,
                                                           nseg, flag);
  HGR_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

template <class T>
bool launch_level_fused(const T* U, T* coef_out, T* zload, T* gather, const LevelArgs<T>& a,
                        int mode, int* flag, cudaStream_t s) {
  // cp.async needs a 16-byte aligned base; dim 0 segments need c0-1 = 2^k
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

template <class T>
bool launch_interp_rec(const T* coef, T* out, const T* C, const T* Z, const LevelArgs<T>& a,
                       bool with, cudaStream_t s) {
  constexpr int B0 = 2, B1 = 16, B2 = 128;
  const int64_t m0 = a.c[0] - 1, m1 = a.c[1] - 1, m2 = a.c[2] - 1;
  const int nb0 = int(std::max<int64_t>(1, (m0 + B0 - 1) / B0));
  const int nb1 = int(std::max<int64_t>(1, (m1 + B1 - 1) / B1));
  const int nb2 = int(std::max<int64_t>(1, (m2 + B2 - 1) / B2));
  const size_t smem = size_t(B0 + 1) * (B1 + 1) * (B2 + 2) * sizeof(T);
  static int attr_dev = -1;
  int dev = 0;
  HGR_CUDA_CHECK(cudaGetDevice(&dev));
  if (attr_dev != dev) {
    HGR_CUDA_CHECK(cudaFuncSetAttribute(k_interp_rec<T, B0, B1, B2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr_dev = dev;
  }
  k_interp_rec<T, B0, B1, B2><<<unsigned(int64_t(nb0) * nb1 * nb2), 2 * B2, smem, s>>>(
      coef, out, C, Z, a, with, nb1, nb2);
  HGR_CUDA_CHECK(cudaGetLastError());
  return true;
}

template bool launch_level_fused<float>(const float*, float*, float*, float*,
                                        const LevelArgs<float>&, int, int*, cudaStream_t);
template bool launch_level_fused<double>(const double*, double*, double*, double*,
                                         const LevelArgs<double>&, int, int*, cudaStream_t);
template bool launch_interp_rec<float>(const float*, float*, const float*, const float*,
                                       const LevelArgs<float>&, bool, cudaStream_t);
template bool launch_interp_rec<double>(const double*, double*, const double*, const double*,
                                        const LevelArgs<double>&, bool, cudaStream_t);

}  // namespace hgrb
