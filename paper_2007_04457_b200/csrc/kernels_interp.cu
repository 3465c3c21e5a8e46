// kernels_interp.cu -- recompose interpolation (GPK^-1, refactor.hpp:77-87):
// out[coarse] = C - Z, out[refined] = coef + interp(C - Z), or the
// interpolation alone for classes above the recompose prefix.
//
// k_interp_march: a CTA (16 warps) owns a (dim1, dim2) tile of TW1 x 64 coarse
// cells (2*TW1 x 128 fine cells) and marches along dim 0 over a segment of
// coarse planes. Per coarse plane m the corrected coarse window (C and Z rows
// by 1D TMA copies) gives, for every thread's cells, the in-plane interpolant
// of fine plane 2m (dim-2 blend on even rows, blend of the even rows above /
// below on odd rows), kept in registers; the odd fine plane 2m-1 blends it
// with plane m-1's (transforms.hpp:41-55 evaluated as a separable product).
// Coefficient planes stream through an NS-slot TMA ring (rows land as their
// 16-byte aligned supersets, read at the row's phase); outputs are coalesced
// row stores. Lane L of column group G owns coarse column t = 32G + L and fine
// cells 2t, 2t+1; the warps of a group own bands of four fine rows. In-place
// safe (every cell is read before it is written, by the CTA that owns it).
// The last fine row and column of the level (the faces) are written by the last
// tile row / column: the lane whose right coarse neighbour is the last coarse
// column computes one extra cell, the band holding the last fine row one extra
// row, so those rows are stored whole (no strided face writes).
#include <algorithm>
#include <type_traits>
#include <cmath>

#include "kernels.cuh"
#include "kernels_fused.cuh"
#include "plan.hpp"
#include "ptx.cuh"
#include "launch.cuh"
#include "tma.hpp"

namespace hgrb {

namespace {

constexpr int kMaxSegI = 32;  // coarse planes per dim-0 segment

template <class T>
struct ICfg {
  // fp64: lane = 1 coarse column, 16 warps in 2 column groups, one CTA per SM;
  // fp32: lane = 2 coarse columns (float4 coefficient loads), 8 warps, two CTAs per SM
  static constexpr bool D = sizeof(T) == 8;
  static constexpr int CPL = D ? 1 : 2;
  static constexpr int NG = D ? 2 : 1;
  static constexpr int NT = D ? 512 : 256, NW = NT / 32, WG = NW / NG;
  static constexpr int MINB = D ? 1 : 2;
  static constexpr int TW2 = 32 * CPL * NG, TW1 = D ? 14 : 16;
  static constexpr int NS = D ? 5 : 4;                         // coefficient plane slots
  static constexpr int V = 16 / int(sizeof(T));
  static constexpr int ALN = 128 / int(sizeof(T));
  static constexpr int FR = 2 * TW1, FC = 2 * TW2;             // fine rows / cols of a tile
  static constexpr int NB = FR / 4;                            // bands of four fine rows
  static_assert(NB <= WG, "one band per warp of a group");
  static constexpr int NCELL = 2 * CPL;
  static constexpr int BOX = (FC + V - 1 + V - 1) / V * V;     // aligned superset of a row
  static constexpr int PITCH = (BOX + ALN - 1) / ALN * ALN;
  static_assert(PITCH >= FC + V + 4, "vector reads stay inside the row");
  static constexpr int SLOT = (FR + 1) * PITCH;                // + the last fine row (face)
  static constexpr int CR = TW1 + 1, CC = TW2 + 1;             // coarse window
  static constexpr int CBOX = (CC + V - 1 + V - 1) / V * V;
  static constexpr int CPITCH = (CBOX + ALN - 1) / ALN * ALN;
  static constexpr int CSLOT = CR * CPITCH;
  static constexpr size_t c_off = size_t(NS) * SLOT * sizeof(T);  // [2 bufs][C, Z][CSLOT]
  static constexpr size_t w_off = c_off + size_t(4) * CSLOT * sizeof(T);
  static constexpr int W0N = kMaxSegI + 2;
  static constexpr size_t bar_off = (w_off + size_t(2) * W0N * sizeof(T) + 15) / 16 * 16;
  static constexpr size_t total = bar_off + (NS + 2) * sizeof(uint64_t);
  static_assert(total * MINB <= 227 * 1024, "shared memory budget");
};

template <int N>
using IC = std::integral_constant<int, N>;

template <class T>
struct Vec2i;
template <>
struct Vec2i<double> { using type = double2; };
template <>
struct Vec2i<float> { using type = float2; };

// v[k] = row[pos + k], k < N (pairs by 2-element vector loads; fp32 N = 4 by float4)
template <class T, int N>
__device__ __forceinline__ void ldn(const T* row, int pos, T (&v)[N]) {
  using T2 = typename Vec2i<T>::type;
  if constexpr (N == 4 && sizeof(T) == 4) {
    const int base = pos & ~3, ph = pos & 3;
    const float4* p = reinterpret_cast<const float4*>(row + base);
    const float4 x = p[0];
    if (ph == 0) {
      v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    } else {
      const float4 y = p[1];
      const float w[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
      if (ph == 1) { v[0] = w[1]; v[1] = w[2]; v[2] = w[3]; v[3] = w[4]; }
      else if (ph == 2) { v[0] = w[2]; v[1] = w[3]; v[2] = w[4]; v[3] = w[5]; }
      else { v[0] = w[3]; v[1] = w[4]; v[2] = w[5]; v[3] = w[6]; }
    }
  } else if constexpr (N == 2) {
    if (!(pos & 1)) {
      const T2 x = *reinterpret_cast<const T2*>(row + pos);
      v[0] = x.x;
      v[1] = x.y;
    } else {
      v[0] = row[pos];
      v[1] = row[pos + 1];
    }
  } else {
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] = row[pos + k];
  }
}

// ldn with the phase of pos known at compile time (pos - PH is 16-byte aligned)
template <class T, int N, int PH>
__device__ __forceinline__ void ldnc(const T* row, int pos, T (&v)[N]) {
  const T* p = row + (pos - PH);
  if constexpr (N == 4 && sizeof(T) == 4) {
    const float4 x = *reinterpret_cast<const float4*>(p);
    if constexpr (PH == 0) {
      v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    } else {
      const float4 y = *reinterpret_cast<const float4*>(p + 4);
      const float w[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = w[PH + k];
    }
  } else if constexpr (N == 2 && sizeof(T) == 8) {
    if constexpr (PH == 0) {
      const double2 x = *reinterpret_cast<const double2*>(p);
      v[0] = x.x;
      v[1] = x.y;
    } else {
      v[0] = p[1];
      v[1] = p[2];
    }
  } else {
    ldn<T, N>(row, pos, v);
  }
}

// SUB (in-place decompose): out = U - interp(C) at refined nodes, U at coarse
// nodes, with U in place of the coefficients (every cell reads only its own U,
// the coarse values come from C) and a non-finite check of every cell into flag.
// E1C, E2C: the extents of dims 1 and 2 at compile time for the large 2^k+1 shapes (0:
// run time), so the address arithmetic folds
template <class T, bool WITH, bool HASZ, bool SUB, int E1C = 0, int E2C = 0>
__global__ void __launch_bounds__(ICfg<T>::NT, ICfg<T>::MINB)
    k_interp_march(const __grid_constant__ CUtensorMap mcoef, const __grid_constant__ CUtensorMap mC,
                   const __grid_constant__ CUtensorMap mZ, int64_t coef_off, int64_t c_off,
                   T* __restrict__ out, LevelArgs<T> a, int S0, int nt1, int nt2, int nseg,
                   int seg_base, int* flag) {
  using C = ICfg<T>;
  ptx::pdl_trigger();
  constexpr int V = C::V, PITCH = C::PITCH, SLOT = C::SLOT, NS = C::NS, NW = C::NW;
  constexpr int TW1 = C::TW1, TW2 = C::TW2, WG = C::WG, NB = C::NB;
  constexpr int CPITCH = C::CPITCH, CSLOT = C::CSLOT, CPL = C::CPL, NCELL = C::NCELL;
  extern __shared__ __align__(128) unsigned char smem[];
  T* ring = reinterpret_cast<T*>(smem);
  T* cbuf = reinterpret_cast<T*>(smem + C::c_off);
  T* w0t = reinterpret_cast<T*>(smem + C::w_off);  // [2][W0N] dim-0 weights of odd planes
  uint64_t* barf = reinterpret_cast<uint64_t*>(smem + C::bar_off);
  uint64_t* barc = barf + NS;

  const int tid = threadIdx.x, lane = tid & 31, warp = ptx::warp_id_uniform();
  const int64_t e0 = a.e[0], e1 = E1C ? E1C : a.e[1], e2 = E2C ? E2C : a.e[2];
  const int64_t c0 = a.c[0], c1 = E1C ? (E1C + 1) / 2 : a.c[1], c2 = E2C ? (E2C + 1) / 2 : a.c[2];
  int bid = blockIdx.x;
  const int t2i = bid % nt2;
  bid /= nt2;
  const int t1i = bid % nt1;
  const int seg = seg_base + bid / nt1;
  const bool lastseg = seg == nseg - 1;
  const int64_t q1a = int64_t(t1i) * TW1, q2a = int64_t(t2i) * TW2;
  const int tw1 = int(c1 - 1 - q1a < TW1 ? c1 - 1 - q1a : TW1);
  const int tw2 = int(c2 - 1 - q2a < TW2 ? c2 - 1 - q2a : TW2);
  const int64_t ka = int64_t(seg) * S0;
  const int64_t kb = lastseg ? c0 - 1 : ka + S0;  // coarse planes ka..kb
  const int64_t jlo = 2 * ka, jhi = lastseg ? e0 - 1 : 2 * kb - 1;  // owned fine planes
  const int frows = 2 * tw1;
  // faces: the last coarse column / row of the level is this tile's +1 neighbour
  const bool xcol = c2 - 1 - q2a <= TW2, xrow = c1 - 1 - q1a <= TW1;

  const int grp = warp / WG, wg = warp % WG;
  const int t0 = CPL * (32 * grp + lane);  // tile-local coarse columns t0..t0+CPL-1
  T hl[CPL], hr[CPL];
  bool cvalid[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    cvalid[c] = t0 + c < tw2;
    hl[c] = cvalid[c] ? a.wl[2][q2a + t0 + c] : T(0);
    hr[c] = cvalid[c] ? a.wr[2][q2a + t0 + c] : T(0);
  }
  // face cell of this lane (the even cell of coarse column tw2 = c2-1): index fk
  // of its NCELL + 1 cells, or -1
  int fk = -1;
  if (xcol && tw2 - t0 >= 0 && tw2 - t0 <= CPL) fk = 2 * (tw2 - t0);
  const bool has_band = wg < NB;
  const int b = 4 * wg;  // fine rows b..b+4 of the tile; coarse rows b/2 .. b/2+2
  // row b+4 is only ever the last fine row of a full-height last tile row
  bool rown[5];
#pragma unroll
  for (int i = 0; i < 5; ++i)
    rown[i] = has_band && (i < 4 ? (b + i < frows || (xrow && b + i == frows))
                                 : (xrow && b + 4 == frows && frows == 2 * TW1));
  T w1l[2] = {T(0), T(0)}, w1r[2] = {T(0), T(0)};  // odd fine rows b+1, b+3
  if (has_band) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int64_t gr = 2 * q1a + b + 1 + 2 * i;
      if (gr < e1 - 1) { w1l[i] = a.wl[1][gr >> 1]; w1r[i] = a.wr[1][gr >> 1]; }
    }
  }

  // ---- TMA: fine coefficient rows and coarse C / Z rows --------------------------------
  const int64_t plane_f = e1 * e2, plane_c = c1 * c2;
  const int frows_ld = frows + (xrow ? 1 : 0);  // + the last fine row
  const uint32_t tx_f = uint32_t(frows_ld) * C::BOX * uint32_t(sizeof(T));
  const int crows = tw1 + 1;
  const uint32_t tx_c = uint32_t(crows) * C::CBOX * uint32_t(sizeof(T)) * (HASZ ? 2u : 1u);
  const uint32_t ring_s = ptx::smem_addr(ring), cbuf_s = ptx::smem_addr(cbuf);
  const uint32_t barf_s = ptx::smem_addr(barf), barc_s = ptx::smem_addr(barc);
  auto issue_f = [&](int64_t j) {  // fine plane j into slot (j - jlo) % NS
    const int sl = int(j - jlo) % NS;
    if (tid == 0) ptx::mbar_arrive_expect_tx(&barf[sl], tx_f);
    if (ptx::elect_one()) {
      const uint32_t dst = ring_s + uint32_t(sl * SLOT * sizeof(T));
      const uint32_t bs = barf_s + uint32_t(sl * sizeof(uint64_t));
      const int64_t base = (j * e1 + 2 * q1a) * e2 + 2 * q2a - coef_off;
      for (int r = warp; r < frows_ld; r += NW) {
        const int64_t f = base + int64_t(r) * e2;
        ptx::tma_load_1d_s(dst + uint32_t(r * PITCH * sizeof(T)), &mcoef, int(f & ~int64_t(V - 1)), bs);
      }
    }
  };
  auto issue_c = [&](int64_t m) {  // coarse plane m into buffer m & 1
    const int bsl = int(m & 1);
    if (tid == 0) ptx::mbar_arrive_expect_tx(&barc[bsl], tx_c);
    if (ptx::elect_one()) {
      const uint32_t dst = cbuf_s + uint32_t(bsl * 2 * CSLOT * sizeof(T));
      const uint32_t bs = barc_s + uint32_t(bsl * sizeof(uint64_t));
      const int64_t base = (m * c1 + q1a) * c2 + q2a - c_off;
      for (int r = warp; r < crows; r += NW) {
        const int64_t f = base + int64_t(r) * c2;
        const int x = int(f & ~int64_t(V - 1));
        ptx::tma_load_1d_s(dst + uint32_t(r * CPITCH * sizeof(T)), &mC, x, bs);
        if (HASZ) ptx::tma_load_1d_s(dst + uint32_t((CSLOT + r * CPITCH) * sizeof(T)), &mZ, x, bs);
      }
    }
  };

  for (int i = tid; i < C::W0N; i += blockDim.x) {
    const int64_t q = ka + i;  // dim-0 interval of odd plane 2q+1
    const bool ok = e0 > 1 && q < c0 - 1;
    w0t[i] = ok ? a.wl[0][q] : T(0);
    w0t[C::W0N + i] = ok ? a.wr[0][q] : T(0);
  }
  if (tid == 0) {
    for (int q = 0; q < NS + 2; ++q) ptx::mbar_init(&barf[q], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  ptx::pdl_wait();  // C, Z and the coefficients come from earlier launches
  if (WITH)
    for (int64_t j = jlo; j <= jhi && j < jlo + NS; ++j) issue_f(j);
  issue_c(ka);
  if (ka + 1 <= kb) issue_c(ka + 1);

  const int e2m = int(e2 & (V - 1)), c2m = int(c2 & (V - 1));
  // 2^k+1 extents: consecutive fine rows advance the phase by one (fp64 only:
  // the fp32 march is at its bandwidth bound and measured no gain)
  const bool ph_regular = sizeof(T) == 8 && e2m == 1;
  // vector output stores: whole tile row owned, output and coefficient map base
  // on the same 16-byte phase (cell phases then follow fpos)
  const bool vstore = tw2 == TW2 && (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
                      (coef_off & (V - 1)) == 0 && (2 * t0) % V == 0;
  const int fph0 = int((2 * q1a * e2 + 2 * q2a) & (V - 1));
  const int cph0 = int((q1a * c2 + q2a) & (V - 1));
  auto fpos = [&](int64_t j, int r) {
    return int((j * plane_f + fph0 + int64_t(r) * e2m) & (V - 1)) + 2 * t0;
  };
  auto cpos = [&](int64_t m, int s) {
    return int((m * plane_c + cph0 + int64_t(s) * c2m) & (V - 1)) + t0;
  };

  constexpr int NC1 = NCELL + 1;  // + the face cell
  T A1p[5][NC1], A1[5][NC1];
#pragma unroll
  for (int i = 0; i < 5; ++i)
#pragma unroll
    for (int k = 0; k < NC1; ++k) A1p[i][k] = A1[i][k] = T(0);
  T* obase = out + (2 * q1a + b) * e2 + 2 * q2a + 2 * t0;
  T bad = T(0);  // SUB: non-finite input seen

  // one fine plane j: out = coef + interp (interp alone at coarse nodes / without coef)
  auto fine_plane = [&](int64_t j, bool odd, T w0l, T w0r) {
    const int p = int(j - jlo);
    const T* S = ring + (p % NS) * SLOT;
    if (WITH) ptx::mbar_wait(&barf[p % NS], uint32_t((p / NS) & 1));
    if (!has_band) return;
    T* o = obase + j * plane_f;
    // one row; PH: the phase of the row's cells (compile time), or -1
    auto row = [&](auto i_c, auto ph_c) {
      constexpr int i = decltype(i_c)::value, PH = decltype(ph_c)::value;
      if (i == 4 && !rown[4]) return;
      T v[NC1];
#pragma unroll
      for (int k = 0; k < NC1; ++k) v[k] = odd ? w0l * A1p[i][k] + w0r * A1[i][k] : A1[i][k];
      if (WITH) {
        T cf[NC1];
        {
          T c4[NCELL];
          const T* rowp = S + (b + i) * PITCH;
          const int pos = fpos(j, b + i);
          if constexpr (PH >= 0) ldnc<T, NCELL, PH>(rowp, pos, c4);
          else ldn<T, NCELL>(rowp, pos, c4);
#pragma unroll
          for (int k = 0; k < NCELL; ++k) cf[k] = c4[k];
          cf[NCELL] = fk == NCELL ? rowp[pos + NCELL] : T(0);
        }
#pragma unroll
        for (int k = 0; k < NC1; ++k) {
          // the coarse nodes (even plane, even row, even column) keep the interpolant
          // (SUB: keep U there, the coefficient U - interp elsewhere)
          const bool refined = odd || (i & 1) || (k & 1);
          if constexpr (SUB) {
            v[k] = refined ? cf[k] - v[k] : cf[k];
            if (rown[i] && (k < NCELL ? cvalid[k >> 1] || k == fk : fk == NCELL))
              bad = cf[k] * T(0) + bad;
          } else if (refined) {
            v[k] += cf[k];
          }
        }
      }
      if (rown[i]) {
        T* orow = o + int64_t(i) * e2;
        if (fk == NCELL) orow[NCELL] = v[NCELL];
        // the output has the coefficients' layout: same phase when both are aligned
        if constexpr (PH >= 0) {
          if (vstore) {
            T v4[NCELL];
#pragma unroll
            for (int k = 0; k < NCELL; ++k) v4[k] = v[k];
            store_cells<T, NCELL, PH>(orow, v4);
            return;
          }
        }
#pragma unroll
        for (int k = 0; k < NCELL; ++k)
          if (cvalid[k >> 1] || k == fk) orow[k] = v[k];
      }
    };
    auto rows4 = [&](auto phb_c) {
      constexpr int P = decltype(phb_c)::value;
      auto ph = [](auto ic) { return IC<P < 0 ? -1 : (P + decltype(ic)::value) & (V - 1)>{}; };
      row(IC<0>{}, ph(IC<0>{}));
      row(IC<1>{}, ph(IC<1>{}));
      row(IC<2>{}, ph(IC<2>{}));
      row(IC<3>{}, ph(IC<3>{}));
      row(IC<4>{}, ph(IC<4>{}));
    };
    if (ph_regular) {
      const int phb = fpos(j, b) & (V - 1);
      if constexpr (V == 2) {
        if (phb == 0) rows4(IC<0>{});
        else rows4(IC<1>{});
      } else {
        switch (phb) {
          case 0: rows4(IC<0>{}); break;
          case 1: rows4(IC<1>{}); break;
          case 2: rows4(IC<2>{}); break;
          default: rows4(IC<3>{}); break;
        }
      }
    } else {
      rows4(IC<-1>{});
    }
  };

  for (int64_t m = ka; m <= kb; ++m) {
    // ---- coarse plane m: corrected window -> in-plane interpolant of fine plane 2m
    const int bsl = int(m & 1);
    ptx::mbar_wait(&barc[bsl], uint32_t(((m - ka) >> 1) & 1));
    if (has_band) {
      const T* Cb = cbuf + bsl * 2 * CSLOT;
      T A2[3][NC1];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int s = b / 2 + k;
        const int ps = cpos(m, s);
        T x[CPL + 1];
        ldn<T, CPL + 1>(Cb + s * CPITCH, ps, x);
        if (HASZ) {
          T z[CPL + 1];
          ldn<T, CPL + 1>(Cb + CSLOT + s * CPITCH, ps, z);
#pragma unroll
          for (int c = 0; c <= CPL; ++c) x[c] -= z[c];
        }
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          A2[k][2 * c] = x[c];
          A2[k][2 * c + 1] = hl[c] * x[c] + hr[c] * x[c + 1];
        }
        A2[k][NCELL] = x[CPL];  // the face cell (coarse column t0 + CPL)
      }
#pragma unroll
      for (int c = 0; c < NC1; ++c) {
        A1[0][c] = A2[0][c];
        A1[1][c] = w1l[0] * A2[0][c] + w1r[0] * A2[1][c];
        A1[2][c] = A2[1][c];
        A1[3][c] = w1l[1] * A2[1][c] + w1r[1] * A2[2][c];
        A1[4][c] = A2[2][c];
      }
    }
    // ---- fine planes 2m-1 (odd) and 2m (even)
    if (m > ka) {
      const int iw = int(m - 1 - ka);
      fine_plane(2 * m - 1, true, w0t[iw], w0t[C::W0N + iw]);
    }
    if (2 * m <= jhi) fine_plane(2 * m, false, T(0), T(0));
#pragma unroll
    for (int i = 0; i < 5; ++i)
#pragma unroll
      for (int k = 0; k < NC1; ++k) A1p[i][k] = A1[i][k];
    __syncthreads();  // slots of planes 2m-1, 2m and coarse buffer m are free
    if (WITH) {
      if (m > ka && 2 * m - 1 + NS <= jhi) issue_f(2 * m - 1 + NS);
      if (2 * m <= jhi && 2 * m + NS <= jhi) issue_f(2 * m + NS);
    }
    if (m + 2 <= kb) issue_c(m + 2);
  }
  if (SUB && flag) {
    const bool nf = !(bad == T(0));
    if (__syncthreads_or(nf) && tid == 0) atomicOr(flag, 1);
  }
}

// The last fine column (e2-1, blockIdx.y = 0) and row (e1-1, columns < e2-1,
// blockIdx.y = 1) of fine plane blockIdx.x: one thread per cell
// (reference-order multilinear interpolation, kernels.cuh).
template <class T>
__global__ void __launch_bounds__(256)
    k_interp_face(const T* coef, T* out, const T* __restrict__ C, const T* __restrict__ Z,
                  LevelArgs<T> a, bool with) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int e1 = int(a.e[1]), e2 = int(a.e[2]);
  const int c1 = int(a.c[1]), c2 = int(a.c[2]);
  const int j = blockIdx.x, face = blockIdx.y;
  auto coarse = [&](int64_t q0, int64_t q1, int64_t q2) {
    const int64_t q = (q0 * c1 + q1) * c2 + q2;
    return Z ? C[q] - Z[q] : C[q];
  };
  const int n = face == 0 ? e1 : e2 - 1;
  const int64_t pbase = int64_t(j) * e1 * e2;
  const int q1 = min(n, int(blockIdx.z + 1) * int(blockDim.x));
  for (int q = int(blockIdx.z * blockDim.x + threadIdx.x); q < q1; q += blockDim.x) {
    const int r = face == 0 ? q : e1 - 1, c = face == 0 ? e2 - 1 : q;
    const int64_t idx = pbase + int64_t(r) * e2 + c;
    if (((j | r | c) & 1) == 0) {
      out[idx] = coarse(j >> 1, r >> 1, c >> 1);
    } else {
      const T ip = interp_node(a, j, r, c, coarse);
      out[idx] = with ? coef[idx] + ip : ip;
    }
  }
}

template <class T>
int interp_tiles(const LevelArgs<T>& a) {
  using Cf = ICfg<T>;
  const int64_t nt1 = (a.c[1] - 1 + Cf::TW1 - 1) / Cf::TW1;
  const int64_t nt2 = (a.c[2] - 1 + Cf::TW2 - 1) / Cf::TW2;
  return int(nt1 * nt2);
}

template <class T>
int interp_heuristic_s0(const LevelArgs<T>& a) {
  const int64_t tiles = interp_tiles(a);
  // B200 autotuning picks 8 coarse planes per CTA on every large level measured
  // (1025^3 / 513^3, fp32 and fp64: 1.47 vs 1.70 ms at 32 for the top fp32 level)
  int S0 = std::min(kMaxSegI, 8);
  while (S0 > 4 && tiles * std::max<int64_t>(1, (a.c[0] - 1) / S0) < 1200) S0 /= 2;
  return S0;
}

template <class T, bool WITH, bool HASZ, bool SUB = false>
void run_interp(const T* coef, T* out, const T* Cv, const T* Zv, const LevelArgs<T>& a,
                cudaStream_t s, int s0, int* flag = nullptr) {
  using Cf = ICfg<T>;
  auto kern = k_interp_march<T, WITH, HASZ, SUB>;
  if (a.e[1] == 1025 && a.e[2] == 1025) kern = k_interp_march<T, WITH, HASZ, SUB, 1025, 1025>;
  else if (a.e[1] == 513 && a.e[2] == 513) kern = k_interp_march<T, WITH, HASZ, SUB, 513, 513>;
  else if (a.e[1] == 513 && a.e[2] == 1025) kern = k_interp_march<T, WITH, HASZ, SUB, 513, 1025>;
  else if (a.e[1] == 257 && a.e[2] == 513) kern = k_interp_march<T, WITH, HASZ, SUB, 257, 513>;
  set_smem_attr(reinterpret_cast<const void*>(kern), Cf::total);
  const int nt1 = int((a.c[1] - 1 + Cf::TW1 - 1) / Cf::TW1);
  const int nt2 = int((a.c[2] - 1 + Cf::TW2 - 1) / Cf::TW2);
  const int64_t tiles = int64_t(nt1) * nt2;
  const int S0 = s0 > 0 ? std::min(s0, kMaxSegI) : interp_heuristic_s0(a);
  const int nseg = int(std::max<int64_t>(1, (a.c[0] - 1) / S0));
  constexpr int V = Cf::V;
  const int64_t plane_f = a.e[1] * a.e[2], plane_c = a.c[1] * a.c[2];
  const int64_t Nf = a.e[0] * plane_f, Nc = a.c[0] * plane_c;
  const int64_t lim = (int64_t(1) << 31) - 4 * int64_t(Cf::BOX);
  int sa = 0;
  while (sa < nseg) {
    // fine planes of segments sa..sb-1: [2*sa*S0, 2*(sb*S0) + 1]; coarse planes up to sb*S0 + 1
    auto f_hi = [&](int sg) { return std::min<int64_t>(a.e[0] - 1, 2 * (int64_t(sg) + 1) * S0); };
    const int64_t f_lo = 2 * int64_t(sa) * S0;
    int sb = sa + 1;
    while (sb < nseg && (f_hi(sb) + 1 - f_lo) * plane_f < lim) ++sb;
    require((f_hi(sb - 1) + 1 - f_lo) * plane_f < lim, "level too large for the 1D TMA path");
    const int64_t coef_off = (f_lo * plane_f) & ~int64_t(V - 1);
    const int64_t c_off = ((int64_t(sa) * S0) * plane_c) & ~int64_t(V - 1);
    CUtensorMap mcoef, mC, mZ;
    make_tma_1d(&mC, Cv + c_off, uint64_t(Nc - c_off), int(sizeof(T)), Cf::CBOX);
    mZ = mC;
    if (HASZ) make_tma_1d(&mZ, Zv + c_off, uint64_t(Nc - c_off), int(sizeof(T)), Cf::CBOX);
    mcoef = mC;
    if (WITH) make_tma_1d(&mcoef, coef + coef_off, uint64_t(Nf - coef_off), int(sizeof(T)), Cf::BOX);
    const int64_t blocks = tiles * (sb - sa);
    launch_pdl(kern, dim3(unsigned(blocks)), dim3(Cf::NT), Cf::total, s, Nf, mcoef, mC, mZ, coef_off, c_off, out, a, S0,
                                                     nt1, nt2, nseg, sa, flag);
    HGR_CUDA_CHECK(cudaGetLastError());
    sa = sb;
  }
}

}  // namespace

template <class T>
bool launch_interp_rec(const T* coef, T* out, const T* C, const T* Z, const LevelArgs<T>& a,
                       bool with, cudaStream_t s, int s0) {
  if (a.e[0] == 1 && a.e[1] == 1) return launch_line_interp<T>(coef, out, C, Z, a, with, s);
  const auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (a.e[1] < 3 || a.e[2] < 3 || !al(C) || (Z && !al(Z)) || (with && !al(coef))) return false;
  if (a.c[0] > 1 && ((a.c[0] - 1) & (a.c[0] - 2)) != 0) return false;
  if (a.c[0] * a.c[1] * a.c[2] >= (int64_t(1) << 31)) return false;
  if (with && Z) run_interp<T, true, true>(coef, out, C, Z, a, s, s0);
  else if (with) run_interp<T, true, false>(coef, out, C, Z, a, s, s0);
  else if (Z) run_interp<T, false, true>(coef, out, C, Z, a, s, s0);
  else run_interp<T, false, false>(coef, out, C, Z, a, s, s0);
  // the faces (last fine row / column) are written by the last tiles
  return true;
}

template <class T>
bool launch_coef_inplace(T* U, const T* C, const LevelArgs<T>& a, int* flag, cudaStream_t s,
                         int s0) {
  if (a.e[0] == 1 && a.e[1] == 1) return false;  // 1D: the line kernels
  const auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (a.e[1] < 3 || a.e[2] < 3 || !al(C) || !al(U)) return false;
  if (a.c[0] > 1 && ((a.c[0] - 1) & (a.c[0] - 2)) != 0) return false;
  if (a.c[0] * a.c[1] * a.c[2] >= (int64_t(1) << 31)) return false;
  run_interp<T, true, false, true>(U, U, C, nullptr, a, s, s0, flag);
  return true;
}

template <class T>
int interp_default_s0(const LevelArgs<T>& a) {
  return interp_heuristic_s0(a);
}

template <class T>
std::vector<SegChoice> interp_candidates(const LevelArgs<T>& a, bool with, bool hasz,
                                         double bw_gbs) {
  using Cf = ICfg<T>;
  const double S = double(sizeof(T));
  const int64_t tiles = interp_tiles(a);
  const double slots = 148.0 * Cf::MINB;
  auto sectors = [&](double elems) { return std::ceil(elems * S / 32.0) * 32.0 / S; };
  std::vector<SegChoice> out;
  int last_nseg = -1;
  for (int S0 = kMaxSegI; S0 >= 1; S0 /= 2) {
    const int nseg = int(std::max<int64_t>(1, (a.c[0] - 1) / S0));
    if (nseg == last_nseg) continue;
    last_nseg = nseg;
    const double fine = std::min<double>(double(a.e[0]), 2.0 * S0 + 1);
    const double coarse = std::min<double>(double(a.c[0]), S0 + 1.0);
    double elems = fine * Cf::FR * sectors(Cf::FC);                       // output rows
    if (with) elems += fine * Cf::FR * sectors(Cf::BOX);                  // coefficient rows
    elems += (hasz ? 2 : 1) * coarse * Cf::CR * sectors(Cf::CBOX);        // coarse (+ Z) rows
    const double blocks = double(tiles) * nseg;
    const double waves = std::ceil(blocks / slots) / (blocks / slots);
    out.push_back({S0, int(blocks), blocks * elems * S / (bw_gbs * 1e3) * waves});
  }
  std::stable_sort(out.begin(), out.end(),
                   [](const SegChoice& x, const SegChoice& y) { return x.model_us < y.model_us; });
  return out;
}

template int interp_default_s0<float>(const LevelArgs<float>&);
template int interp_default_s0<double>(const LevelArgs<double>&);
template std::vector<SegChoice> interp_candidates<float>(const LevelArgs<float>&, bool, bool,
                                                         double);
template std::vector<SegChoice> interp_candidates<double>(const LevelArgs<double>&, bool, bool,
                                                          double);

template bool launch_interp_rec<float>(const float*, float*, const float*, const float*,
                                       const LevelArgs<float>&, bool, cudaStream_t, int);
template bool launch_interp_rec<double>(const double*, double*, const double*, const double*,
                                        const LevelArgs<double>&, bool, cudaStream_t, int);
template bool launch_coef_inplace<float>(float*, const float*, const LevelArgs<float>&, int*,
                                         cudaStream_t, int);
template bool launch_coef_inplace<double>(double*, const double*, const LevelArgs<double>&, int*,
                                          cudaStream_t, int);

}  // namespace hgrb
