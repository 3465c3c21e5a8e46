// kernels_stream.cu -- IPK passes (thomas_pass, correction.hpp:262-278) as
// streaming column solves: one CTA per SM marches down a "matrix" whose columns
// are the lines of the pass, band by band, with the bands arriving by bulk
// copies (TMA engine) into a ring of shared-memory slots several bands ahead.
//
//   A job = W adjacent columns of one matrix (rows = line positions, row pitch
//   = the line stride):
//     dim 0:          the level array as a c0 x (c1*c2) matrix, jobs = column strips;
//     dim 1:          every dim-0 plane as a c1 x c2 matrix, jobs = column strips;
//     dims 1+2 (ROWS) every plane whole (W = c2): each band's rows are solved along
//                     dim 2 first (a warp per row, register chunks + shuffle scans,
//                     thomas_chunk.cuh), then the columns along dim 1 -- one HBM
//                     round trip for both passes.
//   One thread per column. Band b (R positions starting at s):
//     forward   y = x - m * y_prev   (exact: the carry y_prev is the previous
//               band's last y, the bands of a job run in order on one CTA);
//     backward  h = (y - u * h) / p  with zero carry at the band end, kept in
//               the slot; by linearity z = h + c_b * Q with the line-independent
//               product table Q (Q_i = prod_{k=i..e-1} -u_k/p_k) and the carry
//               c_b = z at the next band's first position;
//     band b-K is finished once band b has been solved:
//               c_b(b-K) = sum_t (prod_{t'<t} Q0(b-K+t')) h0(b-K+t),  t = 1..K,
//               dropping the term of z past band b, which every backward factor
//               (<= 1/2, thomas_chunk.cuh) damps by 2^-(K*R) <= 2^-56 (fp64) /
//               2^-26 (fp32) -- the bound of the windowed kernels. The last K
//               bands of a job are finished exactly.
//   Results are written as coalesced rows. A producer warp keeps every free
//   slot of the ring filled (full/empty mbarrier pairs); the ring holds the K
//   unfinished bands plus the bands in flight, so every SM keeps 100+ KB of
//   loads in flight (Little's law at ~44 GB/s per SM) while the consumer warps,
//   each column independent of the others, compute without CTA barriers.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "kernels_fused.cuh"
#include "launch.cuh"
#include "plan.hpp"
#include "ptx.cuh"
#include "thomas_chunk.cuh"

namespace hgrb {

namespace {

using namespace thomas;

constexpr int kStreamR = 16;      // line positions per band
constexpr int kStreamKMax = 4;    // lookahead bands (K * R >= 56)
constexpr int kStreamSlots = 16;  // ring slots (upper bound)

template <class T>
constexpr int sbits() {
  return sizeof(T) == 8 ? 56 : 26;
}

struct StreamGeo {
  int n;           // line length (matrix rows)
  int nb;          // bands of R positions
  int K;           // lookahead bands of the backward carry
  int nslot;       // ring slots
  int W;           // columns per job
  int jpm;         // jobs per matrix
  int ncols;       // columns of a matrix
  int njobs;       // matrices * jpm
  int SP;          // slot row pitch (elements), == pitch (mod 16 bytes)
  int slot;        // slot size (elements), a 16-byte multiple
  int64_t pitch;   // element stride between line positions
  int64_t mstride; // element stride between matrices
};

// shared-memory layout (in T units from the base): slots | tm tu tp tQ (n each,
// rounded up to whole bands and zero past the line) | q0 (nb) | row tables
// (ROWS) | mbarriers
struct StreamLayout {
  int tabs, q0, rows, bars;
  size_t bytes;
};
template <class T>
__host__ __device__ inline StreamLayout stream_layout(const StreamGeo& g, int rnt) {
  constexpr int V = int(16 / sizeof(T));
  StreamLayout L;
  L.tabs = g.nslot * g.slot;
  // whole bands: a band's 16-entry table loads stay inside its own (zeroed) table
  const int nn = (g.n + kStreamR - 1) / kStreamR * kStreamR;
  L.q0 = L.tabs + 4 * nn;
  L.rows = L.q0 + (g.nb + V - 1) / V * V;
  L.bars = L.rows + 5 * rnt;  // 16-byte aligned (every piece is a 16-byte multiple)
  L.bytes = size_t(L.bars) * sizeof(T) + size_t(3 * kStreamSlots) * 8;
  return L;
}

// R consecutive table entries (16-byte aligned) into registers
template <class T, int R>
__device__ __forceinline__ void load_tab(const T* t, T (&v)[R]) {
  using VV = Vec16<T>;
  constexpr int N = VV::N;
#pragma unroll
  for (int i = 0; i < R; i += N) {
    T w[N];
    VV::split(reinterpret_cast<const typename VV::type*>(t)[i / N], w);
#pragma unroll
    for (int k = 0; k < N; ++k) v[i + k] = w[k];
  }
}

// NT consumer threads (one column each; ROWS: also a warp per row) plus one
// producer warp that refills the ring: full[s] completes when slot s's bytes
// have landed, empty[s] when every consumer warp has finished the band in it.
template <class T, int NT, bool ROWS, int CHR, int KR>
__global__ void __launch_bounds__(NT + 32, 1)
    k_thomas_stream(const T* in, T* out, StreamGeo G, const T* __restrict__ mult,
                    const T* __restrict__ rpiv, const T* __restrict__ upper,
                    const T* __restrict__ rmult, const T* __restrict__ rrpiv,
                    const T* __restrict__ rupper) {
  constexpr int V = int(16 / sizeof(T)), R = kStreamR, NWC = NT / 32;
  constexpr int CHRP = ROWS ? chunk_pitch<T, CHR>() : 1;
  constexpr int RNT = ROWS ? 32 * CHRP : 0;
  static_assert(R % V == 0, "bands start on 16-byte table boundaries");
  ptx::pdl_trigger();
  extern __shared__ __align__(128) unsigned char smem_st[];
  T* base = reinterpret_cast<T*>(smem_st);
  const StreamLayout L = stream_layout<T>(G, RNT);
  const int n = G.n, nb = G.nb, K = G.K, nslot = G.nslot;
  T* tm = base + L.tabs;
  const int nn = (n + R - 1) / R * R;  // whole bands (stream_layout)
  T* tu = tm + nn;
  T* tp = tu + nn;
  T* tQ = tp + nn;
  T* q0b = base + L.q0;
  T* rt = base + L.rows;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + L.bars);
  uint64_t* empty = full + kStreamSlots;
  const int tid = threadIdx.x, lane = tid & 31, wp = ptx::warp_id_uniform();

  // ---- tables (plan constants): column line factors (zero past the line),
  // per-band Q products
  for (int i = tid; i < nn; i += NT + 32) {
    const bool in_l = i < n;
    tm[i] = (in_l && i >= 1) ? mult[i - 1] : T(0);
    tp[i] = in_l ? rpiv[i] : T(0);
    tu[i] = (in_l && i < n - 1) ? upper[i] : T(0);
    tQ[i] = T(0);
  }
  if (tid == 0) {
    for (int b = 0; b < nslot; ++b) {
      ptx::mbar_init(&full[b], 1);
      ptx::mbar_init(&empty[b], NWC * 32);  // every consumer lane arrives
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  for (int b = tid; b < nb; b += NT + 32) {
    const int s = b * R, e = min(n, s + R);
    T q = T(1);
    for (int i = e - 1; i >= s; --i) {
      q *= -(tu[i] * tp[i]);
      tQ[i] = q;
    }
    q0b[b] = q;
  }
  if constexpr (ROWS)
    build_tables(rt, rt + RNT, rt + 2 * RNT, rt + 3 * RNT, rt + 4 * RNT, G.ncols, 32, CHR, CHRP,
                 rmult, rrpiv, rupper);  // ends with __syncthreads
  else
    __syncthreads();

  // ---- this CTA's items: (job J = blockIdx.x + jl * gridDim.x, band b), jl-major
  const int G0 = int(gridDim.x);
  const int myjobs = int(blockIdx.x) < G.njobs ? (G.njobs - int(blockIdx.x) + G0 - 1) / G0 : 0;
  const int64_t nitems = int64_t(myjobs) * nb;
  struct Job {
    int64_t g0;  // element offset of (position 0, column 0)
    int w;       // columns
  };
  auto job = [&](int jl) {
    const int J = int(blockIdx.x) + jl * G0;
    const int mat = J / G.jpm, jc = J - mat * G.jpm;
    const int col0 = jc * G.W;
    Job r;
    r.g0 = int64_t(mat) * G.mstride + col0;
    r.w = min(G.W, G.ncols - col0);
    return r;
  };
  ptx::pdl_wait();  // the lines are the previous launches' output

  if (wp == NWC) {
    // ---- producer warp: row r of band b lands at PH0 + r*SP - ph_r (16-byte
    // aligned because SP == pitch (mod V)); a whole-row band is one copy
    const bool whole = G.W == G.ncols && int64_t(G.ncols) == G.pitch;
    int jl = 0, b = 0, sl = 0;
    uint32_t use = 0;
    Job jb = myjobs > 0 ? job(0) : Job{0, 0};
    for (int64_t it = 0; it < nitems; ++it) {
      if (use > 0) ptx::mbar_wait(&empty[sl], (use - 1) & 1);
      const int s = b * R, B = min(R, n - s);
      const int64_t g0 = jb.g0 + int64_t(s) * G.pitch;
      const int ph0 = int(g0 & (V - 1));
      T* dst = base + sl * G.slot;
      if (whole) {
        // one contiguous block, cut into 2 KB pieces issued by the lanes (a
        // single large bulk copy from one thread streams far below the HBM rate)
        constexpr uint32_t PIECE = 2048;
        const uint32_t by = uint32_t((ph0 + B * G.ncols + V - 1) / V * V * sizeof(T));
        if (lane == 0) ptx::mbar_arrive_expect_tx(&full[sl], by);
        __syncwarp();
        const char* src = reinterpret_cast<const char*>(in + (g0 - ph0));
        for (uint32_t off = uint32_t(lane) * PIECE; off < by; off += 32 * PIECE)
          ptx::bulk_g2s(reinterpret_cast<char*>(dst) + off, src + off, min(PIECE, by - off),
                        &full[sl]);
      } else {
        uint32_t mine = 0;
        for (int r = lane; r < B; r += 32) {
          const int phr = int((g0 + int64_t(r) * G.pitch) & (V - 1));
          mine += uint32_t((phr + jb.w + V - 1) / V * V * sizeof(T));
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
        if (lane == 0) ptx::mbar_arrive_expect_tx(&full[sl], mine);
        __syncwarp();
        for (int r = lane; r < B; r += 32) {
          const int64_t gr = g0 + int64_t(r) * G.pitch;
          const int phr = int(gr & (V - 1));
          ptx::bulk_g2s(dst + (ph0 + r * G.SP - phr), in + (gr - phr),
                        uint32_t((phr + jb.w + V - 1) / V * V * sizeof(T)), &full[sl]);
        }
      }
      if (++sl == nslot) {
        sl = 0;
        ++use;
      }
      if (++b == nb) {
        b = 0;
        if (++jl < myjobs) jb = job(jl);
      }
    }
    return;
  }

  // ---- consumers
  T yprev = T(0);
  constexpr bool REGH = KR > 0;  // the KR pending bands live in registers
  T hprev[REGH ? KR : 1][REGH ? R : 1];  // backward-local values of bands b-1 (, b-2)
  T h0r[kStreamKMax + 1];  // h0r[k]: first backward-local value of band b - k
#pragma unroll
  for (int k = 0; k <= kStreamKMax; ++k) h0r[k] = T(0);
  int jl = 0, b = 0, sl = 0;
  uint32_t use = 0;
  Job jb = myjobs > 0 ? job(0) : Job{0, 0};
  // finish band b - d (its slot sf): z = h + c_b * Q, coalesced row stores
  auto finish = [&](int d, int sf, auto full_c) {
    constexpr bool FULL = decltype(full_c)::value;
    const int bf = b - d, s0 = bf * R, Bf = FULL ? R : min(R, n - s0);
    // c_b = sum over bands bf+1 .. b (h0r[d-1] .. h0r[0]) of prod(Q0 before) * h0
    T cb = T(0), coef = T(1);
#pragma unroll
    for (int k = kStreamKMax; k >= 0; --k)
      if (k < d) {
        cb += coef * h0r[k];
        coef *= q0b[b - k];
      }
    const int64_t gf = jb.g0 + int64_t(s0) * G.pitch;
    const T* cf = base + sf * G.slot + int(gf & (V - 1)) + tid;
    T q[R];
    load_tab<T, R>(tQ + s0, q);
    T* o = out + gf + tid;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (FULL || r < Bf) *o = cf[r * G.SP] + cb * q[r];
      o += G.pitch;
    }
  };
  for (int64_t it = 0; it < nitems; ++it) {
    const int s = b * R, B = min(R, n - s);
    T* S = base + sl * G.slot;
    const int ph0 = int((jb.g0 + int64_t(s) * G.pitch) & (V - 1));
    ptx::mbar_wait(&full[sl], use & 1);

    // ---- ROWS: the band's rows along dim 2 (a warp per row, CHR per lane)
    if constexpr (ROWS) {
      constexpr int KD = scan_depth<T, CHR>() < 31 ? scan_depth<T, CHR>() : 31;
      const int P = G.ncols;
      const int q0 = lane * CHR;
      const T* rtm = rt + lane * CHRP;
      const T* rtP = rtm + RNT;
      const T* rtp = rtP + RNT;
      const T* rtu = rtp + RNT;
      const T* rtQ = rtu + RNT;
      const T pend = rtP[CHR - 1], qfirst = rtQ[0];
      // two rows per warp: the per-lane chunk tables are read once for both
      constexpr int RL = 2;
      for (int r0 = RL * wp; r0 < B; r0 += RL * NWC) {
        T y[RL][CHR];
#pragma unroll
        for (int u = 0; u < RL; ++u) {
          const T* row = S + ph0 + (r0 + u) * G.SP + q0;
          const bool ok = r0 + u < B;
#pragma unroll
          for (int k = 0; k < CHR; ++k) y[u][k] = (ok && q0 + k < P) ? row[k] : T(0);
        }
        T e[RL], c[RL];
        ChunkSolveV<T, CHR, RL>::fwd_local(y, rtm, e);
#pragma unroll
        for (int u = 0; u < RL; ++u) c[u] = T(0);
#pragma unroll
        for (int d = 0; d < KD; ++d) {
#pragma unroll
          for (int u = 0; u < RL; ++u) {
            const T t = __shfl_up_sync(0xffffffffu, e[u] + pend * c[u], 1);
            c[u] = lane == 0 ? T(0) : t;
          }
        }
        ChunkSolveV<T, CHR, RL>::apply(y, rtP, c);
        ChunkSolveV<T, CHR, RL>::bwd_local(y, rtu, rtp, e);
#pragma unroll
        for (int u = 0; u < RL; ++u) c[u] = T(0);
#pragma unroll
        for (int d = 0; d < KD; ++d) {
#pragma unroll
          for (int u = 0; u < RL; ++u) {
            const T t = __shfl_down_sync(0xffffffffu, e[u] + qfirst * c[u], 1);
            c[u] = lane == 31 ? T(0) : t;
          }
        }
        ChunkSolveV<T, CHR, RL>::apply(y, rtQ, c);
#pragma unroll
        for (int u = 0; u < RL; ++u) {
          T* row = S + ph0 + (r0 + u) * G.SP + q0;
          if (r0 + u < B) {
#pragma unroll
            for (int k = 0; k < CHR; ++k)
              if (q0 + k < P) row[k] = y[u][k];
          }
        }
      }
      ptx::named_sync(1, NT);
    }

    if (b == 0) yprev = T(0);
    const bool last = b == nb - 1;
    if constexpr (REGH) {
      // ---- K = KR <= 2: the column values go to registers and the slot back to
      // the producer at once; the pending bands' backward-local values wait in
      // registers (hprev) for their carries: c_b(b-1) = h0(b) (K = 1), c_b(b-2) =
      // h0(b-1) + Q0(b-1) h0(b) (K = 2; exact at the line end)
      const bool act = tid < jb.w;
      T x[R];
      const T* col = S + ph0 + tid;
#pragma unroll
      for (int r = 0; r < R; ++r) x[r] = (act && r < B) ? col[r * G.SP] : T(0);
      ptx::mbar_arrive(&empty[sl]);  // each lane releases its own reads
      if (act) {
        T t1[R], t2[R];
        load_tab<T, R>(tm + s, t1);
        T y = yprev;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          y = x[r] - t1[r] * y;  // tm = 0 past the line: y stays 0 there
          x[r] = y;
        }
        yprev = y;
        load_tab<T, R>(tu + s, t1);
        load_tab<T, R>(tp + s, t2);
        T h = T(0);
#pragma unroll
        for (int r = R - 1; r >= 0; --r) {
          h = (x[r] - t1[r] * h) * t2[r];  // tp = 0 past the line: h stays 0 there
          x[r] = h;
        }
        if constexpr (KR == 1) {
          if (b > 0) {  // band b-1 is full
            load_tab<T, R>(tQ + (s - R), t1);
            T* o = out + jb.g0 + int64_t(s - R) * G.pitch + tid;
#pragma unroll
            for (int r = 0; r < R; ++r) {
              *o = hprev[0][r] + h * t1[r];
              o += G.pitch;
            }
          }
        } else {
          if (b >= 2) {  // band b-2 (full)
            const T cb = hprev[0][0] + q0b[b - 1] * h;
            load_tab<T, R>(tQ + (s - 2 * R), t1);
            T* o = out + jb.g0 + int64_t(s - 2 * R) * G.pitch + tid;
#pragma unroll
            for (int r = 0; r < R; ++r) {
              *o = hprev[1][r] + cb * t1[r];
              o += G.pitch;
            }
          }
          if (last && b >= 1) {  // band b-1 (full), exactly
            load_tab<T, R>(tQ + (s - R), t1);
            T* o = out + jb.g0 + int64_t(s - R) * G.pitch + tid;
#pragma unroll
            for (int r = 0; r < R; ++r) {
              *o = hprev[0][r] + h * t1[r];
              o += G.pitch;
            }
          }
        }
        if (last) {  // the line ends here: zero carry
          T* o = out + jb.g0 + int64_t(s) * G.pitch + tid;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (r < B) *o = x[r];
            o += G.pitch;
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if constexpr (KR == 2) hprev[1][r] = hprev[0][r];
          hprev[0][r] = x[r];
        }
      }
    } else {
    // ---- columns: forward with the exact carry, backward-local (kept in the
    // slot), then finish band b - K (every remaining band at the job's end)
    const int nfin = last ? min(K, b) + 1 : (b >= K ? 1 : 0);
    if (tid < jb.w) {
      T* col = S + ph0 + tid;
      auto solve = [&](auto full_c) {
        constexpr bool FULL = decltype(full_c)::value;
        T x[R], t1[R], t2[R];
#pragma unroll
        for (int r = 0; r < R; ++r) x[r] = (FULL || r < B) ? col[r * G.SP] : T(0);
        load_tab<T, R>(tm + s, t1);
        T y = yprev;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          y = x[r] - t1[r] * y;
          x[r] = y;
          if (!FULL && r == B - 1) yprev = y;
        }
        if (FULL) yprev = y;
        load_tab<T, R>(tu + s, t1);
        load_tab<T, R>(tp + s, t2);
        T h = T(0);
#pragma unroll
        for (int r = R - 1; r >= 0; --r) {
          h = (x[r] - t1[r] * h) * t2[r];  // tp = 0 past the line: h stays 0 there
          x[r] = h;
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (FULL || r < B) col[r * G.SP] = x[r];
#pragma unroll
        for (int k = kStreamKMax; k >= 1; --k) h0r[k] = h0r[k - 1];
        h0r[0] = h;
      };
      if (B == R) solve(std::true_type{});
      else solve(std::false_type{});
      if (!last) {
        if (b >= K) {
          int sf = sl - K;
          if (sf < 0) sf += nslot;
          finish(K, sf, std::true_type{});
        }
      } else {
        for (int d = min(K, b); d >= 0; --d) {
          int sf = sl - d;
          if (sf < 0) sf += nslot;
          if (d == 0 && B != R) finish(0, sf, std::false_type{});
          else finish(d, sf, std::true_type{});
        }
      }
    }
    // release the finished bands' slots to the producer (generic-proxy reads and
    // writes of this warp ordered before the next bulk copy into them)
    if (nfin > 0) {
      ptx::fence_proxy_async_smem();
      for (int d = nfin - 1; d >= 0; --d) {  // each lane releases its own accesses
        const int dd = last ? d : K;
        int sf = sl - dd;
        if (sf < 0) sf += nslot;
        ptx::mbar_arrive(&empty[sf]);
      }
    }
    }  // !REGH
    if (++sl == nslot) {
      sl = 0;
      ++use;
    }
    if (last) {
      b = 0;
      if (++jl < myjobs) jb = job(jl);
    } else {
      ++b;
    }
  }
}

// Whole planes, dims 1 + 2, one lookahead band (K = 1, fp32): the row and
// column phases of consecutive bands overlap on separate warps.
//   producer warp     refills free slots (full[s] = bytes landed);
//   RWN row warps     solve the band's rows along dim 2, two rows per warp, in
//                     the slot (rows[s] = every row warp is done);
//   CW column warps   two columns per thread (c and c + 32*CW): load the band's
//                     column values into registers, hand the slot back
//                     (empty[s]), solve along dim 1 and finish band b-1 from
//                     registers with c_b = h0(b).
// So the dim-2 solve of band b+1 runs while the dim-1 solve of band b does.
// registers per thread for one CTA per SM: the warps are spread over the four
// SM sub-partitions, each with a 16K-register file, so the busiest one holds
// ceil(warps / 4) warps (launch bounds alone let ptxas stop below this)
constexpr int ws_maxnreg(int nth) {
  return (16384 / (((nth / 32) + 3) / 4 * 32)) / 8 * 8 > 255
             ? 255
             : (16384 / (((nth / 32) + 3) / 4 * 32)) / 8 * 8;
}

template <class T, int CHR, int CW, int RWN, bool PROV, int PC>
__global__ void __maxnreg__(ws_maxnreg((CW + RWN + 1) * 32))
    k_thomas_planes_ws(const T* in, T* out, StreamGeo G, const T* __restrict__ mult,
                       const T* __restrict__ rpiv, const T* __restrict__ upper,
                       const T* __restrict__ rmult, const T* __restrict__ rrpiv,
                       const T* __restrict__ rupper) {
  constexpr int V = int(16 / sizeof(T)), R = kStreamR, RL = 2;
  constexpr int NTH = (CW + RWN + 1) * 32;
  constexpr int CHRP = chunk_pitch<T, CHR>();
  constexpr int RNT = 32 * CHRP;
  static_assert(RL * RWN >= R, "two rows per row warp cover a band");
  ptx::pdl_trigger();
  extern __shared__ __align__(128) unsigned char smem_st[];
  T* base = reinterpret_cast<T*>(smem_st);
  const StreamLayout L = stream_layout<T>(G, RNT);
  const int n = G.n, nb = G.nb, nslot = G.nslot;
  T* tm = base + L.tabs;
  const int nn = (n + R - 1) / R * R;  // whole bands (stream_layout)
  T* tu = tm + nn;
  T* tp = tu + nn;
  T* tQ = tp + nn;
  T* rt = base + L.rows;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + L.bars);
  uint64_t* rowsd = full + kStreamSlots;
  uint64_t* empty = rowsd + kStreamSlots;
  const int tid = threadIdx.x, lane = tid & 31, wp = ptx::warp_id_uniform();

  for (int i = tid; i < nn; i += NTH) {
    const bool in_l = i < n;
    tm[i] = (in_l && i >= 1) ? mult[i - 1] : T(0);
    tp[i] = in_l ? rpiv[i] : T(0);
    tu[i] = (in_l && i < n - 1) ? upper[i] : T(0);
    tQ[i] = T(0);
  }
  if (tid == 0) {
    for (int b = 0; b < nslot; ++b) {
      ptx::mbar_init(&full[b], 1);
      ptx::mbar_init(&rowsd[b], RWN * 32);  // every lane of the row warps arrives
      ptx::mbar_init(&empty[b], CW * 32);  // every lane of the column warps arrives
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  T* q0b = base + L.q0;
  for (int b = tid; b < nb; b += NTH) {
    const int s = b * R, e = min(n, s + R);
    T q = T(1);
    for (int i = e - 1; i >= s; --i) {
      q *= -(tu[i] * tp[i]);
      tQ[i] = q;
    }
    q0b[b] = q;
  }
  build_tables(rt, rt + RNT, rt + 2 * RNT, rt + 3 * RNT, rt + 4 * RNT, G.ncols, 32, CHR, CHRP, rmult,
               rrpiv, rupper);  // ends with __syncthreads

  // jobs = planes: plane J = blockIdx.x + jl * gridDim.x, bands 0..nb-1
  const int G0 = int(gridDim.x);
  const int myjobs = int(blockIdx.x) < G.njobs ? (G.njobs - int(blockIdx.x) + G0 - 1) / G0 : 0;
  const int64_t nitems = int64_t(myjobs) * nb;
  const int P = PC > 0 ? PC : G.ncols;  // row length == pitch == W (PC: compile time)
  ptx::pdl_wait();  // the planes are the previous launches' output

  if (wp == CW + RWN) {
    // ---- producer: one contiguous block per band, 2 KB pieces over the lanes
    int jl = 0, b = 0, sl = 0;
    uint32_t use = 0;
    for (int64_t it = 0; it < nitems; ++it) {
      if (use > 0) ptx::mbar_wait(&empty[sl], (use - 1) & 1);
      const int s = b * R, B = min(R, n - s);
      const int64_t g0 = int64_t(int(blockIdx.x) + jl * G0) * G.mstride + int64_t(s) * P;
      const int ph0 = int(g0 & (V - 1));
      constexpr uint32_t PIECE = 2048;
      const uint32_t by = uint32_t((ph0 + B * P + V - 1) / V * V * sizeof(T));
      if (lane == 0) ptx::mbar_arrive_expect_tx(&full[sl], by);
      __syncwarp();
      const char* src = reinterpret_cast<const char*>(in + (g0 - ph0));
      char* dst = reinterpret_cast<char*>(base + sl * G.slot);
      for (uint32_t off = uint32_t(lane) * PIECE; off < by; off += 32 * PIECE)
        ptx::bulk_g2s(dst + off, src + off, min(PIECE, by - off), &full[sl]);
      if (++sl == nslot) {
        sl = 0;
        ++use;
      }
      if (++b == nb) {
        b = 0;
        ++jl;
      }
    }
    return;
  }

  if (wp >= CW) {
    // ---- row warps: rows 2*rw, 2*rw+1 of every band along dim 2
    constexpr int KD = scan_depth<T, CHR>() < 31 ? scan_depth<T, CHR>() : 31;
    const int rw = wp - CW;
    const int q0 = lane * CHR;
    const T* rtm = rt + lane * CHRP;
    const T* rtP = rtm + RNT;
    const T* rtp = rtP + RNT;
    const T* rtu = rtp + RNT;
    const T* rtQ = rtu + RNT;
    const T pend = rtP[CHR - 1], qfirst = rtQ[0];
    int jl = 0, b = 0, sl = 0;
    uint32_t use = 0;
    for (int64_t it = 0; it < nitems; ++it) {
      const int s = b * R, B = min(R, n - s);
      const int64_t g0 = int64_t(int(blockIdx.x) + jl * G0) * G.mstride + int64_t(s) * P;
      const int ph0 = int(g0 & (V - 1));
      T* S = base + sl * G.slot;
      ptx::mbar_wait(&full[sl], use & 1);
      const int r0 = RL * rw;
      if (r0 < B) {
        T y[RL][CHR];
#pragma unroll
        for (int u = 0; u < RL; ++u) {
          const T* row = S + ph0 + (r0 + u) * P + q0;
          const bool ok = r0 + u < B;
#pragma unroll
          for (int k = 0; k < CHR; ++k) y[u][k] = (ok && q0 + k < P) ? row[k] : T(0);
        }
        T e[RL], c[RL];
        ChunkSolveV<T, CHR, RL>::fwd_local(y, rtm, e);
#pragma unroll
        for (int u = 0; u < RL; ++u) c[u] = T(0);
#pragma unroll
        for (int d = 0; d < KD; ++d) {
#pragma unroll
          for (int u = 0; u < RL; ++u) {
            const T t = __shfl_up_sync(0xffffffffu, e[u] + pend * c[u], 1);
            c[u] = lane == 0 ? T(0) : t;
          }
        }
        ChunkSolveV<T, CHR, RL>::apply(y, rtP, c);
        ChunkSolveV<T, CHR, RL>::bwd_local(y, rtu, rtp, e);
#pragma unroll
        for (int u = 0; u < RL; ++u) c[u] = T(0);
#pragma unroll
        for (int d = 0; d < KD; ++d) {
#pragma unroll
          for (int u = 0; u < RL; ++u) {
            const T t = __shfl_down_sync(0xffffffffu, e[u] + qfirst * c[u], 1);
            c[u] = lane == 31 ? T(0) : t;
          }
        }
        ChunkSolveV<T, CHR, RL>::apply(y, rtQ, c);
#pragma unroll
        for (int u = 0; u < RL; ++u) {
          T* row = S + ph0 + (r0 + u) * P + q0;
          if (r0 + u < B) {
#pragma unroll
            for (int k = 0; k < CHR; ++k)
              if (q0 + k < P) row[k] = y[u][k];
          }
        }
      }
      ptx::mbar_arrive(&rowsd[sl]);  // each lane releases its own row writes
      if (++sl == nslot) {
        sl = 0;
        ++use;
      }
      if (++b == nb) {
        b = 0;
        ++jl;
      }
    }
    return;
  }

  // ---- column warps: columns tid and tid + 32*CW
  constexpr int CPT = 2;
  const int K = G.K;
  T yprev[CPT], hprev[PROV ? 1 : CPT][PROV ? 1 : R];
  T h0h[PROV ? CPT : 1][kStreamKMax + 1];  // PROV: first backward-local values of bands b-k
#pragma unroll
  for (int u = 0; u < (PROV ? CPT : 1); ++u)
#pragma unroll
    for (int k = 0; k <= kStreamKMax; ++k) h0h[u][k] = T(0);
#pragma unroll
  for (int u = 0; u < CPT; ++u) yprev[u] = T(0);
  int jl = 0, b = 0, sl = 0;
  uint32_t use = 0;
  for (int64_t it = 0; it < nitems; ++it) {
    const int s = b * R, B = min(R, n - s);
    const int64_t gj = int64_t(int(blockIdx.x) + jl * G0) * G.mstride;
    const int64_t g0 = gj + int64_t(s) * P;
    const int ph0 = int(g0 & (V - 1));
    const T* S = base + sl * G.slot + ph0;
    const bool last = b == nb - 1;
    ptx::mbar_wait(&rowsd[sl], use & 1);
    T x[CPT][R];
#pragma unroll
    for (int u = 0; u < CPT; ++u) {
      const int c = tid + u * 32 * CW;
#pragma unroll
      for (int r = 0; r < R; ++r) x[u][r] = (c < P && r < B) ? S[r * P + c] : T(0);
    }
    ptx::mbar_arrive(&empty[sl]);  // each lane releases its own reads
    if (b == 0) {
#pragma unroll
      for (int u = 0; u < CPT; ++u) yprev[u] = T(0);
    }
    T t1[R], t2[R];
    load_tab<T, R>(tm + s, t1);
#pragma unroll
    for (int u = 0; u < CPT; ++u) {
      T y = yprev[u];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        y = x[u][r] - t1[r] * y;  // tm = 0 past the line: y stays 0 there
        x[u][r] = y;
      }
      yprev[u] = y;
    }
    load_tab<T, R>(tu + s, t1);
    load_tab<T, R>(tp + s, t2);
    T h0[CPT];
#pragma unroll
    for (int u = 0; u < CPT; ++u) {
      T h = T(0);
#pragma unroll
      for (int r = R - 1; r >= 0; --r) {
        h = (x[u][r] - t1[r] * h) * t2[r];  // tp = 0 past the line: h stays 0 there
        x[u][r] = h;
      }
      h0[u] = h;
    }
    if constexpr (PROV) {
      // ---- K >= 1 pending bands without registers for them: band b goes out as
      // provisional values (final for the plane's last band), and band b-K is
      // corrected in place (L2-resident: written K bands ago) once c_b is known
#pragma unroll
      for (int u = 0; u < CPT; ++u) {
        const int c = tid + u * 32 * CW;
        if (c < P) {
          T* o = out + g0 + c;
#pragma unroll
          for (int r = 0; r < R; ++r)
            if (r < B) o[r * P] = x[u][r];
        }
#pragma unroll
        for (int k = kStreamKMax; k >= 1; --k) h0h[u][k] = h0h[u][k - 1];
        h0h[u][0] = h0[u];
      }
      auto fix = [&](int d) {  // band b-d (full): z += c_b * Q, c_b from bands b-d+1 .. b
        const int s0 = (b - d) * R;
        load_tab<T, R>(tQ + s0, t1);
#pragma unroll
        for (int u = 0; u < CPT; ++u) {
          const int c = tid + u * 32 * CW;
          T cb = T(0), coef = T(1);
#pragma unroll
          for (int k = kStreamKMax; k >= 0; --k)
            if (k < d) {
              cb += coef * h0h[u][k];
              coef *= q0b[b - k];
            }
          if (c < P) {
            T* o = out + gj + int64_t(s0) * P + c;
            T z[R];
#pragma unroll
            for (int r = 0; r < R; ++r) z[r] = o[r * P];
#pragma unroll
            for (int r = 0; r < R; ++r) o[r * P] = z[r] + cb * t1[r];
          }
        }
      };
      if (!last) {
        if (b >= K) fix(K);
      } else {
        for (int d = min(K, b); d >= 1; --d) fix(d);
      }
    } else {
    if (b > 0) {  // finish band b-1 (full) with c_b = h0(b)
      load_tab<T, R>(tQ + (s - R), t1);
#pragma unroll
      for (int u = 0; u < CPT; ++u) {
        const int c = tid + u * 32 * CW;
        if (c < P) {
          T* o = out + gj + int64_t(s - R) * P + c;
#pragma unroll
          for (int r = 0; r < R; ++r) o[r * P] = hprev[u][r] + h0[u] * t1[r];
        }
      }
    }
    if (last) {  // the plane ends here: zero carry
#pragma unroll
      for (int u = 0; u < CPT; ++u) {
        const int c = tid + u * 32 * CW;
        if (c < P) {
          T* o = out + g0 + c;
#pragma unroll
          for (int r = 0; r < R; ++r)
            if (r < B) o[r * P] = x[u][r];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < CPT; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) hprev[u][r] = x[u][r];
    }  // !PROV
    if (++sl == nslot) {
      sl = 0;
      ++use;
    }
    if (last) {
      b = 0;
      ++jl;
    } else {
      ++b;
    }
  }
}

int stream_sm_count() {
  static std::mutex mu;
  static std::vector<int> cache;
  int dev = 0;
  HGR_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (int(cache.size()) <= dev) cache.resize(std::size_t(dev) + 1, 0);
  if (!cache[std::size_t(dev)])
    HGR_CUDA_CHECK(cudaDeviceGetAttribute(&cache[std::size_t(dev)], cudaDevAttrMultiProcessorCount, dev));
  return cache[std::size_t(dev)];
}

constexpr size_t kStreamSmem = 220 * 1024;

// Fill the ring geometry for a job width W; false if the tables and K + 1
// slots do not fit.
template <class T, int RNT, bool REGH>
bool stream_ring(StreamGeo& g, int min_slots = 0) {  // REGH: no slot holds a pending band
  constexpr int V = int(16 / sizeof(T));
  g.nb = (g.n + kStreamR - 1) / kStreamR;
  // g.K: the plan's lookahead (tables.hpp stream_lookahead), at most nb - 1
  g.K = std::max(1, std::min(g.K, g.nb - 1));
  if (g.K > kStreamKMax) return false;
  const bool whole = g.W == g.ncols && int64_t(g.ncols) == g.pitch;
  if (whole) {
    g.SP = g.ncols;
  } else {
    // smallest pitch >= W + 2V - 2 congruent to the line stride (mod V): the
    // aligned supersets of consecutive rows then never overlap
    const int want = int(g.pitch % V);
    g.SP = g.W + 2 * V - 2;
    while (g.SP % V != want) ++g.SP;
  }
  g.slot = (kStreamR * g.SP + 2 * V + V - 1) / V * V;
  g.nslot = 1;
  const StreamLayout L1 = stream_layout<T>(g, RNT);
  const size_t fixed = L1.bytes - size_t(g.slot) * sizeof(T);
  const size_t per = size_t(g.slot) * sizeof(T);
  const int held = REGH ? 0 : g.K;  // slots of unfinished bands
  const int need = min_slots > 0 ? min_slots : held + 3;
  if (fixed + per * size_t(need) > kStreamSmem) return false;
  const int fit = int((kStreamSmem - fixed) / per);
  g.nslot = std::min(kStreamSlots, fit);
  // more bands in flight than the current one plus two measured slower (A/B at
  // 1025^3 fp32, tools/ab_stream.sh); knob HGR_STREAM_SLOTS caps the ring
  static const int cap = [] {
    const char* v = std::getenv("HGR_STREAM_SLOTS");
    return v ? std::atoi(v) : 0;
  }();
  // (fp32); fp64 bands of 16 rows of 256 doubles take every slot that fits (A/B
  // at 1025^3 fp64: IPK 3.05 -> 2.98 ms with 6 slots instead of 5)
  g.nslot = std::min(g.nslot, cap > 0 ? cap : sizeof(T) == 8 ? g.nslot : std::max(need, held + 3));
  return g.nslot >= need;  // by default the current band and two in flight at least
}

template <class T, int NT, bool ROWS, int CHR>
bool run_stream(const T* in, T* out, StreamGeo g, const T* mult, const T* rpiv, const T* upper,
                const T* rmult, const T* rrpiv, const T* rupper, int64_t level_nodes,
                cudaStream_t s) {
  constexpr int RNT = ROWS ? 32 * chunk_pitch<T, CHR>() : 0;
  auto go = [&](auto kr_c) {
    constexpr int KR = decltype(kr_c)::value;
    if (!stream_ring<T, RNT, (KR > 0)>(g)) return false;
    const size_t smem = stream_layout<T>(g, RNT).bytes;
    auto kern = k_thomas_stream<T, NT, ROWS, CHR, KR>;
    set_smem_attr(reinterpret_cast<const void*>(kern), smem);
    const int grid = std::min(g.njobs, stream_sm_count());
    launch_pdl(kern, dim3(unsigned(grid)), dim3(NT + 32), smem, s, level_nodes, in, out, g, mult,
               rpiv, upper, rmult, rrpiv, rupper);
    return true;
  };
  // one lookahead band: the pending band lives in registers (knob HGR_STREAM_KR:
  // the most bands kept in registers; 2 fits the fp64 strips' 288 threads but
  // measured slower than the shared-memory slots, 3.15 vs 2.98 ms of fp64 IPK
  // per 1025^3 round trip; 0: always shared memory)
  static const int kr_max = [] {
    const char* v = std::getenv("HGR_STREAM_KR");
    return v ? std::atoi(v) : 1;
  }();
  const int nb = (g.n + kStreamR - 1) / kStreamR;
  const int k = std::max(1, std::min(g.K, nb - 1));  // the lookahead stream_ring settles on
  if (k <= 1 && kr_max >= 1) return go(std::integral_constant<int, 1>{});
  if (k == 2 && kr_max >= 2) return go(std::integral_constant<int, 2>{});
  return go(std::integral_constant<int, 0>{});
}

template <class T, int CHR, int CW, int RWN, bool PROV, int PC = 0>
bool run_planes_ws(const T* in, T* out, StreamGeo g, const T* mult, const T* rpiv, const T* upper,
                   const T* rmult, const T* rrpiv, const T* rupper, int64_t level_nodes,
                   cudaStream_t s) {
  constexpr int RNT = 32 * chunk_pitch<T, CHR>();
  if (g.ncols > 2 * 32 * CW || g.ncols > 32 * CHR) return false;
  // PROV (pending bands corrected in place in global memory): two slots suffice,
  // the column warps hand a slot back as soon as its band is in registers
  if (!stream_ring<T, RNT, true>(g, PROV ? 2 : 0)) return false;
  if (PC > 0 && g.ncols != PC) return false;
  auto kern = k_thomas_planes_ws<T, CHR, CW, RWN, PROV, PC>;
  // the ring as deep as one resident CTA allows (shared memory + registers)
  size_t smem = 0;
  for (;; --g.nslot) {
    smem = stream_layout<T>(g, RNT).bytes;
    set_smem_attr(reinterpret_cast<const void*>(kern), smem);
    int per_sm = 0;
    const cudaError_t oe =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (CW + RWN + 1) * 32, smem);
    if (oe != cudaSuccess) {
      cudaGetLastError();
      per_sm = 0;
    }

    if (per_sm > 0) break;
    if (g.nslot <= 2) return false;
  }
  const int grid = std::min(g.njobs, stream_sm_count());
  launch_pdl(kern, dim3(unsigned(grid)), dim3((CW + RWN + 1) * 32), smem, s, level_nodes, in, out, g,
             mult, rpiv, upper, rmult, rrpiv, rupper);
  return true;
}

// Column strips of `nmat` matrices of n rows x ncols columns (row pitch, matrix
// stride): the job width balances the jobs over the SMs (a multiple of 32
// columns, at most NT).
template <class T, int NT>
bool stream_strips(const T* in, T* out, int n, int64_t pitch, int64_t ncols, int64_t nmat,
                   int64_t mstride, int K, const T* mult, const T* rpiv, const T* upper,
                   int64_t level_nodes, cudaStream_t s) {
  if (ncols > (int64_t(1) << 30) || nmat * ncols > (int64_t(1) << 30)) return false;
  const int64_t sms = stream_sm_count();
  // smallest number of waves q such that W = ceil(cols / (q * sms / nmat)) fits NT
  int64_t W = 0, jpm = 0;
  for (int64_t q = 1; q < 4096; ++q) {
    const int64_t jobs = q * sms;
    jpm = std::max<int64_t>(1, (jobs + nmat - 1) / nmat);
    W = (ncols + jpm - 1) / jpm;
    W = (W + 31) / 32 * 32;
    if (W <= NT) break;
  }
  if (W > NT || W < 1) return false;
  jpm = (ncols + W - 1) / W;
  StreamGeo g{};
  g.n = n;
  g.W = int(W);
  g.jpm = int(jpm);
  g.ncols = int(ncols);
  g.njobs = int(nmat * jpm);
  g.pitch = pitch;
  g.mstride = mstride;
  g.K = K;
  return run_stream<T, NT, false, 1>(in, out, g, mult, rpiv, upper, nullptr, nullptr, nullptr,
                                     level_nodes, s);
}

}  // namespace

// IPK of a 3D level in two (fp32) or three (fp64) streaming passes:
//   dim 0 column strips of the c0 x (c1*c2) matrix, in place on src;
//   fp32: dims 1+2 on whole planes (ROWS), src -> dst;
//   fp64: dim 1 column strips of every plane in place, then the dim-2 row
//         kernel (k_thomas_rows) src -> dst.
// Returns the number of launches, 0 (nothing launched) when a pass does not
// fit; the caller then falls back to the other IPK kernels.
template <class T>
bool thomas_stream_supported(const int64_t c[3]) {
  constexpr bool F64 = sizeof(T) == 8;
  if (c[0] < 2 || c[1] < 2 || c[2] < 2) return false;
  if (c[0] > 1100 || c[1] > 1100) return false;  // column tables in shared memory
  if (!F64 && c[2] > 32 * 17) return false;      // plane rows: 17 per lane
  if (F64 && c[2] > 32 * 17) return false;       // k_thomas_rows register tiles
  return c[0] * c[1] * c[2] < (int64_t(1) << 40);
}

template <class T>
int launch_thomas_stream(T* src, T* dst, const int64_t c[3], const T* const mult[3],
                         const T* const rpiv[3], const T* const upper[3], const int K[3],
                         int64_t level_nodes, cudaStream_t s) {
  if (!thomas_stream_supported<T>(c)) return 0;
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) return 0;
  constexpr bool F64 = sizeof(T) == 8;
  const int64_t plane = c[1] * c[2];
  if (!stream_strips<T, F64 ? 256 : 512>(src, src, int(c[0]), plane, plane, 1, 0, K[0], mult[0], rpiv[0],
                                         upper[0], level_nodes, s))
    return 0;
  // fp32 planes whole (ROWS) by default; knob HGR_STREAM_PLANES=0: dim-1 strips
  // plus the row kernel, as fp64
  static const bool planes = [] {
    const char* v = std::getenv("HGR_STREAM_PLANES");
    return !v || v[0] != '0';
  }();
  // fp64 dims 1 + 2 on whole planes, pending bands corrected in place in global
  // memory (knob HGR_STREAM_PLANES64=1): two 66 KB slots only, and the
  // corrections re-write bands L2 has partly evicted (1025^3: 853 us against
  // 380 + 335 us for dim-1 strips + rows), so off by default
  const bool planes64 = [] {  // read per launch: tests switch it within a process
    const char* v = std::getenv("HGR_STREAM_PLANES64");
    return v && v[0] == '1';
  }();
  if (F64 && planes && planes64) {
    // fp64 dims 1 + 2 on whole planes: pending bands corrected in place
    StreamGeo g{};
    g.n = int(c[1]);
    g.W = int(c[2]);
    g.jpm = 1;
    g.ncols = int(c[2]);
    g.njobs = int(c[0]);
    g.pitch = c[2];
    g.mstride = plane;
    g.K = K[1];
    bool ok = false;
    if (c[2] <= 32 * 5)
      ok = run_planes_ws<T, 5, 3, 8, true>(src, dst, g, mult[1], rpiv[1], upper[1], mult[2], rpiv[2],
                                           upper[2], level_nodes, s);
    else if (c[2] <= 32 * 9)
      ok = run_planes_ws<T, 9, 5, 8, true>(src, dst, g, mult[1], rpiv[1], upper[1], mult[2], rpiv[2],
                                           upper[2], level_nodes, s);
    else
      ok = run_planes_ws<T, 17, 9, 8, true>(src, dst, g, mult[1], rpiv[1], upper[1], mult[2], rpiv[2],
                                            upper[2], level_nodes, s);
    if (ok) return 2;
  }
  if (F64 || !planes) {
    require(stream_strips<T, F64 ? 256 : 512>(src, src, int(c[1]), c[2], c[2], c[0], plane, K[1], mult[1], rpiv[1],
                                  upper[1], level_nodes, s),
            "thomas stream: dim-1 strips do not fit after the dim-0 pass ran");
    require(launch_thomas_fast<T>(src, dst, c, 2, mult[2], rpiv[2], upper[2], s),
            "thomas stream: dim-2 rows kernel unavailable after the dim-1 pass ran");
    return 3;
  } else {
    StreamGeo g{};
    g.n = int(c[1]);
    g.W = int(c[2]);
    g.jpm = 1;
    g.ncols = int(c[2]);
    g.njobs = int(c[0]);
    g.pitch = c[2];
    g.mstride = plane;
    g.K = K[1];
    bool ok = false;
    static const bool ws = [] {  // knob HGR_STREAM_WS=0: one warp set for both phases
      const char* v = std::getenv("HGR_STREAM_WS");
      return !v || v[0] != '0';
    }();
    if (ws && std::min(g.K, int((c[1] + kStreamR - 1) / kStreamR) - 1) <= 1) {
#define HGR_WS(CHR, CW, PC)                                                                      \
  run_planes_ws<T, CHR, CW, 8, false, PC>(src, dst, g, mult[1], rpiv[1], upper[1], mult[2], rpiv[2], \
                                          upper[2], level_nodes, s)
      // the 2^k+1 row lengths of the large levels at compile time (address and
      // guard arithmetic folds), any other length at run time
      if (c[2] == 513) ok = HGR_WS(17, 9, 513);
      else if (c[2] == 257) ok = HGR_WS(9, 5, 257);
      else if (c[2] == 129) ok = HGR_WS(5, 3, 129);
      else if (c[2] <= 32 * 5) ok = HGR_WS(5, 3, 0);
      else if (c[2] <= 32 * 9) ok = HGR_WS(9, 5, 0);
      else ok = HGR_WS(17, 9, 0);
#undef HGR_WS
    }
    if (ok) {
    } else if (c[2] <= 32 * 5) ok = run_stream<T, 160, true, 5>(src, dst, g, mult[1], rpiv[1], upper[1],
                                                         mult[2], rpiv[2], upper[2], level_nodes, s);
    else if (c[2] <= 32 * 9) ok = run_stream<T, 288, true, 9>(src, dst, g, mult[1], rpiv[1], upper[1],
                                                              mult[2], rpiv[2], upper[2], level_nodes, s);
    else ok = run_stream<T, 544, true, 17>(src, dst, g, mult[1], rpiv[1], upper[1], mult[2], rpiv[2],
                                           upper[2], level_nodes, s);
    require(ok, "thomas stream: the plane pass does not fit after the dim-0 pass ran");
    return 2;
  }
}

template bool thomas_stream_supported<float>(const int64_t*);
template bool thomas_stream_supported<double>(const int64_t*);
template int launch_thomas_stream<float>(float*, float*, const int64_t*, const float* const*,
                                         const float* const*, const float* const*, const int*,
                                         int64_t, cudaStream_t);
template int launch_thomas_stream<double>(double*, double*, const int64_t*, const double* const*,
                                           const double* const*, const double* const*, const int*,
                                           int64_t, cudaStream_t);

}  // namespace hgrb
