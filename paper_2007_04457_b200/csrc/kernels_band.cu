// kernels_band.cu -- IPK passes of 3D levels (thomas_pass, correction.hpp:262-278)
// solved by thread-block clusters, two passes instead of three:
//
//   k_thomas_band<ROWS = false>  dim 0: a job is W contiguous columns of the
//       (c1 x c2) plane at every dim-0 position;
//   k_thomas_band<ROWS = true>   dims 1 + 2 fused: a job is one dim-0 plane;
//       after the dim-1 solve the same shared-memory tile is solved along its
//       rows (dim 2), so the plane makes one HBM round trip for both passes.
//
// A line of n positions is cut into NB bands, one per CTA of a cluster
// (NB = ceil(n / 33) <= 16): each CTA stages its band of the job with bulk
// copies (TMA engine) into shared memory, and one thread per column solves its
// band with zero carries: g = forward-local(x), hg = backward-local(g). By
// linearity the true solution of band j is
//     z = hg + c_f * hP + c_b * Q
// with line-independent tables hP = backward-local(P) and Q (thomas_chunk.cuh),
// c_f = y at the end of band j-1 and c_b = z at the start of band j+1:
//     c_f(j)   = g_end(j-1)  + Pend(j-1) * c_f(j-1)
//     c_b(j)   = hg_0(j+1)   + c_f(j+1) * hP_0(j+1) + Q_0(j+1) * c_b(j+1)
// where g_end / hg_0 are the neighbours' local summaries, read through
// distributed shared memory after one cluster barrier, and Pend / hP_0 / Q_0
// per-band constants. Every forward multiplier and backward factor is at most
// 1/2 (thomas_chunk.cuh), so a band of B positions damps a carry by 2^-B and
// the chains stop after KB = ceil(bits / B_min) bands (contributions below
// 2^-56 fp64 / 2^-26 fp32 of a summary), exactly like the chunk scans of the
// register-tiled kernels. The reference recurrences (solve_fiber,
// correction.hpp:202-208) are otherwise evaluated in the same order.

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

constexpr int kBandMax = 33;   // positions per band (CTA)
constexpr int kMaxBands = 16;  // non-portable cluster size limit
constexpr int kKBMax = 4;      // carry-chain depth in bands
constexpr int kNbr = 2 * kKBMax + 1;

template <class T>
constexpr int vecn() {
  return int(16 / sizeof(T));
}
template <class T>
constexpr int band_pitch() {  // table stride of a band, 16-byte multiple
  return (kBandMax + vecn<T>() - 1) / vecn<T>() * vecn<T>();
}
template <class T>
constexpr int damp_bits() {
  return sizeof(T) == 8 ? 56 : 26;
}

// Job geometry: element (position p, column w) of job J lives at
//   J * jstride + p * sd + w,   0 <= w < (J == njobs-1 ? Wlast : W).
// ROWS: sd == W == row length c2 (a job is one contiguous plane).
struct BandGeo {
  int n;            // line length
  int nb;           // bands = cluster size
  int kb;           // carry-chain depth (bands)
  int njobs;
  int W, Wlast;     // columns per job
  int64_t sd;       // element stride between line positions
  int64_t jstride;  // element stride between jobs
};

__host__ __device__ inline int band_start(int j, int n, int nb) { return int((int64_t(j) * n) / nb); }

// per-band constants: Pend (forward carry through the band), hP0 (first entry
// of backward-local(P)), Q0 (backward carry through the band)
template <class T>
__device__ __noinline__ void band_constants(int s, int e, int n, const T* __restrict__ mult,
                               const T* __restrict__ rpiv, const T* __restrict__ upper, T& pend,
                               T& hp0, T& q0) {
  T P[kBandMax];
  T a = T(1);
#pragma unroll
  for (int i = 0; i < kBandMax; ++i) {
    const int pos = s + i;
    if (pos < e) a *= -(pos >= 1 ? mult[pos - 1] : T(0));
    P[i] = a;
  }
  pend = a;
  T h = T(0), q = T(1);
#pragma unroll
  for (int i = kBandMax - 1; i >= 0; --i) {
    const int pos = s + i;
    if (pos < e) {
      const T tu = pos < n - 1 ? upper[pos] : T(0), tp = rpiv[pos];
      h = (P[i] - tu * h) * tp;
      q *= -(tu * tp);
    }
  }
  hp0 = h;
  q0 = q;
}

// Shared-memory tile of a job: element (band position i, column c) at
//   ph0 + i * P + c,
// ph0 = the job's 16-byte phase. ROWS: the band is one contiguous block and
// P = the row length. Otherwise every position is its own bulk copy whose
// aligned superset lands at ph0 + i * P - ph_i (16-byte aligned because
// P == sd (mod V)), so the layout stays linear in i and every access is one
// shared-memory instruction with a compile-time offset.
template <class T, bool ROWS, int NT, int P, int CHR, int NBUF>
struct BandCfg {
  static constexpr int V = vecn<T>();
  static constexpr int BP = band_pitch<T>();
  static constexpr int NW = NT / 32;
  static constexpr int CHRP = chunk_pitch<T, CHR>();
  static constexpr int RNTB = ROWS ? 32 * CHRP : 0;  // row-table entries per table
  static constexpr int NCOL = (NT + V - 1) / V * V;  // summary slots (one column per thread)
  static constexpr int TE = (kBandMax * P + 2 * V + V - 1) / V * V;  // tile elements
  // NBUF tiles | band tables | neighbour constants | row tables | mbarriers (NBUF
  // tiles + 2 exchange) | received summaries [2 parity][3 kb - 1 slots][NCOL]
  static constexpr int OFF_TAB = NBUF * TE;
  static constexpr int OFF_NBR = OFF_TAB + 6 * BP;
  static constexpr int OFF_ROWS = OFF_NBR + (3 * kNbr + V - 1) / V * V;
  static constexpr int OFF_BAR = OFF_ROWS + 5 * RNTB;  // in T units; 16-byte aligned
  static constexpr size_t FIXED = size_t(OFF_BAR) * sizeof(T) + 32 + 8 * NBUF;
  static size_t bytes(int kb) {
    return (FIXED + 15) / 16 * 16 + size_t(2) * (3 * kb - 1 > 0 ? 3 * kb - 1 : 0) * NCOL * sizeof(T);
  }
};

// Local (zero-carry) forward and backward solves of one column's band: x ends
// as hg = backward-local(forward-local(column)); gend = forward-local at the
// band's last position, h0 = hg at its first. FULL: B is 32 or 33 (every
// band of a line longer than 33), so only position 32 is predicated.
template <class T, int P, bool FULL>
__device__ __forceinline__ void band_local(const T* col, int B, const T* tm, const T* tu,
                                           const T* tp, T (&x)[kBandMax], T& gend, T& h0) {
  using VV = Vec16<T>;
  constexpr int N = VV::N;
  T g = T(0);
  gend = T(0);
#pragma unroll
  for (int i0 = 0; i0 < kBandMax; i0 += N) {
    T m[N];
    VV::split(reinterpret_cast<const typename VV::type*>(tm)[i0 / N], m);
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int i = i0 + k;
      if (i < kBandMax) {
        const bool in = FULL ? (i < 32 || B > 32) : i < B;
        const T v = in ? col[i * P] : T(0);
        g = v - m[k] * g;
        x[i] = g;
        if (!FULL && i == B - 1) gend = g;
      }
    }
  }
  if (FULL) gend = B > 32 ? x[32] : x[31];
  T h = T(0);
  constexpr int I0 = (kBandMax - 1) / N * N;
#pragma unroll
  for (int i0 = I0; i0 >= 0; i0 -= N) {
    T uu[N], pp[N];
    VV::split(reinterpret_cast<const typename VV::type*>(tu)[i0 / N], uu);
    VV::split(reinterpret_cast<const typename VV::type*>(tp)[i0 / N], pp);
#pragma unroll
    for (int k = N - 1; k >= 0; --k) {
      const int i = i0 + k;
      if (i < kBandMax) {
        h = (x[i] - uu[k] * h) * pp[k];  // tp = 0 past the band: h stays 0 there
        x[i] = h;
      }
    }
  }
  h0 = h;
}

template <class T, bool ROWS, int NT, int P, int CHR, int NBUF, int MINB>
__global__ void __launch_bounds__(NT, MINB)
    k_thomas_band(const T* in, T* out, BandGeo G, const T* __restrict__ mult,
                  const T* __restrict__ rpiv, const T* __restrict__ upper,
                  const T* __restrict__ rmult, const T* __restrict__ rrpiv,
                  const T* __restrict__ rupper) {
  using C = BandCfg<T, ROWS, NT, P, CHR, NBUF>;
  constexpr int V = C::V, BP = C::BP, NW = C::NW, CHRP = C::CHRP, TE = C::TE;
  using VV = Vec16<T>;
  using VT = typename VV::type;
  ptx::pdl_trigger();
  extern __shared__ __align__(16) unsigned char smem_b[];
  T* tiles = reinterpret_cast<T*>(smem_b);
  T* tm = tiles + C::OFF_TAB;
  T* tp = tm + BP;
  T* tu = tp + BP;
  T* tP = tu + BP;
  T* tQ = tP + BP;
  T* thP = tQ + BP;
  T* nPend = tiles + C::OFF_NBR;  // [kNbr] constants of bands j - kKBMax .. j + kKBMax
  T* nhP0 = nPend + kNbr;
  T* nQ0 = nhP0 + kNbr;
  T* rt = tiles + C::OFF_ROWS;  // row tables (ROWS)
  uint64_t* xbar = reinterpret_cast<uint64_t*>(tiles + C::OFF_BAR);  // [2] summary exchange
  uint64_t* bar = xbar + 4;                                          // [NBUF] tile loads
  // summaries received from the neighbouring bands, per parity: slots
  // [0, kb) g_end(j-kb .. j-1), [kb, 2kb-1) g_end(j+1 .. j+kb-1), [2kb-1, 3kb-1) hg_0(j+1 .. j+kb)
  T* rsum = reinterpret_cast<T*>(smem_b + (C::FIXED + 15) / 16 * 16);

  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  const int j = int(ptx::cluster_ctarank());
  const int n = G.n, nb = G.nb, kb = G.kb;
  const int s = band_start(j, n, nb), B = band_start(j + 1, n, nb) - s;

  // ---- tables (plan constants: readable before the previous launch completes)
  if (tid < BP) {
    const int pos = s + tid;
    const bool inb = tid < B;
    tm[tid] = (inb && pos >= 1) ? mult[pos - 1] : T(0);
    tp[tid] = inb ? rpiv[pos] : T(0);
    tu[tid] = (inb && pos < n - 1) ? upper[pos] : T(0);
  }
  if (tid >= 64 - kNbr && tid < 64) {  // NT >= 64
    const int t = tid - (64 - kNbr), k = j + t - kKBMax;
    T pe = T(0), h0 = T(0), q0 = T(0);
    if (k >= 0 && k < nb)
      band_constants<T>(band_start(k, n, nb), band_start(k + 1, n, nb), n, mult, rpiv, upper, pe, h0,
                        q0);
    nPend[t] = pe;
    nhP0[t] = h0;
    nQ0[t] = q0;
  }
  if (tid == 0) {
    for (int b = 0; b < NBUF; ++b) ptx::mbar_init(&bar[b], 1);
    ptx::mbar_init(&xbar[0], 1);
    ptx::mbar_init(&xbar[1], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    T a = T(1);
    for (int i = 0; i < BP; ++i) {
      a *= -tm[i];
      tP[i] = i < B ? a : T(0);
    }
    T h = T(0), q = T(1);
    for (int i = BP - 1; i >= 0; --i) {
      if (i < B) q *= -(tu[i] * tp[i]);
      tQ[i] = i < B ? q : T(0);
      h = (tP[i] - tu[i] * h) * tp[i];
      thP[i] = h;
    }
  }
  if constexpr (ROWS) build_tables(rt, rt + C::RNTB, rt + 2 * C::RNTB, rt + 3 * C::RNTB,
                                   rt + 4 * C::RNTB, P, 32, CHR, CHRP, rmult, rrpiv, rupper);
  ptx::cluster_arrive();  // every CTA's exchange barriers exist before the first push
  ptx::cluster_wait();
  // summary pushes: receiver r of band j's values and the bytes a phase expects
  const int nslot = 3 * kb - 1 > 0 ? 3 * kb - 1 : 0;
  const uint32_t rs_base = ptx::smem_addr(rsum), xb_base = ptx::smem_addr(xbar);
  uint32_t xbytes = 0;
  for (int t = 1; t <= kb; ++t) {
    if (j - t >= 0) xbytes += 1;                    // g_end(j - t)
    if (j + t < nb) xbytes += t < kb ? 2 : 1;       // g_end(j + t) (t < kb), hg_0(j + t)
  }
  xbytes *= uint32_t(NT * sizeof(T));  // every thread pushes one value per slot

  const int ncl = int(gridDim.x) / nb;
  const int cid = int(blockIdx.x) / nb;
  auto jobW = [&](int J) { return J == G.njobs - 1 ? G.Wlast : G.W; };
  // global element offset of (job J, band position 0, column 0)
  auto gbase = [&](int J) { return int64_t(J) * G.jstride + int64_t(s) * G.sd; };
  // the job's bulk copies into buffer b (warp 0: lane 0 posts the bytes)
  auto issue_load = [&](int J, int b) {
    const int w = jobW(J);
    T* tile = tiles + b * TE;
    const int64_t g0 = gbase(J);
    const int ph0 = int(g0 & (V - 1));
    if constexpr (ROWS) {
      if (lane == 0) {
        const uint32_t by = uint32_t((ph0 + B * P + V - 1) / V * V * sizeof(T));
        ptx::mbar_arrive_expect_tx(&bar[b], by);
        ptx::bulk_g2s(tile, in + (g0 - ph0), by, &bar[b]);
      }
    } else {
      uint32_t mine = 0;
      for (int i = lane; i < B; i += 32) {
        const int phi = int((g0 + int64_t(i) * G.sd) & (V - 1));
        mine += uint32_t((phi + w + V - 1) / V * V * sizeof(T));
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
      if (lane == 0) ptx::mbar_arrive_expect_tx(&bar[b], mine);
      __syncwarp();
      for (int i = lane; i < B; i += 32) {
        const int64_t gi = g0 + int64_t(i) * G.sd;
        const int phi = int(gi & (V - 1));
        ptx::bulk_g2s(tile + (ph0 + i * P - phi), in + (gi - phi),
                      uint32_t((phi + w + V - 1) / V * V * sizeof(T)), &bar[b]);
      }
    }
  };

  ptx::pdl_wait();
  if (wp == 0)
    for (int b = 0; b < NBUF; ++b)
      if (cid + b * ncl < G.njobs) issue_load(cid + b * ncl, b);

  const bool full = B >= 32;
  int it = 0;
  for (int J = cid; J < G.njobs; J += ncl, ++it) {
    const int b = NBUF == 1 ? 0 : it % NBUF;
    const int w = jobW(J);
    const int64_t g0 = gbase(J);
    const int ph0 = int(g0 & (V - 1));
    T* tile = tiles + b * TE;
    const int par = it & 1;
    const T* rs = rsum + par * nslot * C::NCOL + tid;
    if (tid == 0 && nb > 1) ptx::mbar_arrive_expect_tx(&xbar[par], xbytes);
    ptx::mbar_wait(&bar[b], uint32_t((it / NBUF) & 1));

    // ---- ROWS: the tile's rows along dim 2 first (the dimension passes
    // commute; only rounding depends on the order), one warp per row, CHR per lane
    if constexpr (ROWS) {
      constexpr int KD = scan_depth<T, CHR>() < 31 ? scan_depth<T, CHR>() : 31;
      const int q0 = lane * CHR;
      const T* rtm = rt + lane * CHRP;
      const T* rtP = rtm + C::RNTB;
      const T* rtp = rtP + C::RNTB;
      const T* rtu = rtp + C::RNTB;
      const T* rtQ = rtu + C::RNTB;
      const T pend = rtP[CHR - 1], qfirst = rtQ[0];
      for (int r = wp; r < B; r += NW) {
        T* row = tile + ph0 + r * P + q0;
        T y[CHR];
#pragma unroll
        for (int k = 0; k < CHR; ++k) y[k] = q0 + k < P ? row[k] : T(0);
        T e = ChunkSolveV<T, CHR>::fwd_local(y, rtm);
        T c = T(0);
#pragma unroll
        for (int d = 0; d < KD; ++d) {
          const T t = __shfl_up_sync(0xffffffffu, e + pend * c, 1);
          c = lane == 0 ? T(0) : t;
        }
        ChunkSolveV<T, CHR>::apply(y, rtP, c);
        e = ChunkSolveV<T, CHR>::bwd_local(y, rtu, rtp);
        c = T(0);
#pragma unroll
        for (int d = 0; d < KD; ++d) {
          const T t = __shfl_down_sync(0xffffffffu, e + qfirst * c, 1);
          c = lane == 31 ? T(0) : t;
        }
        ChunkSolveV<T, CHR>::apply(y, rtQ, c);
#pragma unroll
        for (int k = 0; k < CHR; ++k)
          if (q0 + k < P) row[k] = y[k];
      }
      __syncthreads();
    }

    // ---- lines along the band dimension, one thread per column: local solve
    // in registers; the tile is then free for the job after next
    const bool act = tid < w;
    T x[kBandMax];
    T gend, h0;
    {
      const T* col = tile + ph0 + tid;
      if (full) band_local<T, P, true>(col, B, tm, tu, tp, x, gend, h0);
      else band_local<T, P, false>(col, B, tm, tu, tp, x, gend, h0);
    }
    ptx::fence_proxy_async_smem();  // generic smem traffic before the TMA refill
    __syncthreads();
    {
      const int Jn = J + NBUF * ncl;
      if (wp == 0 && Jn < G.njobs) issue_load(Jn, b);
    }
    // carries from the neighbouring bands' summaries (pushed, not polled)
    T cf = T(0), cb = T(0);
    if (nb > 1) {
      const uint32_t slot_bytes = uint32_t(C::NCOL * sizeof(T));
      const uint32_t mine = uint32_t((par * nslot * C::NCOL + tid) * sizeof(T));
#pragma unroll
      for (int t = 1; t <= kKBMax; ++t) {
        if (t > kb) break;
        if (j + t < nb) {  // receiver after this band: g_end(j) in its slot kb - t
          const uint32_t r = uint32_t(j + t);
          ptx::st_async1(ptx::mapa(rs_base + mine + uint32_t(kb - t) * slot_bytes, r), gend,
                         ptx::mapa(xb_base + uint32_t(par) * 8, r));
        }
        if (j - t >= 0) {  // receiver before: g_end(j) (t < kb), hg_0(j)
          const uint32_t r = uint32_t(j - t);
          const uint32_t rb = ptx::mapa(xb_base + uint32_t(par) * 8, r);
          if (t < kb)
            ptx::st_async1(ptx::mapa(rs_base + mine + uint32_t(kb + t - 1) * slot_bytes, r), gend, rb);
          ptx::st_async1(ptx::mapa(rs_base + mine + uint32_t(2 * kb - 2 + t) * slot_bytes, r), h0, rb);
        }
      }
      ptx::mbar_wait_cluster(&xbar[par], uint32_t((it >> 1) & 1));
#pragma unroll
      for (int t = kKBMax; t >= 1; --t) {  // bands j - t, oldest first
        if (t <= kb && j - t >= 0) cf = rs[(kb - t) * C::NCOL] + nPend[kKBMax - t] * cf;
      }
      T cfn[kKBMax];  // c_f of bands j + 1 .. j + kKBMax
      T prev = cf, pg = gend;
#pragma unroll
      for (int t = 1; t <= kKBMax; ++t) {
        T v = T(0);
        if (t <= kb && j + t < nb) {
          v = pg + nPend[kKBMax + t - 1] * prev;
          if (t < kb && j + t + 1 < nb) pg = rs[(kb + t - 1) * C::NCOL];
        }
        cfn[t - 1] = v;
        prev = v;
      }
#pragma unroll
      for (int t = kKBMax; t >= 1; --t) {
        if (t <= kb && j + t < nb)
          cb = rs[(2 * kb - 2 + t) * C::NCOL] + cfn[t - 1] * nhP0[kKBMax + t] + nQ0[kKBMax + t] * cb;
      }
    }
    // ---- results straight from registers: one coalesced row of columns per position
    if (act) {
      constexpr int N = VV::N;
      T* gcol = out + g0 + tid;
      const int64_t sd = ROWS ? int64_t(P) : G.sd;
#pragma unroll
      for (int i0 = 0; i0 < kBandMax; i0 += N) {
        T a[N], q[N];
        VV::split(reinterpret_cast<const VT*>(thP)[i0 / N], a);
        VV::split(reinterpret_cast<const VT*>(tQ)[i0 / N], q);
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const int i = i0 + k;
          if (i < kBandMax && (i < 32 ? (full || i < B) : i < B))
            gcol[i * sd] = x[i] + cf * a[k] + cb * q[k];
        }
      }
    }
  }
  ptx::cluster_arrive();  // no CTA leaves while its pushes into neighbours may be in flight
  ptx::cluster_wait();
}

// ---- host side --------------------------------------------------------------------

template <class T, bool ROWS, int NT, int P, int CHR, int NBUF, int MINB>
bool run_band(const T* in, T* out, const BandGeo& g, const T* mult, const T* rpiv, const T* upper,
              const T* rmult, const T* rrpiv, const T* rupper, int64_t level_nodes, cudaStream_t s) {
  using C = BandCfg<T, ROWS, NT, P, CHR, NBUF>;
  auto kern = k_thomas_band<T, ROWS, NT, P, CHR, NBUF, MINB>;
  const size_t smem = C::bytes(g.kb);
  if (smem > 227 * 1024) return false;
  set_smem_attr(reinterpret_cast<const void*>(kern), smem);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(g.nb);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_for(level_nodes) ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  // co-resident clusters of this shape (cached per kernel, size, device)
  struct Occ {
    const void* fn;
    int dev, nb, ncl;
    size_t smem;
  };
  static std::mutex mu;
  static std::vector<Occ> cache;
  int dev = 0;
  HGR_CUDA_CHECK(cudaGetDevice(&dev));
  int ncl = -1;
  {
    std::lock_guard<std::mutex> lock(mu);
    for (const auto& o : cache)
      if (o.fn == reinterpret_cast<const void*>(kern) && o.dev == dev && o.nb == g.nb && o.smem == smem)
        ncl = o.ncl;
    if (ncl < 0) {
      if (g.nb > 8)
        HGR_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(kern),
                                            cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      cfg.gridDim = dim3(unsigned(g.nb));
      int v = 0;
      if (cudaOccupancyMaxActiveClusters(&v, kern, &cfg) != cudaSuccess) {
        cudaGetLastError();
        v = 0;
      }
      ncl = v;
      cache.push_back(Occ{reinterpret_cast<const void*>(kern), dev, g.nb, ncl, smem});
    }
  }
  if (ncl <= 0) return false;
  const int clusters = g.njobs < ncl ? g.njobs : ncl;
  cfg.gridDim = dim3(unsigned(clusters * g.nb));
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, in, out, g, mult, rpiv, upper, rmult, rrpiv,
                                           rupper);
  if (e != cudaSuccess) launch_failed(e, reinterpret_cast<const void*>(kern), cfg.gridDim, cfg.blockDim, smem);
  return true;
}

template <class T>
BandGeo band_geo(int n) {
  BandGeo g{};
  g.n = n;
  g.nb = int((n + kBandMax - 1) / kBandMax);
  const int bmin = n / g.nb;
  const int kb = (damp_bits<T>() + bmin - 1) / bmin;
  g.kb = kb < g.nb - 1 ? kb : g.nb - 1;
  return g;
}

// fp32 513-wide planes: two single-buffered CTAs per SM (default; measured
// 1.79 vs 1.83 ms of IPK per 1025^3 round trip) or one double-buffered CTA
// (knob HGR_PLANES_2CTA=0)
inline bool planes_two_ctas() {
  static const bool v = [] {
    const char* e = std::getenv("HGR_PLANES_2CTA");
    return !e || e[0] != '0';
  }();
  return v;
}

// row lengths with a fused dims-1+2 kernel (compile-time tile pitch)
inline bool planes_row_ok(int64_t c2) {
  return c2 == 513 || c2 == 257 || c2 == 129 || c2 == 65 || c2 == 33 || c2 == 17;
}

}  // namespace

template <class T>
bool thomas_band_supported(const int64_t c[3]) {
  constexpr int V = vecn<T>();
  return c[0] >= 2 && c[1] >= 2 && planes_row_ok(c[2]) && c[0] <= kBandMax * kMaxBands &&
         c[1] <= kBandMax * kMaxBands && (c[1] * c[2]) % V == 1 % V &&
         c[0] * c[1] * c[2] < (int64_t(1) << 40);
}

template <class T>
bool launch_thomas_planes(T* src, T* dst, const int64_t c[3], const T* const mult[3],
                          const T* const rpiv[3], const T* const upper[3], int64_t level_nodes,
                          bool band_dim0, cudaStream_t s) {
  if (!thomas_band_supported<T>(c)) return false;
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) return false;
  constexpr bool F64 = sizeof(T) == 8;
  constexpr int V = vecn<T>();
  const int64_t plane = c[1] * c[2];
  // dim 0, in place on src: the register-tiled strided-line kernel, or jobs of
  // W0 contiguous plane columns (35 KB tiles, double-buffered, 3 CTAs per SM;
  // pitch P0 == plane (mod V))
  if (!band_dim0) {
    if (!launch_thomas_fast<T>(src, src, c, 0, mult[0], rpiv[0], upper[0], s)) return false;
  } else {
    constexpr int NT0 = F64 ? 128 : 256;
    constexpr int W0 = NT0 - V;  // a position's phased superset is <= 64 vectors
    constexpr int P0 = W0 + 2 * V + 1;
    BandGeo g = band_geo<T>(int(c[0]));
    g.W = W0;
    g.njobs = int((plane + W0 - 1) / W0);
    g.Wlast = int(plane - int64_t(g.njobs - 1) * W0);
    g.sd = plane;
    g.jstride = W0;
    if (!run_band<T, false, NT0, P0, 1, 2, 3>(src, src, g, mult[0], rpiv[0], upper[0], nullptr,
                                              nullptr, nullptr, level_nodes, s))
      return false;
  }
  // dims 1 + 2: one plane per job, src -> dst
  BandGeo g = band_geo<T>(int(c[1]));
  g.W = g.Wlast = int(c[2]);
  g.njobs = int(c[0]);
  g.sd = c[2];
  g.jstride = plane;
#define HGR_PLANES(NT, C2, CHR, NBUF, MINB)                                                       \
  run_band<T, true, NT, C2, CHR, NBUF, MINB>(src, dst, g, mult[1], rpiv[1], upper[1], mult[2],    \
                                             rpiv[2], upper[2], level_nodes, s)
  bool ok = false;
  switch (int(c[2])) {
    case 513:
      if constexpr (F64) ok = HGR_PLANES(544, 513, 17, 1, 1);
      else if (planes_two_ctas()) ok = HGR_PLANES(544, 513, 17, 1, 2);
      else ok = HGR_PLANES(544, 513, 17, 2, 1);
      break;
    case 257:
      if constexpr (F64) ok = HGR_PLANES(288, 257, 9, 2, 1);
      else ok = HGR_PLANES(288, 257, 9, 2, 2);
      break;
    case 129: ok = HGR_PLANES(160, 129, 5, 2, 2); break;
    case 65: ok = HGR_PLANES(96, 65, 3, 2, 2); break;
    case 33: ok = HGR_PLANES(64, 33, 2, 2, 2); break;
    case 17: ok = HGR_PLANES(64, 17, 1, 2, 2); break;
  }
#undef HGR_PLANES
  require(ok, "thomas planes: the dims-1+2 cluster kernel does not fit after the dim-0 pass ran");
  return true;
}

template bool thomas_band_supported<float>(const int64_t*);
template bool thomas_band_supported<double>(const int64_t*);
template bool launch_thomas_planes<float>(float*, float*, const int64_t*, const float* const*,
                                          const float* const*, const float* const*, int64_t, bool,
                                          cudaStream_t);
template bool launch_thomas_planes<double>(double*, double*, const int64_t*, const double* const*,
                                           const double* const*, const double* const*, int64_t,
                                           bool, cudaStream_t);

}  // namespace hgrb
