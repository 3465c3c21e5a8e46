// thomas_chunk.cuh -- chunked-affine Thomas building blocks shared by the IPK
// kernels (kernels_thomas.cu, kernels_band.cu): line-independent carry tables,
// register-chunk forward / backward solves with zero carry, carry application,
// and the carry-scan depth from the damping bound.
#pragma once

#include <cuda_runtime.h>

namespace hgrb {
namespace thomas {

// Line-independent tables for NC chunks of CH positions over a line of n:
//   tm[i] = m_{i-1} (0 at i = 0 and i >= n), tp[i] = 1/p_i, tu[i] = u_i (0 at
//   i >= n-1), P (forward carry products), Q (backward carry products);
//   positions >= n have tp = 0 so padding never feeds back.
//   With a window start ws the tables cover line positions ws .. ws+NP-1
//   (positions outside the line are padding).
template <class T>
__device__ void build_tables(T* tm, T* tP, T* tp, T* tu, T* tQ, int n, int NC, int CH, int CHP,
                             const T* mult, const T* rpiv, const T* upper, int ws = 0) {
  // chunk q's entries live at q*CHP .. q*CHP+CH-1 (CHP: CH rounded up to a
  // 16-byte multiple, so a chunk's table is read with vector loads); pad = 0
  for (int i = threadIdx.x; i < NC * CHP; i += blockDim.x) {
    const int q = i / CHP, k = i - q * CHP;
    const int pos = ws + q * CH + k;
    const bool in = k < CH;
    tm[i] = (in && pos >= 1 && pos < n) ? mult[pos - 1] : T(0);
    tp[i] = (in && pos >= 0 && pos < n) ? rpiv[pos] : T(0);
    tu[i] = (in && pos >= 0 && pos < n - 1) ? upper[pos] : T(0);
  }
  __syncthreads();
  for (int q = threadIdx.x; q < NC; q += blockDim.x) {
    const int s = q * CHP;
    T a = T(1);
    for (int k = 0; k < CH; ++k) {
      a *= -tm[s + k];
      tP[s + k] = a;
    }
    T b = T(1);
    for (int k = CH - 1; k >= 0; --k) {
      b *= -(tu[s + k] * tp[s + k]);
      tQ[s + k] = b;
    }
    for (int k = CH; k < CHP; ++k) tP[s + k] = tQ[s + k] = T(0);
  }
  __syncthreads();
}

// table stride of a chunk of CH positions: CH rounded up to 16 bytes
template <class T, int CH>
constexpr int chunk_pitch() {
  return (CH + int(16 / sizeof(T)) - 1) / int(16 / sizeof(T)) * int(16 / sizeof(T));
}

// 16-byte vector of T
template <class T>
struct Vec16;
template <>
struct Vec16<float> {
  using type = float4;
  static constexpr int N = 4;
  static __device__ __forceinline__ void split(const float4& v, float (&o)[4]) {
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  }
};
template <>
struct Vec16<double> {
  using type = double2;
  static constexpr int N = 2;
  static __device__ __forceinline__ void split(const double2& v, double (&o)[2]) {
    o[0] = v.x; o[1] = v.y;
  }
};

// Chunk solves reading the (16-byte aligned, chunk-pitched) tables with vector
// loads: one shared-memory load per 16 bytes of table instead of per entry.
template <class T, int CH, int LPT = 1>
struct ChunkSolveV {
  using V = Vec16<T>;
  static constexpr int N = V::N;
  static __device__ __forceinline__ void fwd_local(T (&x)[LPT][CH], const T* tm, T (&g)[LPT]) {
#pragma unroll
    for (int u = 0; u < LPT; ++u) g[u] = T(0);
#pragma unroll
    for (int k0 = 0; k0 < CH; k0 += N) {
      T m[N];
      V::split(reinterpret_cast<const typename V::type*>(tm)[k0 / N], m);
#pragma unroll
      for (int j = 0; j < N; ++j) {
        if (k0 + j < CH) {
#pragma unroll
          for (int u = 0; u < LPT; ++u) {
            g[u] = x[u][k0 + j] - m[j] * g[u];
            x[u][k0 + j] = g[u];
          }
        }
      }
    }
  }
  static __device__ __forceinline__ void apply(T (&x)[LPT][CH], const T* tab, const T (&c)[LPT]) {
#pragma unroll
    for (int k0 = 0; k0 < CH; k0 += N) {
      T t[N];
      V::split(reinterpret_cast<const typename V::type*>(tab)[k0 / N], t);
#pragma unroll
      for (int j = 0; j < N; ++j)
        if (k0 + j < CH) {
#pragma unroll
          for (int u = 0; u < LPT; ++u) x[u][k0 + j] += t[j] * c[u];
        }
    }
  }
  static __device__ __forceinline__ void bwd_local(T (&x)[LPT][CH], const T* tu, const T* tp,
                                                   T (&h)[LPT]) {
#pragma unroll
    for (int u = 0; u < LPT; ++u) h[u] = T(0);
    constexpr int K0 = (CH - 1) / N * N;
#pragma unroll
    for (int k0 = K0; k0 >= 0; k0 -= N) {
      T uu[N], pp[N];
      V::split(reinterpret_cast<const typename V::type*>(tu)[k0 / N], uu);
      V::split(reinterpret_cast<const typename V::type*>(tp)[k0 / N], pp);
#pragma unroll
      for (int j = N - 1; j >= 0; --j) {
        if (k0 + j < CH) {
#pragma unroll
          for (int u = 0; u < LPT; ++u) {
            h[u] = (x[u][k0 + j] - uu[j] * h[u]) * pp[j];
            x[u][k0 + j] = h[u];
          }
        }
      }
    }
  }
  // single-line forms
  static __device__ __forceinline__ T fwd_local(T (&x)[CH], const T* tm) {
    T (&xx)[1][CH] = *reinterpret_cast<T(*)[1][CH]>(&x);
    T g[1];
    ChunkSolveV<T, CH, 1>::fwd_local(xx, tm, g);
    return g[0];
  }
  static __device__ __forceinline__ void apply(T (&x)[CH], const T* tab, T c) {
    T (&xx)[1][CH] = *reinterpret_cast<T(*)[1][CH]>(&x);
    const T cc[1] = {c};
    ChunkSolveV<T, CH, 1>::apply(xx, tab, cc);
  }
  static __device__ __forceinline__ T bwd_local(T (&x)[CH], const T* tu, const T* tp) {
    T (&xx)[1][CH] = *reinterpret_cast<T(*)[1][CH]>(&x);
    T h[1];
    ChunkSolveV<T, CH, 1>::bwd_local(xx, tu, tp, h);
    return h[0];
  }
};

// chunk solves of LPT lines at once (the line-independent table values are
// loaded once for all of them)
template <class T, int CH, int LPT = 1>
struct ChunkSolve {
  // forward local (zero carry) in place; g[u] = the chunk's last value of line u
  static __device__ __forceinline__ void fwd_local(T (&x)[LPT][CH], const T* tm, T (&g)[LPT]) {
#pragma unroll
    for (int u = 0; u < LPT; ++u) g[u] = T(0);
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const T m = tm[k];
#pragma unroll
      for (int u = 0; u < LPT; ++u) {
        g[u] = x[u][k] - m * g[u];
        x[u][k] = g[u];
      }
    }
  }
  static __device__ __forceinline__ void apply(T (&x)[LPT][CH], const T* tab, const T (&c)[LPT]) {
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const T t = tab[k];
#pragma unroll
      for (int u = 0; u < LPT; ++u) x[u][k] += t * c[u];
    }
  }
  // backward local (zero carry) in place; h[u] = the chunk's first value of line u
  static __device__ __forceinline__ void bwd_local(T (&x)[LPT][CH], const T* tu, const T* tp,
                                                   T (&h)[LPT]) {
#pragma unroll
    for (int u = 0; u < LPT; ++u) h[u] = T(0);
#pragma unroll
    for (int k = CH - 1; k >= 0; --k) {
      const T uu = tu[k], pp = tp[k];
#pragma unroll
      for (int u = 0; u < LPT; ++u) {
        h[u] = (x[u][k] - uu * h[u]) * pp;
        x[u][k] = h[u];
      }
    }
  }
  // single-line convenience forms
  static __device__ __forceinline__ T fwd_local(T (&x)[CH], const T* tm) {
    T g = T(0);
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      g = x[k] - tm[k] * g;
      x[k] = g;
    }
    return g;
  }
  static __device__ __forceinline__ void apply(T (&x)[CH], const T* tab, T c) {
#pragma unroll
    for (int k = 0; k < CH; ++k) x[k] += tab[k] * c;
  }
  static __device__ __forceinline__ T bwd_local(T (&x)[CH], const T* tu, const T* tp) {
    T h = T(0);
#pragma unroll
    for (int k = CH - 1; k >= 0; --k) {
      h = (x[k] - tu[k] * h) * tp[k];
      x[k] = h;
    }
    return h;
  }
};

// Carry-scan depth: every forward multiplier m_i = h_i / p_i and backward
// factor u_i / p_i is at most 1/2 (p_i >= 2 h_i + 1.5 h_{i-1}, the first is 1/2),
// so a chunk of CH positions scales the carry through it by at most 2^-CH.
// Chunks further than KD chunks away contribute below 2^-B (B = 56 for fp64, 26
// for fp32) of their summaries and the scan stops there.
template <class T, int CH>
constexpr int scan_depth() {
  return ((sizeof(T) == 8 ? 56 : 26) + CH - 1) / CH + 1;
}

// Overlap (positions) of windowed solves: a carry dropped H positions away is
// damped below 2^-H relative (the bound above).
template <class T>
constexpr int window_halo() {
  return sizeof(T) == 8 ? 56 : 26;
}

}  // namespace thomas
}  // namespace hgrb
