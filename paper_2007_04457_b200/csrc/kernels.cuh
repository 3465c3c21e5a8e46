// kernels.cuh -- launcher declarations for the sm_100a kernels.
#pragma once

#include "common.cuh"

namespace hgrb {

// ---- device helpers ---------------------------------------------------------

// Multilinear interpolation of the coarse neighbours of level-l node (i0,i1,i2)
// (transforms.hpp:20-65). Corner and weight order follow the reference: the
// corner bit of the lowest odd dimension varies fastest and the weight product
// is accumulated over odd dimensions in ascending order.
template <class T, class Coarse>
__device__ __forceinline__ T interp_node(const LevelArgs<T>& a, int64_t i0, int64_t i1,
                                         int64_t i2, const Coarse& coarse) {
  const bool o0 = i0 & 1, o1 = i1 & 1, o2 = i2 & 1;
  const int64_t b0 = i0 >> 1, b1 = i1 >> 1, b2 = i2 >> 1;
  T w0[2] = {T(1), T(0)}, w1[2] = {T(1), T(0)}, w2[2] = {T(1), T(0)};
  if (o0) { w0[0] = a.wl[0][b0]; w0[1] = a.wr[0][b0]; }
  if (o1) { w1[0] = a.wl[1][b1]; w1[1] = a.wr[1][b1]; }
  if (o2) { w2[0] = a.wl[2][b2]; w2[1] = a.wr[2][b2]; }
  T acc = T(0);
#pragma unroll
  for (int k2 = 0; k2 < 2; ++k2) {
    if (k2 && !o2) break;
#pragma unroll
    for (int k1 = 0; k1 < 2; ++k1) {
      if (k1 && !o1) break;
#pragma unroll
      for (int k0 = 0; k0 < 2; ++k0) {
        if (k0 && !o0) break;
        T w = T(1);
        if (o0) w *= w0[k0];
        if (o1) w *= w1[k1];
        if (o2) w *= w2[k2];
        acc += w * coarse(b0 + k0, b1 + k1, b2 + k2);
      }
    }
  }
  return acc;
}

// The lane's NCELL consecutive coefficients into global memory whose first
// element has phase P (elements mod 16 bytes): the widest aligned vector
// stores instead of one store per cell.
template <class T, int NCELL, int P>
__device__ __forceinline__ void store_cells(T* o, const T (&cv)[NCELL]) {
  if constexpr (sizeof(T) == 4) {
    static_assert(NCELL == 4, "fp32 lanes own four cells");
    if constexpr (P == 0) {
      *reinterpret_cast<float4*>(o) = make_float4(cv[0], cv[1], cv[2], cv[3]);
    } else if constexpr (P == 2) {
      *reinterpret_cast<float2*>(o) = make_float2(cv[0], cv[1]);
      *reinterpret_cast<float2*>(o + 2) = make_float2(cv[2], cv[3]);
    } else if constexpr (P == 1) {
      o[0] = cv[0];
      *reinterpret_cast<float2*>(o + 1) = make_float2(cv[1], cv[2]);
      o[3] = cv[3];
    } else {
      o[0] = cv[0];
      *reinterpret_cast<float2*>(o + 1) = make_float2(cv[1], cv[2]);
      o[3] = cv[3];
    }
  } else {
    static_assert(NCELL == 2, "fp64 lanes own two cells");
    if constexpr (P == 0) {
      *reinterpret_cast<double2*>(o) = make_double2(cv[0], cv[1]);
    } else {
      o[0] = cv[0];
      o[1] = cv[1];
    }
  }
}


// ---- launchers (all stream-ordered) -----------------------------------------

// GPK, decompose direction (refactor.hpp:43-47): in place on the compact level-l
// array U: refined nodes -= interp; coarse nodes are gathered into the compact
// level-(l-1) array C. Sets *flag if check_finite and a non-finite value is seen.
template <class T>
void launch_gpk_dec(T* U, T* C, const LevelArgs<T>& a, int* flag, bool check_finite,
                    cudaStream_t s);

// GPK, recompose direction (refactor.hpp:77-87): coarse value = C - Z (Z may be
// null); out[coarse] = coarse value, out[refined] = (with ? coef : 0) + interp.
template <class T>
void launch_gpk_rec(const T* coef, T* out, const T* C, const T* Z, const LevelArgs<T>& a,
                    bool with_coeffs, cudaStream_t s);

// LPK pass along dim (masstrans_pass, correction.hpp:238-260), compact in -> compact out.
template <class T>
void launch_lpk(const T* in, const int64_t in_ext[3], T* out, int dim, int64_t cd,
                const T* taps, bool mask, cudaStream_t s);

// IPK pass along dim (thomas_pass, correction.hpp:262-278) on compact z. If
// apply != null, apply[i] += sign * x[i] and z is not written back.
template <class T>
void launch_thomas(T* z, const int64_t ext[3], int dim, const T* mult, const T* rpiv,
                   const T* upper, T* apply, int sign, cudaStream_t s);

// y[i] += sign * x[i], i < n
template <class T>
void launch_axpy(T* y, const T* x, int64_t n, int sign, cudaStream_t s);

// dst[q] = src[q * stride] (3D), dst extents given.
template <class T>
void launch_gather(const T* src, const int64_t src_ext[3], int64_t stride, T* dst,
                   const int64_t dst_ext[3], cudaStream_t s);

// level-l array even positions <- compact level-(l-1) array (pyramid assembly).
template <class T>
void launch_scatter_even(const T* src, T* dst, const LevelArgs<T>& a, cudaStream_t s);

// compute_coefficients (transforms.hpp:96-111), compact -> compact.
template <class T>
void launch_coefficients(const T* fine, T* coeffs, const LevelArgs<T>& a, cudaStream_t s);

// interpolate_to_fine (transforms.hpp:76-92), compact coarse -> compact fine.
template <class T>
void launch_interpolate(const T* coarse, T* fine, const LevelArgs<T>& a, cudaStream_t s);

// *flag = 1 if any coarse-aligned entry of the level-l array is nonzero
// (correction.hpp:354-360).
template <class T>
void launch_check_coarse_zero(const T* coeffs, const LevelArgs<T>& a, int* flag, cudaStream_t s);

// extract_class / scatter_class (refactor.hpp:134-170) on the finest array.
template <class T>
void launch_class_copy(T* data, const int64_t finest_ext[3], int64_t stride,
                       const int64_t cls_ext[3], bool cls0, T* vals, bool extract,
                       cudaStream_t s);

// *flag = 1 if any of the n values is NaN/Inf (refactor.hpp:36-38)
template <class T>
void check_finite(const T* v, int64_t n, int* flag, cudaStream_t s);

// fiber operators (correction.hpp:43-88, 141-154, 202-208), batched
template <class T>
void launch_fiber_mass(const T* v, T* out, int64_t n, int64_t count, const T* h, cudaStream_t s);
template <class T>
void launch_fiber_masstrans(const T* v, T* out, int64_t n, int64_t count, const T* taps,
                            bool zero_even, cudaStream_t s);
template <class T>
void launch_fiber_transfer(const T* v, T* out, int64_t n, int64_t count, const T* trl,
                           const T* trr, cudaStream_t s);
template <class T>
void launch_fiber_thomas(const T* v, T* out, int64_t n, int64_t count, const T* mult,
                         const T* rpiv, const T* upper, cudaStream_t s);

}  // namespace hgrb
