// cd_common.cuh — complex arithmetic of the complex-diffusion kernels in the canonical
// order of DESIGN.md reading 19 (every operation an explicitly rounded intrinsic).
#pragma once
#include "kernels_cd.h"

namespace mg {
namespace cdk {

__device__ __forceinline__ double dv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float dv(float a, float b) { return __fdiv_rn(a, b); }

template <typename T>
struct C2 {
  T re, im;
};

template <typename T>
__device__ __forceinline__ C2<T> ld(const T* a, long long q) {
  if constexpr (sizeof(T) == 8) {
    const double2 v = *reinterpret_cast<const double2*>(a + 2 * q);
    return {v.x, v.y};
  } else {
    const float2 v = *reinterpret_cast<const float2*>(a + 2 * q);
    return {v.x, v.y};
  }
}
template <typename T>
__device__ __forceinline__ void st(T* a, long long q, C2<T> v) {
  if constexpr (sizeof(T) == 8)
    *reinterpret_cast<double2*>(a + 2 * q) = make_double2(v.re, v.im);
  else
    *reinterpret_cast<float2*>(a + 2 * q) = make_float2(v.re, v.im);
}
template <typename T>
__device__ __forceinline__ C2<T> cmul(C2<T> a, C2<T> b) {
  return {sub(mul(a.re, b.re), mul(a.im, b.im)), add(mul(a.re, b.im), mul(a.im, b.re))};
}
template <typename T>
__device__ __forceinline__ C2<T> cdiv(C2<T> x, C2<T> y) {
  const T den = add(mul(y.re, y.re), mul(y.im, y.im));
  return {dv(add(mul(x.re, y.re), mul(x.im, y.im)), den), dv(sub(mul(x.im, y.re), mul(x.re, y.im)), den)};
}
// Eq. 3 at s = Im u
template <typename T>
__device__ __forceinline__ C2<T> diffusivity(const CdCoef<T>& c, T s) {
  const T q = dv(s, c.kth);
  const T den = add((T)1, mul(q, q));
  return {dv(c.ct, den), dv(c.st, den)};
}

}  // namespace cdk
}  // namespace mg
