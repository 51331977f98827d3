// vec.cuh — 16-byte vectors of W = 16/sizeof(T) consecutive x nodes (FP64: 2, FP32: 4).
#pragma once
#include <cuda_runtime.h>

namespace mg {

template <typename T, int W>
struct Vec {
  T v[W];
};

template <typename T>
__device__ __forceinline__ Vec<T, 16 / sizeof(T)> ld_vec(const T* p) {
  Vec<T, 16 / sizeof(T)> r;
  if constexpr (sizeof(T) == 8) {
    const double2 a = *reinterpret_cast<const double2*>(p);
    r.v[0] = a.x;
    r.v[1] = a.y;
  } else {
    const float4 a = *reinterpret_cast<const float4*>(p);
    r.v[0] = a.x;
    r.v[1] = a.y;
    r.v[2] = a.z;
    r.v[3] = a.w;
  }
  return r;
}

// the same through the read-only (non-coherent) path: only for data no thread of the
// kernel writes
template <typename T>
__device__ __forceinline__ Vec<T, 16 / sizeof(T)> ld_vec_nc(const T* p) {
  Vec<T, 16 / sizeof(T)> r;
  if constexpr (sizeof(T) == 8) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    r.v[0] = a.x;
    r.v[1] = a.y;
  } else {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    r.v[0] = a.x;
    r.v[1] = a.y;
    r.v[2] = a.z;
    r.v[3] = a.w;
  }
  return r;
}

// store the whole vector at p (16-byte aligned)
template <typename T>
__device__ __forceinline__ void st_vec(T* p, const Vec<T, 16 / sizeof(T)>& o) {
  if constexpr (sizeof(T) == 8)
    *reinterpret_cast<double2*>(p) = make_double2(o.v[0], o.v[1]);
  else
    *reinterpret_cast<float4*>(p) = make_float4(o.v[0], o.v[1], o.v[2], o.v[3]);
}

// store the vector at dst[x..x+W), element k only if ok[k]
template <typename T>
__device__ __forceinline__ void store_vec(T* dst, int x, const bool* ok, const Vec<T, 16 / sizeof(T)>& o) {
  constexpr int W = 16 / sizeof(T);
  bool all = true;
#pragma unroll
  for (int k = 0; k < W; k++) all = all && ok[k];
  if (all) {
    if constexpr (sizeof(T) == 8) {
      *reinterpret_cast<double2*>(dst + x) = make_double2(o.v[0], o.v[1]);
    } else {
      *reinterpret_cast<float4*>(dst + x) = make_float4(o.v[0], o.v[1], o.v[2], o.v[3]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < W; k++)
      if (ok[k]) dst[x + k] = o.v[k];
  }
}

// the same with the W flags as the low bits of `ok`
template <typename T>
__device__ __forceinline__ void store_vec_m(T* dst, int x, uint32_t ok, const Vec<T, 16 / sizeof(T)>& o) {
  constexpr int W = 16 / sizeof(T);
  if (ok == (1u << W) - 1u) {
    st_vec(dst + x, o);
  } else {
#pragma unroll
    for (int k = 0; k < W; k++)
      if ((ok >> k) & 1u) dst[x + k] = o.v[k];
  }
}

}  // namespace mg
