// mg_common.cuh — shared device-side definitions of the CUDA path.
//
// Internal data model (DESIGN.md §5 "data layout in HBM"): every level of
// every problem is stored as a dense array [planes][rows][pitch], x fastest.
//   3D: planes = z nodes, rows = y nodes, in-plane y neighbours at +-pitch,
//       plane neighbours at +-plane_stride.
//   2D: the paper's y axis is the PLANE axis (rows = 1, plane stride = pitch),
//       so the slowest axis is always the plane axis — slab decomposition,
//       plane marching and halo exchange are written once for both dims.
// The canonical per-point operation order (reading 13) is then
//   s = cx*(x-1 + x+1); [3D: s = s + cy*(y-1 + y+1)]; s = s + cz*(p-1 + p+1);
//   Au = D*u - s; r = f - Au
// with cz the coefficient of the plane axis (2D: the paper's c_y).  No FMA:
// every product and sum is an explicitly rounded intrinsic.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mg {

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
// nsum + r^2 in FP64.  r from FP32 arithmetic: r^2 is exact in double, so one FMA is bitwise
// the rounded add of the exact product; FP64 r keeps the two roundings (dmul, dadd).
template <typename T>
__device__ __forceinline__ double acc_sq(double nsum, T r) {
  const double d = (double)r;
  if constexpr (sizeof(T) == 4) return __fma_rn(d, d, nsum);
  else return __dadd_rn(nsum, __dmul_rn(d, d));
}
// ... where r is already the double of a value of the kernel's type T
template <typename T>
__device__ __forceinline__ double acc_sq_d(double nsum, double r) {
  if constexpr (sizeof(T) == 4) return __fma_rn(r, r, nsum);
  else return __dadd_rn(nsum, __dmul_rn(r, r));
}
// c ? a : b as one selp: both operands are computed, no branch around an expensive a
__device__ __forceinline__ float selv(bool c, float a, float b) {
  float r;
  asm("{.reg .pred p; setp.ne.u32 p, %3, 0; selp.f32 %0, %1, %2, p;}" : "=f"(r) : "f"(a), "f"(b), "r"((unsigned)c));
  return r;
}
__device__ __forceinline__ double selv(bool c, double a, double b) {
  double r;
  asm("{.reg .pred p; setp.ne.u32 p, %3, 0; selp.f64 %0, %1, %2, p;}" : "=d"(r) : "d"(a), "d"(b), "r"((unsigned)c));
  return r;
}

// Geometry of one level on this rank.
struct Geom {
  int three_d;        // 1: in-plane y neighbours exist (3D problem)
  int nx;             // cells along x (nodes 0..nx)
  int ny;             // cells along in-plane y (3D); 0 in 2D
  int nz;             // GLOBAL cells along the plane axis (3D z, 2D y)
  int rows;           // rows per plane in memory (3D: ny+1, 2D: 1)
  int p_lo, p_hi;     // local planes holding interior nodes to update: [p_lo, p_hi)
  int p_glob0;        // global plane index of local plane 0
  int planes;         // local planes in memory (incl. halo planes of a slab)
  long long pitch;    // elements between rows
  long long pstride;  // elements between planes
};

template <typename T>
struct Coef {
  T cx, cy, cz;  // c_d = a_d / h_{l,d}^2 (cz: plane axis)
  T D;           // 2 * sum c_d
  T wd;          // omega / D
};

// f - A u at linear index p (u interior node), canonical order.
template <typename T>
__device__ __forceinline__ T point_residual(const T* __restrict__ u, long long p, const Geom& g,
                                            const Coef<T>& c, T fp) {
  T s = mul(c.cx, add(u[p - 1], u[p + 1]));
  if (g.three_d) s = add(s, mul(c.cy, add(u[p - g.pitch], u[p + g.pitch])));
  s = add(s, mul(c.cz, add(u[p - g.pstride], u[p + g.pstride])));
  T Au = sub(mul(c.D, u[p]), s);
  return sub(fp, Au);
}

}  // namespace mg
