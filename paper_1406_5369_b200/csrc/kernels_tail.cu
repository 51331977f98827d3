// kernels_tail.cu — the coarse tail of the V-cycle in ONE launch.
//
// Levels below a size threshold are pure latency (each op-by-op pass is a few
// microseconds of launch and barrier for a few thousand nodes).  k_tail runs
// V_lt(0, f_lt) — every operation of Alg. 1 on levels lt..L-1:
// pre-smoothing, residual + full weighting, the coarsest solve, prolongation +
// correction, post-smoothing — inside ONE thread-block cluster (16 CTAs x 512
// threads, one per SM), a cluster barrier (barrier.cluster release/acquire)
// between passes, data in global memory (L2 resident).  Levels of at most a few
// thousand nodes run on CTA 0 alone with block barriers ("solo"), their arrays
// held in CTA 0's shared memory when they fit (a pass is then a few hundred
// cycles: no L2 round trip).  With lt = 0 (small 2D grids such as C1) the whole
// cycle is one launch on one CTA, the level-0 arrays copied in and u copied out.
// Work of a pass is distributed by rows: a warp takes a row of the level (one
// integer division per row, none per node) and its lanes the row's nodes (every
// other node for a red-black colour).  The per-node arithmetic is the same
// canonical device code as every other kernel (mg_common.cuh), so results are
// bitwise identical to the op-by-op schedule.
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "kernels.h"
#include "kernels_tail.h"
#include "launch_util.h"

namespace mg {

namespace {

constexpr int NTT = 512;  // measured: 512 beats 1024 (C1 63.6 -> 59.3 us, C2, C4) and 256
constexpr int WPC = NTT / 32;  // warps per CTA

// all CTAs of the cluster (= the grid): release/acquire at cluster scope makes the
// pass's global writes visible to the next pass (and invalidates L1)
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Work distribution of a pass.  A SOLO level runs on CTA 0 alone with block barriers — a block
// barrier costs a fraction of a cluster barrier and the level's work is too small to pay for 16
// SMs; the other CTAs skip solo passes entirely and meet CTA 0 at the next cluster barrier (the
// transitions in k_tail).  A DIST level is split into slabs of planes, one per CTA, each held
// with a halo plane on either side in that CTA's shared memory (LG::p_lo..p_hi are the CTA's own
// planes): the CTA's warps take its own rows, writes to its first/last plane are mirrored into
// the neighbours' halos through distributed shared memory (Mir), a cluster barrier between passes.
struct Mode {
  bool solo;
  bool dist = false;
  __device__ bool active() const { return !solo || blockIdx.x == 0; }
  __device__ bool local() const { return solo || dist; }
  __device__ int wstart() const {
    return local() ? (int)(threadIdx.x >> 5) : (int)(blockIdx.x * WPC + (threadIdx.x >> 5));
  }
  __device__ int wstride() const { return local() ? WPC : (int)(gridDim.x * WPC); }
  __device__ int start() const { return local() ? (int)threadIdx.x : (int)(blockIdx.x * NTT + threadIdx.x); }
  __device__ int stride() const { return local() ? NTT : (int)(gridDim.x * NTT); }
  __device__ void sync() const {
    if (!solo)
      cluster_sync();
    else if (blockIdx.x == 0)
      __syncthreads();
  }
};

// A level's geometry in registers (32-bit strides: tail levels are small).  Every pass copies
// it out of the kernel parameters once, so the node loops index with plain integer adds.
struct LG {
  int nx, ny, p_lo, p_hi, pg0, sy, sz, planes, rows;
  int shA, shC;  // log2 of the lane group of for_rows: all nodes / one colour of a row
  float inv_nr;  // 1 / rows per plane
  int zoff;      // plane of the array's first stored plane (a dist slab's lower halo; else 0)
};
__device__ __forceinline__ int ceil_log2_32(int v) { return v >= 32 ? 5 : (v <= 1 ? 0 : 32 - __clz(v - 1)); }
__device__ __forceinline__ LG lg_of(const Geom& g) {
  const int ni = g.nx - 1, nr = g.three_d ? g.ny - 1 : 1;
  return LG{g.nx, g.ny, g.p_lo, g.p_hi, g.p_glob0, (int)g.pitch, (int)g.pstride, g.planes, g.rows,
            ceil_log2_32(ni), ceil_log2_32((ni + 1) >> 1), __frcp_rn((float)nr), 0};
}
__device__ __forceinline__ int lin(const LG& g, int i, int j, int pl) { return (pl - g.zoff) * g.sz + j * g.sy + i; }

// A dist level's mirrors: after a pass, the CTA's first (last) own plane of the array it wrote
// is copied whole into the lower (upper) halo of the CTAs whose slab window holds that plane —
// the neighbour, and past it neighbours with empty slabs — through distributed shared memory
// (rem: remote bases shifted to this CTA's local indexing), 16-byte stores by every thread after
// a block barrier; the pass's cluster barrier then publishes them.  (Mirroring each node as it
// was written cost more than the pass: measured 20% more instructions.)
template <typename T>
struct Mir {  // plain data (a __shared__ table): set every field through none()
  int plo, phi, nlo, nhi;
  int sz, zoff;
  T* a[3];            // the local u, t, r arrays (the mirrored ones)
  T* rem[2][3][3];    // [side][target][array]
  __device__ static Mir none() {
    Mir m;
    m.plo = m.phi = -1;
    m.nlo = m.nhi = m.sz = m.zoff = 0;
    m.a[0] = m.a[1] = m.a[2] = nullptr;
    return m;
  }
  __device__ __forceinline__ void push(const T* arr) const {
    if (nlo + nhi == 0) return;  // uniform over the CTA (shared-memory table)
    __syncthreads();
    const int ai = arr == a[0] ? 0 : (arr == a[1] ? 1 : 2);
    const bool v16 = ((long long)sz * (long long)sizeof(T)) % 16 == 0;
    for (int side = 0; side < 2; side++) {
      const int n = side ? nhi : nlo;
      if (n == 0) continue;
      const long long o = (long long)((side ? phi : plo) - zoff) * sz;
      for (int t = 0; t < n; t++) {
        T* dst = rem[side][t][ai] + o;
        const T* src = arr + o;
        if (v16) {
          const int nv = sz * (int)sizeof(T) / 16;
          for (int q = threadIdx.x; q < nv; q += NTT)
            reinterpret_cast<uint4*>(dst)[q] = reinterpret_cast<const uint4*>(src)[q];
        } else {
          for (int q = threadIdx.x; q < sz; q += NTT) dst[q] = src[q];
        }
      }
    }
  }
};

// f - A u at p, canonical order (mg_common.cuh point_residual), DIM known at compile time
template <typename T, int DIM>
__device__ __forceinline__ T pres(const T* u, int p, const LG& g, const Coef<T>& c, T fp) {
  T s = mul(c.cx, add(u[p - 1], u[p + 1]));
  if (DIM == 3) s = add(s, mul(c.cy, add(u[p - g.sy], u[p + g.sy])));
  s = add(s, mul(c.cz, add(u[p - g.sz], u[p + g.sz])));
  return sub(fp, sub(mul(c.D, u[p]), s));
}

// f(i, j, plane, linear index) for the interior nodes of g; par >= 0: only the nodes with
// (i + j + global plane) & 1 == par (a red-black colour).  A warp takes 32/G rows at a time, a
// group of G lanes (G = the power of two >= the nodes to visit per row, at most 32) one row,
// so short rows of small levels do not idle most of the lanes.  Row -> (plane, y) by one
// float multiply: exact for the tail's levels (rows < 2^13, quotient error << 1/(2 nr)).
template <int DIM, class F>
__device__ __forceinline__ void for_rows(const Mode& M, const LG& g, int par, F&& f) {
  if (!M.active()) return;
  const int lane = threadIdx.x & 31;
  const int ni = g.nx - 1;
  const int nr = DIM == 3 ? g.ny - 1 : 1;
  const int nrows = nr * (g.p_hi - g.p_lo);
  const int sh = par < 0 ? g.shA : g.shC;
  const int G = 1 << sh, rpw = 32 >> sh;
  const int sub_ = lane & (G - 1);
  const float inv_nr = g.inv_nr;
  for (int rb = M.wstart() * rpw; rb < nrows; rb += M.wstride() * rpw) {
    const int row = rb + (lane >> sh);
    if (row >= nrows) continue;
    const int dp = DIM == 3 ? __float2int_rz(((float)row + 0.5f) * inv_nr) : row;
    const int pl = g.p_lo + dp;
    const int j = DIM == 3 ? 1 + row - dp * nr : 0;
    const int base = (pl - g.zoff) * g.sz + j * g.sy;
    if (par < 0) {
      for (int i = 1 + sub_; i <= ni; i += G) f(i, j, pl, base + i);
    } else {
      const int i0 = 1 + ((1 + j + pl + g.pg0 + par) & 1);  // first i of the colour
      for (int i = i0 + 2 * sub_; i <= ni; i += 2 * G) f(i, j, pl, base + i);
    }
  }
}

template <typename T>
__device__ void zero_level(const Mode& M, const LG& g, T* u) {
  if (!M.active()) return;
  const int n = g.planes * g.sz;
  for (int q = M.start(); q < n; q += M.stride()) u[q] = (T)0;
}

// one sweep of the smoother; Jacobi ping-pongs (returns the new current buffer)
template <typename T, int DIM>
__device__ T* sweep(const Mode& M, const LG& g, const Coef<T>& c, int rbgs, T* u, T* t, const T* f, const Mir<T>& mi) {
  const bool act = M.active();
  if (rbgs == 2) {  // lexicographic omega-GS: hyperplanes i + j + global plane = s in order
    const int nj = DIM == 3 ? g.ny - 1 : 1;
    const int m = nj * (g.p_hi - g.p_lo);
    const int smin = 1 + (DIM == 3 ? 1 : 0) + g.p_lo + g.pg0;
    const int smax = (g.nx - 1) + (DIM == 3 ? g.ny - 1 : 0) + g.p_hi - 1 + g.pg0;
    for (int s = smin; s <= smax; s++) {
      for (int q = act ? M.start() : m; q < m; q += M.stride()) {
        const int j = DIM == 3 ? 1 + q % nj : 0;
        const int pl = g.p_lo + q / nj;
        const int i = s - j - (pl + g.pg0);
        if (i < 1 || i > g.nx - 1) continue;
        const int p = lin(g, i, j, pl);
        u[p] = add(u[p], mul(c.wd, pres<T, DIM>(u, p, g, c, f[p])));
      }
      M.sync();
    }
    return u;
  }
  if (rbgs) {
    for (int colour = 0; colour < 2; colour++) {
      for_rows<DIM>(M, g, colour,
                    [&](int, int, int, int p) { u[p] = add(u[p], mul(c.wd, pres<T, DIM>(u, p, g, c, f[p]))); });
      mi.push(u);
      M.sync();
    }
    return u;
  }
  for_rows<DIM>(M, g, -1, [&](int, int, int, int p) { t[p] = add(u[p], mul(c.wd, pres<T, DIM>(u, p, g, c, f[p]))); });
  mi.push(t);
  M.sync();
  return t;
}

template <typename T, int DIM>
__device__ void residual(const Mode& M, const LG& g, const Coef<T>& c, const T* u, const T* f, T* r, const Mir<T>& mi) {
  for_rows<DIM>(M, g, -1, [&](int, int, int, int p) { r[p] = pres<T, DIM>(u, p, g, c, f[p]); });
  mi.push(r);
  M.sync();
}

// full weighting, separable x -> y -> plane axis (reading 13)
template <typename T, int DIM>
__device__ void restrict_fw(const Mode& M, const LG& gf, const LG& gc, const T* r, T* fc) {
  const T two = (T)2;
  const T scale = DIM == 3 ? (T)(1.0 / 64.0) : (T)(1.0 / 16.0);
  for_rows<DIM>(M, gc, -1, [&](int I, int J, int PL, int pc) {
    const int pf = 2 * (PL + gc.pg0) - gf.pg0;
    T tz[3];
#pragma unroll
    for (int dz = -1; dz <= 1; dz++) {
      T ty;
      if (DIM == 3) {
        T tx[3];
#pragma unroll
        for (int dy = -1; dy <= 1; dy++) {
          const int p = lin(gf, 2 * I, 2 * J + dy, pf + dz);
          tx[dy + 1] = add(add(r[p - 1], r[p + 1]), mul(two, r[p]));
        }
        ty = add(add(tx[0], tx[2]), mul(two, tx[1]));
      } else {
        const int p = lin(gf, 2 * I, 0, pf + dz);
        ty = add(add(r[p - 1], r[p + 1]), mul(two, r[p]));
      }
      tz[dz + 1] = ty;
    }
    fc[pc] = mul(add(add(tz[0], tz[2]), mul(two, tz[1])), scale);
  });
  M.sync();
}

// the first sweep from a zero iterate (V_H(0, ...)) without a zeroing pass: Jacobi writes
// t = 0 + wd (f - A 0) = 0 + wd f; RBGS's red pass writes 0 + wd f at red nodes and 0 at black
// nodes (the black pass then runs as usual).  With A 0 = D*0 - 0 = +0 and f - (+0) = f the
// values are bitwise those of a sweep over a zeroed array.
template <typename T, int DIM>
__device__ T* sweep_from_zero(const Mode& M, const LG& g, const Coef<T>& c, int rbgs, T* u, T* t, const T* f,
                              const Mir<T>& mi) {
  const T zero = (T)0;
  if (!rbgs) {
    for_rows<DIM>(M, g, -1, [&](int, int, int, int p) { t[p] = add(zero, mul(c.wd, sub(f[p], zero))); });
    mi.push(t);
    M.sync();
    return t;
  }
  for_rows<DIM>(M, g, 0, [&](int, int, int, int p) { u[p] = add(zero, mul(c.wd, sub(f[p], zero))); });  // red
  for_rows<DIM>(M, g, 1, [&](int, int, int, int p) { u[p] = zero; });                                 // black: 0
  mi.push(u);
  M.sync();
  for_rows<DIM>(M, g, 1, [&](int, int, int, int p) {  // black pass
    u[p] = add(u[p], mul(c.wd, pres<T, DIM>(u, p, g, c, f[p])));
  });
  mi.push(u);
  M.sync();
  return u;
}

// u += P e, separable x -> y -> plane axis
template <typename T, int DIM>
__device__ void prolong(const Mode& M, const LG& gf, const LG& gc, const T* e, T* u, const Mir<T>& mi) {
  const T half = (T)0.5;
  for_rows<DIM>(M, gf, -1, [&](int i, int j, int pl, int pu) {
    const int pg = pl + gf.pg0;
    const int I = i >> 1, dx = i & 1;
    const int J = j >> 1, dy = DIM == 3 ? (j & 1) : 0;
    const int P = (pg >> 1) - gc.pg0, dz = pg & 1;
    T vy[2];
    for (int zz = 0; zz <= dz; zz++) {
      T vx[2];
      for (int yy = 0; yy <= dy; yy++) {
        const int p = lin(gc, I, J + yy, P + zz);
        vx[yy] = dx ? mul(half, add(e[p], e[p + 1])) : e[p];
      }
      vy[zz] = dy ? mul(half, add(vx[0], vx[1])) : vx[0];
    }
    const T v = dz ? mul(half, add(vy[0], vy[1])) : vy[0];
    u[pu] = add(u[pu], v);
  });
  mi.push(u);
  M.sync();
}

// the top level's inputs into its shared-memory layout gd: every node (x <= nx, all rows and
// planes) of f, and of u into both U and Tt (with_u); eight elements per thread in flight (a
// warp-per-row copy waited an L2 round trip per element: measured 9.7 us of C1's cycle)
template <typename T>
__device__ void copy_in(const LG& gs, const T* u, const T* f, const LG& gd, T* U, T* Tt, T* F, bool with_u) {
  constexpr int B = 8;
  const int nx1 = gs.nx + 1;
  const int n = nx1 * gs.rows * gs.planes;
  for (int q0 = threadIdx.x; q0 < n; q0 += B * NTT) {
    T vu[B], vf[B];
    int pd[B];
#pragma unroll
    for (int k = 0; k < B; k++) {
      const int q = q0 + k * NTT;
      const int row = q / nx1, i = q - row * nx1;
      const int pl = row / gs.rows, j = row - pl * gs.rows;
      const int ps = pl * gs.sz + j * gs.sy + i;
      pd[k] = pl * gd.sz + j * gd.sy + i;
      if (q < n) {
        vf[k] = f[ps];
        if (with_u) vu[k] = u[ps];
      }
    }
#pragma unroll
    for (int k = 0; k < B; k++)
      if (q0 + k * NTT < n) {
        F[pd[k]] = vf[k];
        if (with_u) {
          U[pd[k]] = vu[k];
          Tt[pd[k]] = vu[k];
        }
      }
  }
}
// every node (x <= nx, all rows) of planes [pa, pb) from the layout gs into gd (a dist slab:
// gd.zoff), into d1 and d2 (if set); eight elements per thread in flight
template <typename T>
__device__ void copy_planes(const LG& gs, const T* src, const LG& gd, T* d1, T* d2, int pa, int pb) {
  constexpr int B = 8;
  const int nx1 = gs.nx + 1;
  const int n = nx1 * gs.rows * (pb - pa);
  for (int q0 = threadIdx.x; q0 < n; q0 += B * NTT) {
    T v[B];
    int pd[B];
#pragma unroll
    for (int k = 0; k < B; k++) {
      const int q = q0 + k * NTT;
      const int row = q / nx1, i = q - row * nx1;
      const int dpl = row / gs.rows, j = row - dpl * gs.rows;
      const int pl = pa + dpl;
      pd[k] = (pl - gd.zoff) * gd.sz + j * gd.sy + i;
      if (q < n) v[k] = src[(pl - gs.zoff) * gs.sz + j * gs.sy + i];
    }
#pragma unroll
    for (int k = 0; k < B; k++)
      if (q0 + k * NTT < n) {
        d1[pd[k]] = v[k];
        if (d2) d2[pd[k]] = v[k];
      }
  }
}
// interior nodes only
template <typename T, int DIM>
__device__ void copy_interior(const Mode& M, const LG& gs, const T* src, const LG& gd, T* dst) {
  for_rows<DIM>(M, gs, -1, [&](int i, int j, int pl, int p) { dst[lin(gd, i, j, pl)] = src[p]; });
}

// a / b correctly rounded (bitwise __ddiv_rn) from y = RN(1/b), without div.rn's reciprocal
// refinement on the critical path (a dependent div.rn measured 440 cycles on this GPU, the
// coarse substitutions of C1 are 18 of them in a chain): q = RN(a y) with one Markstein
// correction, accepted only when the exact remainder a - b q (exact for a faithful q) puts
// a / b strictly inside q's rounding interval — half an ulp each side, a quarter below a power
// of two — else div.rn.  An accepted q is therefore RN(a / b) whatever y was.
__device__ __forceinline__ double div_rn_via(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double q = __fma_rn(__fma_rn(-b, q0, a), y, q0);
  const double r = __fma_rn(-b, q, a);
  const long long bits = __double_as_longlong(q);
  const int e = (int)((bits >> 52) & 0x7ff);
  if (e > 60 && e < 2040) {
    const double hu = __longlong_as_double((long long)(e - 53) << 52);  // half an ulp of q
    const bool below = (r < 0.0) != (b < 0.0);                         // a / b < q
    const bool pow2 = (bits & 0xfffffffffffffll) == 0;
    const double h = __dmul_rn(below && pow2 ? 0.5 * hu : hu, fabs(b));
    if (h > 0x1p-960 && fabs(r) < h) return q;
  }
  return __ddiv_rn(a, b);
}

// ||f - A u|| of a level into *P.norm_out: FP64 sum of squares per thread in for_rows order,
// warp shuffles, the CTA's warps in order, then (cluster mode) the CTAs in rank order — a fixed
// order for a given launch shape (k_tail's norm-only and fused uses share it)
template <typename T>
__device__ double norm_reduce(const Mode& M, double acc, const TailParams<T>& P) {
  __shared__ double wsum[WPC];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < WPC; w++) t = __dadd_rn(t, wsum[w]);
  if (M.solo) {
    if (threadIdx.x == 0) {
      t = __dsqrt_rn(t);
      if (P.norm_out) *P.norm_out = t;
    }
    return t;  // (thread 0 of CTA 0)
  }
  if (threadIdx.x == 0) P.nscratch[blockIdx.x] = t;
  cluster_sync();
  double sum = 0.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int b = 0; b < (int)gridDim.x; b++) sum = __dadd_rn(sum, P.nscratch[b]);
    sum = __dsqrt_rn(sum);
    if (P.norm_out) *P.norm_out = sum;
  }
  return sum;
}

template <typename T, int DIM>
__device__ double tail_norm(const Mode& M, const LG& g, const Coef<T>& c, const T* u, const T* f,
                            const TailParams<T>& P) {
  if (!M.active()) return 0.0;
  double acc = 0.0;
  for_rows<DIM>(M, g, -1, [&](int, int, int, int p) {
    const double r = (double)pres<T, DIM>(u, p, g, c, f[p]);
    acc = __dadd_rn(acc, __dmul_rn(r, r));
  });
  return norm_reduce(M, acc, P);
}

// a Jacobi sweep u -> t that also returns ||f - A u|| of its input (thread 0 of CTA 0): the
// per-node residual the sweep forms anyway, the traversal and the reduction of tail_norm, so
// the value is bitwise tail_norm's.  The one-launch solve takes each iterate's norm from the
// next cycle's first sweep (written to the ping-pong partner: if the stop test then ends the
// solve, the iterate is untouched) instead of a pass of its own.
template <typename T, int DIM>
__device__ double jacobi_norm(const Mode& M, const LG& g, const Coef<T>& c, const T* u, T* t, const T* f,
                              const Mir<T>& mi, const TailParams<T>& P) {
  double acc = 0.0;
  for_rows<DIM>(M, g, -1, [&](int, int, int, int p) {
    const T r = pres<T, DIM>(u, p, g, c, f[p]);
    t[p] = add(u[p], mul(c.wd, r));
    const double rd = (double)r;
    acc = __dadd_rn(acc, __dmul_rn(rd, rd));
  });
  mi.push(t);
  M.sync();
  if (!M.active()) return 0.0;
  return norm_reduce(M, acc, P);
}

template <typename T, int DIM>
__global__ void __launch_bounds__(NTT, 1) k_tail(TailParams<T> P) {
  extern __shared__ __align__(16) unsigned char tsm[];
  if (P.norm_only) {  // the distribution of the cycle's fused norm (a dist level 0: this CTA's slab)
    LG g0 = lg_of(P.g[0]);
    if (P.dist_n > 0) {
      g0.p_lo = P.zr[0][blockIdx.x];
      g0.p_hi = P.zr[0][blockIdx.x + 1];
    }
    tail_norm<T, DIM>(Mode{0 >= P.solo_from, P.dist_n > 0}, g0, P.c[0], P.u[0], P.f[0], P);
    return;
  }
  const bool sm_lv0 = P.smem_from == 0;  // the top tail level lives in shared memory (one CTA)
  // ---- per-level constants, derived once per launch into shared memory: levels >= smem_from
  // keep their four arrays u, t, f, r in CTA 0's shared memory (compact layout P.gs[k]), dist
  // levels (k < dist_n) their slabs in every CTA's, the others live in global memory.
  // (Re-deriving layouts and pointers from the kernel parameters at every use was 30% of a C1
  // cycle's instructions.)
  struct LvRT {
    LG g;
    T* a[4];
    int solo, dist;
  };
  __shared__ LvRT lvt[kTailMax];
  __shared__ Coef<T> lvc[kTailMax];
  __shared__ Mir<T> lvm[kTailDistMax + 1];  // the dist levels' mirrors; [kTailDistMax]: none
  if (threadIdx.x < P.nl) {
    const int k = threadIdx.x;
    const bool sm = k >= P.smem_from;
    LvRT e;
    e.g = lg_of(sm ? P.gs[k] : P.g[k]);
    const int n = P.gs[k].planes * (int)P.gs[k].pstride;
    const int n16 = (n * (int)sizeof(T) + 15) / 16 * 16 / (int)sizeof(T);
    T* base = reinterpret_cast<T*>(tsm + P.soff[k]);
    e.a[0] = sm ? base : P.u[k];
    e.a[1] = sm ? base + n16 : P.t[k];
    e.a[2] = sm ? base + 2 * n16 : P.f[k];
    e.a[3] = sm ? base + 3 * n16 : P.r[k];
    e.solo = k >= P.solo_from;
    e.dist = k < P.dist_n;
    if (e.dist) {
      namespace cg = cooperative_groups;
      const int r = blockIdx.x, C = gridDim.x;
      const int z0 = P.zr[k][r], z1 = P.zr[k][r + 1];
      e.g = lg_of(P.gd[k]);
      e.g.p_lo = z0;
      e.g.p_hi = z1;
      e.g.zoff = z0 - 1;
      T* b = reinterpret_cast<T*>(tsm + P.doff[k]);
      const int m = P.dn16[k];
      e.a[0] = b;                               // u
      e.a[2] = b + m;                           // f
      e.a[3] = b + 2 * m;                       // r
      e.a[1] = P.rbgs ? nullptr : b + 3 * m;    // t (Jacobi)
      Mir<T> mi = Mir<T>::none();
      mi.a[0] = e.a[0];
      mi.a[1] = e.a[1];
      mi.a[2] = e.a[3];
      mi.sz = e.g.sz;
      mi.zoff = e.g.zoff;
      if (z1 > z0) {
        mi.plo = z0;
        mi.phi = z1 - 1;
        const int sz = e.g.sz;
        // ranks whose window [zr[s] - 1, zr[s+1]] holds my first / last plane
        for (int s2 = r - 1; s2 >= 0 && P.zr[k][s2 + 1] == z0 && mi.nlo < 3; s2--, mi.nlo++)
          for (int ai = 0; ai < 3; ai++)
            mi.rem[0][mi.nlo][ai] = mi.a[ai] ? cg::this_cluster().map_shared_rank(mi.a[ai], s2) +
                                                   (z0 - P.zr[k][s2]) * sz
                                             : nullptr;
        for (int s2 = r + 1; s2 < C && P.zr[k][s2] == z1 && mi.nhi < 3; s2++, mi.nhi++)
          for (int ai = 0; ai < 3; ai++)
            mi.rem[1][mi.nhi][ai] = mi.a[ai] ? cg::this_cluster().map_shared_rank(mi.a[ai], s2) +
                                                   (z0 - P.zr[k][s2]) * sz
                                             : nullptr;
      }
      lvm[k] = mi;
    }
    lvt[k] = e;
    lvc[k] = P.c[k];
  }
  if (threadIdx.x == 0) lvm[kTailDistMax] = Mir<T>::none();
  __syncthreads();
  auto mode = [&](int k) { return Mode{lvt[k].solo != 0, lvt[k].dist != 0}; };
  auto MI = [&](int k) -> const Mir<T>& { return lvm[k < P.dist_n ? k : kTailDistMax]; };
  auto G = [&](int k) { return lvt[k].g; };
  auto U = [&](int k) { return lvt[k].a[0]; };
  auto Tt = [&](int k) { return lvt[k].a[1]; };
  auto F = [&](int k) { return lvt[k].a[2]; };
  auto R = [&](int k) { return lvt[k].a[3]; };
  auto zero = [&](const unsigned char* a, const unsigned char* b) {
    for (uint4* q = reinterpret_cast<uint4*>(const_cast<unsigned char*>(a)) + threadIdx.x;
         reinterpret_cast<const unsigned char*>(q) < b; q += NTT)
      *q = make_uint4(0u, 0u, 0u, 0u);
  };
  if (P.dist_n > 0) {
    // every CTA: zeroed slabs (halos, boundaries, coarse guesses), then the top level's inputs
    // when it is dist — f on the own planes, u (also into t) on the window with its halos
    zero(tsm, tsm + P.doff[P.dist_n - 1] + (P.rbgs ? 3 : 4) * P.dn16[P.dist_n - 1] * (int)sizeof(T));
    __syncthreads();
    const LG g0 = lg_of(P.g[0]), d0 = G(0);
    copy_planes<T>(g0, P.f[0], d0, F(0), nullptr, d0.p_lo, d0.p_hi);
    if (!P.zero_first) copy_planes<T>(g0, P.u[0], d0, U(0), Tt(0), d0.p_lo - 1, d0.p_hi + 1);
  }
  if (blockIdx.x == 0 && (P.smem_from < P.nl || P.chol_off >= 0)) {
    // CTA 0's shared memory: the top level's inputs when it lives there (u, also into t: the
    // Jacobi partner's Dirichlet boundary; f), the coarse factor, zeros everywhere else in the
    // shared-memory levels (boundaries, residual borders, coarse guesses); one barrier
    if (P.chol_off >= 0) {
      double* Ls = reinterpret_cast<double*>(tsm + P.chol_off);
      for (int q = threadIdx.x; q < P.m * P.m; q += NTT) Ls[q] = P.chol[q];
    }
    if (P.y_off >= 0) {  // reciprocals of the factor's diagonal behind y (div_rn_via)
      double* rd = reinterpret_cast<double*>(tsm + P.y_off) + P.m;
      for (int i = threadIdx.x; i < P.m; i += NTT) rd[i] = __drcp_rn(P.chol[(long long)i * P.m + i]);
    }
    if (P.smem_from < P.nl) {
      const unsigned char* end = tsm + P.smem_bytes;
      if (sm_lv0) {
        copy_in<T>(lg_of(P.g[0]), P.u[0], P.f[0], G(0), U(0), Tt(0), F(0), !P.zero_first);
        const unsigned char* f0 = reinterpret_cast<const unsigned char*>(F(0));
        if (P.zero_first) zero(tsm + P.soff[0], f0);  // u and t of the zero guess
        zero(reinterpret_cast<const unsigned char*>(R(0)), end);
      } else {
        zero(tsm + P.soff[P.smem_from], end);
      }
    }
  }
  __syncthreads();
  if (P.dist_n > 0) cluster_sync();  // no CTA mirrors into a slab its owner is still zeroing
  // ---- P.solve: the driver loop of mg_solve in this launch — the level arrays stay
  // where they are between cycles (the top level's iterate in cur[0]); else one cycle
  T* cur[kTailMax];
  cur[0] = U(0);
  __shared__ int s_flag;
  auto bcast = [&](int v) -> int {  // thread 0 of CTA 0's decision to every thread
    if (gridDim.x == 1) {
      if (threadIdx.x == 0) s_flag = v;
      __syncthreads();
      return s_flag;
    }
    volatile int* g = reinterpret_cast<volatile int*>(P.nscratch + gridDim.x);
    if (blockIdx.x == 0 && threadIdx.x == 0) *g = v;
    cluster_sync();
    return *g;
  };
  // Jacobi with pre-smoothing: each iterate's norm from the next cycle's first sweep (jacobi_norm)
  const bool fuse_norm = P.solve && P.rbgs == 0 && P.nu1 >= 1 && !P.zero_first;
  if (P.solve && !fuse_norm) {
    const double r0 = tail_norm<T, DIM>(mode(0), G(0), P.c[0], cur[0], F(0), P);
    int go = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) go = loop_begin(r0, P.solve) ? 1 : 0;
    if (!bcast(go)) return;  // u unchanged
  }
  for (int cyc = 0;; cyc++) {
  bool first_done = false;  // level 0's first pre-sweep already ran (fuse_norm)
  if (fuse_norm) {
    T* oth = cur[0] == U(0) ? Tt(0) : U(0);
    const double rk = jacobi_norm<T, DIM>(mode(0), G(0), lvc[0], cur[0], oth, F(0), MI(0), P);
    int go = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0)
      go = (cyc == 0 ? loop_begin(rk, P.solve) : loop_step(rk, P.solve)) ? 1 : 0;
    if (!bcast(go)) break;  // cur[0] still holds the iterate
    cur[0] = oth;
    first_done = true;
  }
  // ---- descend
  for (int k = 1; k < P.nl; k++) cur[k] = U(k);
  for (int k = 0; k < P.nl - 1; k++) {
    const LG g = G(k);
    const Coef<T> c = lvc[k];
    const Mode M = mode(k);
    const bool zero = k > 0 || P.zero_first;  // V_H(0, ...)
    const bool fold = zero && P.nu1 > 0 && P.rbgs != 2;  // the zero guess folded into the first sweep
    if (zero && !fold) {
      zero_level(M, g, cur[k]);
      M.sync();
    }
    for (int s = (k == 0 && first_done) ? 1 : 0; s < P.nu1; s++) {
      T* oth = cur[k] == U(k) ? Tt(k) : U(k);
      cur[k] = (s == 0 && fold) ? sweep_from_zero<T, DIM>(M, g, c, P.rbgs, cur[k], oth, F(k), MI(k))
                                : sweep<T, DIM>(M, g, c, P.rbgs, cur[k], oth, F(k), MI(k));
    }
    // separate residual and restriction passes: measured faster than one fused pass whose
    // coarse threads each evaluate 3^d fine residuals (latency-bound serial chains)
    residual<T, DIM>(M, g, c, cur[k], F(k), R(k), MI(k));
    // the restriction writes level k+1: its mode (a solo coarse level is restricted by CTA 0,
    // reading the residual the cluster barrier above made visible); from a dist level every CTA
    // restricts the coarse planes of its slab (zr[k+1]) from its own residual slab, into the
    // coarse f wherever it lives (its own slab, CTA 0's shared memory, global memory)
    if (M.dist) {
      LG gc = G(k + 1);
      T* fc = F(k + 1);
      if (!mode(k + 1).dist) {
        gc.p_lo = P.zr[k + 1][blockIdx.x];
        gc.p_hi = P.zr[k + 1][blockIdx.x + 1];
        if (k + 1 >= P.smem_from) fc = cooperative_groups::this_cluster().map_shared_rank(fc, 0);
      }
      restrict_fw<T, DIM>(Mode{false, true}, g, gc, R(k), fc);
    } else {
      restrict_fw<T, DIM>(mode(k + 1), g, G(k + 1), R(k), F(k + 1));
    }
  }
  // ---- coarsest level (Alg. 1 line 2)
  {
    const int k = P.nl - 1;
    const LG g = G(k);
    const Coef<T> c = lvc[k];
    const Mode M = mode(k);
    const bool zero = P.nl > 1 || P.zero_first;
    // DIRECT writes every interior node, so its zero guess needs no pass; SWEEPS folds it
    // into the first sweep (lexicographic GS zeroes first)
    const bool fold = zero && P.sweeps && P.ncoarse > 0 && P.rbgs != 2;
    if (zero && P.sweeps && !fold) {
      zero_level(M, g, cur[k]);
      M.sync();
    }
    if (P.sweeps) {
      for (int s = 0; s < P.ncoarse; s++) {
        T* oth = cur[k] == U(k) ? Tt(k) : U(k);
        cur[k] = (s == 0 && fold) ? sweep_from_zero<T, DIM>(M, g, c, P.rbgs, cur[k], oth, F(k), MI(k))
                                  : sweep<T, DIM>(M, g, c, P.rbgs, cur[k], oth, F(k), MI(k));
      }
    } else {
      const int m = P.m;
      if (m > 1 && m <= 32 && P.y_off >= 0) {
        // warp 0, lane i owns row i and node i (the oracle's row order: plane, y, x).  Bitwise
        // the sequential substitutions: forward, column k finalises y_k and every row below
        // subtracts L_ik y_k — row i still subtracts in the order k = 0, 1, ..; backward, x_kk
        // arrives in descending kk, so lane i parks its products L_kk,i x_kk in shared memory
        // and folds them in ascending kk once x_{i+1} is known.  The chains of dependent loads
        // and divisions of one thread (measured 5000 cycles per substitution at m = 9) become
        // one shuffle and one division per step.
        if (blockIdx.x == 0 && threadIdx.x < 32) {
          const int lane = threadIdx.x;
          const bool own = lane < m;
          const int jlo = DIM == 3 ? 1 : 0, nj = DIM == 3 ? g.ny - 1 : 1, ni = g.nx - 1;
          const double* L = P.chol_off >= 0 ? reinterpret_cast<const double*>(tsm + P.chol_off) : P.chol;
          const double* rd = reinterpret_cast<const double*>(tsm + P.y_off) + m;
          double* Ps = reinterpret_cast<double*>(tsm + P.y_off) + 2 * m;  // [kk][i], 32 x 32
          int node = 0;
          if (own) {
            const int r = lane / ni;
            node = lin(g, 1 + lane - r * ni, jlo + r % nj, g.p_lo + r / nj);
          }
          double acc = own ? (double)F(k)[node] : 0.0;
          for (int kk = 0; kk < m; kk++) {
            if (lane == kk) acc = div_rn_via(acc, L[kk * m + kk], rd[kk]);
            const double ykk = __shfl_sync(0xffffffffu, acc, kk);
            if (lane > kk && own) acc = __dsub_rn(acc, __dmul_rn(L[lane * m + kk], ykk));
          }
          for (int i = m - 1; i >= 0; i--) {
            if (lane == i) {
              double sacc = acc;
              for (int kk = i + 1; kk < m; kk++) sacc = __dsub_rn(sacc, Ps[kk * 32 + i]);
              acc = div_rn_via(sacc, L[i * m + i], rd[i]);
            }
            const double xi = __shfl_sync(0xffffffffu, acc, i);
            if (lane < i) Ps[i * 32 + lane] = __dmul_rn(L[i * m + lane], xi);
          }
          if (own) cur[k][node] = (T)acc;
        }
      } else if (blockIdx.x == 0 && threadIdx.x == 0) {
        // same loop order as k_coarse_direct / the oracle
        const int jlo = DIM == 3 ? 1 : 0, jhi = DIM == 3 ? g.ny - 1 : 0;
        // the factor and the vector in shared memory: the substitutions are serial chains of
        // dependent loads (a global y costs an L2 round trip per step: measured 8.5 us at m = 9)
        const double* L = P.chol_off >= 0 ? reinterpret_cast<const double*>(tsm + P.chol_off) : P.chol;
        const T* fk = F(k);
        if (m == 1) {
          const int p = lin(g, 1, jlo, g.p_lo);
          cur[k][p] = (T)div_rn_via((double)fk[p], P.D_coarse, P.rD_coarse);
        } else if (P.y_off >= 0) {  // y and the diagonal's reciprocals (the prologue's) in shared memory
          double* y = reinterpret_cast<double*>(tsm + P.y_off);
          const double* rd = y + m;
          int q = 0;
          for (int pl = g.p_lo; pl < g.p_hi; pl++)
            for (int j = jlo; j <= jhi; j++)
              for (int i = 1; i < g.nx; i++) y[q++] = (double)fk[lin(g, i, j, pl)];
          for (int i = 0; i < m; i++) {
            double sacc = y[i];
            for (int kk = 0; kk < i; kk++) sacc = __dsub_rn(sacc, __dmul_rn(L[(long long)i * m + kk], y[kk]));
            y[i] = div_rn_via(sacc, L[(long long)i * m + i], rd[i]);
          }
          for (int i = m - 1; i >= 0; i--) {
            double sacc = y[i];
            for (int kk = i + 1; kk < m; kk++) sacc = __dsub_rn(sacc, __dmul_rn(L[(long long)kk * m + i], y[kk]));
            y[i] = div_rn_via(sacc, L[(long long)i * m + i], rd[i]);
          }
          q = 0;
          for (int pl = g.p_lo; pl < g.p_hi; pl++)
            for (int j = jlo; j <= jhi; j++)
              for (int i = 1; i < g.nx; i++) cur[k][lin(g, i, j, pl)] = (T)y[q++];
        } else {
          double* y = P.work;
          int q = 0;
          for (int pl = g.p_lo; pl < g.p_hi; pl++)
            for (int j = jlo; j <= jhi; j++)
              for (int i = 1; i < g.nx; i++) y[q++] = (double)fk[lin(g, i, j, pl)];
          for (int i = 0; i < m; i++) {
            double sacc = y[i];
            for (int kk = 0; kk < i; kk++) sacc = __dsub_rn(sacc, __dmul_rn(L[(long long)i * m + kk], y[kk]));
            y[i] = __ddiv_rn(sacc, L[(long long)i * m + i]);
          }
          for (int i = m - 1; i >= 0; i--) {
            double sacc = y[i];
            for (int kk = i + 1; kk < m; kk++) sacc = __dsub_rn(sacc, __dmul_rn(L[(long long)kk * m + i], y[kk]));
            y[i] = __ddiv_rn(sacc, L[(long long)i * m + i]);
          }
          q = 0;
          for (int pl = g.p_lo; pl < g.p_hi; pl++)
            for (int j = jlo; j <= jhi; j++)
              for (int i = 1; i < g.nx; i++) cur[k][lin(g, i, j, pl)] = (T)y[q++];
        }
      }
      M.sync();
    }
  }
  // ---- ascend
  for (int k = P.nl - 2; k >= 0; k--) {
    const Mode M = mode(k);
    const LG g = G(k);
    const Coef<T> c = lvc[k];
    const T* e = cur[k + 1];
    LG ge = G(k + 1);
    if (mode(k + 1).solo && M.dist) {  // read CTA 0's coarse correction in place (DSMEM)
      if (k + 1 >= P.smem_from) e = cooperative_groups::this_cluster().map_shared_rank(cur[k + 1], 0);
      cluster_sync();
    } else if (mode(k + 1).solo && !M.solo) {  // CTA 0's solo levels visible to every CTA
      if (k + 1 >= P.smem_from) {  // the correction lives in CTA 0's shared memory: publish it
        const LG gg = lg_of(P.g[k + 1]);
        if (blockIdx.x == 0) {
          copy_interior<T, DIM>(Mode{true}, ge, e, gg, P.u[k + 1]);
          __syncthreads();
        }
        e = P.u[k + 1];
        ge = gg;
      }
      cluster_sync();
    }
    prolong<T, DIM>(M, g, ge, e, cur[k], MI(k));
    for (int s = 0; s < P.nu2; s++)
      cur[k] = sweep<T, DIM>(M, g, c, P.rbgs, cur[k], cur[k] == U(k) ? Tt(k) : U(k), F(k), MI(k));
  }
  if (!P.solve) break;
  if (!fuse_norm) {
    const double rk = tail_norm<T, DIM>(mode(0), G(0), P.c[0], cur[0], F(0), P);
    int go = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) go = loop_step(rk, P.solve) ? 1 : 0;
    if (!bcast(go)) break;
  }
  }  // for (cyc)
  // result of the top tail level in u[0]
  if (sm_lv0 || cur[0] != P.u[0]) copy_interior<T, DIM>(mode(0), G(0), (const T*)cur[0], lg_of(P.g[0]), P.u[0]);
  if (P.norm_out && !P.solve) tail_norm<T, DIM>(mode(0), G(0), P.c[0], cur[0], F(0), P);
  if (P.dist_n > 0) cluster_sync();  // every slab stays alive until no CTA can touch it
}

}  // namespace

template <typename T>
void tail_prepare(TailParams<T>& q) {
  // 16 CTAs (non-portable) where allowed, else the portable 8; probed once per device (the
  // non-portable opt-in and the shared-memory opt-in are per-device function attributes)
  const int cluster = per_device_once((const void*)k_tail<T, 3>, [] {
    cudaFuncSetAttribute(k_tail<T, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTailSmemCap);
    cudaFuncSetAttribute(k_tail<T, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTailSmemCap);
    int c = 8;
    if (cudaFuncSetAttribute(k_tail<T, 2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
        cudaFuncSetAttribute(k_tail<T, 3>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
      cudaLaunchConfig_t c16 = {};
      c16.gridDim = dim3(16);
      c16.blockDim = dim3(NTT);
      c16.dynamicSmemBytes = kTailSmemCap;
      cudaLaunchAttribute a;
      a.id = cudaLaunchAttributeClusterDimension;
      a.val.clusterDim.x = 16;
      a.val.clusterDim.y = 1;
      a.val.clusterDim.z = 1;
      c16.attrs = &a;
      c16.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, k_tail<T, 3>, &c16) == cudaSuccess && n >= 1) c = 16;
    }
    cudaGetLastError();
    return c;
  });
  auto interior = [](const Geom& g) {
    return (long long)(g.nx - 1) * (g.three_d ? g.ny - 1 : 1) * (g.p_hi - g.p_lo);
  };
  // tiny tails (a few thousand nodes, e.g. the whole 65^2 C1 hierarchy) run on one CTA
  q.csize = interior(q.g[0]) <= 8192 ? 1 : cluster;
  // levels from solo_from on run on CTA 0 alone with block barriers (all of them on one CTA)
  // measured (C2, C3, C4): 2048 interior nodes in 3D (a 17^3 level is faster on the cluster),
  // 8192 in 2D (a 65^2 level is faster on CTA 0 with its arrays in shared memory)
  const long long solo_max = q.g[0].three_d ? 2048 : 8192;
  q.solo_from = q.nl;
  for (int k = 0; k < q.nl; k++)
    if (q.csize == 1 || interior(q.g[k]) <= solo_max) {
      q.solo_from = k;
      break;
    }
  auto bytes16 = [](long long b) { return (b + 15) / 16 * 16; };
  auto words = [&](const Geom& g) { return bytes16((long long)g.planes * g.pstride * (long long)sizeof(T)); };
  auto compact = [](Geom g) {
    g.pitch = g.nx + 1;
    g.pstride = g.three_d ? (long long)(g.ny + 1) * (g.nx + 1) : g.pitch;
    return g;
  };
  // dist levels: the leading cluster levels, split into plane slabs — level 0 evenly over the
  // CTAs, each coarser level by ceil(z / 2) of the finer slab boundaries, so that a CTA owns
  // coarse plane P iff it owns fine plane 2P: the restriction of its coarse planes and the
  // prolongation into its fine planes read only its slabs and their one-plane halos.  They
  // take the front of every CTA's shared memory, as long as they fit.
  q.dist_n = 0;
  long long dbytes = 0;
  if (q.csize > 1 && q.rbgs != 2) {
    const int C = q.csize;
    const int kmax = std::min(q.solo_from, q.nl - 1);  // the coarsest level is never dist
    for (int r = 0; r <= C; r++) q.zr[0][r] = q.g[0].p_lo + (int)((long long)(q.g[0].p_hi - q.g[0].p_lo) * r / C);
    for (int k = 1; k <= kmax; k++)
      for (int r = 0; r <= C; r++) q.zr[k][r] = (q.zr[k - 1][r] + 1) / 2;
    for (int k = 0; k < kmax && k < kTailDistMax; k++) {
      const Geom& g = q.g[k];
      bool ok = g.p_glob0 == 0 && q.zr[k][0] == g.p_lo && q.zr[k][C] == g.p_hi;
      if (k + 1 <= kmax) ok = ok && q.zr[k + 1][0] == q.g[k + 1].p_lo && q.zr[k + 1][C] == q.g[k + 1].p_hi;
      int wmax = 0;
      for (int r = 0; r < C && ok; r++) {
        const int w = q.zr[k][r + 1] - q.zr[k][r];
        wmax = std::max(wmax, w);
        if (w > 0) {  // mirror targets: the neighbour and the empty slabs past it (at most 3)
          int lo = 1, hi = 1;
          for (int s2 = r - 1; s2 > 0 && q.zr[k][s2] == q.zr[k][r]; s2--) lo++;
          for (int s2 = r + 1; s2 < C - 1 && q.zr[k][s2 + 1] == q.zr[k][r + 1]; s2++) hi++;
          ok = lo <= 3 && hi <= 3;
        }
      }
      if (!ok) break;
      Geom gd = compact(g);
      gd.planes = wmax + 2;
      gd.p_glob0 = 0;
      const long long m = words(gd) / (long long)sizeof(T);
      const long long bytes = m * (long long)sizeof(T) * (q.rbgs ? 3 : 4);
      if (dbytes + bytes > kTailSmemMax) break;
      q.gd[k] = gd;
      q.doff[k] = (int)dbytes;
      q.dn16[k] = (int)m;
      dbytes += bytes;
      q.dist_n = k + 1;
    }
  }
  // the solo levels' arrays (u, t, f, r) in CTA 0's shared memory behind the dist slabs,
  // compact layout: the coarsest levels that fit (a solo level above them stays in global memory)
  q.smem_from = q.nl;
  long long total = dbytes;
  for (int k = q.nl - 1; k >= q.solo_from; k--) {
    const Geom g = compact(q.g[k]);
    if (total + 4 * words(g) > kTailSmemMax) break;
    total += 4 * words(g);
    q.gs[k] = g;
    q.smem_from = k;
  }
  long long off = dbytes;
  for (int k = q.smem_from; k < q.nl; k++) {
    q.soff[k] = (int)off;
    off += 4 * words(q.gs[k]);
  }
  q.smem_bytes = (int)off;
  // direct coarsest solve: its vector and (when it fits) the factor behind the levels
  q.chol_off = q.y_off = -1;
  if (!q.sweeps && q.m > 1) {
    // y, 1 / L_ii, and for m <= 32 the backward substitution's 32 x 32 products
    const long long lb = bytes16((long long)q.m * q.m * 8), yb = bytes16((long long)q.m * 16 + (q.m <= 32 ? 8192 : 0));
    if (off + lb + yb <= kTailSmemCap) {
      q.chol_off = (int)off;
      off += lb;
    }
    if (off + yb <= kTailSmemCap) {
      q.y_off = (int)off;
      off += yb;
    }
  }
  q.smem_total = (int)off;
}

template <typename T>
cudaError_t launch_tail(const TailParams<T>& q, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(q.csize);
  cfg.blockDim = dim3(NTT);
  cfg.stream = st;
  cfg.dynamicSmemBytes = q.norm_only ? 0 : q.smem_total;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = q.csize;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = q.csize > 1 ? 1 : 0;
  return q.g[0].three_d ? cudaLaunchKernelEx(&cfg, k_tail<T, 3>, q) : cudaLaunchKernelEx(&cfg, k_tail<T, 2>, q);
}

template void tail_prepare<double>(TailParams<double>&);
template void tail_prepare<float>(TailParams<float>&);
template cudaError_t launch_tail<double>(const TailParams<double>&, cudaStream_t);
template cudaError_t launch_tail<float>(const TailParams<float>&, cudaStream_t);

}  // namespace mg
