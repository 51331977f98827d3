// kernels_cd.cu — complex diffusion with FAS on cell-centred levels (sm_100a):
// the paper's second workload (Eqs. 2-3).
//
//   (A u)(c) = a_c u(c) - sum_{inner faces} w_d g_f u(c+o),   a_c = 1 + sum w_d g_f,
//   g_f = (g(c) + g(c+o)) / 2,  g = e^{i theta} / (1 + (Im u_lag / (k theta))^2)
//
// One thread per cell (complex element = one 8/16-byte vector load); the lagged
// diffusivity g is a stored complex field per level, rebuilt once per cycle
// (k_cd_gfield).  Canonical complex arithmetic (reading 19, the same
// order as oracle/cd_oracle.c, every operation an explicitly rounded intrinsic):
//   cmul(a,b) = (a.re b.re - a.im b.im, a.re b.im + a.im b.re)
//   cdiv(x,y) = ((x.re y.re + x.im y.im)/den, (x.im y.re - x.re y.im)/den), den = |y|^2
//   faces x-, x+, [y-, y+], plane-, plane+ (those inside the domain)
// so the iterates are bitwise those of the oracle.
#include "kernels.h"
#include "kernels_cd.h"
#include <cstdint>
#include <type_traits>

#include "cd_common.cuh"
#include "launch_util.h"

namespace mg {

namespace {
using namespace cdk;

struct Cell {
  int i, j, k;
  long long q;
};


// Visit every cell of a level: blocks stride over rows (one 32-bit division per row, not
// per cell); a block covers 2^r rows at once when a row is narrower than the block.
template <class F>
__device__ __forceinline__ void for_cells(const Geom& g, F fn) {
  const int nr = g.three_d ? g.ny : 1;
  const int rows = nr * g.nz;
  int sh = 0;  // log2(rows per block pass)
  while ((g.nx << (sh + 1)) <= (int)blockDim.x) sh++;
  const int w = (int)blockDim.x >> sh;  // threads per row
  const int sub = (int)threadIdx.x / w, i0 = (int)threadIdx.x - sub * w;
  for (int r0 = (int)blockIdx.x << sh; r0 < rows; r0 += (int)gridDim.x << sh) {
    const int row = r0 + sub;
    if (row >= rows) continue;
    const int j = row % nr, k = row / nr;
    const long long base = (long long)k * g.pstride + (long long)j * g.pitch;
    for (int i = i0; i < g.nx; i += w) fn(Cell{i, j, k, base + i});
  }
}
// the cells of one colour ((i + j + k) & 1 == colour)
template <class F>
__device__ __forceinline__ void for_cells_colour(const Geom& g, int colour, F fn) {
  const int nr = g.three_d ? g.ny : 1;
  const int rows = nr * g.nz;
  const int half = (g.nx + 1) >> 1;
  int sh = 0;
  while ((half << (sh + 1)) <= (int)blockDim.x) sh++;
  const int w = (int)blockDim.x >> sh;
  const int sub = (int)threadIdx.x / w, i0 = (int)threadIdx.x - sub * w;
  for (int r0 = (int)blockIdx.x << sh; r0 < rows; r0 += (int)gridDim.x << sh) {
    const int row = r0 + sub;
    if (row >= rows) continue;
    const int j = row % nr, k = row / nr;
    const int par = (j + k + colour) & 1;
    const long long base = (long long)k * g.pstride + (long long)j * g.pitch;
    for (int ih = i0; ih < half; ih += w) {
      const int i = 2 * ih + par;
      if (i < g.nx) fn(Cell{i, j, k, base + i});
    }
  }
}

// one inner face's contribution: cf = w * (g_c + g_n)/2; acc_a += cf; acc_s += cf * u_n
template <typename T, class GF>
__device__ __forceinline__ void face(T w, C2<T> gc, long long qn, GF gat, const T* u, C2<T>& acc_a, C2<T>& acc_s) {
  const C2<T> gn = gat(qn);
  const T half = (T)0.5;
  const C2<T> cf = {mul(w, mul(half, add(gc.re, gn.re))), mul(w, mul(half, add(gc.im, gn.im)))};
  acc_a = {add(acc_a.re, cf.re), add(acc_a.im, cf.im)};
  const C2<T> t = cmul(cf, ld(u, qn));
  acc_s = {add(acc_s.re, t.re), add(acc_s.im, t.im)};
}

// (A u)(c) and a_c; gat(q) returns the lagged diffusivity of cell q
template <typename T, class GF>
__device__ __forceinline__ C2<T> apply(const Geom& g, const CdCoef<T>& c, GF gat, const T* u, const Cell& x,
                                       C2<T>& diag) {
  const C2<T> gc = gat(x.q);
  C2<T> acc_a = {(T)0, (T)0}, acc_s = {(T)0, (T)0};
  if (x.i > 0) face(c.w[0], gc, x.q - 1, gat, u, acc_a, acc_s);
  if (x.i < g.nx - 1) face(c.w[0], gc, x.q + 1, gat, u, acc_a, acc_s);
  if (g.three_d) {
    if (x.j > 0) face(c.w[1], gc, x.q - g.pitch, gat, u, acc_a, acc_s);
    if (x.j < g.ny - 1) face(c.w[1], gc, x.q + g.pitch, gat, u, acc_a, acc_s);
  }
  if (x.k > 0) face(c.w[2], gc, x.q - g.pstride, gat, u, acc_a, acc_s);
  if (x.k < g.nz - 1) face(c.w[2], gc, x.q + g.pstride, gat, u, acc_a, acc_s);
  diag = {add((T)1, acc_a.re), acc_a.im};
  const C2<T> du = cmul(diag, ld(u, x.q));
  return {sub(du.re, acc_s.re), sub(du.im, acc_s.im)};
}

template <typename T>
struct Stored {  // lagged diffusivity read from the g field
  const T* gd;
  __device__ C2<T> operator()(long long q) const { return ld(gd, q); }
};
template <typename T>
struct OnTheFly {  // g(u) evaluated from u itself (nonlinear residual)
  const CdCoef<T>* c;
  const T* u;
  __device__ C2<T> operator()(long long q) const { return diffusivity(*c, u[2 * q + 1]); }
};

// u + omega * (f - A u) / a_c
template <typename T>
__device__ __forceinline__ C2<T> relax(const Geom& g, const CdCoef<T>& c, const T* gd, const T* u, const T* f,
                                       const Cell& x) {
  C2<T> d;
  const C2<T> Au = apply(g, c, Stored<T>{gd}, u, x, d);
  const C2<T> fu = ld(f, x.q), uu = ld(u, x.q);
  const C2<T> z = cdiv(C2<T>{sub(fu.re, Au.re), sub(fu.im, Au.im)}, d);
  return {add(uu.re, mul(c.omega, z.re)), add(uu.im, mul(c.omega, z.im))};
}

constexpr int NB = 256;

template <typename T>
__global__ void __launch_bounds__(NB) k_cd_gfield(Geom g, CdCoef<T> c, const T* __restrict__ u, T* __restrict__ gd) {
  for_cells(g, [&](const Cell& x) { st(gd, x.q, diffusivity(c, u[2 * x.q + 1])); });
}

template <typename T>
__global__ void __launch_bounds__(NB) k_cd_jacobi(Geom g, CdCoef<T> c, const T* __restrict__ gd,
                                                  const T* __restrict__ uin, const T* __restrict__ f,
                                                  T* __restrict__ uout) {
  for_cells(g, [&](const Cell& x) { st(uout, x.q, relax(g, c, gd, uin, f, x)); });
}

// one colour of red-black GS in place
template <typename T>
__global__ void __launch_bounds__(NB) k_cd_rbgs(Geom g, CdCoef<T> c, const T* __restrict__ gd, T* u,
                                                const T* __restrict__ f, int colour) {
  for_cells_colour(g, colour, [&](const Cell& x) { st(u, x.q, relax(g, c, gd, u, f, x)); });
}

// coarse cell C: x-pairs, then y-pairs, [then z-pairs], times 2^-d (reading 19)
template <typename T, class V>
__device__ __forceinline__ C2<T> average_children(const Geom& gf, const Cell& X, V val) {
  const int nkz = 2;  // plane-axis pair (3D z, 2D y)
  const int njy = gf.three_d ? 2 : 1;
  C2<T> sz[2];
  for (int dz = 0; dz < nkz; dz++) {
    C2<T> sy[2];
    for (int dy = 0; dy < njy; dy++) {
      const int k = 2 * X.k + dz, j = gf.three_d ? 2 * X.j + dy : 0;
      const long long q = (long long)k * gf.pstride + (long long)j * gf.pitch + 2 * X.i;
      Cell a{2 * X.i, j, k, q}, b{2 * X.i + 1, j, k, q + 1};
      const C2<T> va = val(a), vb = val(b);
      sy[dy] = {add(va.re, vb.re), add(va.im, vb.im)};
    }
    sz[dz] = gf.three_d ? C2<T>{add(sy[0].re, sy[1].re), add(sy[0].im, sy[1].im)} : sy[0];
  }
  // 2D: sz[0], sz[1] are the two x-pair sums of rows 2J, 2J+1 (the y-pairs); 3D: the y-pair sums
  // of planes 2K, 2K+1 (the z-pairs)
  const C2<T> s = {add(sz[0].re, sz[1].re), add(sz[0].im, sz[1].im)};
  const T scale = gf.three_d ? (T)0.125 : (T)0.25;
  return {mul(s.re, scale), mul(s.im, scale)};
}

template <typename T>
__global__ void __launch_bounds__(NB) k_cd_restrict(Geom gf, Geom gc, const T* __restrict__ v, T* __restrict__ vh,
                                                    T* __restrict__ vc) {
  for_cells(gc, [&](const Cell& X) {
    const C2<T> o = average_children<T>(gf, X, [&](const Cell& a) { return ld(v, a.q); });
    st(vh, X.q, o);
    if (vc) st(vc, X.q, o);
  });
}

template <typename T>
__global__ void __launch_bounds__(NB) k_cd_fas_rhs(Geom gf, Geom gc, CdCoef<T> cf, CdCoef<T> cc,
                                                   const T* __restrict__ gdf, const T* __restrict__ uf,
                                                   const T* __restrict__ ff, const T* __restrict__ gdc,
                                                   const T* __restrict__ uh, T* __restrict__ fc) {
  for_cells(gc, [&](const Cell& X) {
    // R (f - A_h u_h)
    const C2<T> Rr = average_children<T>(gf, X, [&](const Cell& a) {
      C2<T> d;
      const C2<T> Au = apply(gf, cf, Stored<T>{gdf}, uf, a, d);
      const C2<T> fv = ld(ff, a.q);
      return C2<T>{sub(fv.re, Au.re), sub(fv.im, Au.im)};
    });
    C2<T> d;
    const C2<T> AH = apply(gc, cc, Stored<T>{gdc}, uh, X, d);
    st(fc, X.q, C2<T>{add(AH.re, Rr.re), add(AH.im, Rr.im)});
  });
}

template <typename T>
__global__ void __launch_bounds__(NB) k_cd_prolong(Geom gf, Geom gc, const T* __restrict__ uc,
                                                   const T* __restrict__ uh, T* __restrict__ uf) {
  for_cells(gf, [&](const Cell& x) {
    const long long Q = (long long)(x.k >> 1) * gc.pstride + (long long)(gf.three_d ? (x.j >> 1) : 0) * gc.pitch +
                        (x.i >> 1);
    C2<T> e = ld(uc, Q);
    if (uh) {
      const C2<T> h = ld(uh, Q);
      e = {sub(e.re, h.re), sub(e.im, h.im)};
    }
    const C2<T> u = ld(uf, x.q);
    st(uf, x.q, C2<T>{add(u.re, e.re), add(u.im, e.im)});
  });
}

template <typename T>
__global__ void __launch_bounds__(NB) k_cd_residual(Geom g, CdCoef<T> c, const T* __restrict__ gd,
                                                    const T* __restrict__ u, const T* __restrict__ f,
                                                    T* __restrict__ r) {
  for_cells(g, [&](const Cell& x) {
    C2<T> d;
    const C2<T> Au = apply(g, c, Stored<T>{gd}, u, x, d);
    const C2<T> fv = ld(f, x.q);
    st(r, x.q, C2<T>{sub(fv.re, Au.re), sub(fv.im, Au.im)});
  });
}

template <typename T, bool STORED>
__global__ void __launch_bounds__(NB) k_cd_norm(Geom g, CdCoef<T> c, const T* __restrict__ gd,
                                                const T* __restrict__ u, const T* __restrict__ f,
                                                double* __restrict__ partial) {
  __shared__ double red[NB / 32];
  double s = 0.0;
  const OnTheFly<T> gfly{&c, u};
  for_cells(g, [&](const Cell& x) {
    C2<T> d;
    const C2<T> Au = STORED ? apply(g, c, Stored<T>{gd}, u, x, d) : apply(g, c, gfly, u, x, d);
    const C2<T> fv = ld(f, x.q);
    const double rr = (double)sub(fv.re, Au.re), ri = (double)sub(fv.im, Au.im);
    s = __dadd_rn(s, __dadd_rn(__dmul_rn(rr, rr), __dmul_rn(ri, ri)));
  });
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < NB / 32; w++) tot = __dadd_rn(tot, red[w]);
    partial[blockIdx.x] = tot;
  }
}

template <typename T>
__global__ void __launch_bounds__(NB) k_cd_fill(Geom g, T* __restrict__ dst, uint64_t seed, double lo, double hi) {
  const int nr = g.three_d ? g.ny : 1;
  for_cells(g, [&](const Cell& x) {
    const unsigned long long idx = ((unsigned long long)x.k * nr + x.j) * (unsigned long long)g.nx + x.i;
    unsigned long long z = seed + (idx + 1ull) * 0x9E3779B97F4A7C15ull;  // SplitMix64, reading 10
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const double r = (double)(z >> 11) * 0x1.0p-53;
    const double v = (lo == 0.0 && hi == 1.0) ? r : __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), r));
    st(dst, x.q, C2<T>{(T)v, (T)0});
  });
}

int grid_for(long long n) {
  const int sms = sm_count();
  const long long b = (n + NB - 1) / NB;
  const long long cap = (long long)(sms > 0 ? sms : 148) * 8;  // 8 x 256 threads per SM
  return (int)(b < cap ? (b < 1 ? 1 : b) : cap);
}

// blocks for a row-striding kernel over level g (rows per block pass as in for_cells)
int grid_rows(const Geom& g, int width) {
  const long long rows = (long long)(g.three_d ? g.ny : 1) * g.nz;
  int sh = 0;
  while (((long long)width << (sh + 1)) <= NB) sh++;
  return grid_for(((rows + (1ll << sh) - 1) >> sh) * NB);
}

}  // namespace

// g over the whole pitched array, one 16-byte vector (16 / (2 sizeof T) cells) per thread and
// step: the per-cell function is that of k_cd_gfield (bitwise); pitch cells beyond nx get a
// harmless value that nothing reads (every kernel bounds its faces by nx)
template <typename T>
__global__ void __launch_bounds__(NB) k_cd_gfield_vec(Geom g, CdCoef<T> c, const T* __restrict__ u,
                                                      T* __restrict__ gd, long long nvec) {
  constexpr int CW = 16 / (2 * (int)sizeof(T));
  using V = std::conditional_t<sizeof(T) == 8, double2, float4>;
  for (long long q = (long long)blockIdx.x * NB + threadIdx.x; q < nvec; q += (long long)gridDim.x * NB) {
    const V uv = reinterpret_cast<const V*>(u)[q];
    const T* ur = reinterpret_cast<const T*>(&uv);
    V gv;
    T* gr = reinterpret_cast<T*>(&gv);
#pragma unroll
    for (int j = 0; j < CW; j++) {
      const C2<T> d = diffusivity(c, ur[2 * j + 1]);
      gr[2 * j] = d.re;
      gr[2 * j + 1] = d.im;
    }
    reinterpret_cast<V*>(gd)[q] = gv;
  }
}

template <typename T>
cudaError_t cd_launch_gfield(const Geom& g, const CdCoef<T>& c, const T* u, T* gd, cudaStream_t s) {
  constexpr int CW = 16 / (2 * (int)sizeof(T));
  const long long cells = (long long)g.pstride * g.planes;
  if (cells % CW == 0 && ((uintptr_t)u & 15) == 0 && ((uintptr_t)gd & 15) == 0) {
    const long long nvec = cells / CW;
    const long long want = (nvec + NB - 1) / NB;
    const int nb = (int)(want < 148LL * 16 ? want : 148LL * 16);
    k_cd_gfield_vec<T><<<nb, NB, 0, s>>>(g, c, u, gd, nvec);
  } else {
    k_cd_gfield<T><<<grid_rows(g, g.nx), NB, 0, s>>>(g, c, u, gd);
  }
  return cudaGetLastError();
}
template <typename T>
cudaError_t cd_launch_jacobi(const Geom& g, const CdCoef<T>& c, const T* gd, const T* uin, const T* f, T* uout,
                             cudaStream_t s) {
  k_cd_jacobi<T><<<grid_rows(g, g.nx), NB, 0, s>>>(g, c, gd, uin, f, uout);
  return cudaGetLastError();
}
template <typename T>
cudaError_t cd_launch_rbgs(const Geom& g, const CdCoef<T>& c, const T* gd, T* u, const T* f, int colour,
                           cudaStream_t s) {
  k_cd_rbgs<T><<<grid_rows(g, (g.nx + 1) / 2), NB, 0, s>>>(g, c, gd, u, f, colour);
  return cudaGetLastError();
}
template <typename T>
cudaError_t cd_launch_restrict(const Geom& gf, const Geom& gc, const T* v, T* vh, T* vc, cudaStream_t s) {
  k_cd_restrict<T><<<grid_rows(gc, gc.nx), NB, 0, s>>>(gf, gc, v, vh, vc);
  return cudaGetLastError();
}
template <typename T>
cudaError_t cd_launch_fas_rhs(const Geom& gf, const Geom& gc, const CdCoef<T>& cf, const CdCoef<T>& cc, const T* gdf,
                              const T* uf, const T* ff, const T* gdc, const T* uh, T* fc, cudaStream_t s) {
  k_cd_fas_rhs<T><<<grid_rows(gc, gc.nx), NB, 0, s>>>(gf, gc, cf, cc, gdf, uf, ff, gdc, uh, fc);
  return cudaGetLastError();
}
template <typename T>
cudaError_t cd_launch_prolong(const Geom& gf, const Geom& gc, const T* uc, const T* uh, T* uf, cudaStream_t s) {
  k_cd_prolong<T><<<grid_rows(gf, gf.nx), NB, 0, s>>>(gf, gc, uc, uh, uf);
  return cudaGetLastError();
}
template <typename T>
cudaError_t cd_launch_residual(const Geom& g, const CdCoef<T>& c, const T* gd, const T* u, const T* f, T* r,
                               cudaStream_t s) {
  k_cd_residual<T><<<grid_rows(g, g.nx), NB, 0, s>>>(g, c, gd, u, f, r);
  return cudaGetLastError();
}
int cd_norm_partials(const Geom& g) { return grid_rows(g, g.nx); }
template <typename T>
cudaError_t cd_launch_norm_partial(const Geom& g, const CdCoef<T>& c, const T* gd, const T* u, const T* f,
                                   double* partial, int* npartial, cudaStream_t s) {
  const int nb = grid_rows(g, g.nx);
  *npartial = nb;
  if (gd)
    k_cd_norm<T, true><<<nb, NB, 0, s>>>(g, c, gd, u, f, partial);
  else
    k_cd_norm<T, false><<<nb, NB, 0, s>>>(g, c, gd, u, f, partial);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// coarse tail: the FAS recursion on levels lt..L-1 in one CTA (same per-cell code)
namespace {
constexpr int NTT = 1024;

template <typename T>
__device__ void tail_gfield(const Geom& g, const CdCoef<T>& c, const T* u, T* gd) {
  for_cells(g, [&](const Cell& x) { st(gd, x.q, diffusivity(c, u[2 * x.q + 1])); });
}

// one sweep; Jacobi returns the other buffer as the new current one
template <typename T>
__device__ T* tail_sweep(const Geom& g, const CdCoef<T>& c, int rbgs, const T* gd, T* u, T* t, const T* f) {
  if (!rbgs) {
    for_cells(g, [&](const Cell& x) { st(t, x.q, relax(g, c, gd, u, f, x)); });
    __syncthreads();
    return t;
  }
  for (int colour = 0; colour < 2; colour++) {
    for_cells_colour(g, colour, [&](const Cell& x) { st(u, x.q, relax(g, c, gd, u, f, x)); });
    __syncthreads();
  }
  return u;
}
}  // namespace

template <typename T>
__global__ void __launch_bounds__(NTT, 1) k_cd_tail(const __grid_constant__ CdTail<T> P) {
  T* cur[kCdTailMax];
  T* oth[kCdTailMax];
  for (int k = 0; k < P.nl; k++) {
    cur[k] = P.u[k];
    oth[k] = P.t[k];
  }
  if (!P.g_ready) {
    tail_gfield(P.g[0], P.c[0], cur[0], P.gd[0]);
    __syncthreads();
  }
  const int last = P.nl - 1;
  // descend: pre-smoothing, u^ = R u, coarse g, FAS right-hand side
  for (int k = 0; k < last; k++) {
    const Geom &G = P.g[k], &H = P.g[k + 1];
    const T* f = P.f[k];
    for (int s = 0; s < P.nu1; s++) {
      T* nw = tail_sweep(G, P.c[k], P.rbgs, P.gd[k], cur[k], oth[k], f);
      if (nw != cur[k]) {
        oth[k] = cur[k];
        cur[k] = nw;
      }
    }
    const T* ul = cur[k];
    T* uck = cur[k + 1];
    for_cells(H, [&](const Cell& X) {
      const C2<T> o = average_children<T>(G, X, [&](const Cell& a) { return ld(ul, a.q); });
      st(P.uh[k + 1], X.q, o);
      st(uck, X.q, o);
      st(P.gd[k + 1], X.q, diffusivity(P.c[k + 1], o.im));
    });
    __syncthreads();
    for_cells(H, [&](const Cell& X) {
      const C2<T> Rr = average_children<T>(G, X, [&](const Cell& a) {
        C2<T> d;
        const C2<T> Au = apply(G, P.c[k], Stored<T>{P.gd[k]}, ul, a, d);
        const C2<T> fv = ld(f, a.q);
        return C2<T>{sub(fv.re, Au.re), sub(fv.im, Au.im)};
      });
      C2<T> d;
      const C2<T> AH = apply(H, P.c[k + 1], Stored<T>{P.gd[k + 1]}, P.uh[k + 1], X, d);
      st(P.f[k + 1], X.q, C2<T>{add(AH.re, Rr.re), add(AH.im, Rr.im)});
    });
    __syncthreads();
  }
  // coarsest: ncoarse sweeps
  for (int s = 0; s < P.ncoarse; s++) {
    T* nw = tail_sweep(P.g[last], P.c[last], P.rbgs, P.gd[last], cur[last], oth[last], P.f[last]);
    if (nw != cur[last]) {
      oth[last] = cur[last];
      cur[last] = nw;
    }
  }
  // ascend: u += P(u_H - u^_H), post-smoothing
  for (int k = last - 1; k >= 0; k--) {
    const Geom &G = P.g[k], &H = P.g[k + 1];
    const T* ucn = cur[k + 1];
    const T* uhk = P.uh[k + 1];
    T* uk = cur[k];
    for_cells(G, [&](const Cell& x) {
      const long long Q =
          (long long)(x.k >> 1) * H.pstride + (long long)(G.three_d ? (x.j >> 1) : 0) * H.pitch + (x.i >> 1);
      const C2<T> a = ld(ucn, Q), h = ld(uhk, Q);
      const C2<T> u = ld(uk, x.q);
      st(uk, x.q, C2<T>{add(u.re, sub(a.re, h.re)), add(u.im, sub(a.im, h.im))});
    });
    __syncthreads();
    for (int s = 0; s < P.nu2; s++) {
      T* nw = tail_sweep(G, P.c[k], P.rbgs, P.gd[k], cur[k], oth[k], P.f[k]);
      if (nw != cur[k]) {
        oth[k] = cur[k];
        cur[k] = nw;
      }
    }
  }
  if (cur[0] != P.u[0]) {  // the result belongs in the top level's u
    const T* c0 = cur[0];
    T* u0 = P.u[0];
    for_cells(P.g[0], [&](const Cell& x) { st(u0, x.q, ld(c0, x.q)); });
  }
}

template <typename T>
cudaError_t cd_launch_tail(const CdTail<T>& p, cudaStream_t s) {
  k_cd_tail<T><<<1, NTT, 0, s>>>(p);
  return cudaGetLastError();
}
template <typename T>
cudaError_t cd_launch_fill(const Geom& g, T* dst, uint64_t seed, double lo, double hi, cudaStream_t s) {
  k_cd_fill<T><<<grid_rows(g, g.nx), NB, 0, s>>>(g, dst, seed, lo, hi);
  return cudaGetLastError();
}

#define CD_INST(T)                                                                                                   \
  template cudaError_t cd_launch_gfield<T>(const Geom&, const CdCoef<T>&, const T*, T*, cudaStream_t);              \
  template cudaError_t cd_launch_jacobi<T>(const Geom&, const CdCoef<T>&, const T*, const T*, const T*, T*,          \
                                           cudaStream_t);                                                            \
  template cudaError_t cd_launch_rbgs<T>(const Geom&, const CdCoef<T>&, const T*, T*, const T*, int, cudaStream_t); \
  template cudaError_t cd_launch_restrict<T>(const Geom&, const Geom&, const T*, T*, T*, cudaStream_t);              \
  template cudaError_t cd_launch_fas_rhs<T>(const Geom&, const Geom&, const CdCoef<T>&, const CdCoef<T>&, const T*, \
                                            const T*, const T*, const T*, const T*, T*, cudaStream_t);               \
  template cudaError_t cd_launch_prolong<T>(const Geom&, const Geom&, const T*, const T*, T*, cudaStream_t);         \
  template cudaError_t cd_launch_residual<T>(const Geom&, const CdCoef<T>&, const T*, const T*, const T*, T*,        \
                                             cudaStream_t);                                                          \
  template cudaError_t cd_launch_norm_partial<T>(const Geom&, const CdCoef<T>&, const T*, const T*, const T*, double*, \
                                                 int*, cudaStream_t);                                                \
  template cudaError_t cd_launch_tail<T>(const CdTail<T>&, cudaStream_t);                                           \
  template cudaError_t cd_launch_fill<T>(const Geom&, T*, uint64_t, double, double, cudaStream_t);
CD_INST(float)
CD_INST(double)
#undef CD_INST

}  // namespace mg
