// kernels_baseline.cu — op-by-op level operators, one thread per node.
//
// These are the straightforward data-parallel forms of each step of Alg. 1
// (P:187-219): used for coarse levels (where a launch is latency-bound and
// the level fits in L2) and, with MG_FLAG_BASELINE, for every level — the
// "paper-style" schedule (one kernel per operation, RBGS as two colour
// passes) that the fused plane-marching kernels are measured
// against.  Arithmetic follows the canonical order of mg_common.cuh.
#include <cstdio>

#include "kernels.h"

namespace mg {

namespace {

constexpr int BX = 64, BY = 4;

// Interior nodes of a level enumerated as (i, q) with q = plane-major index
// over the interior (row, plane) pairs.
struct Interior {
  int ni;      // interior nodes along x
  int nrow;    // interior rows per plane (3D: ny-1, 2D: 1)
  int nplane;  // planes to update
};

__host__ __device__ inline Interior interior_of(const Geom& g) {
  Interior it;
  it.ni = g.nx - 1;
  it.nrow = g.three_d ? g.ny - 1 : 1;
  it.nplane = g.p_hi - g.p_lo;
  return it;
}

// Map (blockIdx, threadIdx) to a node; returns false when outside the interior.
__device__ __forceinline__ bool node_of(const Geom& g, int& i, int& j, int& pl) {
  Interior it = interior_of(g);
  i = 1 + blockIdx.y * BX + threadIdx.x;
  long long q = (long long)blockIdx.x * BY + threadIdx.y;
  if (i > it.ni || q >= (long long)it.nrow * it.nplane) return false;
  int jr = (int)(q % it.nrow);
  pl = g.p_lo + (int)(q / it.nrow);
  j = g.three_d ? jr + 1 : 0;
  return true;
}

__device__ __forceinline__ long long lin(const Geom& g, int i, int j, int pl) {
  return (long long)pl * g.pstride + (long long)j * g.pitch + i;
}

inline dim3 grid_of(const Geom& g) {
  Interior it = interior_of(g);
  long long q = (long long)it.nrow * it.nplane;
  return dim3((unsigned)((q + BY - 1) / BY), (it.ni + BX - 1) / BX, 1);  // x: rows (may exceed 65535)
}

inline bool empty(const Geom& g) {
  Interior it = interior_of(g);
  return it.ni <= 0 || it.nrow <= 0 || it.nplane <= 0;
}

// ---- omega-Jacobi sweep (double-buffered, reading 9) ----------------
template <typename T>
__global__ void __launch_bounds__(BX* BY) k_jacobi(Geom g, Coef<T> c, const T* __restrict__ uin,
                                                   const T* __restrict__ f, T* __restrict__ uout) {
  int i, j, pl;
  if (!node_of(g, i, j, pl)) return;
  long long p = lin(g, i, j, pl);
  T r = point_residual(uin, p, g, c, f[p]);
  uout[p] = add(uin[p], mul(c.wd, r));
}

// ---- one colour of red-black Gauss-Seidel, in place (listing P:299-305) ----
template <typename T>
__global__ void __launch_bounds__(BX* BY) k_rbgs_colour(Geom g, Coef<T> c, T* __restrict__ u,
                                                        const T* __restrict__ f, int colour) {
  int i, j, pl;
  if (!node_of(g, i, j, pl)) return;
  if (((i + j + pl + g.p_glob0) & 1) != colour) return;  // global parity (reading 8)
  long long p = lin(g, i, j, pl);
  T r = point_residual(u, p, g, c, f[p]);
  u[p] = add(u[p], mul(c.wd, r));
}

// ---- lexicographic omega-GS (Table 1; "order lex"): one hyperplane
// i + j + global plane = s per launch.  Every node's lower neighbours lie on the
// previous hyperplane (already new), its upper ones on the next (still old), so
// the sweep over s = min..max reproduces the row-major sequential sweep exactly.
template <typename T>
__global__ void __launch_bounds__(256) k_gs_lex_plane(Geom g, Coef<T> c, T* __restrict__ u,
                                                      const T* __restrict__ f, int s) {
  const int nj = g.three_d ? g.ny - 1 : 1;
  const int q = blockIdx.x * 256 + threadIdx.x;
  if (q >= nj * (g.p_hi - g.p_lo)) return;
  const int j = g.three_d ? 1 + q % nj : 0;
  const int pl = g.p_lo + q / nj;
  const int i = s - j - (pl + g.p_glob0);
  if (i < 1 || i > g.nx - 1) return;
  const long long p = lin(g, i, j, pl);
  u[p] = add(u[p], mul(c.wd, point_residual(u, p, g, c, f[p])));
}

// ---- residual r = f - A u (Alg. 1 line 4) ----------------------------------
template <typename T>
__global__ void __launch_bounds__(BX* BY) k_residual(Geom g, Coef<T> c, const T* __restrict__ u,
                                                     const T* __restrict__ f, T* __restrict__ r) {
  int i, j, pl;
  if (!node_of(g, i, j, pl)) return;
  long long p = lin(g, i, j, pl);
  r[p] = point_residual(u, p, g, c, f[p]);
}

// ---- full weighting f_H = R r_h --------------------
// Separable, x then y then plane axis: t = (r[-1] + r[+1]) + 2 r[0]; f = t * 4^-d.
template <typename T>
__global__ void __launch_bounds__(BX* BY) k_restrict(Geom gf, Geom gc, const T* __restrict__ r,
                                                     T* __restrict__ fc) {
  int I, J, P;
  if (!node_of(gc, I, J, P)) return;
  const T two = (T)2;
  int pf = 2 * (P + gc.p_glob0) - gf.p_glob0;  // fine local plane of coarse plane P
  int jf = 2 * J;
  T tz[3];
#pragma unroll
  for (int dz = -1; dz <= 1; dz++) {
    T ty;
    if (gc.three_d) {
      T tx[3];
#pragma unroll
      for (int dy = -1; dy <= 1; dy++) {
        long long q = lin(gf, 2 * I, jf + dy, pf + dz);
        tx[dy + 1] = add(add(r[q - 1], r[q + 1]), mul(two, r[q]));
      }
      ty = add(add(tx[0], tx[2]), mul(two, tx[1]));
    } else {
      long long q = lin(gf, 2 * I, 0, pf + dz);
      ty = add(add(r[q - 1], r[q + 1]), mul(two, r[q]));
    }
    tz[dz + 1] = ty;
  }
  T t = add(add(tz[0], tz[2]), mul(two, tz[1]));
  const T scale = gc.three_d ? (T)(1.0 / 64.0) : (T)(1.0 / 16.0);
  fc[lin(gc, I, J, P)] = mul(t, scale);
}

// ---- bi-/trilinear prolongation + correction u += P e ---
template <typename T>
__global__ void __launch_bounds__(BX* BY) k_prolong_correct(Geom gf, Geom gc, const T* __restrict__ e,
                                                            T* __restrict__ u) {
  int i, j, pl;
  if (!node_of(gf, i, j, pl)) return;
  const T half = (T)0.5;
  int pg = pl + gf.p_glob0;
  int I = i >> 1, dx = i & 1;
  int J = j >> 1, dy = gf.three_d ? (j & 1) : 0;
  int P = (pg >> 1) - gc.p_glob0, dz = pg & 1;
  T vy[2];
#pragma unroll
  for (int zz = 0; zz < 2; zz++) {
    if (zz > dz) break;
    T vx[2];
#pragma unroll
    for (int yy = 0; yy < 2; yy++) {
      if (yy > dy) break;
      long long q = lin(gc, I, J + yy, P + zz);
      vx[yy] = dx ? mul(half, add(e[q], e[q + 1])) : e[q];
    }
    vy[zz] = dy ? mul(half, add(vx[0], vx[1])) : vx[0];
  }
  T v = dz ? mul(half, add(vy[0], vy[1])) : vy[0];
  long long p = lin(gf, i, j, pl);
  u[p] = add(u[p], v);
}

// ---- copy the boundary nodes of the local planes (ping-pong buffers) -------
// One thread per boundary node, enumerated as: (A) whole boundary planes,
// (B) boundary rows of interior planes (3D), (C) the two x-ends of interior rows.
template <typename T>
__global__ void k_copy_boundary(Geom g, const T* __restrict__ src, T* __restrict__ dst, int nplanes) {
  const long long nxn = g.nx + 1;
  const int irows = g.three_d ? g.ny - 1 : 1;  // interior rows per plane
  const int rlo = g.three_d ? 1 : 0;
  // local planes holding global boundary planes
  const int pb0 = 0 - g.p_glob0, pb1 = g.nz - g.p_glob0;
  const bool has0 = pb0 >= 0 && pb0 < nplanes, has1 = pb1 >= 0 && pb1 < nplanes;
  const long long nA = (long long)((has0 ? 1 : 0) + (has1 ? 1 : 0)) * g.rows * nxn;
  const int iplanes = g.p_hi - g.p_lo;  // interior planes
  const long long nB = g.three_d ? (long long)iplanes * 2 * nxn : 0;
  const long long nC = (long long)iplanes * irows * 2;
  const long long n = nA + nB + nC;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    long long off;
    if (t < nA) {
      const long long per = (long long)g.rows * nxn;
      const int which = (int)(t / per);
      const long long rem = t - which * per;
      const int pl = (which == 0 && has0) ? pb0 : pb1;
      off = (long long)pl * g.pstride + (rem / nxn) * g.pitch + rem % nxn;
    } else if (t < nA + nB) {
      const long long q = t - nA;
      const long long per = 2 * nxn;
      const int pl = g.p_lo + (int)(q / per);
      const long long rem = q % per;
      const int row = rem < nxn ? 0 : g.ny;
      off = (long long)pl * g.pstride + (long long)row * g.pitch + rem % nxn;
    } else {
      const long long q = t - nA - nB;
      const long long rr = q >> 1;
      const int pl = g.p_lo + (int)(rr / irows);
      const int row = rlo + (int)(rr % irows);
      off = (long long)pl * g.pstride + (long long)row * g.pitch + ((q & 1) ? g.nx : 0);
    }
    dst[off] = src[off];
  }
}

// ---- deterministic residual norm: fixed blocks, fixed tree ------------------
constexpr int NB = 256;  // threads per norm block
constexpr int NORM_ROWS = 4;  // (row,plane) pairs per norm block

template <typename T>
__global__ void __launch_bounds__(NB) k_norm_partial(Geom g, Coef<T> c, const T* __restrict__ u,
                                                     const T* __restrict__ f, double* __restrict__ partial) {
  Interior it = interior_of(g);
  long long q0 = (long long)blockIdx.x * NORM_ROWS;
  long long nq = (long long)it.nrow * it.nplane;
  double s = 0.0;
  for (int rr = 0; rr < NORM_ROWS; rr++) {
    long long q = q0 + rr;
    if (q >= nq) break;
    int j = g.three_d ? (int)(q % it.nrow) + 1 : 0;
    int pl = g.p_lo + (int)(q / it.nrow);
    for (int i = 1 + threadIdx.x; i <= it.ni; i += NB) {
      long long p = lin(g, i, j, pl);
      double r = (double)point_residual(u, p, g, c, f[p]);
      s = __dadd_rn(s, __dmul_rn(r, r));
    }
  }
  __shared__ double sh[NB / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < NB / 32; w++) t = __dadd_rn(t, sh[w]);
    partial[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) k_norm_final(const double* __restrict__ partial, int n,
                                                     double* __restrict__ out, int take_sqrt) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 1024) s = __dadd_rn(s, partial[i]);
  __shared__ double sh[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 32; w++) t = __dadd_rn(t, sh[w]);
    *out = take_sqrt ? __dsqrt_rn(t) : t;
  }
}

// sqrt of the rank sums added in rank order (identical on every rank)
__global__ void k_norm_combine(const double* __restrict__ sums, int P, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double t = 0.0;
  for (int p = 0; p < P; p++) t = __dadd_rn(t, sums[p]);
  *out = __dsqrt_rn(t);
}

// ---- coarsest direct solve (Alg. 1 line 2; reading 3) ------------
// Same loop order as the definition: Cholesky-Banachiewicz row by row, inner
// sums in increasing index, then forward and backward substitution.  One thread:
// the coarsest system has 1 (paper rule) to a few hundred unknowns.
__device__ __forceinline__ int unk_of(const Geom& g, int i, int j, int pl) {
  int mx = g.nx - 1, my = g.three_d ? g.ny - 1 : 1;
  int jr = g.three_d ? j - 1 : 0;
  return ((pl - g.p_lo) * my + jr) * mx + (i - 1);
}

__global__ void k_cholesky(Geom g, double cx, double cy, double cz, double D, double* __restrict__ L, int m,
                           int* status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  // assemble A into L (lower part used in place as A then overwritten row by row)
  for (long long q = 0; q < (long long)m * m; q++) L[q] = 0.0;
  // A[p][q] entries
  auto A = [&](int r, int s) -> double {
    if (r == s) return D;
    // decode r and s into (i,j,pl) offsets
    int mx = g.nx - 1, my = g.three_d ? g.ny - 1 : 1;
    int ir = r % mx, jr = (r / mx) % my, pr = r / (mx * my);
    int is = s % mx, js = (s / mx) % my, ps = s / (mx * my);
    int di = abs(ir - is), dj = abs(jr - js), dp = abs(pr - ps);
    if (di == 1 && dj == 0 && dp == 0) return -cx;
    if (g.three_d && di == 0 && dj == 1 && dp == 0) return -cy;
    if (di == 0 && dj == 0 && dp == 1) return -cz;
    return 0.0;
  };
  for (int i = 0; i < m; i++) {
    for (int j = 0; j <= i; j++) {
      double s = A(i, j);
      for (int k = 0; k < j; k++) s = __dsub_rn(s, __dmul_rn(L[(long long)i * m + k], L[(long long)j * m + k]));
      if (i == j) {
        if (!(s > 0.0)) { *status = 1; return; }
        L[(long long)i * m + i] = __dsqrt_rn(s);
      } else {
        L[(long long)i * m + j] = __ddiv_rn(s, L[(long long)j * m + j]);
      }
    }
  }
  *status = 0;
}

template <typename T>
__global__ void k_coarse_direct(Geom g, double D, const double* __restrict__ L, int m, const T* __restrict__ f,
                                T* __restrict__ e, double* __restrict__ y) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int jlo = g.three_d ? 1 : 0, jhi = g.three_d ? g.ny - 1 : 0;
  if (m == 1) {
    long long p = lin(g, 1, jlo, g.p_lo);
    e[p] = (T)__ddiv_rn((double)f[p], D);
    return;
  }
  for (int pl = g.p_lo; pl < g.p_hi; pl++)
    for (int j = jlo; j <= jhi; j++)
      for (int i = 1; i < g.nx; i++) y[unk_of(g, i, j, pl)] = (double)f[lin(g, i, j, pl)];
  for (int i = 0; i < m; i++) {
    double s = y[i];
    for (int k = 0; k < i; k++) s = __dsub_rn(s, __dmul_rn(L[(long long)i * m + k], y[k]));
    y[i] = __ddiv_rn(s, L[(long long)i * m + i]);
  }
  for (int i = m - 1; i >= 0; i--) {
    double s = y[i];
    for (int k = i + 1; k < m; k++) s = __dsub_rn(s, __dmul_rn(L[(long long)k * m + i], y[k]));
    y[i] = __ddiv_rn(s, L[(long long)i * m + i]);
  }
  for (int pl = g.p_lo; pl < g.p_hi; pl++)
    for (int j = jlo; j <= jhi; j++)
      for (int i = 1; i < g.nx; i++) e[lin(g, i, j, pl)] = (T)y[unk_of(g, i, j, pl)];
}

// ---- SplitMix64 workload generator (reading 10; NOT method arithmetic)
template <typename T>
__global__ void k_workload_fill(Geom g, uint64_t seed, double lo, double hi, T* __restrict__ dst, int nplanes) {
  long long q = (long long)blockIdx.x * blockDim.y + threadIdx.y;  // (plane,row)
  if (q >= (long long)nplanes * g.rows) return;
  int row = (int)(q % g.rows);
  int pl = (int)(q / g.rows);
  int pg = pl + g.p_glob0;
  for (int i = threadIdx.x; i <= g.nx; i += blockDim.x) {
    bool interior = i > 0 && i < g.nx && pg > 0 && pg < g.nz && (!g.three_d || (row > 0 && row < g.ny));
    double v = 0.0;
    if (interior) {
      unsigned long long idx = ((unsigned long long)pg * (unsigned long long)g.rows + row) * (g.nx + 1ull) + i;
      unsigned long long z = seed + (idx + 1ull) * 0x9E3779B97F4A7C15ull;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      z ^= z >> 31;
      double r = (double)(z >> 11) * 0x1.0p-53;
      v = (lo == 0.0 && hi == 1.0) ? r : __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), r));
    }
    dst[(long long)pl * g.pstride + (long long)row * g.pitch + i] = (T)v;
  }
}

}  // namespace

// ------------------------------------------------------------------ launchers
template <typename T>
cudaError_t launch_jacobi(const Geom& g, const Coef<T>& c, const T* uin, const T* f, T* uout, cudaStream_t st) {
  if (empty(g)) return cudaSuccess;
  k_jacobi<T><<<grid_of(g), dim3(BX, BY), 0, st>>>(g, c, uin, f, uout);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_rbgs_colour(const Geom& g, const Coef<T>& c, T* u, const T* f, int colour, cudaStream_t st) {
  if (empty(g)) return cudaSuccess;
  k_rbgs_colour<T><<<grid_of(g), dim3(BX, BY), 0, st>>>(g, c, u, f, colour);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_gs_lex_plane(const Geom& g, const Coef<T>& c, T* u, const T* f, int s, cudaStream_t st) {
  const int n = (g.three_d ? g.ny - 1 : 1) * (g.p_hi - g.p_lo);
  if (n <= 0) return cudaSuccess;
  k_gs_lex_plane<T><<<(n + 255) / 256, 256, 0, st>>>(g, c, u, f, s);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_residual(const Geom& g, const Coef<T>& c, const T* u, const T* f, T* r, cudaStream_t st) {
  if (empty(g)) return cudaSuccess;
  k_residual<T><<<grid_of(g), dim3(BX, BY), 0, st>>>(g, c, u, f, r);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_restrict(const Geom& gf, const Geom& gc, const T* r, T* fc, cudaStream_t st) {
  if (empty(gc)) return cudaSuccess;
  k_restrict<T><<<grid_of(gc), dim3(BX, BY), 0, st>>>(gf, gc, r, fc);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_prolong_correct(const Geom& gf, const Geom& gc, const T* e, T* u, cudaStream_t st) {
  if (empty(gf)) return cudaSuccess;
  k_prolong_correct<T><<<grid_of(gf), dim3(BX, BY), 0, st>>>(gf, gc, e, u);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_copy_boundary(const Geom& g, const T* src, T* dst, cudaStream_t st) {
  int nplanes = g.planes;
  k_copy_boundary<T><<<148 * 4, 256, 0, st>>>(g, src, dst, nplanes);
  return cudaGetLastError();
}
template <typename T>
int norm_num_partials(const Geom& g) {
  Interior it = interior_of(g);
  long long nq = (long long)it.nrow * it.nplane;
  return (int)((nq + NORM_ROWS - 1) / NORM_ROWS);
}
template <typename T>
cudaError_t launch_norm_partial(const Geom& g, const Coef<T>& c, const T* u, const T* f, double* partial,
                                cudaStream_t st) {
  int nb = norm_num_partials<T>(g);
  if (nb == 0 || empty(g)) return cudaSuccess;
  k_norm_partial<T><<<nb, NB, 0, st>>>(g, c, u, f, partial);
  return cudaGetLastError();
}
cudaError_t launch_norm_final(const double* partial, int n, double* out, cudaStream_t st, bool take_sqrt) {
  k_norm_final<<<1, 1024, 0, st>>>(partial, n, out, take_sqrt ? 1 : 0);
  return cudaGetLastError();
}
cudaError_t launch_norm_combine(const double* sums, int P, double* out, cudaStream_t st) {
  k_norm_combine<<<1, 32, 0, st>>>(sums, P, out);
  return cudaGetLastError();
}
cudaError_t launch_cholesky_factor(const Geom& g, double cx, double cy, double cz, double D, double* L, int m,
                                   int* status, cudaStream_t st) {
  k_cholesky<<<1, 32, 0, st>>>(g, cx, cy, cz, D, L, m, status);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_coarse_direct(const Geom& g, double D, const double* L, int m, const T* f, T* e, double* work,
                                 cudaStream_t st) {
  k_coarse_direct<T><<<1, 32, 0, st>>>(g, D, L, m, f, e, work);
  return cudaGetLastError();
}
template <typename T>
cudaError_t launch_workload_fill(const Geom& g, uint64_t seed, double lo, double hi, T* dst, cudaStream_t st) {
  int nplanes = g.planes;
  long long q = (long long)nplanes * g.rows;
  dim3 blk(128, 2);
  dim3 grd((unsigned)((q + 1) / 2));
  k_workload_fill<T><<<grd, blk, 0, st>>>(g, seed, lo, hi, dst, nplanes);
  return cudaGetLastError();
}

#define MG_INST(T)                                                                                           \
  template cudaError_t launch_jacobi<T>(const Geom&, const Coef<T>&, const T*, const T*, T*, cudaStream_t);  \
  template cudaError_t launch_rbgs_colour<T>(const Geom&, const Coef<T>&, T*, const T*, int, cudaStream_t);  \
  template cudaError_t launch_gs_lex_plane<T>(const Geom&, const Coef<T>&, T*, const T*, int, cudaStream_t); \
  template cudaError_t launch_residual<T>(const Geom&, const Coef<T>&, const T*, const T*, T*, cudaStream_t); \
  template cudaError_t launch_restrict<T>(const Geom&, const Geom&, const T*, T*, cudaStream_t);             \
  template cudaError_t launch_prolong_correct<T>(const Geom&, const Geom&, const T*, T*, cudaStream_t);      \
  template cudaError_t launch_copy_boundary<T>(const Geom&, const T*, T*, cudaStream_t);                     \
  template int norm_num_partials<T>(const Geom&);                                                            \
  template cudaError_t launch_norm_partial<T>(const Geom&, const Coef<T>&, const T*, const T*, double*,      \
                                              cudaStream_t);                                                 \
  template cudaError_t launch_coarse_direct<T>(const Geom&, double, const double*, int, const T*, T*, double*, \
                                               cudaStream_t);                                                \
  template cudaError_t launch_workload_fill<T>(const Geom&, uint64_t, double, double, T*, cudaStream_t);
MG_INST(float)
MG_INST(double)
#undef MG_INST

}  // namespace mg
