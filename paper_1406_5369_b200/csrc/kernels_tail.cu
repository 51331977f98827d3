// kernels_tail.cu — the coarse tail of the V-cycle in ONE launch.
//
// Levels below a size threshold are pure latency (each op-by-op pass is a few
// microseconds of launch and barrier for a few thousand nodes).  k_tail runs
// V_lt(0, f_lt) — every operation of Alg. 1 on levels lt..L-1:
// pre-smoothing, residual + full weighting, the coarsest solve, prolongation +
// correction, post-smoothing — inside ONE thread-block cluster (16 CTAs x 1024
// threads, one per SM), a cluster barrier (barrier.cluster release/acquire,
// ~0.2 us) between passes, data in global memory (L2 resident).  The
// per-node arithmetic is the same canonical device code as every other kernel
// (mg_common.cuh), so results are bitwise identical to the op-by-op schedule.
// With lt = 0 (small 2D grids such as C1) the whole cycle is one launch.
#include <cstdlib>

#include "kernels.h"
#include "kernels_tail.h"
#include "launch_util.h"

namespace mg {

namespace {

constexpr int NTT = 1024;

// all CTAs of the cluster (= the grid): release/acquire at cluster scope makes the
// pass's global writes visible to the next pass (and invalidates L1)
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Work distribution of a pass.  A SOLO level (a few thousand nodes) runs on CTA 0 alone with
// block barriers — a block barrier costs a fraction of a cluster barrier and the level's work
// is too small to pay for 16 SMs; the other CTAs skip solo passes entirely and meet CTA 0 at
// the next cluster barrier (the transitions in k_tail).
struct Mode {
  bool solo;
  __device__ bool active() const { return !solo || blockIdx.x == 0; }
  __device__ int start() const { return solo ? (int)threadIdx.x : (int)(blockIdx.x * NTT + threadIdx.x); }
  __device__ int stride() const { return solo ? NTT : (int)(gridDim.x * NTT); }
  __device__ void sync() const {
    if (!solo)
      cluster_sync();
    else if (blockIdx.x == 0)
      __syncthreads();
  }
};

struct Idx {
  int i, j, pl;
};

// interior node number q -> (i, j, plane)
__device__ __forceinline__ Idx interior_node(const Geom& g, int q) {
  const int ni = g.nx - 1;
  const int nr = g.three_d ? g.ny - 1 : 1;
  Idx d;
  d.i = 1 + q % ni;
  const int t = q / ni;
  d.j = g.three_d ? 1 + t % nr : 0;
  d.pl = g.p_lo + t / nr;
  return d;
}
__device__ __forceinline__ int interior_count(const Geom& g) {
  return (g.nx - 1) * (g.three_d ? g.ny - 1 : 1) * (g.p_hi - g.p_lo);
}
__device__ __forceinline__ long long lin(const Geom& g, int i, int j, int pl) {
  return (long long)pl * g.pstride + (long long)j * g.pitch + i;
}

template <typename T>
__device__ void zero_level(const Mode& M, const Geom& g, T* u) {
  if (!M.active()) return;
  const long long n = (long long)g.planes * g.pstride;
  for (long long q = M.start(); q < n; q += M.stride()) u[q] = (T)0;
}

// one sweep of the smoother; Jacobi ping-pongs (returns the new current buffer)
template <typename T>
__device__ T* sweep(const Mode& M, const Geom& g, const Coef<T>& c, int rbgs, T* u, T* t, const T* f) {
  const bool act = M.active();
  const int n = interior_count(g);
  if (rbgs == 2) {  // lexicographic omega-GS: hyperplanes i + j + global plane = s in order
    const int nj = g.three_d ? g.ny - 1 : 1;
    const int m = nj * (g.p_hi - g.p_lo);
    const int smin = 1 + (g.three_d ? 1 : 0) + g.p_lo + g.p_glob0;
    const int smax = (g.nx - 1) + (g.three_d ? g.ny - 1 : 0) + g.p_hi - 1 + g.p_glob0;
    for (int s = smin; s <= smax; s++) {
      for (int q = act ? M.start() : m; q < m; q += M.stride()) {
        const int j = g.three_d ? 1 + q % nj : 0;
        const int pl = g.p_lo + q / nj;
        const int i = s - j - (pl + g.p_glob0);
        if (i < 1 || i > g.nx - 1) continue;
        const long long p = lin(g, i, j, pl);
        u[p] = add(u[p], mul(c.wd, point_residual(u, p, g, c, f[p])));
      }
      M.sync();
    }
    return u;
  }
  if (rbgs) {
    for (int colour = 0; colour < 2; colour++) {
      for (int q = act ? M.start() : n; q < n; q += M.stride()) {
        const Idx d = interior_node(g, q);
        if (((d.i + d.j + d.pl + g.p_glob0) & 1) != colour) continue;
        const long long p = lin(g, d.i, d.j, d.pl);
        u[p] = add(u[p], mul(c.wd, point_residual(u, p, g, c, f[p])));
      }
      M.sync();
    }
    return u;
  }
  for (int q = act ? M.start() : n; q < n; q += M.stride()) {
    const Idx d = interior_node(g, q);
    const long long p = lin(g, d.i, d.j, d.pl);
    t[p] = add(u[p], mul(c.wd, point_residual(u, p, g, c, f[p])));
  }
  M.sync();
  return t;
}

template <typename T>
__device__ void residual(const Mode& M, const Geom& g, const Coef<T>& c, const T* u, const T* f, T* r) {
  const bool act = M.active();
  const int n = interior_count(g);
  for (int q = act ? M.start() : n; q < n; q += M.stride()) {
    const Idx d = interior_node(g, q);
    const long long p = lin(g, d.i, d.j, d.pl);
    r[p] = point_residual(u, p, g, c, f[p]);
  }
  M.sync();
}

// full weighting, separable x -> y -> plane axis (reading 13)
template <typename T>
__device__ void restrict_fw(const Mode& M, const Geom& gf, const Geom& gc, const T* r, T* fc) {
  const bool act = M.active();
  const int n = interior_count(gc);
  const T two = (T)2;
  const T scale = gc.three_d ? (T)(1.0 / 64.0) : (T)(1.0 / 16.0);
  for (int q = act ? M.start() : n; q < n; q += M.stride()) {
    const Idx d = interior_node(gc, q);
    const int pf = 2 * (d.pl + gc.p_glob0) - gf.p_glob0;
    T tz[3];
    for (int dz = -1; dz <= 1; dz++) {
      T ty;
      if (gc.three_d) {
        T tx[3];
        for (int dy = -1; dy <= 1; dy++) {
          const long long p = lin(gf, 2 * d.i, 2 * d.j + dy, pf + dz);
          tx[dy + 1] = add(add(r[p - 1], r[p + 1]), mul(two, r[p]));
        }
        ty = add(add(tx[0], tx[2]), mul(two, tx[1]));
      } else {
        const long long p = lin(gf, 2 * d.i, 0, pf + dz);
        ty = add(add(r[p - 1], r[p + 1]), mul(two, r[p]));
      }
      tz[dz + 1] = ty;
    }
    fc[lin(gc, d.i, d.j, d.pl)] = mul(add(add(tz[0], tz[2]), mul(two, tz[1])), scale);
  }
  M.sync();
}

// the first sweep from a zero iterate (V_H(0, ...)) without a zeroing pass: Jacobi writes
// t = 0 + wd (f - A 0) = 0 + wd f; RBGS's red pass writes 0 + wd f at red nodes and 0 at black
// nodes (the black pass then runs as usual).  With A 0 = D*0 - 0 = +0 and f - (+0) = f the
// values are bitwise those of a sweep over a zeroed array.
template <typename T>
__device__ T* sweep_from_zero(const Mode& M, const Geom& g, const Coef<T>& c, int rbgs, T* u, T* t, const T* f) {
  const bool act = M.active();
  const int n = interior_count(g);
  const T zero = (T)0;
  if (!rbgs) {
    for (int q = act ? M.start() : n; q < n; q += M.stride()) {
      const Idx d = interior_node(g, q);
      const long long p = lin(g, d.i, d.j, d.pl);
      t[p] = add(zero, mul(c.wd, sub(f[p], zero)));
    }
    M.sync();
    return t;
  }
  for (int q = act ? M.start() : n; q < n; q += M.stride()) {  // red pass (colour 0) + zero black nodes
    const Idx d = interior_node(g, q);
    const long long p = lin(g, d.i, d.j, d.pl);
    u[p] = ((d.i + d.j + d.pl + g.p_glob0) & 1) == 0 ? add(zero, mul(c.wd, sub(f[p], zero))) : zero;
  }
  M.sync();
  for (int q = act ? M.start() : n; q < n; q += M.stride()) {  // black pass
    const Idx d = interior_node(g, q);
    if (((d.i + d.j + d.pl + g.p_glob0) & 1) != 1) continue;
    const long long p = lin(g, d.i, d.j, d.pl);
    u[p] = add(u[p], mul(c.wd, point_residual(u, p, g, c, f[p])));
  }
  M.sync();
  return u;
}

// u += P e, separable x -> y -> plane axis
template <typename T>
__device__ void prolong(const Mode& M, const Geom& gf, const Geom& gc, const T* e, T* u) {
  const bool act = M.active();
  const int n = interior_count(gf);
  const T half = (T)0.5;
  for (int q = act ? M.start() : n; q < n; q += M.stride()) {
    const Idx d = interior_node(gf, q);
    const int pg = d.pl + gf.p_glob0;
    const int I = d.i >> 1, dx = d.i & 1;
    const int J = d.j >> 1, dy = gf.three_d ? (d.j & 1) : 0;
    const int P = (pg >> 1) - gc.p_glob0, dz = pg & 1;
    T vy[2];
    for (int zz = 0; zz <= dz; zz++) {
      T vx[2];
      for (int yy = 0; yy <= dy; yy++) {
        const long long p = lin(gc, I, J + yy, P + zz);
        vx[yy] = dx ? mul(half, add(e[p], e[p + 1])) : e[p];
      }
      vy[zz] = dy ? mul(half, add(vx[0], vx[1])) : vx[0];
    }
    const T v = dz ? mul(half, add(vy[0], vy[1])) : vy[0];
    const long long p = lin(gf, d.i, d.j, d.pl);
    u[p] = add(u[p], v);
  }
  M.sync();
}

template <typename T>
__global__ void __launch_bounds__(NTT, 1) k_tail(TailParams<T> P) {
  auto mode = [&](int k) { return Mode{k >= P.solo_from}; };
  // ---- descend
  T* cur[kTailMax];
  for (int k = 0; k < P.nl; k++) cur[k] = P.u[k];
  for (int k = 0; k < P.nl - 1; k++) {
    const Geom& g = P.g[k];
    const Mode M = mode(k);
    const bool zero = k > 0 || P.zero_first;  // V_H(0, ...)
    const bool fold = zero && P.nu1 > 0 && P.rbgs != 2;  // the zero guess folded into the first sweep
    if (zero && !fold) {
      zero_level(M, g, cur[k]);
      M.sync();
    }
    for (int s = 0; s < P.nu1; s++) {
      T* oth = cur[k] == P.u[k] ? P.t[k] : P.u[k];
      cur[k] = (s == 0 && fold) ? sweep_from_zero(M, g, P.c[k], P.rbgs, cur[k], oth, P.f[k])
                                : sweep(M, g, P.c[k], P.rbgs, cur[k], oth, P.f[k]);
    }
    // separate residual and restriction passes: measured faster than one fused pass whose
    // coarse threads each evaluate 3^d fine residuals (latency-bound serial chains)
    residual(M, g, P.c[k], cur[k], P.f[k], P.r[k]);
    // the restriction writes level k+1: its mode (a solo coarse level is restricted by CTA 0,
    // reading the residual the cluster barrier above made visible)
    restrict_fw(mode(k + 1), g, P.g[k + 1], P.r[k], P.f[k + 1]);
  }
  // ---- coarsest level (Alg. 1 line 2)
  {
    const int k = P.nl - 1;
    const Geom& g = P.g[k];
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
        T* oth = cur[k] == P.u[k] ? P.t[k] : P.u[k];
        cur[k] = (s == 0 && fold) ? sweep_from_zero(M, g, P.c[k], P.rbgs, cur[k], oth, P.f[k])
                                  : sweep(M, g, P.c[k], P.rbgs, cur[k], oth, P.f[k]);
      }
    } else {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        // same loop order as k_coarse_direct / the oracle
        const int jlo = g.three_d ? 1 : 0, jhi = g.three_d ? g.ny - 1 : 0;
        const int m = P.m;
        const double* L = P.chol;
        if (m == 1) {
          const long long p = lin(g, 1, jlo, g.p_lo);
          cur[k][p] = (T)__ddiv_rn((double)P.f[k][p], P.D_coarse);
        } else {
          double* y = P.work;
          int q = 0;
          for (int pl = g.p_lo; pl < g.p_hi; pl++)
            for (int j = jlo; j <= jhi; j++)
              for (int i = 1; i < g.nx; i++) y[q++] = (double)P.f[k][lin(g, i, j, pl)];
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
    const Geom& g = P.g[k];
    const Mode M = mode(k);
    if (mode(k + 1).solo && !M.solo) cluster_sync();  // CTA 0's solo levels visible to every CTA
    prolong(M, g, P.g[k + 1], cur[k + 1], cur[k]);
    for (int s = 0; s < P.nu2; s++)
      cur[k] = sweep(M, g, P.c[k], P.rbgs, cur[k], cur[k] == P.u[k] ? P.t[k] : P.u[k], P.f[k]);
  }
  // result of the top tail level in u[0]
  if (cur[0] != P.u[0]) {
    const Mode M = mode(0);
    const bool act = M.active();
    const Geom& g = P.g[0];
    const int n = interior_count(g);
    for (int q = act ? M.start() : n; q < n; q += M.stride()) {
      const Idx d = interior_node(g, q);
      const long long p = lin(g, d.i, d.j, d.pl);
      P.u[0][p] = cur[0][p];
    }
  }
}

}  // namespace

template <typename T>
cudaError_t launch_tail(const TailParams<T>& p, cudaStream_t st) {
  // 16 CTAs (non-portable) where allowed, else the portable 8; probed once per device (the
  // non-portable opt-in is a per-device function attribute)
  const int cluster = per_device_once((const void*)k_tail<T>, [] {
    int c = 8;
    if (cudaFuncSetAttribute(k_tail<T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(16);
      q.blockDim = dim3(NTT);
      cudaLaunchAttribute a;
      a.id = cudaLaunchAttributeClusterDimension;
      a.val.clusterDim.x = 16;
      a.val.clusterDim.y = 1;
      a.val.clusterDim.z = 1;
      q.attrs = &a;
      q.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, k_tail<T>, &q) == cudaSuccess && n >= 1) c = 16;
    }
    cudaGetLastError();
    return c;
  });
  // tiny tails (a few thousand nodes, e.g. the whole 65^2 C1 hierarchy) run faster on one CTA
  const Geom& g0 = p.g[0];
  const long long top = (long long)(g0.nx - 1) * (g0.three_d ? g0.ny - 1 : 1) * (g0.p_hi - g0.p_lo);
  const int csize = top <= 8192 ? 1 : cluster;
  // levels from solo_from on run on CTA 0 alone with block barriers (all of them on one CTA)
  constexpr long long solo_max = 2048;  // measured: threshold scan 512-8192
  TailParams<T> q = p;
  q.solo_from = p.nl;
  for (int k = 0; k < p.nl; k++) {
    const Geom& g = p.g[k];
    const long long n = (long long)(g.nx - 1) * (g.three_d ? g.ny - 1 : 1) * (g.p_hi - g.p_lo);
    if (csize == 1 || n <= solo_max) {
      q.solo_from = k;
      break;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(csize);
  cfg.blockDim = dim3(NTT);
  cfg.stream = st;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = csize;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = csize > 1 ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_tail<T>, q);
}

template cudaError_t launch_tail<double>(const TailParams<double>&, cudaStream_t);
template cudaError_t launch_tail<float>(const TailParams<float>&, cudaStream_t);

}  // namespace mg
