// kernels_cd.h — complex-diffusion FAS kernels on cell-centred levels (kernels_cd.cu).
//
// A cell-centred level reuses Geom with cells instead of nodes: nx = cells along x,
// ny = cells along the in-plane y (3D), nz = cells along the plane axis (3D z, 2D
// the paper's y), planes = nz, rows = ny (3D) / 1 (2D), p_lo = 0, p_hi = nz; pitch
// and pstride count COMPLEX elements, stored (re, im) interleaved.  No ghost cells:
// boundary faces are dropped from the stencil (zero flux).
#pragma once
#include "mg_common.cuh"

namespace mg {

template <typename T>
struct CdCoef {
  T w[3];      // tau / h_d^2 for x, in-plane y (3D; 0 in 2D), plane axis
  T omega;
  T kth;       // k * theta (Eq. 3)
  T ct, st;    // cos(theta), sin(theta), computed in double on the host and cast once
};

template <typename T>
cudaError_t cd_launch_gfield(const Geom& g, const CdCoef<T>& c, const T* u, T* gd, cudaStream_t st);
template <typename T>
cudaError_t cd_launch_jacobi(const Geom& g, const CdCoef<T>& c, const T* gd, const T* uin, const T* f, T* uout,
                             cudaStream_t st);
template <typename T>
cudaError_t cd_launch_rbgs(const Geom& g, const CdCoef<T>& c, const T* gd, T* u, const T* f, int colour,
                           cudaStream_t st);
// vh = R v (cell average); also vc = vh when vc != nullptr
template <typename T>
cudaError_t cd_launch_restrict(const Geom& gf, const Geom& gc, const T* v, T* vh, T* vc, cudaStream_t st);
// fc = A_c(gdc) uh + R(ff - A_f(gdf) uf)   (FAS coarse right-hand side)
template <typename T>
cudaError_t cd_launch_fas_rhs(const Geom& gf, const Geom& gc, const CdCoef<T>& cf, const CdCoef<T>& cc, const T* gdf,
                              const T* uf, const T* ff, const T* gdc, const T* uh, T* fc, cudaStream_t st);
// uf += P(uc - uh) (constant injection); uh == nullptr: uf += P uc
template <typename T>
cudaError_t cd_launch_prolong(const Geom& gf, const Geom& gc, const T* uc, const T* uh, T* uf, cudaStream_t st);
// r = f - A(gd) u
template <typename T>
cudaError_t cd_launch_residual(const Geom& g, const CdCoef<T>& c, const T* gd, const T* u, const T* f, T* r,
                               cudaStream_t st);
// partial sums of |f - A(g(u)) u|^2, one double per block; g read from gd (which must hold
// g(u)) or, when gd == nullptr, evaluated from u on the fly
template <typename T>
cudaError_t cd_launch_norm_partial(const Geom& g, const CdCoef<T>& c, const T* gd, const T* u, const T* f,
                                   double* partial, int* npartial, cudaStream_t st);
int cd_norm_partials(const Geom& g);
// The coarse tail of the FAS cycle: levels lt..L-1 (k = 0 .. nl-1) in ONE single-CTA launch
// (latency-bound levels; every pass of the recursion separated by __syncthreads).
constexpr int kCdTailMax = 12;
constexpr int kCdTailCells = 4096;  // the top tail level has at most this many cells
template <typename T>
struct CdTail {
  int nl;
  int rbgs, nu1, nu2, ncoarse;
  int g_ready;  // the top level's g field is already g(u_top)
  Geom g[kCdTailMax];
  CdCoef<T> c[kCdTailMax];
  T* u[kCdTailMax];
  T* f[kCdTailMax];
  T* uh[kCdTailMax];
  T* gd[kCdTailMax];
  T* t[kCdTailMax];
};
template <typename T>
cudaError_t cd_launch_tail(const CdTail<T>& p, cudaStream_t st);

// 2D warp-marching Jacobi sweep (kernels_cd2d.cu), bitwise equal to cd_launch_jacobi
bool cd2d_supported(const Geom& g);
template <typename T>
cudaError_t cd2d_launch_jacobi(const Geom& g, const CdCoef<T>& c, const T* gd, const T* uin, const T* f, T* uout,
                               cudaStream_t st);

// its residual-norm variant (g = g(u) stored): partial sums of |f - A u|^2, one per CTA
template <typename T>
int cd2d_norm_partials(const Geom& g);
template <typename T>
cudaError_t cd2d_launch_norm(const Geom& g, const CdCoef<T>& c, const T* gd, const T* u, const T* f,
                             double* partial, int* npartial, cudaStream_t st);
// K (1..3 FP32, 1..2 FP64) omega-Jacobi sweeps with the frozen g in one pass (temporal
// blocking), bitwise equal to K cd2d_launch_jacobi sweeps; partial != nullptr: also the
// partials of |f - A(g) uin|^2 (*npartial of them, at most cd2d_kpartials)
template <typename T>
cudaError_t cd2d_launch_jacobi_k(const Geom& g, const CdCoef<T>& c, int K, const T* gd, const T* uin, const T* f,
                                 T* uout, cudaStream_t st, double* partial = nullptr, int* npartial = nullptr);
template <typename T>
int cd2d_kpartials(const Geom& g);

// 3D plane-marching Jacobi sweep and stored-g residual norm (kernels_cd3d.cu), bitwise equal to
// cd_launch_jacobi / the partials of cd_launch_norm_partial's sum
bool cd3d_supported(const Geom& g);
template <typename T>
cudaError_t cd3d_launch_jacobi(const Geom& g, const CdCoef<T>& c, const T* gd, const T* uin, const T* f, T* uout,
                               cudaStream_t st);
template <typename T>
int cd3d_norm_partials(const Geom& g);
template <typename T>
cudaError_t cd3d_launch_norm(const Geom& g, const CdCoef<T>& c, const T* gd, const T* u, const T* f,
                             double* partial, int* npartial, cudaStream_t st);

// W5 inputs: re = lo + (hi-lo) U[0,1)(global cell index), im = 0
template <typename T>
cudaError_t cd_launch_fill(const Geom& g, T* dst, uint64_t seed, double lo, double hi, cudaStream_t st);

}  // namespace mg
