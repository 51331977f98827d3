// kernels_cd3d.cu — 2.5D plane-marching omega-Jacobi sweep (and its residual-norm variant)
// of the complex-diffusion operator on 3D cell-centred levels (the
// per-cell arithmetic of kernels_cd.cu relax(), reading 19).
//
// A CTA owns a tile of TX x TY cells (TX = 32 lanes x CW complex cells: 64 FP32 / 32 FP64;
// TY = 8 rows, one warp per row) and marches a z-chunk of planes.  Step q of a 4-slot TMA
// ring brings u(q+1) and g(q+1) — tile + a 1-cell ring in x and y — and f(q) (the arrays
// viewed as real arrays twice as wide; zero-filled outside).  Processing plane p reads the
// in-plane neighbours from the boxes of plane p and the z-neighbours from registers, so u,
// g and f are read from HBM once per sweep and u' written once (4 complex words per cell).
// Faces outside the domain (Neumann) are formed anyway and not accumulated (selv), i.e.
// the same operations as relax(): the output is bitwise that of k_cd_jacobi and of the
// oracle.
#include <cstdio>

#include "cd_common.cuh"
#include "kernels_cd.h"
#include "kernels_pm.h"
#include "launch_util.h"
#include "tma.cuh"
#include "vec.cuh"

namespace mg {
namespace cd3 {
using namespace cdk;

constexpr int TY = 8;  // tile rows = warps per CTA
constexpr int NT = 32 * TY;
constexpr int NS = 4;  // ring slots

template <typename T>
struct G {
  static constexpr int CW = 16 / (2 * (int)sizeof(T));  // complex cells per lane
  static constexpr int TX = 32 * CW;                    // tile width in cells
  static constexpr int BXR = 2 * (TX + 2 * CW);         // box row in reals: cells x0-CW .. x0+TX+CW
  static constexpr int UB = (BXR * (TY + 2) * (int)sizeof(T) + 127) / 128 * 128;  // u / g box bytes (ring rows)
  static constexpr int FB = (BXR * TY * (int)sizeof(T) + 127) / 128 * 128;        // f box bytes
  static constexpr int STEP = 2 * UB + FB;
  static constexpr int SMEM = NS * STEP + 128;  // + mbarriers
};

template <typename T>
using VT = Vec<T, 16 / sizeof(T)>;

template <typename T>
__device__ __forceinline__ C2<T> cell(const VT<T>& v, int j) {
  return {v.v[2 * j], v.v[2 * j + 1]};
}

// NORM: instead of the sweep, the partial sums of |f - A(g) u|^2 (FP64), one per CTA
template <typename T, bool NORM>
__global__ void __launch_bounds__(NT) k_cd_jacobi3d(const __grid_constant__ CUtensorMap tm_u,
                                                    const __grid_constant__ CUtensorMap tm_g,
                                                    const __grid_constant__ CUtensorMap tm_f, Geom g, CdCoef<T> c,
                                                    T* __restrict__ uout, int tiles_x, int ntiles, int zc, int nitems,
                                                    double* __restrict__ partial) {
  using V = VT<T>;
  using GG = G<T>;
  constexpr int CW = GG::CW, TX = GG::TX, BXR = GG::BXR;
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + NS * GG::STEP);
  const int tid = threadIdx.x, lane = tid & 31, ry = tid >> 5;
  if (tid == 0) {
    prefetch_tmap(&tm_u);
    prefetch_tmap(&tm_g);
    prefetch_tmap(&tm_f);
    for (int s = 0; s < NS; s++) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto Ub = [&](uint32_t n) { return reinterpret_cast<const T*>(sm + (n % NS) * GG::STEP); };
  auto Gb = [&](uint32_t n) { return reinterpret_cast<const T*>(sm + (n % NS) * GG::STEP + GG::UB); };
  auto Fb = [&](uint32_t n) { return reinterpret_cast<const T*>(sm + (n % NS) * GG::STEP + 2 * GG::UB); };
  const int bo = (ry + 1) * BXR + 2 * (CW + CW * lane);  // the lane's vector in a u / g box
  const int fo = ry * BXR + 2 * (CW + CW * lane);        // ... in an f box
  const T half = (T)0.5;
  uint32_t seq = 0;
  double nsum = 0.0;
  for (int k = blockIdx.x; k < nitems; k += gridDim.x) {
    const int tile = k % ntiles, pa = (k / ntiles) * zc, pb = min(pa + zc, g.nz);
    const int x0 = (tile % tiles_x) * TX, y0 = (tile / tiles_x) * TY;
    const int ox = x0 + CW * lane, oy = y0 + ry;
    bool own[CW], xm[CW], xp[CW];
    bool any = false;
#pragma unroll
    for (int j = 0; j < CW; j++) {
      own[j] = ox + j < g.nx && oy < g.ny;
      xm[j] = ox + j > 0;
      xp[j] = ox + j < g.nx - 1;
      any = any || own[j];
    }
    const bool ym = oy > 0, yp = oy < g.ny - 1;
    // steps q = pa-2 .. pb-1: u, g of plane q+1 (ring rows), f of plane q
    const int qlo = pa - 2, qlast = pb - 1;
    auto N = [&](int q) { return seq + (uint32_t)(q - qlo); };
    auto issue = [&](int q) {  // thread 0
      uint64_t* br = &bar[N(q) % NS];
      mbar_expect_tx(br, (uint32_t)(2 * BXR * (TY + 2) * sizeof(T) + BXR * TY * sizeof(T)));
      T* base = reinterpret_cast<T*>(sm + (N(q) % NS) * GG::STEP);
      tma_load_3d(base, &tm_u, 2 * (x0 - CW), y0 - 1, q + 1, br);
      tma_load_3d(reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(base) + GG::UB), &tm_g, 2 * (x0 - CW),
                  y0 - 1, q + 1, br);
      tma_load_3d(reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(base) + 2 * GG::UB), &tm_f, 2 * (x0 - CW), y0,
                  q, br);
    };
    if (tid == 0)
      for (int q = qlo; q < qlo + NS && q <= qlast; q++) issue(q);
    auto wait = [&](int q) { mbar_wait(&bar[N(q) % NS], (N(q) / NS) & 1u); };
    wait(qlo);
    wait(qlo + 1);
    V um = ld_vec(Ub(N(qlo)) + bo), gm = ld_vec(Gb(N(qlo)) + bo);          // plane pa-1
    V u0 = ld_vec(Ub(N(qlo + 1)) + bo), g0 = ld_vec(Gb(N(qlo + 1)) + bo);  // plane pa
    __syncthreads();  // step qlo lives on in registers only
    if (tid == 0 && qlo + NS <= qlast) {
      fence_proxy_async();
      issue(qlo + NS);
    }
    for (int p = pa; p < pb; p++) {
      wait(p);
      const T* U0 = Ub(N(p - 1));  // u(p) with its ring
      const T* G0 = Gb(N(p - 1));
      const V up = ld_vec(Ub(N(p)) + bo), gp = ld_vec(Gb(N(p)) + bo);  // plane p+1, own cells
      const V fv = ld_vec(Fb(N(p)) + fo);
      const V udn = ld_vec(U0 + bo - BXR), uupv = ld_vec(U0 + bo + BXR);
      const V gdn = ld_vec(G0 + bo - BXR), gupv = ld_vec(G0 + bo + BXR);
      const C2<T> uL = {U0[bo - 2], U0[bo - 1]}, gL = {G0[bo - 2], G0[bo - 1]};
      const C2<T> uR = {U0[bo + 2 * CW], U0[bo + 2 * CW + 1]}, gR = {G0[bo + 2 * CW], G0[bo + 2 * CW + 1]};
      const bool zm = p > 0, zp = p < g.nz - 1;
      V o{};
#pragma unroll
      for (int j = 0; j < CW; j++) {
        const C2<T> uc = cell(u0, j), gc = cell(g0, j);
        C2<T> acc_a = {(T)0, (T)0}, acc_s = {(T)0, (T)0};
        auto face = [&](bool on, T w, C2<T> gn, C2<T> un) {
          const C2<T> cf = {mul(w, mul(half, add(gc.re, gn.re))), mul(w, mul(half, add(gc.im, gn.im)))};
          const C2<T> tt = cmul(cf, un);
          acc_a = {selv(on, add(acc_a.re, cf.re), acc_a.re), selv(on, add(acc_a.im, cf.im), acc_a.im)};
          acc_s = {selv(on, add(acc_s.re, tt.re), acc_s.re), selv(on, add(acc_s.im, tt.im), acc_s.im)};
        };
        face(xm[j], c.w[0], j == 0 ? gL : cell(g0, j > 0 ? j - 1 : 0), j == 0 ? uL : cell(u0, j > 0 ? j - 1 : 0));
        face(xp[j], c.w[0], j == CW - 1 ? gR : cell(g0, j < CW - 1 ? j + 1 : 0),
             j == CW - 1 ? uR : cell(u0, j < CW - 1 ? j + 1 : 0));
        face(ym, c.w[1], cell(gdn, j), cell(udn, j));
        face(yp, c.w[1], cell(gupv, j), cell(uupv, j));
        face(zm, c.w[2], cell(gm, j), cell(um, j));
        face(zp, c.w[2], cell(gp, j), cell(up, j));
        const C2<T> diag = {add((T)1, acc_a.re), acc_a.im};
        const C2<T> du = cmul(diag, uc);
        const C2<T> fc = cell(fv, j);
        const C2<T> res = {sub(fc.re, sub(du.re, acc_s.re)), sub(fc.im, sub(du.im, acc_s.im))};
        if constexpr (NORM) {
          const double rr = selv(own[j], (double)res.re, 0.0), ri = selv(own[j], (double)res.im, 0.0);
          nsum = __dadd_rn(nsum, __dadd_rn(__dmul_rn(rr, rr), __dmul_rn(ri, ri)));
        } else {
          const C2<T> z = cdiv(res, diag);
          o.v[2 * j] = add(uc.re, mul(c.omega, z.re));
          o.v[2 * j + 1] = add(uc.im, mul(c.omega, z.im));
        }
      }
      if (!NORM && any) {
        T* orow = uout + 2 * ((long long)p * g.pstride + (long long)oy * g.pitch);
        bool all = true;
#pragma unroll
        for (int j = 0; j < CW; j++) all = all && own[j];
        if (all) {
          if constexpr (sizeof(T) == 8)
            *reinterpret_cast<double2*>(orow + 2 * ox) = make_double2(o.v[0], o.v[1]);
          else
            *reinterpret_cast<float4*>(orow + 2 * ox) = make_float4(o.v[0], o.v[1], o.v[2], o.v[3]);
        } else {
#pragma unroll
          for (int j = 0; j < CW; j++)
            if (own[j]) {
              orow[2 * (ox + j)] = o.v[2 * j];
              orow[2 * (ox + j) + 1] = o.v[2 * j + 1];
            }
        }
      }
      __syncthreads();  // every warp is past plane p: step p-1 (u(p), g(p), f(p-1)) is free
      if (tid == 0 && p - 1 + NS <= qlast) {
        fence_proxy_async();
        issue(p - 1 + NS);
      }
      um = u0;
      u0 = up;
      gm = g0;
      g0 = gp;
    }
    seq = N(qlast) + 1;
  }
  if constexpr (NORM) {  // fixed-order block reduction -> partial[blockIdx.x]
    __shared__ double red[TY];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nsum = __dadd_rn(nsum, __shfl_down_sync(0xffffffffu, nsum, o));
    if (lane == 0) red[ry] = nsum;
    __syncthreads();
    if (tid == 0) {
      double tot = 0.0;
      for (int w = 0; w < TY; w++) tot = __dadd_rn(tot, red[w]);
      partial[blockIdx.x] = tot;
    }
  }
}

// complex level array viewed as reals: dims (2 nx, ny, nz), box (BXR, rows, 1), zero OOB fill
template <typename T>
static bool encode(CUtensorMap* tm, const T* base, const Geom& g, int rows) {
  const unsigned long long dims[3] = {(unsigned long long)(2 * g.nx), (unsigned long long)g.ny,
                                      (unsigned long long)g.nz};
  const unsigned long long strides[2] = {(unsigned long long)(g.pitch * 2 * sizeof(T)),
                                         (unsigned long long)(g.pstride * 2 * sizeof(T))};
  const unsigned box[3] = {(unsigned)G<T>::BXR, (unsigned)rows, 1u};
  return pm::encode_tiled(tm, sizeof(T) == 8, 3, base, dims, strides, box) == CUDA_SUCCESS;
}

// work items (tile, z-chunk): one wave of resident CTAs, chunks of >= 4 planes
template <typename T, bool NORM>
static void grid_of(const Geom& g, int& tiles_x, int& ntiles, int& zc, int& nitems, int& nb) {
  tiles_x = (g.nx + G<T>::TX - 1) / G<T>::TX;
  ntiles = tiles_x * ((g.ny + TY - 1) / TY);
  const int resident = resident_ctas((const void*)k_cd_jacobi3d<T, NORM>, NT, G<T>::SMEM);  // whole GPU
  int nch = resident / ntiles;
  if (nch < 1) nch = 1;
  if (nch > g.nz / 4) nch = g.nz / 4 > 0 ? g.nz / 4 : 1;
  zc = (g.nz + nch - 1) / nch;
  nitems = ntiles * ((g.nz + zc - 1) / zc);
  nb = nitems < resident ? nitems : resident;
}

}  // namespace cd3

bool cd3d_supported(const Geom& g) { return g.three_d && g.nx >= 32 && g.ny >= 8 && g.nz >= 4; }

template <typename T>
static cudaError_t cd3d_run(const Geom& g, const CdCoef<T>& c, const T* gd, const T* u, const T* f, T* uout,
                            double* partial, int* npartial, cudaStream_t st) {
  using namespace cd3;
  CUtensorMap tu, tg, tf;
  if (!encode<T>(&tu, u, g, TY + 2) || !encode<T>(&tg, gd, g, TY + 2) || !encode<T>(&tf, f, g, TY))
    return cudaErrorInvalidValue;
  int tiles_x, ntiles, zc, nitems, nb;
  if (partial) {
    grid_of<T, true>(g, tiles_x, ntiles, zc, nitems, nb);
    *npartial = nb;
    k_cd_jacobi3d<T, true><<<nb, NT, G<T>::SMEM, st>>>(tu, tg, tf, g, c, nullptr, tiles_x, ntiles, zc, nitems,
                                                       partial);
  } else {
    grid_of<T, false>(g, tiles_x, ntiles, zc, nitems, nb);
    k_cd_jacobi3d<T, false><<<nb, NT, G<T>::SMEM, st>>>(tu, tg, tf, g, c, uout, tiles_x, ntiles, zc, nitems,
                                                        nullptr);
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t cd3d_launch_jacobi(const Geom& g, const CdCoef<T>& c, const T* gd, const T* uin, const T* f, T* uout,
                               cudaStream_t st) {
  return cd3d_run<T>(g, c, gd, uin, f, uout, nullptr, nullptr, st);
}

template <typename T>
int cd3d_norm_partials(const Geom& g) {
  int tiles_x, ntiles, zc, nitems, nb;
  cd3::grid_of<T, true>(g, tiles_x, ntiles, zc, nitems, nb);
  return nb;
}

template <typename T>
cudaError_t cd3d_launch_norm(const Geom& g, const CdCoef<T>& c, const T* gd, const T* u, const T* f,
                             double* partial, int* npartial, cudaStream_t st) {
  return cd3d_run<T>(g, c, gd, u, f, nullptr, partial, npartial, st);
}

#define CD3_INST(T)                                                                                                  \
  template cudaError_t cd3d_launch_jacobi<T>(const Geom&, const CdCoef<T>&, const T*, const T*, const T*, T*,       \
                                             cudaStream_t);                                                          \
  template int cd3d_norm_partials<T>(const Geom&);                                                                   \
  template cudaError_t cd3d_launch_norm<T>(const Geom&, const CdCoef<T>&, const T*, const T*, const T*, double*,    \
                                           int*, cudaStream_t);
CD3_INST(float)
CD3_INST(double)
#undef CD3_INST

}  // namespace mg
