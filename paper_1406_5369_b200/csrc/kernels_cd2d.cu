// kernels_cd2d.cu — warp-marching omega-Jacobi sweep of the complex-diffusion operator on
// 2D cell-centred levels (the skeleton of kernels_pm2d.cu applied to kernels_cd.cu's
// operator).
//
// A warp owns a strip of TX = 32 CW cells (lane = one 16-byte vector of CW = 16/(2 sizeof T)
// complex cells: 2 in FP32, 1 in FP64) and marches a chunk of rows.  Every step of RB rows
// of u, of the lagged diffusivity g and of f arrives by three per-warp 2D TMA boxes
// (the complex arrays viewed as real arrays twice as wide, strip +- CW cells, zero-filled
// outside) in a per-warp shared-memory ring of NS slots.  x-neighbours by warp shuffles
// (lanes 0 / 31 read the strip edge from the box), the rows above and below in registers:
// u, g and f are read from HBM once per sweep, u' written once.  The per-cell arithmetic is
// kernels_cd.cu's relax() in the same canonical order (faces x-, x+, y-, y+), so the
// output is bitwise that of k_cd_jacobi and of the oracle.
#include <cstdio>
#include <cstdlib>

#include "cd_common.cuh"
#include "kernels_cd.h"
#include "kernels_pm.h"
#include "launch_util.h"
#include "tma.cuh"
#include "vec.cuh"

namespace mg {
namespace cd2 {
using namespace cdk;

constexpr int WPB = 4;  // warps per CTA
constexpr int NT = 32 * WPB;
constexpr int RB = 2;  // rows per step
constexpr int NS = 4;  // ring slots per warp
constexpr unsigned FULL = 0xffffffffu;

template <typename T>
struct G {
  static constexpr int CW = 16 / (2 * (int)sizeof(T));  // complex cells per lane
  static constexpr int TX = 32 * CW;                    // strip width in cells
  static constexpr int RW = 2 * (TX + 2 * CW);          // box row in reals: cells x0-CW .. x0+TX+CW
  static constexpr int BOX = RW * RB;
  static constexpr int BOXB = BOX * (int)sizeof(T);               // bytes a box load delivers
  static constexpr int BOXS = (BOXB + 127) / 128 * 128 / (int)sizeof(T);  // box stride (128-B aligned)
  static constexpr int WARP_BYTES = NS * 3 * BOXS * (int)sizeof(T) + 128;  // slots (u, g, f) + mbarriers
  static constexpr int SMEM = WPB * WARP_BYTES;
};

template <typename T>
using VT = Vec<T, 16 / sizeof(T)>;

template <typename T>
__device__ __forceinline__ C2<T> cell(const VT<T>& v, int j) {
  return {v.v[2 * j], v.v[2 * j + 1]};
}
template <typename T>
__device__ __forceinline__ C2<T> shfl_up(C2<T> a) {
  return {__shfl_up_sync(FULL, a.re, 1), __shfl_up_sync(FULL, a.im, 1)};
}
template <typename T>
__device__ __forceinline__ C2<T> shfl_down(C2<T> a) {
  return {__shfl_down_sync(FULL, a.re, 1), __shfl_down_sync(FULL, a.im, 1)};
}

__device__ __forceinline__ void item2(int gw, int nstrips, int nch, int lo, int hi, int& strip, int& pa, int& pb) {
  strip = gw % nstrips;
  const int ch = gw / nstrips;
  const long long n = hi - lo;
  pa = lo + (int)(n * ch / nch);
  pb = lo + (int)(n * (ch + 1) / nch);
}

// A step b of a march starting at row t0: u and g rows t0 + b RB + 1 .. + RB, and (b >= 0)
// f rows t0 + b RB .. + RB - 1; step -1 supplies u, g of rows t0 - RB + 1 .. t0.
template <typename T>
struct Ring {
  using GG = G<T>;
  T* buf;
  uint64_t* bar;
  uint32_t n0;
  int t0, x;  // first row, box x start in reals
  __device__ void init(unsigned char* smem, int wid, int lane) {
    unsigned char* w = smem + wid * GG::WARP_BYTES;
    buf = reinterpret_cast<T*>(w);
    bar = reinterpret_cast<uint64_t*>(w + NS * 3 * GG::BOXS * sizeof(T));
    n0 = 0;
    if (lane == 0) {
      for (int s = 0; s < NS; s++) mbar_init(&bar[s], 1);
      fence_barrier_init();
    }
    __syncwarp();
  }
  __device__ uint32_t N(int b) const { return n0 + (uint32_t)(b + 1); }
  __device__ T* U(int b) const { return buf + (N(b) % NS) * (3 * GG::BOXS); }
  __device__ T* Gd(int b) const { return U(b) + GG::BOXS; }
  __device__ T* F(int b) const { return U(b) + 2 * GG::BOXS; }
  __device__ void wait(int b) const { mbar_wait(&bar[N(b) % NS], (N(b) / NS) & 1u); }
  __device__ void issue(int b, const CUtensorMap* tu, const CUtensorMap* tg, const CUtensorMap* tf) const {
    uint64_t* br = &bar[N(b) % NS];
    const bool lf = b >= 0;
    mbar_expect_tx(br, (uint32_t)((lf ? 3 : 2) * GG::BOXB));
    tma_load_2d(U(b), tu, x, t0 + b * RB + 1, br);
    tma_load_2d(Gd(b), tg, x, t0 + b * RB + 1, br);
    if (lf) tma_load_2d(F(b), tf, x, t0 + b * RB, br);
  }
  __device__ void start(int nsteps, const CUtensorMap* tu, const CUtensorMap* tg, const CUtensorMap* tf) const {
    for (int b = -1; b < NS - 1 && b < nsteps; b++) issue(b, tu, tg, tf);
  }
  __device__ void release(int b, int nsteps, int lane, const CUtensorMap* tu, const CUtensorMap* tg,
                          const CUtensorMap* tf) const {
    __syncwarp();
    if (lane == 0 && b + NS < nsteps) issue(b + NS, tu, tg, tf);
  }
  __device__ void finish(int nsteps) { n0 = N(nsteps - 1) + 1; }
};

// NORM: instead of the sweep, the partial sums of |f - A(g) u|^2 (FP64), one per CTA in a
// fixed order (the nonlinear residual norm of the head, with g = g(u) stored)
template <typename T, bool NORM>
__global__ void __launch_bounds__(NT) k_cd_jacobi2d(const __grid_constant__ CUtensorMap tm_u,
                                                    const __grid_constant__ CUtensorMap tm_g,
                                                    const __grid_constant__ CUtensorMap tm_f, Geom g, CdCoef<T> c,
                                                    T* __restrict__ uout, int nstrips, int nch,
                                                    double* __restrict__ partial) {
  double nsum = 0.0;
  using V = VT<T>;
  using GG = G<T>;
  constexpr int CW = GG::CW, TX = GG::TX, RW = GG::RW;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Ring<T> R;
  R.init(smem, wid, lane);
  if (lane == 0) {
    prefetch_tmap(&tm_u);
    prefetch_tmap(&tm_g);
    prefetch_tmap(&tm_f);
  }
  const int vo = 2 * (CW + CW * lane);                  // the lane's vector in a box row (reals)
  const int eo = lane == 0 ? 2 * (CW - 1) : 2 * (CW + TX);  // strip-edge cell (lane 0: x0-1, 31: x0+TX)
  const T half = (T)0.5;
  for (int gw = blockIdx.x * WPB + wid; gw < nstrips * nch; gw += gridDim.x * WPB) {
    int strip, pa, pb;
    item2(gw, nstrips, nch, 0, g.nz, strip, pa, pb);
    const int x0 = strip * TX, ox = x0 + CW * lane;
    R.t0 = pa;
    R.x = 2 * (x0 - CW);
    const int nsteps = (pb - 1 - pa) / RB + 1;
    if (lane == 0) R.start(nsteps, &tm_u, &tm_g, &tm_f);
    auto edge = [&](const T* row) { return C2<T>{row[eo], row[eo + 1]}; };
    R.wait(-1);
    V um = ld_vec(R.U(-1) + (RB - 2) * RW + vo), gm = ld_vec(R.Gd(-1) + (RB - 2) * RW + vo);
    V u0 = ld_vec(R.U(-1) + (RB - 1) * RW + vo), g0 = ld_vec(R.Gd(-1) + (RB - 1) * RW + vo);
    C2<T> u0e = edge(R.U(-1) + (RB - 1) * RW), g0e = edge(R.Gd(-1) + (RB - 1) * RW);
    R.release(-1, nsteps, lane, &tm_u, &tm_g, &tm_f);
    for (int b = 0; b < nsteps; b++) {
      R.wait(b);
      const T* Ub = R.U(b);
      const T* Gb = R.Gd(b);
      const T* Fb = R.F(b);
#pragma unroll
      for (int i = 0; i < RB; i++) {
        const int t = pa + b * RB + i;
        if (t >= pb) break;
        const V up = ld_vec(Ub + i * RW + vo), gp = ld_vec(Gb + i * RW + vo), fv = ld_vec(Fb + i * RW + vo);
        const C2<T> upe = edge(Ub + i * RW), gpe = edge(Gb + i * RW);
        // x-neighbours of the lane's first / last cell
        C2<T> uL = shfl_up(cell(u0, CW - 1)), gL = shfl_up(cell(g0, CW - 1));
        C2<T> uR = shfl_down(cell(u0, 0)), gR = shfl_down(cell(g0, 0));
        if (lane == 0) {
          uL = u0e;
          gL = g0e;
        }
        if (lane == 31) {
          uR = u0e;
          gR = g0e;
        }
        V o;
#pragma unroll
        for (int j = 0; j < CW; j++) {
          const int ci = ox + j;
          const C2<T> uc = cell(u0, j), gc = cell(g0, j);
          C2<T> acc_a = {(T)0, (T)0}, acc_s = {(T)0, (T)0};
          auto face = [&](T w, C2<T> gn, C2<T> un) {
            const C2<T> cf = {mul(w, mul(half, add(gc.re, gn.re))), mul(w, mul(half, add(gc.im, gn.im)))};
            acc_a = {add(acc_a.re, cf.re), add(acc_a.im, cf.im)};
            const C2<T> tt = cmul(cf, un);
            acc_s = {add(acc_s.re, tt.re), add(acc_s.im, tt.im)};
          };
          if (ci > 0) face(c.w[0], j == 0 ? gL : cell(g0, j > 0 ? j - 1 : 0), j == 0 ? uL : cell(u0, j > 0 ? j - 1 : 0));
          if (ci < g.nx - 1)
            face(c.w[0], j == CW - 1 ? gR : cell(g0, j < CW - 1 ? j + 1 : 0),
                 j == CW - 1 ? uR : cell(u0, j < CW - 1 ? j + 1 : 0));
          if (t > 0) face(c.w[2], cell(gm, j), cell(um, j));
          if (t < g.nz - 1) face(c.w[2], cell(gp, j), cell(up, j));
          const C2<T> diag = {add((T)1, acc_a.re), acc_a.im};
          const C2<T> du = cmul(diag, uc);
          const C2<T> fc = cell(fv, j);
          const C2<T> res = {sub(fc.re, sub(du.re, acc_s.re)), sub(fc.im, sub(du.im, acc_s.im))};
          if constexpr (NORM) {
            if (ci < g.nx) {
              const double rr = (double)res.re, ri = (double)res.im;
              nsum = __dadd_rn(nsum, __dadd_rn(__dmul_rn(rr, rr), __dmul_rn(ri, ri)));
            }
          } else {
            const C2<T> z = cdiv(res, diag);
            o.v[2 * j] = add(uc.re, mul(c.omega, z.re));
            o.v[2 * j + 1] = add(uc.im, mul(c.omega, z.im));
          }
        }
        if (NORM) {
          um = u0;
          gm = g0;
          u0 = up;
          g0 = gp;
          u0e = upe;
          g0e = gpe;
          continue;
        }
        T* orow = uout + (long long)t * g.pstride * 2;
        bool all = true;
#pragma unroll
        for (int j = 0; j < CW; j++) all = all && (ox + j < g.nx);
        if (all) {
          if constexpr (sizeof(T) == 8)
            *reinterpret_cast<double2*>(orow + 2 * ox) = make_double2(o.v[0], o.v[1]);
          else
            *reinterpret_cast<float4*>(orow + 2 * ox) = make_float4(o.v[0], o.v[1], o.v[2], o.v[3]);
        } else {
#pragma unroll
          for (int j = 0; j < CW; j++)
            if (ox + j < g.nx) {
              orow[2 * (ox + j)] = o.v[2 * j];
              orow[2 * (ox + j) + 1] = o.v[2 * j + 1];
            }
        }
        um = u0;
        gm = g0;
        u0 = up;
        g0 = gp;
        u0e = upe;
        g0e = gpe;
      }
      R.release(b, nsteps, lane, &tm_u, &tm_g, &tm_f);
    }
    R.finish(nsteps);
  }
  if constexpr (NORM) {  // fixed-order block reduction -> partial[blockIdx.x]
    __shared__ double red[WPB];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nsum = __dadd_rn(nsum, __shfl_down_sync(FULL, nsum, o));
    if (lane == 0) red[wid] = nsum;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (int w = 0; w < WPB; w++) tot = __dadd_rn(tot, red[w]);
      partial[blockIdx.x] = tot;
    }
  }
}

// ---------------------------------------------------------------------------
template <class K>
static int resident_warps(K kernel, int smem) {
  return resident_ctas((const void*)kernel, NT, smem) * WPB;
}

// complex level array viewed as reals: dims (2 nx, planes), box (RW, RB), zero OOB fill
template <typename T>
static bool encode(CUtensorMap* tm, const T* base, const Geom& g) {
  const unsigned long long dims[2] = {(unsigned long long)(2 * g.nx), (unsigned long long)g.planes};
  const unsigned long long strides[1] = {(unsigned long long)(g.pstride * 2 * sizeof(T))};
  const unsigned box[2] = {(unsigned)G<T>::RW, (unsigned)RB};
  return pm::encode_tiled(tm, sizeof(T) == 8, 2, base, dims, strides, box) == CUDA_SUCCESS;
}

}  // namespace cd2

bool cd2d_supported(const Geom& g) { return !g.three_d && g.nx >= 64 && g.nz >= 8; }

namespace {
template <typename T>
int cd2d_grid(const Geom& g, int& ns, int& nch) {
  using namespace cd2;
  ns = (g.nx + G<T>::TX - 1) / G<T>::TX;
  const int rw = resident_warps(k_cd_jacobi2d<T, false>, G<T>::SMEM);
  nch = rw / ns;
  if (nch > g.nz / 4) nch = g.nz / 4;
  if (nch < 1) nch = 1;
  return (ns * nch + WPB - 1) / WPB;
}
}  // namespace

template <typename T>
cudaError_t cd2d_launch_jacobi(const Geom& g, const CdCoef<T>& c, const T* gd, const T* uin, const T* f, T* uout,
                               cudaStream_t st) {
  using namespace cd2;
  CUtensorMap tu, tg, tf;
  if (!encode<T>(&tu, uin, g) || !encode<T>(&tg, gd, g) || !encode<T>(&tf, f, g)) return cudaErrorInvalidValue;
  int ns, nch;
  const int nb = cd2d_grid<T>(g, ns, nch);
  k_cd_jacobi2d<T, false><<<nb, NT, G<T>::SMEM, st>>>(tu, tg, tf, g, c, uout, ns, nch, nullptr);
  return cudaGetLastError();
}

template <typename T>
int cd2d_norm_partials(const Geom& g) {
  int ns, nch;
  return cd2d_grid<T>(g, ns, nch);
}

template <typename T>
cudaError_t cd2d_launch_norm(const Geom& g, const CdCoef<T>& c, const T* gd, const T* u, const T* f,
                             double* partial, int* npartial, cudaStream_t st) {
  using namespace cd2;
  CUtensorMap tu, tg, tf;
  if (!encode<T>(&tu, u, g) || !encode<T>(&tg, gd, g) || !encode<T>(&tf, f, g)) return cudaErrorInvalidValue;
  int ns, nch;
  const int nb = cd2d_grid<T>(g, ns, nch);
  *npartial = nb;
  resident_warps(k_cd_jacobi2d<T, true>, G<T>::SMEM);  // opt in to the shared-memory size
  k_cd_jacobi2d<T, true><<<nb, NT, G<T>::SMEM, st>>>(tu, tg, tf, g, c, nullptr, ns, nch, partial);
  return cudaGetLastError();
}

template cudaError_t cd2d_launch_jacobi<float>(const Geom&, const CdCoef<float>&, const float*, const float*,
                                               const float*, float*, cudaStream_t);
template cudaError_t cd2d_launch_jacobi<double>(const Geom&, const CdCoef<double>&, const double*, const double*,
                                                const double*, double*, cudaStream_t);
template int cd2d_norm_partials<float>(const Geom&);
template int cd2d_norm_partials<double>(const Geom&);
template cudaError_t cd2d_launch_norm<float>(const Geom&, const CdCoef<float>&, const float*, const float*,
                                             const float*, double*, int*, cudaStream_t);
template cudaError_t cd2d_launch_norm<double>(const Geom&, const CdCoef<double>&, const double*, const double*,
                                              const double*, double*, int*, cudaStream_t);

}  // namespace mg
