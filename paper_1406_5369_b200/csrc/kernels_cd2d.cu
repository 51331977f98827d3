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

// A step b of a march starting at row t0: u and g rows t0 + b RBR + 1 .. + RBR, and (b >= 0)
// f rows t0 + b RBR .. + RBR - 1; step -1 supplies u, g of rows t0 - RBR + 1 .. t0.
template <typename T, int RBR = RB, int NSR = NS>
struct Ring {
  static constexpr int BOXB = G<T>::RW * RBR * (int)sizeof(T);           // bytes a box load delivers
  static constexpr int BOXS = (BOXB + 127) / 128 * 128 / (int)sizeof(T);  // box stride (128-B aligned)
  static constexpr int WARP_BYTES = NSR * 3 * BOXS * (int)sizeof(T) + 128;  // slots (u, g, f) + mbarriers
  static constexpr int SMEM = WPB * WARP_BYTES;
  T* buf;
  uint64_t* bar;
  uint32_t n0;
  int t0, x;  // first row, box x start in reals
  __device__ void init(unsigned char* smem, int wid, int lane) {
    unsigned char* w = smem + wid * WARP_BYTES;
    buf = reinterpret_cast<T*>(w);
    bar = reinterpret_cast<uint64_t*>(w + NSR * 3 * BOXS * sizeof(T));
    n0 = 0;
    if (lane == 0) {
      for (int s = 0; s < NSR; s++) mbar_init(&bar[s], 1);
      fence_barrier_init();
    }
    __syncwarp();
  }
  __device__ uint32_t N(int b) const { return n0 + (uint32_t)(b + 1); }
  __device__ T* U(int b) const { return buf + (N(b) % NSR) * (3 * BOXS); }
  __device__ T* Gd(int b) const { return U(b) + BOXS; }
  __device__ T* F(int b) const { return U(b) + 2 * BOXS; }
  __device__ void wait(int b) const { mbar_wait(&bar[N(b) % NSR], (N(b) / NSR) & 1u); }
  __device__ void issue(int b, const CUtensorMap* tu, const CUtensorMap* tg, const CUtensorMap* tf) const {
    uint64_t* br = &bar[N(b) % NSR];
    const bool lf = b >= 0;
    mbar_expect_tx(br, (uint32_t)((lf ? 3 : 2) * BOXB));
    tma_load_2d(U(b), tu, x, t0 + b * RBR + 1, br);
    tma_load_2d(Gd(b), tg, x, t0 + b * RBR + 1, br);
    if (lf) tma_load_2d(F(b), tf, x, t0 + b * RBR, br);
  }
  __device__ void start(int nsteps, const CUtensorMap* tu, const CUtensorMap* tg, const CUtensorMap* tf) const {
    for (int b = -1; b < NSR - 1 && b < nsteps; b++) issue(b, tu, tg, tf);
  }
  __device__ void release(int b, int nsteps, int lane, const CUtensorMap* tu, const CUtensorMap* tg,
                          const CUtensorMap* tf) const {
    __syncwarp();
    if (lane == 0 && b + NSR < nsteps) issue(b + NSR, tu, tg, tf);
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
        V o{};
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
// K omega-Jacobi sweeps with the frozen g in ONE pass (temporal blocking, the scheme of
// kernels_pm2d.cu k_jacobi2d_k): stage k relaxes row t-k+1 from stage k-1's rows kept in
// a 3-row register window per stage; g rows come from a 3-row window (stage 1) and a
// chain of delayed copies (stage k >= 2 reads rows down to t-k).  Strips overlap by CW
// cells per side, lanes 1..30 store, so a stage-k value is exact K-1 <= CW cells inside
// the box on every stored cell.  The face terms are formed unconditionally and selected
// (selv) where relax() skips them: the same operations on every cell of the domain, so
// the result is bitwise that of K launches of k_cd_jacobi2d.  u, g, f read once, u^(K)
// written once: 4 complex words per pass.  NRM: the partials of |f - A(g) u_in|^2 from
// stage 1 on the stored cells (the solve's head: norm + first pre-smoothing pass).
template <typename T, int K, bool NRM>
__global__ void __launch_bounds__(NT) k_cd_jacobi2d_k(const __grid_constant__ CUtensorMap tm_u,
                                                      const __grid_constant__ CUtensorMap tm_g,
                                                      const __grid_constant__ CUtensorMap tm_f, Geom g, CdCoef<T> c,
                                                      T* __restrict__ uout, int nstrips, int nch,
                                                      double* __restrict__ partial) {
  using V = VT<T>;
  using GG = G<T>;
  constexpr int CW = GG::CW, TX = GG::TX, RW = GG::RW, SX = TX - 2 * CW;
  static_assert(K >= 1 && K <= CW + 1, "overlap CW cells per side");
  constexpr int R3 = 3;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Ring<T, R3, 3> R;
  R.init(smem, wid, lane);
  if (lane == 0) {
    prefetch_tmap(&tm_u);
    prefetch_tmap(&tm_g);
    prefetch_tmap(&tm_f);
  }
  const int vo = 2 * (CW + CW * lane);
  const int eo = lane == 0 ? 2 * (CW - 1) : 2 * (CW + TX);
  const bool stores = lane >= 1 && lane <= 30;
  const T half = (T)0.5;
  double nsum = 0.0;
  for (int gw = blockIdx.x * WPB + wid; gw < nstrips * nch; gw += gridDim.x * WPB) {
    int strip, pa, pb;
    item2(gw, nstrips, nch, 0, g.nz, strip, pa, pb);
    const int x0 = strip * SX - CW, ox = x0 + CW * lane;
    bool xm[CW], xp[CW], own[CW];  // face x- / x+ present; a stored cell of the domain
#pragma unroll
    for (int j = 0; j < CW; j++) {
      xm[j] = ox + j > 0;
      xp[j] = ox + j < g.nx - 1;
      own[j] = stores && ox + j >= 0 && ox + j < g.nx;
    }
    const int ts = pa - K + 1, te = pb + K - 2;
    R.t0 = ts;
    R.x = 2 * (x0 - CW);
    const int nsteps = (te - ts) / R3 + 1;
    if (lane == 0) R.start(nsteps, &tm_u, &tm_g, &tm_f);
    auto edge = [&](const T* row) { return C2<T>{row[eo], row[eo + 1]}; };
    // windows: slot of a row = (row - ts + 1) mod 3
    V S[K + 1][3], Gw[3], Fw[3];
    V Gold[K > 1 ? K - 1 : 1];  // g rows t-2, t-3, ... (stages >= 2)
    C2<T> ue[3], ge[3];         // stage-0 u and g at the strip-edge cell (lanes 0 / 31)
    R.wait(-1);
    {
      const T* U = R.U(-1);
      const T* Gb = R.Gd(-1);
      S[0][0] = ld_vec(U + 1 * RW + vo);  // row ts-1
      S[0][1] = ld_vec(U + 2 * RW + vo);  // row ts
      Gw[0] = ld_vec(Gb + 1 * RW + vo);
      Gw[1] = ld_vec(Gb + 2 * RW + vo);
      ue[0] = edge(U + 1 * RW);
      ue[1] = edge(U + 2 * RW);
      ge[0] = edge(Gb + 1 * RW);
      ge[1] = edge(Gb + 2 * RW);
      Gw[2] = Gw[1];  // row ts-2 is never used by an exact value
#pragma unroll
      for (int k = 0; k < (K > 1 ? K - 1 : 1); k++) Gold[k] = Gw[0];
    }
    R.release(-1, nsteps, lane, &tm_u, &tm_g, &tm_f);
    auto iter = [&](auto PHc, int t, const T* ur, const T* gr, const T* fr) {
      constexpr int PH = decltype(PHc)::value;
      constexpr int sN = (PH + 2) % 3;  // slot of row t+1 (held row t-2)
      if constexpr (K > 1) {
#pragma unroll
        for (int k = K - 2; k > 0; k--) Gold[k] = Gold[k - 1];
        Gold[0] = Gw[sN];
      }
      S[0][sN] = ld_vec(ur + vo);
      Gw[sN] = ld_vec(gr + vo);
      ue[sN] = edge(ur);
      ge[sN] = edge(gr);
      Fw[(PH + 1) % 3] = ld_vec(fr + vo);  // f, row t
#pragma unroll
      for (int k = 1; k <= K; k++) {
        const int s0 = (PH - k + 2 + 6) % 3, sm = (PH - k + 1 + 6) % 3, sp = (PH - k + 6) % 3;
        const int rho = t - k + 1;
        // g row t + d: the window holds rows >= t-1 (slot (PH + 1 + d) mod 3), Gold[i] row t-2-i
        auto grow = [&](int d) -> const V& { return d >= -1 ? Gw[(PH + 4 + d) % 3] : Gold[-2 - d]; };
        const V& g0 = grow(1 - k);
        const V& gmv = grow(-k);
        const V& gpv = grow(2 - k);
        const V& u0 = S[k - 1][s0];
        const V& umv = S[k - 1][sm];
        const V& upv = S[k - 1][sp];
        C2<T> uL = shfl_up(cell(u0, CW - 1)), gL = shfl_up(cell(g0, CW - 1));
        C2<T> uR = shfl_down(cell(u0, 0)), gR = shfl_down(cell(g0, 0));
        if (k == 1) {  // the box supplies the stage-0 cells beyond the strip
          if (lane == 0) {
            uL = ue[s0];
            gL = ge[s0];
          }
          if (lane == 31) {
            uR = ue[s0];
            gR = ge[s0];
          }
        }
        const bool ym = rho > 0, yp = rho < g.nz - 1;
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
          face(ym, c.w[2], cell(gmv, j), cell(umv, j));
          face(yp, c.w[2], cell(gpv, j), cell(upv, j));
          const C2<T> diag = {add((T)1, acc_a.re), acc_a.im};
          const C2<T> du = cmul(diag, uc);
          const C2<T> fc = cell(Fw[s0], j);
          const C2<T> res = {sub(fc.re, sub(du.re, acc_s.re)), sub(fc.im, sub(du.im, acc_s.im))};
          if (NRM && k == 1) {
            const bool on = own[j] && t >= pa && t < pb;
            const double rr = selv(on, (double)res.re, 0.0), ri = selv(on, (double)res.im, 0.0);
            nsum = __dadd_rn(nsum, __dadd_rn(__dmul_rn(rr, rr), __dmul_rn(ri, ri)));
          }
          const C2<T> z = cdiv(res, diag);
          o.v[2 * j] = add(uc.re, mul(c.omega, z.re));
          o.v[2 * j + 1] = add(uc.im, mul(c.omega, z.im));
        }
        S[k][s0] = o;
      }
      const int ro = t - K + 1;
      if (ro >= pa && ro < pb) {
        const V& ov = S[K][(PH - K + 8) % 3];
        T* orow = uout + (long long)ro * g.pstride * 2;
        bool all = true, any = false;
#pragma unroll
        for (int j = 0; j < CW; j++) {
          all = all && own[j];
          any = any || own[j];
        }
        if (all) {
          if constexpr (sizeof(T) == 8)
            *reinterpret_cast<double2*>(orow + 2 * ox) = make_double2(ov.v[0], ov.v[1]);
          else
            *reinterpret_cast<float4*>(orow + 2 * ox) = make_float4(ov.v[0], ov.v[1], ov.v[2], ov.v[3]);
        } else if (any) {
#pragma unroll
          for (int j = 0; j < CW; j++)
            if (own[j]) {
              orow[2 * (ox + j)] = ov.v[2 * j];
              orow[2 * (ox + j) + 1] = ov.v[2 * j + 1];
            }
        }
      }
    };
    for (int b = 0; b < nsteps; b++) {  // rows past te (last box) compute values never stored
      R.wait(b);
      const T* Ub = R.U(b);
      const T* Gb = R.Gd(b);
      const T* Fb = R.F(b);
      const int t = ts + b * R3;
      iter(std::integral_constant<int, 0>(), t, Ub, Gb, Fb);
      iter(std::integral_constant<int, 1>(), t + 1, Ub + RW, Gb + RW, Fb + RW);
      iter(std::integral_constant<int, 2>(), t + 2, Ub + 2 * RW, Gb + 2 * RW, Fb + 2 * RW);
      R.release(b, nsteps, lane, &tm_u, &tm_g, &tm_f);
    }
    R.finish(nsteps);
  }
  if constexpr (NRM) {  // fixed-order block reduction -> partial[blockIdx.x]
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
static bool encode(CUtensorMap* tm, const T* base, const Geom& g, int rows = RB) {
  const unsigned long long dims[2] = {(unsigned long long)(2 * g.nx), (unsigned long long)g.planes};
  const unsigned long long strides[1] = {(unsigned long long)(g.pstride * 2 * sizeof(T))};
  const unsigned box[2] = {(unsigned)G<T>::RW, (unsigned)rows};
  return pm::encode_tiled(tm, sizeof(T) == 8, 2, base, dims, strides, box) == CUDA_SUCCESS;
}

}  // namespace cd2

bool cd2d_supported(const Geom& g) { return !g.three_d && g.nx >= 64 && g.nz >= 8; }

namespace {
template <typename T>
int cd2d_grid(const Geom& g, int& ns, int& nch) {
  using namespace cd2;
  ns = (g.nx + G<T>::TX - 1) / G<T>::TX;
  const int rw = resident_warps(k_cd_jacobi2d<T, false>, Ring<T>::SMEM);
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
  k_cd_jacobi2d<T, false><<<nb, NT, Ring<T>::SMEM, st>>>(tu, tg, tf, g, c, uout, ns, nch, nullptr);
  return cudaGetLastError();
}

template <typename T>
cudaError_t cd2d_launch_jacobi_k(const Geom& g, const CdCoef<T>& c, int K, const T* gd, const T* uin, const T* f,
                                 T* uout, cudaStream_t st, double* partial, int* npartial) {
  using namespace cd2;
  CUtensorMap tu, tg, tf;
  if (!encode<T>(&tu, uin, g, 3) || !encode<T>(&tg, gd, g, 3) || !encode<T>(&tf, f, g, 3))
    return cudaErrorInvalidValue;
  const int ns = (g.nx + G<T>::TX - 2 * G<T>::CW - 1) / (G<T>::TX - 2 * G<T>::CW);
  const int smem = Ring<T, 3, 3>::SMEM;
  int nb = 0;
  auto go = [&](auto kernel) {
    int nch = resident_warps(kernel, smem) / ns;
    if (nch > g.nz / 8) nch = g.nz / 8;
    if (nch < 1) nch = 1;
    nb = (ns * nch + WPB - 1) / WPB;
    kernel<<<nb, NT, smem, st>>>(tu, tg, tf, g, c, uout, ns, nch, partial);
  };
  auto goK = [&](auto Kc) {
    constexpr int KK = decltype(Kc)::value;
    partial ? go(k_cd_jacobi2d_k<T, KK, true>) : go(k_cd_jacobi2d_k<T, KK, false>);
  };
  if (K == 1)
    goK(std::integral_constant<int, 1>());
  else if (K == 2)
    goK(std::integral_constant<int, 2>());
  else if constexpr (G<T>::CW >= 2) {
    if (K != 3) return cudaErrorInvalidValue;
    goK(std::integral_constant<int, 3>());
  } else {
    return cudaErrorInvalidValue;
  }
  if (npartial) *npartial = nb;
  return cudaGetLastError();
}

template <typename T>
int cd2d_kpartials(const Geom& g) {  // the most partials a NRM pass of any K writes
  using namespace cd2;
  const int ns = (g.nx + G<T>::TX - 2 * G<T>::CW - 1) / (G<T>::TX - 2 * G<T>::CW);
  int best = 0;
  auto one = [&](auto kernel) {
    int nch = resident_warps(kernel, Ring<T, 3, 3>::SMEM) / ns;
    if (nch > g.nz / 8) nch = g.nz / 8;
    if (nch < 1) nch = 1;
    const int nb = (ns * nch + WPB - 1) / WPB;
    if (nb > best) best = nb;
  };
  one(k_cd_jacobi2d_k<T, 1, true>);
  one(k_cd_jacobi2d_k<T, 2, true>);
  if constexpr (G<T>::CW >= 2) one(k_cd_jacobi2d_k<T, 3, true>);
  return best;
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
  resident_warps(k_cd_jacobi2d<T, true>, Ring<T>::SMEM);  // opt in to the shared-memory size
  k_cd_jacobi2d<T, true><<<nb, NT, Ring<T>::SMEM, st>>>(tu, tg, tf, g, c, nullptr, ns, nch, partial);
  return cudaGetLastError();
}

template cudaError_t cd2d_launch_jacobi<float>(const Geom&, const CdCoef<float>&, const float*, const float*,
                                               const float*, float*, cudaStream_t);
template cudaError_t cd2d_launch_jacobi<double>(const Geom&, const CdCoef<double>&, const double*, const double*,
                                                const double*, double*, cudaStream_t);
template cudaError_t cd2d_launch_jacobi_k<float>(const Geom&, const CdCoef<float>&, int, const float*, const float*,
                                                 const float*, float*, cudaStream_t, double*, int*);
template cudaError_t cd2d_launch_jacobi_k<double>(const Geom&, const CdCoef<double>&, int, const double*,
                                                  const double*, const double*, double*, cudaStream_t, double*, int*);
template int cd2d_kpartials<float>(const Geom&);
template int cd2d_kpartials<double>(const Geom&);
template int cd2d_norm_partials<float>(const Geom&);
template int cd2d_norm_partials<double>(const Geom&);
template cudaError_t cd2d_launch_norm<float>(const Geom&, const CdCoef<float>&, const float*, const float*,
                                             const float*, double*, int*, cudaStream_t);
template cudaError_t cd2d_launch_norm<double>(const Geom&, const CdCoef<double>&, const double*, const double*,
                                              const double*, double*, int*, cudaStream_t);

}  // namespace mg
