// kernels_pm2d.cu — warp-marching level operators for 2D levels (sm_100a).
//
// A 2D level is [planes = the paper's y][pitch], x fastest (mg_common.cuh).  A
// warp owns a strip of TX = 32 W columns (lane = one 16-byte vector of W =
// 16/sizeof(T) nodes) and marches a chunk of rows.  Rows arrive through a
// warp-private ring of NS shared-memory slots: lane 0 issues, per STEP of RB rows,
// one 2D TMA box load of u and one of f (cp.async.bulk.tensor.2d, RW = TX + 2W
// columns from x0 - W, zero-filled outside the array), completing on the slot's
// mbarrier.  The prefetch costs no registers, and the issue and wait cost is paid
// once per RB rows.  A lane reads its vector from the slot; its x-neighbours come
// from the adjacent lanes by warp shuffles (lanes 0 / 31 read the strip-edge nodes
// from the slot); the rows above and below stay in registers.  No block barriers:
// the warps of a CTA are independent.  A slot is refilled after the warp's
// __syncwarp that ends its reads of it.  Warps with consecutive ids take
// neighbouring strips of the same chunk and the launch is one wave of resident
// warps (rows split evenly), so strip-edge and chunk-halo re-reads hit L2.
//
//  k_jacobi2d          omega-Jacobi sweep, optionally with the residual-norm
//                      partials of its input; MODE 2: norm partials only
//  k_rbgs2d            one red-black Gauss-Seidel sweep in ONE pass (listing P:299-305):
//                      red of row t, then black of row t-1 from the red rows t-2..t,
//                      all in registers
//  k_resid_restrict2d  r = f - A u (Alg. 1 line 4) and full weighting:
//                      read u, f; write f_H (r never leaves registers)
//  k_prolong2d         uout = uin + P e, bilinear
// Arithmetic is the canonical per-point order of mg_common.cuh with explicitly
// rounded intrinsics (no FMA): bitwise identical to the op-by-op kernels and the oracle.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "kernels_pm.h"
#include "kernels_pm2d.h"
#include "launch_util.h"
#include "tma.cuh"
#include "vec.cuh"

namespace mg {
namespace pm2 {

#ifndef MG_PM2_RB
#define MG_PM2_RB 4
#endif
#ifndef MG_PM2_NS
#define MG_PM2_NS 3
#endif
constexpr int WPB = 4;          // warps per CTA
constexpr int NT = 32 * WPB;
constexpr int RB = MG_PM2_RB;   // rows per step (one TMA box of u and one of f)
constexpr int NS = MG_PM2_NS;   // ring slots per warp
constexpr unsigned FULL = 0xffffffffu;

template <typename T>
struct G2 {
  static constexpr int W = 16 / (int)sizeof(T);  // nodes per lane
  static constexpr int TX = 32 * W;              // strip width (64 FP64 / 128 FP32)
  static constexpr int NR = W / 2;               // coarse nodes per lane (restriction)
  static constexpr int RW = TX + 2 * W;          // box row: x in [x0 - W, x0 + TX + W)
  static constexpr int BOX = RW * RB;            // elements per box
  static constexpr int BOXB = BOX * (int)sizeof(T);  // 2176 B
  static constexpr int WARP_BYTES = NS * 2 * BOXB + 128;  // slots (u box, f box) + mbarriers
  static constexpr int SMEM = WPB * WARP_BYTES;
};

template <typename T>
using VT = Vec<T, 16 / sizeof(T)>;

template <typename T>
__device__ __forceinline__ VT<T> zvec() {
  VT<T> z;
#pragma unroll
  for (int k = 0; k < 16 / (int)sizeof(T); k++) z.v[k] = (T)0;
  return z;
}

// 2D operator, canonical order: s = cx*(l+r); s = s + cz*(m+p); A u = D*u - s
// (m, p: the rows below / above, i.e. the paper's y neighbours on the plane axis)
template <typename T>
__device__ __forceinline__ T A2(const Coef<T>& c, T ctr, T l, T r, T m, T p) {
  T s = mul(c.cx, add(l, r));
  s = add(s, mul(c.cz, add(m, p)));
  return sub(mul(c.D, ctr), s);
}
// u + wd*(f - A u)
template <typename T>
__device__ __forceinline__ T relax2(const Coef<T>& c, T ctr, T l, T r, T m, T p, T f) {
  return add(ctr, mul(c.wd, sub(f, A2(c, ctr, l, r, m, p))));
}

// warp gw -> strip and rows [pa, pb) of [lo, hi); consecutive warps: neighbouring strips
__device__ __forceinline__ void item2(int gw, int nstrips, int nch, int lo, int hi, int& strip, int& pa, int& pb) {
  strip = gw % nstrips;
  const int ch = gw / nstrips;
  const long long n = hi - lo;
  pa = lo + (int)(n * ch / nch);
  pb = lo + (int)(n * (ch + 1) / nch);
}

// left / right x-neighbours of a lane's vector: adjacent lanes, or lx / rx at the strip edges
template <typename T>
__device__ __forceinline__ void edges(const VT<T>& v, T lx, T rx, int lane, T& l, T& r) {
  constexpr int W = G2<T>::W;
  l = __shfl_up_sync(FULL, v.v[W - 1], 1);
  r = __shfl_down_sync(FULL, v.v[0], 1);
  if (lane == 0) l = lx;
  if (lane == 31) r = rx;
}

// fixed-order block reduction of the per-thread sums -> partial[blockIdx.x]
__device__ __forceinline__ void block_partial(double nsum, double* partial) {
  __shared__ double red[WPB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nsum = __dadd_rn(nsum, __shfl_down_sync(FULL, nsum, o));
  if (lane == 0) red[wid] = nsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < WPB; w++) t = __dadd_rn(t, red[w]);
    partial[blockIdx.x] = t;
  }
}

// ---------------------------------------------------------------------------
// The warp's ring.  A warp marching rows t0 .. tlast uses steps b = -1, 0, 1, ...:
// step b holds u rows t0 + b RB + 1 .. + RB and (b >= 0) f rows t0 + b RB .. + RB - 1,
// so row t = t0 + b RB + i reads u(t+1) and f(t) from box row i of step b, and step -1
// supplies u(t0 - RB + 1 .. t0) for the registers the march starts with.  Step b lives
// in slot (n0 + b + 1) % NS, mbarrier phase ((n0 + b + 1) / NS) & 1 (n0: steps of the
// warp's earlier items).
template <typename T, int RBR = RB>
struct WRing {
  struct G {  // G2<T> with RBR rows per box; slots 128-B aligned (TMA destinations)
    static constexpr int BOXB = G2<T>::RW * RBR * (int)sizeof(T);
    static constexpr int SLOTB = (BOXB + 127) / 128 * 128;
    static constexpr int BOX = SLOTB / (int)sizeof(T);  // slot stride in elements
  };
  static constexpr int WARP_BYTES = NS * 2 * G::SLOTB + 128;
  static constexpr int SMEM = WPB * WARP_BYTES;
  T* buf;
  uint64_t* bar;
  uint32_t n0;
  int t0, x;  // first row of the march, box x start (x0 - W)

  __device__ void init(unsigned char* smem, int wid, int lane) {
    unsigned char* w = smem + wid * WARP_BYTES;
    buf = reinterpret_cast<T*>(w);
    bar = reinterpret_cast<uint64_t*>(w + NS * 2 * G::SLOTB);
    n0 = 0;
    if (lane == 0) {
      for (int s = 0; s < NS; s++) mbar_init(&bar[s], 1);
      fence_barrier_init();
    }
    __syncwarp();
  }
  __device__ uint32_t N(int b) const { return n0 + (uint32_t)(b + 1); }
  __device__ T* U(int b) const { return buf + (N(b) % NS) * (2 * G::BOX); }
  __device__ T* F(int b) const { return U(b) + G::BOX; }
  __device__ void wait(int b) const { mbar_wait(&bar[N(b) % NS], (N(b) / NS) & 1u); }
  // lane 0: the loads of step b (u unless !load_u; f when b >= 0)
  __device__ void issue(int b, const CUtensorMap* tu, const CUtensorMap* tf, bool load_u) const {
    uint64_t* br = &bar[N(b) % NS];
    const bool lf = b >= 0;
    mbar_expect_tx(br, (uint32_t)((load_u ? G::BOXB : 0) + (lf ? G::BOXB : 0)));
    if (load_u) tma_load_2d(U(b), tu, x, t0 + b * RBR + 1, br);
    if (lf) tma_load_2d(F(b), tf, x, t0 + b * RBR, br);
  }
  // lane 0: steps -1 .. NS-2 (all slots)
  __device__ void start(int nsteps, const CUtensorMap* tu, const CUtensorMap* tf, bool load_u) const {
    for (int b = -1; b < NS - 1 && b < nsteps; b++) issue(b, tu, tf, load_u);
  }
  // after the reads of step b: refill its slot with step b + NS
  __device__ void release(int b, int nsteps, int lane, const CUtensorMap* tu, const CUtensorMap* tf,
                          bool load_u) const {
    __syncwarp();
    if (lane == 0 && b + NS < nsteps) issue(b + NS, tu, tf, load_u);
  }
  __device__ void finish(int nsteps) { n0 = N(nsteps - 1) + 1; }
};

template <typename T>
__device__ __forceinline__ void prefetch_maps(const CUtensorMap* a, const CUtensorMap* b, int lane) {
  if (lane == 0) {
    prefetch_tmap(a);
    prefetch_tmap(b);
  }
}

// ---------------------------------------------------------------------------
// MODE 0: Jacobi sweep uin -> uout; MODE 2: residual-norm partials only.
// ZERO: the input iterate is 0 (first sweep after V_H(0, ...)), u not read.
// NRM (MODE 0): also the norm partials of the sweep's INPUT (fused head sweep).
template <typename T, int MODE, bool ZERO, bool NRM>
__global__ void __launch_bounds__(NT) k_jacobi2d(const __grid_constant__ CUtensorMap tm_u,
                                                 const __grid_constant__ CUtensorMap tm_f, Geom g, Coef<T> c,
                                                 T* __restrict__ uout, int nstrips, int nch,
                                                 double* __restrict__ partial) {
  using V = VT<T>;
  constexpr int W = G2<T>::W, TX = G2<T>::TX, RW = G2<T>::RW;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WRing<T> R;
  R.init(smem, wid, lane);
  prefetch_maps<T>(&tm_u, &tm_f, lane);
  const int vo = W + W * lane;                // the lane's vector in a box row
  const int eo = lane == 0 ? W - 1 : W + TX;  // strip-edge node (lane 0: x0-1, lane 31: x0+TX)
  double nsum = 0.0;
  for (int gw = blockIdx.x * WPB + wid; gw < nstrips * nch; gw += gridDim.x * WPB) {
    int strip, pa, pb;
    item2(gw, nstrips, nch, g.p_lo, g.p_hi, strip, pa, pb);
    const int x0 = strip * TX, ox = x0 + W * lane;
    bool in[W];
#pragma unroll
    for (int j = 0; j < W; j++) in[j] = ox + j >= 1 && ox + j <= g.nx - 1;
    const bool okv = ox <= g.nx;
    R.t0 = pa;
    R.x = x0 - W;
    const int nsteps = (pb - 1 - pa) / RB + 1;
    if (lane == 0) R.start(nsteps, &tm_u, &tm_f, !ZERO);
    auto urow = [&](const T* row, T& e) -> V {
      if (ZERO) {
        e = (T)0;
        return zvec<T>();
      }
      e = row[eo];
      return ld_vec(row + vo);
    };
    T ume, u0s;
    R.wait(-1);
    V um = urow(R.U(-1) + (RB - 2) * RW, ume);  // u(pa-1)
    V u0 = urow(R.U(-1) + (RB - 1) * RW, u0s);  // u(pa)
    R.release(-1, nsteps, lane, &tm_u, &tm_f, !ZERO);
    for (int b = 0; b < nsteps; b++) {
      R.wait(b);
      const T* Ub = R.U(b);
      const T* Fb = R.F(b);
#pragma unroll
      for (int i = 0; i < RB; i++) {
        const int p = pa + b * RB + i;
        if (p >= pb) break;
        T ups;
        const V up = urow(Ub + i * RW, ups);
        const V fv = ld_vec(Fb + i * RW + vo);
        T l0, r0;
        edges(u0, u0s, u0s, lane, l0, r0);
        V o;
#pragma unroll
        for (int j = 0; j < W; j++) {
          const T l = j == 0 ? l0 : u0.v[j > 0 ? j - 1 : 0];
          const T r = j == W - 1 ? r0 : u0.v[j < W - 1 ? j + 1 : 0];
          const T rr = sub(fv.v[j], A2(c, u0.v[j], l, r, um.v[j], up.v[j]));
          if ((MODE == 2 || NRM) && in[j]) nsum = acc_sq<T>(nsum, rr);
          o.v[j] = in[j] ? add(u0.v[j], mul(c.wd, rr)) : u0.v[j];
        }
        if (MODE != 2 && okv) store_vec(uout + (long long)p * g.pstride, ox, in, o);
        um = u0;
        u0 = up;
        u0s = ups;
      }
      R.release(b, nsteps, lane, &tm_u, &tm_f, !ZERO);
    }
    R.finish(nsteps);
  }
  if (MODE == 2 || NRM) block_partial(nsum, partial);
}

// ---------------------------------------------------------------------------
// K omega-Jacobi sweeps in ONE pass (temporal blocking in registers; 2 <= K <= W + 1).
// Stage k (k = 1..K) is the k-th sweep; at iteration t stage k relaxes row t-k+1 from
// stage k-1's rows t-k .. t-k+2, kept in a 3-row register window per stage.  Strips
// OVERLAP: a warp covers TX columns from x0 but only its lanes 1..30 store (columns
// x0+W .. x0+TX-W-1), so the strip stride is TX - 2W.  A stage-k value is exact at least
// K-1 <= W columns inside the strip's box, hence exact on every stored column; the outer
// lanes' values are used only as neighbours of values that are discarded.  No lane-divergent
// edge code.  Every value is a single sweep's canonical arithmetic: bitwise equal to K
// launches of k_jacobi2d.  u, f read once, u^(K) written once: 3 words for K sweeps.
// ZERO: the input iterate is 0 (first sweeps after V_H(0, ...)), u not read.
// NRM: also the norm partials of the INPUT's residual f - A u, from stage 1 on the nodes
// the warp stores (fused head of the pipelined solve: sweep + ||r|| of its input).
// CORR: the input is u + P e (Alg. 1 line 6): stage 0 of every row is
// corrected in registers as it arrives, in k_prolong2d's order (x, then y, then the add),
// so the corrected iterate never makes an HBM round trip (prolongation fused into the
// first post-smoothing pass; e read from L2/HBM once, a quarter word per node).
// RR (K <= W-1): also r = f - A u^(K) of the pass's result (Alg. 1 line 4) and its full
// weighting into the coarse f — k_resid_restrict2d's values and order — as one
// more stage: r of row t-K from the stage-K window, its x-sums (lane shuffles), the last
// three in registers, fine row 2J+1 completing coarse row J.  The march runs 2 rows further
// on each side so r is exact on rows pa-1 .. pb; each coarse row is written by the chunk
// holding its centre row 2J, each coarse column by the lane storing fine column 2I.
template <typename T, int K, bool ZERO, bool NRM, bool CORR, bool RR = false>
__global__ void __launch_bounds__(NT) k_jacobi2d_k(const __grid_constant__ CUtensorMap tm_u,
                                                   const __grid_constant__ CUtensorMap tm_f, Geom g, Coef<T> c,
                                                   T* __restrict__ uout, int nstrips, int nch,
                                                   double* __restrict__ partial, const T* __restrict__ ec, Geom gc,
                                                   T* __restrict__ fcout) {
  using V = VT<T>;
  constexpr int W = G2<T>::W, TX = G2<T>::TX, RW = G2<T>::RW, SX = TX - 2 * W, NRC = W / 2;
  static_assert(K >= 2 && K <= W + 1, "overlap W columns per side");
  static_assert(!RR || K <= W - 1, "r of the stored columns needs u^(K) one column further in");
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int R3 = 3;  // rows per box = the window period: a row's window slots are static
  WRing<T, R3> R;
  R.init(smem, wid, lane);
  prefetch_maps<T>(&tm_u, &tm_f, lane);
  const int vo = W + W * lane;                // the lane's vector in a box row
  const int eo = lane == 0 ? W - 1 : W + TX;  // the column beyond the strip (stage-0 neighbour)
  const bool stores = lane >= 1 && lane <= 30;
  double nsum = 0.0;
  for (int gw = blockIdx.x * WPB + wid; gw < nstrips * nch; gw += gridDim.x * WPB) {
    int strip, pa, pb;
    item2(gw, nstrips, nch, g.p_lo, g.p_hi, strip, pa, pb);
    const int x0 = strip * SX - W, ox = x0 + W * lane;
    bool in[W], any = false;
#pragma unroll
    for (int j = 0; j < W; j++) {
      in[j] = ox + j >= 1 && ox + j <= g.nx - 1;
      any = any || in[j];
    }
    const int ts = pa - K + 1 - (RR ? 2 : 0), te = pb + K - 2 + (RR ? 2 : 0);  // stage-1 rows (= iterations)
    R.t0 = ts;
    R.x = x0 - W;
    const int nsteps = (te - ts) / R3 + 1;
    if (lane == 0) R.start(nsteps, &tm_u, &tm_f, !ZERO);
    auto urow = [&](const T* r, T& e) -> V {
      if (ZERO) {
        e = (T)0;
        return zvec<T>();
      }
      e = r[eo];
      return ld_vec(r + vo);
    };
    // ---- CORR: coarse rows interpolated along x at the lane's columns (V) and at its
    // strip-edge column (lanes 0 / 31); cA = V(cz), cB = V(cz + 1).  Rows advance by one, so
    // cz advances by at most one per row: one refill site, predicated loads, no branches
    const int X = ox >> 1, xe = lane == 0 ? x0 - 1 : x0 + TX, Xe = xe >> 1;
    const bool ein = xe >= 1 && xe <= g.nx - 1, eok = (lane == 0 || lane == 31) && ein;
    bool xok[W / 2 + 1];
#pragma unroll
    for (int i = 0; i <= W / 2; i++) xok[i] = X + i >= 0 && X + i <= gc.nx;
    const T half = (T)0.5;
    auto Vrow = [&](int Z, T& es) -> V {
      const bool rok = Z >= 0 && Z <= gc.nz;
      const T* p0 = ec + (long long)((rok ? Z : gc.p_glob0) - gc.p_glob0) * gc.pstride;
      T a[W / 2 + 1];
#pragma unroll
      for (int i = 0; i <= W / 2; i++) a[i] = (rok && xok[i]) ? __ldg(p0 + X + i) : (T)0;
      V v;
#pragma unroll
      for (int i = 0; i < W / 2; i++) {
        v.v[2 * i] = a[i];
        v.v[2 * i + 1] = mul(half, add(a[i], a[i + 1]));
      }
      const T e1 = (rok && eok) ? __ldg(p0 + Xe) : (T)0;
      const T e2 = (rok && eok && (xe & 1)) ? __ldg(p0 + Xe + 1) : (T)0;
      es = (xe & 1) ? mul(half, add(e1, e2)) : e1;
      return v;
    };
    int cz = 0;
    V cA, cB;
    T eA = (T)0, eB = (T)0;
    if (CORR) {  // prime: cB = V(Z(ts - 1)), so the first row's advance makes it cA
      cz = ((ts - 1 + g.p_glob0) >> 1) - 1;
      cB = Vrow(cz + 1, eB);
    }
    auto correct = [&](V& v, T& es, int row) {  // stage 0 of local row `row` += P e
      const int zg = row + g.p_glob0, Z = zg >> 1;
      if (Z != cz) {
        cA = cB;
        eA = eB;
        cB = Vrow(Z + 1, eB);
        cz = Z;
      }
      const bool zin = zg >= 1 && zg <= g.nz - 1;
      const bool odd = zg & 1;
#pragma unroll
      for (int j = 0; j < W; j++) {
        const T pv = odd ? mul(half, add(cA.v[j], cB.v[j])) : cA.v[j];
        v.v[j] = selv(zin && in[j], add(v.v[j], pv), v.v[j]);
      }
      const T pe = odd ? mul(half, add(eA, eB)) : eA;
      es = selv(zin && ein, add(es, pe), es);
    };
    // window slot of a row: (row - ts + 1) mod 3; S[k][slot] stage k, e0[slot] stage-0 edge
    V S[K + 1][3];
    T e0[3];
    V Fw[3] = {};  // (early slots feed only values that are never stored)
    V Fold;                      // RR with K = 3: f of row t-3 (its window slot is reused by row t)
    T ty1[NRC], ty2[NRC];        // RR: x-sums of the two previous residual rows
#pragma unroll
    for (int i = 0; i < NRC; i++) ty1[i] = ty2[i] = (T)0;
    const T two = (T)2, scale = (T)(1.0 / 16.0);
    R.wait(-1);
    S[0][0] = urow(R.U(-1) + 1 * RW, e0[0]);  // row ts-1
    S[0][1] = urow(R.U(-1) + 2 * RW, e0[1]);  // row ts
    if (CORR) {
      correct(S[0][0], e0[0], ts - 1);
      correct(S[0][1], e0[1], ts);
    }
    R.release(-1, nsteps, lane, &tm_u, &tm_f, !ZERO);
    auto iter = [&](auto PHc, int t, const T* ur, const T* fr) {
      constexpr int PH = decltype(PHc)::value;
      S[0][(PH + 2) % 3] = urow(ur, e0[(PH + 2) % 3]);  // stage 0, row t+1
      if (CORR) correct(S[0][(PH + 2) % 3], e0[(PH + 2) % 3], t + 1);
      if (RR && K == 3) Fold = Fw[(PH + 1) % 3];        // f, row t-3
      Fw[(PH + 1) % 3] = ld_vec(fr + vo);               // f, row t
#pragma unroll
      for (int k = 1; k <= K; k++) {
        const int sm = (PH - k + 1 + 6) % 3, s0 = (PH - k + 2 + 6) % 3, sp = (PH - k + 6) % 3;
        const V& P0 = S[k - 1][s0];
        const int rg = t - k + 1 + g.p_glob0;
        const bool rin = rg >= 1 && rg <= g.nz - 1;
        T l0 = __shfl_up_sync(FULL, P0.v[W - 1], 1), r0 = __shfl_down_sync(FULL, P0.v[0], 1);
        if (k == 1) {  // the box supplies the stage-0 columns beyond the strip; later stages'
          if (lane == 0) l0 = e0[s0];  // out-of-strip neighbours only feed discarded values
          if (lane == 31) r0 = e0[s0];
        }
        V o;
#pragma unroll
        for (int j = 0; j < W; j++) {
          const T l = j == 0 ? l0 : P0.v[j > 0 ? j - 1 : 0];
          const T r = j == W - 1 ? r0 : P0.v[j < W - 1 ? j + 1 : 0];
          const T ctr = P0.v[j];
          const T rr = sub(Fw[s0].v[j], A2(c, ctr, l, r, S[k - 1][sm].v[j], S[k - 1][sp].v[j]));
          o.v[j] = selv(rin && in[j], add(ctr, mul(c.wd, rr)), ctr);
          if (NRM && k == 1) {  // stage 1 row t: the input's residual on the stored nodes
            const double d = selv(stores && rin && in[j] && t >= pa && t < pb, (double)rr, 0.0);
            nsum = __fma_rn(d, d, nsum);  // FP32 rr: d*d is exact, = dadd(nsum, dmul(d, d))
          }
        }
        S[k][s0] = o;
      }
      const int ro = t - K + 1;  // the stage-K row of this iteration
      if (stores && any && ro >= pa && ro < pb) store_vec(uout + (long long)ro * g.pstride, ox, in, S[K][(PH - K + 8) % 3]);
      if constexpr (RR) {  // residual of row t-K from stage-K rows t-K-1 .. t-K+1, restriction
        constexpr int s0 = (PH - K + 1 + 9) % 3, sm = (PH - K + 9) % 3, sp = (PH - K + 2 + 9) % 3;
        const V& P0 = S[K][s0];
        const V& Fr = K == 3 ? Fold : Fw[(PH + 3 - K + 1) % 3];
        const int rg = t - K + g.p_glob0;
        const bool rin = rg >= 1 && rg <= g.nz - 1;
        const T l0 = __shfl_up_sync(FULL, P0.v[W - 1], 1), r0 = __shfl_down_sync(FULL, P0.v[0], 1);
        V rv;
#pragma unroll
        for (int j = 0; j < W; j++) {
          const T l = j == 0 ? l0 : P0.v[j > 0 ? j - 1 : 0];
          const T r = j == W - 1 ? r0 : P0.v[j < W - 1 ? j + 1 : 0];
          rv.v[j] = selv(rin && in[j], sub(Fr.v[j], A2(c, P0.v[j], l, r, S[K][sm].v[j], S[K][sp].v[j])), (T)0);
        }
        const T rl = __shfl_up_sync(FULL, rv.v[W - 1], 1);  // r(ox - 1): exact for lanes 1..30
        T tx[NRC];
#pragma unroll
        for (int i = 0; i < NRC; i++) {
          const T left = i == 0 ? rl : rv.v[i > 0 ? 2 * i - 1 : 0];
          tx[i] = add(add(left, rv.v[2 * i + 1]), mul(two, rv.v[2 * i]));
        }
        if ((rg & 1) == 1) {  // fine row 2J+1 completes coarse row J
          const int J = (rg - 1) >> 1, cr = 2 * J - g.p_glob0;  // the centre row, local
          if (stores && cr >= pa && cr < pb && J >= 1 && J <= gc.nz - 1) {
            T* crow = fcout + (long long)(J - gc.p_glob0) * gc.pstride;
#pragma unroll
            for (int i = 0; i < NRC; i++) {
              const int I = (ox >> 1) + i;
              if (I >= 1 && I <= gc.nx - 1) crow[I] = mul(add(add(ty2[i], tx[i]), mul(two, ty1[i])), scale);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < NRC; i++) {
          ty2[i] = ty1[i];
          ty1[i] = tx[i];
        }
      }
    };
    // rows past te (in the last box) compute values that are never stored
    for (int b = 0; b < nsteps; b++) {
      R.wait(b);
      const T* Ub = R.U(b);
      const T* Fb = R.F(b);
      const int t = ts + b * R3;
      iter(std::integral_constant<int, 0>(), t, Ub, Fb);
      iter(std::integral_constant<int, 1>(), t + 1, Ub + RW, Fb + RW);
      iter(std::integral_constant<int, 2>(), t + 2, Ub + 2 * RW, Fb + 2 * RW);
      R.release(b, nsteps, lane, &tm_u, &tm_f, !ZERO);
    }
    R.finish(nsteps);
  }
  if (NRM) block_partial(nsum, partial);
}

// ---------------------------------------------------------------------------
// One red-black GS sweep uin -> uout in one pass.  Iteration t computes the red
// nodes of row t ("post-red" row pr(t): red entries relaxed, black entries old) and
// then the black nodes of row t-1 from pr(t-2), pr(t-1), pr(t); rows pa-1 and pb get
// their red nodes only (neighbour chunks' rows, recomputed, never written).  Colour:
// red = even global i + j (reading 8); strips start at even x, so the colour of a
// lane's element j in row t is (j + t + p_glob0) & 1, uniform over the warp.
// Strip-edge (ring) nodes: lane 0 relaxes x0-1, lane 31 x0+TX when they are red.
template <typename T, bool ZERO, bool NRM>
__global__ void __launch_bounds__(NT) k_rbgs2d(const __grid_constant__ CUtensorMap tm_u,
                                               const __grid_constant__ CUtensorMap tm_f, Geom g, Coef<T> c,
                                               T* __restrict__ uout, int nstrips, int nch,
                                               double* __restrict__ partial) {
  using V = VT<T>;
  constexpr int W = G2<T>::W, TX = G2<T>::TX, NR = G2<T>::NR, RW = G2<T>::RW;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WRing<T> R;
  R.init(smem, wid, lane);
  prefetch_maps<T>(&tm_u, &tm_f, lane);
  const int vo = W + W * lane;
  // ring node e1 and its outer neighbour e2: lane 0 (x0-1, x0-2), lane 31 (x0+TX, x0+TX+1)
  const int e1o = lane == 0 ? W - 1 : W + TX, e2o = lane == 0 ? W - 2 : W + TX + 1;
  double nsum = 0.0;
  for (int gw = blockIdx.x * WPB + wid; gw < nstrips * nch; gw += gridDim.x * WPB) {
    int strip, pa, pb;
    item2(gw, nstrips, nch, g.p_lo, g.p_hi, strip, pa, pb);
    const int x0 = strip * TX, ox = x0 + W * lane;
    const int pg0 = g.p_glob0;
    bool in[W];
#pragma unroll
    for (int j = 0; j < W; j++) in[j] = ox + j >= 1 && ox + j <= g.nx - 1;
    const bool okv = ox <= g.nx;
    const bool ring_ok = lane == 0 ? x0 - 1 >= 1 : (lane == 31 && x0 + TX <= g.nx - 1);
    auto plin = [&](int p) {
      const int pg = p + pg0;
      return pg >= 1 && pg <= g.nz - 1;
    };
    R.t0 = pa - 1;
    R.x = x0 - W;
    const int nsteps = (pb - (pa - 1)) / RB + 1;
    if (lane == 0) R.start(nsteps, &tm_u, &tm_f, !ZERO);
    auto urow = [&](const T* row, T& e1, T& e2) -> V {
      if (ZERO) {
        e1 = e2 = (T)0;
        return zvec<T>();
      }
      e1 = row[e1o];
      e2 = row[e2o];
      return ld_vec(row + vo);
    };
    T Bx1, Bx2, Cx1, Cx2;
    R.wait(-1);
    V B = urow(R.U(-1) + (RB - 2) * RW, Bx1, Bx2);  // u(pa-2) = pr(pa-2) at its black (old) entries
    V Bo = B;                                       // u_old(t-1) (NRM)
    V C = urow(R.U(-1) + (RB - 1) * RW, Cx1, Cx2);  // u_old(pa-1)
    R.release(-1, nsteps, lane, &tm_u, &tm_f, !ZERO);
    V A = zvec<T>();     // pr(t-2)
    V Fm1 = zvec<T>();   // f(t-1)
    T ring_prev = (T)0;  // relaxed ring node of row t-1 (when red)
    for (int b = 0; b < nsteps; b++) {
      R.wait(b);
      const T* Ub = R.U(b);
      const T* Fb = R.F(b);
#pragma unroll
      for (int i = 0; i < RB; i++) {
        const int t = pa - 1 + b * RB + i;
        if (t > pb) break;
        T Dx1, Dx2;
        const V Dn = urow(Ub + i * RW, Dx1, Dx2);  // u_old(t+1)
        const V fv = ld_vec(Fb + i * RW + vo);
        const T fe = Fb[i * RW + e1o];
        const bool pin = plin(t);
        T Cl, Cr;
        edges(C, Cx1, Cx1, lane, Cl, Cr);
        if (NRM && t >= pa && t < pb) {  // ||f - A u_in||^2 of row t (all old values)
#pragma unroll
          for (int j = 0; j < W; j++) {
            const T l = j == 0 ? Cl : C.v[j > 0 ? j - 1 : 0];
            const T r = j == W - 1 ? Cr : C.v[j < W - 1 ? j + 1 : 0];
            const T rr = sub(fv.v[j], A2(c, C.v[j], l, r, Bo.v[j], Dn.v[j]));
            if (in[j]) nsum = acc_sq<T>(nsum, rr);
          }
        }
        V prT = C;
        T ring_cur = Cx1;
        auto body = [&](auto KRc) {
          constexpr int KR = decltype(KRc)::value;  // red elements of row t: j = KR + 2m
          if (pin) {
#pragma unroll
            for (int m = 0; m < NR; m++) {
              const int j = KR + 2 * m;
              const T l = j == 0 ? Cl : C.v[j > 0 ? j - 1 : 0];
              const T r = j == W - 1 ? Cr : C.v[j < W - 1 ? j + 1 : 0];
              if (in[j]) prT.v[j] = relax2(c, C.v[j], l, r, B.v[j], Dn.v[j], fv.v[j]);
            }
            // ring node: lane 0's x0-1 is red in row t iff KR == 1, lane 31's x0+TX iff KR == 0
            if (ring_ok && ((lane == 0) == (KR == 1)))
              ring_cur = lane == 0 ? relax2(c, Cx1, Cx2, C.v[0], Bx1, Dx1, fe)
                                   : relax2(c, Cx1, C.v[W - 1], Cx2, Bx1, Dx1, fe);
          }
          if (t - 1 >= pa) {  // black nodes of row t-1: the same elements j = KR + 2m
            T Bl, Br;
            edges(B, ring_prev, ring_prev, lane, Bl, Br);
            V o = B;
#pragma unroll
            for (int m = 0; m < NR; m++) {
              const int j = KR + 2 * m;
              const T l = j == 0 ? Bl : B.v[j > 0 ? j - 1 : 0];
              const T r = j == W - 1 ? Br : B.v[j < W - 1 ? j + 1 : 0];
              if (in[j]) o.v[j] = relax2(c, B.v[j], l, r, A.v[j], prT.v[j], Fm1.v[j]);
            }
            if (okv) store_vec(uout + (long long)(t - 1) * g.pstride, ox, in, o);
          }
        };
        if ((t + pg0) & 1)
          body(std::integral_constant<int, 1>());
        else
          body(std::integral_constant<int, 0>());
        A = B;
        B = prT;
        if (NRM) Bo = C;
        Bx1 = Cx1;
        Bx2 = Cx2;
        C = Dn;
        Cx1 = Dx1;
        Cx2 = Dx2;
        Fm1 = fv;
        ring_prev = ring_cur;
      }
      R.release(b, nsteps, lane, &tm_u, &tm_f, !ZERO);
    }
    R.finish(nsteps);
  }
  if (NRM) block_partial(nsum, partial);
}

// ---------------------------------------------------------------------------
// Fused residual + full weighting.  Warp = a coarse strip (TX/2 coarse nodes = the
// fine strip x0 .. x0+TX) and a chunk [Pa, Pb) of coarse rows.  Per fine row t: r of
// the lane's W nodes (lane 0 also r(x0-1)), the x-sums of its NR coarse nodes, and
// the last three x-sums in registers; fine row 2J+1 completes coarse row J.
template <typename T>
__global__ void __launch_bounds__(NT) k_resid_restrict2d(const __grid_constant__ CUtensorMap tm_u,
                                                         const __grid_constant__ CUtensorMap tm_f, Geom gf, Geom gc,
                                                         Coef<T> c, T* __restrict__ fc, int nstrips, int nch) {
  using V = VT<T>;
  constexpr int W = G2<T>::W, TX = G2<T>::TX, NR = G2<T>::NR, RW = G2<T>::RW;
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WRing<T> R;
  R.init(smem, wid, lane);
  prefetch_maps<T>(&tm_u, &tm_f, lane);
  const int vo = W + W * lane;
  const int e1o = lane == 0 ? W - 1 : W + TX, e2o = lane == 0 ? W - 2 : W + TX + 1;
  const T two = (T)2, scale = (T)(1.0 / 16.0);
  for (int gw = blockIdx.x * WPB + wid; gw < nstrips * nch; gw += gridDim.x * WPB) {
    int strip, Pa, Pb;
    item2(gw, nstrips, nch, gc.p_lo, gc.p_hi, strip, Pa, Pb);
    const int x0 = strip * TX, ox = x0 + W * lane;
    bool in[W];
#pragma unroll
    for (int j = 0; j < W; j++) in[j] = ox + j >= 1 && ox + j <= gf.nx - 1;
    const bool ring_ok = lane == 0 && x0 - 1 >= 1;  // r(x0-1) is an interior residual
    auto plin = [&](int t) {
      const int tg = t + gf.p_glob0;
      return tg >= 1 && tg <= gf.nz - 1;
    };
    const int qf0 = 2 * (Pa + gc.p_glob0) - gf.p_glob0;      // fine centre row of coarse row Pa
    const int qf1 = 2 * (Pb - 1 + gc.p_glob0) - gf.p_glob0;  // ... of coarse row Pb-1
    const int rlo = qf0 - 1, rhi = qf1 + 1;
    R.t0 = rlo;
    R.x = x0 - W;
    const int nsteps = (rhi - rlo) / RB + 1;
    if (lane == 0) R.start(nsteps, &tm_u, &tm_f, true);
    auto urow = [&](const T* row, T& e1, T& e2) -> V {
      e1 = row[e1o];
      e2 = row[e2o];
      return ld_vec(row + vo);
    };
    T umx1, umx2, u0x1, u0x2;
    R.wait(-1);
    V um = urow(R.U(-1) + (RB - 2) * RW, umx1, umx2);
    V u0 = urow(R.U(-1) + (RB - 1) * RW, u0x1, u0x2);
    R.release(-1, nsteps, lane, &tm_u, &tm_f, true);
    T ty1[NR], ty2[NR];
#pragma unroll
    for (int i = 0; i < NR; i++) ty1[i] = ty2[i] = (T)0;
    const int I0 = ox >> 1;
    for (int b = 0; b < nsteps; b++) {
      R.wait(b);
      const T* Ub = R.U(b);
      const T* Fb = R.F(b);
#pragma unroll
      for (int ii = 0; ii < RB; ii++) {
        const int t = rlo + b * RB + ii;
        if (t > rhi) break;
        T upx1, upx2;
        const V up = urow(Ub + ii * RW, upx1, upx2);
        const V fv = ld_vec(Fb + ii * RW + vo);
        const T fe = Fb[ii * RW + e1o];
        const bool pin = plin(t);
        T l0, r0;
        edges(u0, u0x1, u0x1, lane, l0, r0);
        V rv;
#pragma unroll
        for (int j = 0; j < W; j++) {
          const T l = j == 0 ? l0 : u0.v[j > 0 ? j - 1 : 0];
          const T r = j == W - 1 ? r0 : u0.v[j < W - 1 ? j + 1 : 0];
          const T rr = sub(fv.v[j], A2(c, u0.v[j], l, r, um.v[j], up.v[j]));
          rv.v[j] = pin && in[j] ? rr : (T)0;
        }
        T rx = (T)0;  // lane 0: r(x0-1)
        if (pin && ring_ok) rx = sub(fe, A2(c, u0x1, u0x2, u0.v[0], umx1, upx1));
        T rl = __shfl_up_sync(FULL, rv.v[W - 1], 1);
        if (lane == 0) rl = rx;
        T tx[NR];
#pragma unroll
        for (int i = 0; i < NR; i++) {
          const T left = i == 0 ? rl : rv.v[i > 0 ? 2 * i - 1 : 0];
          tx[i] = add(add(left, rv.v[2 * i + 1]), mul(two, rv.v[2 * i]));
        }
        const int tg = t + gf.p_glob0;
        if ((tg & 1) == 1 && t >= qf0 + 1) {  // fine row 2J+1 completes coarse row J
          const int J = (tg - 1) >> 1;
          T* crow = fc + (long long)(J - gc.p_glob0) * gc.pstride;
          if (J >= 1 && J <= gc.nz - 1) {
#pragma unroll
            for (int i = 0; i < NR; i++) {
              const int I = I0 + i;
              if (I >= 1 && I <= gc.nx - 1) crow[I] = mul(add(add(ty2[i], tx[i]), mul(two, ty1[i])), scale);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < NR; i++) {
          ty2[i] = ty1[i];
          ty1[i] = tx[i];
        }
        um = u0;
        umx1 = u0x1;
        u0 = up;
        u0x1 = upx1;
        u0x2 = upx2;
      }
      R.release(b, nsteps, lane, &tm_u, &tm_f, true);
    }
    R.finish(nsteps);
  }
}

// ---------------------------------------------------------------------------
// uout = uin + P e on interior fine nodes (uout == uin: in place; out of place, uout's
// boundary must already hold the Dirichlet data).  Fine row z = 2Z + dz gets
// dz ? (V(Z) + V(Z+1))/2 : V(Z), V(K) = coarse row K interpolated along x (reading 13
// order: x, then y).
template <typename T>
__global__ void __launch_bounds__(NT) k_prolong2d(Geom gf, Geom gc, const T* __restrict__ e, const T* uin, T* uout,
                                                  int nstrips, int nch) {
  using V = VT<T>;
  constexpr int W = G2<T>::W, TX = G2<T>::TX, NR = G2<T>::NR;
  const int lane = threadIdx.x & 31, gw = blockIdx.x * WPB + (threadIdx.x >> 5);
  if (gw >= nstrips * nch) return;
  int strip, pa, pb;
  item2(gw, nstrips, nch, gf.p_lo, gf.p_hi, strip, pa, pb);
  const int ox = strip * TX + W * lane;
  bool in[W], any = false, all = true;
#pragma unroll
  for (int j = 0; j < W; j++) {
    in[j] = ox + j >= 1 && ox + j <= gf.nx - 1;
    any = any || in[j];
    all = all && in[j];
  }
  if (!any) return;
  const T half = (T)0.5;
  const int X = ox >> 1;
  auto Vz = [&](int Zg) -> V {
    const T* p0 = e + (long long)(Zg - gc.p_glob0) * gc.pstride + X;
    T a[NR + 1];
#pragma unroll
    for (int i = 0; i <= NR; i++) a[i] = X + i <= gc.nx ? __ldg(p0 + i) : (T)0;
    V v;
#pragma unroll
    for (int i = 0; i < NR; i++) {
      v.v[2 * i] = a[i];
      v.v[2 * i + 1] = mul(half, add(a[i], a[i + 1]));
    }
    return v;
  };
  int Z = (pa + gf.p_glob0) >> 1;
  V Av = Vz(Z), Bv = Av;
  bool haveB = false;
  for (int z = pa; z < pb; z++) {
    const int zg = z + gf.p_glob0;
    if ((zg >> 1) != Z) {
      Z++;
      Av = haveB ? Bv : Vz(Z);
      haveB = false;
    }
    V v = Av;
    if (zg & 1) {
      if (!haveB) {
        Bv = Vz(Z + 1);
        haveB = true;
      }
#pragma unroll
      for (int j = 0; j < W; j++) v.v[j] = mul(half, add(Av.v[j], Bv.v[j]));
    }
    const T* ui = uin + (long long)z * gf.pstride;
    T* uo = uout + (long long)z * gf.pstride;
    if (all) {
      const V uu = ld_vec(ui + ox);
      V o;
#pragma unroll
      for (int j = 0; j < W; j++) o.v[j] = add(uu.v[j], v.v[j]);
      store_vec(uo, ox, in, o);
    } else {
#pragma unroll
      for (int j = 0; j < W; j++)
        if (in[j]) uo[ox + j] = add(ui[ox + j], v.v[j]);
    }
  }
}

// ---------------------------------------------------------------------------
// launch geometry: one wave of resident warps; rows split evenly, >= kMinRows per chunk
constexpr int kMinRows = 4;  // measured on C4: 16 -> 1.70 ms, 8 -> 1.63, 4 -> 1.61

template <class K>
static int resident_warps(K kernel, int smem) {
  return resident_ctas((const void*)kernel, NT, smem) * WPB;
}

static void split(int nstrips, int rows, int rw, int& nch, int& nblocks) {
  constexpr int min_rows = kMinRows;
  nch = rw / nstrips;
  const int cap = rows / min_rows;
  if (nch > cap) nch = cap;
  if (nch < 1) nch = 1;
  nblocks = (nstrips * nch + WPB - 1) / WPB;
}

template <typename T>
static int strips(const Geom& g) {
  return (g.nx + G2<T>::TX - 1) / G2<T>::TX;  // covers x in [0, nx): every interior column
}

// 2D tensor map of a level array: dims (nx+1, planes), box (RW, RB) — OOB reads are zero
// overlapping strips of the fused Jacobi passes: stride TX - 2W covering the columns 0 .. nx
template <typename T>
static int kstrips(const Geom& g) {
  constexpr int SX = G2<T>::TX - 2 * G2<T>::W;
  return (g.nx + 1 + SX - 1) / SX;
}

template <typename T>
static bool encode2d(CUtensorMap* tm, const T* base, const Geom& g, int rows = RB) {
  const unsigned long long dims[2] = {(unsigned long long)(g.nx + 1), (unsigned long long)g.planes};
  const unsigned long long strides[1] = {(unsigned long long)(g.pstride * sizeof(T))};
  const unsigned box[2] = {(unsigned)G2<T>::RW, (unsigned)rows};
  return pm::encode_tiled(tm, sizeof(T) == 8, 2, base, dims, strides, box) == CUDA_SUCCESS;
}

bool supported(const Geom& g, int min_nx) {
  return !g.three_d && g.nx >= (min_nx < 16 ? 16 : min_nx) && (g.p_hi - g.p_lo) >= 4;
}

template <typename T>
cudaError_t launch_sweep(const Geom& g, const Coef<T>& c, bool rbgs, const T* uin, const T* f, T* uout, bool zero_in,
                         cudaStream_t st, double* partial, int* npartial) {
  const bool nrm = partial && !zero_in;
  CUtensorMap tu, tf;
  if (!encode2d<T>(&tu, uin ? uin : f, g) || !encode2d<T>(&tf, f, g)) return cudaErrorInvalidValue;
  const int ns = strips<T>(g), smem = G2<T>::SMEM;
  int nch, nb;
  auto go = [&](auto kernel) {
    split(ns, g.p_hi - g.p_lo, resident_warps(kernel, smem), nch, nb);
    if (npartial) *npartial = nb;
    kernel<<<nb, NT, smem, st>>>(tu, tf, g, c, uout, ns, nch, partial);
  };
  if (rbgs) {
    if (nrm)
      go(k_rbgs2d<T, false, true>);
    else
      zero_in ? go(k_rbgs2d<T, true, false>) : go(k_rbgs2d<T, false, false>);
  } else {
    if (nrm)
      go(k_jacobi2d<T, 0, false, true>);
    else
      zero_in ? go(k_jacobi2d<T, 0, true, false>) : go(k_jacobi2d<T, 0, false, false>);
  }
  return cudaGetLastError();
}

template <typename T>
bool rr_fusable(int K) {
  return K >= 2 && K <= G2<T>::W - 1;
}

template <typename T>
cudaError_t launch_jacobi_k(const Geom& g, const Coef<T>& c, int K, const T* uin, const T* f, T* uout, bool zero_in,
                            cudaStream_t st, double* partial, int* npartial, const T* e, const Geom* gc, T* fc) {
  CUtensorMap tu, tf;
  if (!encode2d<T>(&tu, uin ? uin : f, g, 3) || !encode2d<T>(&tf, f, g, 3)) return cudaErrorInvalidValue;
  if ((partial && zero_in) || (e && (zero_in || partial || !gc)) || (fc && (e || !gc || !rr_fusable<T>(K))))
    return cudaErrorInvalidValue;
  const int ns = kstrips<T>(g);
  const int smem = WRing<T, 3>::SMEM;
  const Geom gcv = gc ? *gc : g;
  int nch, nb;
  auto go = [&](auto kernel) {
    split(ns, g.p_hi - g.p_lo, resident_warps(kernel, smem), nch, nb);
    kernel<<<nb, NT, smem, st>>>(tu, tf, g, c, uout, ns, nch, partial, e, gcv, fc);
  };
  auto goK = [&](auto Kc) {
    constexpr int KK = decltype(Kc)::value;
    if constexpr (KK <= G2<T>::W - 1) {  // RR variants (FP32: K = 2, 3)
      if (fc) {
        if (partial)
          go(k_jacobi2d_k<T, KK, false, true, false, true>);
        else
          zero_in ? go(k_jacobi2d_k<T, KK, true, false, false, true>) : go(k_jacobi2d_k<T, KK, false, false, false, true>);
        return;
      }
    }
    if (partial)
      go(k_jacobi2d_k<T, KK, false, true, false>);
    else if (e)
      go(k_jacobi2d_k<T, KK, false, false, true>);
    else
      zero_in ? go(k_jacobi2d_k<T, KK, true, false, false>) : go(k_jacobi2d_k<T, KK, false, false, false>);
  };
  if (K == 2)
    goK(std::integral_constant<int, 2>());
  else if constexpr (G2<T>::W >= 3) {
    if (K != 3) return cudaErrorInvalidValue;
    goK(std::integral_constant<int, 3>());
  } else {
    return cudaErrorInvalidValue;
  }
  if (npartial) *npartial = nb;
  return cudaGetLastError();
}

template <typename T>
int sweep_partials(const Geom& g, bool rbgs) {
  int nch, nb;
  const int smem = G2<T>::SMEM;
  const int rw = rbgs ? resident_warps(k_rbgs2d<T, false, true>, smem)
                      : resident_warps(k_jacobi2d<T, 0, false, true>, smem);
  split(strips<T>(g), g.p_hi - g.p_lo, rw, nch, nb);
  if (!rbgs) {  // the fused head (k_jacobi2d_k NRM, K = 2 or 3)
    int nb2;
    split(kstrips<T>(g), g.p_hi - g.p_lo, resident_warps(k_jacobi2d_k<T, 2, false, true, false>, WRing<T, 3>::SMEM), nch,
          nb2);
    nb = nb2 > nb ? nb2 : nb;
    if constexpr (G2<T>::W >= 3) {  // the head with the fused residual + restriction
      split(kstrips<T>(g), g.p_hi - g.p_lo,
            resident_warps(k_jacobi2d_k<T, 2, false, true, false, true>, WRing<T, 3>::SMEM), nch, nb2);
      nb = nb2 > nb ? nb2 : nb;
    }
    if constexpr (G2<T>::W >= 4) {
      split(kstrips<T>(g), g.p_hi - g.p_lo,
            resident_warps(k_jacobi2d_k<T, 3, false, true, false, true>, WRing<T, 3>::SMEM), nch, nb2);
    }
    nb = nb2 > nb ? nb2 : nb;
    if constexpr (G2<T>::W >= 3) {
      split(kstrips<T>(g), g.p_hi - g.p_lo, resident_warps(k_jacobi2d_k<T, 3, false, true, false>, WRing<T, 3>::SMEM), nch,
            nb2);
      nb = nb2 > nb ? nb2 : nb;
    }
  }
  return nb;
}

template <typename T>
cudaError_t launch_norm(const Geom& g, const Coef<T>& c, const T* u, const T* f, double* partial, int* npartial,
                        cudaStream_t st) {
  CUtensorMap tu, tf;
  if (!encode2d<T>(&tu, u, g) || !encode2d<T>(&tf, f, g)) return cudaErrorInvalidValue;
  auto kernel = k_jacobi2d<T, 2, false, false>;
  const int ns = strips<T>(g), smem = G2<T>::SMEM;
  int nch, nb;
  split(ns, g.p_hi - g.p_lo, resident_warps(kernel, smem), nch, nb);
  *npartial = nb;
  kernel<<<nb, NT, smem, st>>>(tu, tf, g, c, nullptr, ns, nch, partial);
  return cudaGetLastError();
}

template <typename T>
int norm_partials(const Geom& g) {
  int nch, nb;
  split(strips<T>(g), g.p_hi - g.p_lo, resident_warps(k_jacobi2d<T, 2, false, false>, G2<T>::SMEM), nch, nb);
  return nb;
}

template <typename T>
cudaError_t launch_resid_restrict(const Geom& gf, const Geom& gc, const Coef<T>& c, const T* u, const T* f, T* fc,
                                  cudaStream_t st) {
  CUtensorMap tu, tf;
  if (!encode2d<T>(&tu, u, gf) || !encode2d<T>(&tf, f, gf)) return cudaErrorInvalidValue;
  auto kernel = k_resid_restrict2d<T>;
  const int ns = strips<T>(gf), smem = G2<T>::SMEM;
  int nch, nb;
  split(ns, gc.p_hi - gc.p_lo, resident_warps(kernel, smem), nch, nb);
  kernel<<<nb, NT, smem, st>>>(tu, tf, gf, gc, c, fc, ns, nch);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_prolong(const Geom& gf, const Geom& gc, const T* e, const T* uin, T* uout, cudaStream_t st) {
  auto kernel = k_prolong2d<T>;
  const int ns = strips<T>(gf);
  int nch, nb;
  split(ns, gf.p_hi - gf.p_lo, resident_warps(kernel, 0), nch, nb);
  kernel<<<nb, NT, 0, st>>>(gf, gc, e, uin, uout, ns, nch);
  return cudaGetLastError();
}

template cudaError_t launch_sweep<double>(const Geom&, const Coef<double>&, bool, const double*, const double*,
                                          double*, bool, cudaStream_t, double*, int*);
template cudaError_t launch_sweep<float>(const Geom&, const Coef<float>&, bool, const float*, const float*, float*,
                                         bool, cudaStream_t, double*, int*);
template cudaError_t launch_jacobi_k<double>(const Geom&, const Coef<double>&, int, const double*, const double*,
                                             double*, bool, cudaStream_t, double*, int*, const double*, const Geom*,
                                             double*);
template cudaError_t launch_jacobi_k<float>(const Geom&, const Coef<float>&, int, const float*, const float*, float*,
                                            bool, cudaStream_t, double*, int*, const float*, const Geom*, float*);
template bool rr_fusable<double>(int);
template bool rr_fusable<float>(int);
template int sweep_partials<double>(const Geom&, bool);
template int sweep_partials<float>(const Geom&, bool);
template cudaError_t launch_norm<double>(const Geom&, const Coef<double>&, const double*, const double*, double*,
                                         int*, cudaStream_t);
template cudaError_t launch_norm<float>(const Geom&, const Coef<float>&, const float*, const float*, double*, int*,
                                        cudaStream_t);
template int norm_partials<double>(const Geom&);
template int norm_partials<float>(const Geom&);
template cudaError_t launch_resid_restrict<double>(const Geom&, const Geom&, const Coef<double>&, const double*,
                                                   const double*, double*, cudaStream_t);
template cudaError_t launch_resid_restrict<float>(const Geom&, const Geom&, const Coef<float>&, const float*,
                                                  const float*, float*, cudaStream_t);
template cudaError_t launch_prolong<double>(const Geom&, const Geom&, const double*, const double*, double*,
                                            cudaStream_t);
template cudaError_t launch_prolong<float>(const Geom&, const Geom&, const float*, const float*, float*, cudaStream_t);

}  // namespace pm2
}  // namespace mg
