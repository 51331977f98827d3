// kernels_pm.cu — 2.5D plane-marching level operators for 3D levels (sm_100a).
//
// Work decomposition: a level's interior is a set of (x,y)-tiles of TX x TY
// nodes, each a column of planes along z cut into z-chunks; an item is one
// (tile, chunk).  Consecutive items are neighbouring tiles of the same chunk, so
// CTAs resident together march the same planes and their ring re-reads hit L2;
// the chunk length is chosen so the last wave of resident CTAs is nearly full.
// Each CTA marches its item plane by plane; u and f planes (tile + ring) are
// staged in shared memory by TMA (cp.async.bulk.tensor.3d) into an NS-deep
// slot ring signalled by mbarriers, so every HBM byte is read once per sweep.
//
// Thread t owns the x-pair (ox, ox+1) = (x0 + 2*(t%32), y0 + t/32); a warp is
// one tile row, so every colour decision is warp-uniform.  The pair's values
// of planes p-1, p, p+1 live in registers (z-neighbours never touch smem).
// Arithmetic is the canonical per-point order of mg_common.cuh (no FMA):
// results are bitwise identical to the op-by-op kernels and to the oracle.
//
//  k_sweep3d<RB>     RB: one red-black Gauss-Seidel sweep in ONE pass
//                    (listing P:299-305), ping-pong u_old -> u_new: red
//                    ("post-red", PR) values of plane p on the tile + 1-node
//                    ring, then the black nodes of plane p-1 from PR.  No CTA
//                    reads what another CTA writes: race free.  Jacobi: one
//                    omega-Jacobi sweep.  Both 3 words/node of HBM.
//  k_resid_restrict3d  r = f - A u (Alg. 1 line 4) per fine plane into smem,
//                    full weighting as x/y sums per plane and the z
//                    sum in registers: read u, f; write f_H = 2 + 1/8 words.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels_pm.h"
#include "tma.cuh"

namespace mg {
namespace pm {

#ifndef MG_PM_TY
#define MG_PM_TY 16
#endif
constexpr int TX = 64, TY = MG_PM_TY;  // output tile (fine nodes) per CTA and plane
constexpr int NT = (TX / 2) * TY;      // one thread per x-pair, one warp per tile row
constexpr int RCOL = TY / 2;           // red ring nodes per ring column and plane
constexpr int PX = TX + 2, PY = TY + 2;  // PR / r planes: tile + 1-node ring

__host__ __device__ constexpr int rup(int a, int b) { return (a + b - 1) / b * b; }

// Measured on B200 (sm_100a, driver 580): a tiled TMA load whose x start is not
// a multiple of 16 BYTES raises "illegal instruction", so boxes start HX =
// 16/sizeof(T) nodes left of the tile (2 in FP64, 4 in FP32).
template <typename T>
struct Geo {
  static constexpr int HX = 16 / (int)sizeof(T);
  static constexpr int BX = TX + 2 * HX;  // box width (u and f)
  static constexpr int BYU = TY + 4;      // u box rows: ring 2
  static constexpr int BYF = TY + 2;      // f box rows: ring 1
  static constexpr int UB = rup(BX * BYU * (int)sizeof(T), 128);
  static constexpr int FB = rup(BX * BYF * (int)sizeof(T), 128);
  static constexpr int PB = rup(PX * PY * (int)sizeof(T), 128);
  static constexpr int NS = 4;  // step slots (power of two): 2 steps in flight
  // resident CTAs per SM (registers / shared memory)
  static constexpr int MINB = TY == 8 ? (sizeof(T) == 8 ? 3 : 6) : (sizeof(T) == 8 ? 2 : 3);
  // layout: [NS u boxes][NS f boxes][NS mbarriers][3 PR / r planes][(CORR) 3 coarse boxes]
  static constexpr int BAR_OFF = NS * (UB + FB);
  static constexpr int PR_OFF = BAR_OFF + 128;
  static constexpr int SMEM = PR_OFF + 3 * PB;
  // coarse boxes of the fused prolongation (CORR): x from X0 - 16/sizeof(T), y from Y0 - 1
  static constexpr int CHX = 16 / (int)sizeof(T);
  static constexpr int CBX = rup(TX / 2 + 2 + CHX, CHX);  // 36 (FP64) / 40 (FP32)
  static constexpr int CBY = TY / 2 + 3;
  static constexpr int CB = rup(CBX * CBY * (int)sizeof(T), 128);
  static constexpr int COFF = PR_OFF + 2 * PB;  // CORR keeps 2 PR planes (two barriers per plane)
  static constexpr int SMEM_CORR = COFF + 3 * CB;
};

template <typename T>
struct V2;
template <>
struct V2<double> {
  using t = double2;
};
template <>
struct V2<float> {
  using t = float2;
};

template <typename T>
struct Pair {
  T x, y;
};

template <typename T>
__device__ __forceinline__ Pair<T> ld_pair(const T* p) {
  typename V2<T>::t v = *reinterpret_cast<const typename V2<T>::t*>(p);
  return Pair<T>{v.x, v.y};
}

template <typename T>
__device__ __forceinline__ void store_pair(T* dst, int x, bool ok0, bool ok1, T v0, T v1) {
  if (ok0 && ok1) {
    typename V2<T>::t v;
    v.x = v0;
    v.y = v1;
    *reinterpret_cast<typename V2<T>::t*>(dst + x) = v;
  } else {
    if (ok0) dst[x] = v0;
    if (ok1) dst[x + 1] = v1;
  }
}

// A u at a node in the canonical order: D*u - [cx*(l+r) + cy*(d+u) + cz*(m+p)]
template <typename T>
__device__ __forceinline__ T apply_A(const Coef<T>& c, T ctr, T l, T r, T d, T u, T m, T p) {
  T s = mul(c.cx, add(l, r));
  s = add(s, mul(c.cy, add(d, u)));
  s = add(s, mul(c.cz, add(m, p)));
  return sub(mul(c.D, ctr), s);
}
// u + wd*(f - A u)
template <typename T>
__device__ __forceinline__ T relax(const Coef<T>& c, T ctr, T l, T r, T d, T u, T m, T p, T f) {
  return add(ctr, mul(c.wd, sub(f, apply_A(c, ctr, l, r, d, u, m, p))));
}

// ---------------------------------------------------------------------------
// Slot ring shared by the kernels.  Loads are issued as numbered STEPS n = 0, 1,
// ... per CTA; step n goes to slot n % NS (completing phase (n/NS)&1) and
// carries u of plane q+1 and f of plane q, where q = first plane + n.  While
// plane q is processed only steps q-1 (u(q), f(q-1)) and q (u(q+1), f(q)) are
// read, so NS-2 steps stream in behind them.
template <typename T>
struct Ring {
  unsigned char* sm;
  uint64_t* full;
  __device__ T* U(uint32_t n) const { return reinterpret_cast<T*>(sm + (n % Geo<T>::NS) * Geo<T>::UB); }
  __device__ T* F(uint32_t n) const {
    return reinterpret_cast<T*>(sm + Geo<T>::NS * Geo<T>::UB + (n % Geo<T>::NS) * Geo<T>::FB);
  }
  __device__ void wait(uint32_t n) const { mbar_wait(&full[n % Geo<T>::NS], (n / Geo<T>::NS) & 1u); }
  // step n: u plane qu (unless !load_u), f plane qf
  __device__ void issue(uint32_t n, const CUtensorMap* tu, const CUtensorMap* tf, int x, int y, int qu, int qf,
                        bool load_u) const {
    uint64_t* bar = &full[n % Geo<T>::NS];
    const uint32_t ub = (uint32_t)(Geo<T>::BX * Geo<T>::BYU * sizeof(T));
    const uint32_t fb = (uint32_t)(Geo<T>::BX * Geo<T>::BYF * sizeof(T));
    mbar_expect_tx(bar, (load_u ? ub : 0u) + fb);
    if (load_u) tma_load_3d(U(n), tu, x - Geo<T>::HX, y - 2, qu, bar);
    tma_load_3d(F(n), tf, x - Geo<T>::HX, y - 1, qf, bar);
  }
};

template <typename T>
__device__ __forceinline__ Ring<T> ring_setup(unsigned char* sm, const CUtensorMap* tu, const CUtensorMap* tf) {
  Ring<T> R;
  R.sm = sm;
  R.full = reinterpret_cast<uint64_t*>(sm + Geo<T>::BAR_OFF);
  if (threadIdx.x == 0) {
    prefetch_tmap(tu);
    prefetch_tmap(tf);
    for (int s = 0; s < Geo<T>::NS; s++) mbar_init(&R.full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  return R;
}

// Work item k: tile k % ntiles, planes [p_lo + zc*(k / ntiles), ... + zc) — consecutive
// items are neighbouring tiles of the same z-chunk, so CTAs resident together
// march the same planes and re-read each other's rings from L2.
__device__ __forceinline__ void item_of(int k, int ntiles, int zc, int p_lo, int p_hi, int& tile, int& pa,
                                        int& pb) {
  tile = k % ntiles;
  pa = p_lo + (k / ntiles) * zc;
  pb = min(pa + zc, p_hi);
}

// ---------------------------------------------------------------------------
template <typename T, bool ZERO>
struct Sweep {
  const Coef<T>& c;
  const Ring<T>& R;
  __device__ T u(const T* base, int off) const { return ZERO ? (T)0 : base[off]; }
  __device__ Pair<T> upair(const T* base, int off) const { return ZERO ? Pair<T>{0, 0} : ld_pair(base + off); }
};

// red node (ox + KR) of plane p; returns its post-red value and stores it in PR
template <typename T, bool ZERO, int KR>
__device__ __forceinline__ T red_node(const Sweep<T, ZERO>& S, const T* U0, const T* F0, T* PR, int bo, int fo,
                                      int po, const Pair<T>& um, const Pair<T>& u0, const Pair<T>& up, bool ok) {
  constexpr int BX = Geo<T>::BX;
  const T ctr = KR ? u0.y : u0.x;
  const T l = KR ? u0.x : S.u(U0, bo - 1);
  const T r = KR ? S.u(U0, bo + 2) : u0.y;
  const T v = relax(S.c, ctr, l, r, S.u(U0, bo + KR - BX), S.u(U0, bo + KR + BX), KR ? um.y : um.x,
                    KR ? up.y : up.x, F0[fo + KR]);
  const T pr = ok ? v : ctr;
  PR[po + KR] = pr;
  return pr;
}

// black node (ox + KB) of plane bp from the post-red values
template <typename T, int KB>
__device__ __forceinline__ void black_node(const Coef<T>& c, const T* P, const T* Fb, int fo, int po, T ctr,
                                           T pr_own, T pr_below, T pr_above, bool in0, bool in1, T* orow, int ox) {
  const T l = KB ? pr_own : P[po - 1];
  const T r = KB ? P[po + 2] : pr_own;
  const T v = relax(c, ctr, l, r, P[po + KB - PX], P[po + KB + PX], pr_below, pr_above, Fb[fo + KB]);
  const T o = (KB ? in1 : in0) ? v : ctr;
  store_pair(orow, ox, in0, in1, KB ? pr_own : o, KB ? o : pr_own);
}

// MODE 0: Jacobi sweep; 1: red-black GS sweep; 2: residual-norm partials (one
// double per CTA in `partial`, fixed reduction tree: deterministic).
// NRM (modes 0, 1): also accumulate ||f - A u_in||^2 partials of the sweep's INPUT
// (the norm after the previous cycle comes for free with the next cycle's first
// sweep: u and f are read anyway).
// CORR (modes 0, 1): the sweep's input is u + P e (Alg. 1 line 6), the
// coarse-grid correction applied to every u box in shared memory as it arrives, so
// the corrected iterate never makes an HBM round trip (prolongation fused into the
// first post-smoothing sweep).  Same separable order as k_prolong3d.
constexpr int NRING_CORR = 4 * (TX + 4) + 4 * TY;  // box nodes outside the tile that are read

template <typename T, int MODE, bool ZERO, bool NRM = false, bool CORR = false>
__global__ void __launch_bounds__(NT, Geo<T>::MINB)
    k_sweep3d(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_f, Geom g,
              Coef<T> c, T* __restrict__ unew, int tiles_x, int ntiles, int zc, int nitems,
              double* __restrict__ partial, const __grid_constant__ CUtensorMap tm_e, Geom gc) {
  constexpr bool RB = MODE == 1;
  extern __shared__ __align__(128) unsigned char sm[];
  using G = Geo<T>;
  constexpr int BX = G::BX, HX = G::HX;
  const Ring<T> R = ring_setup<T>(sm, &tm_u, &tm_f);
  // One barrier per plane (3 PR planes, refill one plane later) except with CORR, whose
  // in-smem correction pass needs the shared-memory budget of the third PR plane.
  constexpr bool ONESYNC = !CORR;
  T* spr = reinterpret_cast<T*>(sm + G::PR_OFF);
  auto PRb = [&](int q) {
    return spr + (size_t)(ONESYNC ? ((q % 3) + 3) % 3 : (q & 1)) * (G::PB / sizeof(T));
  };
  const Sweep<T, ZERO> S{c, R};

  const int tid = threadIdx.x, lane = tid & 31, ry = tid >> 5;
  const int pg0 = g.p_glob0;
  const int bo = (ry + 2) * BX + 2 * lane + HX;  // u-box offset of (ox, oy)
  const int fo = (ry + 1) * BX + 2 * lane + HX;  // f-box offset of (ox, oy)
  const int po = (ry + 1) * PX + 2 * lane + 1;    // PR offset of (ox, oy)
  uint32_t seq = 0;
  double nsum = 0.0;  // MODE 2 / NRM: this thread's sum of r^2
  // r^2 of the pair at plane p from the registers u(p-1), u(p), u(p+1) and smem u(p), f(p)
  auto acc_norm = [&](const T* U0, const T* F0, const Pair<T>& um, const Pair<T>& u0, const Pair<T>& up, bool ok0,
                      bool ok1) {
    const Pair<T> fp = ld_pair(F0 + fo);
    const double r0 =
        (double)sub(fp.x, apply_A(c, u0.x, S.u(U0, bo - 1), u0.y, S.u(U0, bo - BX), S.u(U0, bo + BX), um.x, up.x));
    const double r1 = (double)sub(
        fp.y, apply_A(c, u0.y, u0.x, S.u(U0, bo + 2), S.u(U0, bo + 1 - BX), S.u(U0, bo + 1 + BX), um.y, up.y));
    if (ok0) nsum = __dadd_rn(nsum, __dmul_rn(r0, r0));
    if (ok1) nsum = __dadd_rn(nsum, __dmul_rn(r1, r1));
  };
  for (int k = blockIdx.x; k < nitems; k += gridDim.x) {
    int tile, pa, pb;
    item_of(k, ntiles, zc, g.p_lo, g.p_hi, tile, pa, pb);
    const int x0 = (tile % tiles_x) * TX, y0 = (tile / tiles_x) * TY;
    const int ox = x0 + 2 * lane, oy = y0 + ry;
    const bool rin = oy >= 1 && oy <= g.ny - 1;
    const bool in0 = rin && ox >= 1 && ox <= g.nx - 1;
    const bool in1 = rin && ox + 1 <= g.nx - 1;
    T* orow = unew + (long long)oy * g.pitch;
    // step for plane q carries u(q+1), f(q); steps q = qlo .. qlast
    const int qlo = RB ? pa - 3 : pa - 2, qlast = RB ? pb : pb - 1;
    const uint32_t nlo = seq;
    auto N = [&](int q) { return nlo + (uint32_t)(q - qlo); };
    // CORR: coarse plane K lives in coarse slot K % 3; step q (fine u plane z = q+1) also
    // loads coarse plane (z+1)/2 when z is odd (first needed there), the first step also
    // z/2 (TMA, zero-filled outside the coarse array)
    const int X0c = x0 / 2, Y0c = y0 / 2;
    auto Cs = [&](int K) -> T* {
      return reinterpret_cast<T*>(sm + G::COFF + (size_t)(((K % 3) + 3) % 3) * G::CB);
    };
    auto issue_step = [&](int q) {  // thread 0
      if (CORR) {
        uint64_t* bar = &R.full[N(q) % G::NS];
        const int zg = q + 1 + pg0;
        auto ld = [&](int K) {
          mbar_add_tx(bar, (uint32_t)(G::CBX * G::CBY * sizeof(T)));
          tma_load_3d(Cs(K), &tm_e, X0c - G::CHX, Y0c - 1, K - gc.p_glob0, bar);
        };
        if (q == qlo) ld(zg >> 1);
        if (zg & 1) ld((zg + 1) >> 1);
      }
      R.issue(N(q), &tm_u, &tm_f, x0, y0, q + 1, q, !ZERO);
    };
    if (tid == 0)
      for (int q = qlo; q < qlo + G::NS && q <= qlast; q++) issue_step(q);
    // ---- CORR: u += P e on the u box of fine local plane zl (in smem, right after its arrival)
    const T half = (T)0.5;
    int cZ = -1000000;
    Pair<T> cA{0, 0}, cB{0, 0};
    bool cHaveB = false;
    auto e_at = [&](int X, int Y, int Zg) -> T {
      return Cs(Zg)[(Y - Y0c + 1) * G::CBX + (X - X0c + G::CHX)];
    };
    auto Vpair = [&](int Zg) -> Pair<T> {  // pair (2X, 2X+1) of row oy after the x- and y-interpolation
      const int X = ox >> 1, Y = oy >> 1;
      const T a0 = e_at(X, Y, Zg), a1 = e_at(X + 1, Y, Zg);
      Pair<T> v{a0, mul(half, add(a0, a1))};
      if (oy & 1) {
        const T b0 = e_at(X, Y + 1, Zg), b1 = e_at(X + 1, Y + 1, Zg);
        v = Pair<T>{mul(half, add(v.x, b0)), mul(half, add(v.y, mul(half, add(b0, b1))))};
      }
      return v;
    };
    auto interp = [&](int x, int y, int zg) -> T {  // single node, reading 13 order
      const int X = x >> 1, dx = x & 1, Y = y >> 1, dy = y & 1, Z = zg >> 1, dz = zg & 1;
      T vy[2];
      for (int zz = 0; zz <= dz; zz++) {
        T vx[2];
        for (int yy = 0; yy <= dy; yy++)
          vx[yy] = dx ? mul(half, add(e_at(X, Y + yy, Z + zz), e_at(X + 1, Y + yy, Z + zz))) : e_at(X, Y + yy, Z + zz);
        vy[zz] = dy ? mul(half, add(vx[0], vx[1])) : vx[0];
      }
      return dz ? mul(half, add(vy[0], vy[1])) : vy[0];
    };
    auto correct = [&](T* Ub, int zl) {
      const int zg = zl + pg0;
      if (zg < 1 || zg > g.nz - 1) return;  // boundary / outside planes: no correction
      if (in0 || in1) {
        if ((zg >> 1) != cZ) {
          cA = (cHaveB && (zg >> 1) == cZ + 1) ? cB : Vpair(zg >> 1);
          cZ = zg >> 1;
          cHaveB = false;
        }
        Pair<T> v = cA;
        if (zg & 1) {
          if (!cHaveB) {
            cB = Vpair(cZ + 1);
            cHaveB = true;
          }
          v = Pair<T>{mul(half, add(cA.x, cB.x)), mul(half, add(cA.y, cB.y))};
        }
        T* up_ = Ub + bo;
        if (in0) up_[0] = add(up_[0], v.x);
        if (in1) up_[1] = add(up_[1], v.y);
      }
      if (tid < NRING_CORR) {  // box nodes around the tile that the stencils read
        int x, y;
        if (tid < 4 * (TX + 4)) {
          const int rr = tid / (TX + 4);
          y = rr < 2 ? y0 - 2 + rr : y0 + TY + rr - 2;
          x = x0 - 2 + tid % (TX + 4);
        } else {
          const int t2 = tid - 4 * (TX + 4), cc = t2 / TY;
          x = cc < 2 ? x0 - 2 + cc : x0 + TX + cc - 2;
          y = y0 + t2 % TY;
        }
        if (x >= 1 && x <= g.nx - 1 && y >= 1 && y <= g.ny - 1) {
          T* q = Ub + (y - y0 + 2) * BX + (x - x0 + HX);
          *q = add(*q, interp(x, y, zg));
        }
      }
    };
    R.wait(N(qlo));
    R.wait(N(qlo + 1));
    if (CORR) {
      correct(R.U(N(qlo)), qlo + 1);
      correct(R.U(N(qlo + 1)), qlo + 2);
      __syncthreads();
    }
    Pair<T> um = S.upair(R.U(N(qlo)), bo), u0 = S.upair(R.U(N(qlo + 1)), bo), up;
    T rzm = (T)0;  // RB ring thread: u(p-1) at its plane-p ring node
    if (RB && (ry < 2 || (ry == 2 && lane < 2 * RCOL))) {
      const int pgl = pa - 1 + pg0;
      int x, y;
      if (ry < 2) {
        y = ry == 0 ? y0 - 1 : y0 + TY;
        x = x0 + 2 * lane + ((y + pgl) & 1);
      } else {
        x = lane < RCOL ? x0 - 1 : x0 + TX;
        y = y0 + 2 * (lane % RCOL) + ((x + y0 + pgl) & 1);
      }
      rzm = S.u(R.U(N(qlo)), (y - y0 + 2) * BX + (x - x0 + HX));
    }
    __syncthreads();  // step qlo lives on in registers only: refill its slot
    if (tid == 0 && qlo + G::NS <= qlast) {
      fence_proxy_async();
      issue_step(qlo + G::NS);
    }
    if (RB) {
      // ring threads: warp 0 top row (y0-1), warp 1 bottom row (y0+TY), warp 2 lanes [0,RCOL) left column
      // (x0-1), lanes [RCOL,2 RCOL) right column (x0+TX); each computes the red ring node of its slot
      const bool ring = ry < 2 || (ry == 2 && lane < 2 * RCOL);
      auto ring_pos = [&](int pgl, int& x, int& y) {
        if (ry < 2) {
          y = ry == 0 ? y0 - 1 : y0 + TY;
          x = x0 + 2 * lane + ((y + pgl) & 1);  // x0 even
        } else if (lane < RCOL) {
          x = x0 - 1;
          y = y0 + 2 * lane + ((x + y0 + pgl) & 1);
        } else {
          x = x0 + TX;
          y = y0 + 2 * (lane - RCOL) + ((x + y0 + pgl) & 1);
        }
      };
      T pr1 = (T)0, pr2 = (T)0;  // own red value of planes p-1, p-2
      for (int p = pa - 1; p <= pb; p++) {
        R.wait(N(p));
        if (CORR) {
          correct(R.U(N(p)), p + 1);
          __syncthreads();
        }
        const T* U0 = R.U(N(p - 1));  // u(p)
        const T* Up = R.U(N(p));      // u(p+1)
        const T* F0 = R.F(N(p));      // f(p)
        T* PR = PRb(p);
        up = S.upair(Up, bo);
        const int pgl = p + pg0;
        const bool pl_in = pgl >= 1 && pgl <= g.nz - 1;
        const int kr = (oy + pgl) & 1;  // warp uniform
        if (NRM && p >= pa && p < pb) acc_norm(U0, F0, um, u0, up, in0, in1);
        const T pr0 = kr ? red_node<T, ZERO, 1>(S, U0, F0, PR, bo, fo, po, um, u0, up, pl_in && in1)
                         : red_node<T, ZERO, 0>(S, U0, F0, PR, bo, fo, po, um, u0, up, pl_in && in0);
        if (ring) {  // red ring node of plane p
          int x, y;
          ring_pos(pgl, x, y);
          const int rb = (y - y0 + 2) * BX + (x - x0 + HX);
          const T ctr = S.u(U0, rb);
          const T v = relax(c, ctr, S.u(U0, rb - 1), S.u(U0, rb + 1), S.u(U0, rb - BX), S.u(U0, rb + BX), rzm,
                            S.u(Up, rb), F0[(y - y0 + 1) * BX + (x - x0 + HX)]);
          const bool ok = pl_in && x >= 1 && x <= g.nx - 1 && y >= 1 && y <= g.ny - 1;
          PR[(y - y0 + 1) * PX + (x - x0 + 1)] = ok ? v : ctr;
          ring_pos(pgl + 1, x, y);  // next plane's node: its z-neighbour below is u(p)
          rzm = S.u(U0, (y - y0 + 2) * BX + (x - x0 + HX));
        }
        __syncthreads();
        // ONESYNC: every thread has finished plane p-2's black update: step p-2 is free
        if (ONESYNC && tid == 0 && p >= pa && p - 2 + G::NS <= qlast) {
          fence_proxy_async();
          issue_step(p - 2 + G::NS);
        }
        const int bp = p - 1;  // black nodes of plane p-1: they sit where plane p's red nodes are
        if (bp >= pa) {
          const T* P = PRb(bp);
          const T* Fb = R.F(N(bp));
          T* orow_b = orow + (long long)bp * g.pstride;
          if (kr)
            black_node<T, 1>(c, P, Fb, fo, po, um.y, pr1, pr2, pr0, in0, in1, orow_b, ox);
          else
            black_node<T, 0>(c, P, Fb, fo, po, um.x, pr1, pr2, pr0, in0, in1, orow_b, ox);
        }
        if (!ONESYNC) {
          __syncthreads();
          if (tid == 0 && p - 1 + G::NS <= qlast) {  // step p-1 (u(p), f(p-1)) is consumed
            fence_proxy_async();
            issue_step(p - 1 + G::NS);
          }
        }
        um = u0;
        u0 = up;
        pr2 = pr1;
        pr1 = pr0;
      }
    } else {
      for (int p = pa; p < pb; p++) {
        R.wait(N(p));
        if (CORR) {
          correct(R.U(N(p)), p + 1);
          __syncthreads();
        }
        const T* U0 = R.U(N(p - 1));
        up = S.upair(R.U(N(p)), bo);
        const Pair<T> fp = ld_pair(R.F(N(p)) + fo);
        if (MODE == 2 || NRM) acc_norm(U0, R.F(N(p)), um, u0, up, in0, in1);  // r = f - A u, FP64 squares
        if (MODE != 2) {
          const T v0 =
              relax(c, u0.x, S.u(U0, bo - 1), u0.y, S.u(U0, bo - BX), S.u(U0, bo + BX), um.x, up.x, fp.x);
          const T v1 =
              relax(c, u0.y, u0.x, S.u(U0, bo + 2), S.u(U0, bo + 1 - BX), S.u(U0, bo + 1 + BX), um.y, up.y, fp.y);
          store_pair(orow + (long long)p * g.pstride, ox, in0, in1, in0 ? v0 : u0.x, in1 ? v1 : u0.y);
        }
        __syncthreads();
        if (tid == 0 && p - 1 + G::NS <= qlast) {
          fence_proxy_async();
          issue_step(p - 1 + G::NS);
        }
        um = u0;
        u0 = up;
      }
    }
    seq = N(qlast) + 1;
    __syncthreads();
  }
  if (MODE == 2 || NRM) {  // fixed-order block reduction -> one partial per CTA
    double* red = reinterpret_cast<double*>(sm);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nsum = __dadd_rn(nsum, __shfl_down_sync(0xffffffffu, nsum, o));
    if (lane == 0) red[ry] = nsum;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w2 = 0; w2 < NT / 32; w2++) t = __dadd_rn(t, red[w2]);
      partial[blockIdx.x] = t;
    }
  }
}

// ---------------------------------------------------------------------------
// Fused residual + full-weighting restriction.  Work items are (coarse tile,
// coarse z-chunk); the fine tile is 2x the coarse tile (x0 = 2 X0).  Per fine
// plane q: r for every pair of the tile (u column in registers) and the 73
// low-side ring nodes (row y0-1, column x0-1) into smem; then the 128 coarse
// nodes form their x- then y-sums of plane q and keep the last three in
// registers: when q = 2P+1 the z-sum gives f_H(P) (reading 13 order).
template <typename T>
__global__ void __launch_bounds__(NT, Geo<T>::MINB)
    k_resid_restrict3d(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_f,
                       Geom gf, Geom gc, Coef<T> c, T* __restrict__ fc, int tiles_x, int ntiles, int zcc,
                       int nitems) {
  extern __shared__ __align__(128) unsigned char sm[];
  using G = Geo<T>;
  constexpr int BX = G::BX, HX = G::HX;
  const Ring<T> R = ring_setup<T>(sm, &tm_u, &tm_f);
  T* Rr = reinterpret_cast<T*>(sm + G::PR_OFF);

  const int tid = threadIdx.x, lane = tid & 31, ry = tid >> 5;
  const int pgf0 = gf.p_glob0;
  const int bo = (ry + 2) * BX + 2 * lane + HX;
  const int fo = (ry + 1) * BX + 2 * lane + HX;
  const int po = (ry + 1) * PX + 2 * lane + 1;
  const T two = (T)2;
  const T scale = (T)(1.0 / 64.0);
  uint32_t seq = 0;
  for (int k = blockIdx.x; k < nitems; k += gridDim.x) {
    int tile, Pa, Pb;
    item_of(k, ntiles, zcc, gc.p_lo, gc.p_hi, tile, Pa, Pb);
    const int X0 = (tile % tiles_x) * (TX / 2), Y0 = (tile / tiles_x) * (TY / 2);
    const int x0 = 2 * X0, y0 = 2 * Y0;
    const int ox = x0 + 2 * lane, oy = y0 + ry;
    const bool rin = oy >= 1 && oy <= gf.ny - 1;
    const bool in0 = rin && ox >= 1 && ox <= gf.nx - 1;
    const bool in1 = rin && ox + 1 <= gf.nx - 1;
    // low-side ring: row y0-1 for x in [x0-1, x0+TX-1] (65 nodes), column x0-1 for y in [y0, y0+TY-1] (TY)
    const bool has_ring = tid < TX + 1 + TY;
    const int rx = tid < TX + 1 ? x0 - 1 + tid : x0 - 1;
    const int ryy = tid < TX + 1 ? y0 - 1 : y0 + tid - (TX + 1);
    const bool ring_in = rx >= 1 && rx <= gf.nx - 1 && ryy >= 1 && ryy <= gf.ny - 1;
    const int rb = (ryy - y0 + 2) * BX + (rx - x0 + HX);
    const int rf = (ryy - y0 + 1) * BX + (rx - x0 + HX);
    const int rpo = (ryy - y0 + 1) * PX + (rx - x0 + 1);
    // coarse node of threads 0..127: warp = coarse row, lane = coarse column
    const int I = X0 + lane, J = Y0 + ry;
    const bool cnode = ry < TY / 2 && I >= 1 && I <= gc.nx - 1 && J >= 1 && J <= gc.ny - 1;
    const int co = (2 * ry + 1) * PX + 2 * lane + 1;  // r offset of fine (2I, 2J)
    T* crow = fc + (long long)J * gc.pitch + I;

    const int qf0 = 2 * (Pa + gc.p_glob0) - pgf0;      // fine centre of the first coarse plane
    const int qf1 = 2 * (Pb - 1 + gc.p_glob0) - pgf0;  // ... of the last
    const int rlo = qf0 - 1, rhi = qf1 + 1;              // r planes needed
    const int qlo = rlo - 2, qlast = rhi;                // steps: u(q+1), f(q)
    const uint32_t nlo = seq;
    auto N = [&](int q) { return nlo + (uint32_t)(q - qlo); };
    if (tid == 0)
      for (int q = qlo; q < qlo + G::NS && q <= qlast; q++) R.issue(N(q), &tm_u, &tm_f, x0, y0, q + 1, q, true);
    R.wait(N(qlo));
    R.wait(N(qlo + 1));
    Pair<T> um = ld_pair(R.U(N(qlo)) + bo), u0 = ld_pair(R.U(N(qlo + 1)) + bo), up;
    T rzm = has_ring ? R.U(N(qlo))[rb] : (T)0;
    __syncthreads();  // step qlo lives on in registers only: refill its slot
    if (tid == 0 && qlo + G::NS <= qlast) {
      fence_proxy_async();
      R.issue(N(qlo + G::NS), &tm_u, &tm_f, x0, y0, qlo + G::NS + 1, qlo + G::NS, true);
    }
    T ty1 = (T)0, ty2 = (T)0;
    for (int q = rlo; q <= rhi; q++) {
      R.wait(N(q));
      const T* U0 = R.U(N(q - 1));
      const T* Up = R.U(N(q));
      const T* F0 = R.F(N(q));
      up = ld_pair(Up + bo);
      const int pgl = q + pgf0;
      const bool pl_in = pgl >= 1 && pgl <= gf.nz - 1;
      {
        const Pair<T> fp = ld_pair(F0 + fo);
        const T r0 = sub(fp.x, apply_A(c, u0.x, U0[bo - 1], u0.y, U0[bo - BX], U0[bo + BX], um.x, up.x));
        const T r1 = sub(fp.y, apply_A(c, u0.y, u0.x, U0[bo + 2], U0[bo + 1 - BX], U0[bo + 1 + BX], um.y, up.y));
        Rr[po] = pl_in && in0 ? r0 : (T)0;
        Rr[po + 1] = pl_in && in1 ? r1 : (T)0;
      }
      if (has_ring) {
        const T uc = U0[rb];
        const T r = sub(F0[rf], apply_A(c, uc, U0[rb - 1], U0[rb + 1], U0[rb - BX], U0[rb + BX], rzm, Up[rb]));
        Rr[rpo] = pl_in && ring_in ? r : (T)0;
        rzm = uc;
      }
      __syncthreads();
      if (ry < TY / 2) {
        T tx[3];
#pragma unroll
        for (int dy = -1; dy <= 1; dy++) {
          const T* row = Rr + co + dy * PX;
          tx[dy + 1] = add(add(row[-1], row[1]), mul(two, row[0]));
        }
        const T ty0 = add(add(tx[0], tx[2]), mul(two, tx[1]));
        if (cnode && (pgl & 1) == 1 && q >= qf0 + 1) {  // fine plane 2P+1 completes coarse plane P
          const int Pc = ((pgl - 1) >> 1) - gc.p_glob0;
          crow[(long long)Pc * gc.pstride] = mul(add(add(ty2, ty0), mul(two, ty1)), scale);
        }
        ty2 = ty1;
        ty1 = ty0;
      }
      __syncthreads();
      if (tid == 0 && q - 1 + G::NS <= qlast) {
        fence_proxy_async();
        R.issue(N(q - 1 + G::NS), &tm_u, &tm_f, x0, y0, q + G::NS, q - 1 + G::NS, true);
      }
      um = u0;
      u0 = up;
    }
    seq = N(qlast) + 1;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// cuTensorMapEncodeTiled through the runtime's driver entry point, so that the
// library does not link libcuda (it must load on GPU-less hosts for the ABI tests).
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static CUresult encode(CUtensorMap* tm, const void* base, const Geom& g, int esz, int box_rows) {
  PFN_cuTensorMapEncodeTiled_v12000 cuTensorMapEncodeTiled = encode_fn();
  if (!cuTensorMapEncodeTiled) return CUDA_ERROR_NOT_FOUND;
  cuuint64_t dims[3] = {(cuuint64_t)(g.nx + 1), (cuuint64_t)g.rows, (cuuint64_t)g.planes};
  cuuint64_t strides[2] = {(cuuint64_t)(g.pitch * esz), (cuuint64_t)(g.pstride * esz)};
  cuuint32_t box[3] = {(cuuint32_t)(TX + 2 * (16 / esz)), (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return cuTensorMapEncodeTiled(tm, esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                                const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

// Plane marching pays off once a level has enough planes per CTA to hide the
// per-plane barrier latency: measured, a 65^3 level is 2x slower marched than
// with the one-thread-per-node kernels, 129^3 is ~1.5x faster.  The plan passes
// mg_config.pm_min_nx (default 128; tests lower it to cover small grids).
static CUresult encode_coarse(CUtensorMap* tm, const void* base, const Geom& g, int esz, int box_x, int box_y) {
  PFN_cuTensorMapEncodeTiled_v12000 cuTensorMapEncodeTiled = encode_fn();
  if (!cuTensorMapEncodeTiled) return CUDA_ERROR_NOT_FOUND;
  cuuint64_t dims[3] = {(cuuint64_t)(g.nx + 1), (cuuint64_t)g.rows, (cuuint64_t)g.planes};
  cuuint64_t strides[2] = {(cuuint64_t)(g.pitch * esz), (cuuint64_t)(g.pstride * esz)};
  cuuint32_t box[3] = {(cuuint32_t)box_x, (cuuint32_t)box_y, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return cuTensorMapEncodeTiled(tm, esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                                const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

bool supported(const Geom& g, int min_nx) {
  return g.three_d && g.nx >= (min_nx < 16 ? 16 : min_nx) && g.ny >= 16 && (g.p_hi - g.p_lo) >= 4;
}

// First use of a kernel: opt in to its dynamic shared memory and return the
// number of CTAs the device keeps resident (cached per kernel).
template <class K>
static int prepare_kernel(K kernel, int smem) {
  static const void* keys[32];
  static int vals[32];
  static int n = 0;
  for (int i = 0; i < n; i++)
    if (keys[i] == (const void*)kernel) return vals[i];
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int sms = 0, occ = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, NT, smem);
  const int r = (occ < 1 ? 1 : occ) * (sms < 1 ? 1 : sms);
  if (n < 32) {
    keys[n] = (const void*)kernel;
    vals[n++] = r;
  }
  return r;
}

// z-chunk size.  Measured on the 513^3 RBGS sweep (tools/scan_zc.py): what
// matters is a nearly full last wave of resident CTAs and enough waves (>= ~8)
// to balance SMs; the halo re-loads of short chunks mostly hit L2.  So: among
// chunk lengths >= 16 planes, minimise (ceil(waves)/waves) * (1 + halo/(2 zc))
// plus a small penalty below 8 waves.
static int choose_zc(long long ntiles, int np, int resident, int halo) {
  int best = np;
  double best_cost = 1e300;
  for (int c = 1; c <= 256 && c <= np; c++) {
    const int zc = (np + c - 1) / c;
    if (zc < 16 && c > 1) break;
    const int chunks = (np + zc - 1) / zc;
    const long long items = ntiles * chunks;
    const double wx = (double)items / resident;
    const double wc = (double)((items + resident - 1) / resident);
    const double cost = (wc / wx) * (1.0 + 0.5 * halo / zc) + (wx < 8.0 ? 0.02 * (8.0 - wx) : 0.0);
    if (cost < best_cost - 1e-12) {
      best_cost = cost;
      best = zc;
    }
  }
  return best;
}

static CUresult encode_coarse(CUtensorMap* tm, const void* base, const Geom& g, int esz, int box_x, int box_y);

template <typename T>
cudaError_t launch_sweep(const Geom& g, const Coef<T>& c, bool rbgs, const T* uin, const T* f, T* uout, bool zero_in,
                         int zc_override, cudaStream_t st, double* partial, int* npartial, const T* ecoarse,
                         const Geom* gcoarse) {
  const Geom gce = gcoarse ? *gcoarse : Geom{};
  CUtensorMap te;
  memset(&te, 0, sizeof te);
  if (ecoarse && encode_coarse(&te, ecoarse, gce, sizeof(T), Geo<T>::CBX, Geo<T>::CBY) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  using G = Geo<T>;
  CUtensorMap tu, tf;
  CUresult e1 = encode(&tu, uin ? uin : f, g, sizeof(T), G::BYU), e2 = encode(&tf, f, g, sizeof(T), G::BYF);
  if (getenv("MG_DEBUG")) fprintf(stderr, "launch_sweep: encode %d %d nx=%d ny=%d rows=%d np=%d\n", (int)e1, (int)e2, g.nx, g.ny, g.rows, g.p_hi - g.p_lo);
  if (e1 != CUDA_SUCCESS || e2 != CUDA_SUCCESS) return cudaErrorInvalidValue;
  const int tiles_x = (g.nx + TX - 1) / TX, tiles_y = (g.ny + TY - 1) / TY;
  const int ntiles = tiles_x * tiles_y;
  const int np = g.p_hi - g.p_lo;
  auto go = [&](auto kernel) {
    const int resident = prepare_kernel(kernel, ecoarse ? G::SMEM_CORR : G::SMEM);
    const int zc = zc_override > 0 ? zc_override : choose_zc(ntiles, np, resident, rbgs ? 4 : 2);
    const int nitems = ntiles * ((np + zc - 1) / zc);
    if (getenv("MG_DEBUG"))
      fprintf(stderr, "launch_sweep: resident=%d zc=%d nitems=%d smem=%d\n", resident, zc, nitems, G::SMEM);
    if (npartial) *npartial = nitems;
    const int smem = ecoarse ? G::SMEM_CORR : G::SMEM;
    const int resident2 = ecoarse ? prepare_kernel(kernel, smem) : resident;
    (void)resident2;
    kernel<<<nitems, NT, smem, st>>>(tu, tf, g, c, uout, tiles_x, ntiles, zc, nitems, partial, te, gce);
  };
  if (ecoarse)
    rbgs ? go(k_sweep3d<T, 1, false, false, true>) : go(k_sweep3d<T, 0, false, false, true>);
  else if (partial && !zero_in)
    rbgs ? go(k_sweep3d<T, 1, false, true>) : go(k_sweep3d<T, 0, false, true>);
  else if (rbgs)
    zero_in ? go(k_sweep3d<T, 1, true>) : go(k_sweep3d<T, 1, false>);
  else
    zero_in ? go(k_sweep3d<T, 0, true>) : go(k_sweep3d<T, 0, false>);
  return cudaGetLastError();
}

// upper bound of the partials launch_sweep(..., partial, ...) writes for a level
template <typename T>
int sweep_partials(const Geom& g, bool rbgs) {
  using G = Geo<T>;
  const int ntiles = ((g.nx + TX - 1) / TX) * ((g.ny + TY - 1) / TY);
  const int np = g.p_hi - g.p_lo;
  const int resident = rbgs ? prepare_kernel(k_sweep3d<T, 1, false, true>, G::SMEM)
                            : prepare_kernel(k_sweep3d<T, 0, false, true>, G::SMEM);
  int best = 0;
  for (int halo : {2, 4}) {
    const int zc = choose_zc(ntiles, np, resident, halo);
    const int n = ntiles * ((np + zc - 1) / zc);
    if (n > best) best = n;
  }
  return best;
}

template <typename T>
int norm_partials(const Geom& g) {
  using G = Geo<T>;
  const int ntiles = ((g.nx + TX - 1) / TX) * ((g.ny + TY - 1) / TY);
  const int np = g.p_hi - g.p_lo;
  const int resident = prepare_kernel(k_sweep3d<T, 2, false>, G::SMEM);
  const int zc = choose_zc(ntiles, np, resident, 2);
  return ntiles * ((np + zc - 1) / zc);
}

template <typename T>
cudaError_t launch_norm(const Geom& g, const Coef<T>& c, const T* u, const T* f, double* partial, int* npartial,
                        cudaStream_t st) {
  using G = Geo<T>;
  CUtensorMap tu, tf;
  if (encode(&tu, u, g, sizeof(T), G::BYU) != CUDA_SUCCESS || encode(&tf, f, g, sizeof(T), G::BYF) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const int tiles_x = (g.nx + TX - 1) / TX, tiles_y = (g.ny + TY - 1) / TY;
  const int ntiles = tiles_x * tiles_y;
  const int np = g.p_hi - g.p_lo;
  auto kernel = k_sweep3d<T, 2, false>;
  const int resident = prepare_kernel(kernel, G::SMEM);
  const int zc = choose_zc(ntiles, np, resident, 2);
  const int nitems = ntiles * ((np + zc - 1) / zc);
  *npartial = nitems;
  CUtensorMap te;
  memset(&te, 0, sizeof te);
  kernel<<<nitems, NT, G::SMEM, st>>>(tu, tf, g, c, nullptr, tiles_x, ntiles, zc, nitems, partial, te, Geom{});
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Bi-/trilinear prolongation + correction u += P e, 3D.
// Pointwise in u, so no staging: thread = fine x-pair (2X, 2X+1) of one row,
// marching z.  The pair's coarse values after the x- and y-interpolation of a
// coarse plane K, V(K), stay in registers for the 3 fine planes that use it;
// fine plane z = 2Z+dz gets dz ? (V(Z)+V(Z+1))/2 : V(Z) (reading 13 order).
template <typename T>
__global__ void __launch_bounds__(NT) k_prolong3d(Geom gf, Geom gc, const T* __restrict__ e, T* __restrict__ u,
                                                 int tiles_x, int ntiles, int zc, int nitems) {
  const int lane = threadIdx.x & 31, ry = threadIdx.x >> 5;
  const T half = (T)0.5;
  for (int k = blockIdx.x; k < nitems; k += gridDim.x) {
    int tile, pa, pb;
    item_of(k, ntiles, zc, gf.p_lo, gf.p_hi, tile, pa, pb);
    const int x0 = (tile % tiles_x) * TX, y0 = (tile / tiles_x) * TY;
    const int ox = x0 + 2 * lane, oy = y0 + ry;
    const bool rin = oy >= 1 && oy <= gf.ny - 1;
    const bool in0 = rin && ox >= 1 && ox <= gf.nx - 1;
    const bool in1 = rin && ox + 1 <= gf.nx - 1;
    if (!(in0 || in1)) continue;
    const int X = ox >> 1, Y = oy >> 1, dy = oy & 1;
    const T* ec = e + (long long)Y * gc.pitch + X;
    auto V = [&](int Zg) -> Pair<T> {  // x- then y-interpolated pair of coarse plane Zg (global)
      const T* p0 = ec + (long long)(Zg - gc.p_glob0) * gc.pstride;
      const T a0 = __ldg(p0), a1 = __ldg(p0 + 1);
      Pair<T> v{a0, mul(half, add(a0, a1))};
      if (dy) {
        const T b0 = __ldg(p0 + gc.pitch), b1 = __ldg(p0 + gc.pitch + 1);
        const Pair<T> w{b0, mul(half, add(b0, b1))};
        v = Pair<T>{mul(half, add(v.x, w.x)), mul(half, add(v.y, w.y))};
      }
      return v;
    };
    T* urow = u + (long long)oy * gf.pitch + ox;
    int Z = (pa + gf.p_glob0) >> 1;
    Pair<T> A = V(Z), B = A;
    bool haveB = false;
    for (int z = pa; z < pb; z++) {
      const int zg = z + gf.p_glob0;
      if ((zg >> 1) != Z) {
        Z++;
        A = haveB ? B : V(Z);
        haveB = false;
      }
      Pair<T> v = A;
      if (zg & 1) {
        if (!haveB) {
          B = V(Z + 1);
          haveB = true;
        }
        v = Pair<T>{mul(half, add(A.x, B.x)), mul(half, add(A.y, B.y))};
      }
      T* up = urow + (long long)z * gf.pstride;
      if (in0 && in1) {
        const Pair<T> uu = ld_pair(up);
        typename V2<T>::t o;
        o.x = add(uu.x, v.x);
        o.y = add(uu.y, v.y);
        *reinterpret_cast<typename V2<T>::t*>(up) = o;
      } else {
        if (in0) up[0] = add(up[0], v.x);
        if (in1) up[1] = add(up[1], v.y);
      }
    }
  }
}

template <typename T>
cudaError_t launch_prolong(const Geom& gf, const Geom& gc, const T* e, T* u, cudaStream_t st) {
  const int tiles_x = (gf.nx + TX - 1) / TX, tiles_y = (gf.ny + TY - 1) / TY;
  const int ntiles = tiles_x * tiles_y;
  const int np = gf.p_hi - gf.p_lo;
  static int resident = 0;
  if (!resident) {
    int sms = 0, occ = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_prolong3d<T>, NT, 0);
    resident = (occ < 1 ? 1 : occ) * (sms < 1 ? 1 : sms);
  }
  const int zc = choose_zc(ntiles, np, resident, 0);
  const int nitems = ntiles * ((np + zc - 1) / zc);
  k_prolong3d<T><<<nitems, NT, 0, st>>>(gf, gc, e, u, tiles_x, ntiles, zc, nitems);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_resid_restrict(const Geom& gf, const Geom& gc, const Coef<T>& c, const T* u, const T* f, T* fc,
                                  int zc_override, cudaStream_t st) {
  using G = Geo<T>;
  CUtensorMap tu, tf;
  if (encode(&tu, u, gf, sizeof(T), G::BYU) != CUDA_SUCCESS || encode(&tf, f, gf, sizeof(T), G::BYF) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const int tiles_x = (gc.nx + TX / 2 - 1) / (TX / 2), tiles_y = (gc.ny + TY / 2 - 1) / (TY / 2);
  const int ntiles = tiles_x * tiles_y;
  const int npc = gc.p_hi - gc.p_lo;
  auto kernel = k_resid_restrict3d<T>;
  const int resident = prepare_kernel(kernel, G::SMEM);
  const int zcc = zc_override > 0 ? zc_override : choose_zc(ntiles, npc, resident, 2);
  const int nitems = ntiles * ((npc + zcc - 1) / zcc);
  kernel<<<nitems, NT, G::SMEM, st>>>(tu, tf, gf, gc, c, fc, tiles_x, ntiles, zcc, nitems);
  return cudaGetLastError();
}

template cudaError_t launch_sweep<double>(const Geom&, const Coef<double>&, bool, const double*, const double*,
                                          double*, bool, int, cudaStream_t, double*, int*, const double*,
                                          const Geom*);
template cudaError_t launch_sweep<float>(const Geom&, const Coef<float>&, bool, const float*, const float*, float*,
                                         bool, int, cudaStream_t, double*, int*, const float*, const Geom*);
template int sweep_partials<double>(const Geom&, bool);
template int sweep_partials<float>(const Geom&, bool);
template int norm_partials<double>(const Geom&);
template int norm_partials<float>(const Geom&);
template cudaError_t launch_norm<double>(const Geom&, const Coef<double>&, const double*, const double*, double*,
                                         int*, cudaStream_t);
template cudaError_t launch_norm<float>(const Geom&, const Coef<float>&, const float*, const float*, double*, int*,
                                        cudaStream_t);
template cudaError_t launch_prolong<double>(const Geom&, const Geom&, const double*, double*, cudaStream_t);
template cudaError_t launch_prolong<float>(const Geom&, const Geom&, const float*, float*, cudaStream_t);
template cudaError_t launch_resid_restrict<double>(const Geom&, const Geom&, const Coef<double>&, const double*,
                                                   const double*, double*, int, cudaStream_t);
template cudaError_t launch_resid_restrict<float>(const Geom&, const Geom&, const Coef<float>&, const float*,
                                                  const float*, float*, int, cudaStream_t);

}  // namespace pm
}  // namespace mg
