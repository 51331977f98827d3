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
// Thread t owns one 16-byte x-vector (W = 2 FP64 / 4 FP32 nodes) of RPT = 2
// consecutive tile rows; a warp is a pair of tile rows, so every colour decision
// is warp-uniform.  Its values of planes p-1, p, p+1 live in registers
// (z-neighbours never touch smem; y-neighbours inside the thread's rows neither).
// Arithmetic is the canonical per-point order of mg_common.cuh (no FMA):
// results are bitwise identical to the op-by-op kernels and to the oracle.
//
//  k_sweep3d_rows    RB: one red-black Gauss-Seidel sweep in ONE pass
//                    (listing P:299-305), ping-pong u_old -> u_new: red
//                    ("post-red", PR) values of plane p on the tile + 1-node
//                    ring, then the black nodes of plane p-1 from PR.  No CTA
//                    reads what another CTA writes: race free.  Jacobi: one
//                    omega-Jacobi sweep.  Both 3 words/node of HBM.
//                    A thread owns RPT rows of its x-vector.  Variants: the
//                    residual norm of the input / of the output's black nodes,
//                    a zero input, the prolongation fused in (CORR).
//  k_resid_restrict3d_rows  r = f - A u (Alg. 1 line 4) per fine plane into
//                    smem, full weighting as x/y sums per plane and
//                    the z sum in registers: read u, f; write f_H = 2 + 1/8 words.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <utility>

#include "kernels_pm.h"
#include "kernels_pm2d.h"
#include "launch_util.h"
#include "tma.cuh"
#include "vec.cuh"

namespace mg {
namespace pm {

#ifndef MG_PM_TY
#define MG_PM_TY 16
#endif
// A thread owns one 16-byte vector of W consecutive x nodes (W = 2 in FP64, 4 in
// FP32: the same bytes per instruction in both precisions); a warp is one tile row
// of TX = 32 W nodes, so every colour decision is warp-uniform.
constexpr int TY = MG_PM_TY;  // tile rows
constexpr int NT = 32 * TY;   // threads per CTA

__host__ __device__ constexpr int rup(int a, int b) { return (a + b - 1) / b * b; }

// Measured on B200 (sm_100a, driver 580): a tiled TMA load whose x start is not
// a multiple of 16 BYTES raises "illegal instruction", so boxes start HX =
// 16/sizeof(T) nodes left of the tile (2 in FP64, 4 in FP32).
template <typename T>
struct Geo {
  static constexpr int W = 16 / (int)sizeof(T);  // nodes per thread
  static constexpr int TX = 32 * W;              // tile width (64 / 128)
  static constexpr int HX = W;
  static constexpr int PY = TY + 2;                // PR / r planes: tile + 1-node ring rows
  static constexpr int BX = TX + 2 * HX;  // box width (u and f)
  static constexpr int BYU = TY + 4;      // u box rows: ring 2
  static constexpr int BYF = TY + 2;      // f box rows: ring 1
  static constexpr int UB = rup(BX * BYU * (int)sizeof(T), 128);
  static constexpr int FB = rup(BX * BYF * (int)sizeof(T), 128);
  // PR / r planes use the box row stride BX and x offset HX, so per-thread vectors are 16-B aligned
  static constexpr int PX = BX;
  static constexpr int PB = rup(PX * PY * (int)sizeof(T), 128);
  static constexpr int NS = 4;     // step slots (power of two)
  static constexpr int MINB = 2;   // resident CTAs per SM (shared memory: ~111 KB each)
  // layout: [NS u boxes][NS f boxes][NS mbarriers][3 PR / r planes][(CORR) 3 coarse boxes]
  static constexpr int BAR_OFF = NS * (UB + FB);
  static constexpr int PR_OFF = BAR_OFF + 128;
  static constexpr int SMEM = PR_OFF + 3 * PB;
  // coarse boxes of the fused prolongation (CORR): x from X0 - CHX, y from Y0 - 1
  static constexpr int CHX = W;
  static constexpr int CBX = rup(TX / 2 + 2 + CHX, CHX);  // 36 (FP64) / 72 (FP32)
  static constexpr int CBY = TY / 2 + 3;
  static constexpr int CB = rup(CBX * CBY * (int)sizeof(T), 128);
  static constexpr int NRED = W / 2;  // red (and black) nodes per thread and plane
  static constexpr int RCOL = TY / 2;  // red ring nodes per ring column and plane
};

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
template <typename T, int NSR = Geo<T>::NS>
struct Ring {
  static constexpr int NS = NSR;
  static constexpr int BAR_OFF = NSR * (Geo<T>::UB + Geo<T>::FB);  // then NSR mbarriers (128 B)
  unsigned char* sm;
  uint64_t* full;
  __device__ T* U(uint32_t n) const { return reinterpret_cast<T*>(sm + (n % NSR) * Geo<T>::UB); }
  __device__ T* F(uint32_t n) const {
    return reinterpret_cast<T*>(sm + NSR * Geo<T>::UB + (n % NSR) * Geo<T>::FB);
  }
  __device__ void wait(uint32_t n) const { mbar_wait(&full[n % NSR], (n / NSR) & 1u); }
  // step n: u plane qu (unless !load_u), f plane qf
  __device__ void issue(uint32_t n, const CUtensorMap* tu, const CUtensorMap* tf, int x, int y, int qu, int qf,
                        bool load_u) const {
    uint64_t* bar = &full[n % NSR];
    const uint32_t ub = (uint32_t)(Geo<T>::BX * Geo<T>::BYU * sizeof(T));
    const uint32_t fb = (uint32_t)(Geo<T>::BX * Geo<T>::BYF * sizeof(T));
    mbar_expect_tx(bar, (load_u ? ub : 0u) + fb);
    if (load_u) tma_load_3d(U(n), tu, x - Geo<T>::HX, y - 2, qu, bar);
    tma_load_3d(F(n), tf, x - Geo<T>::HX, y - 1, qf, bar);
  }
};

template <typename T, int NSR = Geo<T>::NS>
__device__ __forceinline__ Ring<T, NSR> ring_setup(unsigned char* sm, const CUtensorMap* tu, const CUtensorMap* tf) {
  Ring<T, NSR> R;
  R.sm = sm;
  R.full = reinterpret_cast<uint64_t*>(sm + Ring<T, NSR>::BAR_OFF);
  if (threadIdx.x == 0) {
    prefetch_tmap(tu);
    prefetch_tmap(tf);
    for (int s = 0; s < NSR; s++) mbar_init(&R.full[s], 1);
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
// Row-blocked sweep (the default for every variant but CORR): the same tile, boxes, ring,
// arithmetic and red/black schedule as k_sweep3d, but a thread owns RPT consecutive tile
// rows of its x-vector (NTH = 32 TY / RPT threads per CTA).  The y-neighbours of a row that
// lie inside the thread's own rows come from registers: its rows' u(p) for the red stage,
// its rows' post-red values of plane p-1 for the black stage (the black node at (j, row k)
// has its y-neighbours at the red positions of rows k-1 / k+1 with the same index m).  Only
// the outer rows read the row above / below from shared memory.  Per-plane fixed costs
// (ring waits, slot addresses, barrier, loop control) are shared by RPT rows, and the
// register budget per thread (NTH threads, 2 CTAs per SM) doubles.  Bitwise identical
// results (the per-node operations and their order are those of k_sweep3d).
template <int N, class F, int... I>
__device__ __forceinline__ void sfor_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>()), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  sfor_impl<N>(f, std::make_integer_sequence<int, N>());
}

// NM (RB / Jacobi): 0 no norm; 1 ||f - A u_in||^2 partials of the sweep's INPUT (the solve's
// first head); 2 the same, red nodes only (RB: a later head of the solve, whose black nodes'
// input residuals were accumulated by the previous cycle's last level-0 sweep); 3 (RB) the
// residuals of the black nodes of the sweep's OUTPUT: a black node's neighbours are all red
// and final when it is relaxed, so the stencil sum s of its relaxation is the sum the norm
// forms at the output, and r = f - (D v - s) is that residual bitwise (3 more operations)
//
// CORR (the first post-smoothing sweep, the default on 3D levels): the sweep's input is u + P e (Alg. 1
// line 6).  The coarse planes of e arrive by TMA with the u box (3 slots; the u/f
// ring has 3 slots then, for shared memory).  While plane p is processed, the box of plane p+1
// (just arrived) is corrected in place: every thread its own rows (in registers, then written
// back), the box ring nodes by all threads, the red ring threads the one node of that box they
// read during plane p themselves; nothing else reads that box before the plane barrier, so
// one barrier per plane remains.  The corrected iterate never reaches HBM.  Same separable
// interpolation order as k_prolong3d_flat (bitwise equal to the separate prolongation).
template <typename T, int MODE, bool ZERO, int NM, int RPT, bool CORR = false>
__global__ void __launch_bounds__(32 * TY / RPT, Geo<T>::MINB)
    k_sweep3d_rows(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_f, Geom g,
                   Coef<T> c, T* __restrict__ unew, int tiles_x, int ntiles, int zc, int nitems,
                   double* __restrict__ partial, const __grid_constant__ CUtensorMap tm_e, Geom gc) {
  using G = Geo<T>;
  using V = Vec<T, G::W>;
  constexpr int W = G::W, TX = G::TX, BX = G::BX, HX = G::HX, PX = G::PX, NR = G::NRED, RCOL = G::RCOL;
  constexpr int NTH = 32 * TY / RPT;
  constexpr bool RB = MODE == 1;
  constexpr bool NRM = NM == 1 || NM == 2;  // input residuals (NM 2: red nodes only)
  static_assert(TY % RPT == 0, "rows per thread");
  static_assert(NM != 3 || RB, "output black residuals: RBGS only");
  static_assert(!CORR || (NM == 0 && !ZERO && MODE != 2), "CORR: a plain sweep");
  constexpr int NSR = CORR ? 3 : G::NS;                     // u/f ring slots
  constexpr int PR_OFF = Ring<T, NSR>::BAR_OFF + 128;       // 3 PR planes, then (CORR) 3 coarse boxes
  constexpr int COFF = PR_OFF + 3 * G::PB;
  extern __shared__ __align__(128) unsigned char sm[];
  const Ring<T, NSR> R = ring_setup<T, NSR>(sm, &tm_u, &tm_f);
  T* spr = reinterpret_cast<T*>(sm + PR_OFF);
  auto su = [&](const T* base, int off) -> T { return ZERO ? (T)0 : base[off]; };
  auto svec = [&](const T* base, int off) -> V {
    if (ZERO) {
      V z;
#pragma unroll
      for (int k = 0; k < W; k++) z.v[k] = (T)0;
      return z;
    }
    return ld_vec(base + off);
  };

  const int tid = threadIdx.x, lane = tid & 31, wr = tid >> 5;
  const int ty0 = wr * RPT;                        // first tile row of the thread
  const int bo = (ty0 + 2) * BX + W * lane + HX;  // u-box offset of (ox, row 0); row k: + k BX
  const int fo = (ty0 + 1) * BX + W * lane + HX;  // f-box offset
  const int po = (ty0 + 1) * PX + W * lane + HX;  // PR offset
  uint32_t seq = 0;
  double nsum = 0.0;

  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    int tile, pa, pb;
    item_of(it, ntiles, zc, g.p_lo, g.p_hi, tile, pa, pb);
    const int x0 = (tile % tiles_x) * TX, y0 = (tile / tiles_x) * TY;
    const int ox = x0 + W * lane, oy0 = y0 + ty0;
    // interior flags of the thread's nodes as bits (k W + j): one register instead of RPT W
    // predicates, which the register-tight variants would otherwise recompute at every use
    uint32_t inm = 0;
#pragma unroll
    for (int k = 0; k < RPT; k++) {
      const bool rin = oy0 + k >= 1 && oy0 + k <= g.ny - 1;
#pragma unroll
      for (int j = 0; j < W; j++)
        if (rin && ox + j >= 1 && ox + j <= g.nx - 1) inm |= 1u << (k * W + j);
    }
    auto in = [&](int k, int j) -> bool { return (inm >> (k * W + j)) & 1u; };
    auto inrow = [&](int k) -> uint32_t { return (inm >> (k * W)) & ((1u << W) - 1u); };
    T* orow = unew + (long long)oy0 * g.pitch;
    // CORR (128 registers): the interior mask and the output row in shared memory, reloaded per
    // plane, so that their live ranges end at the plane instead of being rematerialised at every
    // use (measured FP32 0.449 -> 0.405 ms per level-0 launch; FP64 unchanged)
    constexpr int TCOFF = PR_OFF + 3 * G::PB + 3 * G::CB;
    if constexpr (CORR) {
      reinterpret_cast<uint32_t*>(sm + TCOFF)[tid] = inm;
      reinterpret_cast<T**>(sm + TCOFF + 1024)[tid] = orow;
    }

    const int qlo = RB ? pa - 3 : pa - 2, qlast = RB ? pb : pb - 1;
    const uint32_t nlo = seq;
    auto N = [&](int q) { return nlo + (uint32_t)(q - qlo); };
    // CORR: coarse plane K lives in coarse slot K % 3; step q (fine u plane z = q+1) also loads
    // coarse plane (z+1)/2 when z is odd (first needed there), the first step also z/2
    const int X0c = x0 / 2, Y0c = y0 / 2;
    auto Cs = [&](int K) -> T* { return reinterpret_cast<T*>(sm + COFF + (size_t)(((K % 3) + 3) % 3) * G::CB); };
    auto issue_step = [&](int q) {
      if (CORR) {
        uint64_t* bar = &R.full[N(q) % NSR];
        const int zg = q + 1 + g.p_glob0;
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
      for (int q = qlo; q < qlo + NSR && q <= qlast; q++) issue_step(q);

    // ---- CORR: u += P e (reading 13 order: x, then y, then z interpolation)
    const T half = (T)0.5;
    // V(x, y, Zg): the W nodes (x .. x+W-1, x even) of row y after the x- and y-interpolation of
    // coarse plane Zg; fine plane z then takes V(z/2), or (V(Z) + V(Z+1)) / 2 when z is odd
    auto Vxy = [&](const T* cb, bool yodd) -> V {  // cb: the coarse box at (x/2, y/2)
      T a[NR + 1], b[NR + 1];
#pragma unroll
      for (int i = 0; i <= NR; i++) a[i] = cb[i];
      V v;
#pragma unroll
      for (int i = 0; i < NR; i++) {
        v.v[2 * i] = a[i];
        v.v[2 * i + 1] = mul(half, add(a[i], a[i + 1]));
      }
      if (yodd) {
#pragma unroll
        for (int i = 0; i <= NR; i++) b[i] = cb[G::CBX + i];
#pragma unroll
        for (int i = 0; i < NR; i++) {
          v.v[2 * i] = mul(half, add(v.v[2 * i], b[i]));
          v.v[2 * i + 1] = mul(half, add(v.v[2 * i + 1], mul(half, add(b[i], b[i + 1]))));
        }
      }
      return v;
    };
    // The box vectors around the tile that the stencils read, one per thread of warps 0-5:
    // rows y0-1 / y0+TY (warps 0 / 1: the ring rows whose red nodes those warps relax), the
    // halo vectors of the tile rows (warp 2, which relaxes the ring columns), rows y0-2 /
    // y0+TY+1 (warps 3 / 4), the corner vectors (warp 5)
    constexpr int VH = TX / W + 1;  // index of the right halo vector (left: 0)
    int rvy = -1000000, rvi = 0;
    if (CORR) {
      if (wr == 0 || wr == 1 || wr == 3 || wr == 4) {
        rvy = wr == 0 ? y0 - 1 : wr == 1 ? y0 + TY : wr == 3 ? y0 - 2 : y0 + TY + 1;
        rvi = lane + 1;
      } else if (wr == 2) {
        rvy = y0 + (lane & 15);
        rvi = lane < 16 ? 0 : VH;
      } else if (wr == 5 && lane < 8) {
        const int rr = lane & 3;
        rvy = rr < 2 ? y0 - 2 + rr : y0 + TY + rr - 2;
        rvi = lane < 4 ? 0 : VH;
      }
    }
    const bool has_rv = rvy > -1000000;
    const int rvx = x0 - HX + W * rvi;
    const int rbo = (rvy - y0 + 2) * BX + W * rvi;
    uint32_t rinm = 0;  // interior flags of the ring vector's nodes
#pragma unroll
    for (int j = 0; j < W; j++)
      if (has_rv && rvy >= 1 && rvy <= g.ny - 1 && rvx + j >= 1 && rvx + j <= g.nx - 1) rinm |= 1u << j;
    bool own_all = true;
#pragma unroll
    for (int k = 0; k < RPT; k++)
#pragma unroll
      for (int j = 0; j < W; j++) own_all = own_all && in(k, j);
    int cZ = -1000000;  // coarse plane of cA (cB: cZ + 1 when cHaveB)
    V cA[RPT + 1], cB[RPT + 1];  // [RPT]: the ring vector
    bool cHaveB = false;
    // offsets of the thread's vectors in a coarse box (constant over the item's planes)
    int coff[RPT + 1];
#pragma unroll
    for (int k = 0; k < RPT; k++) coff[k] = (((oy0 + k) >> 1) - Y0c + 1) * G::CBX + ((ox >> 1) - X0c + G::CHX);
    coff[RPT] = has_rv ? ((rvy >> 1) - Y0c + 1) * G::CBX + ((rvx >> 1) - X0c + G::CHX) : 0;
    auto cache_row = [&](int k, const T* base) {
      return Vxy(base + coff[k], k < RPT ? (((oy0 + k) & 1) != 0) : ((rvy & 1) != 0));
    };
    // fine plane zl (local): the own rows uv[k] += P e in registers, the ring vector in the box Ub
    auto correct = [&](V* uv, int zl, T* Ub) {
      const int zg = zl + g.p_glob0;
      if (zg < 1 || zg > g.nz - 1) return;  // boundary / outside planes: no correction
      const int nk = has_rv ? RPT + 1 : RPT;
      if ((zg >> 1) != cZ) {
        if (cHaveB && (zg >> 1) == cZ + 1) {
#pragma unroll
          for (int k = 0; k <= RPT; k++) cA[k] = cB[k];
        } else {
          const T* base = Cs(zg >> 1);
#pragma unroll
          for (int k = 0; k <= RPT; k++)
            if (k < nk) cA[k] = cache_row(k, base);
        }
        cZ = zg >> 1;
        cHaveB = false;
      }
      if ((zg & 1) && !cHaveB) {
        const T* base = Cs(cZ + 1);
#pragma unroll
        for (int k = 0; k <= RPT; k++)
          if (k < nk) cB[k] = cache_row(k, base);
        cHaveB = true;
      }
      // the plane parity is CTA-uniform and most threads' nodes are all interior: branch on both
      // instead of selecting per element
      auto apply = [&](auto ODDc) {
        constexpr bool ODD = decltype(ODDc)::value;
        auto pe = [&](int k, int j) { return ODD ? mul(half, add(cA[k].v[j], cB[k].v[j])) : cA[k].v[j]; };
        if (own_all) {
#pragma unroll
          for (int k = 0; k < RPT; k++)
#pragma unroll
            for (int j = 0; j < W; j++) uv[k].v[j] = add(uv[k].v[j], pe(k, j));
        } else {
#pragma unroll
          for (int k = 0; k < RPT; k++)
#pragma unroll
            for (int j = 0; j < W; j++)
              if (in(k, j)) uv[k].v[j] = add(uv[k].v[j], pe(k, j));
        }
        if (has_rv) {
          V rv = ld_vec(Ub + rbo);
#pragma unroll
          for (int j = 0; j < W; j++)
            if ((rinm >> j) & 1u) rv.v[j] = add(rv.v[j], pe(RPT, j));
          st_vec(Ub + rbo, rv);
        }
      };
      if (zg & 1)
        apply(std::true_type());
      else
        apply(std::false_type());
    };

    R.wait(N(qlo));
    R.wait(N(qlo + 1));
    V um[RPT], u0[RPT], up[RPT];
    if constexpr (CORR) {  // the first two boxes, in shared memory, before anyone reads them
#pragma unroll
      for (int b = 0; b < 2; b++) {
        T* Ub = R.U(N(qlo + b));
        V own[RPT];
#pragma unroll
        for (int k = 0; k < RPT; k++) own[k] = ld_vec(Ub + bo + k * BX);
        correct(own, qlo + 1 + b, Ub);
#pragma unroll
        for (int k = 0; k < RPT; k++) st_vec(Ub + bo + k * BX, own[k]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < RPT; k++) {
      um[k] = svec(R.U(N(qlo)), bo + k * BX);
      u0[k] = svec(R.U(N(qlo + 1)), bo + k * BX);
    }

    // RB ring threads: the red nodes of the ring rows y0-1 / y0+TY and of the ring columns
    // x0-1 / x0+TX, one node per lane (FP32, NR = 2 per lane and row: warps 0-3, warp w row
    // w & 1, node w >> 1), the columns by warp RWARPS.  CORR: warps 0 / 1 take both nodes of
    // their lane's vector (the vector they corrected), the columns warp 2.
    constexpr int RWARPS = CORR ? 2 : 2 * NR;
    constexpr int MPL = CORR ? NR : 1;  // ring-row nodes per lane
    static_assert(RWARPS < NTH / 32, "ring warps");
    const bool ring_row = RB && wr < RWARPS;
    const bool ring_col = RB && wr == RWARPS && lane < 2 * RCOL;
    const int mring = (ring_row && !CORR) ? (wr >> 1) : 0;
    const int nring = ring_row ? MPL : (ring_col ? 1 : 0);
    auto ring_pos = [&](int pgl, int m, int& x, int& y) {
      if (wr < RWARPS) {
        y = (wr & 1) == 0 ? y0 - 1 : y0 + TY;
        x = x0 + W * lane + 2 * m + ((y + pgl) & 1);
      } else {
        x = lane < RCOL ? x0 - 1 : x0 + TX;
        y = y0 + 2 * (lane % RCOL) + ((x + y0 + pgl) & 1);
      }
    };
    T rzm[MPL];  // ring thread: u(p-1) at its plane-p ring node(s)
#pragma unroll
    for (int mm = 0; mm < MPL; mm++) {
      rzm[mm] = (T)0;
      if (mm < nring) {
        int x, y;
        ring_pos(pa - 1 + g.p_glob0, mring + mm, x, y);
        rzm[mm] = su(R.U(N(qlo)), (y - y0 + 2) * BX + (x - x0 + HX));
      }
    }
    __syncthreads();  // step qlo lives on in registers only: refill its slot
    if (tid == 0 && qlo + NSR <= qlast) {
      fence_proxy_async();
      issue_step(qlo + NSR);
    }

    if constexpr (RB) {
      T pr1[RPT][NR], pr2[RPT][NR];  // own red values of planes p-1, p-2, per row
      V fprev[RPT];                   // f(p-1)
#pragma unroll
      for (int k = 0; k < RPT; k++) {
#pragma unroll
        for (int m = 0; m < NR; m++) pr1[k][m] = pr2[k][m] = (T)0;
#pragma unroll
        for (int j = 0; j < W; j++) fprev[k].v[j] = (T)0;
      }
      int ps = (((pa - 1) % 3) + 3) % 3;  // PR slot of plane p (rotates 0, 1, 2)
      for (int p = pa - 1; p <= pb; p++) {
        R.wait(N(p));
        if constexpr (CORR) {
          inm = reinterpret_cast<volatile uint32_t*>(sm + TCOFF)[tid];
          orow = reinterpret_cast<T* volatile*>(sm + TCOFF + 1024)[tid];
        }
        const T* U0 = R.U(N(p - 1));  // u(p)
        const T* Up = R.U(N(p));      // u(p+1)
        const T* F0 = R.F(N(p));      // f(p)
        T* PR = spr + (size_t)ps * (G::PB / sizeof(T));
#pragma unroll
        for (int k = 0; k < RPT; k++) up[k] = svec(Up, bo + k * BX);
        const int pgl = p + g.p_glob0;
        if constexpr (CORR) {  // plane p+1's box: own rows (registers + write-back) and the ring vectors
          correct(up, p + 1, const_cast<T*>(Up));
#pragma unroll
          for (int k = 0; k < RPT; k++) st_vec(const_cast<T*>(Up) + bo + k * BX, up[k]);
          if (wr == RWARPS) __syncwarp();  // the ring columns' z+1 nodes, corrected by other lanes
        }
        const bool pl_in = pgl >= 1 && pgl <= g.nz - 1;
        const int kr0 = (oy0 + pgl) & 1;  // red offset of row 0 (row k: kr0 ^ (k & 1)), warp uniform
        const bool nrm_here = NRM && p >= pa && p < pb;
        T pr0[RPT][NR];
        V fcur[RPT];
#pragma unroll
        for (int k = 0; k < RPT; k++) fcur[k] = ld_vec(F0 + fo + k * BX);
        auto red_stage = [&](auto KR0c) {
          static_for<RPT>([&](auto Kc) {
            constexpr int K = decltype(Kc)::value;
            constexpr int KR = decltype(KR0c)::value ^ (K & 1);
            const V dn = K == 0 ? svec(U0, bo - BX) : u0[K > 0 ? K - 1 : 0];
            const V upr = K == RPT - 1 ? svec(U0, bo + (K + 1) * BX) : u0[K < RPT - 1 ? K + 1 : 0];
            const T edge = KR == 0 ? su(U0, bo + K * BX - 1) : su(U0, bo + K * BX + W);
            if constexpr (NM == 1) {
              if (nrm_here) {  // black nodes of plane p: residual of the old iterate
                const T oedge = KR == 0 ? su(U0, bo + K * BX + W) : su(U0, bo + K * BX - 1);
#pragma unroll
                for (int m = 0; m < NR; m++) {
                  const int j = (1 - KR) + 2 * m;
                  const T l = j == 0 ? oedge : u0[K].v[j > 0 ? j - 1 : 0];
                  const T r = j == W - 1 ? oedge : u0[K].v[j < W - 1 ? j + 1 : 0];
                  const double rr = (double)sub(
                      fcur[K].v[j], apply_A(c, u0[K].v[j], l, r, dn.v[j], upr.v[j], um[K].v[j], up[K].v[j]));
                  if (in(K, j)) nsum = acc_sq_d<T>(nsum, rr);
                }
              }
            }
            V pv = u0[K];
#pragma unroll
            for (int m = 0; m < NR; m++) {
              const int j = KR + 2 * m;
              const T ctr = u0[K].v[j];
              const T l = j == 0 ? edge : u0[K].v[j > 0 ? j - 1 : 0];
              const T r = j == W - 1 ? edge : u0[K].v[j < W - 1 ? j + 1 : 0];
              const T res = sub(fcur[K].v[j], apply_A(c, ctr, l, r, dn.v[j], upr.v[j], um[K].v[j], up[K].v[j]));
              const T v = add(ctr, mul(c.wd, res));
              if (NRM && nrm_here && in(K, j)) nsum = acc_sq<T>(nsum, res);
              const T prv = (pl_in && in(K, j)) ? v : ctr;
              pv.v[j] = prv;
              pr0[K][m] = prv;
            }
            if constexpr (sizeof(T) == 8)
              *reinterpret_cast<double2*>(PR + po + K * PX) = make_double2(pv.v[0], pv.v[1]);
            else
              *reinterpret_cast<float4*>(PR + po + K * PX) = make_float4(pv.v[0], pv.v[1], pv.v[2], pv.v[3]);
          });
        };
        if (kr0)
          red_stage(std::integral_constant<int, 1>());
        else
          red_stage(std::integral_constant<int, 0>());
#pragma unroll
        for (int mm = 0; mm < MPL; mm++) {  // the red ring node(s) of plane p
          if (mm < nring) {
            int x, y;
            ring_pos(pgl, mring + mm, x, y);
            const int rb = (y - y0 + 2) * BX + (x - x0 + HX);
            const T ctr = su(U0, rb);
            const T v = relax(c, ctr, su(U0, rb - 1), su(U0, rb + 1), su(U0, rb - BX), su(U0, rb + BX), rzm[mm],
                              su(Up, rb), F0[(y - y0 + 1) * BX + (x - x0 + HX)]);
            const bool ok = pl_in && x >= 1 && x <= g.nx - 1 && y >= 1 && y <= g.ny - 1;
            PR[(y - y0 + 1) * PX + (x - x0 + HX)] = ok ? v : ctr;
            ring_pos(pgl + 1, mring + mm, x, y);
            rzm[mm] = su(U0, (y - y0 + 2) * BX + (x - x0 + HX));
          }
        }
        __syncthreads();
        // every thread is past plane p-2's black update and plane p's red stage: step p-1
        // (u(p), f(p-1); f(p-1) is in registers) is consumed
        if (tid == 0 && p >= pa - 1 && p - 1 + NSR <= qlast) {
          fence_proxy_async();
          issue_step(p - 1 + NSR);
        }
        const int bp = p - 1;
        if (bp >= pa) {
          const T* P = spr + (size_t)(ps == 0 ? 2 : ps - 1) * (G::PB / sizeof(T));
          auto black_stage = [&](auto KB0c) {
            static_for<RPT>([&](auto Kc) {
              constexpr int K = decltype(Kc)::value;
              constexpr int KB = decltype(KB0c)::value ^ (K & 1);
              T pdn[NR], pup[NR];
              if constexpr (K == 0) {
                if constexpr (W == 4) {
                  const V a = ld_vec(P + po - PX);
#pragma unroll
                  for (int m = 0; m < NR; m++) pdn[m] = a.v[KB + 2 * m];
                } else {
                  pdn[0] = P[po + KB - PX];
                }
              } else {
#pragma unroll
                for (int m = 0; m < NR; m++) pdn[m] = pr1[K > 0 ? K - 1 : 0][m];
              }
              if constexpr (K == RPT - 1) {
                if constexpr (W == 4) {
                  const V a = ld_vec(P + po + (K + 1) * PX);
#pragma unroll
                  for (int m = 0; m < NR; m++) pup[m] = a.v[KB + 2 * m];
                } else {
                  pup[0] = P[po + (K + 1) * PX + KB];
                }
              } else {
#pragma unroll
                for (int m = 0; m < NR; m++) pup[m] = pr1[K < RPT - 1 ? K + 1 : 0][m];
              }
              const T edge = KB == 0 ? P[po + K * PX - 1] : P[po + K * PX + W];
              V o;
#pragma unroll
              for (int m = 0; m < NR; m++) o.v[(1 - KB) + 2 * m] = pr1[K][m];
#pragma unroll
              for (int m = 0; m < NR; m++) {
                const int j = KB + 2 * m;
                const T ctr = um[K].v[j];
                const T l = (KB == 0 && m == 0) ? edge : pr1[K][KB == 1 ? m : (m > 0 ? m - 1 : 0)];
                const T r = (KB == 1 && m == NR - 1) ? edge : pr1[K][KB == 0 ? m : (m + 1 < NR ? m + 1 : 0)];
                // relax() written out: s is also the stencil sum of the output's residual (NM 3)
                T sm_ = mul(c.cx, add(l, r));
                sm_ = add(sm_, mul(c.cy, add(pdn[m], pup[m])));
                sm_ = add(sm_, mul(c.cz, add(pr2[K][m], pr0[K][m])));
                const T fb = fprev[K].v[j];
                const T v = add(ctr, mul(c.wd, sub(fb, sub(mul(c.D, ctr), sm_))));
                if constexpr (NM == 3) {
                  if (in(K, j)) nsum = acc_sq<T>(nsum, sub(fb, sub(mul(c.D, v), sm_)));
                }
                o.v[j] = in(K, j) ? v : ctr;
              }
              store_vec_m(orow + (long long)K * g.pitch + (long long)bp * g.pstride, ox, inrow(K), o);
            });
          };
          if (kr0)
            black_stage(std::integral_constant<int, 1>());
          else
            black_stage(std::integral_constant<int, 0>());
        }
        ps = ps == 2 ? 0 : ps + 1;
#pragma unroll
        for (int k = 0; k < RPT; k++) {
          um[k] = u0[k];
          u0[k] = up[k];
          fprev[k] = fcur[k];
#pragma unroll
          for (int m = 0; m < NR; m++) {
            pr2[k][m] = pr1[k][m];
            pr1[k][m] = pr0[k][m];
          }
        }
      }
    } else {
      for (int p = pa; p < pb; p++) {
        R.wait(N(p));
        const T* U0 = R.U(N(p - 1));
        const T* F0 = R.F(N(p));
#pragma unroll
        for (int k = 0; k < RPT; k++) up[k] = svec(R.U(N(p)), bo + k * BX);
        if constexpr (CORR) {
          T* Upw = R.U(N(p));
          correct(up, p + 1, Upw);
#pragma unroll
          for (int k = 0; k < RPT; k++) st_vec(Upw + bo + k * BX, up[k]);
        }
        static_for<RPT>([&](auto Kc) {
          constexpr int K = decltype(Kc)::value;
          const V fv = ld_vec(F0 + fo + K * BX);
          const V dn = K == 0 ? svec(U0, bo - BX) : u0[K > 0 ? K - 1 : 0];
          const V upr = K == RPT - 1 ? svec(U0, bo + (K + 1) * BX) : u0[K < RPT - 1 ? K + 1 : 0];
          const T el = su(U0, bo + K * BX - 1), er = su(U0, bo + K * BX + W);
          V o;
#pragma unroll
          for (int j = 0; j < W; j++) {
            const T l = j == 0 ? el : u0[K].v[j > 0 ? j - 1 : 0];
            const T r = j == W - 1 ? er : u0[K].v[j < W - 1 ? j + 1 : 0];
            const T res = sub(fv.v[j], apply_A(c, u0[K].v[j], l, r, dn.v[j], upr.v[j], um[K].v[j], up[K].v[j]));
            if (MODE == 2) {
              if (in(K, j)) nsum = acc_sq_d<T>(nsum, (double)res);
            } else {
              if (NRM && in(K, j)) nsum = acc_sq<T>(nsum, res);
              o.v[j] = in(K, j) ? add(u0[K].v[j], mul(c.wd, res)) : u0[K].v[j];
            }
          }
          if (MODE != 2) store_vec_m(orow + (long long)K * g.pitch + (long long)p * g.pstride, ox, inrow(K), o);
        });
        __syncthreads();
        if (tid == 0 && p - 1 + NSR <= qlast) {
          fence_proxy_async();
          issue_step(p - 1 + NSR);
        }
#pragma unroll
        for (int k = 0; k < RPT; k++) {
          um[k] = u0[k];
          u0[k] = up[k];
        }
      }
    }
    seq = N(qlast) + 1;
    __syncthreads();
  }
  if (MODE == 2 || NM != 0) {  // fixed-order block reduction -> one partial per CTA
    double* red = reinterpret_cast<double*>(sm);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nsum = __dadd_rn(nsum, __shfl_down_sync(0xffffffffu, nsum, o));
    if (lane == 0) red[wr] = nsum;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w2 = 0; w2 < NTH / 32; w2++) t = __dadd_rn(t, red[w2]);
      partial[blockIdx.x] = t;
    }
  }
}

// ---------------------------------------------------------------------------
// Fused residual + full-weighting restriction.  Work items are (coarse tile,
// coarse z-chunk); the fine tile is 2x the coarse tile (x0 = 2 X0).  Per fine
// plane q: r for every node of the tile (u column in registers) and the
// low-side ring nodes (row y0-1, column x0-1) into smem; then the coarse nodes
// of the tile form their x- then y-sums of plane q and keep the last three in
// registers: when q = 2P+1 the z-sum gives f_H(P) (reading 13 order).
// Row-blocked residual + restriction (the default): as k_resid_restrict3d, but a thread owns
// RPT consecutive fine rows of its x-vector (the rows' u(q) y-neighbours inside the thread
// come from registers) and CN / NTH coarse nodes.  Bitwise identical results.
template <typename T, int RPT>
__global__ void __launch_bounds__(32 * TY / RPT, Geo<T>::MINB)
    k_resid_restrict3d_rows(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_f,
                            Geom gf, Geom gc, Coef<T> c, T* __restrict__ fc, int tiles_x, int ntiles, int zcc,
                            int nitems) {
  using G = Geo<T>;
  using V = Vec<T, G::W>;
  constexpr int W = G::W, TX = G::TX, BX = G::BX, HX = G::HX, PX = G::PX;
  constexpr int NTH = 32 * TY / RPT;
  extern __shared__ __align__(128) unsigned char sm[];
  const Ring<T> R = ring_setup<T>(sm, &tm_u, &tm_f);
  T* const Rr2 = reinterpret_cast<T*>(sm + G::PR_OFF);

  const int tid = threadIdx.x, lane = tid & 31, wr = tid >> 5;
  const int ty0 = wr * RPT;
  const int pgf0 = gf.p_glob0;
  const int bo = (ty0 + 2) * BX + W * lane + HX;
  const int fo = (ty0 + 1) * BX + W * lane + HX;
  const int po = (ty0 + 1) * PX + W * lane + HX;
  const T two = (T)2;
  const T scale = (T)(1.0 / 64.0);
  constexpr int CNX = TX / 2, CN = (TX / 2) * (TY / 2), NC = CN / NTH;  // coarse nodes per thread
  static_assert(CN % NTH == 0 && CNX % 32 == 0, "coarse mapping: whole warps per coarse row");
  uint32_t seq = 0;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    int tile, Pa, Pb;
    item_of(it, ntiles, zcc, gc.p_lo, gc.p_hi, tile, Pa, Pb);
    const int X0 = (tile % tiles_x) * (TX / 2), Y0 = (tile / tiles_x) * (TY / 2);
    const int x0 = 2 * X0, y0 = 2 * Y0;
    const int ox = x0 + W * lane, oy0 = y0 + ty0;
    uint32_t inm = 0;  // interior flags (bit k W + j), as in k_sweep3d_rows
#pragma unroll
    for (int k = 0; k < RPT; k++) {
      const bool rin = oy0 + k >= 1 && oy0 + k <= gf.ny - 1;
#pragma unroll
      for (int j = 0; j < W; j++)
        if (rin && ox + j >= 1 && ox + j <= gf.nx - 1) inm |= 1u << (k * W + j);
    }
    // low-side ring: row y0-1 for x in [x0-1, x0+TX-1] (TX+1 nodes), column x0-1 for y in [y0, y0+TY-1]
    constexpr int NRING = TX + 1 + TY;
    constexpr int RING_PER = (NRING + NTH - 1) / NTH;  // ring nodes per thread (1 or 2)
    int rb[RING_PER], rf[RING_PER], rpo[RING_PER];
    bool has_ring[RING_PER], ring_in[RING_PER];
#pragma unroll
    for (int s = 0; s < RING_PER; s++) {
      const int e = tid + s * NTH;
      has_ring[s] = e < NRING;
      const int rx = e < TX + 1 ? x0 - 1 + e : x0 - 1;
      const int ryy = e < TX + 1 ? y0 - 1 : y0 + e - (TX + 1);
      ring_in[s] = rx >= 1 && rx <= gf.nx - 1 && ryy >= 1 && ryy <= gf.ny - 1;
      rb[s] = (ryy - y0 + 2) * BX + (rx - x0 + HX);
      rf[s] = (ryy - y0 + 1) * BX + (rx - x0 + HX);
      rpo[s] = (ryy - y0 + 1) * PX + (rx - x0 + HX);
    }
    int co[NC];
    bool cnode[NC];
    T* crow[NC];
#pragma unroll
    for (int s = 0; s < NC; s++) {
      const int ci = tid + s * NTH, ccx = ci % CNX, ccy = ci / CNX;
      co[s] = (2 * ccy + 1) * PX + 2 * ccx + HX;  // r offset of fine (2I, 2J)
      const int I = X0 + ccx, J = Y0 + ccy;
      cnode[s] = I >= 1 && I <= gc.nx - 1 && J >= 1 && J <= gc.ny - 1;
      crow[s] = fc + (long long)J * gc.pitch + I;
    }

    const int qf0 = 2 * (Pa + gc.p_glob0) - pgf0;
    const int qf1 = 2 * (Pb - 1 + gc.p_glob0) - pgf0;
    const int rlo = qf0 - 1, rhi = qf1 + 1;
    const int qlo = rlo - 2, qlast = rhi;
    const uint32_t nlo = seq;
    auto N = [&](int q) { return nlo + (uint32_t)(q - qlo); };
    if (tid == 0)
      for (int q = qlo; q < qlo + G::NS && q <= qlast; q++) R.issue(N(q), &tm_u, &tm_f, x0, y0, q + 1, q, true);
    R.wait(N(qlo));
    R.wait(N(qlo + 1));
    V um[RPT], u0[RPT], up[RPT];
#pragma unroll
    for (int k = 0; k < RPT; k++) {
      um[k] = ld_vec(R.U(N(qlo)) + bo + k * BX);
      u0[k] = ld_vec(R.U(N(qlo + 1)) + bo + k * BX);
    }
    T rzm[RING_PER];
#pragma unroll
    for (int s = 0; s < RING_PER; s++) rzm[s] = has_ring[s] ? R.U(N(qlo))[rb[s]] : (T)0;
    __syncthreads();
    if (tid == 0 && qlo + G::NS <= qlast) {
      fence_proxy_async();
      R.issue(N(qlo + G::NS), &tm_u, &tm_f, x0, y0, qlo + G::NS + 1, qlo + G::NS, true);
    }
    T ty1[NC], ty2[NC];
#pragma unroll
    for (int s = 0; s < NC; s++) ty1[s] = ty2[s] = (T)0;
    for (int q = rlo; q <= rhi; q++) {
      R.wait(N(q));
      const T* U0 = R.U(N(q - 1));
      const T* Up = R.U(N(q));
      const T* F0 = R.F(N(q));
      T* Rr = Rr2 + (size_t)(q & 1) * (G::PB / sizeof(T));
#pragma unroll
      for (int k = 0; k < RPT; k++) up[k] = ld_vec(Up + bo + k * BX);
      const int pgl = q + pgf0;
      const bool pl_in = pgl >= 1 && pgl <= gf.nz - 1;
      static_for<RPT>([&](auto Kc) {
        constexpr int K = decltype(Kc)::value;
        const V fv = ld_vec(F0 + fo + K * BX);
        const V dn = K == 0 ? ld_vec(U0 + bo - BX) : u0[K > 0 ? K - 1 : 0];
        const V upr = K == RPT - 1 ? ld_vec(U0 + bo + (K + 1) * BX) : u0[K < RPT - 1 ? K + 1 : 0];
        const T el = U0[bo + K * BX - 1], er = U0[bo + K * BX + W];
        V rv;
#pragma unroll
        for (int j = 0; j < W; j++) {
          const T l = j == 0 ? el : u0[K].v[j > 0 ? j - 1 : 0];
          const T r = j == W - 1 ? er : u0[K].v[j < W - 1 ? j + 1 : 0];
          const T rr = sub(fv.v[j], apply_A(c, u0[K].v[j], l, r, dn.v[j], upr.v[j], um[K].v[j], up[K].v[j]));
          rv.v[j] = pl_in && ((inm >> (K * W + j)) & 1u) ? rr : (T)0;
        }
        if constexpr (sizeof(T) == 8)
          *reinterpret_cast<double2*>(Rr + po + K * PX) = make_double2(rv.v[0], rv.v[1]);
        else
          *reinterpret_cast<float4*>(Rr + po + K * PX) = make_float4(rv.v[0], rv.v[1], rv.v[2], rv.v[3]);
      });
#pragma unroll
      for (int s = 0; s < RING_PER; s++) {
        if (has_ring[s]) {
          const int b = rb[s];
          const T uc = U0[b];
          const T r = sub(F0[rf[s]], apply_A(c, uc, U0[b - 1], U0[b + 1], U0[b - BX], U0[b + BX], rzm[s], Up[b]));
          Rr[rpo[s]] = pl_in && ring_in[s] ? r : (T)0;
          rzm[s] = uc;
        }
      }
      __syncthreads();
      if (tid == 0 && q - 1 + G::NS <= qlast) {
        fence_proxy_async();
        R.issue(N(q - 1 + G::NS), &tm_u, &tm_f, x0, y0, q + G::NS, q - 1 + G::NS, true);
      }
      using P2 = std::conditional_t<sizeof(T) == 8, double2, float2>;
#pragma unroll
      for (int s = 0; s < NC; s++) {
        T tx[3];
#pragma unroll
        for (int dy = -1; dy <= 1; dy++) {
          const T* row = Rr + co[s] + dy * PX;
          const P2 pr = *reinterpret_cast<const P2*>(row);
          T left = __shfl_up_sync(0xffffffffu, pr.y, 1);
          if (lane == 0) left = row[-1];
          tx[dy + 1] = add(add(left, pr.y), mul(two, pr.x));
        }
        const T ty0v = add(add(tx[0], tx[2]), mul(two, tx[1]));
        if (cnode[s] && (pgl & 1) == 1 && q >= qf0 + 1) {
          const int Pc = ((pgl - 1) >> 1) - gc.p_glob0;
          crow[s][(long long)Pc * gc.pstride] = mul(add(add(ty2[s], ty0v), mul(two, ty1[s])), scale);
        }
        ty2[s] = ty1[s];
        ty1[s] = ty0v;
      }
#pragma unroll
      for (int k = 0; k < RPT; k++) {
        um[k] = u0[k];
        u0[k] = up[k];
      }
    }
    seq = N(qlast) + 1;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// cuTensorMapEncodeTiled through the runtime's driver entry point, so that the
// library does not link libcuda (it must load on GPU-less hosts for the ABI tests).
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {  // thread-safe one-time lookup
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
  }();
  return fn;
}

CUresult encode_tiled(CUtensorMap* tm, bool fp64, int rank, const void* base, const unsigned long long* dims,
                      const unsigned long long* strides, const unsigned* box) {
  PFN_cuTensorMapEncodeTiled_v12000 cuTensorMapEncodeTiled = encode_fn();
  if (!cuTensorMapEncodeTiled) return CUDA_ERROR_NOT_FOUND;
  cuuint64_t d[5], sd[4];
  cuuint32_t b[5], estr[5];
  for (int i = 0; i < rank; i++) {
    d[i] = dims[i];
    b[i] = box[i];
    estr[i] = 1;
    if (i + 1 < rank) sd[i] = strides[i];
  }
  return cuTensorMapEncodeTiled(tm, fp64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                (cuuint32_t)rank, const_cast<void*>(base), d, sd, b, estr,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

static CUresult encode(CUtensorMap* tm, const void* base, const Geom& g, int esz, int box_rows) {
  PFN_cuTensorMapEncodeTiled_v12000 cuTensorMapEncodeTiled = encode_fn();
  if (!cuTensorMapEncodeTiled) return CUDA_ERROR_NOT_FOUND;
  cuuint64_t dims[3] = {(cuuint64_t)(g.nx + 1), (cuuint64_t)g.rows, (cuuint64_t)g.planes};
  cuuint64_t strides[2] = {(cuuint64_t)(g.pitch * esz), (cuuint64_t)(g.pstride * esz)};
  const int tx = 32 * (16 / esz);  // Geo<T>::TX
  cuuint32_t box[3] = {(cuuint32_t)(tx + 2 * (16 / esz)), (cuuint32_t)box_rows, 1};
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
  if (!g.three_d) return pm2::supported(g, min_nx);
  return g.three_d && g.nx >= (min_nx < 16 ? 16 : min_nx) && g.ny >= 16 && (g.p_hi - g.p_lo) >= 4;
}

// First use of a kernel: opt in to its dynamic shared memory and return the
// number of CTAs the device keeps resident (cached per kernel).
template <class K>
static int prepare_kernel(K kernel, int smem, int threads = NT) {
  return resident_ctas((const void*)kernel, threads, smem);
}

// rows per thread of the row-blocked sweep (k_sweep3d_rows) and its CTA size
constexpr int RPT = 2;
constexpr int NTR = 32 * TY / RPT;

// z-chunk size.  Measured on the 513^3 RBGS sweep (tools/scan_zc.py): what
// matters is a nearly full last wave of resident CTAs and enough waves (>= ~8)
// to balance SMs; the halo re-loads of short chunks mostly hit L2.  So: among
// chunk lengths >= 16 planes, minimise (ceil(waves)/waves) * (1 + halo/(2 zc))
// plus a small penalty below 8 waves.
// L2-resident levels (three arrays < 100 MB of the 126 MB L2) may use chunks down to 4 planes: their halo
// re-reads are L2 hits, and 16-plane chunks leave most of the GPU idle on 129^3 (measured C2
// 0.190 -> 0.165 ms moving this bound from 48 to 100 MB: the 129^3 FP64 level is 55 MB).
static int min_zc_for(const Geom& g, size_t esz) {
  return (double)g.planes * (double)g.pstride * (double)esz * 3.0 < 100e6 ? 4 : 16;
}

static int choose_zc(long long ntiles, int np, int resident, int halo, int min_zc = 16) {
  int best = np;
  double best_cost = 1e300;
  for (int c = 1; c <= 256 && c <= np; c++) {
    const int zc = (np + c - 1) / c;
    if (zc < min_zc && c > 1) break;
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
                         cudaStream_t st, double* partial, int* npartial, const T* ecoarse,
                         const Geom* gcoarse, SweepNorm nm) {
  if (!g.three_d) {
    if (ecoarse || (partial && nm != SN_INPUT)) return cudaErrorInvalidValue;  // 3D only
    return pm2::launch_sweep<T>(g, c, rbgs, uin, f, uout, zero_in, st, partial, npartial);
  }
  const Geom gce = gcoarse ? *gcoarse : Geom{};
  CUtensorMap te;
  memset(&te, 0, sizeof te);
  if (ecoarse && encode_coarse(&te, ecoarse, gce, sizeof(T), Geo<T>::CBX, Geo<T>::CBY) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  using G = Geo<T>;
  CUtensorMap tu, tf;
  CUresult e1 = encode(&tu, uin ? uin : f, g, sizeof(T), G::BYU), e2 = encode(&tf, f, g, sizeof(T), G::BYF);
  if (e1 != CUDA_SUCCESS || e2 != CUDA_SUCCESS) return cudaErrorInvalidValue;
  const int tiles_x = (g.nx + G::TX - 1) / G::TX, tiles_y = (g.ny + TY - 1) / TY;
  const int ntiles = tiles_x * tiles_y;
  const int np = g.p_hi - g.p_lo;
  auto gor = [&](auto kernel, int smem) {
    const int resident = prepare_kernel(kernel, smem, NTR);
    const int zc = choose_zc(ntiles, np, resident, rbgs ? 4 : 2, min_zc_for(g, sizeof(T)));
    const int nitems = ntiles * ((np + zc - 1) / zc);
    if (npartial) *npartial = nitems;
    kernel<<<nitems, NTR, smem, st>>>(tu, tf, g, c, uout, tiles_x, ntiles, zc, nitems, partial, te, gce);
  };
  if (ecoarse) {  // CORR: 3-slot u/f ring + 3 coarse boxes
    constexpr int smem_corr = Ring<T, 3>::BAR_OFF + 128 + 3 * G::PB + 3 * G::CB + 1024 + 2048;
    static_assert(smem_corr <= G::SMEM, "CORR fits the plain sweep's shared memory");
    rbgs ? gor(k_sweep3d_rows<T, 1, false, 0, RPT, true>, smem_corr)
         : gor(k_sweep3d_rows<T, 0, false, 0, RPT, true>, smem_corr);
  } else if (partial && !zero_in) {
    if (!rbgs) {
      if (nm != SN_INPUT) return cudaErrorInvalidValue;
      gor(k_sweep3d_rows<T, 0, false, 1, RPT>, G::SMEM);
    } else if (nm == SN_INPUT) {
      gor(k_sweep3d_rows<T, 1, false, 1, RPT>, G::SMEM);
    } else if (nm == SN_INPUT_RED) {
      gor(k_sweep3d_rows<T, 1, false, 2, RPT>, G::SMEM);
    } else {
      gor(k_sweep3d_rows<T, 1, false, 3, RPT>, G::SMEM);
    }
  } else if (rbgs)
    zero_in ? gor(k_sweep3d_rows<T, 1, true, 0, RPT>, G::SMEM) : gor(k_sweep3d_rows<T, 1, false, 0, RPT>, G::SMEM);
  else
    zero_in ? gor(k_sweep3d_rows<T, 0, true, 0, RPT>, G::SMEM) : gor(k_sweep3d_rows<T, 0, false, 0, RPT>, G::SMEM);
  return cudaGetLastError();
}

// upper bound of the partials launch_sweep(..., partial, ...) writes for a level
template <typename T>
int sweep_partials(const Geom& g, bool rbgs) {
  if (!g.three_d) return pm2::sweep_partials<T>(g, rbgs);
  using G = Geo<T>;
  const int ntiles = ((g.nx + G::TX - 1) / G::TX) * ((g.ny + TY - 1) / TY);
  const int np = g.p_hi - g.p_lo;
  const int resident = rbgs ? prepare_kernel(k_sweep3d_rows<T, 1, false, 1, RPT>, G::SMEM, NTR)
                            : prepare_kernel(k_sweep3d_rows<T, 0, false, 1, RPT>, G::SMEM, NTR);
  int best = 0;
  for (int halo : {2, 4}) {
    const int zc = choose_zc(ntiles, np, resident, halo, min_zc_for(g, sizeof(T)));
    const int n = ntiles * ((np + zc - 1) / zc);
    if (n > best) best = n;
  }
  return best;
}

template <typename T>
int sweep_items(const Geom& g, bool rbgs) {
  using G = Geo<T>;
  const int ntiles = ((g.nx + G::TX - 1) / G::TX) * ((g.ny + TY - 1) / TY);
  const int np = g.p_hi - g.p_lo;
  const int resident = rbgs ? prepare_kernel(k_sweep3d_rows<T, 1, false, 1, RPT>, G::SMEM, NTR)
                            : prepare_kernel(k_sweep3d_rows<T, 0, false, 1, RPT>, G::SMEM, NTR);
  const int zc = choose_zc(ntiles, np, resident, rbgs ? 4 : 2, min_zc_for(g, sizeof(T)));
  return ntiles * ((np + zc - 1) / zc);
}

template <typename T>
int norm_partials(const Geom& g) {
  if (!g.three_d) return pm2::norm_partials<T>(g);
  using G = Geo<T>;
  const int ntiles = ((g.nx + G::TX - 1) / G::TX) * ((g.ny + TY - 1) / TY);
  const int np = g.p_hi - g.p_lo;
  const int resident = prepare_kernel(k_sweep3d_rows<T, 2, false, 0, RPT>, G::SMEM, NTR);
  const int zc = choose_zc(ntiles, np, resident, 2, min_zc_for(g, sizeof(T)));
  return ntiles * ((np + zc - 1) / zc);
}

template <typename T>
cudaError_t launch_norm(const Geom& g, const Coef<T>& c, const T* u, const T* f, double* partial, int* npartial,
                        cudaStream_t st) {
  if (!g.three_d) return pm2::launch_norm<T>(g, c, u, f, partial, npartial, st);
  using G = Geo<T>;
  CUtensorMap tu, tf;
  if (encode(&tu, u, g, sizeof(T), G::BYU) != CUDA_SUCCESS || encode(&tf, f, g, sizeof(T), G::BYF) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const int tiles_x = (g.nx + G::TX - 1) / G::TX, tiles_y = (g.ny + TY - 1) / TY;
  const int ntiles = tiles_x * tiles_y;
  const int np = g.p_hi - g.p_lo;
  auto kernel = k_sweep3d_rows<T, 2, false, 0, RPT>;
  const int resident = prepare_kernel(kernel, G::SMEM, NTR);
  const int zc = choose_zc(ntiles, np, resident, 2, min_zc_for(g, sizeof(T)));
  const int nitems = ntiles * ((np + zc - 1) / zc);
  *npartial = nitems;
  CUtensorMap te;
  memset(&te, 0, sizeof te);
  kernel<<<nitems, NTR, G::SMEM, st>>>(tu, tf, g, c, nullptr, tiles_x, ntiles, zc, nitems, partial, te, Geom{});
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Bi-/trilinear prolongation + correction u += P e, 3D.
// Pointwise in u, so no staging: thread = W fine nodes (2X .. 2X+W-1) of one row,
// marching z.  The thread's coarse values after the x- and y-interpolation of a
// coarse plane K, V(K), stay in registers for the 3 fine planes that use it;
// fine plane z = 2Z+dz gets dz ? (V(Z)+V(Z+1))/2 : V(Z) (reading 13 order).
// (Used with MG_FLAG_SEPARATE_PROLONG; by default the first post-sweep does it, CORR.)
// KZ planes per batch; MINB resident CTAs per SM (register cap); PIPE: the next batch's
// u vectors are loaded before the current batch is stored (software pipelining).
template <typename T, int KZ, int MINB, bool PIPE>
__global__ void __launch_bounds__(NT, MINB) k_prolong3d(Geom gf, Geom gc, const T* __restrict__ e, T* __restrict__ u,
                                                       int tiles_x, int ntiles, int zc, int nitems) {
  using G = Geo<T>;
  using Vt = Vec<T, G::W>;
  constexpr int W = G::W, NR = G::NRED;
  const int lane = threadIdx.x & 31, ry = threadIdx.x >> 5;
  const T half = (T)0.5;
  for (int k = blockIdx.x; k < nitems; k += gridDim.x) {
    int tile, pa, pb;
    item_of(k, ntiles, zc, gf.p_lo, gf.p_hi, tile, pa, pb);
    const int x0 = (tile % tiles_x) * G::TX, y0 = (tile / tiles_x) * TY;
    const int ox = x0 + W * lane, oy = y0 + ry;
    const bool rin = oy >= 1 && oy <= gf.ny - 1;
    bool in[W], any = false;
#pragma unroll
    for (int j = 0; j < W; j++) {
      in[j] = rin && ox + j >= 1 && ox + j <= gf.nx - 1;
      any = any || in[j];
    }
    if (!any) continue;
    const int X = ox >> 1, Y = oy >> 1, dy = oy & 1;
    const T* ec = e + (long long)Y * gc.pitch + X;
    auto Vz = [&](int Zg) -> Vt {  // x- then y-interpolated nodes of coarse plane Zg (global)
      const T* p0 = ec + (long long)(Zg - gc.p_glob0) * gc.pstride;
      T a[NR + 1];
#pragma unroll
      for (int i = 0; i <= NR; i++) a[i] = __ldg(p0 + i);
      Vt v;
#pragma unroll
      for (int i = 0; i < NR; i++) {
        v.v[2 * i] = a[i];
        v.v[2 * i + 1] = mul(half, add(a[i], a[i + 1]));
      }
      if (dy) {
#pragma unroll
        for (int i = 0; i <= NR; i++) a[i] = __ldg(p0 + gc.pitch + i);
#pragma unroll
        for (int i = 0; i < NR; i++) {
          v.v[2 * i] = mul(half, add(v.v[2 * i], a[i]));
          v.v[2 * i + 1] = mul(half, add(v.v[2 * i + 1], mul(half, add(a[i], a[i + 1]))));
        }
      }
      return v;
    };
    T* urow = u + (long long)oy * gf.pitch;
    int Z = (pa + gf.p_glob0) >> 1;
    Vt A = Vz(Z), B = A;
    bool haveB = false;
    bool all = true;
#pragma unroll
    for (int j = 0; j < W; j++) all = all && in[j];
    // KZ planes per iteration: their u vectors are loaded before any store (more bytes in
    // flight per thread; the compiler cannot reorder loads of u across stores to u)
    Vt uu[KZ], un[KZ];
    auto load_batch = [&](Vt* dst, int zb) {
      if (all) {
#pragma unroll
        for (int k = 0; k < KZ; k++)
          if (zb + k < pb) dst[k] = ld_vec(urow + (long long)(zb + k) * gf.pstride + ox);
      }
    };
    if (PIPE) load_batch(uu, pa);
    for (int z0 = pa; z0 < pb; z0 += KZ) {
      if (PIPE) {
        if (z0 + KZ < pb) load_batch(un, z0 + KZ);
      } else {
        load_batch(uu, z0);
      }
#pragma unroll
      for (int k = 0; k < KZ; k++) {
        const int z = z0 + k;
        if (z >= pb) break;
        const int zg = z + gf.p_glob0;
        if ((zg >> 1) != Z) {
          Z++;
          A = haveB ? B : Vz(Z);
          haveB = false;
        }
        Vt v = A;
        if (zg & 1) {
          if (!haveB) {
            B = Vz(Z + 1);
            haveB = true;
          }
#pragma unroll
          for (int j = 0; j < W; j++) v.v[j] = mul(half, add(A.v[j], B.v[j]));
        }
        T* up = urow + (long long)z * gf.pstride;
        if (all) {
          Vt o;
#pragma unroll
          for (int j = 0; j < W; j++) o.v[j] = add(uu[k].v[j], v.v[j]);
          store_vec(up, ox, in, o);
        } else {
#pragma unroll
          for (int j = 0; j < W; j++)
            if (in[j]) up[ox + j] = add(up[ox + j], v.v[j]);
        }
      }
      if (PIPE) {
#pragma unroll
        for (int k = 0; k < KZ; k++) uu[k] = un[k];
      }
    }
  }
}

// Flat variant: no z-marching.  Thread item = one 16-byte vector of W fine nodes of row y
// and the (up to) two fine planes 2Z, 2Z+1 of coarse plane Z; both u vectors are loaded
// before either is stored.  Memory-level parallelism from occupancy (256-thread CTAs,
// grid-stride) instead of per-thread z batches.  Same per-node arithmetic as k_prolong3d.
template <typename T, int MINB>
__global__ void __launch_bounds__(256, MINB)
    k_prolong3d_flat(Geom gf, Geom gc, const T* __restrict__ e, T* __restrict__ u, unsigned nvec, unsigned nrow,
                     unsigned nitems, int zg_lo, int zg_hi) {
  using G = Geo<T>;
  using Vt = Vec<T, G::W>;
  constexpr int W = G::W, NR = G::NRED;
  const T half = (T)0.5;
  for (unsigned it = blockIdx.x * 256u + threadIdx.x; it < nitems; it += gridDim.x * 256u) {
    const unsigned xv = it % nvec, t = it / nvec;
    const int oy = 1 + (int)(t % nrow), Z = (int)(t / nrow) + (zg_lo >> 1);
    const int ox = W * (int)xv;
    bool in[W], all = true;
#pragma unroll
    for (int j = 0; j < W; j++) {
      in[j] = ox + j >= 1 && ox + j <= gf.nx - 1;
      all = all && in[j];
    }
    const int X = ox >> 1, Y = oy >> 1, dy = oy & 1;
    const T* ec = e + (long long)Y * gc.pitch + X;
    auto Vz = [&](int Zg) -> Vt {
      const T* p0 = ec + (long long)(Zg - gc.p_glob0) * gc.pstride;
      T a[NR + 1];
#pragma unroll
      for (int i = 0; i <= NR; i++) a[i] = __ldg(p0 + i);
      Vt v;
#pragma unroll
      for (int i = 0; i < NR; i++) {
        v.v[2 * i] = a[i];
        v.v[2 * i + 1] = mul(half, add(a[i], a[i + 1]));
      }
      if (dy) {
#pragma unroll
        for (int i = 0; i <= NR; i++) a[i] = __ldg(p0 + gc.pitch + i);
#pragma unroll
        for (int i = 0; i < NR; i++) {
          v.v[2 * i] = mul(half, add(v.v[2 * i], a[i]));
          v.v[2 * i + 1] = mul(half, add(v.v[2 * i + 1], mul(half, add(a[i], a[i + 1]))));
        }
      }
      return v;
    };
    const int ze = 2 * Z, zo = 2 * Z + 1;  // global fine planes
    const bool he = ze >= zg_lo && ze < zg_hi, ho = zo >= zg_lo && zo < zg_hi;
    T* urow = u + (long long)oy * gf.pitch;
    T* pe = urow + (long long)(ze - gf.p_glob0) * gf.pstride;
    T* po = urow + (long long)(zo - gf.p_glob0) * gf.pstride;
    Vt ue, uo;
    if (all) {
      if (he) ue = ld_vec(pe + ox);
      if (ho) uo = ld_vec(po + ox);
    }
    const Vt A = Vz(Z);
    auto put = [&](T* p, const Vt& uv, const Vt& v) {
      if (all) {
        Vt o;
#pragma unroll
        for (int j = 0; j < W; j++) o.v[j] = add(uv.v[j], v.v[j]);
        store_vec(p, ox, in, o);
      } else {
#pragma unroll
        for (int j = 0; j < W; j++)
          if (in[j]) p[ox + j] = add(p[ox + j], v.v[j]);
      }
    };
    if (he) put(pe, ue, A);
    if (ho) {
      const Vt B = Vz(Z + 1);
      Vt v;
#pragma unroll
      for (int j = 0; j < W; j++) v.v[j] = mul(half, add(A.v[j], B.v[j]));
      put(po, uo, v);
    }
  }
}

template <typename T>
cudaError_t launch_prolong(const Geom& gf, const Geom& gc, const T* e, T* u, cudaStream_t st) {
  if (!gf.three_d) return pm2::launch_prolong<T>(gf, gc, e, u, u, st);
  using G = Geo<T>;
  const int tiles_x = (gf.nx + G::TX - 1) / G::TX, tiles_y = (gf.ny + TY - 1) / TY;
  const int ntiles = tiles_x * tiles_y;
  const int np = gf.p_hi - gf.p_lo;
  auto go = [&](auto kernel) {
    const int resident = resident_ctas((const void*)kernel, NT, 0);
    const int zc = choose_zc(ntiles, np, resident, 0, min_zc_for(gf, sizeof(T)));
    const int nitems = ntiles * ((np + zc - 1) / zc);
    kernel<<<nitems, NT, 0, st>>>(gf, gc, e, u, tiles_x, ntiles, zc, nitems);
    return cudaGetLastError();
  };
  auto go_flat = [&](auto kernel) {
    // rows 1 .. ny-1, vectors covering x = 0 .. nx, coarse planes of fine planes [p_lo, p_hi)
    const int zg_lo = gf.p_lo + gf.p_glob0, zg_hi = gf.p_hi + gf.p_glob0;
    const unsigned nvec = (unsigned)((gf.nx + G::W) / G::W), nrow = (unsigned)(gf.ny - 1);
    const unsigned nz = (unsigned)(((zg_hi - 1) >> 1) - (zg_lo >> 1) + 1);
    const unsigned long long n = (unsigned long long)nvec * nrow * nz;
    if (zg_hi <= zg_lo || nrow == 0) return cudaSuccess;
    if (n >= (1ull << 31)) return go(k_prolong3d<T, 4, 2, false>);
    int per_sm = 0, nsm = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0);
    const unsigned long long want = (n + 255) / 256, cap = (unsigned long long)nsm * (per_sm > 0 ? per_sm : 1) * 4;
    const int grid = (int)(want < cap ? want : cap);
    kernel<<<grid, 256, 0, st>>>(gf, gc, e, u, nvec, nrow, (unsigned)n, zg_lo, zg_hi);
    return cudaGetLastError();
  };
  // measured on C3 L0: flat<6> 0.411 ms FP64 / 0.225 ms FP32 beat the z-marching
  // variants (0.419-0.425 / 0.228-0.238) and other occupancies; the marching kernel is kept for
  // levels with >= 2^31 thread items
  return go_flat(k_prolong3d_flat<T, 6>);
}

template <typename T>
cudaError_t launch_resid_restrict(const Geom& gf, const Geom& gc, const Coef<T>& c, const T* u, const T* f, T* fc,
                                  cudaStream_t st) {
  if (!gf.three_d) return pm2::launch_resid_restrict<T>(gf, gc, c, u, f, fc, st);
  using G = Geo<T>;
  CUtensorMap tu, tf;
  if (encode(&tu, u, gf, sizeof(T), G::BYU) != CUDA_SUCCESS || encode(&tf, f, gf, sizeof(T), G::BYF) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const int tiles_x = (gc.nx + G::TX / 2 - 1) / (G::TX / 2), tiles_y = (gc.ny + TY / 2 - 1) / (TY / 2);
  const int ntiles = tiles_x * tiles_y;
  const int npc = gc.p_hi - gc.p_lo;
  auto kernel = k_resid_restrict3d_rows<T, RPT>;
  const int resident = prepare_kernel(kernel, G::SMEM, NTR);
  const int zcc = choose_zc(ntiles, npc, resident, 2, min_zc_for(gf, sizeof(T)));
  const int nitems = ntiles * ((npc + zcc - 1) / zcc);
  kernel<<<nitems, NTR, G::SMEM, st>>>(tu, tf, gf, gc, c, fc, tiles_x, ntiles, zcc, nitems);
  return cudaGetLastError();
}

template cudaError_t launch_sweep<double>(const Geom&, const Coef<double>&, bool, const double*, const double*,
                                          double*, bool, cudaStream_t, double*, int*, const double*,
                                          const Geom*, SweepNorm);
template cudaError_t launch_sweep<float>(const Geom&, const Coef<float>&, bool, const float*, const float*, float*,
                                         bool, cudaStream_t, double*, int*, const float*, const Geom*, SweepNorm);
template int sweep_partials<double>(const Geom&, bool);
template int sweep_partials<float>(const Geom&, bool);
template int sweep_items<double>(const Geom&, bool);
template int sweep_items<float>(const Geom&, bool);
template int norm_partials<double>(const Geom&);
template int norm_partials<float>(const Geom&);
template cudaError_t launch_norm<double>(const Geom&, const Coef<double>&, const double*, const double*, double*,
                                         int*, cudaStream_t);
template cudaError_t launch_norm<float>(const Geom&, const Coef<float>&, const float*, const float*, double*, int*,
                                        cudaStream_t);
template cudaError_t launch_prolong<double>(const Geom&, const Geom&, const double*, double*, cudaStream_t);
template cudaError_t launch_prolong<float>(const Geom&, const Geom&, const float*, float*, cudaStream_t);
template cudaError_t launch_resid_restrict<double>(const Geom&, const Geom&, const Coef<double>&, const double*,
                                                   const double*, double*, cudaStream_t);
template cudaError_t launch_resid_restrict<float>(const Geom&, const Geom&, const Coef<float>&, const float*,
                                                  const float*, float*, cudaStream_t);

}  // namespace pm
}  // namespace mg
