// kernels_pm.cu — 2.5D plane-marching level operators for 3D levels (sm_100a).
//
// Each CTA owns a TX x TY tile of an (x,y) plane and marches a chunk of planes
// along z.  u and f planes (tile + a 2-node ring) are staged in shared memory
// by TMA (cp.async.bulk.tensor.3d) into an NS-deep ring of slots signalled by
// mbarriers, so every HBM byte is read once per sweep and the ring re-reads of
// neighbouring tiles hit L2.  Arithmetic is the canonical per-point order of
// mg_common.cuh (no FMA), so results are bitwise identical to the op-by-op
// kernels and to the oracle.
//
//  k_sweep3d<RB=true>   one red-black Gauss-Seidel sweep in ONE pass:
//                       ping-pong u_old -> u_new.  For output plane b the red
//                       ("post-red", PR) values of planes b-1..b+1 are computed
//                       on the tile + 1-node ring from u_old (a 3-plane smem
//                       ring), then black nodes of plane b are updated from PR.
//                       No CTA reads what another CTA writes: race free.
//                       HBM: read u_old, f; write u_new = 3 words per node.
//  k_sweep3d<RB=false>  one omega-Jacobi sweep (reading 9), 3 words/node.
//  k_resid_restrict3d   r = f - A u (Alg. 1 line 4) on the fine tile + ring,
//                       kept in a 3-plane smem ring, and full weighting
//                        of every completed coarse plane; r never
//                       touches HBM: read u, f; write f_H = 2 + 1/8 words.
#include <cuda.h>

#include "kernels_pm.h"
#include "tma.cuh"

namespace mg {
namespace pm {

constexpr int TX = 64, TY = 8;      // output tile (fine nodes) per CTA and plane
constexpr int NT = (TX / 2) * TY;   // 256 threads: one x-pair each
// TMA box: tile + 2-node ring in y and >= 2 in x.  Measured on B200 (sm_100a,
// driver 580): a tiled TMA load whose x start is not a multiple of 16 BYTES
// raises "illegal instruction", so the box starts HX = 16/sizeof(T) nodes left
// of the tile (2 in FP64, 4 in FP32) and is 2*HX wider than the tile.
template <typename T>
struct Box {
  static constexpr int HX = 16 / (int)sizeof(T);
  static constexpr int BX = TX + 2 * HX;
};
constexpr int BYU = TY + 4;
constexpr int PX = TX + 2, PY = TY + 2;    // PR / r planes: tile + 1-node ring

__host__ __device__ constexpr int rup(int a, int b) { return (a + b - 1) / b * b; }

template <typename T>
struct Lay {
  static constexpr int BXU = Box<T>::BX;
  static constexpr int HX = Box<T>::HX;
  static constexpr int UB = rup(BYU * BXU * (int)sizeof(T), 128);  // bytes per box slot
  static constexpr int PB = rup(PY * PX * (int)sizeof(T), 128);    // bytes per PR plane
  static constexpr int smem(int ns) { return 2 * ns * UB + 3 * PB + ns * 8; }      // resid-restrict
  static constexpr int smem_sweep(int ns) { return 2 * ns * UB + 2 * PB + ns * 8; }
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

// ---------------------------------------------------------------------------
// Thread t owns the x-pair (ox, ox+1) = (x0 + 2*(t%32), y0 + t/32) of the tile:
// in every plane one node of the pair is red, the other black.  The pair's u
// values of planes p-1, p, p+1 and its red (post-red) values of the last two
// planes live in registers; only in-plane neighbours come from shared memory.
// 144 "ring" threads additionally compute the red nodes on the 1-node ring
// around the tile that the tile's black nodes read.
template <typename T>
struct Pair {
  T x, y;
};

template <typename T>
__device__ __forceinline__ Pair<T> ld_pair(const T* p) {
  typename V2<T>::t v = *reinterpret_cast<const typename V2<T>::t*>(p);
  return Pair<T>{v.x, v.y};
}

// canonical update u + wd*(f - (D*u - [cx*(l+r) + cy*(d+u) + cz*(m+p)]))
template <typename T>
__device__ __forceinline__ T relax(const Coef<T>& c, T ctr, T l, T r, T d, T u, T m, T p, T f) {
  T s = mul(c.cx, add(l, r));
  s = add(s, mul(c.cy, add(d, u)));
  s = add(s, mul(c.cz, add(m, p)));
  T Au = sub(mul(c.D, ctr), s);
  return add(ctr, mul(c.wd, sub(f, Au)));
}

// A u at a node (canonical order); the residual is f - Au
template <typename T>
__device__ __forceinline__ T relax_au(const Coef<T>& c, T ctr, T l, T r, T d, T u, T m, T p) {
  T s = mul(c.cx, add(l, r));
  s = add(s, mul(c.cy, add(d, u)));
  s = add(s, mul(c.cz, add(m, p)));
  return sub(mul(c.D, ctr), s);
}

template <typename T, bool RB, int NS>
__global__ void __launch_bounds__(NT, 3)
    k_sweep3d(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_f, Geom g,
              Coef<T> c, T* __restrict__ unew, int zc, int tiles_x, int tiles_y, int zero_in) {
  extern __shared__ __align__(128) unsigned char sm[];
  using L = Lay<T>;
  constexpr int BXU = L::BXU, HX = L::HX;
  T* su = reinterpret_cast<T*>(sm);
  T* sf = reinterpret_cast<T*>(sm + NS * L::UB);
  T* spr = reinterpret_cast<T*>(sm + 2 * NS * L::UB);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + 2 * NS * L::UB + 2 * L::PB);
  auto slot = [](int q) { return ((q % NS) + NS) % NS; };
  auto U = [&](int q) { return su + (size_t)slot(q) * (L::UB / sizeof(T)); };
  auto F = [&](int q) { return sf + (size_t)slot(q) * (L::UB / sizeof(T)); };
  auto PRb = [&](int q) { return spr + (size_t)(q & 1) * (L::PB / sizeof(T)); };

  const int tid = threadIdx.x;
  int b = blockIdx.x;
  const int tix = b % tiles_x;
  b /= tiles_x;
  const int tiy = b % tiles_y;
  b /= tiles_y;
  const int x0 = tix * TX, y0 = tiy * TY;
  const int pz0 = g.p_lo + b * zc;
  const int pz1 = min(pz0 + zc, g.p_hi);
  const int qlo = pz0 - (RB ? 2 : 1);
  const int qlast = RB ? pz1 + 1 : pz1;
  const uint32_t boxb = (uint32_t)(BYU * BXU * sizeof(T));
  const uint32_t tx_bytes = (zero_in ? 0u : boxb) + boxb;

  if (tid == 0) {
    prefetch_tmap(&tm_u);
    prefetch_tmap(&tm_f);
    for (int s2 = 0; s2 < NS; s2++) mbar_init(&full[s2], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int q) {  // thread 0 only
    uint64_t* bar = &full[slot(q)];
    mbar_expect_tx(bar, tx_bytes);
    if (!zero_in) tma_load_3d(U(q), &tm_u, x0 - HX, y0 - 2, q, bar);
    tma_load_3d(F(q), &tm_f, x0 - HX, y0 - 2, q, bar);
  };
  if (tid == 0)
    for (int q = qlo; q < qlo + NS && q <= qlast; q++) issue(q);
  auto wait = [&](int q) { mbar_wait(&full[slot(q)], (uint32_t)(((q - qlo) / NS) & 1)); };

  const int pg0 = g.p_glob0;
  const int px = tid & 31, ry = tid >> 5;
  const int ox = x0 + 2 * px, oy = y0 + ry;
  const int bo = (ry + 2) * BXU + 2 * px + HX;  // box offset of (ox, oy)
  const int po = (ry + 1) * PX + 2 * px + 1;     // PR offset of (ox, oy)
  const bool rin = oy >= 1 && oy <= g.ny - 1;
  const bool in0 = rin && ox >= 1 && ox <= g.nx - 1;
  const bool in1 = rin && ox + 1 <= g.nx - 1;
  T* orow = unew + (long long)oy * g.pitch;
  const Pair<T> zero2{(T)0, (T)0};
  auto ldu = [&](const T* base) -> Pair<T> { return zero_in ? zero2 : ld_pair(base + bo); };
  auto sldu = [&](const T* base, int off) -> T { return zero_in ? (T)0 : base[off]; };

  if (RB) {
    // ring position of threads 0..143: top row, bottom row, left column, right column
    int rxr = 0, ryr = 0;
    if (tid < 64) { rxr = x0 + tid; ryr = y0 - 1; }
    else if (tid < 128) { rxr = x0 + tid - 64; ryr = y0 + TY; }
    else if (tid < 136) { rxr = x0 - 1; ryr = y0 + tid - 128; }
    else if (tid < 144) { rxr = x0 + TX; ryr = y0 + tid - 136; }
    const bool has_ring = tid < 144;
    const bool ring_in = has_ring && rxr >= 1 && rxr <= g.nx - 1 && ryr >= 1 && ryr <= g.ny - 1;
    const int rbo = (ryr - y0 + 2) * BXU + (rxr - x0 + HX);
    const int rpo = (ryr - y0 + 1) * PX + (rxr - x0 + 1);

    wait(qlo);
    wait(qlo + 1);
    Pair<T> um = ldu(U(qlo)), u0 = ldu(U(qlo + 1)), up;
    T pr1 = (T)0, pr2 = (T)0;  // own red value of planes p-1 and p-2
    for (int p = pz0 - 1; p <= pz1; p++) {
      wait(p + 1);
      const T* U0 = U(p);
      up = ldu(U(p + 1));
      const int pgl = p + pg0;
      const bool pl_in = pgl >= 1 && pgl <= g.nz - 1;
      const int kr = (oy + pgl) & 1;  // red node of the pair: ox + kr
      // ---- red node of plane p (post-red value)
      T pr0;
      {
        const T ctr = kr ? u0.y : u0.x;
        pr0 = ctr;
        if (pl_in && (kr ? in1 : in0)) {
          const T l = kr ? u0.x : sldu(U0, bo - 1);
          const T r = kr ? sldu(U0, bo + 2) : u0.y;
          pr0 = relax(c, ctr, l, r, sldu(U0, bo + kr - BXU), sldu(U0, bo + kr + BXU), kr ? um.y : um.x,
                      kr ? up.y : up.x, F(p)[bo + kr]);
        }
        PRb(p)[po + kr] = pr0;
      }
      if (has_ring && ((rxr + ryr + pgl) & 1) == 0) {  // red ring node
        const T* Um = U(p - 1);
        const T* Up = U(p + 1);
        T v = sldu(U0, rbo);
        if (pl_in && ring_in)
          v = relax(c, v, sldu(U0, rbo - 1), sldu(U0, rbo + 1), sldu(U0, rbo - BXU), sldu(U0, rbo + BXU),
                    sldu(Um, rbo), sldu(Up, rbo), F(p)[rbo]);
        PRb(p)[rpo] = v;
      }
      __syncthreads();
      // ---- black node of plane bp = p-1 (its red neighbours are final)
      const int bp = p - 1;
      if (bp >= pz0) {
        const int kb = kr;  // black node of plane p-1 sits where plane p's red node is
        const T* P = PRb(bp);
        const T ctr = kb ? um.y : um.x;
        T v = ctr;
        if (kb ? in1 : in0) {
          const T l = kb ? pr1 : P[po - 1];
          const T r = kb ? P[po + 2] : pr1;
          v = relax(c, ctr, l, r, P[po + kb - PX], P[po + kb + PX], pr2, pr0, F(bp)[bo + kb]);
        }
        const T o0 = kb ? pr1 : v, o1 = kb ? v : pr1;
        store_pair(orow + (long long)bp * g.pstride, ox, in0, in1, o0, o1);
      }
      __syncthreads();
      if (tid == 0) {
        const int q = p - 1 + NS;  // plane p-1 is no longer needed
        if (q <= qlast) {
          fence_proxy_async();
          issue(q);
        }
      }
      um = u0;
      u0 = up;
      pr2 = pr1;
      pr1 = pr0;
    }
  } else {
    wait(qlo);
    wait(qlo + 1);
    Pair<T> um = ldu(U(qlo)), u0 = ldu(U(qlo + 1)), up;
    for (int p = pz0; p < pz1; p++) {
      wait(p + 1);
      const T* U0 = U(p);
      up = ldu(U(p + 1));
      const Pair<T> fp = ld_pair(F(p) + bo);
      T o0 = u0.x, o1 = u0.y;
      if (in0)
        o0 = relax(c, u0.x, sldu(U0, bo - 1), u0.y, sldu(U0, bo - BXU), sldu(U0, bo + BXU), um.x, up.x, fp.x);
      if (in1)
        o1 = relax(c, u0.y, u0.x, sldu(U0, bo + 2), sldu(U0, bo + 1 - BXU), sldu(U0, bo + 1 + BXU), um.y, up.y,
                   fp.y);
      store_pair(orow + (long long)p * g.pstride, ox, in0, in1, o0, o1);
      __syncthreads();
      if (tid == 0) {
        const int q = p - 1 + NS;
        if (q <= qlast) {
          fence_proxy_async();
          issue(q);
        }
      }
      um = u0;
      u0 = up;
    }
  }
}

// ---------------------------------------------------------------------------
// Fused residual + full-weighting restriction.  Fine tile = 2x the coarse tile
// (TX x TY fine nodes, x0 = 2 X0).  Per fine plane q: every thread computes r
// for its x-pair (u column in registers), 73 ring threads the low-side ring
// (row y0-1, column x0-1) that the tile's coarse nodes also need; then the
// 128 coarse nodes of the tile form their x- and y-sums of plane q (reading r
// from smem) and keep the last three in registers: when q = 2P+1 the z-sum
// gives f_H(P).  Canonical order (reading 13): x, then y, then z.
template <typename T, int NS>
__global__ void __launch_bounds__(NT, 3)
    k_resid_restrict3d(const __grid_constant__ CUtensorMap tm_u, const __grid_constant__ CUtensorMap tm_f,
                       Geom gf, Geom gc, Coef<T> c, T* __restrict__ fc, int zcc, int tiles_x, int tiles_y) {
  extern __shared__ __align__(128) unsigned char sm[];
  using L = Lay<T>;
  constexpr int BXU = L::BXU, HX = L::HX;
  T* su = reinterpret_cast<T*>(sm);
  T* sf = reinterpret_cast<T*>(sm + NS * L::UB);
  T* R = reinterpret_cast<T*>(sm + 2 * NS * L::UB);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + 2 * NS * L::UB + 2 * L::PB);
  auto slot = [](int q) { return ((q % NS) + NS) % NS; };
  auto U = [&](int q) { return su + (size_t)slot(q) * (L::UB / sizeof(T)); };
  auto F = [&](int q) { return sf + (size_t)slot(q) * (L::UB / sizeof(T)); };

  const int tid = threadIdx.x;
  int b = blockIdx.x;
  const int tix = b % tiles_x;
  b /= tiles_x;
  const int tiy = b % tiles_y;
  b /= tiles_y;
  const int X0 = tix * (TX / 2), Y0 = tiy * (TY / 2);
  const int x0 = 2 * X0, y0 = 2 * Y0;
  const int P0c = gc.p_lo + b * zcc;  // coarse output planes [P0c, P1c)
  const int P1c = min(P0c + zcc, gc.p_hi);
  const int qf0 = 2 * (P0c + gc.p_glob0) - gf.p_glob0;      // fine centre of the first coarse plane
  const int qf1 = 2 * (P1c - 1 + gc.p_glob0) - gf.p_glob0;  // ... of the last
  const int rlo = qf0 - 1, rhi = qf1 + 1;                    // r planes needed
  const int qlo = rlo - 1, qlast = rhi + 1;                  // u/f planes loaded
  const uint32_t tx_bytes = 2u * (uint32_t)(BYU * BXU * sizeof(T));

  if (tid == 0) {
    prefetch_tmap(&tm_u);
    prefetch_tmap(&tm_f);
    for (int s2 = 0; s2 < NS; s2++) mbar_init(&full[s2], 1);
    fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int q) {
    uint64_t* bar = &full[slot(q)];
    mbar_expect_tx(bar, tx_bytes);
    tma_load_3d(U(q), &tm_u, x0 - HX, y0 - 2, q, bar);
    tma_load_3d(F(q), &tm_f, x0 - HX, y0 - 2, q, bar);
  };
  if (tid == 0)
    for (int q = qlo; q < qlo + NS && q <= qlast; q++) issue(q);
  auto wait = [&](int q) { mbar_wait(&full[slot(q)], (uint32_t)(((q - qlo) / NS) & 1)); };

  const int pgf0 = gf.p_glob0;
  const int px = tid & 31, ry = tid >> 5;
  const int ox = x0 + 2 * px, oy = y0 + ry;
  const int bo = (ry + 2) * BXU + 2 * px + HX;
  const int po = (ry + 1) * PX + 2 * px + 1;
  const bool rin = oy >= 1 && oy <= gf.ny - 1;
  const bool in0 = rin && ox >= 1 && ox <= gf.nx - 1;
  const bool in1 = rin && ox + 1 <= gf.nx - 1;
  // low-side ring: row y0-1 for x in [x0-1, x0+TX-1] (65), column x0-1 for y in [y0, y0+TY-1] (8)
  int rxr = 0, ryr = 0;
  if (tid < TX + 1) { rxr = x0 - 1 + tid; ryr = y0 - 1; }
  else if (tid < TX + 1 + TY) { rxr = x0 - 1; ryr = y0 + tid - (TX + 1); }
  const bool has_ring = tid < TX + 1 + TY;
  const bool ring_in = has_ring && rxr >= 1 && rxr <= gf.nx - 1 && ryr >= 1 && ryr <= gf.ny - 1;
  const int rbo = (ryr - y0 + 2) * BXU + (rxr - x0 + HX);
  const int rpo = (ryr - y0 + 1) * PX + (rxr - x0 + 1);
  // coarse node of threads 0..127
  const int ccx = tid % (TX / 2), ccy = tid / (TX / 2);
  const int I = X0 + ccx, J = Y0 + ccy;
  const bool cnode = tid < (TX / 2) * (TY / 2) && I >= 1 && I <= gc.nx - 1 && J >= 1 && J <= gc.ny - 1;
  const int co = (2 * ccy + 1) * PX + 2 * ccx + 1;  // r offset of fine (2I, 2J)
  T* crow = fc + (long long)J * gc.pitch + I;
  const T two = (T)2;
  const T scale = (T)(1.0 / 64.0);

  wait(qlo);
  wait(qlo + 1);
  Pair<T> um = ld_pair(U(qlo) + bo), u0 = ld_pair(U(qlo + 1) + bo), up;
  T ty1 = (T)0, ty2 = (T)0;
  for (int q = rlo; q <= rhi; q++) {
    wait(q + 1);
    const T* U0 = U(q);
    const T* F0 = F(q);
    up = ld_pair(U(q + 1) + bo);
    const int pgl = q + pgf0;
    const bool pl_in = pgl >= 1 && pgl <= gf.nz - 1;
    {
      const Pair<T> fp = ld_pair(F0 + bo);
      T r0 = (T)0, r1 = (T)0;
      if (pl_in && in0) r0 = sub(fp.x, relax_au(c, u0.x, U0[bo - 1], u0.y, U0[bo - BXU], U0[bo + BXU], um.x, up.x));
      if (pl_in && in1)
        r1 = sub(fp.y, relax_au(c, u0.y, u0.x, U0[bo + 2], U0[bo + 1 - BXU], U0[bo + 1 + BXU], um.y, up.y));
      R[po] = r0;
      R[po + 1] = r1;
    }
    if (has_ring) {
      T r = (T)0;
      if (pl_in && ring_in)
        r = sub(F0[rbo], relax_au(c, U0[rbo], U0[rbo - 1], U0[rbo + 1], U0[rbo - BXU], U0[rbo + BXU],
                                  U(q - 1)[rbo], U(q + 1)[rbo]));
      R[rpo] = r;
    }
    __syncthreads();
    if (cnode) {
      T tx[3];
#pragma unroll
      for (int dy = -1; dy <= 1; dy++) {
        const T* row = R + co + dy * PX;
        tx[dy + 1] = add(add(row[-1], row[1]), mul(two, row[0]));
      }
      const T ty0 = add(add(tx[0], tx[2]), mul(two, tx[1]));
      if ((pgl & 1) == 1 && q >= qf0 + 1) {  // fine plane 2P+1 completes coarse plane P
        const int Pc = ((pgl - 1) >> 1) - gc.p_glob0;
        const T t = add(add(ty2, ty0), mul(two, ty1));
        crow[(long long)Pc * gc.pstride] = mul(t, scale);
      }
      ty2 = ty1;
      ty1 = ty0;
    }
    __syncthreads();
    if (tid == 0) {
      const int qq = q - 1 + NS;
      if (qq <= qlast) {
        fence_proxy_async();
        issue(qq);
      }
    }
    um = u0;
    u0 = up;
  }
}

// ---------------------------------------------------------------------------
static CUresult encode(CUtensorMap* tm, const void* base, const Geom& g, int esz) {
  cuuint64_t dims[3] = {(cuuint64_t)(g.nx + 1), (cuuint64_t)g.rows, (cuuint64_t)(g.p_hi + 1)};
  cuuint64_t strides[2] = {(cuuint64_t)(g.pitch * esz), (cuuint64_t)(g.pstride * esz)};
  cuuint32_t box[3] = {(cuuint32_t)(TX + 2 * (16 / esz)), BYU, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return cuTensorMapEncodeTiled(tm, esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                                const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

// slots per CTA: FP64 4 (3 CTAs/SM), FP32 6 (4 CTAs/SM)
template <typename T>
constexpr int ns_sweep() { return sizeof(T) == 8 ? 4 : 6; }


bool supported(const Geom& g) { return g.three_d && g.nx >= 16 && g.ny >= 16 && (g.p_hi - g.p_lo) >= 4; }

template <typename T>
cudaError_t launch_sweep(const Geom& g, const Coef<T>& c, bool rbgs, const T* uin, const T* f, T* uout, bool zero_in,
                         int zc, cudaStream_t st) {
  CUtensorMap tu, tf;
  if (encode(&tu, uin ? uin : f, g, sizeof(T)) != CUDA_SUCCESS || encode(&tf, f, g, sizeof(T)) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const int tiles_x = (g.nx + TX - 1) / TX, tiles_y = (g.ny + TY - 1) / TY;
  const int nplanes = g.p_hi - g.p_lo;
  const int chunks = (nplanes + zc - 1) / zc;
  constexpr int NS = ns_sweep<T>();
  const int smem = Lay<T>::smem_sweep(NS);
  dim3 grid((unsigned)(tiles_x * tiles_y * chunks));
  if (rbgs) {
    auto k = k_sweep3d<T, true, NS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<grid, NT, smem, st>>>(tu, tf, g, c, uout, zc, tiles_x, tiles_y, zero_in ? 1 : 0);
  } else {
    auto k = k_sweep3d<T, false, NS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<grid, NT, smem, st>>>(tu, tf, g, c, uout, zc, tiles_x, tiles_y, zero_in ? 1 : 0);
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_resid_restrict(const Geom& gf, const Geom& gc, const Coef<T>& c, const T* u, const T* f, T* fc,
                                  int zcc, cudaStream_t st) {
  CUtensorMap tu, tf;
  if (encode(&tu, u, gf, sizeof(T)) != CUDA_SUCCESS || encode(&tf, f, gf, sizeof(T)) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  const int tiles_x = (gc.nx + TX / 2 - 1) / (TX / 2), tiles_y = (gc.ny + TY / 2 - 1) / (TY / 2);
  const int nplanes = gc.p_hi - gc.p_lo;
  const int chunks = (nplanes + zcc - 1) / zcc;
  constexpr int NS = ns_sweep<T>();
  const int smem = Lay<T>::smem_sweep(NS);
  auto k = k_resid_restrict3d<T, NS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<dim3((unsigned)(tiles_x * tiles_y * chunks)), NT, smem, st>>>(tu, tf, gf, gc, c, fc, zcc, tiles_x, tiles_y);
  return cudaGetLastError();
}

template cudaError_t launch_sweep<double>(const Geom&, const Coef<double>&, bool, const double*, const double*,
                                          double*, bool, int, cudaStream_t);
template cudaError_t launch_sweep<float>(const Geom&, const Coef<float>&, bool, const float*, const float*, float*,
                                         bool, int, cudaStream_t);
template cudaError_t launch_resid_restrict<double>(const Geom&, const Geom&, const Coef<double>&, const double*,
                                                   const double*, double*, int, cudaStream_t);
template cudaError_t launch_resid_restrict<float>(const Geom&, const Geom&, const Coef<float>&, const float*,
                                                  const float*, float*, int, cudaStream_t);

}  // namespace pm
}  // namespace mg
