// kernels_tail.h — single-CTA coarse tail of the V-cycle (kernels_tail.cu).
#pragma once
#include "mg_common.cuh"
#include "loop_state.cuh"

namespace mg {

constexpr int kTailMax = 12;  // levels handled by one tail launch
constexpr int kTailCluster = 16;  // CTAs of the largest tail cluster
constexpr int kTailDistMax = 4;   // dist levels at most
constexpr int kTailSmemMax = 200 * 1024;  // CTA 0's shared memory for the solo levels' arrays
constexpr int kTailSmemCap = 222 * 1024;  // all dynamic shared memory (+ the coarse factor; 5 KB static below 227 KB)

template <typename T>
struct TailParams {
  int nl;          // tail levels (index 0 = the top tail level lt)
  int rbgs;        // smoother: 1 red-black GS, 0 Jacobi, 2 lexicographic GS
  int nu1, nu2;
  int sweeps;      // coarsest: 1 = ncoarse sweeps, 0 = direct
  int ncoarse;
  int zero_first;  // the top tail level starts from a zero guess (always, unless it is level 0)
  int solo_from;   // levels >= solo_from run on CTA 0 alone (set by launch_tail)
  int smem_from;   // levels >= smem_from (all solo) keep u, t, f, r in CTA 0's shared memory (launch_tail)
  int smem_bytes;  // their dynamic shared memory
  int smem_total;  // all dynamic shared memory (levels, coarse factor and vector)
  int soff[kTailMax];   // byte offset of level k's four arrays
  Geom gs[kTailMax];    // level k's compact shared-memory layout (pitch nx+1, no padding)
  int csize;       // CTAs (one cluster; set by tail_prepare)
  // dist levels: the leading dist_n cluster levels are split into slabs of planes,
  // CTA r holding planes [zr[k][r], zr[k][r+1]) plus a halo plane each side in its own shared
  // memory at doff[k] (arrays u, f, r[, t] of dn16[k] elements, compact layout gd[k] whose
  // `planes` is the largest window); zr is also set for level dist_n (the restriction into it)
  int dist_n;
  int zr[kTailMax][kTailCluster + 1];
  int doff[kTailMax];
  int dn16[kTailMax];
  Geom gd[kTailMax];
  int m;           // coarsest unknowns (direct)
  double D_coarse;
  double rD_coarse;  // RN(1 / D_coarse) (m = 1)
  const double* chol;
  double* work;
  int chol_off;    // direct solve: byte offset of the staged factor in shared memory, -1: read global
  int y_off;       // ... and of its right-hand side / solution vector (m doubles) + 1 / L_ii (m)
  // the residual norm ||f - A u|| of the top tail level when it is level 0:
  // norm_only = 1 evaluates it for (u[0], f[0]) without a cycle; otherwise, with norm_out set,
  // of the cycle's result.  Both run the same distribution and reduction order, so the
  // solve's history is bitwise that of mg_residual_norm.
  int norm_only;
  double* norm_out;
  double* nscratch;  // csize doubles (per-CTA sums)
  LoopState* solve;  // lt = 0: the whole driver loop in this launch (r0, cycles, norms, stop test)
  Geom g[kTailMax];
  Coef<T> c[kTailMax];
  T* u[kTailMax];
  T* t[kTailMax];
  T* r[kTailMax];
  T* f[kTailMax];
};

// work distribution and shared-memory layout (solo_from, smem_from, soff, gs, smem_bytes,
// csize, chol_off, y_off) from the levels: call once before launch_tail
template <typename T>
void tail_prepare(TailParams<T>& p);
template <typename T>
cudaError_t launch_tail(const TailParams<T>& p, cudaStream_t st);

}  // namespace mg
