// kernels_tail.h — single-CTA coarse tail of the V-cycle (kernels_tail.cu).
#pragma once
#include "mg_common.cuh"

namespace mg {

constexpr int kTailMax = 12;  // levels handled by one tail launch
constexpr int kTailSmemMax = 200 * 1024;  // CTA 0's shared memory for the solo levels' arrays

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
  int soff[kTailMax];   // byte offset of level k's four arrays
  Geom gs[kTailMax];    // level k's compact shared-memory layout (pitch nx+1, no padding)
  int m;           // coarsest unknowns (direct)
  double D_coarse;
  const double* chol;
  double* work;
  Geom g[kTailMax];
  Coef<T> c[kTailMax];
  T* u[kTailMax];
  T* t[kTailMax];
  T* r[kTailMax];
  T* f[kTailMax];
};

template <typename T>
cudaError_t launch_tail(const TailParams<T>& p, cudaStream_t st);

}  // namespace mg
