// loop_state.cuh — the device driver loop's state and its per-cycle check (loop.cu), shared
// with the whole-cycle tail kernel, which runs the check itself (kernels_tail.cu).
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace mg {

struct LoopState {
  double rtol;     // in: stopping tolerance (r_k <= rtol * r0)
  double r0;       // out: initial norm
  double* hist;    // in: device history buffer (max+1 doubles) or NULL
  int32_t max;     // in: max_cycles
  int32_t k;       // out: cycles run
  int32_t status;  // out: 0 ok, 1 r0 non-finite, 2 r_k non-finite
  int32_t pad;
};

// the initial norm: record r0; false: stop (non-finite r0, or max = 0).  One thread.
__device__ __forceinline__ bool loop_begin(double r0, LoopState* st) {
  const bool fin = isfinite(r0);
  st->r0 = r0;
  st->k = 0;
  st->status = fin ? 0 : 1;
  if (st->hist) st->hist[0] = r0;
  return fin && st->max > 0;
}

// after cycle k: record r_k; false: stop on a non-finite norm, k = max or r_k <= rtol r0
// (rtol < 0: no test).  One thread.
__device__ __forceinline__ bool loop_step(double rk, LoopState* st) {
  const int k = st->k + 1;
  const bool fin = isfinite(rk);
  st->k = k;
  if (st->hist) st->hist[k] = rk;
  if (!fin) st->status = 2;
  return !(!fin || k >= st->max || (st->rtol >= 0.0 && rk <= st->rtol * st->r0));
}

// the graph loop's check: the WHILE node's condition
__device__ __forceinline__ void loop_check(double rk, LoopState* st, cudaGraphConditionalHandle h) {
  cudaGraphSetConditional(h, loop_step(rk, st) ? 1u : 0u);
}

}  // namespace mg
