// loop.cu — the driver loop of the `Application` listing on the device.
//
//   r0 = ||f - A u||;  repeat { V-cycle; r_k = ||f - A u|| } until r_k <= rtol r0 or k = max
//
// is ONE CUDA graph: the initial norm, then a conditional WHILE node whose body is
// one cycle plus its norm and a one-thread check kernel that records r_k and sets
// the loop condition with cudaGraphSetConditional.  The host enqueues the graph
// once and synchronises once per solve instead of once per cycle (SURVEY §8(f)
// NEXT-1).  With the pipelined split (plan_can_split) the body is tail + head, the
// same kernels, in the same order, as the host loop in api.cu, so the iterates and
// norms are bitwise those of the host loop.
//
// NCCL calls cannot live inside a conditional body, so slab runs with nranks > 1
// keep the host loop (plan_loop_supported).
#include <cmath>
#include <cstdio>

#include "plan.h"

namespace mg {

__global__ void k_loop_init(const double* __restrict__ d_norm, LoopState* st, cudaGraphConditionalHandle h) {
  cudaGraphSetConditional(h, loop_begin(*d_norm, st) ? 1u : 0u);
}

__global__ void k_loop_check(const double* __restrict__ d_norm, LoopState* st, cudaGraphConditionalHandle h) {
  loop_check(*d_norm, st, h);
}

static mg_status cuda_fail(mg_solver* s, cudaError_t e, const char* what) {
  char buf[384];
  snprintf(buf, sizeof buf, "driver loop: %s: %s", what, cudaGetErrorString(e));
  return plan_fail(s, MG_ERR_CUDA, buf);
}

bool plan_loop_supported(mg_solver* s) { return !comm_active(s); }

// Capture: [head | norm] -> init -> WHILE { [tail + head | cycle + norm (part 5)] -> check }.
static mg_status build_loop_graph(mg_solver* s, void* u, const void* f, cudaGraphExec_t* out) {
  const bool split = plan_can_split(s);
  cudaStream_t cs = s->cap_stream;
  cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return cuda_fail(s, e, "cudaStreamBeginCapture");
  cudaGraph_t graph = nullptr;
  mg_status r = MG_OK;
  auto abort_capture = [&](mg_status st) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(cs, &g);
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    return st;
  };
  cudaStreamCaptureStatus cst;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  if ((e = cudaStreamGetCaptureInfo(cs, &cst, nullptr, &graph, nullptr, nullptr)) != cudaSuccess)
    return abort_capture(cuda_fail(s, e, "cudaStreamGetCaptureInfo"));
  cudaGraphConditionalHandle h;
  if ((e = cudaGraphConditionalHandleCreate(&h, graph, 0, 0)) != cudaSuccess)
    return abort_capture(cuda_fail(s, e, "cudaGraphConditionalHandleCreate"));
  // r0
  if ((r = plan_run_part(s, split ? 1 : 3, u, f, cs)) != MG_OK) return abort_capture(r);
  k_loop_init<<<1, 1, 0, cs>>>(s->d_norm, s->d_loop, h);
  if ((e = cudaGetLastError()) != cudaSuccess) return abort_capture(cuda_fail(s, e, "k_loop_init"));
  // WHILE node after everything captured so far
  if ((e = cudaStreamGetCaptureInfo(cs, &cst, nullptr, nullptr, &deps, &ndeps)) != cudaSuccess)
    return abort_capture(cuda_fail(s, e, "cudaStreamGetCaptureInfo"));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t wnode;
  if ((e = cudaGraphAddNode(&wnode, graph, deps, ndeps, &np)) != cudaSuccess)
    return abort_capture(cuda_fail(s, e, "cudaGraphAddNode(WHILE)"));
  if ((e = cudaStreamUpdateCaptureDependencies(cs, &wnode, 1, cudaStreamSetCaptureDependencies)) != cudaSuccess)
    return abort_capture(cuda_fail(s, e, "cudaStreamUpdateCaptureDependencies"));
  // body
  cudaGraph_t body = np.conditional.phGraph_out[0];
  cudaStream_t bs = s->cap_body;
  if ((e = cudaStreamBeginCaptureToGraph(bs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal)) !=
      cudaSuccess)
    return abort_capture(cuda_fail(s, e, "cudaStreamBeginCaptureToGraph"));
  // 4: no refresh; 5: the cycle and its norm
  mg_status rb = split ? plan_run_part(s, 2, u, f, bs) : plan_run_part(s, 5, u, f, bs);
  if (rb == MG_OK && split) rb = plan_run_part(s, 4, u, f, bs);
  if (rb == MG_OK) {
    k_loop_check<<<1, 1, 0, bs>>>(s->d_norm, s->d_loop, h);
    if ((e = cudaGetLastError()) != cudaSuccess) rb = cuda_fail(s, e, "k_loop_check");
  }
  cudaGraph_t bout = nullptr;
  e = cudaStreamEndCapture(bs, &bout);
  if (rb != MG_OK) return abort_capture(rb);
  if (e != cudaSuccess) return abort_capture(cuda_fail(s, e, "cudaStreamEndCapture(body)"));
  cudaGraph_t whole = nullptr;
  if ((e = cudaStreamEndCapture(cs, &whole)) != cudaSuccess) {
    cudaGetLastError();
    return cuda_fail(s, e, "cudaStreamEndCapture");
  }
  e = cudaGraphInstantiate(out, whole, 0);
  cudaGraphDestroy(whole);
  if (e != cudaSuccess) return cuda_fail(s, e, "cudaGraphInstantiate");
  return MG_OK;
}

mg_status plan_solve_device(mg_solver* s, void* u, const void* f, double rtol, int32_t max_cycles, int32_t* cycles,
                            double* history, cudaStream_t st, bool eager) {
  // a whole-cycle tail grid runs the loop inside one kernel (plan_solve_in_tail, part 6):
  // launched directly when eager, else as a one-launch graph; other grids: the WHILE graph
  const bool in_tail = plan_solve_in_tail(s);
  auto it = s->graphs.end();
  if (!in_tail) {
    auto key = std::make_tuple(u, f, 16);
    it = s->graphs.find(key);
    if (it == s->graphs.end()) {
      cudaGraphExec_t exec;
      mg_status r = build_loop_graph(s, u, f, &exec);
      if (r != MG_OK) return r;
      if (s->graphs.size() >= 16) {
        cudaGraphExecDestroy(s->graphs.begin()->second);
        s->graphs.erase(s->graphs.begin());
      }
      it = s->graphs.emplace(key, exec).first;
    }
  }
  if (history && (int64_t)max_cycles + 1 > s->hist_cap) {
    cudaFree(s->d_hist);
    s->d_hist = nullptr;
    s->hist_cap = 0;
    if (cudaMalloc(&s->d_hist, sizeof(double) * ((size_t)max_cycles + 1)) != cudaSuccess) {
      cudaGetLastError();
      return plan_fail(s, MG_ERR_OOM, "allocation of the residual history failed");
    }
    s->hist_cap = (int64_t)max_cycles + 1;
  }
  LoopState* hl = s->h_loop;
  hl->rtol = rtol;
  hl->r0 = 0.0;
  hl->hist = history ? s->d_hist : nullptr;
  hl->max = max_cycles;
  hl->k = 0;
  hl->status = 0;
  cudaError_t e = cudaMemcpyAsync(s->d_loop, hl, sizeof(LoopState), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(s, e, "solve");
  if (in_tail) {
    const mg_status r = eager ? plan_run_part(s, 6, u, f, st) : plan_graph_part(s, 6, u, f, st);
    if (r != MG_OK) return r;
  } else {
    e = cudaGraphLaunch(it->second, st);
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(hl, s->d_loop, sizeof(LoopState), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(s, e, "solve");
  const int k = hl->k;
  if (history) {
    e = cudaMemcpy(history, s->d_hist, sizeof(double) * ((size_t)k + 1), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(s, e, "history readback");
  }
  if (hl->status == 1) return plan_fail(s, MG_ERR_NONFINITE, "initial residual norm is not finite");
  if (cycles) *cycles = k;
  if (hl->status == 2) {
    char buf[128];
    snprintf(buf, sizeof buf, "residual norm not finite after cycle %d (S:535)", k);
    return plan_fail(s, MG_ERR_NONFINITE, buf);
  }
  return MG_OK;
}

}  // namespace mg
