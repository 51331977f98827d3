// api.cu — the C ABI (include/mg.h): validation, level hierarchy, buffers,
// the V-cycle schedule of Alg. 1, CUDA-graph capture/replay and
// per-kernel event timing.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <initializer_list>
#include <map>
#include <string>
#include <vector>

#include <nccl.h>

#include "mg.h"
#include "partition.h"
#include "plan.h"
#include "comm.h"

using namespace mg;

static thread_local std::string g_last_error;

static mg_status fail(mg_solver* s, mg_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  if (s) {
    s->err = buf;
    if (st == MG_ERR_CUDA || st == MG_ERR_NCCL) s->poisoned = true;
  }
  return st;
}

#define CK(call)                                                                                 \
  do {                                                                                           \
    cudaError_t e_ = (call);                                                                     \
    if (e_ != cudaSuccess)                                                                       \
      return fail(s, MG_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
  } while (0)

extern "C" void mg_config_default(mg_config* c, int32_t dim, int64_t nodes) {
  memset(c, 0, sizeof *c);
  c->dim = dim;
  for (int d = 0; d < 3; d++) {
    c->nodes[d] = d < dim ? nodes : 1;
    c->coeff[d] = 1.0;
    c->h[d] = 0.0;
  }
  c->levels = 0;
  c->smoother = MG_RBGS;
  c->omega = 1.0;
  c->nu1 = 2;
  c->nu2 = 2;
  c->coarse = MG_COARSE_DIRECT;
  c->ncoarse = 10;
  c->dtype = MG_FP64;
  c->device = 0;
  c->rank = 0;
  c->nranks = 1;
  c->nccl_id = nullptr;
  c->flags = 0;
  c->problem = MG_PROBLEM_POISSON;
  c->tau = 0.1;  // complex diffusion defaults (the paper gives none)
  c->theta = M_PI / 30.0;
  c->kappa = 2.0;
}

// complex diffusion (cell-centred FAS): nodes[d] are cells; coarsest level has 2 cells
// along the shortest axis (< 3 unknowns per direction)
static mg_status validate_cd(const mg_config* c, int* levels_out) {
  mg_solver* s = nullptr;
  if (c->smoother != MG_JACOBI && c->smoother != MG_RBGS) return fail(s, MG_ERR_INVALID, "bad smoother");
  if (!(c->omega > 0.0 && c->omega < 2.0)) return fail(s, MG_ERR_INVALID, "omega must be in (0,2) (S:46)");
  if (c->nu1 < 0 || c->nu2 < 0) return fail(s, MG_ERR_INVALID, "nu1, nu2 must be >= 0");
  if (c->coarse != MG_COARSE_SWEEPS || c->ncoarse < 1)
    return fail(s, MG_ERR_INVALID, "complex diffusion needs coarse = MG_COARSE_SWEEPS, ncoarse >= 1 (FAS, S:437)");
  if (c->dtype != MG_FP64 && c->dtype != MG_FP32) return fail(s, MG_ERR_INVALID, "bad dtype");
  if (c->nranks != 1) return fail(s, MG_ERR_INVALID, "complex diffusion runs on one rank (nranks = 1)");
  if (c->flags & (MG_FLAG_SLAB | MG_FLAG_SEPARATE_PROLONG))
    return fail(s, MG_ERR_INVALID, "MG_FLAG_SLAB / MG_FLAG_SEPARATE_PROLONG do not apply to complex diffusion");
  if (!(c->tau > 0.0) || !(c->theta > 0.0 && c->theta < M_PI / 2) || !(c->kappa > 0.0))
    return fail(s, MG_ERR_INVALID, "need tau > 0, theta in (0, pi/2), kappa > 0 (S:303)");
  int64_t mincells = INT64_MAX;
  for (int d = 0; d < c->dim; d++) {
    const int64_t n = c->nodes[d];
    if (n < 1 || n > (1ll << 30)) return fail(s, MG_ERR_INVALID, "cells[%d] out of range", d);
    if (c->h[d] < 0.0) return fail(s, MG_ERR_INVALID, "h[%d] < 0", d);
    if (n < mincells) mincells = n;
  }
  int L = c->levels;
  if (L < 0) return fail(s, MG_ERR_INVALID, "levels < 0");
  if (L == 0) {
    L = 1;
    while ((mincells >> L) >= 2 && ((mincells >> L) << L) == mincells) L++;
  }
  for (int d = 0; d < c->dim; d++) {
    const int64_t n = c->nodes[d];
    if (L - 1 >= 62 || (n % (1ll << (L - 1))) != 0 || (n >> (L - 1)) < 1)
      return fail(s, MG_ERR_NOT_COARSENABLE, "cells[%d] = %lld not divisible by 2^(levels-1) = 2^%d", d,
                  (long long)n, L - 1);
  }
  *levels_out = L;
  return MG_OK;
}

// ------------------------------------------------------------------ creation
static mg_status validate(const mg_config* c, int* levels_out) {
  mg_solver* s = nullptr;
  if (!c) return fail(s, MG_ERR_INVALID, "config is NULL");
  if (c->dim != 2 && c->dim != 3) return fail(s, MG_ERR_INVALID, "dim must be 2 or 3 (got %d)", c->dim);
  if (c->problem == MG_PROBLEM_COMPLEX_DIFFUSION) return validate_cd(c, levels_out);
  if (c->problem != MG_PROBLEM_POISSON) return fail(s, MG_ERR_INVALID, "bad problem %d", c->problem);
  if (c->smoother != MG_JACOBI && c->smoother != MG_RBGS && c->smoother != MG_GS_LEX)
    return fail(s, MG_ERR_INVALID, "bad smoother");
  if (c->smoother == MG_GS_LEX && (c->nranks > 1 || (c->flags & MG_FLAG_SLAB)))
    return fail(s, MG_ERR_INVALID, "the lexicographic smoother is sequential across the domain: nranks = 1, no MG_FLAG_SLAB");
  if (!(c->omega > 0.0 && c->omega < 2.0)) return fail(s, MG_ERR_INVALID, "omega must be in (0,2) (S:46)");
  if (c->nu1 < 0 || c->nu2 < 0) return fail(s, MG_ERR_INVALID, "nu1, nu2 must be >= 0");
  if (c->coarse != MG_COARSE_DIRECT && c->coarse != MG_COARSE_SWEEPS) return fail(s, MG_ERR_INVALID, "bad coarse");
  if (c->coarse == MG_COARSE_SWEEPS && c->ncoarse < 0) return fail(s, MG_ERR_INVALID, "ncoarse < 0");
  if (c->dtype != MG_FP64 && c->dtype != MG_FP32) return fail(s, MG_ERR_INVALID, "bad dtype");
  if (c->nranks < 1 || c->rank < 0 || c->rank >= c->nranks) return fail(s, MG_ERR_INVALID, "bad rank/nranks");
  int64_t mincells = INT64_MAX;
  for (int d = 0; d < c->dim; d++) {
    int64_t n = c->nodes[d] - 1;
    if (n < 2) return fail(s, MG_ERR_INVALID, "nodes[%d] must be >= 3", d);
    if (n > (1ll << 30)) return fail(s, MG_ERR_INVALID, "nodes[%d] too large", d);
    if (!(c->coeff[d] > 0.0)) return fail(s, MG_ERR_INVALID, "coeff[%d] must be > 0", d);
    if (c->h[d] < 0.0) return fail(s, MG_ERR_INVALID, "h[%d] < 0", d);
    if (n < mincells) mincells = n;
  }
  int L = c->levels;
  if (L < 0) return fail(s, MG_ERR_INVALID, "levels < 0");
  if (L == 0) {  // paper rule: coarsest level has one interior node along the shortest axis
    // "direct coarsening down to less than three unknowns per direction"
    L = 1;
    while ((mincells >> L) >= 2 && ((mincells >> L) << L) == mincells) L++;
    if ((mincells >> (L - 1)) > 3)
      return fail(s, MG_ERR_NOT_COARSENABLE,
                  "cannot coarsen %lld cells down to < 3 unknowns per direction (P:568); give levels explicitly",
                  (long long)mincells);
  }
  for (int d = 0; d < c->dim; d++) {
    int64_t n = c->nodes[d] - 1;
    if (L - 1 >= 62 || (n % (1ll << (L - 1))) != 0)
      return fail(s, MG_ERR_NOT_COARSENABLE, "nodes[%d]-1 = %lld not divisible by 2^(levels-1) = 2^%d (S:242)", d,
                  (long long)n, L - 1);
    if ((n >> (L - 1)) < 2)
      return fail(s, MG_ERR_NOT_COARSENABLE, "coarsest level has no interior node along axis %d", d);
  }
  *levels_out = L;
  mg::Partition pt;
  std::string perr;
  mg_status ps = mg::compute_partition(c, L, &pt, &perr);
  if (ps != MG_OK) return fail(s, ps, "%s", perr.c_str());
  return MG_OK;
}

extern "C" mg_status mg_partition(const mg_config* cfg, int32_t level, int64_t* first_plane, int64_t* owned_planes,
                                  int32_t* distributed, int32_t* halo) {
  int L = 0;
  mg_status st = validate(cfg, &L);
  if (st != MG_OK) return st;
  if (cfg->problem != MG_PROBLEM_POISSON) return fail(nullptr, MG_ERR_INVALID, "complex diffusion is not decomposed");
  if (level < 0 || level >= L) return fail(nullptr, MG_ERR_INVALID, "level %d out of range", level);
  mg::Partition pt;
  std::string perr;
  st = mg::compute_partition(cfg, L, &pt, &perr);
  if (st != MG_OK) return fail(nullptr, st, "%s", perr.c_str());
  const bool dist = pt.slab && level < pt.la;
  if (first_plane) *first_plane = dist ? pt.a[level] : 0;
  if (owned_planes) *owned_planes = dist ? pt.b[level] - pt.a[level] : pt.n[level] + 1;
  if (distributed) *distributed = dist ? 1 : 0;
  if (halo) *halo = dist ? pt.H : 0;
  return MG_OK;
}

extern "C" mg_status mg_create(const mg_config* cfg, mg_solver** out) {
  if (!out) return fail(nullptr, MG_ERR_INVALID, "out is NULL");
  *out = nullptr;
  int L = 0;
  mg_status st = validate(cfg, &L);
  if (st != MG_OK) return st;
  if (cfg->nranks > 1 && !cfg->nccl_id && !cfg->loopback)
    return fail(nullptr, MG_ERR_INVALID, "nranks > 1 needs nccl_id (ncclUniqueId) or a loopback group");
  if (cfg->nranks > 1 && cfg->loopback) {
    if (mg::loop_group_size(static_cast<mg::LoopGroup*>(cfg->loopback)) != cfg->nranks)
      return fail(nullptr, MG_ERR_INVALID, "loopback group size != nranks");
  }
  int ndev = 0;
  cudaError_t ce = cudaGetDeviceCount(&ndev);
  if (ce != cudaSuccess || ndev == 0)
    return fail(nullptr, MG_ERR_CUDA, "no CUDA device (%s); there is no CPU fallback", cudaGetErrorString(ce));
  if (cfg->device < 0 || cfg->device >= ndev) return fail(nullptr, MG_ERR_INVALID, "bad device %d", cfg->device);

  if (!(cfg->comm_timeout_s >= 0.0) || !std::isfinite(cfg->comm_timeout_s))
    return fail(nullptr, MG_ERR_INVALID, "comm_timeout_s must be finite and >= 0");
  mg_solver* s = new mg_solver();
  s->cfg = *cfg;
  s->L = L;
  s->comm_timeout_s = cfg->comm_timeout_s > 0.0 ? cfg->comm_timeout_s : 300.0;
  s->esz = cfg->dtype == MG_FP64 ? 8 : 4;
  st = plan_build(s);
  if (st != MG_OK) {
    plan_free(s);
    delete s;
    return st;
  }
  *out = s;
  return MG_OK;
}

extern "C" mg_status mg_fault_inject(mg_solver* s, int32_t kind, int32_t countdown) {
  if (!s) return fail(s, MG_ERR_INVALID, "solver is NULL");
  if (kind < MG_FAULT_NONE || kind > MG_FAULT_HALO_CORRUPT || (kind != MG_FAULT_NONE && countdown < 1))
    return fail(s, MG_ERR_INVALID, "bad fault kind %d / countdown %d", kind, countdown);
  if (kind != MG_FAULT_NONE && !mg::comm_active(s))
    return fail(s, MG_ERR_INVALID, "fault injection needs a multi-rank exchange (nranks > 1)");
  s->fault_kind = kind;
  s->fault_count = kind == MG_FAULT_NONE ? 0 : countdown;
  return MG_OK;
}

extern "C" void mg_destroy(mg_solver* s) {
  if (!s) return;
  plan_free(s);
  delete s;
}

extern "C" const char* mg_error_string(const mg_solver* s) {
  if (s && !s->err.empty()) return s->err.c_str();
  return g_last_error.c_str();
}

extern "C" int32_t mg_num_levels(const mg_solver* s) { return s ? s->L : 0; }

extern "C" mg_status mg_layout(const mg_solver* s, int64_t shape[3], int64_t* first, int64_t* owned) {
  if (!s || !shape) return fail(nullptr, MG_ERR_INVALID, "NULL argument");
  const Level& lv = s->lv[0];
  for (int d = 0; d < 3; d++) shape[d] = lv.shape[d];
  if (first) *first = lv.dist ? s->pt.a[0] : 0;
  if (owned) *owned = lv.dist ? s->pt.b[0] - s->pt.a[0] : lv.shape[0];
  return MG_OK;
}

extern "C" mg_status mg_level_layout(const mg_solver* s, int32_t level, int64_t shape[3]) {
  if (!s || !shape) return fail(nullptr, MG_ERR_INVALID, "NULL argument");
  if (level < 0 || level >= s->L) return fail(nullptr, MG_ERR_INVALID, "level %d out of range", level);
  for (int d = 0; d < 3; d++) shape[d] = s->lv[level].shape[d];
  return MG_OK;
}

extern "C" int64_t mg_launches_per_cycle(const mg_solver* s) { return s ? s->launches_per_cycle : -1; }

// ------------------------------------------------------------------ execution
static mg_status guard(mg_solver* s) {
  if (!s) return fail(nullptr, MG_ERR_INVALID, "solver is NULL");
  if (s->poisoned) return fail(s, MG_ERR_POISONED, "solver poisoned by an earlier error: %s", s->err.c_str());
  cudaError_t e = cudaSetDevice(s->cfg.device);
  if (e != cudaSuccess) return fail(s, MG_ERR_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
  return MG_OK;
}

static bool aligned(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// device arrays: non-NULL and 16-byte aligned (TMA boxes and vector accesses need it)
static mg_status check_arrays(mg_solver* s, std::initializer_list<const void*> ps) {
  for (const void* p : ps) {
    if (!p) return fail(s, MG_ERR_INVALID, "NULL array argument");
    if (!aligned(p)) return fail(s, MG_ERR_LAYOUT, "device arrays must be 16-byte aligned");
  }
  return MG_OK;
}

extern "C" mg_status mg_vcycle(mg_solver* s, void* u, const void* f, void* stream) {
  mg_status st = guard(s);
  if (st != MG_OK) return st;
  if (!u || !f) return fail(s, MG_ERR_INVALID, "u or f is NULL");
  if (u == f) return fail(s, MG_ERR_INVALID, "u and f must not alias");
  if (!aligned(u) || !aligned(f)) return fail(s, MG_ERR_LAYOUT, "u and f must be 16-byte aligned");
  cudaStream_t cs = (cudaStream_t)stream;
  bool eager = (s->cfg.flags & MG_FLAG_NO_GRAPH) || s->prof_on;
  if (eager) return plan_run_vcycle(s, u, f, cs);
  return plan_graph_vcycle(s, u, f, cs);
}

extern "C" mg_status mg_residual_norm(mg_solver* s, const void* u, const void* f, double* out, void* stream) {
  mg_status st = guard(s);
  if (st != MG_OK) return st;
  if (!out) return fail(s, MG_ERR_INVALID, "NULL argument");
  if ((st = check_arrays(s, {u, f})) != MG_OK) return st;
  return plan_norm(s, 0, u, f, out, (cudaStream_t)stream, true);
}

extern "C" mg_status mg_solve(mg_solver* s, void* u, const void* f, double rtol, int32_t max_cycles, int32_t* cycles,
                              double* history, void* stream) {
  mg_status st = guard(s);
  if (st != MG_OK) return st;
  if (max_cycles < 0 || std::isnan(rtol)) return fail(s, MG_ERR_INVALID, "bad argument");
  const bool test_on = rtol >= 0.0;  // rtol < 0: exactly max_cycles cycles (no residual test)
  if ((st = check_arrays(s, {u, f})) != MG_OK) return st;
  if (u == f) return fail(s, MG_ERR_INVALID, "u and f must not alias");
  cudaStream_t cs = (cudaStream_t)stream;
  const bool eager_mode = (s->cfg.flags & MG_FLAG_NO_GRAPH) || s->prof_on;
  if (!(s->cfg.flags & MG_FLAG_HOST_LOOP)) {
    if (plan_solve_in_tail(s))  // one launch for the whole solve (eager: without a graph)
      return plan_solve_device(s, u, f, rtol, max_cycles, cycles, history, cs, eager_mode);
    if (!eager_mode && plan_loop_supported(s)) return plan_solve_device(s, u, f, rtol, max_cycles, cycles, history, cs);
  }
  // host-driven loop with the device loop's parts: pipelined split (plan_can_split) — head(k) =
  // first sweep of cycle k+1 into the ping-pong buffer + ||f - A u_k|| of its input, tail(k) =
  // the rest of cycle k+1 (u holds u_k whenever a norm is read, so stopping after a head is
  // exact); unsplit — the norm of u_0, then per cycle the cycle and the norm of its result
  const bool split = plan_can_split(s);
  const bool eager = (s->cfg.flags & MG_FLAG_NO_GRAPH) || s->prof_on;
  auto part = [&](int p) { return eager ? plan_run_part(s, p, u, f, cs) : plan_graph_part(s, p, u, f, cs); };
  auto read = [&](double* out) -> mg_status {
    CK(cudaMemcpyAsync(s->h_norm, s->d_norm, sizeof(double), cudaMemcpyDeviceToHost, cs));
    const mg_status w = plan_wait(s, cs, "mg_solve: norm readback");
    if (w != MG_OK) return w;
    *out = *s->h_norm;
    return MG_OK;
  };
  double r0 = 0.0;
  if ((st = part(split ? 1 : 3)) != MG_OK || (st = read(&r0)) != MG_OK) return st;
  if (history) history[0] = r0;
  if (!std::isfinite(r0)) return fail(s, MG_ERR_NONFINITE, "initial residual norm is not finite");
  int k = 0;
  while (k < max_cycles) {
    if ((st = part(split ? 2 : 5)) != MG_OK) return st;
    k++;
    double rk = 0.0;
    if (split && (st = part(4)) != MG_OK) return st;  // head w/o the boundary refresh
    if ((st = read(&rk)) != MG_OK) return st;
    if (history) history[k] = rk;
    if (!std::isfinite(rk)) {
      if (cycles) *cycles = k;
      return fail(s, MG_ERR_NONFINITE, "residual norm not finite after cycle %d (S:535)", k);
    }
    if (test_on && rk <= rtol * r0) break;
  }
  if (cycles) *cycles = k;
  return MG_OK;
}

// On an error return, copies queued before the failure may still reference the caller's host
// buffers: drain the streams involved (their own errors ignored) before returning.
static void drain_host_copies(mg_solver* s, cudaStream_t cs) {
  if (s->h2d_stream) cudaStreamSynchronize(s->h2d_stream);
  if (s->d2h_stream) cudaStreamSynchronize(s->d2h_stream);
  cudaStreamSynchronize(cs);
  cudaGetLastError();
}

static mg_status vcycle_host_run(mg_solver* s, void* u_host, const void* f_host, int32_t ncycles,
                                 double* norm_out, void* stream) {
  mg_status st = MG_OK;
  cudaStream_t cs = (cudaStream_t)stream;
  const Level& lv = s->lv[0];
  size_t bytes = lv.elems * s->esz * (s->cfg.problem == MG_PROBLEM_COMPLEX_DIFFUSION ? 2 : 1);
  if (!s->stage_u) {
    if (cudaMalloc(&s->stage_u, bytes) != cudaSuccess || cudaMalloc(&s->stage_f, bytes) != cudaSuccess) {
      cudaGetLastError();
      return fail(s, MG_ERR_OOM, "staging allocation failed");
    }
  }
  CK(cudaMemcpyAsync(s->stage_f, f_host, bytes, cudaMemcpyHostToDevice, cs));
  CK(cudaMemcpyAsync(s->stage_u, u_host, bytes, cudaMemcpyHostToDevice, cs));
  for (int c = 0; c < ncycles; c++) {
    st = mg_vcycle(s, s->stage_u, s->stage_f, stream);
    if (st != MG_OK) return st;
  }
  if (norm_out) {
    st = plan_norm(s, 0, s->stage_u, s->stage_f, norm_out, cs, false);
    if (st != MG_OK) return st;
  }
  CK(cudaMemcpyAsync(u_host, s->stage_u, bytes, cudaMemcpyDeviceToHost, cs));
  if ((st = plan_wait(s, cs, "mg_vcycle_host")) != MG_OK) return st;
  if (norm_out) *norm_out = *s->h_norm;
  return MG_OK;
}

extern "C" mg_status mg_vcycle_host(mg_solver* s, void* u_host, const void* f_host, int32_t ncycles,
                                    double* norm_out, void* stream) {
  mg_status st = guard(s);
  if (st != MG_OK) return st;
  if (!u_host || !f_host || ncycles < 0) return fail(s, MG_ERR_INVALID, "bad argument");
  st = vcycle_host_run(s, u_host, f_host, ncycles, norm_out, stream);
  if (st != MG_OK) drain_host_copies(s, (cudaStream_t)stream);
  return st;
}

static mg_status host_batch_run(mg_solver* s, const void* const* u_in, void* const* u_out, const void* const* f_in,
                                int32_t nbatch, int32_t ncycles, double* norms, void* stream);

extern "C" mg_status mg_vcycle_host_batch(mg_solver* s, const void* const* u_in, void* const* u_out,
                                          const void* const* f_in, int32_t nbatch, int32_t ncycles, double* norms,
                                          void* stream) {
  mg_status st = guard(s);
  if (st != MG_OK) return st;
  if (!u_in || !u_out || !f_in || nbatch < 0 || ncycles < 0) return fail(s, MG_ERR_INVALID, "bad argument");
  for (int b = 0; b < nbatch; b++)
    if (!u_in[b] || !u_out[b] || !f_in[b]) return fail(s, MG_ERR_INVALID, "NULL host buffer of problem %d", b);
  st = host_batch_run(s, u_in, u_out, f_in, nbatch, ncycles, norms, stream);
  if (st != MG_OK) drain_host_copies(s, (cudaStream_t)stream);
  return st;
}

static mg_status host_batch_run(mg_solver* s, const void* const* u_in, void* const* u_out, const void* const* f_in,
                                int32_t nbatch, int32_t ncycles, double* norms, void* stream) {
  mg_status st = MG_OK;
  cudaStream_t cs = (cudaStream_t)stream;
  const Level& lv = s->lv[0];
  const size_t bytes = lv.elems * s->esz * (s->cfg.problem == MG_PROBLEM_COMPLEX_DIFFUSION ? 2 : 1);
  if (!s->h2d_stream) {
    for (int k = 0; k < 2; k++) {
      if (cudaMalloc(&s->bstage_u[k], bytes) != cudaSuccess || cudaMalloc(&s->bstage_f[k], bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(s, MG_ERR_OOM, "staging allocation failed");
      }
      CK(cudaEventCreateWithFlags(&s->ev_h2d[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&s->ev_comp[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&s->ev_d2h[k], cudaEventDisableTiming));
    }
    CK(cudaStreamCreateWithFlags(&s->h2d_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s->d2h_stream, cudaStreamNonBlocking));
  }
  if (norms && nbatch > s->h_norms_cap) {
    if (s->h_norms) cudaFreeHost(s->h_norms);
    s->h_norms = nullptr;
    s->h_norms_cap = 0;
    CK(cudaMallocHost(&s->h_norms, sizeof(double) * nbatch));
    s->h_norms_cap = nbatch;
  }
  // the pipeline starts after everything already queued on the caller's stream
  CK(cudaEventRecord(s->ev_comp[0], cs));
  CK(cudaStreamWaitEvent(s->h2d_stream, s->ev_comp[0], 0));
  for (int b = 0; b < nbatch; b++) {
    const int k = b & 1;
    void* su = s->bstage_u[k];
    void* sf = s->bstage_f[k];
    // H2D of problem b into set k once problem b-2 (same set) has been copied out
    if (b >= 2) CK(cudaStreamWaitEvent(s->h2d_stream, s->ev_d2h[k], 0));
    CK(cudaMemcpyAsync(sf, f_in[b], bytes, cudaMemcpyHostToDevice, s->h2d_stream));
    CK(cudaMemcpyAsync(su, u_in[b], bytes, cudaMemcpyHostToDevice, s->h2d_stream));
    CK(cudaEventRecord(s->ev_h2d[k], s->h2d_stream));
    // cycles + norm on the caller's stream
    CK(cudaStreamWaitEvent(cs, s->ev_h2d[k], 0));
    for (int c = 0; c < ncycles; c++)
      if ((st = mg_vcycle(s, su, sf, stream)) != MG_OK) return st;
    if (norms) {
      if ((st = plan_norm(s, 0, su, sf, nullptr, cs, false)) != MG_OK) return st;  // -> d_norm
      CK(cudaMemcpyAsync(s->h_norms + b, s->d_norm, sizeof(double), cudaMemcpyDeviceToHost, cs));
    }
    CK(cudaEventRecord(s->ev_comp[k], cs));
    // D2H of the result on the other copy engine
    CK(cudaStreamWaitEvent(s->d2h_stream, s->ev_comp[k], 0));
    CK(cudaMemcpyAsync(u_out[b], su, bytes, cudaMemcpyDeviceToHost, s->d2h_stream));
    CK(cudaEventRecord(s->ev_d2h[k], s->d2h_stream));
  }
  if ((st = plan_wait(s, s->d2h_stream, "mg_vcycle_host_batch")) != MG_OK) return st;
  if ((st = plan_wait(s, cs, "mg_vcycle_host_batch")) != MG_OK) return st;
  if (norms)
    for (int b = 0; b < nbatch; b++) norms[b] = s->h_norms[b];
  return MG_OK;
}

// ------------------------------------------------------------------ per-op entry points
#define LEVEL_CHECK(l)                                                                        \
  do {                                                                                        \
    if ((l) < 0 || (l) >= s->L) return fail(s, MG_ERR_INVALID, "level %d out of range", (l)); \
  } while (0)

extern "C" mg_status mg_op_smooth(mg_solver* s, int32_t level, const void* u_in, const void* f, void* u_out,
                                  void* stream) {
  mg_status st = guard(s);
  if (st != MG_OK) return st;
  LEVEL_CHECK(level);
  if ((st = check_arrays(s, {u_in, f, u_out})) != MG_OK) return st;
  return plan_op_smooth(s, level, u_in, f, u_out, (cudaStream_t)stream);
}
extern "C" mg_status mg_op_residual(mg_solver* s, int32_t level, const void* u, const void* f, void* r,
                                    void* stream) {
  mg_status st = guard(s);
  if (st != MG_OK) return st;
  LEVEL_CHECK(level);
  if ((st = check_arrays(s, {u, f, r})) != MG_OK) return st;
  return plan_op_residual(s, level, u, f, r, (cudaStream_t)stream);
}
extern "C" mg_status mg_op_restrict(mg_solver* s, int32_t level, const void* r, void* fc, void* stream) {
  mg_status st = guard(s);
  if (st != MG_OK) return st;
  LEVEL_CHECK(level + 1);
  if ((st = check_arrays(s, {r, fc})) != MG_OK) return st;
  return plan_op_restrict(s, level, r, fc, (cudaStream_t)stream);
}
extern "C" mg_status mg_op_prolong_correct(mg_solver* s, int32_t level, const void* e, void* u, void* stream) {
  mg_status st = guard(s);
  if (st != MG_OK) return st;
  LEVEL_CHECK(level + 1);
  if ((st = check_arrays(s, {e, u})) != MG_OK) return st;
  return plan_op_prolong(s, level, e, u, (cudaStream_t)stream);
}
extern "C" mg_status mg_op_coarse_solve(mg_solver* s, const void* f, void* e, void* stream) {
  mg_status st = guard(s);
  if (st != MG_OK) return st;
  if ((st = check_arrays(s, {f, e})) != MG_OK) return st;
  return plan_op_coarse(s, f, e, (cudaStream_t)stream);
}
extern "C" mg_status mg_op_norm(mg_solver* s, int32_t level, const void* u, const void* f, double* out,
                                void* stream) {
  mg_status st = guard(s);
  if (st != MG_OK) return st;
  LEVEL_CHECK(level);
  if (!out) return fail(s, MG_ERR_INVALID, "NULL argument");
  if ((st = check_arrays(s, {u, f})) != MG_OK) return st;
  return plan_norm(s, level, u, f, out, (cudaStream_t)stream, true);
}

extern "C" mg_status mg_workload_fill(mg_solver* s, void* dst, uint64_t seed, double lo, double hi, void* stream) {
  mg_status st = guard(s);
  if (st != MG_OK) return st;
  if ((st = check_arrays(s, {dst})) != MG_OK) return st;
  return plan_workload_fill(s, dst, seed, lo, hi, (cudaStream_t)stream);
}

// ------------------------------------------------------------------ profiling
extern "C" mg_status mg_profile_enable(mg_solver* s, int32_t on) {
  mg_status st = guard(s);
  if (st != MG_OK) return st;
  return plan_profile_enable(s, on != 0);
}

extern "C" int32_t mg_profile_read(mg_solver* s, int32_t cap, const char** names, double* ms, int64_t* count,
                                   double* bytes) {
  if (!s) return -1;
  return plan_profile_read(s, cap, names, ms, count, bytes);
}

// used by plan.cu for error reporting
mg_status mg::plan_fail(mg_solver* s, mg_status st, const char* msg) { return fail(s, st, "%s", msg); }

extern "C" mg_status mg_loopback_group_create(int32_t nranks, void** group) {
  if (!group || nranks < 1) return fail(nullptr, MG_ERR_INVALID, "bad argument");
  *group = mg::loop_group_create(nranks);
  return MG_OK;
}

extern "C" void mg_loopback_group_destroy(void* group) { mg::loop_group_destroy(static_cast<mg::LoopGroup*>(group)); }

extern "C" mg_status mg_nccl_unique_id(void* out128) {
  if (!out128) return fail(nullptr, MG_ERR_INVALID, "out is NULL");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, MG_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  memcpy(out128, &id, sizeof id);
  return MG_OK;
}
