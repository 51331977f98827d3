// plan.cu — level hierarchy, buffers and the V-cycle schedule (Alg. 1,
// P:187-219; Layer-4 VCycle listing P:278-297), executed eagerly or captured
// once per (u, f) pair into a CUDA graph and replayed.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>

#include <nccl.h>

#include "kernels.h"
#include "partition.h"
#include "kernels_pm.h"
#include "kernels_pm2d.h"
#include "kernels_tail.h"
#include <cstdlib>
#include "plan.h"

namespace mg {

enum Kind {
  K_JACOBI = 0,
  K_RBGS_COLOUR,
  K_RESIDUAL,
  K_RESTRICT,
  K_PROLONG,
  K_COPY_BOUNDARY,
  K_COPY_INTERIOR,
  K_NORM_PARTIAL,
  K_NORM_FINAL,
  K_COARSE_DIRECT,
  K_MEMSET,
  K_ADD,
  K_SWEEP_RBGS,
  K_SWEEP_JACOBI,
  K_RESID_RESTRICT,
  K_HALO,
  K_ALLGATHER,
  K_SWEEP_NORM,
  K_TAIL,
  K_SWEEP_CORR,
  K_CD_GFIELD,
  K_CD_JACOBI,
  K_CD_RBGS,
  K_CD_RESTRICT,
  K_CD_FAS_RHS,
  K_CD_PROLONG,
  K_CD_NORM,
  K_CD_RESIDUAL,
  K_CD_COPY,
  K_CD_TAIL,
  K_GS_LEX,
  K_SWEEP_JACOBI_K,
  K_SWEEP_NORM_K,
  K_PROLONG_JACOBI_K,
  K_CD_JACOBI_K,
  K_CD_JACOBI_K_NORM,
  K_SWEEP_RR_K,
  K_TAIL_NORM,
  K_TAIL_NORM_FUSED,
  K_TAIL_SOLVE,
  K_NUM
};
static const char* kKindName[K_NUM] = {"jacobi",        "rbgs_colour",   "residual",     "restrict",
                                       "prolong_correct", "copy_boundary", "copy_interior", "norm_partial",
                                       "norm_final",    "coarse_direct", "memset",       "add_interior",
                                       "rbgs_fused",    "jacobi_pm",     "resid_restrict",
                                       "nccl_halo",     "nccl_allgather", "sweep+norm",
                                       "coarse_tail",   "prolong+sweep",
                                       "cd_gfield",     "cd_jacobi",     "cd_rbgs_colour", "cd_restrict",
                                       "cd_fas_rhs",    "cd_prolong",    "cd_norm_partial", "cd_residual",
                                       "cd_copy",       "cd_tail",       "gs_lex_plane",  "jacobi_pm_xK",
                                       "jacobi_pm_xK+norm", "prolong+jacobi_xK",
                                       "cd_jacobi_xK",  "cd_jacobi_xK+norm", "jacobi_xK+resid_restrict",
                                       "tail_norm",     "coarse_tail+norm", "coarse_tail_solve"};

static mg_status cuda_fail(mg_solver* s, cudaError_t e, const char* what) {
  char buf[384];
  snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
  return plan_fail(s, MG_ERR_CUDA, buf);
}

// One kernel launch through the instrumentation wrapper.
template <class Fn>
static mg_status launch(mg_solver* s, cudaStream_t st, Kind kind, int level, double bytes, Fn&& fn) {
  ProfRec rec{};
  bool prof = s->prof_on;
  if (prof) {
    rec.kind = kind;
    rec.level = level;
    rec.bytes = bytes;
    if (cudaEventCreate(&rec.a) != cudaSuccess || cudaEventCreate(&rec.b) != cudaSuccess ||
        cudaEventRecord(rec.a, st) != cudaSuccess) {  // instrumentation only: skip this record
      if (rec.a) cudaEventDestroy(rec.a);
      if (rec.b) cudaEventDestroy(rec.b);
      cudaGetLastError();
      prof = false;
    }
  }
  cudaError_t e = fn();
  if (prof) {
    if (cudaEventRecord(rec.b, st) == cudaSuccess) {
      s->prof.push_back(rec);
    } else {
      cudaEventDestroy(rec.a);
      cudaEventDestroy(rec.b);
      cudaGetLastError();
    }
  }
  if (kind != K_MEMSET && kind != K_HALO && kind != K_ALLGATHER) s->launch_counter++;  // our kernels only
  if (e != cudaSuccess) {
    if (s->comm_failed) {  // an exchange failed (comm.cu): the communication error, not a CUDA one
      s->comm_failed = false;
      return plan_fail(s, MG_ERR_NCCL, s->comm_msg.c_str());
    }
    return cuda_fail(s, e, kKindName[kind]);
  }
  return MG_OK;
}

static double nodes_of(const Level& L) { return (double)(L.g.nx + 1) * L.shape[1] * L.shape[0]; }

// ---------------------------------------------------------------- small kernels
template <typename T>
__global__ void k_copy_interior(Geom g, const T* __restrict__ src, T* __restrict__ dst) {
  long long q = (long long)blockIdx.x * blockDim.y + threadIdx.y;
  int nrow = g.three_d ? g.ny - 1 : 1;
  if (q >= (long long)nrow * (g.p_hi - g.p_lo)) return;
  int j = g.three_d ? (int)(q % nrow) + 1 : 0;
  int pl = g.p_lo + (int)(q / nrow);
  long long base = (long long)pl * g.pstride + (long long)j * g.pitch;
  for (int i = 1 + threadIdx.x; i < g.nx; i += blockDim.x)
    dst[base + i] = src[base + i];
}

template <typename T>
__global__ void k_add_interior(Geom g, const T* __restrict__ e, T* __restrict__ u) {
  long long q = (long long)blockIdx.x * blockDim.y + threadIdx.y;
  int nrow = g.three_d ? g.ny - 1 : 1;
  if (q >= (long long)nrow * (g.p_hi - g.p_lo)) return;
  int j = g.three_d ? (int)(q % nrow) + 1 : 0;
  int pl = g.p_lo + (int)(q / nrow);
  long long base = (long long)pl * g.pstride + (long long)j * g.pitch;
  for (int i = 1 + threadIdx.x; i < g.nx; i += blockDim.x)
    u[base + i] = add(u[base + i], e[base + i]);
}

static dim3 rows_grid(const Geom& g) {
  int nrow = g.three_d ? g.ny - 1 : 1;
  long long q = (long long)nrow * (g.p_hi - g.p_lo);
  return dim3((unsigned)((q + 1) / 2));
}

static mg_status cd_build(mg_solver* s);
static mg_status alloc_common(mg_solver* s, int np);

// norm partials / scalar, capture streams, driver-loop state (both problems)
static mg_status alloc_common(mg_solver* s, int np) {
  if (np < 64) np = 64;  // also the coarse tail's scratch (per-CTA norm sums + its loop flag)
  s->n_partial_cap = np;
  if (cudaMalloc(&s->d_partial, sizeof(double) * np) != cudaSuccess ||
      cudaMalloc(&s->d_norm, sizeof(double)) != cudaSuccess ||
      cudaMalloc(&s->d_rank_sums, sizeof(double) * s->cfg.nranks) != cudaSuccess ||
      cudaMallocHost(&s->h_norm, sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    return plan_fail(s, MG_ERR_OOM, "allocation of norm buffers failed");
  }
  cudaError_t e = cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s->cap_body, cudaStreamNonBlocking);
  if (e == cudaSuccess && comm_active(s)) {  // halo exchanges overlapped with interior sweeps
    e = cudaStreamCreateWithFlags(&s->comm_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming);
  }
  if (e != cudaSuccess) return cuda_fail(s, e, "cudaStreamCreate");
  if (cudaMalloc(&s->d_loop, sizeof(LoopState)) != cudaSuccess ||
      cudaMallocHost(&s->h_loop, sizeof(LoopState)) != cudaSuccess) {
    cudaGetLastError();
    return plan_fail(s, MG_ERR_OOM, "allocation of the driver-loop state failed");
  }
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(s, e, "setup");
  return MG_OK;
}

// ---------------------------------------------------------------- build / free
mg_status plan_build(mg_solver* s) {
  const mg_config& c = s->cfg;
  cudaError_t e = cudaSetDevice(c.device);
  if (e != cudaSuccess) return cuda_fail(s, e, "cudaSetDevice");
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, c.device);
  if (major != 10) {
    char buf[128];
    snprintf(buf, sizeof buf, "device %d has compute capability %d.x; libmgb200 is built for sm_100a only", c.device,
             major);
    return plan_fail(s, MG_ERR_CUDA, buf);
  }
  if (c.problem == MG_PROBLEM_COMPLEX_DIFFUSION) return cd_build(s);
  const int esz = (int)s->esz;
  const int64_t align = 128 / esz;
  {
    std::string perr;
    mg_status ps = compute_partition(&c, s->L, &s->pt, &perr);
    if (ps != MG_OK) return plan_fail(s, ps, perr.c_str());
  }
  if (c.nranks > 1 && c.loopback) {  // loopback transport: ranks of this process on this device
    s->loop = static_cast<LoopGroup*>(c.loopback);
    if (cudaEventCreateWithFlags(&s->lb_ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->lb_done, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      return plan_fail(s, MG_ERR_CUDA, "loopback events");
    }
  } else if (c.nranks > 1) {  // NCCL communicator over NVLink (unique id broadcast by the caller)
    // (ncclCommInitRank blocks until every rank has joined: mg_create is collective)
    ncclUniqueId id;
    memcpy(&id, c.nccl_id, sizeof id);
    ncclResult_t nr = ncclCommInitRank(&s->comm, c.nranks, id, c.rank);
    if (nr != ncclSuccess) {
      s->comm = nullptr;
      return plan_fail(s, MG_ERR_NCCL, ncclGetErrorString(nr));
    }
  }
  s->lv.resize(s->L);
  for (int l = 0; l < s->L; l++) {
    Level& L = s->lv[l];
    int64_t n[3];
    double hh[3];
    for (int d = 0; d < 3; d++) {
      n[d] = d < c.dim ? (c.nodes[d] - 1) >> l : 0;
      double h0 = c.h[d] > 0.0 ? c.h[d] : (d < c.dim ? 1.0 / (double)(c.nodes[d] - 1) : 0.0);
      hh[d] = std::ldexp(h0, l);
    }
    // coefficients in double in the paper's axis order x, y, z (reading 13)
    double cd[3] = {0, 0, 0}, sum = 0.0;
    for (int d = 0; d < c.dim; d++) {
      cd[d] = c.coeff[d] / (hh[d] * hh[d]);
      sum += cd[d];
    }
    double D = 2.0 * sum, wd = c.omega / D;
    Geom& g = L.g;
    g.three_d = c.dim == 3;
    g.nx = (int)n[0];
    if (c.dim == 3) {
      g.ny = (int)n[1];
      g.nz = (int)n[2];
      g.rows = g.ny + 1;
      L.cx = cd[0];
      L.cy = cd[1];
      L.cz = cd[2];
    } else {
      g.ny = 0;
      g.nz = (int)n[1];  // the paper's y is the plane axis
      g.rows = 1;
      L.cx = cd[0];
      L.cy = 0.0;
      L.cz = cd[1];
    }
    L.D = D;
    g.pitch = (g.nx + 1 + align - 1) / align * align;
    g.pstride = g.pitch * g.rows;
    g.p_lo = 1;
    g.p_hi = g.nz;
    g.p_glob0 = 0;
    g.planes = g.nz + 1;
    L.dist = s->pt.slab && l < s->pt.la;
    if (L.dist) {  // slab: owned planes [a, b) + H halo planes on each side
      const int H = s->pt.H;
      const int a = (int)s->pt.a[l], b = (int)s->pt.b[l];
      g.p_glob0 = a - H;
      g.planes = (b - a) + 2 * H;
      g.p_lo = H + (a == 0 ? 1 : 0);
      g.p_hi = H + ((b < g.nz ? b : g.nz) - a);
    }
    L.gown = g;
    if (s->pt.slab && l == s->pt.la) {  // first full level: this rank restricts into its own planes
      const int a = (int)s->pt.a[l], b = (int)s->pt.b[l];
      L.gown.p_lo = a > 1 ? a : 1;
      L.gown.p_hi = b < g.nz ? b : g.nz;
    }
    L.shape[0] = g.planes;
    L.shape[1] = g.rows;
    L.shape[2] = g.pitch;
    L.elems = (size_t)L.shape[0] * L.shape[1] * L.shape[2];
    L.c64 = Coef<double>{L.cx, L.cy, L.cz, D, wd};
    L.c32 = Coef<float>{(float)L.cx, (float)L.cy, (float)L.cz, (float)D, (float)wd};
    size_t bytes = L.elems * esz;
    void** bufs[4] = {&L.u, &L.f, &L.r, &L.t};
    for (int b = 0; b < 4; b++) {
      if (l == 0 && b < 2) continue;  // level 0 u, f are the caller's
      if (cudaMalloc(bufs[b], bytes) != cudaSuccess) {
        cudaGetLastError();
        return plan_fail(s, MG_ERR_OOM, "device allocation of level buffers failed");
      }
      e = cudaMemset(*bufs[b], 0, bytes);
      if (e != cudaSuccess) return cuda_fail(s, e, "cudaMemset");
    }
  }
  // norm partials sized for the largest level
  int np = 1;
  for (int l = 0; l < s->L; l++) {
    int a = s->esz == 8 ? norm_num_partials<double>(s->lv[l].g) : norm_num_partials<float>(s->lv[l].g);
    if (a > np) np = a;
    if (pm::supported(s->lv[l].g, 16)) {
      a = s->esz == 8 ? pm::norm_partials<double>(s->lv[l].g) : pm::norm_partials<float>(s->lv[l].g);
      if (a > np) np = a;
    }
  }
  if (pm::supported(s->lv[0].g, 16)) {
    const bool rb = c.smoother == MG_RBGS;
    int a = s->esz == 8 ? pm::sweep_partials<double>(s->lv[0].g, rb) : pm::sweep_partials<float>(s->lv[0].g, rb);
    if (2 * a > np) np = 2 * a;  // the split norm: the tail's black partials + the head's red ones
  }
  // coarsest-level direct solve: factor once (reading 3)
  Level& C = s->lv[s->L - 1];
  int m = (C.g.nx - 1) * (C.g.three_d ? C.g.ny - 1 : 1) * (C.g.nz - 1);
  s->m_coarse = m;
  if (c.coarse == MG_COARSE_DIRECT && m > 1) {
    if (m > 1024) {
      char buf[200];
      snprintf(buf, sizeof buf,
               "DIRECT coarse solve with %d unknowns exceeds the 1024 limit: use more levels or MG_COARSE_SWEEPS", m);
      return plan_fail(s, MG_ERR_INVALID, buf);
    }
    int* d_status = nullptr;
    if (cudaMalloc(&s->d_chol, sizeof(double) * (size_t)m * m) != cudaSuccess ||
        cudaMalloc(&s->d_work, sizeof(double) * m) != cudaSuccess || cudaMalloc(&d_status, sizeof(int)) != cudaSuccess) {
      cudaGetLastError();
      return plan_fail(s, MG_ERR_OOM, "allocation of the coarse factor failed");
    }
    e = launch_cholesky_factor(C.g, C.cx, C.cy, C.cz, C.D, s->d_chol, m, d_status, 0);
    int hs = 1;
    if (e == cudaSuccess) e = cudaMemcpy(&hs, d_status, sizeof(int), cudaMemcpyDeviceToHost);
    cudaFree(d_status);
    if (e != cudaSuccess) return cuda_fail(s, e, "coarse Cholesky factorisation");
    if (hs != 0) return plan_fail(s, MG_ERR_INVALID, "coarsest matrix is not positive definite");
  }
  return alloc_common(s, np);
}

void plan_free(mg_solver* s) {
  cudaSetDevice(s->cfg.device);
  // a poisoned solver's NCCL kernels may wait on a dead peer: abort before anything synchronises
  if (s->comm && s->poisoned) plan_comm_abort(s);
  for (auto& kv : s->graphs) cudaGraphExecDestroy(kv.second);
  s->graphs.clear();
  for (auto& L : s->lv) {
    cudaFree(L.u);
    cudaFree(L.f);
    cudaFree(L.r);
    cudaFree(L.t);
    cudaFree(L.uh);
    cudaFree(L.gd);
  }
  s->lv.clear();
  cudaFree(s->d_chol);
  cudaFree(s->d_work);
  cudaFree(s->d_partial);
  cudaFree(s->d_norm);
  cudaFree(s->d_rank_sums);
  if (s->comm) {  // a poisoned solver's peers may be gone: abort instead of a collective teardown
    if (s->poisoned) ncclCommAbort(s->comm);
    else ncclCommDestroy(s->comm);
    s->comm = nullptr;
  }
  if (s->lb_ready) cudaEventDestroy(s->lb_ready);
  if (s->lb_done) cudaEventDestroy(s->lb_done);
  if (s->h_norm) cudaFreeHost(s->h_norm);
  cudaFree(s->stage_u);
  cudaFree(s->stage_f);
  for (int k = 0; k < 2; k++) {
    cudaFree(s->bstage_u[k]);
    cudaFree(s->bstage_f[k]);
    if (s->ev_h2d[k]) cudaEventDestroy(s->ev_h2d[k]);
    if (s->ev_comp[k]) cudaEventDestroy(s->ev_comp[k]);
    if (s->ev_d2h[k]) cudaEventDestroy(s->ev_d2h[k]);
  }
  if (s->h2d_stream) cudaStreamDestroy(s->h2d_stream);
  if (s->d2h_stream) cudaStreamDestroy(s->d2h_stream);
  if (s->h_norms) cudaFreeHost(s->h_norms);
  for (auto& r : s->prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  if (s->cap_stream) cudaStreamDestroy(s->cap_stream);
  if (s->cap_body) cudaStreamDestroy(s->cap_body);
  if (s->comm_stream) cudaStreamDestroy(s->comm_stream);
  if (s->ev_fork) cudaEventDestroy(s->ev_fork);
  if (s->ev_join) cudaEventDestroy(s->ev_join);
  cudaFree(s->d_loop);
  cudaFree(s->d_hist);
  if (s->h_loop) cudaFreeHost(s->h_loop);
}

// ---------------------------------------------------------------- typed schedule
template <typename T>
struct Exec {
  mg_solver* s;
  cudaStream_t st;
  const Coef<T>& coef(int l) const;
  double w(int l) const { return nodes_of(s->lv[l]) * sizeof(T); }  // one word per node of level l

  bool pm(int l) const {
    return !(s->cfg.flags & MG_FLAG_BASELINE) && s->cfg.smoother != MG_GS_LEX && pm::supported(s->lv[l].g, s->cfg.pm_min_nx ? s->cfg.pm_min_nx : 128);
  }
  // First level of the single-CTA coarse tail (levels >= lt run in one launch): the
  // first non-distributed level whose interior has <= 48K nodes.  L if none / disabled.
  int tail_level() const {
    if (s->cfg.flags & MG_FLAG_BASELINE) return s->L;
    const int first = s->pt.slab ? s->pt.la : 0;
    constexpr long long tail_max = 48ll * 1024;  // measured on C2/C3/C4
    for (int l = first; l < s->L; l++) {
      const Geom& g = s->lv[l].g;
      const long long n = (long long)(g.nx - 1) * (g.three_d ? g.ny - 1 : 1) * (g.nz - 1);
      if (n <= tail_max && s->L - l <= kTailMax && (l > 0 || s->L > 1)) return l;
    }
    return s->L;
  }

  // the coarse tail (levels lt..L-1) in one launch; norm_out: also ||f - A u|| of the result
  // (lt = 0); norm_only: only that norm of (u_top, f_top), no cycle
  mg_status run_tail(int lt, T* u_top, const T* f_top, double* norm_out = nullptr, bool norm_only = false) {
    TailParams<T> P = tail_params(lt, u_top, f_top);
    P.norm_out = norm_out;
    P.norm_only = norm_only ? 1 : 0;
    P.nscratch = s->d_partial;
    if (norm_only) return launch(s, st, K_TAIL_NORM, 0, 2 * w(0), [&] { return launch_tail<T>(P, st); });
    // only Jacobi with level 0 in global memory uses the global partner t (whose boundary must
    // hold u's): in shared memory, one CTA's or dist slabs, the kernel copies u into both
    if (lt == 0 && P.rbgs == 0 && P.smem_from != 0 && P.dist_n == 0) {
      const mg_status r = cycle_start(u_top, f_top);
      if (r != MG_OK) return r;
    }
    double bytes = 0;
    for (int k = 0; k < P.nl; k++) bytes += w(lt + k) * (3.0 * (P.nu1 + P.nu2) + 6.0);
    return launch(s, st, norm_out ? K_TAIL_NORM_FUSED : K_TAIL, lt, bytes, [&] { return launch_tail<T>(P, st); });
  }
  // mg_solve on a whole-cycle tail grid (tail_level() = 0): r0, the cycles, their norms and
  // the stop test in ONE launch, the hierarchy resident in shared memory across cycles; the
  // loop state (rtol, max, history, results) in s->d_loop as for the graph loop
  mg_status solve_tail(T* u, const T* f) {
    TailParams<T> P = tail_params(0, u, f);
    P.solve = s->d_loop;
    P.nscratch = s->d_partial;
    if (P.rbgs == 0 && P.smem_from != 0 && P.dist_n == 0) {  // the global Jacobi partner's boundary
      const mg_status r = cycle_start(u, f);
      if (r != MG_OK) return r;
    }
    double bytes = 0;
    for (int k = 0; k < P.nl; k++) bytes += w(k) * (3.0 * (P.nu1 + P.nu2) + 6.0);
    return launch(s, st, K_TAIL_SOLVE, 0, bytes, [&] { return launch_tail<T>(P, st); });
  }
  TailParams<T> tail_params(int lt, T* u_top, const T* f_top) {
    TailParams<T> P{};
    P.nl = s->L - lt;
    P.rbgs = s->cfg.smoother == MG_RBGS ? 1 : (s->cfg.smoother == MG_GS_LEX ? 2 : 0);
    P.nu1 = s->cfg.nu1;
    P.nu2 = s->cfg.nu2;
    P.sweeps = s->cfg.coarse == MG_COARSE_SWEEPS;
    P.ncoarse = s->cfg.ncoarse;
    P.zero_first = lt > 0;
    P.m = s->m_coarse;
    P.D_coarse = s->lv[s->L - 1].D;
    P.rD_coarse = 1.0 / P.D_coarse;  // IEEE division: RN(1 / D)
    P.chol = s->d_chol;
    P.work = s->d_work;
    for (int k = 0; k < P.nl; k++) {
      const Level& L = s->lv[lt + k];
      P.g[k] = L.g;
      P.c[k] = coef(lt + k);
      P.u[k] = k == 0 ? u_top : (T*)L.u;
      P.f[k] = k == 0 ? const_cast<T*>(f_top) : (T*)L.f;
      P.t[k] = (T*)L.t;
      P.r[k] = (T*)L.r;
    }
    tail_prepare<T>(P);
    return P;
  }


  // Slab halo exchange of a distributed level: my h top owned planes
  // go to rank+1's lower halo, my h bottom owned planes to rank-1's upper halo.
  mg_status exchange(int l, T* buf, int h) { return exchange_on(l, buf, h, st); }
  mg_status exchange_on(int l, T* buf, int h, cudaStream_t st) {
    const Level& L = s->lv[l];
    if (!L.dist || !comm_active(s)) return MG_OK;
    const int H = s->pt.H;
    const size_t ps = (size_t)L.g.pstride;
    const int owned = L.g.planes - 2 * H;
    return launch(s, st, K_HALO, l, 2.0 * h * ps * sizeof(T),
                  [&] { return comm_halo(s, buf, ps * sizeof(T), H, owned, h, st); });
  }

  // Agglomeration: every rank restricted into its own planes of the full first
  // undistributed level; all-gather the equal chunks (the top boundary plane stays 0).
  mg_status allgather_level(int l, T* buf) {
    const Level& L = s->lv[l];
    if (!comm_active(s)) return MG_OK;
    const size_t ps = (size_t)L.g.pstride;
    const size_t chunk = (size_t)(s->pt.n[l] / s->pt.P) * ps;
    return launch(s, st, K_ALLGATHER, l, (double)chunk * s->pt.P * sizeof(T),
                  [&] { return comm_allgather(s, buf, chunk * sizeof(T), st); });
  }

  // one sweep; zero_in: the iterate is known to be 0 (first sweep after V_H(0,...))
  // bpart != nullptr (3D RBGS marching level, not distributed): also write the black nodes'
  // residual partials of the sweep's output there (pm::SN_OUT_BLACK; the split norm)
  mg_status smooth(int l, T*& cur, T*& other, const T* f, bool zero_in = false, double* bpart = nullptr) {
    const Level& L = s->lv[l];
    if (bpart) {
      T* in = cur;
      T* out = other;
      mg_status r = launch(s, st, K_SWEEP_RBGS, l, 3 * w(l), [&] {
        int nb = 0;
        cudaError_t e = pm::launch_sweep<T>(L.g, coef(l), true, in, f, out, false, st, bpart, &nb, nullptr, nullptr,
                                            pm::SN_OUT_BLACK);
        return (e == cudaSuccess && nb != black_items()) ? cudaErrorInvalidValue : e;
      });
      std::swap(cur, other);
      return r;
    }
    if (pm(l)) {
      const bool rb = s->cfg.smoother == MG_RBGS;
      T* in = cur;
      T* out = other;
      const Kind kind = rb ? K_SWEEP_RBGS : K_SWEEP_JACOBI;
      const int B = rb ? 2 : 1;  // planes next to the slab faces that read halo planes
      auto sweep_range = [&](int lo, int hi) {
        Geom gr = L.g;
        gr.p_lo = lo;
        gr.p_hi = hi;
        return launch(s, st, kind, l, (zero_in ? 2 : 3) * w(l) * (hi - lo) / (L.g.p_hi - L.g.p_lo), [&] {
          return pm::launch_sweep<T>(gr, coef(l), rb, zero_in ? nullptr : in, f, out, zero_in, st);
        });
      };
      mg_status r;
      if (!zero_in && L.dist && L.g.p_hi - L.g.p_lo >= 2 * B + 8) {
        // slab: the halo exchange runs on the comm stream while the interior planes, which
        // read no halo, are swept; then the B planes next to each face.  The
        // plane ranges split the same per-plane arithmetic: bitwise identical to one launch.
        const int lo = L.g.p_lo, hi = L.g.p_hi;
        if (comm_active(s)) {
          cudaError_t e = cudaEventRecord(s->ev_fork, st);
          if (e == cudaSuccess) e = cudaStreamWaitEvent(s->comm_stream, s->ev_fork, 0);
          if (e != cudaSuccess) return cuda_fail(s, e, "halo fork");
          if ((r = exchange_on(l, in, B, s->comm_stream)) != MG_OK) return r;
          e = cudaEventRecord(s->ev_join, s->comm_stream);
          if (e != cudaSuccess) return cuda_fail(s, e, "halo join");
        }
        if ((r = sweep_range(lo + B, hi - B)) != MG_OK) return r;
        if (comm_active(s)) {
          cudaError_t e = cudaStreamWaitEvent(st, s->ev_join, 0);
          if (e != cudaSuccess) return cuda_fail(s, e, "halo join");
        }
        if ((r = sweep_range(lo, lo + B)) != MG_OK || (r = sweep_range(hi - B, hi)) != MG_OK) return r;
        std::swap(cur, other);
        return MG_OK;
      }
      if (!zero_in && (r = exchange(l, cur, B)) != MG_OK) return r;
      r = sweep_range(L.g.p_lo, L.g.p_hi);
      std::swap(cur, other);
      return r;
    }
    if (zero_in) {
      mg_status r = memset0(l, cur);
      if (r != MG_OK) return r;
    }
    if (s->cfg.smoother == MG_JACOBI) {
      mg_status r = exchange(l, cur, 1);
      if (r != MG_OK) return r;
      r = launch(s, st, K_JACOBI, l, 3 * w(l), [&] { return launch_jacobi<T>(L.g, coef(l), cur, f, other, st); });
      std::swap(cur, other);
      return r;
    }
    if (s->cfg.smoother == MG_GS_LEX) {  // one launch per hyperplane (nranks == 1)
      const int a = gs_lex_smin(L.g), b = gs_lex_smax(L.g);
      T* u = cur;
      for (int hp = a; hp <= b; hp++) {
        mg_status r = launch(s, st, K_GS_LEX, l, 3 * w(l) / (b - a + 1),
                             [&] { return launch_gs_lex_plane<T>(L.g, coef(l), u, f, hp, st); });
        if (r != MG_OK) return r;
      }
      return MG_OK;
    }
    for (int colour = 0; colour < 2; colour++) {
      mg_status r = exchange(l, cur, 1);
      if (r != MG_OK) return r;
      r = launch(s, st, K_RBGS_COLOUR, l, 3 * w(l),
                           [&] { return launch_rbgs_colour<T>(L.g, coef(l), cur, f, colour, st); });
      if (r != MG_OK) return r;
    }
    return MG_OK;
  }

  // n sweeps; 2D plane-marching Jacobi levels (not slab-distributed) run them K at a time in
  // one pass (k_jacobi2d_k: K = 3 in FP32, 2 in FP64), bitwise equal to n single sweeps
  // 2D omega-Jacobi on a marching level: n sweeps run as passes of up to 3 (FP32) / 2 (FP64)
  // fused sweeps (pm2::launch_jacobi_k, temporal blocking; bitwise equal to single sweeps)
  bool kfusable(int l) const {
    const bool off = s->cfg.flags & MG_FLAG_NO_KFUSE;
    const Level& L = s->lv[l];
    return !off && pm(l) && !L.g.three_d && s->cfg.smoother == MG_JACOBI && !L.dist;
  }
  int passes(int l, int n) const {
    const int kmax = sizeof(T) == 4 ? 3 : 2;
    return kfusable(l) ? (n + kmax - 1) / kmax : n;
  }

  // rr_fc != nullptr: the LAST pass also writes the restriction of its result's residual
  // into rr_fc (level l+1) when it can (rr_last(l, n)); the caller skips its own then
  mg_status smooth_n(int l, T*& cur, T*& other, const T* f, int n, bool zero_in, T* rr_fc = nullptr,
                     double* bpart = nullptr) {
    const Level& L = s->lv[l];
    const int p = passes(l, n);
    mg_status r = MG_OK;
    if (bpart) {  // the split norm's black partials from the last sweep (single sweeps: not kfusable)
      for (int k = 0; k < n; k++)
        if ((r = smooth(l, cur, other, f, zero_in && k == 0, k == n - 1 ? bpart : nullptr)) != MG_OK) return r;
      return r;
    }
    for (int k = 0, i = 0; k < n; i++) {
      const int K = n / p + (i < n % p ? 1 : 0);
      if (K >= 2) {
        T* in = cur;
        T* out = other;
        const bool z = zero_in && k == 0;
        T* fcl = (rr_fc && k + K == n) ? rr_fc : nullptr;
        const Geom gcg = s->lv[l + (l + 1 < s->L ? 1 : 0)].g;
        if ((r = launch(s, st, fcl ? K_SWEEP_RR_K : K_SWEEP_JACOBI_K, l,
                        (z ? 2 : 3) * w(l) + (fcl ? w(l + 1) : 0.0), [&] {
                          return pm2::launch_jacobi_k<T>(L.g, coef(l), K, z ? nullptr : in, f, out, z, st, nullptr,
                                                         nullptr, nullptr, fcl ? &gcg : nullptr, fcl);
                        })) != MG_OK)
          return r;
        std::swap(cur, other);
      } else if ((r = smooth(l, cur, other, f, zero_in && k == 0)) != MG_OK) {
        return r;
      }
      k += K;
    }
    return r;
  }

  mg_status memset0(int l, T* p) {
    return launch(s, st, K_MEMSET, l, w(l),
                  [&] { return cudaMemsetAsync(p, 0, s->lv[l].elems * sizeof(T), st); });
  }

  mg_status coarse(T* e, const T* f, T*& cur, T*& other) {
    int l = s->L - 1;
    const Level& L = s->lv[l];
    if (s->cfg.coarse == MG_COARSE_SWEEPS) {
      for (int k = 0; k < s->cfg.ncoarse; k++) {
        mg_status r = smooth(l, cur, other, f);
        if (r != MG_OK) return r;
      }
      return MG_OK;
    }
    return launch(s, st, K_COARSE_DIRECT, l, 2 * w(l), [&] {
      return launch_coarse_direct<T>(L.g, L.D, s->d_chol, s->m_coarse, f, e, s->d_work, st);
    });
  }

  // The cycle can be split into a HEAD (boundary refresh, f halo, first pre-sweep of
  // level 0 with the residual norm of its input accumulated on the fly) and a TAIL
  // (the rest).  mg_solve pipelines tail(k) + head(k+1): the norm after cycle k is
  // computed by the next cycle's first sweep, which reads u and f anyway.
  bool can_split() const { return s->L > 1 && s->cfg.nu1 >= 1 && pm(0) && tail_level() > 0; }
  // The split norm: with RBGS on a 3D marching level 0 held whole by this rank,
  // the tail's last level-0 post-sweep writes the black nodes' residual partials of the new
  // iterate (pm::SN_OUT_BLACK) into d_partial[0, black_items()), and the next head adds only
  // the red nodes' residuals of its input (pm::SN_INPUT_RED) behind them.
  bool split_norm() const {
    const Level& L = s->lv[0];
    return can_split() && s->cfg.smoother == MG_RBGS && L.g.three_d && !L.dist && s->cfg.nu2 >= 1 &&
           !(fuse_prolong(0) && s->cfg.nu2 == 1);
  }
  int black_items() const { return pm::sweep_items<T>(s->lv[0].g, true); }
  // the prolongation + correction of level l rides on its first post-sweep (3D marching levels;
  // measured C3 FP64 3.52 -> 3.31 ms); MG_FLAG_SEPARATE_PROLONG keeps its own pass
  bool fuse_prolong(int l) const {
    return pm(l) && s->lv[l].g.three_d && s->cfg.nu2 >= 1 && l + 1 < s->L && !(s->cfg.flags & MG_FLAG_SEPARATE_PROLONG);
  }

  mg_status cycle_start(T* u0, const T* f0) {
    const bool jac = s->cfg.smoother == MG_JACOBI;
    mg_status r;
    // ping-pong partners: t's boundary must hold u's Dirichlet data
    if ((jac || pm(0)) && (s->cfg.nu1 + s->cfg.nu2 > 0 || s->L == 1)) {
      r = launch(s, st, K_COPY_BOUNDARY, 0, 0,
                 [&] { return launch_copy_boundary<T>(s->lv[0].g, u0, (T*)s->lv[0].t, st); });
      if (r != MG_OK) return r;
    }
    // f is constant during the cycle: one halo exchange of level 0 (caller halo planes are scratch)
    return exchange(0, const_cast<T*>(f0), 1);
  }

  // head: cycle_start + the first level-0 sweep u0 -> t0 + ||f - A u0|| into out_dev
  // refresh = false: a later head of the same solve — the ping-pong partner's boundary and
  // f's halo planes still hold what the first head wrote (no kernel writes boundary nodes,
  // f is constant during the solve)
  mg_status head(T* u0, const T* f0, double* out_dev, bool refresh = true) {
    mg_status r = refresh ? cycle_start(u0, f0) : MG_OK;
    if (r != MG_OK) return r;
    if ((r = exchange(0, u0, s->cfg.smoother == MG_RBGS ? 2 : 1)) != MG_OK) return r;
    const Level& L = s->lv[0];
    const bool rb = s->cfg.smoother == MG_RBGS;
    int np = 0;
    T* t0 = (T*)L.t;
    const int hk = head_sweeps();
    if (hk > 1) {  // fused Jacobi passes: the head is the first pass, up to 3 sweeps
      const bool rr = head_rr();  // ... and, running every pre-sweep, the level-0 restriction
      T* fc = rr ? (T*)s->lv[1].f : nullptr;
      const Geom gcg = s->lv[s->L > 1 ? 1 : 0].g;
      if ((r = launch(s, st, K_SWEEP_NORM_K, 0, 3 * w(0) + (rr ? w(1) : 0.0), [&] {
             return pm2::launch_jacobi_k<T>(L.g, coef(0), hk, u0, f0, t0, false, st, s->d_partial, &np, nullptr,
                                            rr ? &gcg : nullptr, fc);
           })) != MG_OK)
        return r;
      return norm_finish(0, np, out_dev);
    }
    if (!refresh && split_norm()) {  // a later head: the previous tail wrote the black partials
      const int nb = black_items();
      if ((r = launch(s, st, K_SWEEP_NORM, 0, 3 * w(0), [&] {
             return pm::launch_sweep<T>(L.g, coef(0), rb, u0, f0, t0, false, st, s->d_partial + nb, &np, nullptr,
                                        nullptr, pm::SN_INPUT_RED);
           })) != MG_OK)
        return r;
      return norm_finish(0, nb + np, out_dev);
    }
    if ((r = launch(s, st, K_SWEEP_NORM, 0, 3 * w(0), [&] {
           return pm::launch_sweep<T>(L.g, coef(0), rb, u0, f0, t0, false, st, s->d_partial, &np);
         })) != MG_OK)
      return r;
    return norm_finish(0, np, out_dev);
  }

  // sweeps in the first of the passes(l, n) passes (smooth_n's split); 1 when not fusable
  int first_k(int l, int n) const {
    const int p = passes(l, n);
    return p > 0 ? n / p + (n % p ? 1 : 0) : 0;
  }
  // the last of the passes of n pre-sweeps on level l carries the residual + restriction
  bool rr_last(int l, int n) const {
    if (!kfusable(l) || n < 2 || l + 1 >= s->L || s->lv[l + 1].dist || (s->pt.slab && l + 1 == s->pt.la)) return false;
    const int p = passes(l, n);
    return pm2::rr_fusable<T>(n / p);  // the last pass has n / p sweeps
  }
  // the solve's head carries the level-0 residual + restriction (it runs every pre-sweep)
  bool head_rr() const { return kfusable(0) && head_sweeps() == s->cfg.nu1 && rr_last(0, s->cfg.nu1); }
  // level-0 pre-sweeps the head runs: the first fused pass, else one sweep
  int head_sweeps() const { return kfusable(0) ? first_k(0, s->cfg.nu1) : 1; }

  mg_status vcycle(T* u0, const T* f0) { return vcycle_impl(u0, f0, false); }
  // a cycle and the residual norm of its result into out_dev: one launch when the whole
  // cycle is the tail (C1-sized grids), else the cycle followed by norm()
  mg_status cycle_norm(T* u0, const T* f0, double* out_dev) {
    if (tail_level() == 0) return vcycle_impl(u0, f0, false, out_dev);
    const mg_status r = vcycle_impl(u0, f0, false);
    return r != MG_OK ? r : norm(0, u0, f0, out_dev);
  }
  mg_status tail(T* u0, const T* f0) { return vcycle_impl(u0, f0, true); }

  // after_head: the head already ran (first level-0 sweep result is in t0)
  // norm_out (lt = 0 only): the whole-cycle tail also writes ||f - A u|| of its result there
  mg_status vcycle_impl(T* u0, const T* f0, bool after_head, double* norm_out = nullptr) {
    const int Lv = s->L;
    std::vector<T*> cur(Lv), oth(Lv);
    mg_status r;
    const int lt = tail_level();
    if (lt == 0) return run_tail(0, u0, f0, norm_out);  // small grid: the whole cycle in one launch
    if (!after_head && (r = cycle_start(u0, f0)) != MG_OK) return r;
    for (int l = 0; l < Lv; l++) {
      cur[l] = l == 0 ? u0 : (T*)s->lv[l].u;
      oth[l] = (T*)s->lv[l].t;
    }
    if (after_head) std::swap(cur[0], oth[0]);
    const bool bnorm = after_head && split_norm();  // this tail writes the split norm's black partials
    if (Lv == 1) {
      // single-level hierarchy: solve in correction form (honours Dirichlet data)
      if (s->cfg.coarse == MG_COARSE_SWEEPS) {
        r = coarse(nullptr, f0, cur[0], oth[0]);
        if (r != MG_OK) return r;
      } else {
        const Level& L = s->lv[0];
        T* res = (T*)L.r;
        T* e = (T*)L.t;
        if ((r = launch(s, st, K_RESIDUAL, 0, 3 * w(0),
                        [&] { return launch_residual<T>(L.g, coef(0), u0, f0, res, st); })) != MG_OK)
          return r;
        if ((r = coarse(e, res, cur[0], oth[0])) != MG_OK) return r;
        if ((r = launch(s, st, K_ADD, 0, 3 * w(0), [&] {
               k_add_interior<T><<<rows_grid(L.g), dim3(128, 2), 0, st>>>(L.g, e, u0);
               return cudaGetLastError();
             })) != MG_OK)
          return r;
      }
    } else {
      // ---- descend: pre-smooth, residual, restrict (Alg. 1 lines 3-5)
      for (int l = 0; l < Lv - 1 && l < lt; l++) {
        const Level& L = s->lv[l];
        const T* f = l == 0 ? f0 : (const T*)L.f;
        // V_H(0, ...): the zero guess is folded into the first sweep (bitwise identical)
        if (l > 0 && s->cfg.nu1 == 0 && (r = memset0(l, cur[l])) != MG_OK) return r;
        T* fc = (T*)s->lv[l + 1].f;
        bool rr_done = false;  // the residual + restriction rode on the last pre-smoothing pass
        {
          const int k0 = (after_head && l == 0) ? head_sweeps() : 0;
          const int n = s->cfg.nu1 - k0;
          if (k0 > 0 && n == 0) {
            rr_done = head_rr();  // the head pass carried it
          } else {
            rr_done = rr_last(l, n);
          }
          if ((r = smooth_n(l, cur[l], oth[l], f, n, l > 0 && k0 == 0, (rr_done && n > 0) ? fc : nullptr)) != MG_OK)
            return r;
        }
        T* res = (T*)L.r;
        const Level& C = s->lv[l + 1];
        // coarse planes this rank produces: all of a distributed or single-GPU level, its own
        // chunk of the first agglomerated level
        const Geom gcw = (s->pt.slab && l + 1 == s->pt.la) ? C.gown : C.g;
        if (rr_done) {
          // done by the pass
        } else if (pm(l)) {
          if ((r = exchange(l, cur[l], 2)) != MG_OK) return r;
          const T* uc = cur[l];
          if ((r = launch(s, st, K_RESID_RESTRICT, l, 2 * w(l) + w(l + 1), [&] {
                 return pm::launch_resid_restrict<T>(L.g, gcw, coef(l), uc, f, fc, st);
               })) != MG_OK)
            return r;
        } else {
          if ((r = exchange(l, cur[l], 1)) != MG_OK) return r;
          if ((r = launch(s, st, K_RESIDUAL, l, 3 * w(l),
                          [&] { return launch_residual<T>(L.g, coef(l), cur[l], f, res, st); })) != MG_OK)
            return r;
          if ((r = exchange(l, res, 1)) != MG_OK) return r;
          if ((r = launch(s, st, K_RESTRICT, l, w(l) + w(l + 1),
                          [&] { return launch_restrict<T>(L.g, gcw, res, fc, st); })) != MG_OK)
            return r;
        }
        if (C.dist) {
          if ((r = exchange(l + 1, fc, 1)) != MG_OK) return r;
        } else if (s->pt.slab && l + 1 == s->pt.la) {
          if ((r = allgather_level(l + 1, fc)) != MG_OK) return r;
        }
      }
      if (lt < Lv) {
        // ---- levels lt..L-1: V_lt(0, f_lt) in one single-CTA launch (kernels_tail.cu)
        if ((r = run_tail(lt, (T*)s->lv[lt].u, (const T*)s->lv[lt].f)) != MG_OK) return r;
        cur[lt] = (T*)s->lv[lt].u;
      } else {
        // ---- coarsest level (Alg. 1 line 2)
        int l = Lv - 1;
        if (s->cfg.coarse == MG_COARSE_SWEEPS && (r = memset0(l, cur[l])) != MG_OK) return r;
        if ((r = coarse(cur[l], (const T*)s->lv[l].f, cur[l], oth[l])) != MG_OK) return r;
      }
      // ---- ascend: prolongate + correct, post-smooth (Alg. 1 lines 6-7)
      for (int l = (lt < Lv ? lt : Lv - 1) - 1; l >= 0; l--) {
        const Level& L = s->lv[l];
        const T* f = l == 0 ? f0 : (const T*)L.f;
        // e_H neighbour planes (slabs); the fused first post-sweep also corrects the u halo planes,
        // whose top one (odd, above the slab) reads the second coarse plane above
        if ((r = exchange(l + 1, cur[l + 1], fuse_prolong(l) ? 2 : 1)) != MG_OK) return r;
        const T* e = cur[l + 1];
        const bool pml = pm(l);
        if (fuse_prolong(l)) {
          // prolongation + correction fused into the first post-sweep: u + P e is formed in
          // shared memory, only S(u + P e) is written
          const bool rb = s->cfg.smoother == MG_RBGS;
          if ((r = exchange(l, cur[l], rb ? 2 : 1)) != MG_OK) return r;
          T* in = cur[l];
          T* out = oth[l];
          const Geom gcg = s->lv[l + 1].g;
          if ((r = launch(s, st, K_SWEEP_CORR, l, (3 + 1.0 / (1 << s->cfg.dim)) * w(l), [&] {
                 return pm::launch_sweep<T>(L.g, coef(l), rb, in, f, out, false, st, nullptr, nullptr, e, &gcg);
               })) != MG_OK)
            return r;
          std::swap(cur[l], oth[l]);
          for (int k = 1; k < s->cfg.nu2; k++)
            if ((r = smooth(l, cur[l], oth[l], f, false,
                            (bnorm && l == 0 && k == s->cfg.nu2 - 1) ? s->d_partial : nullptr)) != MG_OK)
              return r;
          continue;
        }
        // level 0: the ping-pong buffers swap once per pass; when fused passes change the
        // parity of the sweep count, the prolongation writes out of place (same traffic) so
        // the cycle still ends in u without a copy-back
        const int hk = after_head ? head_sweeps() : 0, n0 = s->cfg.nu1 - hk;
        const bool flip = l == 0 && kfusable(0) &&
                          (((hk ? 1 : 0) + passes(0, n0) + passes(0, s->cfg.nu2) - s->cfg.nu1 - s->cfg.nu2) & 1);
        const int k1 = first_k(l, s->cfg.nu2);
        if (kfusable(l) && !flip && k1 >= 2) {
          // prolongation + correction fused into the first post-smoothing pass: u + P e is
          // formed in registers, only the pass's result is written (cur[l] is not modified)
          const T* in = cur[l];
          T* out = oth[l];
          const Geom gcg = s->lv[l + 1].g;
          if ((r = launch(s, st, K_PROLONG_JACOBI_K, l, 3 * w(l) + w(l + 1), [&] {
                 return pm2::launch_jacobi_k<T>(L.g, coef(l), k1, in, f, out, false, st, nullptr, nullptr, e, &gcg);
               })) != MG_OK)
            return r;
          std::swap(cur[l], oth[l]);
          if ((r = smooth_n(l, cur[l], oth[l], f, s->cfg.nu2 - k1, false)) != MG_OK) return r;
          continue;
        }
        if ((r = launch(s, st, K_PROLONG, l, 2 * w(l) + w(l + 1), [&] {
               return flip ? pm2::launch_prolong<T>(L.g, s->lv[l + 1].g, e, cur[l], oth[l], st)
                      : pml ? pm::launch_prolong<T>(L.g, s->lv[l + 1].g, e, cur[l], st)
                            : launch_prolong_correct<T>(L.g, s->lv[l + 1].g, e, cur[l], st);
             })) != MG_OK)
          return r;
        if (flip) std::swap(cur[l], oth[l]);
        if ((r = smooth_n(l, cur[l], oth[l], f, s->cfg.nu2, false, nullptr, (bnorm && l == 0) ? s->d_partial : nullptr)) !=
            MG_OK)
          return r;
      }
    }
    if (cur[0] != u0) {
      const Level& L = s->lv[0];
      T* src = cur[0];
      if ((r = launch(s, st, K_COPY_INTERIOR, 0, 2 * w(0), [&] {
             k_copy_interior<T><<<rows_grid(L.g), dim3(128, 2), 0, st>>>(L.g, src, u0);
             return cudaGetLastError();
           })) != MG_OK)
        return r;
    }
    return MG_OK;
  }

  mg_status norm(int l, const T* u, const T* f, double* out_dev) {
    const Level& L = s->lv[l];
    // whole-cycle tails evaluate the norm with the tail's own distribution and order (the
    // fused norm of cycle_norm is then bitwise this one)
    if (l == 0 && tail_level() == 0) return run_tail(0, const_cast<T*>(u), f, out_dev, true);
    int np = norm_num_partials<T>(L.g);
    const bool pml = pm(l);
    // slabs: the residual of the owned face planes reads the neighbours' planes, and the
    // cycle's last sweep left u's halo planes stale (halos are library scratch)
    mg_status r = exchange(l, const_cast<T*>(u), 1);
    if (r != MG_OK) return r;
    r = launch(s, st, K_NORM_PARTIAL, l, 2 * w(l), [&] {
      return pml ? pm::launch_norm<T>(L.g, coef(l), u, f, s->d_partial, &np, st)
                 : launch_norm_partial<T>(L.g, coef(l), u, f, s->d_partial, st);
    });
    if (r != MG_OK) return r;
    return norm_finish(l, np, out_dev);
  }

  // partials (np doubles in d_partial) -> ||r|| in out_dev (rank sums all-gathered on slabs)
  mg_status norm_finish(int l, int np, double* out_dev) {
    const Level& L = s->lv[l];
    mg_status r;
    if (!L.dist)
      return launch(s, st, K_NORM_FINAL, l, 8.0 * np,
                    [&] { return launch_norm_final(s->d_partial, np, out_dev, st); });
    // slabs: per-rank sum of r^2 -> all-gather -> summed in rank order (identical on every rank)
    double* mine = s->d_rank_sums + s->pt.rank;
    if ((r = launch(s, st, K_NORM_FINAL, l, 8.0 * np,
                    [&] { return launch_norm_final(s->d_partial, np, mine, st, false); })) != MG_OK)
      return r;
    if (comm_active(s) && (r = launch(s, st, K_ALLGATHER, l, 8.0 * s->pt.P, [&] {
                             return comm_allgather(s, s->d_rank_sums, sizeof(double), st);
                           })) != MG_OK)
      return r;
    return launch(s, st, K_NORM_FINAL, l, 8.0 * s->pt.P,
                  [&] { return launch_norm_combine(s->d_rank_sums, s->pt.P, out_dev, st); });
  }
};

template <>
const Coef<double>& Exec<double>::coef(int l) const {
  return s->lv[l].c64;
}
template <>
const Coef<float>& Exec<float>::coef(int l) const {
  return s->lv[l].c32;
}


// ================================================================ complex diffusion (FAS)
// One implicit-Euler step of nonlinear complex diffusion on a cell-centred grid, FAS
// V-cycle with lagged diffusivity (oracle/cd_oracle.c), kernels in
// kernels_cd.cu.  Level l: cells n_d >> l, h_l = 2^l h, w_d = tau / h_{l,d}^2.
static bool is_cd(const mg_solver* s) { return s->cfg.problem == MG_PROBLEM_COMPLEX_DIFFUSION; }

static mg_status cd_build(mg_solver* s) {
  const mg_config& c = s->cfg;
  const int esz = (int)s->esz;
  const int64_t align = 128 / (2 * esz);  // complex elements per 128 B
  s->lv.resize(s->L);
  int np = 1;
  for (int l = 0; l < s->L; l++) {
    Level& L = s->lv[l];
    int64_t n[3];
    double w[3] = {0, 0, 0};
    for (int d = 0; d < 3; d++) {
      n[d] = d < c.dim ? c.nodes[d] >> l : 1;
      const double h0 = c.h[d] > 0.0 ? c.h[d] : (d < c.dim ? 1.0 / (double)c.nodes[d] : 0.0);
      const double h = std::ldexp(h0, l);
      if (d < c.dim) w[d] = c.tau / (h * h);
    }
    Geom& g = L.g;
    g.three_d = c.dim == 3;
    g.nx = (int)n[0];
    g.ny = c.dim == 3 ? (int)n[1] : 0;
    g.nz = c.dim == 3 ? (int)n[2] : (int)n[1];
    g.rows = c.dim == 3 ? g.ny : 1;
    g.planes = g.nz;
    g.p_lo = 0;
    g.p_hi = g.nz;
    g.p_glob0 = 0;
    g.pitch = (g.nx + align - 1) / align * align;
    g.pstride = g.pitch * g.rows;
    L.gown = g;
    // coefficients in double, cast once: x, in-plane y (3D), plane axis (3D z, 2D y)
    const double wx = w[0], wy = c.dim == 3 ? w[1] : 0.0, wz = c.dim == 3 ? w[2] : w[1];
    const double kth = c.kappa * c.theta, ct = std::cos(c.theta), sn = std::sin(c.theta);
    L.cd64 = CdCoef<double>{{wx, wy, wz}, c.omega, kth, ct, sn};
    L.cd32 = CdCoef<float>{{(float)wx, (float)wy, (float)wz}, (float)c.omega, (float)kth, (float)ct, (float)sn};
    L.shape[0] = g.planes;
    L.shape[1] = g.rows;
    L.shape[2] = g.pitch;
    L.elems = (size_t)L.shape[0] * L.shape[1] * L.shape[2];
    const size_t bytes = L.elems * 2 * esz;
    void** bufs[5] = {&L.u, &L.f, &L.uh, &L.gd, &L.t};
    for (int b = 0; b < 5; b++) {
      if (l == 0 && (b < 3)) continue;  // level 0 u, f are the caller's; no u^ on level 0
      if (cudaMalloc(bufs[b], bytes) != cudaSuccess) {
        cudaGetLastError();
        return plan_fail(s, MG_ERR_OOM, "device allocation of level buffers failed");
      }
      cudaError_t e = cudaMemset(*bufs[b], 0, bytes);
      if (e != cudaSuccess) return cuda_fail(s, e, "cudaMemset");
    }
    int a = cd_norm_partials(g);
    if (a > np) np = a;
    if (cd2d_supported(g)) {
      a = esz == 8 ? cd2d_norm_partials<double>(g) : cd2d_norm_partials<float>(g);
      if (a > np) np = a;
      a = esz == 8 ? cd2d_kpartials<double>(g) : cd2d_kpartials<float>(g);  // fused head pass
      if (a > np) np = a;
    }
    if (cd3d_supported(g)) {
      a = esz == 8 ? cd3d_norm_partials<double>(g) : cd3d_norm_partials<float>(g);
      if (a > np) np = a;
    }
  }
  return alloc_common(s, np);
}

template <typename T>
struct CdExec {
  mg_solver* s;
  cudaStream_t st;
  const CdCoef<T>& cc(int l) const;
  double cw(int l) const {  // one complex word per cell of level l
    const Geom& g = s->lv[l].g;
    return (double)g.nx * (g.three_d ? g.ny : 1) * g.nz * 2.0 * sizeof(T);
  }
  const Geom& G(int l) const { return s->lv[l].g; }
  T* gd(int l) const { return (T*)s->lv[l].gd; }

  mg_status gfield(int l, const T* u) {
    return launch(s, st, K_CD_GFIELD, l, 2 * cw(l), [&] { return cd_launch_gfield<T>(G(l), cc(l), u, gd(l), st); });
  }
  // one sweep with the frozen g of level l; Jacobi ping-pongs cur <-> oth
  mg_status smooth(int l, T*& cur, T*& oth, const T* f) {
    if (s->cfg.smoother == MG_JACOBI) {
      T* in = cur;
      T* out = oth;
      const bool opt = !(s->cfg.flags & MG_FLAG_BASELINE);
      const bool m2 = opt && cd2d_supported(G(l)), m3 = opt && cd3d_supported(G(l));
      mg_status r = launch(s, st, K_CD_JACOBI, l, 4 * cw(l), [&] {
        return m2   ? cd2d_launch_jacobi<T>(G(l), cc(l), gd(l), in, f, out, st)
               : m3 ? cd3d_launch_jacobi<T>(G(l), cc(l), gd(l), in, f, out, st)
                    : cd_launch_jacobi<T>(G(l), cc(l), gd(l), in, f, out, st);
      });
      std::swap(cur, oth);
      return r;
    }
    for (int colour = 0; colour < 2; colour++) {
      T* u = cur;
      mg_status r = launch(s, st, K_CD_RBGS, l, 2.5 * cw(l),
                           [&] { return cd_launch_rbgs<T>(G(l), cc(l), gd(l), u, f, colour, st); });
      if (r != MG_OK) return r;
    }
    return MG_OK;
  }
  // Jacobi on a 2D marching level: n sweeps as passes of up to kmax fused sweeps
  // (cd2d_launch_jacobi_k, temporal blocking; bitwise equal to single sweeps).  Measured on
  // CD2: the complex sweep is already issue-bound alone, so K = 2 passes
  // are SLOWER than two single sweeps (0.37 vs 0.25 ms at 4096^2 FP32); kmax defaults to 1
  // and the fused kernel serves the solve's head (first sweep + the input's norm in one
  // pass).  MG_FLAG_CD_KFUSE re-enables multi-sweep passes (3 FP32 / 2 FP64).
  bool kfusable(int l) const {
    const bool off = s->cfg.flags & MG_FLAG_NO_KFUSE;
    return !off && s->cfg.smoother == MG_JACOBI && !(s->cfg.flags & MG_FLAG_BASELINE) && cd2d_supported(G(l));
  }
  int kmax() const {
    return (s->cfg.flags & MG_FLAG_CD_KFUSE) ? (sizeof(T) == 4 ? 3 : 2) : 1;
  }
  int passes(int l, int n) const { return kfusable(l) ? (n + kmax() - 1) / kmax() : n; }
  int first_k(int l, int n) const {
    const int p = passes(l, n);
    return p > 0 ? n / p + (n % p ? 1 : 0) : 0;
  }
  // level-0 pre-sweeps the solve's head runs (its first pass, with the input's norm)
  int head_sweeps() const {
    return (kfusable(0) && s->L > 1 && tail_level() > 0 && s->cfg.nu1 >= 1) ? first_k(0, s->cfg.nu1) : 0;
  }
  // n sweeps in p passes (p = 0: passes(l, n))
  mg_status smooth_n(int l, T*& cur, T*& oth, const T* f, int n, int p = 0) {
    if (!kfusable(l)) {
      for (int k = 0; k < n; k++) {
        mg_status r = smooth(l, cur, oth, f);
        if (r != MG_OK) return r;
      }
      return MG_OK;
    }
    if (p <= 0) p = passes(l, n);
    for (int k = 0, i = 0; k < n; i++) {
      const int K = n / p + (i < n % p ? 1 : 0);
      T* in = cur;
      T* out = oth;
      mg_status r = K == 1 ? smooth(l, cur, oth, f) : launch(s, st, K_CD_JACOBI_K, l, 4 * cw(l), [&] {
        return cd2d_launch_jacobi_k<T>(G(l), cc(l), K, gd(l), in, f, out, st);
      });
      if (r != MG_OK) return r;
      if (K > 1) std::swap(cur, oth);
      k += K;
    }
    return MG_OK;
  }
  mg_status copy(int l, const T* src, T* dst) {
    const Geom& g = G(l);
    const size_t w = (size_t)g.nx * 2 * sizeof(T), p = (size_t)g.pitch * 2 * sizeof(T);
    return launch(s, st, K_CD_COPY, l, 2 * cw(l), [&] {
      return cudaMemcpy2DAsync(dst, p, src, p, w, (size_t)g.rows * g.planes, cudaMemcpyDeviceToDevice, st);
    });
  }
  // first level of the single-CTA coarse tail (kernels_cd.cu): <= kCdTailCells cells; L if none
  int tail_level() const {
    if (s->cfg.flags & MG_FLAG_BASELINE) return s->L;
    for (int l = 0; l < s->L; l++) {
      const Geom& g = G(l);
      if ((long long)g.nx * (g.three_d ? g.ny : 1) * g.nz <= kCdTailCells && s->L - l <= kCdTailMax) return l;
    }
    return s->L;
  }
  mg_status run_tail(int lt, std::vector<T*>& cur, std::vector<T*>& oth, const T* f_top, bool g_ready) {
    CdTail<T> P{};
    P.nl = s->L - lt;
    P.rbgs = s->cfg.smoother == MG_RBGS;
    P.nu1 = s->cfg.nu1;
    P.nu2 = s->cfg.nu2;
    P.ncoarse = s->cfg.ncoarse;
    P.g_ready = g_ready;
    double bytes = 0;
    for (int k = 0; k < P.nl; k++) {
      Level& L = s->lv[lt + k];
      P.g[k] = L.g;
      P.c[k] = cc(lt + k);
      P.u[k] = cur[lt + k];
      P.t[k] = oth[lt + k];
      P.f[k] = k == 0 ? const_cast<T*>(f_top) : (T*)L.f;
      P.uh[k] = (T*)L.uh;
      P.gd[k] = gd(lt + k);
      bytes += cw(lt + k) * (2 + 4.0 * (P.nu1 + P.nu2) + 10);
    }
    return launch(s, st, K_CD_TAIL, lt, bytes, [&] { return cd_launch_tail<T>(P, st); });
  }
  // FAS V-cycle at level l; g_ready: g of level l already built from cur[l]
  // skip: level-0 pre-sweeps the head already ran
  mg_status rec(int l, std::vector<T*>& cur, std::vector<T*>& oth, const T* f, bool g_ready, int skip = 0) {
    mg_status r;
    if (l == tail_level()) return run_tail(l, cur, oth, f, g_ready);  // the result lands in cur[l]
    if (!g_ready && (r = gfield(l, cur[l])) != MG_OK) return r;  // lagged diffusivity, frozen in the cycle
    if (l == s->L - 1) return smooth_n(l, cur[l], oth[l], f, s->cfg.ncoarse);
    if ((r = smooth_n(l, cur[l], oth[l], f, s->cfg.nu1 - skip)) != MG_OK) return r;
    Level& C = s->lv[l + 1];
    T* uh = (T*)C.uh;
    T* fc = (T*)C.f;
    const T* ul = cur[l];
    T* uc = cur[l + 1];
    // u^_H = R u_h, u_H = u^_H
    if ((r = launch(s, st, K_CD_RESTRICT, l, cw(l) + 2 * cw(l + 1),
                    [&] { return cd_launch_restrict<T>(G(l), G(l + 1), ul, uh, uc, st); })) != MG_OK)
      return r;
    if ((r = gfield(l + 1, uh)) != MG_OK) return r;  // coarse operator from the restricted lagged solution
    // f_H = A_H(u^_H) u^_H + R (f_h - A_h u_h)
    if ((r = launch(s, st, K_CD_FAS_RHS, l, 3 * cw(l) + 3 * cw(l + 1), [&] {
           return cd_launch_fas_rhs<T>(G(l), G(l + 1), cc(l), cc(l + 1), gd(l), ul, f, gd(l + 1), uh, fc, st);
         })) != MG_OK)
      return r;
    if ((r = rec(l + 1, cur, oth, fc, true)) != MG_OK) return r;
    // u_h += P (u_H - u^_H)
    const T* ucn = cur[l + 1];
    T* ulw = cur[l];
    if ((r = launch(s, st, K_CD_PROLONG, l, 2 * cw(l) + 2 * cw(l + 1),
                    [&] { return cd_launch_prolong<T>(G(l), G(l + 1), ucn, uh, ulw, st); })) != MG_OK)
      return r;
    // level 0: when fused passes change the ping-pong parity, one more post pass keeps the
    // result in u (no copy-back)
    int p2 = 0;
    if (l == 0 && kfusable(0)) {
      const int nu1 = s->cfg.nu1, nu2 = s->cfg.nu2;
      p2 = passes(0, nu2);
      if ((((skip ? 1 : 0) + passes(0, nu1 - skip) + p2 - nu1 - nu2) & 1) && p2 < nu2) p2++;
    }
    return smooth_n(l, cur[l], oth[l], f, s->cfg.nu2, p2);
  }
  // g_ready: lv[0].gd already holds g(u0) (the head computed it for the norm); after_head:
  // the head also ran the first level-0 pre-smoothing pass (u0 -> lv[0].t)
  mg_status vcycle(T* u0, const T* f0, bool g_ready = false, bool after_head = false) {
    std::vector<T*> cur(s->L), oth(s->L);
    for (int l = 0; l < s->L; l++) {
      cur[l] = l == 0 ? u0 : (T*)s->lv[l].u;
      oth[l] = (T*)s->lv[l].t;
    }
    const int hk = after_head ? head_sweeps() : 0;
    if (hk > 0) std::swap(cur[0], oth[0]);
    mg_status r = rec(0, cur, oth, f0, g_ready, hk);
    if (r != MG_OK) return r;
    if (cur[0] != u0) return copy(0, cur[0], u0);
    return MG_OK;
  }
  // pipelined driver loop (mg_solve): head = g(u_k) for the next cycle + ||f - A(g(u_k)) u_k||
  // from the stored field; tail = the cycle with g ready
  mg_status head(const T* u0, const T* f0, double* out_dev) {
    mg_status r = gfield(0, u0);
    if (r != MG_OK) return r;
    const int hk = head_sweeps();
    if (hk == 0) return norm(0, u0, f0, out_dev, gd(0));
    // the first pre-smoothing pass also accumulates ||f - A(g(u0)) u0||: one pass instead of two
    int np = 0;
    T* t0 = (T*)s->lv[0].t;
    if ((r = launch(s, st, K_CD_JACOBI_K_NORM, 0, 4 * cw(0), [&] {
           return cd2d_launch_jacobi_k<T>(G(0), cc(0), hk, gd(0), u0, f0, t0, st, s->d_partial, &np);
         })) != MG_OK)
      return r;
    return launch(s, st, K_NORM_FINAL, 0, 8.0 * np, [&] { return launch_norm_final(s->d_partial, np, out_dev, st); });
  }
  mg_status norm(int l, const T* u, const T* f, double* out_dev, const T* gstored = nullptr) {
    int np = 0;
    const bool opt = gstored && !(s->cfg.flags & MG_FLAG_BASELINE);
    const bool m2 = opt && cd2d_supported(G(l)), m3 = opt && cd3d_supported(G(l));
    mg_status r = launch(s, st, K_CD_NORM, l, (gstored ? 3 : 2) * cw(l), [&] {
      return m2   ? cd2d_launch_norm<T>(G(l), cc(l), gstored, u, f, s->d_partial, &np, st)
             : m3 ? cd3d_launch_norm<T>(G(l), cc(l), gstored, u, f, s->d_partial, &np, st)
                  : cd_launch_norm_partial<T>(G(l), cc(l), gstored, u, f, s->d_partial, &np, st);
    });
    if (r != MG_OK) return r;
    return launch(s, st, K_NORM_FINAL, l, 8.0 * np, [&] { return launch_norm_final(s->d_partial, np, out_dev, st); });
  }
  mg_status op_smooth(int l, const T* uin, const T* f, T* uout) {
    mg_status r = gfield(l, uin);
    if (r != MG_OK) return r;
    if (s->cfg.smoother == MG_JACOBI) {
      T* dst = uin == uout ? (T*)s->lv[l].t : uout;
      if ((r = launch(s, st, K_CD_JACOBI, l, 4 * cw(l),
                      [&] { return cd_launch_jacobi<T>(G(l), cc(l), gd(l), uin, f, dst, st); })) != MG_OK)
        return r;
      return dst == uout ? MG_OK : copy(l, dst, uout);
    }
    if (uin != uout && (r = copy(l, uin, uout)) != MG_OK) return r;
    T* cur = uout;
    T* oth = nullptr;
    return smooth(l, cur, oth, f);
  }
  mg_status op_residual(int l, const T* u, const T* f, T* res) {
    mg_status r = gfield(l, u);
    if (r != MG_OK) return r;
    return launch(s, st, K_CD_RESIDUAL, l, 3 * cw(l),
                  [&] { return cd_launch_residual<T>(G(l), cc(l), gd(l), u, f, res, st); });
  }
};
template <>
const CdCoef<double>& CdExec<double>::cc(int l) const {
  return s->lv[l].cd64;
}
template <>
const CdCoef<float>& CdExec<float>::cc(int l) const {
  return s->lv[l].cd32;
}

template <typename T>
static mg_status cd_run_part_T(mg_solver* s, int part, T* u, const T* f, cudaStream_t st) {
  CdExec<T> x{s, st};
  switch (part) {
    case 1:
    case 4: return x.head(u, f, s->d_norm);
    case 2: return x.vcycle(u, f, true, true);
    case 3: return x.norm(0, u, f, s->d_norm);
    case 5: {
      const mg_status r = x.vcycle(u, f);
      return r != MG_OK ? r : x.norm(0, u, f, s->d_norm);
    }
    default: return x.vcycle(u, f);
  }
}
static mg_status cd_run_part(mg_solver* s, int part, void* u, const void* f, cudaStream_t st) {
  return s->esz == 8 ? cd_run_part_T<double>(s, part, (double*)u, (const double*)f, st)
                     : cd_run_part_T<float>(s, part, (float*)u, (const float*)f, st);
}

// ---------------------------------------------------------------- entry points
// part: 0 whole cycle, 1 head (first sweep + norm of the input into d_norm), 2 tail,
// 3 norm of (u, f) into d_norm, 4 head of a later cycle of the same solve (no refresh of the
// ping-pong partner's boundary or of f's halo planes), 5 whole cycle + norm of its result
// into d_norm (the unsplit driver loop's body), 6 the whole driver loop in one launch
// (plan_solve_in_tail; loop state in d_loop)
template <typename T>
static mg_status run_part(mg_solver* s, int part, void* u, const void* f, cudaStream_t st) {
  Exec<T> x{s, st};
  if (part == 1 || part == 4) return x.head((T*)u, (const T*)f, s->d_norm, part == 1);
  if (part == 2) return x.tail((T*)u, (const T*)f);
  if (part == 3) return x.norm(0, (const T*)u, (const T*)f, s->d_norm);
  if (part == 5) return x.cycle_norm((T*)u, (const T*)f, s->d_norm);
  if (part == 6) return x.solve_tail((T*)u, (const T*)f);
  return x.vcycle((T*)u, (const T*)f);
}

mg_status plan_run_part(mg_solver* s, int part, void* u, const void* f, cudaStream_t st) {
  s->launch_counter = 0;
  mg_status r = is_cd(s) ? cd_run_part(s, part, u, f, st)
                         : s->esz == 8 ? run_part<double>(s, part, u, f, st) : run_part<float>(s, part, u, f, st);
  // launches of one cycle: the whole cycle (5: with its norm), or head + tail of the pipelined split
  if (part == 0 || part == 5) s->launches_per_cycle = s->launch_counter;
  if (part == 1 || part == 4) s->head_launches = s->launch_counter;
  if (part == 2) s->tail_launches = s->launch_counter;
  if (part == 2 || part == 4) s->launches_per_cycle = s->head_launches + s->tail_launches;
  return r;
}

mg_status plan_run_vcycle(mg_solver* s, void* u, const void* f, cudaStream_t st) {
  return plan_run_part(s, 0, u, f, st);
}

bool plan_solve_in_tail(mg_solver* s) {
  if (is_cd(s) || comm_active(s)) return false;
  return s->esz == 8 ? Exec<double>{s, 0}.tail_level() == 0 : Exec<float>{s, 0}.tail_level() == 0;
}

bool plan_can_split(mg_solver* s) {
  if (is_cd(s)) return true;  // head = g(u_k) + norm from the stored field, tail = the cycle
  return s->esz == 8 ? Exec<double>{s, 0}.can_split() : Exec<float>{s, 0}.can_split();
}

mg_status plan_graph_part(mg_solver* s, int part, void* u, const void* f, cudaStream_t st) {
  if (s->loop && comm_active(s)) return loop_graph_part(s, part, u, f, st);  // one graph for the group
  auto key = std::make_tuple(u, f, part);
  auto it = s->graphs.find(key);
  if (it == s->graphs.end()) {
    cudaGraph_t graph;
    cudaError_t e = cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return cuda_fail(s, e, "cudaStreamBeginCapture");
    mg_status r = plan_run_part(s, part, u, f, s->cap_stream);
    e = cudaStreamEndCapture(s->cap_stream, &graph);
    if (r != MG_OK) return r;
    if (e != cudaSuccess) return cuda_fail(s, e, "cudaStreamEndCapture");
    cudaGraphExec_t exec;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(s, e, "cudaGraphInstantiate");
    if (s->graphs.size() >= 16) {  // bound the cache
      cudaGraphExecDestroy(s->graphs.begin()->second);
      s->graphs.erase(s->graphs.begin());
    }
    it = s->graphs.emplace(key, exec).first;
  }
  cudaError_t e = cudaGraphLaunch(it->second, st);
  if (e != cudaSuccess) return cuda_fail(s, e, "cudaGraphLaunch");
  return MG_OK;
}

mg_status plan_graph_vcycle(mg_solver* s, void* u, const void* f, cudaStream_t st) {
  return plan_graph_part(s, 0, u, f, st);
}

mg_status plan_norm(mg_solver* s, int level, const void* u, const void* f, double* out, cudaStream_t st, bool sync) {
  mg_status r = is_cd(s) ? (s->esz == 8 ? CdExec<double>{s, st}.norm(level, (const double*)u, (const double*)f, s->d_norm)
                                        : CdExec<float>{s, st}.norm(level, (const float*)u, (const float*)f, s->d_norm))
              : s->esz == 8 ? Exec<double>{s, st}.norm(level, (const double*)u, (const double*)f, s->d_norm)
                            : Exec<float>{s, st}.norm(level, (const float*)u, (const float*)f, s->d_norm);
  if (r != MG_OK) return r;
  cudaError_t e = cudaMemcpyAsync(s->h_norm, s->d_norm, sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) return cuda_fail(s, e, "norm readback");
  if (sync) {
    if ((r = plan_wait(s, st, "norm synchronise")) != MG_OK) return r;
    *out = *s->h_norm;
  }
  return MG_OK;
}

template <typename T>
static mg_status op_smooth_T(mg_solver* s, int l, const T* uin, const T* f, T* uout, cudaStream_t st) {
  Exec<T> x{s, st};
  const Level& L = s->lv[l];
  const bool pingpong = s->cfg.smoother == MG_JACOBI || x.pm(l);
  if (pingpong) {
    T* dst = uin == uout ? (T*)L.t : uout;  // in place: sweep into t, copy back
    mg_status r = launch(s, st, K_COPY_BOUNDARY, l, 0, [&] { return launch_copy_boundary<T>(L.g, uin, dst, st); });
    if (r != MG_OK) return r;
    T* cur = (T*)uin;
    T* oth = dst;
    if ((r = x.smooth(l, cur, oth, f)) != MG_OK) return r;
    if (dst == uout) return MG_OK;
    return launch(s, st, K_COPY_INTERIOR, l, 0, [&] {
      k_copy_interior<T><<<rows_grid(L.g), dim3(128, 2), 0, st>>>(L.g, dst, uout);
      return cudaGetLastError();
    });
  }
  if (uin != uout) {
    cudaError_t e = cudaMemcpyAsync(uout, uin, L.elems * sizeof(T), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_fail(s, e, "copy");
  }
  T* cur = uout;
  T* oth = (T*)L.t;
  return x.smooth(l, cur, oth, f);
}

mg_status plan_op_smooth(mg_solver* s, int l, const void* uin, const void* f, void* uout, cudaStream_t st) {
  if (is_cd(s))
    return s->esz == 8 ? CdExec<double>{s, st}.op_smooth(l, (const double*)uin, (const double*)f, (double*)uout)
                       : CdExec<float>{s, st}.op_smooth(l, (const float*)uin, (const float*)f, (float*)uout);
  if (s->esz == 8) return op_smooth_T<double>(s, l, (const double*)uin, (const double*)f, (double*)uout, st);
  return op_smooth_T<float>(s, l, (const float*)uin, (const float*)f, (float*)uout, st);
}

mg_status plan_op_residual(mg_solver* s, int l, const void* u, const void* f, void* r, cudaStream_t st) {
  if (is_cd(s))
    return s->esz == 8 ? CdExec<double>{s, st}.op_residual(l, (const double*)u, (const double*)f, (double*)r)
                       : CdExec<float>{s, st}.op_residual(l, (const float*)u, (const float*)f, (float*)r);
  const Level& L = s->lv[l];
  return launch(s, st, K_RESIDUAL, l, 0, [&] {
    return s->esz == 8 ? launch_residual<double>(L.g, L.c64, (const double*)u, (const double*)f, (double*)r, st)
                       : launch_residual<float>(L.g, L.c32, (const float*)u, (const float*)f, (float*)r, st);
  });
}

mg_status plan_op_restrict(mg_solver* s, int l, const void* r, void* fc, cudaStream_t st) {
  if (is_cd(s))
    return launch(s, st, K_CD_RESTRICT, l, 0, [&] {
      const Geom &gf = s->lv[l].g, &gc = s->lv[l + 1].g;
      return s->esz == 8 ? cd_launch_restrict<double>(gf, gc, (const double*)r, (double*)fc, nullptr, st)
                         : cd_launch_restrict<float>(gf, gc, (const float*)r, (float*)fc, nullptr, st);
    });
  const Level& F = s->lv[l];
  const Level& C = s->lv[l + 1];
  cudaError_t e = cudaMemsetAsync(fc, 0, C.elems * s->esz, st);
  if (e != cudaSuccess) return cuda_fail(s, e, "memset");
  return launch(s, st, K_RESTRICT, l, 0, [&] {
    return s->esz == 8 ? launch_restrict<double>(F.g, C.g, (const double*)r, (double*)fc, st)
                       : launch_restrict<float>(F.g, C.g, (const float*)r, (float*)fc, st);
  });
}

mg_status plan_op_prolong(mg_solver* s, int l, const void* e, void* u, cudaStream_t st) {
  if (is_cd(s))
    return launch(s, st, K_CD_PROLONG, l, 0, [&] {
      const Geom &gf = s->lv[l].g, &gc = s->lv[l + 1].g;
      return s->esz == 8 ? cd_launch_prolong<double>(gf, gc, (const double*)e, nullptr, (double*)u, st)
                         : cd_launch_prolong<float>(gf, gc, (const float*)e, nullptr, (float*)u, st);
    });
  const Level& F = s->lv[l];
  const Level& C = s->lv[l + 1];
  return launch(s, st, K_PROLONG, l, 0, [&] {
    return s->esz == 8 ? launch_prolong_correct<double>(F.g, C.g, (const double*)e, (double*)u, st)
                       : launch_prolong_correct<float>(F.g, C.g, (const float*)e, (float*)u, st);
  });
}

template <typename T>
static mg_status op_coarse_T(mg_solver* s, const T* f, T* e, cudaStream_t st) {
  Exec<T> x{s, st};
  int l = s->L - 1;
  cudaError_t ce = cudaMemsetAsync(e, 0, s->lv[l].elems * sizeof(T), st);
  if (ce != cudaSuccess) return cuda_fail(s, ce, "memset");
  T* cur = e;
  T* oth = (T*)s->lv[l].t;
  mg_status r = x.coarse(e, f, cur, oth);
  if (r != MG_OK) return r;
  if (cur != e) {
    ce = cudaMemcpyAsync(e, cur, s->lv[l].elems * sizeof(T), cudaMemcpyDeviceToDevice, st);
    if (ce != cudaSuccess) return cuda_fail(s, ce, "copy");
  }
  return MG_OK;
}

mg_status plan_op_coarse(mg_solver* s, const void* f, void* e, cudaStream_t st) {
  if (is_cd(s)) return plan_fail(s, MG_ERR_INVALID, "complex diffusion: the FAS coarsest level is ncoarse sweeps");
  if (s->esz == 8) return op_coarse_T<double>(s, (const double*)f, (double*)e, st);
  return op_coarse_T<float>(s, (const float*)f, (float*)e, st);
}

mg_status plan_workload_fill(mg_solver* s, void* dst, uint64_t seed, double lo, double hi, cudaStream_t st) {
  if (is_cd(s)) {
    const Geom& g = s->lv[0].g;
    cudaError_t e = s->esz == 8 ? cd_launch_fill<double>(g, (double*)dst, seed, lo, hi, st)
                                : cd_launch_fill<float>(g, (float*)dst, seed, lo, hi, st);
    if (e != cudaSuccess) return cuda_fail(s, e, "workload_fill");
    return MG_OK;
  }
  const Level& L = s->lv[0];
  cudaError_t e = s->esz == 8 ? launch_workload_fill<double>(L.g, seed, lo, hi, (double*)dst, st)
                              : launch_workload_fill<float>(L.g, seed, lo, hi, (float*)dst, st);
  if (e != cudaSuccess) return cuda_fail(s, e, "workload_fill");
  return MG_OK;
}

// ---------------------------------------------------------------- profiling
static void prof_drain(mg_solver* s) {
  if (s->prof.empty()) return;
  cudaDeviceSynchronize();
  for (auto& r : s->prof) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    char name[64];
    snprintf(name, sizeof name, "%s@L%d", kKindName[r.kind], r.level);
    ProfSum* sum = nullptr;
    for (auto& p : s->prof_done)
      if (p.name == name) sum = &p;
    if (!sum) {
      s->prof_done.push_back(ProfSum{name, 0, 0, 0});
      sum = &s->prof_done.back();
    }
    sum->ms += ms;
    sum->bytes += r.bytes;  // summed: launches of one kind can differ (zero-guess sweeps skip u)
    sum->count++;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  s->prof.clear();
}

mg_status plan_profile_enable(mg_solver* s, bool on) {
  if (on) {
    prof_drain(s);
    s->prof_done.clear();
  }
  s->prof_on = on;
  return MG_OK;
}

int plan_profile_read(mg_solver* s, int cap, const char** names, double* ms, int64_t* count, double* bytes) {
  prof_drain(s);
  int n = (int)s->prof_done.size();
  for (int i = 0; i < n && i < cap; i++) {
    if (names) names[i] = s->prof_done[i].name.c_str();
    if (ms) ms[i] = s->prof_done[i].ms;
    if (count) count[i] = s->prof_done[i].count;
    if (bytes) bytes[i] = s->prof_done[i].count ? s->prof_done[i].bytes / s->prof_done[i].count : 0.0;
  }
  return n;
}

}  // namespace mg
