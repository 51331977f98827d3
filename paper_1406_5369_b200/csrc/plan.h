// plan.h — solver state shared by api.cu and plan.cu (host side only).
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <tuple>
#include <string>
#include <utility>
#include <vector>

#include "mg.h"
#include "mg_common.cuh"
#include "partition.h"
#include "kernels_cd.h"
#include "comm.h"
#include "checked.h"
#include "loop_state.cuh"

typedef struct ncclComm* ncclComm_t;

namespace mg {

struct Level {
  Geom g;
  Geom gown;              // g restricted to the planes this rank writes when restricting into it
  bool dist = false;      // slab-distributed level
  Coef<double> c64;
  Coef<float> c32;
  double cx, cy, cz, D;   // double-precision coefficients (coarse direct solve)
  int64_t shape[3];       // [planes][rows][pitch]
  size_t elems;           // planes*rows*pitch
  void* u = nullptr;      // library-owned iterate (levels >= 1)
  void* f = nullptr;      // library-owned right-hand side (levels >= 1)
  void* r = nullptr;      // residual scratch (op-by-op schedule)
  void* t = nullptr;      // ping-pong partner of u
  // complex diffusion (cell-centred FAS): restricted lagged solution u^ and diffusivity g
  void* uh = nullptr;
  void* gd = nullptr;
  CdCoef<double> cd64{};
  CdCoef<float> cd32{};
};

// state of the on-device driver loop (loop.cu); written by the host before each solve

struct ProfRec {
  int kind;               // index into the kernel-name table
  int level;
  double bytes;           // algorithmic bytes of this launch
  cudaEvent_t a, b;
};

struct ProfSum {
  std::string name;
  double ms = 0, bytes = 0;
  int64_t count = 0;
};

}  // namespace mg

struct mg_solver {
  mg_config cfg;
  int L = 0;
  size_t esz = 8;
  std::vector<mg::Level> lv;
  // coarsest direct solve
  int m_coarse = 0;
  double* d_chol = nullptr;
  double* d_work = nullptr;
  // slab decomposition / NCCL
  mg::Partition pt;
  ncclComm_t comm = nullptr;
  mg::LoopGroup* loop = nullptr;  // loopback transport (ranks of one process on one device; tests)
  cudaEvent_t lb_ready = nullptr, lb_done = nullptr;
  double* d_rank_sums = nullptr;  // per-rank sums of r^2 (all-gathered)
  // norm
  double* d_partial = nullptr;
  int n_partial_cap = 0;
  double* d_norm = nullptr;
  double* h_norm = nullptr;  // pinned
  // graphs keyed by (u, f)
  cudaStream_t cap_stream = nullptr;
  cudaStream_t cap_body = nullptr;   // captures the body of the driver loop's WHILE node
  cudaStream_t comm_stream = nullptr;  // slab halo exchanges overlapped with interior sweeps
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  mg::LoopState* d_loop = nullptr;
  mg::LoopState* h_loop = nullptr;   // pinned
  double* d_hist = nullptr;
  int64_t hist_cap = 0;
  std::map<std::tuple<void*, const void*, int>, cudaGraphExec_t> graphs;  // (u, f, part)
  // e2e staging (mg_vcycle_host), and the double-buffered pipeline of mg_vcycle_host_batch
  void* stage_u = nullptr;
  void* stage_f = nullptr;
  void* bstage_u[2] = {nullptr, nullptr};
  void* bstage_f[2] = {nullptr, nullptr};
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr}, ev_d2h[2] = {nullptr, nullptr};
  double* h_norms = nullptr;  // pinned, batch norms
  int h_norms_cap = 0;
  // instrumentation
  int64_t launches_per_cycle = 0;
  int64_t head_launches = 0, tail_launches = 0;
  int64_t launch_counter = 0;
  bool prof_on = false;
  std::vector<mg::ProfRec> prof;
  std::vector<mg::ProfSum> prof_done;
  // errors
  std::string err;
  bool poisoned = false;
  // multi-rank failure path: the last exchange's communication failure (set by comm.cu, mapped
  // to MG_ERR_NCCL by the plan), fault injection (mg_fault_inject), the blocking-wait limit
  bool comm_failed = false;
  std::string comm_msg;
  int fault_kind = 0, fault_count = 0;
  double comm_timeout_s = 300.0;
};

namespace mg {
mg_status plan_fail(mg_solver* s, mg_status st, const char* msg);
mg_status plan_build(mg_solver* s);
void plan_free(mg_solver* s);
mg_status plan_run_vcycle(mg_solver* s, void* u, const void* f, cudaStream_t st);
mg_status plan_graph_vcycle(mg_solver* s, void* u, const void* f, cudaStream_t st);
// part: 0 whole cycle, 1 head (first sweep + input norm -> d_norm), 2 tail, 3 norm -> d_norm,
// 4 later head, 5 cycle + its norm, 6 the whole solve in one launch (see plan.cu)
mg_status plan_run_part(mg_solver* s, int part, void* u, const void* f, cudaStream_t st);
mg_status plan_graph_part(mg_solver* s, int part, void* u, const void* f, cudaStream_t st);
bool plan_can_split(mg_solver* s);
// on-device driver loop (loop.cu): one graph launch runs the whole mg_solve loop
bool plan_loop_supported(mg_solver* s);
// the whole loop as one tail launch (tail_level() = 0: the grid is a whole-cycle tail)
bool plan_solve_in_tail(mg_solver* s);
// eager: launch plan_solve_in_tail's kernel directly (no graph; MG_FLAG_NO_GRAPH / profiling)
mg_status plan_solve_device(mg_solver* s, void* u, const void* f, double rtol, int32_t max_cycles, int32_t* cycles,
                            double* history, cudaStream_t st, bool eager = false);
mg_status plan_norm(mg_solver* s, int level, const void* u, const void* f, double* out, cudaStream_t st, bool sync);
// wait for `st`: cudaStreamSynchronize, or with an NCCL communicator a poll of the stream and of
// ncclCommGetAsyncError with the solver's timeout (abort + MG_ERR_NCCL on error or timeout)
mg_status plan_wait(mg_solver* s, cudaStream_t st, const char* what);
// abort the NCCL communicator (a poisoned solver's; nothing without one)
void plan_comm_abort(mg_solver* s);
mg_status plan_op_smooth(mg_solver* s, int level, const void* uin, const void* f, void* uout, cudaStream_t st);
mg_status plan_op_residual(mg_solver* s, int level, const void* u, const void* f, void* r, cudaStream_t st);
mg_status plan_op_restrict(mg_solver* s, int level, const void* r, void* fc, cudaStream_t st);
mg_status plan_op_prolong(mg_solver* s, int level, const void* e, void* u, cudaStream_t st);
mg_status plan_op_coarse(mg_solver* s, const void* f, void* e, cudaStream_t st);
mg_status plan_workload_fill(mg_solver* s, void* dst, uint64_t seed, double lo, double hi, cudaStream_t st);
mg_status plan_profile_enable(mg_solver* s, bool on);
int plan_profile_read(mg_solver* s, int cap, const char** names, double* ms, int64_t* count, double* bytes);
}  // namespace mg
