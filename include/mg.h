/*
 * mg.h — C ABI of libmgb200.so: a B200-native (sm_100a) geometric multigrid
 * V-cycle for finite-difference Poisson-type problems on regular node-based
 * 2D/3D grids, the data-parallel hot path of arXiv:1406.5369 (Koestler et al.,
 * "A Scala Prototype to Generate Multigrid Solver Implementations ...").
 *
 * Citation keys: P:n = PAPER.md line n (the LaTeX source of arXiv:1406.5369);
 * Alg. 1 = the recursive V-cycle; the Layer-4 listing = P:263-320.
 *
 * Conventions (all entry points):
 *  - Every function returns an mg_status; nothing throws or aborts across the
 *    ABI.  On error, mg_error_string(solver) (or mg_error_string(NULL) for a
 *    failed mg_create) describes the last failure of the calling thread.
 *  - `u`, `f`, `r`, `e` are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 *    of the solver's dtype, laid out as a dense C-order array of shape
 *    [planes][rows][pitch] (x fastest), see mg_layout / mg_level_layout.
 *    3D: planes = z nodes, rows = y nodes; 2D: planes = y nodes, rows = 1.
 *    Node (i,j,k) includes the boundary: i = 0..nx, etc. (cells per axis nx).
 *    Padding elements (x > nx) of caller arrays are never written; a kernel may
 *    read them as part of a whole 16-byte vector, and their values never affect
 *    a result (no NaN/Inf check, no arithmetic that reaches a stored node).
 *  - Caller-owned buffers must stay alive until the stream work completes.
 *    `u` and `f` must not alias.  The library never writes boundary nodes of
 *    the caller's `u` (they hold the Dirichlet data).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  All GPU work
 *    is enqueued on it; entry points returning a host scalar synchronise it.
 *  - The library owns coarse-level buffers, the ping-pong buffer, reduction
 *    partials and cached CUDA graphs (keyed by the (u, f) pointers).
 *  - There is NO CPU fallback: without a usable sm_100 device every
 *    compute entry point fails with MG_ERR_CUDA.
 *  - One solver is used by one host thread at a time.
 */
#ifndef MG_H
#define MG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mg_solver mg_solver;

typedef enum {
    MG_OK = 0,
    MG_ERR_INVALID = 1,          /* bad argument / configuration              */
    MG_ERR_NOT_COARSENABLE = 2,  /* (nodes-1) not divisible by 2^(levels-1)   */
    MG_ERR_OOM = 3,              /* device allocation failed                  */
    MG_ERR_CUDA = 4,             /* CUDA runtime / launch failure (poisons)   */
    MG_ERR_NCCL = 5,             /* NCCL failure (poisons the solver)         */
    MG_ERR_NONFINITE = 6,        /* NaN/Inf residual norm             */
    MG_ERR_LAYOUT = 7,           /* pointer misaligned for the layout         */
    MG_ERR_POISONED = 8          /* an earlier CUDA/NCCL error poisoned it    */
} mg_status;

/* omega-Jacobi, red-black GS, lexicographic omega-GS (Table 1, "order lex";
 * one hyperplane i+j+k = s at a time on the GPU, nranks = 1, Poisson only) */
typedef enum { MG_JACOBI = 0, MG_RBGS = 1, MG_GS_LEX = 2 } mg_smoother;
typedef enum { MG_FP64 = 0, MG_FP32 = 1 } mg_dtype;           /* Table 1 */
typedef enum { MG_COARSE_DIRECT = 0, MG_COARSE_SWEEPS = 1 } mg_coarse;
/* The problem (Table 1 "Operator"):
 *  MG_PROBLEM_POISSON: A = -sum a_d d^2/dx_d^2 on a NODE-based grid, Dirichlet data in
 *    u's boundary nodes, correction-scheme V-cycle (Alg. 1).
 *  MG_PROBLEM_COMPLEX_DIFFUSION: one implicit-Euler step of nonlinear isotropic complex
 *    diffusion u - tau div(g(Im u) grad u) = f, g = e^{i theta}/(1 + (Im u/(kappa theta))^2)
 *    (Eqs. 2-3), averaged finite differences on a CELL-centred grid with
 *    Neumann (zero-flux) boundaries, FAS V-cycle with lagged diffusivity, cell-average
 *    restriction and constant interpolation.  Arrays hold COMPLEX
 *    values, (re, im) interleaved, of the precision `dtype`; nodes[d] then counts CELLS
 *    (the unknowns) per axis; there are no boundary entries; coarse must be
 *    MG_COARSE_SWEEPS (ncoarse sweeps on the coarsest level); nranks must be 1. */
typedef enum { MG_PROBLEM_POISSON = 0, MG_PROBLEM_COMPLEX_DIFFUSION = 1 } mg_problem;

/* flags */
#define MG_FLAG_NO_GRAPH 1u   /* launch eagerly instead of replaying a CUDA graph   */
#define MG_FLAG_BASELINE 2u   /* op-by-op kernels only (no fusion; two-pass RBGS)   */
#define MG_FLAG_SLAB 4u       /* slab layout (halos, agglomeration) even with nranks == 1 */
#define MG_FLAG_SEPARATE_PROLONG 8u /* 3D marching levels: prolongation + correction as its own pass; by
                                       default it is fused into the first post-sweep (u + P e formed in
                                       shared memory, never stored); A/B switch, bitwise equal */
#define MG_FLAG_HOST_LOOP 16u   /* mg_solve: host-driven loop (one synchronisation per cycle) instead of
                                   the on-device loop (one CUDA graph with a conditional WHILE node) */
#define MG_FLAG_NO_KFUSE 32u   /* 2D omega-Jacobi: one sweep per HBM pass instead of the temporally blocked
                                   passes of up to 3 (FP32) / 2 (FP64) sweeps (A/B measurement; bitwise equal) */
#define MG_FLAG_CD_KFUSE 64u   /* complex diffusion, 2D Jacobi: multi-sweep passes (3 FP32 / 2 FP64; measured
                                   slower than single sweeps; bitwise equal) */

typedef struct {
    int32_t dim;         /* 2 or 3                                        */
    int64_t nodes[3];    /* global nodes per axis incl. boundary (x, y, z); z ignored in 2D.
                            (nodes[d]-1) % 2^(levels-1) == 0                  */
    int32_t levels;      /* >= 1; 0 => paper rule: coarsen until the coarsest level has
                            1 interior node along the shortest axis    */
    double coeff[3];     /* a_d of A = -sum_d a_d d^2/dx_d^2; Poisson = {1,1,1} */
    double h[3];         /* fine spacing per axis; 0 => unit domain 1/(nodes-1) */
    int32_t smoother;    /* mg_smoother (default RBGS, the listing's GaussSeidel P:236) */
    double omega;        /* default 1.0 for RBGS, 0.8 for Jacobi       */
    int32_t nu1, nu2;    /* pre/post sweeps (Alg. 1); default 2, 2 (V(2,2))     */
    int32_t coarse;      /* mg_coarse, default DIRECT (reading 3)                      */
    int32_t ncoarse;     /* sweeps on the coarsest level in SWEEPS mode, def 10 */
    int32_t dtype;       /* mg_dtype                                                    */
    int32_t device;      /* CUDA device ordinal                                         */
    int32_t rank, nranks;/* slab decomposition along the slowest (plane) axis over nranks
                            GPUs, one process per GPU                   */
    const void* nccl_id; /* 128-byte ncclUniqueId when nranks > 1 (the same bytes on every
                            rank, e.g. broadcast with torch.distributed), else NULL.
                            mg_create is then collective: all ranks must call it.      */
    uint32_t flags;      /* MG_FLAG_*                                                   */
    int32_t pm_min_nx;   /* smallest x-extent (cells) of a level that uses the plane-
                            marching kernels; 0 => 128.  Smaller levels use one thread per
                            node.  Results are bitwise identical either way.              */
    int32_t problem;     /* mg_problem (default MG_PROBLEM_POISSON)                     */
    double tau;          /* complex diffusion: implicit-Euler time step (default 0.1)    */
    double theta;        /* complex diffusion: angle of Eq. 3 (default pi/30)            */
    double kappa;        /* complex diffusion: scaling k of Eq. 3 (default 2); the paper
                            gives no values                                        */
    void* loopback;      /* nranks > 1 without NCCL: a group from mg_loopback_group_create
                            shared by `nranks` solvers of THIS process on the same device,
                            each driven by its own host thread (the collectives rendezvous
                            on the host and copy device-to-device); requires
                            MG_FLAG_NO_GRAPH.  For testing the multi-rank path on one GPU. */
    double comm_timeout_s; /* nranks > 1: a blocking entry point that waits on the device polls
                            the communicator (ncclCommGetAsyncError) and gives up after this many
                            seconds without completion: the communicator is aborted
                            (ncclCommAbort), the call returns MG_ERR_NCCL and the solver is
                            poisoned.  The loopback rendezvous uses the same limit.  0 => 300.  */
} mg_config;

/* Fill `cfg` with the defaults above for a `dim`-D grid of `nodes` per axis
 * (complex diffusion: set problem, coarse = MG_COARSE_SWEEPS and nodes = cells). */
void mg_config_default(mg_config* cfg, int32_t dim, int64_t nodes);

/* Validate `cfg`, build the level hierarchy (h_l = 2^l h, re-discretised
 * coefficients c_d = a_d/h_{l,d}^2, D = 2 sum c_d), allocate the
 * library-owned buffers and, for DIRECT coarse mode with >1 coarsest unknown,
 * factor the coarsest matrix on the device.  On failure nothing is allocated
 * and *out is NULL. */
mg_status mg_create(const mg_config* cfg, mg_solver** out);

/* Shape [planes][rows][pitch] (elements) of this rank's level-0 u and f; the
 * slab of global planes it owns is [*first_plane, *first_plane + *owned).  In slab
 * mode (nranks > 1 or MG_FLAG_SLAB) local plane i holds global plane
 * first_plane - halo + i (halo from mg_partition); the halo planes are library
 * scratch (rewritten by halo exchanges), the owned planes are the caller's. */
mg_status mg_layout(const mg_solver* s, int64_t shape[3], int64_t* first_plane, int64_t* owned);
/* Host-only (no GPU needed): the slab decomposition mg_create would use for
 * `cfg` at `level`: owned global planes [*first_plane, +*owned_planes), whether
 * the level is distributed (else held in full on every rank: agglomeration),
 * and the halo depth.  Rank p owns planes [p n_l/P, (p+1) n_l/P), the last rank
 * also plane n_l; levels stay distributed while n_l/P >= 8 and even. */
mg_status mg_partition(const mg_config* cfg, int32_t level, int64_t* first_plane, int64_t* owned_planes,
                       int32_t* distributed, int32_t* halo);
/* Shape of the level-l arrays used by the per-operation entry points below. */
mg_status mg_level_layout(const mg_solver* s, int32_t level, int64_t shape[3]);
int32_t mg_num_levels(const mg_solver* s);

/* One V(nu1,nu2)-cycle of Alg. 1 — for complex diffusion one FAS
 * V-cycle — in place on u, asynchronous on `stream`.  Replays a cached CUDA graph for this (u, f) unless
 * MG_FLAG_NO_GRAPH. */
mg_status mg_vcycle(mg_solver* s, void* u, const void* f, void* stream);

/* ||f - A u||_2 over interior nodes, unscaled (L2Residual),
 * FP64 accumulation, deterministic reduction order.  Blocking.  Complex diffusion:
 * the nonlinear residual ||f - A(u) u||_2 with the diffusivity evaluated from u. */
mg_status mg_residual_norm(mg_solver* s, const void* u, const void* f, double* out, void* stream);

/* Driver loop of the `Application` listing: r0 = norm; repeat
 * { V-cycle; r_k = norm } until r_k <= rtol * r0 or max_cycles.  rtol < 0 turns
 * the residual test off: exactly max_cycles cycles (a fixed-work loop that does not
 * stop when an iterate reaches an exact solution); NaN rtol is MG_ERR_INVALID.  history (if
 * not NULL, host memory) receives r_0..r_k (room for max_cycles+1 doubles),
 * history[0] = r0; *cycles = k.  Blocking.  Returns MG_ERR_NONFINITE if a
 * norm is NaN/Inf (the loop stops at that cycle).
 * By default the whole loop runs on the device: one CUDA graph whose WHILE
 * node repeats {cycle, norm, test} with the stopping test evaluated by a kernel,
 * one host synchronisation per solve.  On grids whose whole cycle is the coarse tail
 * (small levels only, e.g. 65^2) the loop runs inside ONE kernel launch instead (also
 * with MG_FLAG_NO_GRAPH or profiling).  MG_FLAG_HOST_LOOP, MG_FLAG_NO_GRAPH,
 * profiling, or nranks > 1 (NCCL cannot run inside a conditional node) select
 * the host loop; all give bitwise identical iterates and norms. */
mg_status mg_solve(mg_solver* s, void* u, const void* f, double rtol, int32_t max_cycles,
                   int32_t* cycles, double* history, void* stream);

/* End-to-end variant with HOST buffers u_host, f_host (dense [planes][rows][pitch],
 * preferably pinned): copies f and u to library-owned device buffers, runs
 * `ncycles` V-cycles, computes the residual norm into *norm_out (may be NULL),
 * copies u back.  Blocking. */
mg_status mg_vcycle_host(mg_solver* s, void* u_host, const void* f_host, int32_t ncycles,
                         double* norm_out, void* stream);

/* End-to-end for a stream of `nbatch` independent problems in HOST memory (pinned):
 * problem b copies f_in[b] and u_in[b] to the device, runs `ncycles` cycles, computes
 * its residual norm into norms[b] (may be NULL) and copies u back to u_out[b] (u_out[b]
 * may equal u_in[b]).  Copies and compute are pipelined over two library-owned staging
 * sets and two copy streams: the H2D of problem b+1 and the D2H of problem b-1 overlap
 * problem b's cycles (PCIe is full duplex).  Blocking; the host buffers of all problems
 * must stay valid and unaliased across problems until it returns. */
mg_status mg_vcycle_host_batch(mg_solver* s, const void* const* u_in, void* const* u_out,
                               const void* const* f_in, int32_t nbatch, int32_t ncycles,
                               double* norms, void* stream);

/* ---- per-operation entry points (one step of Alg. 1 each, for parity tests).
 * Arrays use mg_level_layout(level).  Asynchronous unless stated.
 * Complex diffusion: mg_op_smooth freezes the diffusivity at g(u_in) (lagged) and
 * sweeps once; mg_op_residual gives f - A(g(u)) u; mg_op_restrict is the cell average;
 * mg_op_prolong_correct adds the parent cell's value (constant interpolation);
 * mg_op_norm is the nonlinear residual norm; mg_op_coarse_solve is not available
 * (MG_ERR_INVALID: the FAS coarsest level is ncoarse sweeps). */
/* one sweep of the configured smoother S_h (listing P:299-305):
 * u_out = S(u_in); u_out may equal u_in.  Boundary nodes of u_out := u_in's. */
mg_status mg_op_smooth(mg_solver* s, int32_t level, const void* u_in, const void* f, void* u_out, void* stream);
/* r = f - A u on interior, 0 on boundary (Alg. 1 line 4) */
mg_status mg_op_residual(mg_solver* s, int32_t level, const void* u, const void* f, void* r, void* stream);
/* f_{l+1} = R r_l, full weighting (listing P:307-312); coarse boundary := 0 */
mg_status mg_op_restrict(mg_solver* s, int32_t level, const void* r, void* f_coarse, void* stream);
/* u_l += P e_{l+1}, bi/trilinear (listing P:314-319) */
mg_status mg_op_prolong_correct(mg_solver* s, int32_t level, const void* e_coarse, void* u, void* stream);
/* e = A_{L-1}^{-1} f on the coarsest level (Alg. 1 line 2) */
mg_status mg_op_coarse_solve(mg_solver* s, const void* f, void* e, void* stream);
/* residual norm of level `level`; blocking */
mg_status mg_op_norm(mg_solver* s, int32_t level, const void* u, const void* f, double* out, void* stream);

/* ---- synthetic inputs (NOT method arithmetic): the counter-based SplitMix64
 * generator of DESIGN.md reading 10 on the device.  dst (level-0 layout of
 * this rank) gets lo + (hi-lo) * U[0,1) of the GLOBAL unpadded node index on
 * interior nodes and 0 on boundary nodes. */
mg_status mg_workload_fill(mg_solver* s, void* dst, uint64_t seed, double lo, double hi, void* stream);

/* ---- instrumentation */
/* number of kernel launches per mg_vcycle (counted at plan build) */
int64_t mg_launches_per_cycle(const mg_solver* s);
/* enable (1) / disable (0) per-kernel CUDA-event timing; while enabled
 * mg_vcycle launches eagerly and records events around every launch. */
mg_status mg_profile_enable(mg_solver* s, int32_t on);
/* Per-kernel timing since enable: for entry i (< n), names[i] points to a static string
 * "<kernel>@L<level>", ms[i] = summed device time, count[i] = launches,
 * bytes[i] = mean ALGORITHMIC bytes per launch (launches of one kernel may
 * differ, e.g. a zero-guess first sweep does not read u).  Returns the number of entries
 * (may exceed cap; only min(n,cap) written).  Synchronises the device. */
int32_t mg_profile_read(mg_solver* s, int32_t cap, const char** names, double* ms,
                        int64_t* count, double* bytes);

/* Fault injection for tests of the failure path: the `countdown`-th halo exchange
 * from now of this rank (1 = the next one) fails.  MG_FAULT_COMM_ERROR: the exchange reports a
 * communication error, as a failed ncclSend/ncclRecv would (the call returns MG_ERR_NCCL, the
 * solver is poisoned).  MG_FAULT_HALO_CORRUPT: the exchange completes but the received halo
 * planes are overwritten with a wrong finite value (silent data corruption, for showing that
 * the parity tests catch it).  MG_FAULT_NONE disarms.  Host-only; MG_ERR_INVALID on a
 * solver without a multi-rank exchange. */
typedef enum { MG_FAULT_NONE = 0, MG_FAULT_COMM_ERROR = 1, MG_FAULT_HALO_CORRUPT = 2 } mg_fault;
mg_status mg_fault_inject(mg_solver* s, int32_t kind, int32_t countdown);

/* Loopback group of `nranks` ranks for mg_config.loopback (see there); destroy it after
 * every solver of the group has been destroyed. */
mg_status mg_loopback_group_create(int32_t nranks, void** group);
void mg_loopback_group_destroy(void* group);

/* Host-only: write a fresh 128-byte ncclUniqueId into out (rank 0 calls it and
 * broadcasts the bytes to the other ranks before mg_create). */
mg_status mg_nccl_unique_id(void* out128);

const char* mg_error_string(const mg_solver* s);
void mg_destroy(mg_solver* s);

#ifdef __cplusplus
}
#endif
#endif /* MG_H */
