/*
 * mg_oracle.h — plain, slow, obviously-correct CPU oracle of the geometric
 * multigrid V-cycle of arXiv:1406.5369 (Koestler et al.).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1406_5369_b200/, libmgb200.so) never links,
 * imports or calls anything under oracle/; the two share no code.
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * "reading k" = DESIGN.md §3 table row k (the readings of the paper).
 *
 * Storage: every level is a dense, UNPADDED node array including boundary
 * nodes, x fastest: idx(i,j,k) = (k*(ny+1) + j)*(nx+1) + i, where n{x,y,z} are
 * the CELLS per axis of that level (nodes = cells+1).  2D problems have
 * nz = 0, i.e. a single plane (2D vs 3D is only the domain).
 *
 * The library is compiled twice from one source: -DOR_REAL=double
 * (liboracle_f64.so) and -DOR_REAL=float (liboracle_f32.so).  Coefficients
 * are always computed in double and cast once (reading 13).
 */
#ifndef MG_ORACLE_H
#define MG_ORACLE_H

#include <stdint.h>

#ifndef OR_REAL
#define OR_REAL double
#endif
typedef OR_REAL real;

#define OR_JACOBI 0
#define OR_RBGS 1
#define OR_GS_LEX 2
#define OR_COARSE_DIRECT 0
#define OR_COARSE_SWEEPS 1

typedef struct {
    int dim;          /* 2 or 3 (Table 1 "UnitSquare, UnitCube") */
    int n[3];         /* cells per axis at level 0 (x,y,z); n[2] = 0 in 2D   */
    int levels;       /* L >= 1; level 0 finest, level L-1 coarsest  */
    double a[3];      /* A = -sum_d a_d d^2/dx_d^2 ; Poisson: a = 1  */
    double h[3];      /* fine spacing per axis; unit domain: 1/n[d]  */
    int smoother;     /* OR_JACOBI | OR_RBGS | OR_GS_LEX (Table 1)    */
    double omega;     /* damping                              */
    int nu1, nu2;     /* pre/post smoothing steps (Alg. 1)        */
    int coarse;       /* OR_COARSE_DIRECT | OR_COARSE_SWEEPS  */
    int ncoarse;      /* sweeps on the coarsest level in SWEEPS mode */
} or_config;

/* level coefficients (reading 13): c_d = a_d / h_{l,d}^2, D = 2*sum c_d,
 * wd = omega / D, h_{l,d} = 2^l h_d (direct coarse-grid approximation) */
void or_coeffs(const or_config* cfg, int l, double c[3], double* D, double* wd);
int64_t or_level_nodes(const or_config* cfg, int l);

/* single level operators (arrays of level l unless stated) */
void or_residual(const or_config* cfg, int l, const real* u, const real* f, real* r);
void or_jacobi(const or_config* cfg, int l, const real* u_in, const real* f, real* u_out);
void or_rbgs(const or_config* cfg, int l, real* u, const real* f);
void or_gs_lex(const or_config* cfg, int l, real* u, const real* f);
void or_smooth(const or_config* cfg, int l, real* u, const real* f, real* tmp);
void or_restrict(const or_config* cfg, int l, const real* r_fine, real* f_coarse);
void or_prolong_correct(const or_config* cfg, int l, const real* e_coarse, real* u_fine);
/* coarsest level solve A e = f (l = levels-1); returns 0 or -1 on failure */
int or_coarse_solve(const or_config* cfg, real* e, const real* f);
double or_norm(const or_config* cfg, int l, const real* u, const real* f);

/* whole method: one V-cycle in place on level-0 arrays (Alg. 1) */
int or_vcycle(const or_config* cfg, real* u, const real* f);
/* driver loop: history[0] = ||r0||, history[k] after cycle k.
 * Stops at the first k with history[k] <= rtol*history[0] or k = max_cycles.
 * Returns the number of cycles done, or -1 on failure (non-finite norm). */
int or_solve(const or_config* cfg, real* u, const real* f, double rtol,
             int max_cycles, double* history);

/* threads the OpenMP runtime will use (1 when built without OpenMP) */
int or_num_threads(void);

#endif
