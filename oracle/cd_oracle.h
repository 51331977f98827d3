/*
 * cd_oracle.h — plain CPU oracle of the paper's second workload: one implicit-
 * Euler step of nonlinear isotropic complex diffusion (Eqs. 2-3)
 * solved by a Full Approximation Scheme V-cycle with lagged diffusivity on a
 * CELL-CENTRED grid with Neumann (zero-flux) boundaries, cell-average
 * restriction and constant interpolation (Table 1 P:347-352;
 * SURVEY §8(f) NEXT-2 and NEXT-4).
 *
 * TEST INFRASTRUCTURE ONLY (same rules as mg_oracle.h): only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * load it; it shares no code with the CUDA path.
 *
 * Problem.  u - tau div(g(Im u) grad u) = f   (implicit Euler, f = u^n)
 *   g(s) = e^{i theta} / (1 + (s / (k theta))^2)                       (Eq. 3)
 * Discretisation ("averaged finite differences"): cell c, face to
 * neighbour c + o:  g_f = (g(c) + g(c+o)) / 2 from the LAGGED field; with
 * w_d = tau / h_d^2,
 *   (A u)(c) = a_c u(c) - sum_{faces f inside the domain} w_d g_f u(c+o),
 *   a_c = 1 + sum_{faces inside} w_d g_f     (boundary faces: zero flux, dropped)
 * Transfers: R = average of the 2^d children, P = constant injection
 * (R = 2^-d P^T).  Coarse operators are re-discretised at H = 2h from the
 * restricted lagged solution.
 * FAS V-cycle: g_l := g(u_l) once at cycle entry, frozen; nu1
 * sweeps; u^_H = R u_l; u_H = u^_H; f_H = A_H(u^_H) u^_H + R(f_l - A_l u_l);
 * recurse; u_l += P(u_H - u^_H); nu2 sweeps.  Coarsest level: ncoarse sweeps.
 *
 * Canonical arithmetic (reading 19): complex numbers are (re, im)
 * pairs of `real`; every product / sum / quotient is rounded in `real`, in this
 * order, without contraction:
 *   mul(a,b) = (a.re b.re - a.im b.im,  a.re b.im + a.im b.re)
 *   div(x,y) = ((x.re y.re + x.im y.im)/den, (x.im y.re - x.re y.im)/den),
 *              den = y.re y.re + y.im y.im
 *   g(s):  q = s / kth;  den = 1 + q q;  g = (cos_t / den, sin_t / den)
 *          (kth = k theta, cos_t, sin_t computed in double and cast once)
 *   per cell: faces in the order x-, x+, y-, y+, z-, z+ (those inside the
 *   domain): gf = 0.5 (g_c + g_nb) per component; cf = w_d gf per component;
 *   acc_a += cf; acc_s += mul(cf, u_nb)   (acc_* start at 0)
 *   a_c = (1 + acc_a.re, acc_a.im);  A u = mul(a_c, u_c) - acc_s
 *   smoother: u' = u + omega * div(f - A u, a_c)   (per component)
 *   restriction: x-pairs, then y-pairs, then z-pairs summed, times 2^-d
 * Red cells: even sum of 0-based global cell indices; red first (reading 8).
 *
 * Storage: dense unpadded complex arrays (re, im interleaved) of the level's
 * cells, x fastest: idx(i,j,k) = (k*ny + j)*nx + i; 2D: nz = 1.
 */
#ifndef CD_ORACLE_H
#define CD_ORACLE_H

#include <stdint.h>

#ifndef OR_REAL
#define OR_REAL double
#endif
typedef OR_REAL real;

typedef struct {
    int dim;          /* 2 or 3                                             */
    int n[3];         /* cells per axis at level 0; n[2] = 1 in 2D          */
    int levels;       /* L >= 1                                             */
    double h[3];      /* fine cell size per axis (unit domain: 1/n[d])      */
    int smoother;     /* 0 omega-Jacobi, 1 red-black GS (Table 1)           */
    double omega;
    int nu1, nu2, ncoarse;
    double tau, theta, kappa;   /* time step, angle, scaling k (Eq. 3)       */
} cd_config;

/* cells of level l */
int64_t cd_level_cells(const cd_config* c, int l);
/* Eq. 3 at Im u = s: out[0] = Re g, out[1] = Im g */
void cd_diffusivity(const cd_config* c, real s, real out[2]);
/* g field of level l from the lagged iterate ul (both complex arrays of level l) */
void cd_gfield(const cd_config* c, int l, const real* ul, real* g);
/* A u and the diagonal a_c with the frozen field g */
void cd_apply(const cd_config* c, int l, const real* g, const real* u, real* Au, real* diag);
/* one smoothing sweep in place (Jacobi double-buffered internally) */
void cd_smooth(const cd_config* c, int l, const real* g, real* u, const real* f);
/* cell-average restriction v_fine (level l) -> v_coarse (level l+1) */
void cd_restrict(const cd_config* c, int l, const real* vf, real* vc);
/* u_fine (level l) += P e_coarse (constant injection) */
void cd_prolong_add(const cd_config* c, int l, const real* ec, real* uf);
/* || f - A(u) u ||_2 with g = g(u) (the nonlinear residual), FP64 accumulation */
double cd_norm(const cd_config* c, int l, const real* u, const real* f);
/* one FAS V-cycle in place on level-0 arrays; returns 0, -1 on allocation failure */
int cd_cycle(const cd_config* c, real* u, const real* f);
/* driver loop (P:264-276 with the nonlinear residual); as or_solve */
int cd_solve(const cd_config* c, real* u, const real* f, double rtol, int max_cycles, double* history);

#endif
