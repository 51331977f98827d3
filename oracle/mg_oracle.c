/*
 * mg_oracle.c — the CPU oracle of the V-cycle of arXiv:1406.5369.
 *
 * TEST INFRASTRUCTURE ONLY (see mg_oracle.h).  Plain loops, no blocking, no
 * fusion, no reordering beyond the canonical per-point operation order fixed
 * in DESIGN.md §3 (reading 13).  Compiled with -O2 -ffp-contract=off so that
 * no multiply-add is ever contracted.  OpenMP (optional) only splits the
 * outermost loop of pointwise-independent loops; results do not depend on
 * the thread count (the norm sums per plane, then planes in order).
 *
 * Each function cites the passage it follows.
 */
#include "mg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---- hierarchy ("xcoarsefac = 2"; reading 1, 2) ---------------- */

static int nx_of(const or_config* c, int l) { return c->n[0] >> l; }
static int ny_of(const or_config* c, int l) { return c->n[1] >> l; }
static int nz_of(const or_config* c, int l) { return c->dim == 3 ? (c->n[2] >> l) : 0; }

int64_t or_level_nodes(const or_config* cfg, int l) {
    return (int64_t)(nx_of(cfg, l) + 1) * (ny_of(cfg, l) + 1) * (nz_of(cfg, l) + 1);
}

#define IDX(i, j, k) ((((int64_t)(k)) * (ny + 1) + (j)) * (nx + 1) + (i))

/* Direct coarse-grid approximation (Table 1 "direct
 * (re-discretization)"): the level-l operator is the same FD stencil at
 * spacing h_l = 2^l h.  Computed in double (reading 13). */
void or_coeffs(const or_config* cfg, int l, double c[3], double* D, double* wd) {
    double sum = 0.0;
    for (int d = 0; d < 3; d++) {
        c[d] = 0.0;
        if (d < cfg->dim) {
            double hl = ldexp(cfg->h[d], l);
            c[d] = cfg->a[d] / (hl * hl);
            sum += c[d];
        }
    }
    *D = 2.0 * sum;
    *wd = cfg->omega / *D;
}

/* The 5-/7-point stencil of A = -Delta_h (reading 6)
 * applied at an interior node, in the canonical order of reading 13:
 *   s  = cx*(u[x-1]+u[x+1]);  s = s + cy*(u[y-1]+u[y+1]);
 *   s  = s + cz*(u[z-1]+u[z+1]) (3D only);  Au = D*u_c - s;  r = f - Au     */
static real point_residual(int dim, const real* u, int64_t p, int64_t sy, int64_t sz,
                           real cx, real cy, real cz, real D, real fp) {
    real s = cx * (u[p - 1] + u[p + 1]);
    s = s + cy * (u[p - sy] + u[p + sy]);
    if (dim == 3) s = s + cz * (u[p - sz] + u[p + sz]);
    real Au = D * u[p] - s;
    return fp - Au;
}

typedef struct {
    int nx, ny, nz, kmin, kmax;
    int64_t sy, sz;
    real cx, cy, cz, D, wd;
} lvl;

static lvl level_of(const or_config* cfg, int l) {
    lvl L;
    double c[3], D, wd;
    or_coeffs(cfg, l, c, &D, &wd);
    L.nx = nx_of(cfg, l);
    L.ny = ny_of(cfg, l);
    L.nz = nz_of(cfg, l);
    /* interior planes: 1..nz-1 in 3D; the single plane 0 in 2D */
    L.kmin = cfg->dim == 3 ? 1 : 0;
    L.kmax = cfg->dim == 3 ? L.nz - 1 : 0;
    L.sy = L.nx + 1;
    L.sz = (int64_t)(L.nx + 1) * (L.ny + 1);
    L.cx = (real)c[0];
    L.cy = (real)c[1];
    L.cz = (real)c[2];
    L.D = (real)D;
    L.wd = (real)wd;
    return L;
}

/* Residual r = f - A u on interior nodes, r = 0 on the boundary
 * (Alg. 1 line 4; `Residual(lev)` P:288). */
void or_residual(const or_config* cfg, int l, const real* u, const real* f, real* r) {
    lvl L = level_of(cfg, l);
    int nx = L.nx, ny = L.ny;
    memset(r, 0, sizeof(real) * or_level_nodes(cfg, l));
#pragma omp parallel for schedule(static)
    for (int k = L.kmin; k <= L.kmax; k++)
        for (int j = 1; j < ny; j++)
            for (int i = 1; i < nx; i++) {
                int64_t p = IDX(i, j, k);
                r[p] = point_residual(cfg->dim, u, p, L.sy, L.sz, L.cx, L.cy, L.cz, L.D, f[p]);
            }
}

/* omega-Jacobi sweep (Table 1; omega = 0.8 P:568), double-buffered
 * (reading 9): u_out = u_in + (omega/D)*(f - A u_in) on the
 * interior; boundary nodes copied unchanged. */
void or_jacobi(const or_config* cfg, int l, const real* u_in, const real* f, real* u_out) {
    lvl L = level_of(cfg, l);
    int nx = L.nx, ny = L.ny;
    memcpy(u_out, u_in, sizeof(real) * or_level_nodes(cfg, l));
#pragma omp parallel for schedule(static)
    for (int k = L.kmin; k <= L.kmax; k++)
        for (int j = 1; j < ny; j++)
            for (int i = 1; i < nx; i++) {
                int64_t p = IDX(i, j, k);
                real r = point_residual(cfg->dim, u_in, p, L.sy, L.sz, L.cx, L.cy, L.cz, L.D, f[p]);
                u_out[p] = u_in[p] + L.wd * r;
            }
}

/* Red-black Gauss-Seidel sweep (Layer-4 listing P:299-305,
 * "loop innerpoints ... order rb": u = u + inverse(diag(Lapl))*omega*(f - Lapl*u)).
 * Red = interior nodes whose GLOBAL level index sum i+j(+k) is even, updated
 * first; then black (reading 8).  In place: each point reads
 * the current values of its (other-colour) neighbours. */
static void rbgs_colour(const or_config* cfg, const lvl* L, real* u, const real* f, int colour) {
    int nx = L->nx, ny = L->ny;
#pragma omp parallel for schedule(static)
    for (int k = L->kmin; k <= L->kmax; k++)
        for (int j = 1; j < ny; j++)
            for (int i = 1; i < nx; i++) {
                if (((i + j + k) & 1) != colour) continue;
                int64_t p = IDX(i, j, k);
                real r = point_residual(cfg->dim, u, p, L->sy, L->sz, L->cx, L->cy, L->cz, L->D, f[p]);
                u[p] = u[p] + L->wd * r;
            }
}

void or_rbgs(const or_config* cfg, int l, real* u, const real* f) {
    lvl L = level_of(cfg, l);
    rbgs_colour(cfg, &L, u, f, 0); /* red   */
    rbgs_colour(cfg, &L, u, f, 1); /* black */
}

/* Lexicographic omega-Gauss-Seidel sweep (Table 1 "omega-Gauss-Seidel", P:351;
 * S:416 "order lex -> one nest, row-major"): interior nodes in row-major order
 * (x fastest, then y, then z), in place, each reading the latest values:
 * u(x) = u(x) + (omega/D)(f - A u)(x).  Sequential by definition. */
void or_gs_lex(const or_config* cfg, int l, real* u, const real* f) {
    lvl L = level_of(cfg, l);
    int nx = L.nx, ny = L.ny;
    for (int k = L.kmin; k <= L.kmax; k++)
        for (int j = 1; j < ny; j++)
            for (int i = 1; i < nx; i++) {
                int64_t p = IDX(i, j, k);
                real r = point_residual(cfg->dim, u, p, L.sy, L.sz, L.cx, L.cy, L.cz, L.D, f[p]);
                u[p] = u[p] + L.wd * r;
            }
}

/* one sweep of the configured smoother S_h (Alg. 1 lines 3 and 7) */
void or_smooth(const or_config* cfg, int l, real* u, const real* f, real* tmp) {
    if (cfg->smoother == OR_JACOBI) {
        or_jacobi(cfg, l, u, f, tmp);
        memcpy(u, tmp, sizeof(real) * or_level_nodes(cfg, l));
    } else if (cfg->smoother == OR_GS_LEX) {
        or_gs_lex(cfg, l, u, f);
    } else {
        or_rbgs(cfg, l, u, f);
    }
}

/* Full-weighting restriction f_{l+1} = R r_l (Alg. 1 line 5, P:202;
 * `restr_order = 2` => full weighting; listing P:307-312).
 * R = 2^-d P^T (reading 7), i.e. tensor product of [1 2 1]/4 per axis,
 * evaluated separably x, then y, then z (reading 13):
 *   t = (r[-1] + r[+1]) + 2*r[0] along each axis in turn; f = t * 4^-d. */
void or_restrict(const or_config* cfg, int l, const real* r_fine, real* f_coarse) {
    lvl F = level_of(cfg, l);
    lvl C = level_of(cfg, l + 1);
    int nx = C.nx, ny = C.ny; /* IDX below addresses the coarse array */
    const real scale = cfg->dim == 3 ? (real)(1.0 / 64.0) : (real)(1.0 / 16.0);
    memset(f_coarse, 0, sizeof(real) * or_level_nodes(cfg, l + 1));
    int dzlo = cfg->dim == 3 ? -1 : 0, dzhi = cfg->dim == 3 ? 1 : 0;
#pragma omp parallel for schedule(static)
    for (int K = C.kmin; K <= C.kmax; K++)
        for (int J = 1; J < ny; J++)
            for (int I = 1; I < nx; I++) {
                real tx[3][3]; /* [dz+1][dy+1] */
                for (int dz = dzlo; dz <= dzhi; dz++)
                    for (int dy = -1; dy <= 1; dy++) {
                        int64_t q = ((int64_t)(2 * K + dz) * (F.ny + 1) + (2 * J + dy)) * (F.nx + 1) + 2 * I;
                        tx[dz + 1][dy + 1] = (r_fine[q - 1] + r_fine[q + 1]) + (real)2 * r_fine[q];
                    }
                real ty[3];
                for (int dz = dzlo; dz <= dzhi; dz++)
                    ty[dz + 1] = (tx[dz + 1][0] + tx[dz + 1][2]) + (real)2 * tx[dz + 1][1];
                real t = ty[1];
                if (cfg->dim == 3) t = (ty[0] + ty[2]) + (real)2 * ty[1];
                f_coarse[IDX(I, J, K)] = t * scale;
            }
}

/* Bi-/trilinear prolongation and coarse-grid correction
 * u_l += P e_{l+1} (Alg. 1 line 6; `int_order = 2`, P:246, P:255;
 * `interpolatecorr`).  Fine node x = 2X + delta, delta in {0,1}^d;
 * the coarse boundary of e is 0 (homogeneous error equation).  Separable,
 * x then y then z (reading 13):
 *   v_x = dx ? 0.5*(e(X)+e(X+1)) : e(X);  likewise along y, then z;  u += v. */
void or_prolong_correct(const or_config* cfg, int l, const real* e_coarse, real* u_fine) {
    lvl F = level_of(cfg, l);
    lvl C = level_of(cfg, l + 1);
    int nx = F.nx, ny = F.ny; /* IDX addresses the fine array */
    const real half = (real)0.5;
#pragma omp parallel for schedule(static)
    for (int k = F.kmin; k <= F.kmax; k++)
        for (int j = 1; j < ny; j++)
            for (int i = 1; i < nx; i++) {
                int I = i >> 1, J = j >> 1, K = k >> 1;
                int dx = i & 1, dy = j & 1, dz = cfg->dim == 3 ? (k & 1) : 0;
                real vx[2][2]; /* [zz][yy] */
                for (int zz = 0; zz <= dz; zz++)
                    for (int yy = 0; yy <= dy; yy++) {
                        int64_t q = ((int64_t)(K + zz) * (C.ny + 1) + (J + yy)) * (C.nx + 1) + I;
                        vx[zz][yy] = dx ? half * (e_coarse[q] + e_coarse[q + 1]) : e_coarse[q];
                    }
                real vy[2];
                for (int zz = 0; zz <= dz; zz++)
                    vy[zz] = dy ? half * (vx[zz][0] + vx[zz][1]) : vx[zz][0];
                real v = dz ? half * (vy[0] + vy[1]) : vy[0];
                int64_t p = IDX(i, j, k);
                u_fine[p] = u_fine[p] + v;
            }
}

/* Coarsest-level direct solve (Alg. 1 line 2, "direct solver"; reading 3):
 * one interior unknown: e = f / D.  Otherwise: assemble the dense matrix of
 * the coarsest stencil (interior unknowns, lexicographic, x fastest) in
 * double, Cholesky-Banachiewicz (row by row, inner sums in increasing index),
 * forward then backward substitution, then round to real (reading 13). */
int or_coarse_solve(const or_config* cfg, real* e, const real* f) {
    int l = cfg->levels - 1;
    lvl L = level_of(cfg, l);
    int nx = L.nx, ny = L.ny;
    double c[3], D, wd;
    or_coeffs(cfg, l, c, &D, &wd);
    int mx = nx - 1, my = ny - 1, mz = cfg->dim == 3 ? L.nz - 1 : 1;
    int m = mx * my * mz;
    memset(e, 0, sizeof(real) * or_level_nodes(cfg, l));
    if (m <= 0) return 0;
#define UNK(i, j, k) ((((k)-L.kmin) * my + ((j)-1)) * mx + ((i)-1))
    if (m == 1) {
        int64_t p = IDX(1, 1, L.kmin);
        e[p] = (real)((double)f[p] / D);
        return 0;
    }
    double* A = (double*)calloc((size_t)m * m, sizeof(double));
    double* Lf = (double*)calloc((size_t)m * m, sizeof(double));
    double* y = (double*)calloc((size_t)m, sizeof(double));
    if (!A || !Lf || !y) { free(A); free(Lf); free(y); return -1; }
    for (int k = L.kmin; k <= L.kmax; k++)
        for (int j = 1; j < ny; j++)
            for (int i = 1; i < nx; i++) {
                int p = UNK(i, j, k);
                A[(size_t)p * m + p] = D;
                if (i > 1) A[(size_t)p * m + UNK(i - 1, j, k)] = -c[0];
                if (i < nx - 1) A[(size_t)p * m + UNK(i + 1, j, k)] = -c[0];
                if (j > 1) A[(size_t)p * m + UNK(i, j - 1, k)] = -c[1];
                if (j < ny - 1) A[(size_t)p * m + UNK(i, j + 1, k)] = -c[1];
                if (cfg->dim == 3 && k > 1) A[(size_t)p * m + UNK(i, j, k - 1)] = -c[2];
                if (cfg->dim == 3 && k < L.nz - 1) A[(size_t)p * m + UNK(i, j, k + 1)] = -c[2];
            }
    /* Cholesky-Banachiewicz: L[i][j] = (A[i][j] - sum_{k<j} L[i][k] L[j][k]) / L[j][j],
     * L[i][i] = sqrt(A[i][i] - sum_{k<i} L[i][k]^2) */
    for (int i = 0; i < m; i++) {
        for (int j = 0; j <= i; j++) {
            double s = A[(size_t)i * m + j];
            for (int k = 0; k < j; k++) s = s - Lf[(size_t)i * m + k] * Lf[(size_t)j * m + k];
            if (i == j) {
                if (!(s > 0.0)) { free(A); free(Lf); free(y); return -1; }
                Lf[(size_t)i * m + i] = sqrt(s);
            } else {
                Lf[(size_t)i * m + j] = s / Lf[(size_t)j * m + j];
            }
        }
    }
    /* forward: L y = f (increasing index) */
    for (int k = L.kmin; k <= L.kmax; k++)
        for (int j = 1; j < ny; j++)
            for (int i = 1; i < nx; i++) y[UNK(i, j, k)] = (double)f[IDX(i, j, k)];
    for (int i = 0; i < m; i++) {
        double s = y[i];
        for (int k = 0; k < i; k++) s = s - Lf[(size_t)i * m + k] * y[k];
        y[i] = s / Lf[(size_t)i * m + i];
    }
    /* backward: L^T x = y (decreasing index) */
    for (int i = m - 1; i >= 0; i--) {
        double s = y[i];
        for (int k = i + 1; k < m; k++) s = s - Lf[(size_t)k * m + i] * y[k];
        y[i] = s / Lf[(size_t)i * m + i];
    }
    for (int k = L.kmin; k <= L.kmax; k++)
        for (int j = 1; j < ny; j++)
            for (int i = 1; i < nx; i++) e[IDX(i, j, k)] = (real)y[UNK(i, j, k)];
#undef UNK
    free(A);
    free(Lf);
    free(y);
    return 0;
}

/* ||f - A u||_2 over the interior, unscaled (`L2Residual`, P:266-274;
 * reading 11), squares accumulated in double in z, y, x order: per
 * plane first, then the plane sums in increasing plane order. */
double or_norm(const or_config* cfg, int l, const real* u, const real* f) {
    lvl L = level_of(cfg, l);
    int nx = L.nx, ny = L.ny;
    int nplanes = L.kmax - L.kmin + 1;
    double* part = (double*)calloc((size_t)nplanes, sizeof(double));
#pragma omp parallel for schedule(static)
    for (int k = L.kmin; k <= L.kmax; k++) {
        double s = 0.0;
        for (int j = 1; j < ny; j++)
            for (int i = 1; i < nx; i++) {
                int64_t p = IDX(i, j, k);
                double r = (double)point_residual(cfg->dim, u, p, L.sy, L.sz, L.cx, L.cy, L.cz, L.D, f[p]);
                s = s + r * r;
            }
        part[k - L.kmin] = s;
    }
    double s = 0.0;
    for (int q = 0; q < nplanes; q++) s = s + part[q];
    free(part);
    return sqrt(s);
}

/* ---- the recursive V-cycle, Algorithm 1 and the Layer-4
 *      VCycle listing ---------------------------------------- */

typedef struct {
    real** u;   /* u[l], l >= 1: coarse error iterates      */
    real** f;   /* f[l], l >= 1: restricted residuals       */
    real** r;   /* r[l]: residual of level l                */
    real** tmp; /* tmp[l]: Jacobi double buffer             */
} hier;

static void hier_free(const or_config* cfg, hier* H) {
    for (int l = 0; l < cfg->levels; l++) {
        if (H->u && l > 0) free(H->u[l]);
        if (H->f && l > 0) free(H->f[l]);
        if (H->r) free(H->r[l]);
        if (H->tmp) free(H->tmp[l]);
    }
    free(H->u);
    free(H->f);
    free(H->r);
    free(H->tmp);
}

static int hier_alloc(const or_config* cfg, hier* H) {
    int L = cfg->levels;
    H->u = (real**)calloc(L, sizeof(real*));
    H->f = (real**)calloc(L, sizeof(real*));
    H->r = (real**)calloc(L, sizeof(real*));
    H->tmp = (real**)calloc(L, sizeof(real*));
    if (!H->u || !H->f || !H->r || !H->tmp) return -1;
    for (int l = 0; l < L; l++) {
        size_t n = (size_t)or_level_nodes(cfg, l);
        if (l > 0) {
            H->u[l] = (real*)calloc(n, sizeof(real));
            H->f[l] = (real*)calloc(n, sizeof(real));
            if (!H->u[l] || !H->f[l]) return -1;
        }
        H->r[l] = (real*)calloc(n, sizeof(real));
        H->tmp[l] = (real*)calloc(n, sizeof(real));
        if (!H->r[l] || !H->tmp[l]) return -1;
    }
    return 0;
}

static int vcycle_rec(const or_config* cfg, hier* H, int l) {
    real* u = H->u[l];
    const real* f = H->f[l];
    if (l == cfg->levels - 1) {
        /* Alg. 1 line 2: coarsest level */
        if (cfg->coarse == OR_COARSE_SWEEPS) {
            /* Layer-4 listing P:280-283: repeat ncoarse GaussSeidel(lev) */
            for (int s = 0; s < cfg->ncoarse; s++) or_smooth(cfg, l, u, f, H->tmp[l]);
            return 0;
        }
        if (l == 0) {
            /* single-level hierarchy: solve in correction form so that
             * non-zero Dirichlet data of the caller's u is honoured */
            or_residual(cfg, 0, u, f, H->r[0]);
            if (or_coarse_solve(cfg, H->tmp[0], H->r[0])) return -1;
            int64_t n = or_level_nodes(cfg, 0);
            for (int64_t p = 0; p < n; p++) u[p] = u[p] + H->tmp[0][p];
            return 0;
        }
        return or_coarse_solve(cfg, u, f);
    }
    for (int s = 0; s < cfg->nu1; s++) or_smooth(cfg, l, u, f, H->tmp[l]); /* line 3 */
    or_residual(cfg, l, u, f, H->r[l]);                                    /* line 4 */
    or_restrict(cfg, l, H->r[l], H->f[l + 1]);                             /* line 5 */
    memset(H->u[l + 1], 0, sizeof(real) * or_level_nodes(cfg, l + 1));    /* V_H(0, ..) */
    if (vcycle_rec(cfg, H, l + 1)) return -1;                              /* line 6 */
    or_prolong_correct(cfg, l, H->u[l + 1], u);                            /* line 7 */
    for (int s = 0; s < cfg->nu2; s++) or_smooth(cfg, l, u, f, H->tmp[l]); /* line 8 */
    return 0;
}

int or_vcycle(const or_config* cfg, real* u, const real* f) {
    hier H;
    memset(&H, 0, sizeof(H));
    if (hier_alloc(cfg, &H)) { hier_free(cfg, &H); return -1; }
    H.u[0] = u;
    H.f[0] = (real*)f;
    int rc = vcycle_rec(cfg, &H, 0);
    H.u[0] = NULL;
    H.f[0] = NULL;
    hier_free(cfg, &H);
    return rc;
}

/* `Application`: res0 = L2Residual(0); repeat { VCycle(0);
 * res = L2Residual(0) }, stopped at rtol (reading 12). */
int or_solve(const or_config* cfg, real* u, const real* f, double rtol,
             int max_cycles, double* history) {
    double r0 = or_norm(cfg, 0, u, f);
    if (history) history[0] = r0;
    if (!isfinite(r0)) return -1;
    int k = 0;
    while (k < max_cycles) {
        if (or_vcycle(cfg, u, f)) return -1;
        k++;
        double rk = or_norm(cfg, 0, u, f);
        if (history) history[k] = rk;
        if (!isfinite(rk)) return -1;
        if (rk <= rtol * r0) break;
    }
    return k;
}
