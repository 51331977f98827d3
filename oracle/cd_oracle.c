/*
 * cd_oracle.c — plain CPU oracle of the cell-centred complex-diffusion FAS
 * V-cycle (see cd_oracle.h for the problem, the canonical arithmetic and the
 * citations).  TEST INFRASTRUCTURE ONLY.  Straight loops, one function per
 * step of the method, in the paper's order.
 */
#include "cd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    real re, im;
} cplx;

static cplx cmul(cplx a, cplx b) {
    cplx r;
    r.re = a.re * b.re - a.im * b.im;
    r.im = a.re * b.im + a.im * b.re;
    return r;
}
static cplx cdiv(cplx x, cplx y) {
    const real den = y.re * y.re + y.im * y.im;
    cplx r;
    r.re = (x.re * y.re + x.im * y.im) / den;
    r.im = (x.im * y.re - x.re * y.im) / den;
    return r;
}

typedef struct {
    int nx, ny, nz;       /* cells of the level (nz = 1 in 2D) */
    real w[3];            /* tau / h_{l,d}^2 */
} clvl;

static clvl level_of(const cd_config* c, int l) {
    clvl L;
    L.nx = c->n[0] >> l;
    L.ny = c->n[1] >> l;
    L.nz = c->dim == 3 ? (c->n[2] >> l) : 1;
    for (int d = 0; d < 3; d++) {
        const double h = ldexp(c->h[d], l);
        L.w[d] = d < c->dim ? (real)(c->tau / (h * h)) : (real)0;
    }
    return L;
}

int64_t cd_level_cells(const cd_config* c, int l) {
    const clvl L = level_of(c, l);
    return (int64_t)L.nx * L.ny * L.nz;
}

static cplx at(const real* a, int64_t q) {
    cplx r;
    r.re = a[2 * q];
    r.im = a[2 * q + 1];
    return r;
}
static void put(real* a, int64_t q, cplx v) {
    a[2 * q] = v.re;
    a[2 * q + 1] = v.im;
}

/* Eq. 3: g(s) = e^{i theta} / (1 + (s/(k theta))^2) */
void cd_diffusivity(const cd_config* c, real s, real out[2]) {
    const real kth = (real)(c->kappa * c->theta);
    const real ct = (real)cos(c->theta), st = (real)sin(c->theta);
    const real q = s / kth;
    const real den = (real)1 + q * q;
    out[0] = ct / den;
    out[1] = st / den;
}

void cd_gfield(const cd_config* c, int l, const real* ul, real* g) {
    const int64_t n = cd_level_cells(c, l);
    for (int64_t q = 0; q < n; q++) cd_diffusivity(c, ul[2 * q + 1], g + 2 * q);
}

/* (A u)(c) and a_c at cell (i,j,k), faces x-, x+, y-, y+, z-, z+ */
static void point_apply(const clvl* L, int dim, const real* g, const real* u, int i, int j, int k, cplx* Au,
                        cplx* diag) {
    const int64_t sy = L->nx, sz = (int64_t)L->nx * L->ny;
    const int64_t q = (int64_t)k * sz + (int64_t)j * sy + i;
    const cplx gc = at(g, q);
    cplx acc_a = {0, 0}, acc_s = {0, 0};
    const int idx[3] = {i, j, k};
    const int ext[3] = {L->nx, L->ny, L->nz};
    const int64_t str[3] = {1, sy, sz};
    for (int d = 0; d < dim; d++) {
        for (int side = -1; side <= 1; side += 2) {
            const int nb = idx[d] + side;
            if (nb < 0 || nb >= ext[d]) continue;  /* boundary face: zero flux */
            const int64_t qn = q + side * str[d];
            const cplx gn = at(g, qn);
            cplx gf, cf;
            gf.re = (real)0.5 * (gc.re + gn.re);
            gf.im = (real)0.5 * (gc.im + gn.im);
            cf.re = L->w[d] * gf.re;
            cf.im = L->w[d] * gf.im;
            acc_a.re = acc_a.re + cf.re;
            acc_a.im = acc_a.im + cf.im;
            const cplx t = cmul(cf, at(u, qn));
            acc_s.re = acc_s.re + t.re;
            acc_s.im = acc_s.im + t.im;
        }
    }
    diag->re = (real)1 + acc_a.re;
    diag->im = acc_a.im;
    const cplx du = cmul(*diag, at(u, q));
    Au->re = du.re - acc_s.re;
    Au->im = du.im - acc_s.im;
}

void cd_apply(const cd_config* c, int l, const real* g, const real* u, real* Au, real* diag) {
    const clvl L = level_of(c, l);
    for (int k = 0; k < L.nz; k++)
        for (int j = 0; j < L.ny; j++)
            for (int i = 0; i < L.nx; i++) {
                cplx a, d;
                point_apply(&L, c->dim, g, u, i, j, k, &a, &d);
                const int64_t q = ((int64_t)k * L.ny + j) * L.nx + i;
                put(Au, q, a);
                if (diag) put(diag, q, d);
            }
}

/* u' = u + omega * (f - A u) / a_c at one cell (reading u from `src`) */
static cplx relax(const cd_config* c, const clvl* L, const real* g, const real* src, const real* f, int i, int j,
                  int k) {
    cplx a, d;
    point_apply(L, c->dim, g, src, i, j, k, &a, &d);
    const int64_t q = ((int64_t)k * L->ny + j) * L->nx + i;
    const cplx fu = at(f, q), uu = at(src, q);
    cplx r;
    r.re = fu.re - a.re;
    r.im = fu.im - a.im;
    const cplx z = cdiv(r, d);
    const real om = (real)c->omega;
    cplx o;
    o.re = uu.re + om * z.re;
    o.im = uu.im + om * z.im;
    return o;
}

void cd_smooth(const cd_config* c, int l, const real* g, real* u, const real* f) {
    const clvl L = level_of(c, l);
    const int64_t n = cd_level_cells(c, l);
    if (c->smoother == 0) { /* omega-Jacobi: all reads from the old iterate (reading 9) */
        real* old = (real*)malloc(sizeof(real) * 2 * n);
        memcpy(old, u, sizeof(real) * 2 * n);
        for (int k = 0; k < L.nz; k++)
            for (int j = 0; j < L.ny; j++)
                for (int i = 0; i < L.nx; i++)
                    put(u, ((int64_t)k * L.ny + j) * L.nx + i, relax(c, &L, g, old, f, i, j, k));
        free(old);
        return;
    }
    for (int colour = 0; colour < 2; colour++) /* red (even i+j+k) first, in place */
        for (int k = 0; k < L.nz; k++)
            for (int j = 0; j < L.ny; j++)
                for (int i = 0; i < L.nx; i++)
                    if (((i + j + k) & 1) == colour)
                        put(u, ((int64_t)k * L.ny + j) * L.nx + i, relax(c, &L, g, u, f, i, j, k));
}

/* coarse cell = average of its 2^d children; sums x, then y, then z, times 2^-d */
void cd_restrict(const cd_config* c, int l, const real* vf, real* vc) {
    const clvl F = level_of(c, l), C = level_of(c, l + 1);
    const real scale = (real)ldexp(1.0, -c->dim);
    for (int K = 0; K < C.nz; K++)
        for (int J = 0; J < C.ny; J++)
            for (int I = 0; I < C.nx; I++) {
                cplx sz[2];
                const int nkz = c->dim == 3 ? 2 : 1;
                for (int dz = 0; dz < nkz; dz++) {
                    cplx sy[2];
                    for (int dy = 0; dy < 2; dy++) {
                        const int k = c->dim == 3 ? 2 * K + dz : 0, j = 2 * J + dy;
                        const int64_t q = ((int64_t)k * F.ny + j) * F.nx + 2 * I;
                        const cplx a = at(vf, q), b = at(vf, q + 1);
                        sy[dy].re = a.re + b.re;
                        sy[dy].im = a.im + b.im;
                    }
                    sz[dz].re = sy[0].re + sy[1].re;
                    sz[dz].im = sy[0].im + sy[1].im;
                }
                cplx s = sz[0];
                if (c->dim == 3) {
                    s.re = sz[0].re + sz[1].re;
                    s.im = sz[0].im + sz[1].im;
                }
                cplx o;
                o.re = s.re * scale;
                o.im = s.im * scale;
                put(vc, ((int64_t)K * C.ny + J) * C.nx + I, o);
            }
}

/* fine cell gets the value of its parent cell floor(c/2) */
void cd_prolong_add(const cd_config* c, int l, const real* ec, real* uf) {
    const clvl F = level_of(c, l), C = level_of(c, l + 1);
    for (int k = 0; k < F.nz; k++)
        for (int j = 0; j < F.ny; j++)
            for (int i = 0; i < F.nx; i++) {
                const int K = c->dim == 3 ? k / 2 : 0;
                const cplx e = at(ec, ((int64_t)K * C.ny + j / 2) * C.nx + i / 2);
                const int64_t q = ((int64_t)k * F.ny + j) * F.nx + i;
                cplx u = at(uf, q);
                u.re = u.re + e.re;
                u.im = u.im + e.im;
                put(uf, q, u);
            }
}

double cd_norm(const cd_config* c, int l, const real* u, const real* f) {
    const int64_t n = cd_level_cells(c, l);
    real* g = (real*)malloc(sizeof(real) * 2 * n);
    real* Au = (real*)malloc(sizeof(real) * 2 * n);
    cd_gfield(c, l, u, g);
    cd_apply(c, l, g, u, Au, NULL);
    double s = 0.0;
    for (int64_t q = 0; q < n; q++) {
        const double rr = (double)(f[2 * q] - Au[2 * q]), ri = (double)(f[2 * q + 1] - Au[2 * q + 1]);
        s += rr * rr + ri * ri;
    }
    free(g);
    free(Au);
    return sqrt(s);
}

typedef struct {
    real *u, *f, *uh, *g;
} clevel;

/* FAS V-cycle at level l */
static void fas_rec(const cd_config* c, clevel* H, int l) {
    clevel* X = &H[l];
    const int64_t n = cd_level_cells(c, l);
    cd_gfield(c, l, X->u, X->g); /* lagged diffusivity: rebuilt once per cycle, frozen */
    if (l == c->levels - 1) {
        for (int s = 0; s < c->ncoarse; s++) cd_smooth(c, l, X->g, X->u, X->f);
        return;
    }
    for (int s = 0; s < c->nu1; s++) cd_smooth(c, l, X->g, X->u, X->f);
    clevel* Y = &H[l + 1];
    const int64_t m = cd_level_cells(c, l + 1);
    cd_restrict(c, l, X->u, Y->uh); /* u^_H = R u_h */
    memcpy(Y->u, Y->uh, sizeof(real) * 2 * m);
    /* f_H = A_H(u^_H) u^_H + R (f_h - A_h u_h) */
    real* Au = (real*)malloc(sizeof(real) * 2 * n);
    cd_apply(c, l, X->g, X->u, Au, NULL);
    for (int64_t q = 0; q < 2 * n; q++) Au[q] = X->f[q] - Au[q];
    real* Rr = (real*)malloc(sizeof(real) * 2 * m);
    cd_restrict(c, l, Au, Rr);
    real* gH = (real*)malloc(sizeof(real) * 2 * m);
    real* AH = (real*)malloc(sizeof(real) * 2 * m);
    cd_gfield(c, l + 1, Y->uh, gH);
    cd_apply(c, l + 1, gH, Y->uh, AH, NULL);
    for (int64_t q = 0; q < 2 * m; q++) Y->f[q] = AH[q] + Rr[q];
    free(Au);
    free(Rr);
    free(gH);
    free(AH);
    fas_rec(c, H, l + 1);
    /* u_h += P (u_H - u^_H) */
    real* e = (real*)malloc(sizeof(real) * 2 * m);
    for (int64_t q = 0; q < 2 * m; q++) e[q] = Y->u[q] - Y->uh[q];
    cd_prolong_add(c, l, e, X->u);
    free(e);
    for (int s = 0; s < c->nu2; s++) cd_smooth(c, l, X->g, X->u, X->f);
}

int cd_cycle(const cd_config* c, real* u, const real* f) {
    clevel* H = (clevel*)calloc((size_t)c->levels, sizeof(clevel));
    if (!H) return -1;
    int ok = 1;
    for (int l = 0; l < c->levels; l++) {
        const int64_t n = cd_level_cells(c, l);
        H[l].g = (real*)malloc(sizeof(real) * 2 * n);
        if (l > 0) {
            H[l].u = (real*)malloc(sizeof(real) * 2 * n);
            H[l].f = (real*)malloc(sizeof(real) * 2 * n);
            H[l].uh = (real*)malloc(sizeof(real) * 2 * n);
            ok = ok && H[l].u && H[l].f && H[l].uh;
        }
        ok = ok && H[l].g;
    }
    if (ok) {
        H[0].u = u;
        H[0].f = (real*)f;
        fas_rec(c, H, 0);
    }
    for (int l = 0; l < c->levels; l++) {
        free(H[l].g);
        if (l > 0) {
            free(H[l].u);
            free(H[l].f);
            free(H[l].uh);
        }
    }
    free(H);
    return ok ? 0 : -1;
}

int cd_solve(const cd_config* c, real* u, const real* f, double rtol, int max_cycles, double* history) {
    const double r0 = cd_norm(c, 0, u, f);
    history[0] = r0;
    if (!isfinite(r0)) return -1;
    int k = 0;
    while (k < max_cycles) {
        if (cd_cycle(c, u, f) != 0) return -1;
        k++;
        const double rk = cd_norm(c, 0, u, f);
        history[k] = rk;
        if (!isfinite(rk)) return -1;
        if (rk <= rtol * r0) break;
    }
    return k;
}
