"""Pins of the complex-diffusion FAS oracle (oracle/cd_oracle.c) against what the
paper, SPEC and the mathematics fix — dense matrices assembled here from the
definitions (never from the oracle), closed forms, SPEC's worked examples,
fixed-point and linear-equivalence properties of FAS, and the paper's 10^5 claim.

P:521-535 (Eqs. 2-3, FAS, lagged diffusivity, cell-centred transfers)
(discretisation and its examples), S:337-342 (transfers), S:431-439 (FAS)."""
import math

import numpy as np
import pytest

from oracle.cd import CDConfig, CDOracle, JACOBI, RBGS
from paper_1406_5369_b200 import workloads as wl

TH, KA, TAU = math.pi / 30, 2.0, 0.1


def rand_c(shape, seed, scale=1.0):
    r = np.random.default_rng(seed)
    return (scale * (r.uniform(-1, 1, shape) + 1j * r.uniform(-1, 1, shape))).astype(np.complex128)


# ------------------------------------------------------------------ dense definitions
def g_of(s, theta=TH, kappa=KA):
    """Eq. 3 written out: e^{i theta} / (1 + (s/(k theta))^2)."""
    return np.exp(1j * theta) / (1.0 + (s / (kappa * theta)) ** 2)


def dense_A(g, h, tau=TAU):
    """A = I - tau div(g grad) by averaged FD; g per cell, boundary faces dropped."""
    shape = g.shape
    n = g.size
    idx = np.arange(n).reshape(shape)
    A = np.zeros((n, n), complex)
    dim = g.ndim
    for q in np.ndindex(shape):
        p = idx[q]
        A[p, p] += 1.0
        for ax in range(dim):  # array axes: (y, x) or (z, y, x); h given per array axis
            for s in (-1, 1):
                nb = list(q)
                nb[ax] += s
                if nb[ax] < 0 or nb[ax] >= shape[ax]:
                    continue
                gf = 0.5 * (g[q] + g[tuple(nb)])
                w = tau / h[ax] ** 2
                A[p, p] += w * gf
                A[p, idx[tuple(nb)]] -= w * gf
    return A


def dense_R(shape):
    """coarse cell = mean of its 2^d children."""
    dim = len(shape)
    cs = tuple(s // 2 for s in shape)
    R = np.zeros((int(np.prod(cs)), int(np.prod(shape))))
    ci = np.arange(R.shape[0]).reshape(cs)
    fi = np.arange(R.shape[1]).reshape(shape)
    for q in np.ndindex(shape):
        R[ci[tuple(x // 2 for x in q)], fi[q]] = 2.0 ** -dim
    return R


def dense_P(shape):
    """constant injection (each fine cell takes its parent's value)."""
    dim = len(shape)
    return dense_R(shape).T * 2.0 ** dim


def color_mask(shape, colour):
    return np.array([(sum(q) & 1) == colour for q in np.ndindex(shape)])


def dense_smooth(A, f, u, omega, smoother, shape):
    D = np.diag(A)
    if smoother == JACOBI:
        return u + omega * (f - A @ u) / D
    for colour in (0, 1):  # red (even index sum) first
        m = color_mask(shape, colour)
        u = u + m * omega * (f - A @ u) / D
    return u


# ------------------------------------------------------------------ pins
def test_diffusivity_spec_examples():
    O = CDOracle(CDConfig(dim=2, cells=(4, 4)))
    assert abs(O.diffusivity(0.0) - np.exp(1j * TH)) < 1e-15
    assert abs(O.diffusivity(KA * TH) - np.exp(1j * TH) / 2) < 1e-15
    vals = [abs(O.diffusivity(s)) for s in (0.0, 0.1, 0.5, 2.0, 50.0)]
    assert all(a > b for a, b in zip(vals, vals[1:])) and vals[0] <= 1.0
    assert O.diffusivity(0.3) == O.diffusivity(-0.3)                        # even


@pytest.mark.parametrize("dim,cells", [(2, (6, 4)), (2, (8, 8)), (3, (4, 4, 2))])
def test_operator_equals_dense_assembly(dim, cells):
    cfg = CDConfig(dim=dim, cells=cells)
    O = CDOracle(cfg)
    shape = cfg.shape(0)
    ul = rand_c(shape, 1, 0.5)
    u = rand_c(shape, 2)
    g = O.gfield(0, ul)
    np.testing.assert_allclose(g, g_of(ul.imag), rtol=1e-15, atol=0)
    Au, diag = O.apply(0, g, u)
    h = [1.0 / c for c in reversed(cells)]  # per array axis
    A = dense_A(g, h)
    np.testing.assert_allclose(Au.ravel(), A @ u.ravel(), rtol=1e-13, atol=1e-12 * np.abs(A @ u.ravel()).max())
    np.testing.assert_allclose(diag.ravel(), np.diag(A), rtol=1e-14)


def test_operator_spec_examples():
    """real constant lagged field -> g = e^{i theta}, interior centre 1 + 4 tau e^{i theta}/h^2,
    neighbours -tau e^{i theta}/h^2; corner cell centre 1 + 2 tau g/h^2; a 1x1 grid is the identity."""
    cfg = CDConfig(dim=2, cells=(4, 4), levels=1)
    O = CDOracle(cfg)
    g = O.gfield(0, np.full((4, 4), 0.7 + 0j))
    e = np.zeros((4, 4), complex)
    e[1, 1] = 1.0
    Au, diag = O.apply(0, g, e)
    w = TAU * 16.0
    ge = np.exp(1j * TH)
    assert abs(diag[1, 1] - (1 + 4 * w * ge)) < 1e-12
    assert abs(diag[0, 0] - (1 + 2 * w * ge)) < 1e-12
    assert abs(Au[1, 2] - (-w * ge)) < 1e-12 and abs(Au[0, 1] - (-w * ge)) < 1e-12
    assert Au[3, 3] == 0
    O1 = CDOracle(CDConfig(dim=2, cells=(1, 1), levels=1))
    u1 = np.array([[0.3 - 0.2j]])
    Au1, d1 = O1.apply(0, O1.gfield(0, u1), u1)
    assert Au1[0, 0] == u1[0, 0] and d1[0, 0] == 1


def test_constants_in_kernel_of_flux():
    """Zero-flux Neumann: A c = c for a constant field (the diffusion part annihilates constants)."""
    cfg = CDConfig(dim=3, cells=(4, 4, 4))
    O = CDOracle(cfg)
    g = O.gfield(0, rand_c(cfg.shape(), 3))
    c = np.full(cfg.shape(), 0.25 - 0.5j)
    Au, _ = O.apply(0, g, c)
    np.testing.assert_allclose(Au, c, rtol=0, atol=1e-11)


@pytest.mark.parametrize("smoother,omega", [(JACOBI, 0.8), (RBGS, 1.0), (RBGS, 1.15)])
@pytest.mark.parametrize("dim,cells", [(2, (8, 6)), (3, (4, 4, 4))])
def test_smoother_equals_dense(smoother, omega, dim, cells):
    cfg = CDConfig(dim=dim, cells=cells, smoother=smoother, omega=omega)
    O = CDOracle(cfg)
    shape = cfg.shape()
    g = O.gfield(0, rand_c(shape, 4, 0.3))
    u, f = rand_c(shape, 5), rand_c(shape, 6)
    got = O.smooth(0, g, u, f)
    A = dense_A(g, [1.0 / c for c in reversed(cells)])
    ref = dense_smooth(A, f.ravel(), u.ravel(), omega, smoother, shape)
    np.testing.assert_allclose(got.ravel(), ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("dim,cells", [(2, (8, 4)), (3, (4, 4, 2))])
def test_transfers_equal_dense(dim, cells):
    cfg = CDConfig(dim=dim, cells=cells)
    O = CDOracle(cfg)
    shape = cfg.shape()
    v = rand_c(shape, 7)
    R = dense_R(shape)
    np.testing.assert_allclose(O.restrict(0, v).ravel(), R @ v.ravel(), rtol=1e-15, atol=1e-16)
    e = rand_c(cfg.shape(1), 8)
    u = rand_c(shape, 9)
    P = dense_P(shape)
    np.testing.assert_allclose(O.prolong_add(0, e, u).ravel(), u.ravel() + P @ e.ravel(), rtol=1e-15)
    np.testing.assert_array_equal(R, P.T / 2 ** dim)  # R = 2^-d P^T


def test_restriction_spec_example():
    O = CDOracle(CDConfig(dim=2, cells=(2, 2)))
    assert O.restrict(0, np.array([[1, 2], [3, 4]], complex))[0, 0] == 2.5


def test_fas_fixed_point():
    """a converged iterate is a fixed point of the FAS cycle (zero residual ->
    zero coarse correction, smoothing does nothing)."""
    cfg = CDConfig(dim=2, cells=(16, 16), levels=3)
    O = CDOracle(cfg)
    us = rand_c(cfg.shape(), 10, 0.3)
    A = dense_A(g_of(us.imag), [1 / 16, 1 / 16])
    f = (A @ us.ravel()).reshape(us.shape)
    out = O.cycle(us, f)
    assert np.abs(out - us).max() <= 1e-12 * np.abs(us).max()


@pytest.mark.parametrize("smoother,omega", [(JACOBI, 0.8), (RBGS, 1.0)])
def test_fas_with_linear_operator_equals_correction_scheme(smoother, omega):
    """with a linear operator (k -> infinity makes g = e^{i theta} exactly) the FAS
    cycle equals the correction-scheme V-cycle, here evaluated in dense algebra
    (3 levels, coarsest = ncoarse sweeps from a zero correction)."""
    cells = (16, 8)
    cfg = CDConfig(dim=2, cells=cells, levels=3, smoother=smoother, omega=omega, kappa=1e30, ncoarse=4)
    O = CDOracle(cfg)
    shapes = [cfg.shape(l) for l in range(3)]
    As = [dense_A(np.full(s, np.exp(1j * TH)), [2.0 ** l / cells[1], 2.0 ** l / cells[0]]) for l, s in enumerate(shapes)]

    def cs(l, u, f):
        sh = shapes[l]
        if l == 2:
            for _ in range(cfg.ncoarse):
                u = dense_smooth(As[l], f, u, omega, smoother, sh)
            return u
        for _ in range(cfg.nu1):
            u = dense_smooth(As[l], f, u, omega, smoother, sh)
        r = dense_R(sh) @ (f - As[l] @ u)
        e = cs(l + 1, np.zeros(r.size, complex), r)
        u = u + dense_P(sh) @ e
        for _ in range(cfg.nu2):
            u = dense_smooth(As[l], f, u, omega, smoother, sh)
        return u

    u0, f = rand_c(shapes[0], 11), rand_c(shapes[0], 12)
    ref = cs(0, u0.ravel(), f.ravel())
    got = O.cycle(u0, f).ravel()
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("smoother,omega", [(RBGS, 1.0), (JACOBI, 0.8)])
def test_paper_claim_1e5_in_five_cycles(smoother, omega):
    """'for complex diffusion [the residual is reduced] by a factor of 10^5' within
    5 V(2,2) cycles; SPEC S:632's configuration: 128^2 cells, Neumann, one implicit-Euler
    step, tau = 0.1, theta = pi/30, k = 2, noisy-image initial state (W5)."""
    cfg = CDConfig(dim=2, cells=(128, 128), smoother=smoother, omega=omega)
    O = CDOracle(cfg)
    u, f = wl.cd_workload(2, (128, 128), 42)
    _, k, hist = O.solve(u, f, 0.0, 5)
    assert k == 5 and hist[5] <= 1e-5 * hist[0], hist / hist[0]


def test_fp32_build_tracks_fp64():
    cfg = CDConfig(dim=2, cells=(32, 32))
    u, f = wl.cd_workload(2, (32, 32), 3)
    a = CDOracle(cfg).cycle(u, f)
    b = CDOracle(cfg, np.complex64).cycle(u.astype(np.complex64), f.astype(np.complex64))
    assert np.abs(a - b).max() <= 1e-5 * np.abs(a).max()


# ------------------------------------------------------------------ the nonlinear residual norm
@pytest.mark.parametrize("dim,cells", [(2, (6, 4)), (2, (9, 9)), (3, (4, 3, 2))])
def test_norm_equals_dense_nonlinear_residual(dim, cells):
    """S:540-548 (l2_residual): sqrt of the sum over the cells of |f - A u|^2 with the complex
    modulus, where for complex diffusion A = A(g(u)) is assembled from the diffusivity of the
    iterate whose residual is taken (reading 21: the driver loop's norm is the nonlinear
    residual).  Dense A from the definition (dense_A, g_of); negative controls: the squared sum
    (no sqrt), the real parts only, and A built from a different (lagged) field all differ."""
    cfg = CDConfig(dim=dim, cells=cells)
    O = CDOracle(cfg)
    shape = cfg.shape()
    u, f = rand_c(shape, 21, 0.8), rand_c(shape, 22)
    h = [1.0 / c for c in reversed(cells)]
    r = f.ravel() - dense_A(g_of(u.imag), h) @ u.ravel()
    ref = math.sqrt(float(np.sum(r.real ** 2 + r.imag ** 2)))
    got = O.norm(0, u, f)
    assert abs(got - ref) <= 1e-14 * ref, (got, ref)
    assert abs(got ** 2 - ref) > 1e-3 * ref                                  # sqrt taken
    assert abs(got - np.linalg.norm(r.real)) > 1e-3 * ref                     # complex modulus
    lag = rand_c(shape, 23, 0.8)                                              # g from another field
    r_lag = f.ravel() - dense_A(g_of(lag.imag), h) @ u.ravel()
    assert abs(got - np.linalg.norm(r_lag)) > 1e-6 * ref


def test_norm_spec_examples():
    """u = 0, f = 1 on m cells -> sqrt(m); the exact solution of a 1-cell system -> 0."""
    cfg = CDConfig(dim=2, cells=(5, 7), levels=1)
    O = CDOracle(cfg)
    assert O.norm(0, np.zeros(cfg.shape(), complex), np.ones(cfg.shape(), complex)) == math.sqrt(35)
    O1 = CDOracle(CDConfig(dim=2, cells=(1, 1), levels=1))
    u1 = np.array([[0.4 - 0.9j]])
    assert O1.norm(0, u1, u1) == 0.0  # A = I on one cell (no interior faces)


# ------------------------------------------------------------------ FAS with the nonlinear operator
def dense_fas(u, f, cells, levels, smoother, omega, nu1, nu2, ncoarse, coarse_g="restricted_u"):
    """S:431-439 / S:355 written out in dense algebra, nonlinear operator, recursion over `levels`.
    At every level visit the lagged diffusivity g = g(Im u_l) is formed ONCE from the level's
    current iterate ('rebuilt from the current solution once per cycle before smoothing,
    frozen within the cycle'); the coarse operator of the FAS right-hand side is re-discretised
    from the restricted iterate u^_H = R u_h (S:355 'ComplexDiffusion: rebuilt from the restricted
    lagged solution'; S:434 'f_H = A_H(u^_H) + R(f_h - A_h u_h)').  coarse_g selects a WRONG rule
    for the negative controls ('restricted_g': g_H = R g_h; 'fine_lagged': g_H = g(R u_h at the
    START of the cycle, before pre-smoothing))."""
    dim = len(cells)
    shapes = [tuple(c >> l for c in reversed(cells)) for l in range(levels)]

    def hs(l):
        return [2.0 ** l / c for c in reversed(cells)]

    def rec(l, u, f, g_hint=None):
        sh = shapes[l]
        g = g_of(u.reshape(sh).imag) if g_hint is None else g_hint
        A = dense_A(g, hs(l))
        if l == levels - 1:
            for _ in range(ncoarse):
                u = dense_smooth(A, f, u, omega, smoother, sh)
            return u
        u_start = u.copy()
        for _ in range(nu1):
            u = dense_smooth(A, f, u, omega, smoother, sh)
        R, P = dense_R(sh), dense_P(sh)
        uh = R @ u
        if coarse_g == "restricted_u":
            gH = g_of(uh.reshape(shapes[l + 1]).imag)
        elif coarse_g == "restricted_g":
            gH = (R @ g.ravel()).reshape(shapes[l + 1])
        else:
            gH = g_of((R @ u_start).reshape(shapes[l + 1]).imag)
        AH = dense_A(gH, hs(l + 1))
        fH = AH @ uh + R @ (f - A @ u)
        uH = rec(l + 1, uh.copy(), fH, None if coarse_g == "restricted_u" else gH)
        u = u + P @ (uH - uh)
        for _ in range(nu2):
            u = dense_smooth(A, f, u, omega, smoother, sh)
        return u

    return rec(0, u.ravel(), f.ravel()).reshape(shapes[0])


@pytest.mark.parametrize("smoother,omega,levels,cells", [(RBGS, 1.0, 2, (8, 8)), (JACOBI, 0.8, 2, (8, 4)),
                                                         (RBGS, 1.0, 3, (16, 8)), (JACOBI, 0.8, 2, (4, 4, 4))])
def test_fas_nonlinear_cycle_equals_dense(smoother, omega, levels, cells):
    """one nonlinear FAS V(2,2) cycle of the oracle equals the cycle
    evaluated in dense algebra with the coarse operator rebuilt from g(R u_h), for a strongly
    nonlinear state (|Im u| ~ 1 >> k*theta = 0.21, so g varies by ~10x over the grid).  Negative
    controls: the same dense cycle with the coarse diffusivity taken from R g_h, or from R of the
    pre-smoothing iterate, differs from the oracle by far more than the tolerance."""
    dim = len(cells)
    cfg = CDConfig(dim=dim, cells=cells, levels=levels, smoother=smoother, omega=omega, ncoarse=3)
    O = CDOracle(cfg)
    u0, f = rand_c(cfg.shape(), 31, 1.0), rand_c(cfg.shape(), 32, 1.0)
    got = O.cycle(u0, f)
    ref = dense_fas(u0, f, cells, levels, smoother, omega, 2, 2, 3)
    scale = np.abs(ref).max()
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12 * scale)
    for wrong in ("restricted_g", "fine_lagged"):
        bad = dense_fas(u0, f, cells, levels, smoother, omega, 2, 2, 3, coarse_g=wrong)
        assert np.abs(bad - ref).max() > 1e-6 * scale, wrong


def test_fp32_build_ops_within_rounding_bound_of_dense():
    """The complex64 oracle build, op by op, against the dense FP64 definitions applied to the
    same complex64 inputs: g (Eq. 3), A(g)u, the omega-Jacobi sweep and the cell-average
    restriction, each within a bound of a few float32 roundings per term."""
    eps = float(np.finfo(np.float32).eps)
    cells = (8, 6)
    cfg = CDConfig(dim=2, cells=cells, smoother=JACOBI, omega=0.8)
    O = CDOracle(cfg, np.complex64)
    shape = cfg.shape()
    ul = rand_c(shape, 51, 0.5).astype(np.complex64)
    u, f = rand_c(shape, 52).astype(np.complex64), rand_c(shape, 53).astype(np.complex64)
    g = O.gfield(0, ul)
    g_ref = g_of(ul.imag.astype(np.float64))
    assert np.all(np.abs(g - g_ref) <= 8 * eps * np.abs(g_ref))
    g64 = g.astype(np.complex128)
    h = [1.0 / c for c in reversed(cells)]
    A = dense_A(g64, h)
    u64, f64 = u.astype(np.complex128).ravel(), f.astype(np.complex128).ravel()
    Au, _ = O.apply(0, g, u)
    absAu = np.abs(A) @ np.abs(u64)
    assert np.all(np.abs(Au.ravel() - A @ u64) <= 24 * eps * absAu)
    out = O.smooth(0, g, u, f).ravel()
    ref = dense_smooth(A, f64, u64, 0.8, JACOBI, shape)
    D = np.abs(np.diag(A))
    assert np.all(np.abs(out - ref) <= 48 * eps * (np.abs(u64) + (np.abs(f64) + absAu) / D))
    rc = O.restrict(0, f).ravel()
    assert np.all(np.abs(rc - dense_R(shape) @ f64) <= 8 * eps * (dense_R(shape) @ np.abs(f64)))
