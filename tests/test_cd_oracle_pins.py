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
