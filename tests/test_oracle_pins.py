"""Pins of the CPU oracle against what the paper and the mathematics fix
(DESIGN.md §5).  CPU only.  None of these re-types the oracle's formula:
each compares it with a dense brute-force matrix built from the definitions
(tests/dense.py), a closed form, an invariant, or an externally computed value.
"""
import json
import math
import os

import numpy as np
import pytest

import dense
import oracle as orc
from paper_1406_5369_b200 import workloads as wl

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "survey_dense_vcycle.json")))


def cfg(dim, cells, levels=0, smoother="rbgs", omega=None, nu1=2, nu2=2, coarse=orc.COARSE_DIRECT, ncoarse=10):
    sm = {"rbgs": orc.RBGS, "gs_lex": orc.GS_LEX}.get(smoother, orc.JACOBI)
    if omega is None:
        omega = 0.8 if sm == orc.JACOBI else 1.0
    return orc.Config(dim=dim, cells=tuple(cells), levels=levels, smoother=sm, omega=omega,
                      nu1=nu1, nu2=nu2, coarse=coarse, ncoarse=ncoarse)


def rnd(shape, seed, interior_only=True):
    r = np.random.default_rng(seed).uniform(-1, 1, size=shape)
    if interior_only:
        m = np.zeros(shape, bool)
        m[(slice(1, -1),) * len(shape)] = True
        r[~m] = 0.0
    return r


SMALL = [(2, (8, 8)), (2, (16, 8)), (3, (8, 8, 8)), (3, (8, 4, 16))]


# ---------------------------------------------------------------- operator A
@pytest.mark.parametrize("dim,cells", SMALL)
def test_residual_equals_dense_matvec(dim, cells):
    """stencil application equals the dense assembled matvec."""
    O = orc.Oracle(cfg(dim, cells, levels=1))
    u, f = rnd(O.shape(0), 1), rnd(O.shape(0), 2)
    c, D, _ = dense.coeffs(list(cells), 0)
    A = dense.assemble_A(list(cells), c)
    r = O.residual(0, u, f)
    ref = dense.interior(f) - A @ dense.interior(u)
    np.testing.assert_allclose(dense.interior(r), ref, rtol=0, atol=1e-12 * np.abs(A).max())
    # boundary of r is zero
    assert np.all(r[~np.pad(np.ones([s - 2 for s in r.shape], bool), 1)] == 0)


@pytest.mark.parametrize("dim,cells", [(2, (32, 32)), (3, (16, 16, 16))])
def test_sine_mode_eigenvalue(dim, cells):
    """Closed form: A phi_k = sum_d 4 c_d sin^2(k_d pi h_d / 2) phi_k."""
    O = orc.Oracle(cfg(dim, cells, levels=1))
    xs = wl.coords(dim, cells)
    for k in [(1, 1, 1), (3, 7, 2), (cells[0] - 1, 1, cells[-1] - 1)]:
        phi = np.ones(O.shape(0))
        lam = 0.0
        for d in range(dim):
            phi = phi * np.sin(k[d] * np.pi * xs[d])
            h = 1.0 / cells[d]
            lam += 4.0 / h ** 2 * math.sin(k[d] * math.pi * h / 2) ** 2
        r = O.residual(0, phi, np.zeros_like(phi))  # r = -A phi
        np.testing.assert_allclose(-dense.interior(r), lam * dense.interior(phi), rtol=0,
                                   atol=1e-9 * lam)


def test_polynomial_is_discretely_exact():
    """W3: u* = prod x(1-x) has -Delta_h u* = -Delta u* exactly (quadratic per axis)."""
    for dim, cells in [(2, (16, 16)), (3, (8, 8, 8))]:
        O = orc.Oracle(cfg(dim, cells, levels=1))
        _, f = wl.workload("W3", dim, cells)
        us = wl.exact_solution("W3", dim, cells)
        r = O.residual(0, us, f)
        assert np.abs(r).max() < 1e-12 * np.abs(f).max()


# ---------------------------------------------------------------- smoothers
@pytest.mark.parametrize("dim,cells", SMALL)
@pytest.mark.parametrize("omega", [0.8, 1.0, 0.0])
def test_jacobi_equals_dense(dim, cells, omega):
    """one Jacobi sweep equals u + omega D^-1 (f - A u); omega=0 is identity."""
    O = orc.Oracle(cfg(dim, cells, levels=1, smoother="jacobi", omega=omega))
    u, f = rnd(O.shape(0), 3), rnd(O.shape(0), 4)
    c, D, _ = dense.coeffs(list(cells), 0)
    A = dense.assemble_A(list(cells), c)
    out = O.jacobi(0, u, f)
    ref = dense.jacobi(A, D, omega, dense.interior(u), dense.interior(f))
    np.testing.assert_allclose(dense.interior(out), ref, rtol=1e-13, atol=1e-13)
    if omega == 0.0:
        assert np.array_equal(out, u)


@pytest.mark.parametrize("dim,cells", SMALL)
@pytest.mark.parametrize("omega", [1.0, 1.15])
def test_rbgs_equals_dense(dim, cells, omega):
    """One RBGS sweep = S_B S_R with S_C = I - omega E_C D^-1 A (red first, reading 8)."""
    O = orc.Oracle(cfg(dim, cells, levels=1, smoother="rbgs", omega=omega))
    u, f = rnd(O.shape(0), 5), rnd(O.shape(0), 6)
    c, D, _ = dense.coeffs(list(cells), 0)
    A = dense.assemble_A(list(cells), c)
    out = O.rbgs(0, u, f)
    ref = dense.rbgs(A, D, omega, dense.interior(u), dense.interior(f), list(cells))
    np.testing.assert_allclose(dense.interior(out), ref, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("dim,cells", SMALL)
@pytest.mark.parametrize("omega", [1.0, 1.2])
def test_gs_lex_equals_dense_sor(dim, cells, omega):
    """Lexicographic omega-GS (Table 1, S:416 'order lex') = the SOR matrix iteration
    u + omega (D - omega L)^-1 (f - A u), L the strictly lower part in row-major order."""
    O = orc.Oracle(cfg(dim, cells, levels=1, smoother="gs_lex", omega=omega))
    u, f = rnd(O.shape(0), 25), rnd(O.shape(0), 26)
    c, D, _ = dense.coeffs(list(cells), 0)
    A = dense.assemble_A(list(cells), c)
    out = O.gs_lex(0, u, f)
    ref = dense.gs_lex(A, D, omega, dense.interior(u), dense.interior(f))
    np.testing.assert_allclose(dense.interior(out), ref, rtol=1e-13, atol=1e-13)


def test_gs_lex_last_node_residual_zero():
    """omega = 1: the last node in lexicographic order has no later neighbour, so its
    residual is exactly solved away (to rounding) by the sweep."""
    for dim, cells in [(2, (8, 6)), (3, (4, 6, 4))]:
        O = orc.Oracle(cfg(dim, cells, levels=1, smoother="gs_lex", omega=1.0))
        u, f = rnd(O.shape(0), 27), rnd(O.shape(0), 28)
        out = O.gs_lex(0, u, f)
        r = O.residual(0, out, f)
        last = (-2,) * dim
        assert abs(r[last]) <= 1e-12 * np.abs(f).max() * 4 * cells[0] ** 2, r[last]


def test_rbgs_black_residual_zero_and_single_unknown_exact():
    """After an omega=1 RBGS sweep the residual vanishes at black nodes;
    one unknown + omega=1 gives the exact solution."""
    cells = (16, 16)
    O = orc.Oracle(cfg(2, cells, levels=1))
    u, f = rnd(O.shape(0), 7), rnd(O.shape(0), 8)
    out = O.rbgs(0, u, f)
    r = O.residual(0, out, f)
    j, i = np.indices(r.shape)
    black = ((i + j) % 2 == 1)
    black[0, :] = black[-1, :] = black[:, 0] = black[:, -1] = False
    assert np.abs(r[black]).max() < 1e-12 * np.abs(r).max()
    O1 = orc.Oracle(cfg(2, (2, 2), levels=1))
    f1 = np.zeros((3, 3)); f1[1, 1] = 1.0
    u1 = O1.rbgs(0, np.zeros((3, 3)), f1)
    assert O1.norm(0, u1, f1) == 0.0


def test_rbgs_energy_norm_nonincreasing():
    """for SPD A and GS with omega=1 the A-norm of the error does not increase."""
    cells = [16, 16]
    O = orc.Oracle(cfg(2, cells, levels=1))
    c, D, _ = dense.coeffs(cells, 0)
    A = dense.assemble_A(cells, c)
    f = rnd(O.shape(0), 9)
    x = np.linalg.solve(A, dense.interior(f))
    u = rnd(O.shape(0), 10)
    prev = np.inf
    for _ in range(6):
        e = dense.interior(u) - x
        en = e @ A @ e
        assert en <= prev * (1 + 1e-12)
        prev = en
        u = O.rbgs(0, u, f)


def test_jacobi_sine_mode_factor():
    """Closed form: with f=0 Jacobi multiplies phi_k by 1 - omega(1 - (1/d) sum cos(k pi h)).
    SURVEY §8(c): 2D n=64, omega=0.8: k=1 -> 0.999036, k=32 -> 0.2, k=63 -> -0.599036."""
    cells = (64, 64)
    O = orc.Oracle(cfg(2, cells, levels=1, smoother="jacobi", omega=0.8))
    x, y = wl.coords(2, cells)
    for k, expect in [(1, 0.999036), (32, 0.2), (63, -0.599036)]:
        phi = np.sin(k * np.pi * x) * np.sin(k * np.pi * y)
        out = O.jacobi(0, phi, np.zeros_like(phi))
        fac = 1 - 0.8 * (1 - math.cos(k * math.pi / 64))
        np.testing.assert_allclose(out, fac * phi, atol=1e-13)
        assert abs(fac - expect) < 5e-7


# ---------------------------------------------------------------- transfers
@pytest.mark.parametrize("dim,cells", SMALL)
def test_restriction_equals_dense_FW(dim, cells):
    """R = 2^-d P^T (reading 7) applied to a random residual."""
    O = orc.Oracle(cfg(dim, cells, levels=2))
    r = rnd(O.shape(0), 11)
    fc = O.restrict(0, r)
    R = dense.assemble_R([n // 2 for n in cells])
    np.testing.assert_allclose(dense.interior(fc), R @ dense.interior(r), rtol=1e-14, atol=1e-15)
    assert np.all(fc[~np.pad(np.ones([s - 2 for s in fc.shape], bool), 1)] == 0)


def test_restriction_constant_impulse_and_symbol():
    """FW of a constant is the constant; 2D impulse -> 4/16 (3D: 8/64);
    LFA symbol: R phi_k^h = prod cos^2(k pi h/2) phi_k^H."""
    O = orc.Oracle(cfg(2, (16, 16), levels=2))
    fc = O.restrict(0, np.full(O.shape(0), 3.0))
    assert np.all(fc[1:-1, 1:-1] == 3.0)
    imp = np.zeros(O.shape(0)); imp[8, 8] = 1.0
    assert O.restrict(0, imp)[4, 4] == 4.0 / 16.0
    O3 = orc.Oracle(cfg(3, (8, 8, 8), levels=2))
    imp3 = np.zeros(O3.shape(0)); imp3[4, 4, 4] = 1.0
    assert O3.restrict(0, imp3)[2, 2, 2] == 8.0 / 64.0
    x, y = wl.coords(2, (16, 16))
    X, Y = wl.coords(2, (8, 8))
    for k in [(1, 2), (3, 5), (7, 7)]:
        phi = np.sin(k[0] * np.pi * x) * np.sin(k[1] * np.pi * y)
        sym = math.cos(k[0] * math.pi / 32) ** 2 * math.cos(k[1] * math.pi / 32) ** 2
        PhiH = np.sin(k[0] * np.pi * X) * np.sin(k[1] * np.pi * Y)
        np.testing.assert_allclose(O.restrict(0, phi)[1:-1, 1:-1], sym * PhiH[1:-1, 1:-1], atol=1e-14)


@pytest.mark.parametrize("dim,cells", SMALL)
def test_prolongation_equals_dense(dim, cells):
    """u += P e with P the bi-/trilinear tensor-product interpolation."""
    O = orc.Oracle(cfg(dim, cells, levels=2))
    u = rnd(O.shape(0), 12)
    e = rnd(O.shape(1), 13)
    out = O.prolong_correct(0, e, u)
    P = dense.assemble_P([n // 2 for n in cells])
    np.testing.assert_allclose(dense.interior(out), dense.interior(u) + P @ dense.interior(e),
                               rtol=1e-14, atol=1e-15)
    # boundary of u untouched
    bd = ~np.pad(np.ones([s - 2 for s in u.shape], bool), 1)
    assert np.array_equal(out[bd], u[bd])


def test_prolongation_reproduces_linear_functions():
    """Bi-/trilinear interpolation is exact for (multi)linear coarse functions."""
    for dim, cells in [(2, (16, 8)), (3, (8, 8, 8))]:
        O = orc.Oracle(cfg(dim, cells, levels=2))
        xs = wl.coords(dim, cells)
        Xs = wl.coords(dim, [n // 2 for n in cells])
        coef = [0.5, 0.25, 0.125]
        lin_f = 1.0 + sum(coef[d] * xs[d] for d in range(dim))
        lin_c = 1.0 + sum(coef[d] * Xs[d] for d in range(dim))
        out = O.prolong_correct(0, lin_c, np.zeros(O.shape(0)))
        m = np.pad(np.ones([s - 2 for s in out.shape], bool), 1)
        np.testing.assert_allclose(out[m], lin_f[m], rtol=0, atol=1e-15)


# ---------------------------------------------------------------- coarse solve
@pytest.mark.parametrize("dim,cells,levels", [(2, (64, 64), 5), (3, (16, 16, 16), 3), (2, (16, 16), 4)])
def test_coarse_direct_equals_dense_solve(dim, cells, levels):
    O = orc.Oracle(cfg(dim, cells, levels=levels))
    lc = [n >> (levels - 1) for n in cells]
    f = rnd(O.shape(levels - 1), 14)
    e = O.coarse_solve(f)
    c, D, _ = dense.coeffs(list(cells), levels - 1)
    A = dense.assemble_A(lc, c)
    np.testing.assert_allclose(dense.interior(e), np.linalg.solve(A, dense.interior(f)), rtol=1e-12)


def test_coarse_single_unknown_is_division():
    O = orc.Oracle(cfg(3, (8, 8, 8), levels=3))
    f = np.zeros(O.shape(2)); f[1, 1, 1] = 3.0
    _, D, _ = dense.coeffs([8, 8, 8], 2)
    assert O.coarse_solve(f)[1, 1, 1] == 3.0 / D


# ---------------------------------------------------------------- whole cycle
DENSE_CASES = [
    (2, (8, 8), 3, "rbgs", 1.0, 2, 2),
    (2, (16, 16), 3, "jacobi", 0.8, 2, 2),
    (2, (16, 8), 2, "rbgs", 1.0, 1, 0),
    (2, (16, 16), 4, "jacobi", 0.8, 3, 3),
    (3, (8, 8, 8), 2, "rbgs", 1.0, 2, 2),
    (3, (8, 8, 8), 3, "jacobi", 0.8, 2, 2),
    (3, (8, 8, 16), 3, "rbgs", 1.0, 2, 1),
    (2, (16, 8), 3, "gs_lex", 1.0, 2, 2),
    (3, (8, 8, 8), 2, "gs_lex", 1.15, 1, 1),
]


@pytest.mark.parametrize("dim,cells,levels,sm,omega,nu1,nu2", DENSE_CASES)
def test_vcycle_equals_dense_algorithm1(dim, cells, levels, sm, omega, nu1, nu2):
    """The oracle's V-cycle equals Alg. 1 evaluated in dense algebra (two-grid and
    multigrid error propagation) on random u and f."""
    O = orc.Oracle(cfg(dim, cells, levels, sm, omega, nu1, nu2))
    M = dense.DenseMG(cells, levels, sm, omega, nu1, nu2)
    u, f = rnd(O.shape(0), 15), rnd(O.shape(0), 16)
    out = O.vcycle(u, f)
    ref = M.vcycle(dense.interior(u), dense.interior(f) * 1.0)
    np.testing.assert_allclose(dense.interior(out), ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def test_vcycle_coarse_sweeps_mode_equals_dense():
    """Listing P:280-283: coarsest level = ncoarse smoother sweeps from e = 0."""
    O = orc.Oracle(cfg(2, (16, 16), 3, coarse=orc.COARSE_SWEEPS, ncoarse=10))
    M = dense.DenseMG((16, 16), 3, "rbgs", 1.0, 2, 2, coarse="sweeps", ncoarse=10)
    u, f = rnd(O.shape(0), 17), rnd(O.shape(0), 18)
    np.testing.assert_allclose(dense.interior(O.vcycle(u, f)), M.vcycle(dense.interior(u), dense.interior(f)),
                               rtol=1e-12, atol=1e-13)


def test_single_level_direct_is_exact():
    O = orc.Oracle(cfg(2, (8, 8), 1))
    u, f = rnd(O.shape(0), 19), rnd(O.shape(0), 20)
    assert O.norm(0, O.vcycle(u, f), f) < 1e-12 * O.norm(0, u, f)


def _u0(case, shape):
    if case["u0"] == "ones":
        u = np.ones(shape)
    elif case["u0"] == "ijmod7":
        j, i = np.indices(shape)
        u = ((i * j) % 7) / 7.0
    else:
        u = wl.workload("W1", case["dim"], case["cells"], seed=case["seed"])[0]
    u[~np.pad(np.ones([s - 2 for s in shape], bool), 1)] = 0.0
    return u


@pytest.mark.parametrize("case", GOLD["cases"], ids=[c["name"] for c in GOLD["cases"]])
def test_survey_dense_vcycle_histories(case):
    """Residual-ratio histories from the survey's exact dense calculation
    (tests/golden/survey_dense_vcycle.json), 5 significant digits."""
    O = orc.Oracle(cfg(case["dim"], case["cells"], case["levels"], case["smoother"], case["omega"],
                       case["nu1"], case["nu2"]))
    u = _u0(case, O.shape(0))
    f = np.zeros_like(u)
    _, k, hist = O.solve(u, f, 0.0, 10)
    assert k == 10
    ratios = hist[1:] / hist[0]
    if "r0" in case:
        assert abs(hist[0] / case["r0"] - 1) < 1e-10
    if "ratios" in case:
        np.testing.assert_allclose(ratios, case["ratios"], rtol=6e-5)
    for kk, v in case.get("ratios_at", {}).items():
        assert abs(ratios[int(kk) - 1] / v - 1) < 6e-5, (kk, ratios[int(kk) - 1], v)


@pytest.mark.parametrize("case", [c for c in GOLD["cases"] if "rho" in c], ids=lambda c: c["name"])
def test_survey_spectral_radius(case):
    """rho(M_V) from the survey by power iteration through the oracle (f = 0)."""
    O = orc.Oracle(cfg(case["dim"], case["cells"], case["levels"], case["smoother"], case["omega"],
                       case["nu1"], case["nu2"]))
    u = rnd(O.shape(0), 21)
    f = np.zeros_like(u)
    logs = []
    for it in range(500):  # geometric mean of the growth: robust to complex/negative pairs
        v = O.vcycle(u, f)
        n = np.linalg.norm(v)
        logs.append(math.log(n / np.linalg.norm(u)))
        u = v / n
    rho = math.exp(np.mean(logs[400:]))
    assert abs(rho / case["rho"] - 1) < 1e-3, rho


def test_paper_claim_2d_rbgs_1e8_in_5_cycles():
    """'the L2-norm of the residual is reduced by a factor of more than 10^8
    within 5 V(2,2)-cycles' — reproducible for 2D RBGS (reading 17)."""
    for cells in [(64, 64), (128, 128)]:
        for seed in (42, 7, 1234):
            O = orc.Oracle(cfg(2, cells))
            u, f = wl.workload("W1", 2, cells, seed=seed)
            _, k, hist = O.solve(u, f, 1e-8, 5)
            assert hist[-1] / hist[0] < 1e-8, (cells, seed, hist[-1] / hist[0])


def test_h_independence():
    """asymptotic V(2,2) RBGS factors at 63^2, 127^2, 255^2 agree within +-25%."""
    rates = []
    for n in (64, 128, 256):
        O = orc.Oracle(cfg(2, (n, n)))
        u, f = wl.workload("W1", 2, (n, n), seed=42)
        _, k, hist = O.solve(u, f, 0.0, 8)
        rates.append(hist[8] / hist[7])
    assert max(rates) <= 1.25 * min(rates), rates


def test_manufactured_solutions_converge():
    """W3 converges to the exact discrete solution; W2 to (theta/sin theta)^2 u*
    (closed form, SURVEY §8(c) 'Converged solution')."""
    for dim, cells in [(2, (32, 32)), (3, (16, 16, 16))]:
        O = orc.Oracle(cfg(dim, cells))
        u, f = wl.workload("W3", dim, cells)
        u, k, hist = O.solve(u, f, 1e-13, 30)
        assert np.abs(u - wl.exact_solution("W3", dim, cells)).max() < 1e-12
    for n, expect in zip(GOLD["w2_max_error"]["n"], GOLD["w2_max_error"]["value"]):
        O = orc.Oracle(cfg(2, (n, n)))
        u, f = wl.workload("W2", 2, (n, n))
        u, k, hist = O.solve(u, f, 1e-13, 30)
        err = np.abs(u - wl.exact_solution("W2", 2, (n, n))).max()
        theta = math.pi / n / 2
        assert abs(err - ((theta / math.sin(theta)) ** 2 - 1)) < 1e-10
        assert abs(err / expect - 1) < 5e-4


def test_fp32_oracle_tracks_fp64():
    """The FP32 build computes the same algorithm: one cycle agrees with FP64 to float rounding."""
    c = cfg(3, (16, 16, 16))
    u, f = wl.workload("W4", 3, (16, 16, 16))
    u64 = orc.Oracle(c, np.float64).vcycle(u, f)
    u32 = orc.Oracle(c, np.float32).vcycle(u.astype(np.float32), f.astype(np.float32))
    assert np.abs(u32 - u64).max() < 1e-5 * np.abs(u64).max()


def test_prng_goldens():
    """SplitMix64 input generator (reading 10): survey goldens and a pure-Python recomputation."""
    g = GOLD["prng_seed42"]
    vals = wl.splitmix64_uniform(42, np.array(g["idx"], np.uint64))
    assert list(vals) == g["value"]

    def py(seed, i):
        M = (1 << 64) - 1
        z = (seed + (i + 1) * 0x9E3779B97F4A7C15) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        z ^= z >> 31
        return (z >> 11) * 2.0 ** -53
    for i in [0, 5, 12345, 2 ** 40]:
        assert wl.splitmix64_uniform(7, np.array([i], np.uint64))[0] == py(7, i)


def test_oracle_thread_count_independent(tmp_path):
    """Determinism and reading 13: results are bitwise identical for any
    OpenMP thread count (the pointwise loops are split by plane only)."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r); import oracle as orc;"
        "from paper_1406_5369_b200 import workloads as wl;"
        "c = orc.Config(dim=3, cells=(32,32,32));"
        "u, f = wl.workload('W4', 3, (32,32,32)); O = orc.Oracle(c);"
        "u, k, h = O.solve(u, f, 0.0, 3); np.save(sys.argv[1], np.concatenate([u.ravel(), h]))"
    ) % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for nt in ("1", "4"):
        p = str(tmp_path / f"o{nt}.npy")
        env = dict(os.environ, OMP_NUM_THREADS=nt)
        subprocess.run([sys.executable, "-c", code, p], check=True, env=env)
        outs.append(np.load(p))
    assert np.array_equal(outs[0], outs[1])


# ---------------------------------------------------------------- the FP32 build, op by op
EPS32 = float(np.finfo(np.float32).eps)


@pytest.mark.parametrize("dim,cells", [(2, (16, 8)), (3, (8, 8, 8)), (3, (8, 4, 16))])
def test_fp32_ops_within_rounding_bound_of_dense(dim, cells):
    """Each FP32 oracle operation equals its dense FP64 definition (tests/dense.py) applied to the
    same float32 inputs, within a forward rounding-error bound of a few float32 roundings per term
    (standard model |fl(a op b) - (a op b)| <= eps |a op b|, summed over the ~10 operations of a
    node): residual, omega-Jacobi, RBGS, full weighting, prolongation + correction.  A dropped
    term, a wrong sign or a transposed operand moves a value by O(|A||u|) >> the bound."""
    O = orc.Oracle(cfg(dim, cells, levels=2, smoother="jacobi", omega=0.8), np.float32)
    u = rnd(O.shape(0), 41).astype(np.float32)
    f = rnd(O.shape(0), 42).astype(np.float32)
    c, D, _ = dense.coeffs(list(cells), 0)
    A = dense.assemble_A(list(cells), c)
    ui, fi = dense.interior(u).astype(np.float64), dense.interior(f).astype(np.float64)
    absAu = np.abs(A) @ np.abs(ui)
    # residual: ~8 roundings on terms of size |f| + |A||u|
    r = dense.interior(O.residual(0, u, f)).astype(np.float64)
    assert np.all(np.abs(r - (fi - A @ ui)) <= 8 * EPS32 * (np.abs(fi) + absAu))
    # omega-Jacobi
    wd = 0.8 / D
    scale = np.abs(ui) + wd * (np.abs(fi) + absAu)
    out = dense.interior(O.jacobi(0, u, f)).astype(np.float64)
    assert np.all(np.abs(out - dense.jacobi(A, D, 0.8, ui, fi)) <= 10 * EPS32 * scale)
    # RBGS (omega = 1): black nodes read the rounded red values, one more level of propagation
    O1 = orc.Oracle(cfg(dim, cells, levels=2, smoother="rbgs"), np.float32)
    out = dense.interior(O1.rbgs(0, u, f)).astype(np.float64)
    ref = dense.rbgs(A, D, 1.0, ui, fi, list(cells))
    sc = np.abs(ui) + (np.abs(fi) + np.abs(A) @ (np.abs(ui) + np.abs(ref))) / D
    assert np.all(np.abs(out - ref) <= 24 * EPS32 * sc)
    # full weighting and prolongation + correction: sums of nonnegative weights
    R = dense.assemble_R([n // 2 for n in cells])
    P = dense.assemble_P([n // 2 for n in cells])
    fc = dense.interior(O.restrict(0, f)).astype(np.float64)
    assert np.all(np.abs(fc - R @ fi) <= 8 * EPS32 * (np.abs(R) @ np.abs(fi)))
    e = rnd(O.shape(1), 43).astype(np.float32)
    ei = dense.interior(e).astype(np.float64)
    pc = dense.interior(O.prolong_correct(0, e, u)).astype(np.float64)
    assert np.all(np.abs(pc - (ui + P @ ei)) <= 8 * EPS32 * (np.abs(ui) + P @ np.abs(ei)))
    # the bound is tight enough to see float32 at all: the FP32 results are not the FP64 ones
    assert np.abs(out - ref).max() > 0
