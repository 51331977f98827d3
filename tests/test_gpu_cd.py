"""Complex diffusion with FAS on cell-centred grids (SURVEY §8(f) NEXT-2/NEXT-4,
kernels_cd.cu) against the oracle (oracle/cd_oracle.c, pinned in
test_cd_oracle_pins.py): per cycle bitwise in FP64 and FP32 (same canonical
complex operation order, no FMA), per operation, the driver loop's cycle counts and
residual histories, the device input generator, and the paper's 10^5 claim."""
import numpy as np
import pytest

from oracle.cd import CDConfig, CDOracle, JACOBI, RBGS
from paper_1406_5369_b200 import workloads as wl

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-12, "f32": 1e-5}


def make(dim, cells, levels=0, smoother="rbgs", omega=None, nu1=2, nu2=2, ncoarse=10, dtype="f64", flags=0,
         tau=0.1, theta=np.pi / 30, kappa=2.0):
    import paper_1406_5369_b200 as mgb
    if omega is None:
        omega = 1.0 if smoother == "rbgs" else 0.8
    S = mgb.Solver(dim, tuple(cells), levels=levels, smoother=smoother, omega=omega, nu1=nu1, nu2=nu2,
                   coarse="sweeps", ncoarse=ncoarse, dtype=dtype, flags=flags, problem="complex_diffusion",
                   tau=tau, theta=theta, kappa=kappa)
    O = CDOracle(CDConfig(dim=dim, cells=tuple(cells), levels=S.levels, smoother=RBGS if smoother == "rbgs" else JACOBI,
                          omega=omega, nu1=nu1, nu2=nu2, ncoarse=ncoarse, tau=tau, theta=theta, kappa=kappa),
                 np.complex128 if dtype == "f64" else np.complex64)
    return S, O


def relerr(a, b):
    return np.abs(np.asarray(a, np.complex128) - np.asarray(b, np.complex128)).max() / max(np.abs(b).max(), 1e-300)


CASES = [
    dict(dim=2, cells=(64, 64), smoother="rbgs"),
    dict(dim=2, cells=(64, 64), smoother="jacobi"),
    dict(dim=2, cells=(96, 80), levels=4, smoother="rbgs", nu1=1, nu2=2),   # non-square, odd sweep count
    dict(dim=2, cells=(128, 64), smoother="jacobi", nu1=3, nu2=3, dtype="f32"),
    dict(dim=3, cells=(32, 32, 32), smoother="rbgs"),
    dict(dim=3, cells=(16, 32, 8), smoother="jacobi"),
    dict(dim=3, cells=(32, 32, 32), smoother="rbgs", dtype="f32"),
    dict(dim=2, cells=(256, 256), smoother="rbgs", omega=1.15),
    dict(dim=2, cells=(200, 48), levels=3, smoother="jacobi", dtype="f32"),  # ragged warp strips
    dict(dim=2, cells=(200, 48), levels=3, smoother="jacobi"),
    # 3D plane-marching Jacobi (kernels_cd3d.cu): tiles ragged in x (32 / 64 cells) and y (8 rows)
    dict(dim=3, cells=(72, 44, 20), levels=2, smoother="jacobi"),
    dict(dim=3, cells=(100, 36, 16), levels=2, smoother="jacobi", dtype="f32"),
    dict(dim=3, cells=(64, 64, 64), smoother="jacobi", dtype="f32"),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_cd_cycle_parity(case):
    dt = case.get("dtype", "f64")
    S, O = make(**case)
    u, f = wl.cd_workload(case["dim"], case["cells"], seed=42, dtype=S.np_dtype)
    du, df = S.from_numpy(u), S.from_numpy(f)
    uo = u.copy()
    for k in range(3):
        S.vcycle(du, df)
        uo = O.cycle(uo, f)
        got = S.to_numpy(du)
        assert relerr(got, uo) <= TOL[dt], (k, relerr(got, uo))
        assert np.array_equal(got, uo), ("expected bitwise equality", k, relerr(got, uo))
        assert abs(S.residual_norm(du, df) / O.norm(0, uo, f) - 1) <= (1e-12 if dt == "f64" else 1e-6)


@pytest.mark.parametrize("sm", ["rbgs", "jacobi"])
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_cd_per_op_parity(sm, dt):
    cells = (48, 32)
    S, O = make(2, cells, 3, sm, dtype=dt)
    rng = np.random.default_rng(3)
    for l in range(S.levels - 1):
        shp = O.shape(l)
        u = (rng.uniform(-1, 1, shp) + 1j * rng.uniform(-1, 1, shp)).astype(S.np_dtype)
        f = (rng.uniform(-1, 1, shp) + 1j * rng.uniform(-1, 1, shp)).astype(S.np_dtype)
        du, df = S.from_numpy(u, l), S.from_numpy(f, l)
        g = O.gfield(l, u)
        out = S.empty(l)
        S.op_smooth(l, du, df, out)
        assert np.array_equal(S.to_numpy(out, l), O.smooth(l, g, u, f)), ("smooth", l)
        r = S.empty(l)
        S.op_residual(l, du, df, r)
        Au, _ = O.apply(l, g, u)
        assert np.array_equal(S.to_numpy(r, l), (f - Au).astype(S.np_dtype)), ("residual", l)
        assert abs(S.op_norm(l, du, df) / O.norm(l, u, f) - 1) <= (1e-12 if dt == "f64" else 1e-6)
        fc = S.empty(l + 1)
        S.op_restrict(l, du, fc)
        assert np.array_equal(S.to_numpy(fc, l + 1), O.restrict(l, u)), ("restrict", l)
        e = (rng.uniform(-1, 1, O.shape(l + 1)) + 1j * rng.uniform(-1, 1, O.shape(l + 1))).astype(S.np_dtype)
        uu = du.clone()
        S.op_prolong_correct(l, S.from_numpy(e, l + 1), uu)
        assert np.array_equal(S.to_numpy(uu, l), O.prolong_add(l, e, u)), ("prolong", l)


@pytest.mark.parametrize("loop", ["device", "host"])
def test_cd_solve_parity_and_paper_claim(loop):
    """Identical cycle counts and residual histories; P:578's 10^5 within 5 V(2,2) cycles."""
    import paper_1406_5369_b200 as mgb
    for sm in ("rbgs", "jacobi"):
        S, O = make(2, (128, 128), smoother=sm, flags=0 if loop == "device" else mgb.FLAG_HOST_LOOP)
        u, f = wl.cd_workload(2, (128, 128), seed=42)
        du, df = S.from_numpy(u), S.from_numpy(f)
        k, hist = S.solve(du, df, 1e-5, 20)
        uo, k_or, hist_or = O.solve(u, f, 1e-5, 20)
        assert k == k_or and k <= 5, (k, k_or)
        np.testing.assert_allclose(hist, hist_or, rtol=1e-12)
        assert np.array_equal(S.to_numpy(du), uo)


def test_cd_workload_fill_matches_generator():
    for dim, cells, dt in [(2, (64, 48), "f64"), (3, (16, 8, 32), "f32")]:
        S, _ = make(dim, cells, dtype=dt)
        d = S.empty()
        S.workload_fill(d, 42)
        ref, _ = wl.cd_workload(dim, cells, 42, S.np_dtype)
        assert np.array_equal(S.to_numpy(d), ref)


def test_cd_graph_and_eager_identical():
    import paper_1406_5369_b200 as mgb
    outs = []
    for flags in (0, mgb.FLAG_NO_GRAPH):
        S, _ = make(2, (256, 128))
        u, f = wl.cd_workload(2, (256, 128), seed=5)
        du, df = S.from_numpy(u), S.from_numpy(f)
        for _ in range(2):
            S.vcycle(du, df)
        outs.append(S.to_numpy(du))
    assert np.array_equal(outs[0], outs[1])


def test_cd_vcycle_host_e2e():
    """mg_vcycle_host with pinned host complex buffers (the bench's e2e path) == oracle."""
    S, O = make(2, (512, 256), smoother="jacobi")
    u, f = wl.cd_workload(2, (512, 256), seed=9)
    hu = S.from_numpy(u).cpu().pin_memory()
    hf = S.from_numpy(f).cpu().pin_memory()
    n = S.vcycle_host(hu, hf, 2)
    ref = O.cycle(O.cycle(u, f), f)
    assert np.array_equal(S.to_numpy(hu.cuda()), ref)
    assert abs(n / O.norm(0, ref, f) - 1) <= 1e-12


def test_cd_vcycle_host_batch():
    S, O = make(2, (256, 128), smoother="rbgs")
    ins = [wl.cd_workload(2, (256, 128), seed=s) for s in (3, 4)]
    hu = [S.from_numpy(u).cpu().pin_memory() for u, _ in ins]
    hf = [S.from_numpy(f).cpu().pin_memory() for _, f in ins]
    ho = [h.clone().pin_memory() for h in hu]
    norms = S.vcycle_host_batch(hu, ho, hf, 2)
    for b, (u, f) in enumerate(ins):
        ref = O.cycle(O.cycle(u, f), f)
        assert np.array_equal(S.to_numpy(ho[b].cuda()), ref)
        assert abs(norms[b] / O.norm(0, ref, f) - 1) <= 1e-12
