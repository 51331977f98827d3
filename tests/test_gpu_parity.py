"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element
by element on the same seeded inputs.  Tolerances are the ones
BASELINE.json's north_star states: <= 1e-12 relative max-norm difference per
grid value in FP64, <= 1e-5 in FP32, after every cycle; identical iteration
counts to a fixed residual reduction.  (Canonical operation order and no FMA
on both sides make the expected difference exactly 0; that is checked too
where it is guaranteed.)"""
import numpy as np
import pytest

import oracle as orc
from paper_1406_5369_b200 import workloads as wl

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-12, "f32": 1e-5}


def make(dim, cells, levels=0, smoother="rbgs", omega=None, nu1=2, nu2=2, dtype="f64", coarse="direct",
         ncoarse=10, flags=0, pm_min_nx=16):
    import paper_1406_5369_b200 as mgb
    if omega is None:
        omega = 0.8 if smoother == "jacobi" else 1.0
    S = mgb.Solver(dim, tuple(c + 1 for c in cells), levels=levels, smoother=smoother, omega=omega, nu1=nu1,
                   nu2=nu2, coarse=coarse, ncoarse=ncoarse, dtype=dtype, flags=flags, pm_min_nx=pm_min_nx)
    O = orc.Oracle(orc.Config(dim=dim, cells=tuple(cells), levels=S.levels,
                              smoother={"rbgs": orc.RBGS, "gs_lex": orc.GS_LEX}.get(smoother, orc.JACOBI),
                              omega=omega, nu1=nu1,
                              nu2=nu2, coarse=orc.COARSE_DIRECT if coarse == "direct" else orc.COARSE_SWEEPS,
                              ncoarse=ncoarse),
                   np.float64 if dtype == "f64" else np.float32)
    return S, O


def relerr(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = max(np.abs(b).max(), 1e-300)
    return np.abs(a - b).max() / den


def rnd(shape, seed, dtype):
    r = np.random.default_rng(seed).uniform(-1, 1, size=shape)
    r[~np.pad(np.ones([s - 2 for s in shape], bool), 1)] = 0.0
    return r.astype(dtype)


OP_CASES = [
    (2, (64, 64), 5, "jacobi", "f64"),
    (2, (128, 64), 0, "rbgs", "f64"),
    (2, (256, 256), 0, "jacobi", "f32"),
    (3, (32, 32, 32), 0, "rbgs", "f64"),
    (3, (32, 16, 64), 3, "jacobi", "f64"),
    (3, (64, 64, 64), 0, "rbgs", "f32"),
    (3, (96, 96, 96), 5, "rbgs", "f64"),   # ragged: 95 interior nodes, tiles do not divide it
]


@pytest.mark.parametrize("dim,cells,levels,sm,dt", OP_CASES)
def test_per_op_parity(dim, cells, levels, sm, dt):
    S, O = make(dim, cells, levels, sm, dtype=dt)
    npdt = S.np_dtype
    for l in range(S.levels):
        shp = O.shape(l)
        u, f = rnd(shp, 100 + l, npdt), rnd(shp, 200 + l, npdt)
        du, df = S.from_numpy(u, l), S.from_numpy(f, l)
        # smoother
        out = S.empty(l)
        S.op_smooth(l, du, df, out)
        ref = O.smooth(l, u, f)
        assert relerr(S.to_numpy(out, l), ref) <= TOL[dt], ("smooth", l)
        # residual
        r = S.empty(l)
        S.op_residual(l, du, df, r)
        ref_r = O.residual(l, u, f)
        assert relerr(S.to_numpy(r, l), ref_r) <= TOL[dt], ("residual", l)
        # norm
        assert abs(S.op_norm(l, du, df) / O.norm(l, u, f) - 1) <= 1e-12, ("norm", l)
        if l + 1 < S.levels:
            fc = S.empty(l + 1)
            S.op_restrict(l, r, fc)
            assert relerr(S.to_numpy(fc, l + 1), O.restrict(l, ref_r.astype(npdt))) <= TOL[dt], ("restrict", l)
            e = rnd(O.shape(l + 1), 300 + l, npdt)
            uu = du.clone()
            S.op_prolong_correct(l, S.from_numpy(e, l + 1), uu)
            assert relerr(S.to_numpy(uu, l), O.prolong_correct(l, e, u)) <= TOL[dt], ("prolong", l)
        else:
            e = S.empty(l)
            S.op_coarse_solve(df, e)
            assert relerr(S.to_numpy(e, l), O.coarse_solve(f)) <= TOL[dt], "coarse"


CYCLE_CASES = [
    # C1 exactly: 2D 65^2, 5 levels, Jacobi omega=0.8, V(2,2), FP64
    dict(dim=2, cells=(64, 64), levels=5, smoother="jacobi"),
    dict(dim=2, cells=(64, 64), levels=5, smoother="jacobi", dtype="f32"),
    dict(dim=2, cells=(128, 64), smoother="rbgs"),
    dict(dim=2, cells=(256, 256), smoother="jacobi", nu1=3, nu2=3, dtype="f32"),
    dict(dim=3, cells=(32, 32, 32), smoother="rbgs"),
    dict(dim=3, cells=(32, 32, 32), smoother="rbgs", dtype="f32"),
    dict(dim=3, cells=(32, 16, 64), levels=3, smoother="jacobi", nu1=2, nu2=1),  # odd nu1+nu2: copy-back
    dict(dim=3, cells=(48, 48, 48), levels=4, smoother="rbgs", nu1=1, nu2=1),    # ragged tiles
    dict(dim=3, cells=(16, 16, 16), levels=2, smoother="rbgs", coarse="sweeps", ncoarse=10),
    dict(dim=2, cells=(32, 32), levels=1, smoother="rbgs"),                       # single level, direct
    dict(dim=3, cells=(128, 128, 128), smoother="rbgs"),                          # C2 grid
]


@pytest.mark.parametrize("case", CYCLE_CASES, ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_vcycle_parity_per_cycle(case):
    dt = case.get("dtype", "f64")
    S, O = make(**case)
    u, f = wl.workload("W1", case["dim"], case["cells"], seed=42, dtype=S.np_dtype)
    if case["cells"] == (32, 32) or case.get("coarse") == "sweeps":
        u, f = wl.workload("W4", case["dim"], case["cells"], seed=7, dtype=S.np_dtype)
    du, df = S.from_numpy(u), S.from_numpy(f)
    uo = u.copy()
    for k in range(4):
        S.vcycle(du, df)
        O.vcycle_inplace(uo, f)
        got = S.to_numpy(du)
        assert relerr(got, uo) <= TOL[dt], (k, relerr(got, uo))
        if dt == "f64":
            assert np.array_equal(got, uo), ("expected bitwise equality", k)
        assert abs(S.residual_norm(du, df) / O.norm(0, uo, f) - 1) <= 1e-12


@pytest.mark.parametrize("case", [
    dict(dim=2, cells=(64, 64), levels=5, smoother="jacobi"),   # C1
    dict(dim=3, cells=(128, 128, 128), smoother="rbgs"),        # C2
    dict(dim=3, cells=(64, 64, 64), smoother="rbgs", dtype="f32"),
    dict(dim=2, cells=(512, 512), smoother="jacobi", nu1=3, nu2=3, dtype="f32"),
], ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_iteration_count_parity(case):
    """Identical iteration count to a 1e-10 residual reduction (north_star)."""
    S, O = make(**case)
    u, f = wl.workload("W1", case["dim"], case["cells"], seed=42, dtype=S.np_dtype)
    du, df = S.from_numpy(u), S.from_numpy(f)
    k_gpu, hist_gpu = S.solve(du, df, 1e-10, 40)
    _, k_or, hist_or = O.solve(u, f, 1e-10, 40)
    assert k_gpu == k_or, (k_gpu, k_or)
    np.testing.assert_allclose(hist_gpu, hist_or, rtol=1e-12 if S.np_dtype == np.float64 else 1e-5)
    assert hist_gpu[-1] <= 1e-10 * hist_gpu[0]


def test_c1_survey_history_on_gpu():
    """C1 residual history from the survey's dense calculation (golden) reproduced on the GPU."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "survey_dense_vcycle.json")))
    case = [c for c in g["cases"] if c["name"].startswith("C1 on W1")][0]
    S, _ = make(2, (64, 64), 5, "jacobi")
    u, f = wl.workload("W1", 2, (64, 64), seed=42)
    du, df = S.from_numpy(u), S.from_numpy(f)
    k, hist = S.solve(du, df, 0.0, 10)
    assert abs(hist[0] / case["r0"] - 1) < 1e-10
    np.testing.assert_allclose(np.array(hist[1:]) / hist[0], case["ratios"], rtol=6e-5)


def test_workload_fill_matches_numpy_generator():
    for dim, cells, dt in [(3, (32, 16, 8), "f64"), (2, (64, 32), "f32")]:
        S, _ = make(dim, cells, 2, dtype=dt)
        d = S.empty()
        S.workload_fill(d, 42)
        ref = wl.random_interior(dim, cells, 42, S.np_dtype)
        assert np.array_equal(S.to_numpy(d), ref)
        S.workload_fill(d, 7, -1.0, 1.0)
        ref = wl.random_interior(dim, cells, 7, S.np_dtype, -1.0, 1.0)
        assert np.array_equal(S.to_numpy(d), ref)


def test_graph_and_eager_identical_and_deterministic():
    import paper_1406_5369_b200 as mgb
    outs = []
    for flags in (0, mgb.FLAG_NO_GRAPH, 0):
        S, _ = make(3, (64, 64, 64), flags=flags)
        u, f = wl.workload("W4", 3, (64, 64, 64), seed=3)
        du, df = S.from_numpy(u), S.from_numpy(f)
        for _ in range(3):
            S.vcycle(du, df)
        outs.append(S.to_numpy(du))
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_vcycle_host_e2e_matches_device_path():
    import torch
    S, O = make(3, (32, 32, 32))
    u, f = wl.workload("W1", 3, (32, 32, 32), seed=42)
    hu = S.from_numpy(u).cpu().pin_memory()
    hf = S.from_numpy(f).cpu().pin_memory()
    n = S.vcycle_host(hu, hf, 2)
    ref = O.vcycle(O.vcycle(u, f), f)
    got = S.to_numpy(hu.cuda())
    assert np.array_equal(got, ref)
    assert abs(n / O.norm(0, ref, f) - 1) < 1e-12
    del torch


def test_boundary_and_padding_untouched():
    """The library never writes boundary nodes or padding of the caller's u."""
    import torch
    S, _ = make(3, (32, 32, 32))
    u, f = wl.workload("W4", 3, (32, 32, 32), seed=9)
    du, df = S.from_numpy(u), S.from_numpy(f)
    du[:, :, 33:] = 123.0  # padding sentinel
    du[0] = 5.0            # non-zero Dirichlet plane
    before = du.clone()
    S.vcycle(du, df)
    assert torch.equal(du[:, :, 33:], before[:, :, 33:])
    assert torch.equal(du[0], before[0])
    assert torch.equal(du[-1], before[-1])
    assert torch.equal(du[:, 0], before[:, 0]) and torch.equal(du[:, :, 0], before[:, :, 0])


def test_profile_counts_launches():
    S, _ = make(3, (64, 64, 64))
    u, f = wl.workload("W1", 3, (64, 64, 64), seed=42)
    du, df = S.from_numpy(u), S.from_numpy(f)
    S.vcycle(du, df)
    n = S.launches_per_cycle
    assert n > 0
    S.profile_enable(True)
    S.vcycle(du, df)
    recs = S.profile_read()
    S.profile_enable(False)
    assert sum(r["count"] for r in recs if not r["name"].startswith("memset")) == n
    assert all(r["ms"] > 0 for r in recs)


@pytest.mark.parametrize("variant", ["default-threshold", "baseline", "separate-prolong"])
def test_schedule_variants_identical(variant):
    """The plane-marching, mixed (default threshold) and op-by-op (MG_FLAG_BASELINE)
    schedules give bitwise identical iterates (same canonical arithmetic)."""
    import paper_1406_5369_b200 as mgb
    kw = {"default-threshold": dict(pm_min_nx=0), "baseline": dict(flags=mgb.FLAG_BASELINE),
          "separate-prolong": dict(flags=mgb.FLAG_SEPARATE_PROLONG)}[variant]
    outs = []
    for extra in (dict(), kw):
        S, _ = make(3, (128, 128, 128), **extra)
        u, f = wl.workload("W4", 3, (128, 128, 128), seed=11)
        du, df = S.from_numpy(u), S.from_numpy(f)
        for _ in range(2):
            S.vcycle(du, df)
        outs.append(S.to_numpy(du))
    assert np.array_equal(outs[0], outs[1])


SLAB_CASES = [
    dict(dim=3, cells=(128, 128, 128), smoother="rbgs"),
    dict(dim=3, cells=(64, 64, 64), smoother="jacobi", nu1=2, nu2=1),
    dict(dim=2, cells=(64, 64), levels=5, smoother="jacobi"),
    dict(dim=3, cells=(64, 64, 64), smoother="rbgs", dtype="f32"),
]


@pytest.mark.parametrize("case", SLAB_CASES, ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_slab_mode_single_rank(case):
    """Slab layout (halo planes, p_glob0 != 0, agglomerated coarse levels, rank-sum norm)
    on one GPU (MG_FLAG_SLAB, nranks = 1): bitwise identical to the oracle."""
    import paper_1406_5369_b200 as mgb
    dt = case.get("dtype", "f64")
    S, O = make(**case, flags=mgb.FLAG_SLAB)
    assert S.distributed and S.halo == 2
    u, f = wl.workload("W1", case["dim"], case["cells"], seed=42, dtype=S.np_dtype)
    du, df = S.from_numpy(u), S.from_numpy(f)
    uo = u.copy()
    for k in range(3):
        S.vcycle(du, df)
        O.vcycle_inplace(uo, f)
        got = S.to_numpy(du)
        assert relerr(got, uo) <= TOL[dt], (k, relerr(got, uo))
        if dt == "f64":
            assert np.array_equal(got, uo), ("expected bitwise equality", k)
        assert abs(S.residual_norm(du, df) / O.norm(0, uo, f) - 1) <= 1e-12


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_separate_prolongation_parity(dt):
    """MG_FLAG_SEPARATE_PROLONG (the prolongation + correction as its own pass instead of fused
    into the first post-sweep, the default) against the oracle per cycle, both smoothers."""
    import paper_1406_5369_b200 as mgb
    for sm in ("rbgs", "jacobi"):
        S, O = make(3, (128, 128, 128), smoother=sm, dtype=dt, flags=mgb.FLAG_SEPARATE_PROLONG)
        u, f = wl.workload("W4", 3, (128, 128, 128), seed=3, dtype=S.np_dtype)
        du, df = S.from_numpy(u), S.from_numpy(f)
        uo = u.copy()
        for k in range(2):
            S.vcycle(du, df)
            O.vcycle_inplace(uo, f)
            got = S.to_numpy(du)
            assert relerr(got, uo) <= TOL[dt]
            if dt == "f64":
                assert np.array_equal(got, uo)


def test_vcycle_host_batch_pipeline():
    """mg_vcycle_host_batch: independent problems from pinned host buffers, pipelined copies;
    each result equals the oracle's cycle of that problem (in != out and in-place)."""
    S, O = make(3, (64, 64, 64))
    probs = [wl.workload("W4", 3, (64, 64, 64), seed=s) for s in (1, 2, 3)]
    hu = [S.from_numpy(u + wl.random_interior(3, (64, 64, 64), 10 + i)).cpu().pin_memory()
          for i, (u, _) in enumerate(probs)]
    hf = [S.from_numpy(f).cpu().pin_memory() for _, f in probs]
    refs = [O.vcycle(S.to_numpy(h.cuda()), f) for h, (_, f) in zip(hu, probs)]
    ho = [h.clone().pin_memory() for h in hu]
    norms = S.vcycle_host_batch(hu, ho, hf, 1)
    for b in range(3):
        assert np.array_equal(S.to_numpy(ho[b].cuda()), refs[b]), b
        assert abs(norms[b] / O.norm(0, refs[b], probs[b][1]) - 1) < 1e-12
    norms2 = S.vcycle_host_batch(hu, hu, hf, 1)  # in place
    for b in range(3):
        assert np.array_equal(S.to_numpy(hu[b].cuda()), refs[b]), b
        assert norms2[b] == norms[b]


@pytest.mark.parametrize("case", [
    dict(dim=3, cells=(128, 64, 64), coeff=(1.0, 2.0, 0.5), h=(0.5 / 128, 1.0 / 64, 2.0 / 64)),
    dict(dim=2, cells=(256, 128), coeff=(3.0, 0.25), h=(1.0 / 256, 4.0 / 128), smoother="jacobi"),
    dict(dim=3, cells=(64, 64, 128), coeff=(0.7, 1.3, 1.0), h=None, dtype="f32"),
], ids=["3d-aniso", "2d-aniso-jacobi", "3d-aniso-f32"])
def test_anisotropic_coefficients_and_spacing(case):
    """A = -sum a_d d^2/dx_d^2 with a_d != 1 and h_d != 1/n_d (mg_config.coeff / h, P:111,
    P:226): every kernel family (plane-marching, warp-marching, op-by-op, coarse tail)
    against the oracle, per cycle."""
    import paper_1406_5369_b200 as mgb
    dim, cells, dt = case["dim"], case["cells"], case.get("dtype", "f64")
    sm = case.get("smoother", "rbgs")
    omega = 0.8 if sm == "jacobi" else 1.0
    coeff = tuple(case["coeff"]) + (1.0,) * (3 - dim)
    S = mgb.Solver(dim, tuple(c + 1 for c in cells), smoother=sm, omega=omega, dtype=dt, coeff=coeff,
                   h=case["h"], pm_min_nx=16)
    O = orc.Oracle(orc.Config(dim=dim, cells=tuple(cells), levels=S.levels,
                              smoother=orc.RBGS if sm == "rbgs" else orc.JACOBI, omega=omega,
                              a=coeff, h=case["h"]),
                   np.float64 if dt == "f64" else np.float32)
    u, f = wl.workload("W4", dim, cells, seed=17, dtype=S.np_dtype)
    u = u + wl.random_interior(dim, cells, 18, S.np_dtype)
    du, df = S.from_numpy(u), S.from_numpy(f)
    uo = u.copy()
    for _ in range(2):
        S.vcycle(du, df)
        O.vcycle_inplace(uo, f)
        got = S.to_numpy(du)
        assert relerr(got, uo) <= TOL[dt]
        assert np.array_equal(got, uo)
