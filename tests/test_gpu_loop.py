"""On-device driver loop (loop.cu): mg_solve as one CUDA graph
with a conditional WHILE node — or, for grids whose whole cycle is the coarse tail, as
one kernel launch — against the host-driven loop (MG_FLAG_HOST_LOOP) and
the oracle's or_solve (the `Application` listing): identical cycle
counts, bitwise identical iterates and residual histories."""
import numpy as np
import pytest

import oracle as orc  # noqa: F401  (make() builds the oracle)
from paper_1406_5369_b200 import workloads as wl

from test_gpu_parity import make

pytestmark = pytest.mark.gpu

LOOP_CASES = [
    dict(dim=3, cells=(128, 128, 128), smoother="rbgs"),                  # pipelined split (head/tail)
    dict(dim=3, cells=(64, 64, 64), smoother="jacobi", nu1=2, nu2=1),    # split, odd sweep count
    dict(dim=2, cells=(64, 64), levels=5, smoother="jacobi"),            # C1: no split (cycle + norm)
    dict(dim=3, cells=(64, 64, 64), smoother="rbgs", dtype="f32"),
    dict(dim=2, cells=(32, 32), levels=1, smoother="rbgs"),               # single level, direct
    dict(dim=3, cells=(16, 16, 16), levels=2, smoother="rbgs", coarse="sweeps", ncoarse=10),
    # whole-cycle tails (tail_level 0): mg_solve is ONE launch (plan_solve_in_tail) — on one CTA
    # with the hierarchy in shared memory, or on the 16-CTA cluster with level 0 in global memory
    dict(dim=2, cells=(64, 64), levels=5, smoother="jacobi", dtype="f32"),
    dict(dim=3, cells=(32, 32, 32), smoother="rbgs"),
    dict(dim=2, cells=(128, 128), smoother="jacobi", nu1=3, nu2=3),
    dict(dim=2, cells=(64, 64), levels=4, smoother="rbgs"),              # direct coarse 7^2 (m = 49)
]


def _flags(name):
    import paper_1406_5369_b200 as mgb
    return {"host": mgb.FLAG_HOST_LOOP, "device": 0, "baseline": mgb.FLAG_BASELINE,
            "slab": mgb.FLAG_SLAB}[name]


@pytest.mark.parametrize("case", LOOP_CASES, ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_device_loop_matches_host_loop_and_oracle(case):
    case = dict(case)
    dt = case.get("dtype", "f64")
    res = {}
    for mode in ("device", "host"):
        S, O = make(**case, flags=_flags(mode))
        u, f = wl.workload("W1", case["dim"], case["cells"], seed=42, dtype=S.np_dtype)
        du, df = S.from_numpy(u), S.from_numpy(f)
        k, hist = S.solve(du, df, 1e-10, 40)
        res[mode] = (k, np.array(hist), S.to_numpy(du))
    assert res["device"][0] == res["host"][0]
    assert np.array_equal(res["device"][1], res["host"][1])
    assert np.array_equal(res["device"][2], res["host"][2])
    uo, k_or, hist_or = O.solve(u, f, 1e-10, 40)
    assert res["device"][0] == k_or
    np.testing.assert_allclose(res["device"][1], hist_or, rtol=1e-12 if dt == "f64" else 1e-5)
    if dt == "f64":
        assert np.array_equal(res["device"][2], uo)


@pytest.mark.parametrize("variant", ["baseline", "slab"])
def test_device_loop_other_schedules(variant):
    """Op-by-op (no split) and slab-layout schedules inside the WHILE body."""
    case = dict(dim=3, cells=(64, 64, 64), smoother="rbgs")
    S, O = make(**case, flags=_flags(variant))
    u, f = wl.workload("W1", 3, (64, 64, 64), seed=5)
    du, df = S.from_numpy(u), S.from_numpy(f)
    k, hist = S.solve(du, df, 1e-9, 30)
    uo, k_or, hist_or = O.solve(u, f, 1e-9, 30)
    assert k == k_or
    np.testing.assert_allclose(hist, hist_or, rtol=1e-12)
    assert np.array_equal(S.to_numpy(du), uo)


def test_device_loop_stopping_rules_and_graph_reuse():
    """max_cycles = 0, early stop on rtol, and a cached graph reused with new rtol/max."""
    S, O = make(3, (64, 64, 64))
    u, f = wl.workload("W1", 3, (64, 64, 64), seed=42)
    du, df = S.from_numpy(u), S.from_numpy(f)
    k, hist = S.solve(du, df, 0.0, 0)
    assert k == 0 and len(hist) == 1 and abs(hist[0] / O.norm(0, u, f) - 1) <= 1e-12
    assert np.array_equal(S.to_numpy(du), u)
    k1, h1 = S.solve(du, df, 0.5, 20)          # one V(2,2) cycle reduces the residual by far more than 2x
    assert k1 == 1
    u1 = O.vcycle(u, f)
    assert np.array_equal(S.to_numpy(du), u1)
    k2, h2 = S.solve(du, df, 0.0, 3)            # same (u, f): same graph, new parameters
    assert k2 == 3 and h2[0] == h1[1]
    uo = u1
    for _ in range(3):
        uo = O.vcycle(uo, f)
    assert np.array_equal(S.to_numpy(du), uo)


@pytest.mark.parametrize("mode", ["device", "host"])
def test_nonfinite_initial_residual(mode):
    import paper_1406_5369_b200 as mgb
    S, _ = make(3, (32, 32, 32), flags=_flags(mode))
    u, f = wl.workload("W1", 3, (32, 32, 32), seed=1)
    f[5, 6, 7] = np.nan
    du, df = S.from_numpy(u), S.from_numpy(f)
    with pytest.raises(mgb.MGError) as ei:
        S.solve(du, df, 1e-10, 5)
    assert ei.value.status == 6
    assert np.array_equal(S.to_numpy(du), u)   # no cycle ran
    # the solver is not poisoned: a clean solve works afterwards
    f[5, 6, 7] = 0.0
    df = S.from_numpy(f)
    k, _ = S.solve(du, df, 0.0, 1)
    assert k == 1


@pytest.mark.parametrize("host", [False, True], ids=["device", "host"])
def test_negative_rtol_runs_exactly_max_cycles(host):
    """rtol < 0 switches the residual test off (mg.h): a solve from the exact solution
    (u = f = 0, r0 = 0) runs every requested cycle, while rtol = 0 stops after one
    (r1 = 0 <= 0 * r0).  The bench relies on it: W1 (f = 0) decays ~10x per cycle and
    reaches an exact zero after a few hundred cycles.  NaN rtol is rejected."""
    import paper_1406_5369_b200 as mgb
    flags = mgb.FLAG_HOST_LOOP if host else 0
    S, _ = make(3, (32, 32, 32), smoother="rbgs", flags=flags)
    u, f = S.empty(), S.empty()
    k, hist = S.solve(u, f, 0.0, 7)
    assert k == 1 and hist[0] == 0.0 and hist[1] == 0.0
    k, hist = S.solve(u, f, -1.0, 7)
    assert k == 7 and len(hist) == 8 and all(h == 0.0 for h in hist)
    with pytest.raises(mgb.MGError):
        S.solve(u, f, float("nan"), 3)


@pytest.mark.parametrize("case", [dict(dim=2, cells=(64, 64), levels=5, smoother="jacobi"),
                                  dict(dim=3, cells=(32, 32, 32), smoother="rbgs")],
                         ids=["C1-one-CTA", "3D-cluster"])
def test_whole_cycle_tail_solve_is_one_launch(case):
    """On a grid whose whole cycle is the coarse tail, mg_solve is ONE kernel launch (r0, the
    cycles, their norms and the stop test inside k_tail; profiling makes the launch eager, the
    same kernel), and its results are bitwise those of the per-cycle host loop."""
    import paper_1406_5369_b200 as mgb
    S, O = make(**case)
    u, f = wl.workload("W1", case["dim"], case["cells"], seed=3, dtype=S.np_dtype)
    du, df = S.from_numpy(u), S.from_numpy(f)
    S.profile_enable(True)
    k, hist = S.solve(du, df, 0.0, 6)
    recs = S.profile_read()
    S.profile_enable(False)
    ours = [r for r in recs if not r["name"].startswith("memset")]
    assert [r["name"].split("@")[0] for r in ours] == ["coarse_tail_solve"]
    assert ours[0]["count"] == 1
    H, _ = make(**case, flags=mgb.FLAG_HOST_LOOP)
    dh = H.from_numpy(u)
    kh, hh = H.solve(dh, H.from_numpy(f), 0.0, 6)
    assert k == kh and np.array_equal(np.array(hist), np.array(hh))
    assert np.array_equal(S.to_numpy(du), H.to_numpy(dh))


@pytest.mark.parametrize("host", [False, True], ids=["device", "host"])
def test_whole_cycle_tail_jacobi_stopping_rules(host):
    """The one-launch Jacobi solve takes each norm from the next cycle's first sweep: max_cycles
    = 0, a non-finite r0, rtol < 0 (exactly max cycles) and an early rtol stop must leave u
    exactly as the per-cycle loop does."""
    import paper_1406_5369_b200 as mgb
    flags = mgb.FLAG_HOST_LOOP if host else 0
    case = dict(dim=2, cells=(64, 64), levels=5, smoother="jacobi")
    S, O = make(**case, flags=flags)
    u, f = wl.workload("W1", 2, (64, 64), seed=11)
    du, df = S.from_numpy(u), S.from_numpy(f)
    k, hist = S.solve(du, df, 0.0, 0)
    assert k == 0 and len(hist) == 1 and abs(hist[0] / O.norm(0, u, f) - 1) <= 1e-12
    assert np.array_equal(S.to_numpy(du), u)
    k, hist = S.solve(du, df, -1.0, 3)
    assert k == 3 and len(hist) == 4
    uo = u
    for _ in range(3):
        uo = O.vcycle(uo, f)
    assert np.array_equal(S.to_numpy(du), uo)
    k, hist = S.solve(du, df, 0.5, 10)
    assert k == 1
    assert np.array_equal(S.to_numpy(du), O.vcycle(uo, f))
    f2 = f.copy()
    f2[7, 9] = np.nan
    d2 = S.from_numpy(u)
    with pytest.raises(mgb.MGError) as ei:
        S.solve(d2, S.from_numpy(f2), 1e-10, 5)
    assert ei.value.status == 6
    assert np.array_equal(S.to_numpy(d2), u)
