"""2D warp-marching kernels (kernels_pm2d.cu) against the oracle: per operation and
per cycle, bitwise in FP64 (canonical operation order, no FMA), <= 1e-5 in FP32;
ragged strips (x extent not a multiple of the 64/128-node strip), odd sweep
counts, slab layout, and the C4 grid (8193^2, FP32, Jacobi V(3,3)) at full size."""
import numpy as np
import pytest

from paper_1406_5369_b200 import workloads as wl

from test_gpu_parity import TOL, make, relerr

pytestmark = pytest.mark.gpu

CASES_2D = [
    dict(dim=2, cells=(64, 64), smoother="rbgs"),
    dict(dim=2, cells=(64, 64), smoother="jacobi"),
    dict(dim=2, cells=(96, 80), levels=4, smoother="rbgs"),                 # ragged strips, 95 interior
    dict(dim=2, cells=(96, 80), levels=4, smoother="jacobi", nu1=3, nu2=3),
    dict(dim=2, cells=(320, 64), levels=4, smoother="rbgs", nu1=1, nu2=2),  # odd sweep count, 3 strips
    dict(dim=2, cells=(256, 256), smoother="jacobi", nu1=3, nu2=3, dtype="f32"),
    dict(dim=2, cells=(256, 128), smoother="rbgs", dtype="f32"),
    dict(dim=2, cells=(1024, 1024), smoother="rbgs"),
]


def _ids(c):
    return "-".join(f"{k}{v}" for k, v in c.items())


@pytest.mark.parametrize("case", CASES_2D, ids=_ids)
def test_2d_cycle_parity(case):
    dt = case.get("dtype", "f64")
    S, O = make(**case)
    u, f = wl.workload("W4", 2, case["cells"], seed=13, dtype=S.np_dtype)
    u = u + wl.random_interior(2, case["cells"], 3, S.np_dtype)  # non-zero guess and rhs
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


@pytest.mark.parametrize("sm", ["rbgs", "jacobi"])
@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_2d_per_op_parity(sm, dt):
    cells = (192, 96)
    S, O = make(2, cells, 4, sm, dtype=dt)
    u = wl.random_interior(2, cells, 5, S.np_dtype, -1.0, 1.0)
    u[0, :] = 0.25  # Dirichlet data on one edge (never written)
    f = wl.random_interior(2, cells, 6, S.np_dtype, -1.0, 1.0)
    du, df = S.from_numpy(u), S.from_numpy(f)
    out = S.empty(0)
    S.op_smooth(0, du, df, out)
    assert relerr(S.to_numpy(out, 0), O.smooth(0, u, f)) <= TOL[dt]
    if dt == "f64":
        assert np.array_equal(S.to_numpy(out, 0), O.smooth(0, u, f))
    assert abs(S.op_norm(0, du, df) / O.norm(0, u, f) - 1) <= 1e-12
    e = wl.random_interior(2, (96, 48), 8, S.np_dtype, -1.0, 1.0)
    du2 = S.from_numpy(u)
    S.op_prolong_correct(0, S.from_numpy(e, 1), du2)
    assert relerr(S.to_numpy(du2, 0), O.prolong_correct(0, e, u)) <= TOL[dt]


@pytest.mark.parametrize("sm", ["rbgs", "jacobi"])
def test_2d_slab_mode_single_rank(sm):
    import paper_1406_5369_b200 as mgb
    S, O = make(2, (256, 256), smoother=sm, flags=mgb.FLAG_SLAB)
    assert S.distributed and S.halo == 2
    u, f = wl.workload("W1", 2, (256, 256), seed=42)
    du, df = S.from_numpy(u), S.from_numpy(f)
    uo = u.copy()
    for _ in range(2):
        S.vcycle(du, df)
        O.vcycle_inplace(uo, f)
        assert np.array_equal(S.to_numpy(du), uo)


def test_2d_schedules_identical():
    """warp-marching (default) == op-by-op (MG_FLAG_BASELINE), bitwise, both smoothers."""
    import paper_1406_5369_b200 as mgb
    for sm in ("rbgs", "jacobi"):
        outs = []
        for flags in (0, mgb.FLAG_BASELINE):
            S, _ = make(2, (512, 512), smoother=sm, flags=flags, pm_min_nx=0)
            u, f = wl.workload("W4", 2, (512, 512), seed=2)
            du, df = S.from_numpy(u), S.from_numpy(f)
            for _ in range(2):
                S.vcycle(du, df)
            outs.append(S.to_numpy(du))
        assert np.array_equal(outs[0], outs[1]), sm


def test_c4_fullsize_cycle_vs_oracle():
    """C4 (8193^2 nodes, FP32, Jacobi V(3,3), 13 levels) in the bench's launch
    configuration: one cycle against the FP32 oracle."""
    S, O = make(2, (8192, 8192), smoother="jacobi", nu1=3, nu2=3, dtype="f32", pm_min_nx=0)
    u, f = wl.workload("W1", 2, (8192, 8192), seed=42, dtype=np.float32)
    du, df = S.from_numpy(u), S.from_numpy(f)
    S.vcycle(du, df)
    uo = O.vcycle(u, f)
    got = S.to_numpy(du)
    assert relerr(got, uo) <= TOL["f32"]
    assert np.array_equal(got, uo)  # same canonical order in FP32: bitwise too
