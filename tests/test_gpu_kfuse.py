"""Temporal blocking of the 2D omega-Jacobi smoother (kernels_pm2d.cu k_jacobi2d_k):
n sweeps run as passes of up to 3 (FP32) / 2 (FP64) fused sweeps over overlapping
strips, and the level-0 prolongation writes out of place when the pass count changes
the ping-pong parity.  Every value is a single sweep's canonical arithmetic, so the
cycle is bitwise the oracle's (P:287-292 Jacobi, Alg. 1) in both precisions, for
every (nu1, nu2) — odd and even pass counts, zero-guess first passes on coarse
levels — and on strips whose overlap meets the ragged domain edge."""
import numpy as np
import pytest

from paper_1406_5369_b200 import workloads as wl

from test_gpu_parity import make

pytestmark = pytest.mark.gpu

NU = [(1, 1), (2, 1), (2, 2), (3, 3), (4, 4), (5, 2), (0, 3), (3, 0), (6, 5)]


@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("nu", NU, ids=lambda n: f"nu{n[0]}{n[1]}")
def test_kfused_jacobi_cycle_bitwise(nu, dt):
    cells = (304, 192)  # 305 x 193 nodes: 3 overlapping FP32 strips (stride 120), 6 FP64 (stride 60)
    S, O = make(2, cells, 5, "jacobi", nu1=nu[0], nu2=nu[1], dtype=dt, pm_min_nx=0)
    u, f = wl.workload("W4", 2, cells, seed=21, dtype=S.np_dtype)
    u = u + wl.random_interior(2, cells, 4, S.np_dtype)
    du, df = S.from_numpy(u), S.from_numpy(f)
    uo = u.copy()
    for k in range(2):
        S.vcycle(du, df)
        O.vcycle_inplace(uo, f)
        assert np.array_equal(S.to_numpy(du), uo), (nu, dt, k)


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_kfused_jacobi_solve_bitwise(dt):
    """mg_solve pipelines tail(k) + head(k+1): the head's sweep + norm precedes the fused
    pre-smoothing passes; iterates and the residual history stay the oracle's."""
    cells = (512, 384)
    S, O = make(2, cells, smoother="jacobi", nu1=3, nu2=3, dtype=dt, pm_min_nx=0)
    u, f = wl.workload("W1", 2, cells, seed=5, dtype=S.np_dtype)
    du, df = S.from_numpy(u), S.from_numpy(f)
    k, hist = S.solve(du, df, 0.0, 3)
    uo, k_or, hist_or = O.solve(u, f, 0.0, 3)
    assert k == k_or == 3
    assert np.array_equal(S.to_numpy(du), uo)
    assert all(abs(a / b - 1) <= 1e-12 for a, b in zip(hist, hist_or))


def test_kfused_wide_domain_strip_edges():
    """x extents around the strip stride (FP32: 120 columns per strip, 4 overlap each side):
    the stored columns of neighbouring strips tile [0, nx] exactly."""
    for nx in (112, 120, 128, 232, 240, 248, 360):
        for cells in ((nx, 40), (40, nx)):  # either axis may be the strip (pitch) axis
            S, O = make(2, cells, 3, "jacobi", nu1=3, nu2=3, dtype="f32", pm_min_nx=0)
            u, f = wl.workload("W4", 2, cells, seed=nx, dtype=S.np_dtype)
            du, df = S.from_numpy(u), S.from_numpy(f)
            S.vcycle(du, df)
            assert np.array_equal(S.to_numpy(du), O.vcycle(u, f)), cells
