"""Temporal blocking of the 2D complex-diffusion Jacobi smoother (kernels_cd2d.cu
k_cd_jacobi2d_k): up to 3 (FP32) / 2 (FP64) sweeps with the frozen lagged diffusivity
per pass over overlapping strips (opt-in, MG_FLAG_CD_KFUSE; measured slower than single sweeps,
DESIGN.md §10), one more level-0 post pass when the pass count would change the
ping-pong parity, and the solve's head = g(u) + the first pre-smoothing pass with
||f - A(g(u)) u|| accumulated by its first stage (default).  Every cell value is a single
sweep's canonical complex arithmetic (reading 19), so iterates stay
bitwise the oracle's (oracle/cd_oracle.c) for every (nu1, nu2)."""
import numpy as np
import pytest

from paper_1406_5369_b200 import workloads as wl

from test_gpu_cd import make

pytestmark = pytest.mark.gpu

NU = [(1, 1), (2, 1), (1, 2), (2, 2), (3, 3), (4, 3), (0, 2), (5, 4)]


@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("nu", NU, ids=lambda n: f"nu{n[0]}{n[1]}")
def test_cd_kfused_cycle_bitwise(nu, dt):
    cells = (248, 72)  # FP32: 5 overlapping strips of 60 cells (ragged), FP64: 9 of 30
    S, O = make(2, cells, 3, "jacobi", nu1=nu[0], nu2=nu[1], dtype=dt)
    u, f = wl.cd_workload(2, cells, seed=7, dtype=S.np_dtype)
    du, df = S.from_numpy(u), S.from_numpy(f)
    uo = u.copy()
    for k in range(2):
        S.vcycle(du, df)
        uo = O.cycle(uo, f)
        assert np.array_equal(S.to_numpy(du), uo), (nu, dt, k)


@pytest.mark.parametrize("dt", ["f32", "f64"])
@pytest.mark.parametrize("nu", [(2, 2), (3, 1), (1, 1)], ids=lambda n: f"nu{n[0]}{n[1]}")
def test_cd_kfused_solve_head(nu, dt):
    """mg_solve: the head's fused pass (norm of the input + first pre-sweeps) and the tail
    reproduce the oracle's iterates and residual history."""
    cells = (256, 192)
    S, O = make(2, cells, smoother="jacobi", nu1=nu[0], nu2=nu[1], dtype=dt)
    u, f = wl.cd_workload(2, cells, seed=3, dtype=S.np_dtype)
    du, df = S.from_numpy(u), S.from_numpy(f)
    k, hist = S.solve(du, df, 0.0, 3)
    uo, k_or, hist_or = O.solve(u, f, 0.0, 3)
    assert k == k_or == 3
    assert np.array_equal(S.to_numpy(du), uo)
    np.testing.assert_allclose(hist, hist_or, rtol=1e-12 if dt == "f64" else 1e-10)


def test_cd_kfused_strip_edges():
    """x extents around the FP32 strip stride (60 cells): stored cells of neighbouring
    strips tile [0, nx) exactly, Neumann faces at both ends."""
    for nx in (64, 120, 124, 180, 184):
        cells = (nx, 32)
        S, O = make(2, cells, 2, "jacobi", nu1=3, nu2=3, dtype="f32")
        u, f = wl.cd_workload(2, cells, seed=nx, dtype=S.np_dtype)
        du, df = S.from_numpy(u), S.from_numpy(f)
        S.vcycle(du, df)
        assert np.array_equal(S.to_numpy(du), O.cycle(u, f)), cells


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_cd_multisweep_passes_bitwise(dt):
    """MG_FLAG_CD_KFUSE: passes of 3 (FP32) / 2 (FP64) sweeps, every (nu1, nu2) of NU; solve and
    vcycle bitwise equal to the oracle."""
    import paper_1406_5369_b200 as mgb
    bad = []
    for nu in NU:
        S, O = make(2, (248, 72), 3, "jacobi", nu1=nu[0], nu2=nu[1], dtype=dt, flags=mgb.FLAG_CD_KFUSE)
        u, f = wl.cd_workload(2, (248, 72), seed=7, dtype=S.np_dtype)
        du, df = S.from_numpy(u), S.from_numpy(f)
        k, hist = S.solve(du, df, 0.0, 2)
        uo, k_or, hist_or = O.solve(u, f, 0.0, 2)
        if not np.array_equal(S.to_numpy(du), uo):
            bad.append(nu)
        S.vcycle(du, df)
        uo = O.cycle(uo, f)
        if not np.array_equal(S.to_numpy(du), uo):
            bad.append((nu, "vcycle"))
    assert not bad, bad
