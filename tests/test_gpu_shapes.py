"""3D plane-marching kernels on non-cubic grids that are ragged in BOTH tile axes
(x: tiles of 64 FP64 / 128 FP32 nodes, y: 16 rows) and span several tiles, plus short
z extents (few planes per z-chunk): two cycles bitwise equal to the oracle (Alg. 1 with
the canonical per-node order), both smoothers, both precisions, and the opt-in fused
prolongation.  pm_min_nx = 0 puts every level above the tail on the marching kernels."""
import numpy as np
import pytest

from paper_1406_5369_b200 import workloads as wl

from test_gpu_parity import make

pytestmark = pytest.mark.gpu

SHAPES = [(160, 104, 40), (200, 56, 24), (72, 136, 16)]


@pytest.mark.parametrize("dt", ["f64", "f32"])
@pytest.mark.parametrize("sm", ["rbgs", "jacobi"])
@pytest.mark.parametrize("cells", SHAPES, ids=lambda c: "x".join(map(str, c)))
def test_ragged_3d_bitwise(cells, sm, dt):
    S, O = make(3, cells, 4, sm, dtype=dt, pm_min_nx=0)  # coarsest <= 912 unknowns (direct)
    u, f = wl.workload("W4", 3, cells, seed=11, dtype=S.np_dtype)
    u = u + wl.random_interior(3, cells, 12, S.np_dtype)
    du, df = S.from_numpy(u), S.from_numpy(f)
    uo = u.copy()
    for k in range(2):
        S.vcycle(du, df)
        O.vcycle_inplace(uo, f)
        assert np.array_equal(S.to_numpy(du), uo), (cells, sm, dt, k)
    assert abs(S.residual_norm(du, df) / O.norm(0, uo, f) - 1) <= 1e-12


@pytest.mark.parametrize("dt", ["f64", "f32"])
def test_ragged_3d_separate_prolongation(dt):
    import paper_1406_5369_b200 as mgb
    cells = (160, 104, 40)
    S, O = make(3, cells, 4, "rbgs", dtype=dt, pm_min_nx=0, flags=mgb.FLAG_SEPARATE_PROLONG)
    u, f = wl.workload("W4", 3, cells, seed=13, dtype=S.np_dtype)
    du, df = S.from_numpy(u), S.from_numpy(f)
    uo = u.copy()
    for k in range(2):
        S.vcycle(du, df)
        O.vcycle_inplace(uo, f)
        assert np.array_equal(S.to_numpy(du), uo), (dt, k)
