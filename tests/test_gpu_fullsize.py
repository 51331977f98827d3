"""Full-size parity at BASELINE.json's configurations, in the launch
configuration bench.py times (default solver options: plane-marching kernels,
CUDA graphs, the pipelined mg_solve driver loop).  The oracle runs the same
cycles on the host (OpenMP), C5 (1025^3, 8.6 GB per array) included; C5 is also
checked through a property that holds at any size: bitwise agreement of the fused
and the op-by-op schedules."""
import numpy as np
import pytest

import oracle as orc
from paper_1406_5369_b200 import workloads as wl

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _pair(dim, nodes, smoother, nu1, nu2, dtype, levels=0):
    import paper_1406_5369_b200 as mgb
    omega = 1.0 if smoother == "rbgs" else 0.8
    S = mgb.Solver(dim, nodes, levels=levels, smoother=smoother, omega=omega, nu1=nu1, nu2=nu2, dtype=dtype)
    O = orc.Oracle(orc.Config(dim=dim, cells=(nodes - 1,) * dim, levels=S.levels,
                              smoother=orc.RBGS if smoother == "rbgs" else orc.JACOBI, omega=omega, nu1=nu1, nu2=nu2),
                   S.np_dtype)
    return S, O


@pytest.mark.parametrize("cfg", [
    ("C3-f64", 3, 513, "rbgs", 2, 2, "f64"),
    ("C3-f32", 3, 513, "rbgs", 2, 2, "f32"),
    ("C4", 2, 8193, "jacobi", 3, 3, "f32"),
    ("C2", 3, 129, "rbgs", 2, 2, "f64"),
], ids=lambda c: c[0])
def test_fullsize_solve_to_1e10_matches_oracle(cfg):
    """North star: reduce the residual by 1e-10 with the identical iteration count; the final
    iterate within 1e-12 (FP64; bitwise expected) / 1e-5 (FP32) relative max-norm."""
    name, dim, nodes, sm, nu1, nu2, dt = cfg
    S, O = _pair(dim, nodes, sm, nu1, nu2, dt)
    u, f = wl.workload("W1", dim, (nodes - 1,) * dim, seed=42, dtype=S.np_dtype)
    du, df = S.from_numpy(u), S.from_numpy(f)
    k_gpu, hist_gpu = S.solve(du, df, 1e-10, 30)
    uo, k_or, hist_or = O.solve(u, f, 1e-10, 30)
    assert k_gpu == k_or, (k_gpu, k_or)
    np.testing.assert_allclose(hist_gpu, hist_or, rtol=1e-12 if dt == "f64" else 1e-5)
    got = S.to_numpy(du)
    den = np.abs(uo).max()
    rel = np.abs(got.astype(np.float64) - uo).max() / den
    assert rel <= (1e-12 if dt == "f64" else 1e-5), rel
    if dt == "f64":
        assert np.array_equal(got, uo)


def test_c5_solve_to_1e10_matches_oracle():
    """1025^3 FP64 RBGS V(2,2) (C5, 8.6 GB per array; SURVEY §8(d) row C5 "plus the 1e-10 count"):
    mg_solve to a 1e-10 residual reduction against the oracle on the host: the identical cycle
    count, the norm histories to 1e-12, and the full final iterate bitwise."""
    S, O = _pair(3, 1025, "rbgs", 2, 2, "f64")
    u, f = wl.workload("W1", 3, (1024,) * 3, seed=42)
    du, df = S.from_numpy(u), S.from_numpy(f)
    k, hist = S.solve(du, df, 1e-10, 30)
    uo, k_or, hist_or = O.solve(u, f, 1e-10, 30)
    del u
    assert k == k_or, (k, k_or)
    np.testing.assert_allclose(hist, hist_or, rtol=1e-12)
    assert hist[-1] <= 1e-10 * hist[0] and hist[-2] > 1e-10 * hist[0]
    got = S.to_numpy(du)
    assert np.array_equal(got, uo)
    assert all(hist[i + 1] / hist[i] < 0.2 for i in range(k)), hist


def test_c5_fused_equals_op_by_op():
    """Property at any size: the fused plane-marching schedule and the op-by-op schedule give
    bitwise identical iterates (every 64th plane compared) and norms to 1e-12."""
    import torch

    import paper_1406_5369_b200 as mgb
    outs, hists = [], []
    for flags in (0, mgb.FLAG_BASELINE):
        S = mgb.Solver(3, 1025, smoother="rbgs", flags=flags)
        u, f = S.empty(), S.empty()
        S.workload_fill(u, 42)
        k, hist = S.solve(u, f, 0.0, 2)
        hists.append(hist)
        outs.append(u[::64].clone())
        del u, f, S
        torch.cuda.empty_cache()
    assert torch.equal(outs[0], outs[1])
    np.testing.assert_allclose(hists[0], hists[1], rtol=1e-12)
