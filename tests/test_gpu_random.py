"""Seeded randomized configurations against the oracle: dimension, extents (ragged against
every tile / strip width), smoother, (nu1, nu2) including every pass split and parity case of
the fused 2D Jacobi passes, precision, levels and coarse solver; the plane/warp-marching
kernels are forced onto every level above the tail (pm_min_nx = 0).  Two cycles through
mg_vcycle and a short mg_solve (pipelined head) must equal the oracle bitwise."""
import numpy as np
import pytest

from paper_1406_5369_b200 import workloads as wl

from test_gpu_parity import make

pytestmark = pytest.mark.gpu


def _configs(n, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        dim = int(rng.choice([2, 3]))
        levels = int(rng.integers(2, 5))
        m = 1 << (levels - 1)
        hi = 96 if dim == 3 else 640
        cells = tuple(int(m * rng.integers(max(2, 16 // m), hi // m + 1)) for _ in range(dim))
        sm = str(rng.choice(["rbgs", "jacobi"]))
        nu1, nu2 = int(rng.integers(0, 5)), int(rng.integers(0, 5))
        if nu1 + nu2 == 0:
            continue
        dt = str(rng.choice(["f64", "f32"]))
        coarse_cells = [c // m for c in cells]
        unknowns = int(np.prod([c - 1 for c in coarse_cells]))
        coarse = "direct" if unknowns <= 1024 else "sweeps"
        out.append(dict(dim=dim, cells=cells, levels=levels, smoother=sm, nu1=nu1, nu2=nu2, dtype=dt, coarse=coarse))
    return out


CASES = _configs(40) + _configs(80, seed=7)


@pytest.mark.parametrize("case", CASES, ids=lambda c: "{dim}d-{c}-L{levels}-{smoother}-nu{nu1}{nu2}-{dtype}-{coarse}".format(
    c="x".join(map(str, c["cells"])), **c))
def test_random_config_bitwise(case):
    S, O = make(case["dim"], case["cells"], case["levels"], case["smoother"], nu1=case["nu1"], nu2=case["nu2"],
                dtype=case["dtype"], coarse=case["coarse"], pm_min_nx=0)
    u, f = wl.workload("W4", case["dim"], case["cells"], seed=17, dtype=S.np_dtype)
    u = u + wl.random_interior(case["dim"], case["cells"], 18, S.np_dtype)
    du, df = S.from_numpy(u), S.from_numpy(f)
    uo = u.copy()
    for k in range(2):
        S.vcycle(du, df)
        O.vcycle_inplace(uo, f)
        assert np.array_equal(S.to_numpy(du), uo), ("vcycle", k)
    du2 = S.from_numpy(u)
    k, hist = S.solve(du2, df, 0.0, 2)
    uo2, k_or, hist_or = O.solve(u, f, 0.0, 2)
    assert k == k_or
    assert np.array_equal(S.to_numpy(du2), uo2), "solve"
    assert all(abs(a / b - 1) <= 1e-12 for a, b in zip(hist, hist_or) if b != 0)
