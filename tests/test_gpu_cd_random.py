"""Seeded randomized complex-diffusion configurations against oracle/cd_oracle.c: dimension,
cell extents (ragged against the 2D strips and 3D tiles), smoother, (nu1, nu2), precision and
levels; the FAS cycle must equal the oracle bitwise through mg_vcycle and the pipelined solve
(fused head), which exercises the warp-marching (2D) and plane-marching (3D) kernels and the
single-CTA tail."""
import numpy as np
import pytest

from paper_1406_5369_b200 import workloads as wl

from test_gpu_cd import make

pytestmark = pytest.mark.gpu


def _configs(n, seed=99):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        dim = int(rng.choice([2, 3]))
        levels = int(rng.integers(2, 4))
        m = 1 << (levels - 1)
        hi = 72 if dim == 3 else 400
        cells = tuple(int(m * rng.integers(max(2, 8 // m), hi // m + 1)) for _ in range(dim))
        sm = str(rng.choice(["rbgs", "jacobi"]))
        nu1, nu2 = int(rng.integers(0, 4)), int(rng.integers(0, 4))
        if nu1 + nu2 == 0:
            continue
        out.append(dict(dim=dim, cells=cells, levels=levels, smoother=sm, nu1=nu1, nu2=nu2,
                        dtype=str(rng.choice(["f64", "f32"]))))
    return out


CASES = _configs(30) + _configs(50, seed=3)


@pytest.mark.parametrize("case", CASES, ids=lambda c: "{dim}d-{c}-L{levels}-{smoother}-nu{nu1}{nu2}-{dtype}".format(
    c="x".join(map(str, c["cells"])), **c))
def test_cd_random_config_bitwise(case):
    S, O = make(case["dim"], case["cells"], case["levels"], case["smoother"], nu1=case["nu1"], nu2=case["nu2"],
                dtype=case["dtype"])
    u, f = wl.cd_workload(case["dim"], case["cells"], seed=5, dtype=S.np_dtype)
    du, df = S.from_numpy(u), S.from_numpy(f)
    uo = u.copy()
    for k in range(2):
        S.vcycle(du, df)
        uo = O.cycle(uo, f)
        assert np.array_equal(S.to_numpy(du), uo), ("vcycle", k)
    du2 = S.from_numpy(u)
    k, hist = S.solve(du2, df, 0.0, 2)
    uo2, k_or, hist_or = O.solve(u, f, 0.0, 2)
    assert k == k_or
    assert np.array_equal(S.to_numpy(du2), uo2), "solve"
    np.testing.assert_allclose(hist, hist_or, rtol=1e-12 if case["dtype"] == "f64" else 1e-10)
