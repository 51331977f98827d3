"""Degenerate and edge configurations against the oracle, bitwise: one unknown, the
smallest grids, no pre- or post-smoothing, nu1 = 0 (no pipelined head), coarse SWEEPS
with a single sweep, and mg_solve with rtol = 0 / a zero residual."""
import numpy as np
import pytest

from paper_1406_5369_b200 import workloads as wl

from test_gpu_parity import make

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", [
    dict(dim=2, cells=(2, 2), levels=1),                                   # one unknown, f/D
    dict(dim=3, cells=(2, 2, 2), levels=1),
    dict(dim=2, cells=(4, 2), levels=1),                                   # 3 unknowns, Cholesky
    dict(dim=3, cells=(4, 4, 4), levels=2, smoother="jacobi"),
    dict(dim=3, cells=(64, 64, 64), nu1=0, nu2=2),                         # no head sweep to pipeline
    dict(dim=3, cells=(64, 64, 64), nu1=2, nu2=0),
    dict(dim=2, cells=(128, 128), nu1=0, nu2=0, smoother="jacobi"),        # pure coarse-grid correction
    dict(dim=3, cells=(32, 32, 32), coarse="sweeps", ncoarse=1),
    dict(dim=2, cells=(256, 4), levels=2),                                 # very flat 2D grid
], ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
def test_degenerate_cycle_parity(case):
    S, O = make(**case)
    u, f = wl.workload("W4", case["dim"], case["cells"], seed=3, dtype=S.np_dtype)
    u = u + wl.random_interior(case["dim"], case["cells"], 4, S.np_dtype)
    du, df = S.from_numpy(u), S.from_numpy(f)
    uo = u.copy()
    for _ in range(2):
        S.vcycle(du, df)
        O.vcycle_inplace(uo, f)
        assert np.array_equal(S.to_numpy(du), uo)
    k, hist = S.solve(du, df, 0.0, 2)
    uo2, k2, hist2 = O.solve(uo, f, 0.0, 2)
    assert k == k2  # (2 unless the iterate is already exact: r0 = 0 stops after one cycle)
    np.testing.assert_allclose(hist, hist2, rtol=1e-12, atol=1e-300)
    assert np.array_equal(S.to_numpy(du), uo2)


def test_one_unknown_is_exact_in_one_cycle():
    S, O = make(2, (2, 2), levels=1)
    u, f = wl.workload("W4", 2, (2, 2), seed=5)
    du, df = S.from_numpy(u), S.from_numpy(f)
    k, hist = S.solve(du, df, 1e-300, 5)
    assert hist[1] == 0.0 and k == 1


def test_zero_residual_stops_after_one_cycle():
    """u = 0, f = 0: r0 = 0, and the stopping test r_k <= rtol r0 holds at k = 1."""
    S, _ = make(3, (32, 32, 32))
    du, df = S.empty(), S.empty()
    k, hist = S.solve(du, df, 1e-10, 10)
    assert k == 1 and hist == [0.0, 0.0]


def test_bad_arguments_fail_without_poisoning():
    """Misaligned or NULL device arrays are rejected up front (MG_ERR_LAYOUT / MG_ERR_INVALID)
    and leave the solver usable."""
    import ctypes
    import paper_1406_5369_b200 as mgb
    S, O = make(3, (32, 32, 32))
    u, f = wl.workload("W1", 3, (32, 32, 32), seed=42)
    du, df = S.from_numpy(u), S.from_numpy(f)
    bad = ctypes.c_void_p(du.data_ptr() + 8)
    out = ctypes.c_double()
    assert S.lib.mg_residual_norm(S.h, bad, S._p(df), ctypes.byref(out), None) == 7
    assert S.lib.mg_vcycle(S.h, bad, S._p(df), None) == 7
    k = ctypes.c_int32()
    assert S.lib.mg_solve(S.h, None, S._p(df), 0.0, 1, ctypes.byref(k), None, None) == 1
    assert S.lib.mg_op_smooth(S.h, 0, S._p(du), bad, S._p(du), None) == 7
    S.vcycle(du, df)  # still usable
    assert np.array_equal(S.to_numpy(du), O.vcycle(u, f))


def test_binding_rejects_bad_tensors():
    """The Python binding checks what a raw pointer cannot carry (device, dtype, layout
    shape, contiguity) before the C ABI sees it: no kernel ever touches a wrong-sized array."""
    import torch
    from test_gpu_parity import make
    S, _ = make(3, (32, 32, 32), smoother="rbgs")
    u, f = S.empty(), S.empty()
    bad = [
        (u.cpu(), TypeError, ValueError),                     # host tensor
        (u.float(), TypeError, ValueError),                   # wrong dtype
        (u[:, :, :-8], ValueError, TypeError),                # wrong shape
        (u.transpose(0, 2).contiguous(), ValueError, TypeError),
        (torch.empty_strided(u.shape, (1, u.shape[0], u.shape[0] * u.shape[1]), dtype=u.dtype, device=u.device),
         ValueError, TypeError),                              # non-contiguous
    ]
    for t, *errs in bad:
        with pytest.raises(tuple(errs)):
            S.vcycle(t, f)
        with pytest.raises(tuple(errs)):
            S.solve(u, t, 0.0, 1)
    with pytest.raises(ValueError):
        S.op_restrict(0, S.empty(0), S.empty(0))  # fc must have the level-1 layout
    S.vcycle(u, f)  # the solver is still usable
