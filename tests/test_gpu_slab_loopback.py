"""The multi-rank (z-slab) path of libmgb200 executed on ONE GPU: P solvers of this
process (ranks 0..P-1), each driven by its own host thread and stream, joined by the
library's loopback transport (mg_loopback_group_create: the halo exchanges, the
agglomeration all-gather and the rank-sum norm become device-to-device copies ordered
by CUDA events and a host rendezvous — no kernel waits on another rank's kernel), eagerly
and replayed from one CUDA graph of the whole group.
Everything else — partition, halo planes, the overlapped interior/face sweeps, the
agglomerated coarse levels run redundantly, the deterministic norm — is the code NCCL
runs drive.  The gathered iterate must equal the single-domain oracle BIT FOR BIT."""
import threading

import numpy as np
import pytest

from paper_1406_5369_b200 import workloads as wl

from test_gpu_parity import make

pytestmark = pytest.mark.gpu


def _run_ranks(P, case, cycles, u, f, graph=False):
    import torch
    import paper_1406_5369_b200 as mgb
    group = mgb.LoopbackGroup(P)
    solvers = []
    for p in range(P):
        S = mgb.Solver(case["dim"], tuple(c + 1 for c in case["cells"]), levels=case.get("levels", 0),
                       smoother=case.get("smoother", "rbgs"), omega=case.get("omega"), nu1=case.get("nu1", 2),
                       nu2=case.get("nu2", 2), coarse=case.get("coarse", "direct"), dtype=case.get("dtype", "f64"),
                       rank=p, nranks=P, loopback=group, flags=0 if graph else mgb.FLAG_NO_GRAPH, pm_min_nx=16)
        solvers.append(S)
    streams = [torch.cuda.Stream() for _ in range(P)]
    dus = [S.from_numpy(u) for S in solvers]
    dfs = [S.from_numpy(f) for S in solvers]
    torch.cuda.synchronize()
    norms = [[None] * cycles for _ in range(P)]
    errors = []

    def work(p):
        try:
            S = solvers[p]
            for k in range(cycles):
                S.vcycle(dus[p], dfs[p], stream=streams[p])
                norms[p][k] = S.residual_norm(dus[p], dfs[p], stream=streams[p])
            streams[p].synchronize()
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)

    ts = [threading.Thread(target=work, args=(p,), daemon=True) for p in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errors, errors
    assert not any(t.is_alive() for t in ts), "rank thread hung"
    parts = [S.to_numpy(du) for S, du in zip(solvers, dus)]
    dist = solvers[0].distributed
    for S in solvers:
        S.close()
    group.close()
    return np.concatenate(parts, axis=0), norms, dist


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("case", [
    dict(dim=3, cells=(128, 128, 128), smoother="rbgs"),
    dict(dim=3, cells=(64, 64, 64), smoother="jacobi", nu1=2, nu2=1),
    dict(dim=2, cells=(256, 256), smoother="rbgs"),
    dict(dim=3, cells=(128, 128, 128), smoother="rbgs", dtype="f32"),
], ids=lambda c: "-".join(f"{k}{v}" for k, v in c.items()))
@pytest.mark.parametrize("graph", [False, True], ids=["eager", "graph"])
def test_slab_loopback_bitwise_vs_oracle(P, case, graph):
    """graph: every rank's cycle replayed from ONE CUDA graph of the loopback group (comm.cu
    loop_graph_part: the exchanges' cross-rank event edges captured), as NCCL runs capture
    their per-rank graphs with the send/recv inside."""
    cycles = 2
    S0, O = make(**case)
    u, f = wl.workload("W1", case["dim"], case["cells"], seed=42, dtype=S0.np_dtype)
    got, norms, dist = _run_ranks(P, case, cycles, u, f, graph)
    assert dist, "the level-0 grid should be distributed"
    uo = u.copy()
    for _ in range(cycles):
        O.vcycle_inplace(uo, f)
    if case.get("dtype", "f64") == "f64":
        assert np.array_equal(got, uo)
    else:
        assert np.abs(got - uo).max() <= 1e-5 * np.abs(uo).max()
        assert np.array_equal(got, uo)
    ref = O.norm(0, uo, f)
    for p in range(P):
        assert norms[p][-1] == norms[0][-1]  # every rank sums the rank partials in rank order
        assert abs(norms[p][-1] / ref - 1) <= 1e-12


@pytest.mark.parametrize("graph", [False, True], ids=["eager", "graph"])
def test_slab_loopback_solve_and_p8(graph):
    """mg_solve on 8 ranks (the pipelined host loop of the multi-rank path: the norm after
    each cycle comes from the next cycle's first sweep): the cycle count and history equal
    the single-domain oracle's, the iterate bitwise."""
    import torch
    import paper_1406_5369_b200 as mgb
    P, cells = 8, (128, 128, 128)
    S0, O = make(3, cells)
    u, f = wl.workload("W1", 3, cells, seed=42)
    group = mgb.LoopbackGroup(P)
    solvers = [mgb.Solver(3, tuple(c + 1 for c in cells), rank=p, nranks=P, loopback=group,
                          flags=0 if graph else mgb.FLAG_NO_GRAPH, pm_min_nx=16) for p in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    dus = [S.from_numpy(u) for S in solvers]
    dfs = [S.from_numpy(f) for S in solvers]
    torch.cuda.synchronize()
    out = [None] * P
    errors = []

    def work(p):
        try:
            out[p] = solvers[p].solve(dus[p], dfs[p], 1e-10, 40, stream=streams[p])
        except Exception as e:  # pragma: no cover
            errors.append(e)

    ts = [threading.Thread(target=work, args=(p,), daemon=True) for p in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not errors, errors
    uo, k_or, hist_or = O.solve(u, f, 1e-10, 40)
    for p in range(P):
        k, hist = out[p]
        assert k == k_or
        np.testing.assert_allclose(hist, hist_or, rtol=1e-12)
    got = np.concatenate([S.to_numpy(du) for S, du in zip(solvers, dus)], axis=0)
    assert np.array_equal(got, uo)
    for S in solvers:
        S.close()
    group.close()


def _random_slab_cases(n, seed=31):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        dim = int(rng.choice([2, 3]))
        P = int(rng.choice([2, 4]))
        levels = int(rng.integers(3, 5))
        m = 1 << (levels - 1)
        hi = 48 if dim == 3 else 320
        cells = [int(m * rng.integers(2, hi // m + 1)) for _ in range(dim)]
        cells[-1] = P * m * int(rng.integers(2, 5))  # slab axis: >= 8 (even) planes per rank on level 0
        unknowns = int(np.prod([c // m - 1 for c in cells]))
        out.append(dict(P=P, dim=dim, cells=tuple(cells), levels=levels, smoother=str(rng.choice(["rbgs", "jacobi"])),
                        nu1=int(rng.integers(1, 4)), nu2=int(rng.integers(1, 4)),
                        dtype=str(rng.choice(["f64", "f32"])), coarse="direct" if unknowns <= 1024 else "sweeps"))
    return out


@pytest.mark.parametrize("case", _random_slab_cases(30),
                         ids=lambda c: "P{P}-{dim}d-{c}-L{levels}-{smoother}-nu{nu1}{nu2}-{dtype}".format(
                             c="x".join(map(str, c["cells"])), **c))
@pytest.mark.parametrize("graph", [False, True], ids=["eager", "graph"])
def test_slab_loopback_random_bitwise(case, graph):
    """Seeded random slab decompositions: ragged in-plane extents, both smoothers, odd and even
    sweep counts, FP32/FP64 — the gathered iterate equals the single-domain oracle bitwise."""
    case = dict(case)
    P = case.pop("P")
    S0, O = make(case["dim"], case["cells"], case["levels"], case["smoother"], nu1=case["nu1"], nu2=case["nu2"],
                 dtype=case["dtype"], coarse=case["coarse"])
    u, f = wl.workload("W4", case["dim"], case["cells"], seed=9, dtype=S0.np_dtype)
    got, norms, dist = _run_ranks(P, case, 2, u, f, graph)
    assert dist
    uo = u.copy()
    for _ in range(2):
        O.vcycle_inplace(uo, f)
    assert np.array_equal(got, uo)
