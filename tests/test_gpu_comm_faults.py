"""The multi-rank failure path (mg.h mg_fault_inject, comm_timeout_s) on one GPU
through the loopback transport: a failed halo exchange returns MG_ERR_NCCL and poisons the
solver (every later call: MG_ERR_POISONED); a rank whose peer failed does not hang but gives up
after comm_timeout_s with MG_ERR_NCCL; a silently corrupted halo is caught by the bitwise parity
check against the oracle; destroying poisoned solvers returns."""
import threading

import numpy as np
import pytest

from paper_1406_5369_b200 import workloads as wl

pytestmark = pytest.mark.gpu

CELLS = (32, 32, 32)


def _ranks(P, timeout=0.0):
    import paper_1406_5369_b200 as mgb
    group = mgb.LoopbackGroup(P)
    solvers = [mgb.Solver(3, tuple(c + 1 for c in CELLS), rank=p, nranks=P, loopback=group,
                          flags=mgb.FLAG_NO_GRAPH, pm_min_nx=16, comm_timeout_s=timeout) for p in range(P)]
    return group, solvers


def _drive(solvers, fn, join_s=120):
    import torch
    out = [None] * len(solvers)
    streams = [torch.cuda.Stream() for _ in solvers]

    def work(p):
        try:
            out[p] = ("ok", fn(p, solvers[p], streams[p]))
        except Exception as e:
            out[p] = ("err", e)

    ts = [threading.Thread(target=work, args=(p,), daemon=True) for p in range(len(solvers))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=join_s)
    assert not any(t.is_alive() for t in ts), "a rank thread hung"
    return out


def _inputs(S):
    u, f = wl.workload("W1", 3, CELLS, seed=42)
    return S.from_numpy(u), S.from_numpy(f), u, f


def test_injected_comm_error_returns_nccl_status_and_poisons():
    import paper_1406_5369_b200 as mgb
    group, solvers = _ranks(2)
    data = [_inputs(S) for S in solvers]
    for S in solvers:
        S.fault_inject(mgb.FAULT_COMM_ERROR, 3)

    def fn(p, S, st):
        du, df = data[p][0], data[p][1]
        S.vcycle(du, df, stream=st)
        st.synchronize()

    res = _drive(solvers, fn)
    for kind, e in res:
        assert kind == "err" and isinstance(e, mgb.MGError) and e.status == 5, res  # MG_ERR_NCCL
        assert "injected" in str(e)
    for p, S in enumerate(solvers):  # poisoned: every later call fails fast
        with pytest.raises(mgb.MGError) as ei:
            S.vcycle(data[p][0], data[p][1])
        assert ei.value.status == 8  # MG_ERR_POISONED
    for S in solvers:
        S.close()
    group.close()


def test_peer_failure_times_out_instead_of_hanging():
    """Rank 1's exchange fails; rank 0 waits in the rendezvous for a peer that never comes and
    gives up after comm_timeout_s (2 s) with MG_ERR_NCCL rather than blocking forever."""
    import time

    import paper_1406_5369_b200 as mgb
    group, solvers = _ranks(2, timeout=2.0)
    data = [_inputs(S) for S in solvers]
    solvers[1].fault_inject(mgb.FAULT_COMM_ERROR, 2)
    t0 = time.time()

    def fn(p, S, st):
        for _ in range(3):
            S.vcycle(data[p][0], data[p][1], stream=st)
        st.synchronize()

    res = _drive(solvers, fn, join_s=60)
    assert time.time() - t0 < 30
    assert all(kind == "err" and e.status == 5 for kind, e in res), res
    assert "injected" in str(res[1][1]) and "peer" in str(res[0][1])
    for S in solvers:
        S.close()
    group.close()


def test_corrupted_halo_is_caught_by_parity():
    """MG_FAULT_HALO_CORRUPT: the exchange completes with wrong halo values; the gathered iterate
    is then no longer the oracle's, while the same run without the fault is bitwise equal."""
    import oracle as orc
    import paper_1406_5369_b200 as mgb
    u, f = wl.workload("W1", 3, CELLS, seed=42)
    ref = orc.Oracle(orc.Config(dim=3, cells=CELLS), np.float64).vcycle(u, f)
    for corrupt in (False, True):
        group, solvers = _ranks(2)
        dus = [S.from_numpy(u) for S in solvers]
        dfs = [S.from_numpy(f) for S in solvers]
        if corrupt:
            for S in solvers:
                S.fault_inject(mgb.FAULT_HALO_CORRUPT, 2)

        def fn(p, S, st):
            S.vcycle(dus[p], dfs[p], stream=st)
            st.synchronize()

        res = _drive(solvers, fn)
        assert all(kind == "ok" for kind, _ in res), res
        got = np.concatenate([S.to_numpy(du) for S, du in zip(solvers, dus)], axis=0)
        assert np.array_equal(got, ref) != corrupt
        for S in solvers:
            S.close()
        group.close()


def test_fault_inject_validation():
    import paper_1406_5369_b200 as mgb
    S = mgb.Solver(3, 33)
    with pytest.raises(mgb.MGError) as ei:
        S.fault_inject(mgb.FAULT_COMM_ERROR, 1)  # single rank: nothing to inject into
    assert ei.value.status == 1
    S.close()
    group, solvers = _ranks(2)
    with pytest.raises(mgb.MGError):
        solvers[0].fault_inject(7, 1)
    with pytest.raises(mgb.MGError):
        solvers[0].fault_inject(mgb.FAULT_COMM_ERROR, 0)
    solvers[0].fault_inject(mgb.FAULT_NONE, 0)
    for S in solvers:
        S.close()
    group.close()
