"""World-size-2 gloo tests of the multi-GPU (slab) path's host logic on CPU:
libmgb200's partition (mg_partition, no GPU needed), and the schedule of halo
exchanges / agglomeration / deterministic norm that Exec implements with NCCL,
emulated by tests/slab_emulator.py.  The gathered iterate after each V-cycle
must equal the single-domain oracle's BIT FOR BIT."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as orc
import paper_1406_5369_b200 as mgb
from paper_1406_5369_b200 import workloads as wl


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    from slab_emulator import SlabMG
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        dim, nodes, sm, omega, nu1, nu2, levels, wk = case
        cells = (nodes - 1,) * dim
        u, f = wl.workload(wk, dim, cells, seed=42 if wk == "W1" else 5)
        if dim == 2:
            u, f = u[:, None, :], f[:, None, :]
        E = SlabMG(dim, nodes, sm, omega, nu1, nu2, levels, rank, world)
        U, F = E.from_global(0, u), E.from_global(0, f)
        lo, hi = E.owned_local(0)
        first = E.part[0][0]
        owned_sets, norms = [], []
        for _ in range(2):
            U = E.vcycle(U, F)
            mine = (first, U[E.H: E.H + E.part[0][1]].copy())
            got = [None] * world
            dist.all_gather_object(got, mine)
            owned_sets.append(got)
            norms.append(E.norm(U, F))
        if rank == 0:
            np.save(os.path.join(outdir, "norms.npy"), np.array(norms))
            for c, got in enumerate(owned_sets):
                full = np.zeros_like(u)
                for a, arr in got:
                    full[a: a + arr.shape[0]] = arr
                np.save(os.path.join(outdir, f"u{c}.npy"), full)
        del torch
    finally:
        dist.destroy_process_group()


CASES = [
    (3, 33, "rbgs", 1.0, 2, 2, 0, "W1"),
    (3, 33, "jacobi", 0.8, 2, 1, 0, "W4"),
    (2, 65, "jacobi", 0.8, 2, 2, 5, "W1"),    # C1 layout (2D: plane axis = y)
    (2, 129, "rbgs", 1.0, 1, 1, 0, "W4"),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}D-{c[1]}-{c[2]}-V{c[4]}{c[5]}")
def test_slab_schedule_world2_matches_oracle(case, tmp_path):
    dim, nodes, sm, omega, nu1, nu2, levels, wk = case
    cells = (nodes - 1,) * dim
    L = levels or orc.Config(dim=dim, cells=cells).resolved_levels()
    case = (dim, nodes, sm, omega, nu1, nu2, L, wk)
    # the partition the library would use: 2 ranks, nested slabs, agglomeration below 8 planes/rank
    parts = [mgb.partition(l, dim=dim, nodes=nodes, levels=L, nranks=2, rank=1) for l in range(L)]
    assert parts[0][2] and not parts[-1][2]
    mp.spawn(_worker, args=(2, _free_port(), case, str(tmp_path)), nprocs=2, join=True)
    O = orc.Oracle(orc.Config(dim=dim, cells=cells, levels=L, smoother=orc.RBGS if sm == "rbgs" else orc.JACOBI,
                              omega=omega, nu1=nu1, nu2=nu2))
    u, f = wl.workload(wk, dim, cells, seed=42 if wk == "W1" else 5)
    norms = np.load(tmp_path / "norms.npy")
    for c in range(2):
        u = O.vcycle(u, f)
        got = np.load(tmp_path / f"u{c}.npy")
        got = got[:, 0, :] if dim == 2 else got
        assert np.array_equal(got, u), (c, np.abs(got - u).max())
        assert abs(norms[c] / O.norm(0, u, f) - 1) < 1e-12


def test_partition_rules():
    """Nesting, ownership and agglomeration rules of mg_partition (host only)."""
    for dim, nodes, P in [(3, 513, 2), (3, 513, 8), (3, 1025, 8), (2, 8193, 8), (3, 257, 4)]:
        L = orc.Config(dim=dim, cells=(nodes - 1,) * dim).resolved_levels()
        for rank in range(P):
            prev = None
            for l in range(L):
                first, owned, distd, halo = mgb.partition(l, dim=dim, nodes=nodes, nranks=P, rank=rank)
                n = (nodes - 1) >> l
                if distd:
                    assert halo == 2
                    assert first == rank * (n // P)
                    assert owned == n // P + (1 if rank == P - 1 else 0)
                    assert (n // P) >= 8 and (n // P) % 2 == 0
                    if prev is not None:
                        assert first * 2 == prev  # nested slabs
                    prev = first
                else:
                    assert (first, owned, halo) == (0, n + 1, 0)
        # ranks tile the finest level exactly
        tot = sum(mgb.partition(0, dim=dim, nodes=nodes, nranks=P, rank=r)[1] for r in range(P))
        assert tot == nodes
    with pytest.raises(mgb.MGError):
        mgb.partition(0, dim=3, nodes=17, nranks=4, rank=0)  # 16/4 = 4 planes per rank: too thin
