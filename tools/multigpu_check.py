"""Multi-GPU correctness check of the NCCL slab path (run under torchrun on >= 2 GPUs):
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/multigpu_check.py
Each rank runs the z-slab-decomposed V-cycle; rank 0 gathers the owned planes and
compares them with the single-domain CPU oracle bit for bit (FP64), in graph and
eager modes, and checks the residual norms."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as orc  # noqa: E402
import paper_1406_5369_b200 as mgb  # noqa: E402
from paper_1406_5369_b200 import workloads as wl  # noqa: E402


def run(dim, nodes, sm, flags):
    rank, world = dist.get_rank(), dist.get_world_size()
    cells = (nodes - 1,) * dim
    S = mgb.distributed_solver(dim, nodes, smoother=sm, flags=flags)
    u, f = wl.workload("W1", dim, cells, seed=42)
    du, df = S.from_numpy(u), S.from_numpy(f)
    O = orc.Oracle(orc.Config(dim=dim, cells=cells, levels=S.levels,
                              smoother=orc.RBGS if sm == "rbgs" else orc.JACOBI,
                              omega=1.0 if sm == "rbgs" else 0.8)) if rank == 0 else None
    ok = True
    for k in range(3):
        S.vcycle(du, df)
        nrm = S.residual_norm(du, df)
        got = [None] * world
        dist.all_gather_object(got, (S.first_plane, S.to_numpy(du)))
        if rank == 0:
            u = O.vcycle(u, f)
            full = np.zeros_like(u)
            for a, arr in got:
                full[a: a + arr.shape[0]] = arr
            same = np.array_equal(full, u)
            rel = abs(nrm / O.norm(0, u, f) - 1)
            print(f"{dim}D {nodes} {sm} flags={flags} cycle {k}: bitwise={same} norm_rel={rel:.1e}", flush=True)
            ok = ok and same and rel < 1e-12
    return ok


def run_solve(dim, nodes, sm):
    """mg_solve over NCCL (host loop: NCCL cannot run in a conditional graph body) to 1e-10:
    the cycle count and the norm history against the oracle."""
    rank = dist.get_rank()
    cells = (nodes - 1,) * dim
    S = mgb.distributed_solver(dim, nodes, smoother=sm)
    u, f = wl.workload("W1", dim, cells, seed=42)
    du, df = S.from_numpy(u), S.from_numpy(f)
    k, hist = S.solve(du, df, 1e-10, 30)
    ok = True
    if rank == 0:
        O = orc.Oracle(orc.Config(dim=dim, cells=cells, levels=S.levels,
                                  smoother=orc.RBGS if sm == "rbgs" else orc.JACOBI,
                                  omega=1.0 if sm == "rbgs" else 0.8))
        _, k_or, hist_or = O.solve(u, f, 1e-10, 30)
        rel = max(abs(a / b - 1) for a, b in zip(hist, hist_or))
        ok = k == k_or and rel < 1e-12
        print(f"{dim}D {nodes} {sm} solve: cycles {k} (oracle {k_or}) hist_rel={rel:.1e}", flush=True)
    S.close()
    return ok


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ok = True
    for dim, nodes, sm in [(3, 129, "rbgs"), (3, 257, "rbgs"), (2, 1025, "jacobi")]:
        for flags in (0, mgb.FLAG_NO_GRAPH):
            ok = run(dim, nodes, sm, flags) and ok
    ok = run_solve(3, 257, "rbgs") and ok
    if dist.get_rank() == 0:
        print("MULTIGPU_CHECK", "PASS" if ok else "FAIL", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
