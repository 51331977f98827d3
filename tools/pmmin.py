"""C2 step time (solve loop on the device) for several pm_min_nx thresholds."""
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_1406_5369_b200 as mgb

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
dim, nodes, sm, nu1, nu2, dt, levels, omega = bench.CONFIGS[cfg]
for pmn in (128, 64, 32, 16):
    S = mgb.Solver(dim, nodes, levels=levels, smoother=sm, omega=omega, nu1=nu1, nu2=nu2, dtype=dt, pm_min_nx=pmn)
    u, f = S.empty(), S.empty()
    S.workload_fill(u, 42)
    S.solve(u, f, 0.0, 5)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    k_done = None
    for _ in range(5):
        S.workload_fill(u, 42)  # fresh start: 50 cycles of W1 stay far from underflow
        torch.cuda.synchronize()
        e0.record()
        k_done, _ = S.solve(u, f, 0.0, 50)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 50)
    print(cfg, "pm_min_nx", pmn, "ms/cycle", round(best, 4), "cycles", k_done, "launches/cycle", S.launches_per_cycle)
