# A/B: solve time per cycle (device loop) for configs with different pm_min_nx
import sys
sys.path.insert(0, ".")
import torch, bench
import paper_1406_5369_b200 as mgb
for spec in sys.argv[1:]:
    cfg, pmn = spec.split(":")
    dim, nodes, sm, nu1, nu2, dt, levels, omega = bench.CONFIGS[cfg]
    S = mgb.Solver(dim, nodes, levels=levels, smoother=sm, omega=omega, nu1=nu1, nu2=nu2, dtype=dt, pm_min_nx=int(pmn))
    u, f = S.empty(), S.empty(); S.workload_fill(u, 42)
    S.solve(u, f, 0.0, 5); torch.cuda.synchronize()
    best = 1e9
    for rep in range(5):
        S.workload_fill(u, 42); torch.cuda.synchronize()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(S.stream if hasattr(S, "stream") else None) if False else a.record()
        k, h = S.solve(u, f, -1.0, 50)
        b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 50)
    print(spec, "ms/cycle %.4f" % best, "cycles", k, "last", h[-1])
    S.close()
