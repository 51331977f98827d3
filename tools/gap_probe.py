"""Sum of per-kernel device time (instrumented eager pass) vs the graph-timed step: the
difference bounds what launch gaps cost (what programmatic dependent launch could hide)."""
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_1406_5369_b200 as mgb

for cfg in sys.argv[1:]:
    dim, nodes, sm, nu1, nu2, dt, levels, omega = bench.CONFIGS[cfg]
    S = mgb.Solver(dim, nodes, levels=levels, smoother=sm, omega=omega, nu1=nu1, nu2=nu2, dtype=dt)
    u, f = S.empty(), S.empty()
    S.workload_fill(u, 42)
    st = torch.cuda.Stream()
    S.solve(u, f, 0.0, 5, stream=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    S.solve(u, f, 0.0, 20, stream=st)
    e1.record(st)
    torch.cuda.synchronize()
    step = e0.elapsed_time(e1) / 20
    S.profile_enable(True)
    S.solve(u, f, 0.0, 10, stream=st)
    recs = S.profile_read()
    S.profile_enable(False)
    ktot = sum(r["ms"] for r in recs) / 10
    n = sum(r["count"] for r in recs) / 10
    print(f"{cfg}: step {step:.4f} ms, kernels {ktot:.4f} ms, {n:.1f} launches, gap {step - ktot:.4f} ms "
          f"({(step - ktot) / max(n, 1) * 1e3:.2f} us/launch)")
