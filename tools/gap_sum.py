"""Step time (graph, device loop) vs the summed per-kernel CUDA-event time of the same cycles."""
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_1406_5369_b200 as mgb

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3-f64"
dim, nodes, sm, nu1, nu2, dt, levels, omega = bench.CONFIGS[cfg]
S = mgb.Solver(dim, nodes, levels=levels, smoother=sm, omega=omega, nu1=nu1, nu2=nu2, dtype=dt)
u, f = S.empty(), S.empty()
S.workload_fill(u, 42)
S.solve(u, f, -1.0, 5)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 30
e0.record()
S.solve(u, f, -1.0, K)
e1.record()
torch.cuda.synchronize()
graph = e0.elapsed_time(e1) / K
S.profile_enable(True)
S.solve(u, f, -1.0, K)
recs = S.profile_read()
S.profile_enable(False)
ksum = sum(r["ms"] for r in recs) / K
print(cfg, f"graph step {graph:.4f} ms, summed kernel events {ksum:.4f} ms, launches/step {sum(r['count'] for r in recs)/K:.1f}")
