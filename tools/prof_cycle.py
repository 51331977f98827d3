"""Run a few V-cycles of a bench config (for ncu captures): python tools/prof_cycle.py [config] [cycles]"""
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_1406_5369_b200 as mgb

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3-f64"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dim, nodes, sm, nu1, nu2, dt, levels, omega = bench.CONFIGS[cfg]
S = mgb.Solver(dim, nodes, levels=levels, smoother=sm, omega=omega, nu1=nu1, nu2=nu2, dtype=dt,
               flags=mgb.FLAG_HOST_LOOP)
u, f = S.empty(), S.empty()
S.workload_fill(u, 42)
for _ in range(n):
    S.vcycle(u, f)
    r = S.residual_norm(u, f)
torch.cuda.synchronize()
print("ok", cfg, r)
