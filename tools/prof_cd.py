"""Run a few complex-diffusion FAS cycles of a bench config (for ncu captures)."""
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_1406_5369_b200 as mgb

cfg = sys.argv[1] if len(sys.argv) > 1 else "CD2-f32"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dim, cells, sm, nu1, nu2, dt, omega = bench.CD_CONFIGS[cfg]
S = mgb.Solver(dim, (cells,) * dim, smoother=sm, omega=omega, nu1=nu1, nu2=nu2, dtype=dt,
               problem="complex_diffusion", coarse="sweeps", flags=mgb.FLAG_NO_GRAPH)  # ncu: no conditional graphs
u, f = S.empty(), S.empty()
S.workload_fill(u, 42)
S.workload_fill(f, 42)
k, hist = S.solve(u, f, 0.0, n)
torch.cuda.synchronize()
print("ok", cfg, hist[-1] / hist[0])
