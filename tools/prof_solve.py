"""Run mg_solve with the host loop, eager launches (ncu cannot profile kernels inside conditional graphs):
python tools/prof_solve.py [config] [cycles] [separate-prolong] [device] — the same kernels as the bench's
timed steps; `device`: the device-side loop without graphs (a whole-cycle tail grid's one-launch solve)."""
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_1406_5369_b200 as mgb

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dim, nodes, sm, nu1, nu2, dt, levels, omega = bench.CONFIGS[cfg]
S = mgb.Solver(dim, nodes, levels=levels, smoother=sm, omega=omega, nu1=nu1, nu2=nu2, dtype=dt,
               flags=(0 if "device" in sys.argv[3:] else mgb.FLAG_HOST_LOOP) | mgb.FLAG_NO_GRAPH | (mgb.FLAG_SEPARATE_PROLONG if "separate-prolong" in sys.argv[3:] else 0))
u, f = S.empty(), S.empty()
S.workload_fill(u, 42)
k, hist = S.solve(u, f, 0.0, n)
torch.cuda.synchronize()
print("ok", cfg, k, hist[-1])
