"""Time one level-0 sweep / resid-restrict / norm of a bench config for several z-chunk sizes."""
import os
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_1406_5369_b200 as mgb

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3-f64"
dim, nodes, sm, nu1, nu2, dt, levels, omega = bench.CONFIGS[cfg]
S = mgb.Solver(dim, nodes, levels=levels, smoother=sm, omega=omega, nu1=nu1, nu2=nu2, dtype=dt, flags=mgb.FLAG_NO_GRAPH)
u, f, o = S.empty(), S.empty(), S.empty()
S.workload_fill(u, 42)
S.workload_fill(f, 7, -1, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for zc in [0, 16, 24, 32, 40, 48, 57, 64, 73, 86, 103, 128, 171, 256, 511]:
    os.environ["MG_ZC"] = str(zc)
    S.op_smooth(0, u, f, o)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        S.op_smooth(0, u, f, o)
    e1.record()
    torch.cuda.synchronize()
    print(f"zc={zc:4d} op_smooth(L0) {e0.elapsed_time(e1) / 10:.4f} ms", flush=True)
