"""Debug helper: residual norm of complex diffusion with exact-size allocations."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1406_5369_b200 as mgb
from paper_1406_5369_b200 import workloads as wl

for n in (64, 128, 256, 512):
    for dt in ("f32", "f64"):
        S = mgb.Solver(2, (n, n), smoother="jacobi", omega=0.8, dtype=dt, problem="complex_diffusion", flags=1)
        u, f = wl.cd_workload(2, (n, n), 42, S.np_dtype)
        du, df = S.from_numpy(u), S.from_numpy(f)
        try:
            print(n, dt, S.residual_norm(du, df), flush=True)
        except Exception as e:
            print(n, dt, "FAIL", e, flush=True)
            sys.exit(1)
