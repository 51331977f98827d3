"""Debug helper: mg_vcycle_host on complex diffusion at several sizes."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1406_5369_b200 as mgb
from paper_1406_5369_b200 import workloads as wl

for n in [int(a) for a in sys.argv[1:]] or [64, 512, 4096]:
    S = mgb.Solver(2, (n, n), smoother="jacobi", omega=0.8, dtype="f32", problem="complex_diffusion")
    u, f = wl.cd_workload(2, (n, n), 42, np.complex64)
    du, df = S.from_numpy(u), S.from_numpy(f)
    hu = du.cpu().pin_memory()
    hf = df.cpu().pin_memory()
    print(n, "shape", S.shape, hu.shape, hu.dtype, hu.is_contiguous(), flush=True)
    try:
        r = S.vcycle_host(hu, hf, 1)
        print(n, "vcycle_host ok", r, flush=True)
    except Exception as e:
        print(n, "FAIL", e, flush=True)
        break
