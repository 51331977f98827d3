"""Debug helper: complex-diffusion vcycle parity at growing sizes, graph and eager."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1406_5369_b200 as mgb
from paper_1406_5369_b200 import workloads as wl
from oracle.cd import CDConfig, CDOracle

sm = sys.argv[1]
for n in [int(a) for a in sys.argv[2:]]:
    for flags in (mgb.FLAG_NO_GRAPH, 0):
        S = mgb.Solver(2, (n, n), smoother=sm, omega=0.8 if sm == "jacobi" else 1.0, dtype="f32",
                       problem="complex_diffusion", flags=flags)
        u, f = wl.cd_workload(2, (n, n), 42, np.complex64)
        du, df = S.from_numpy(u), S.from_numpy(f)
        try:
            S.vcycle(du, df)
            torch.cuda.synchronize()
            O = CDOracle(CDConfig(dim=2, cells=(n, n), smoother=0 if sm == "jacobi" else 1,
                                  omega=0.8 if sm == "jacobi" else 1.0), np.complex64)
            ok = np.array_equal(S.to_numpy(du), O.cycle(u, f))
            print(n, "flags", flags, "ok" if ok else "MISMATCH", flush=True)
        except Exception as e:
            print(n, "flags", flags, "FAIL", e, flush=True)
            sys.exit(1)
