"""Debug helper: bisect mg_vcycle_host on complex diffusion (eager launches)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1406_5369_b200 as mgb
from paper_1406_5369_b200 import workloads as wl

n = int(sys.argv[1])
flags = int(sys.argv[2])
S = mgb.Solver(2, (n, n), smoother="jacobi", omega=0.8, dtype="f32", problem="complex_diffusion", flags=flags)
u, f = wl.cd_workload(2, (n, n), 42, np.complex64)
du, df = S.from_numpy(u), S.from_numpy(f)
hu = du.cpu().pin_memory()
hf = df.cpu().pin_memory()
for nc in (0, 1):
    for norm in (False, True):
        try:
            out = mgb.ctypes.c_double()
            st = S.lib.mg_vcycle_host(S.h, mgb.ctypes.c_void_p(hu.data_ptr()), mgb.ctypes.c_void_p(hf.data_ptr()), nc,
                                      mgb.ctypes.byref(out) if norm else None, S._stream(None))
            print("ncycles", nc, "norm", norm, "status", st, S.lib.mg_error_string(S.h).decode() if st else out.value,
                  flush=True)
            if st:
                sys.exit(1)
        except Exception as e:
            print("EXC", e)
            sys.exit(1)
