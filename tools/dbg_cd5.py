"""Debug helper: complex-diffusion residual norm on raw cudaMalloc buffers (exact size)."""
import ctypes
import glob
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1406_5369_b200 as mgb
from paper_1406_5369_b200 import workloads as wl

rt = ctypes.CDLL(glob.glob("/usr/local/cuda/lib64/libcudart.so*")[0])
n = int(sys.argv[1])
S = mgb.Solver(2, (n, n), smoother="jacobi", omega=0.8, dtype="f32", problem="complex_diffusion", flags=1)
u, f = wl.cd_workload(2, (n, n), 42, S.np_dtype)
du, df = S.from_numpy(u), S.from_numpy(f)
nbytes = du.numel() * du.element_size()
pu, pf = ctypes.c_void_p(), ctypes.c_void_p()
print("malloc", rt.cudaMalloc(ctypes.byref(pu), ctypes.c_size_t(nbytes)), rt.cudaMalloc(ctypes.byref(pf), ctypes.c_size_t(nbytes)))
hu, hf = du.cpu().numpy(), df.cpu().numpy()
print("copy", rt.cudaMemcpy(pu, hu.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(nbytes), 1),
      rt.cudaMemcpy(pf, hf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(nbytes), 1))
out = ctypes.c_double()
st = S.lib.mg_residual_norm(S.h, pu, pf, ctypes.byref(out), None)
print("raw buffers:", st, out.value if st == 0 else S.lib.mg_error_string(S.h).decode(), flush=True)
