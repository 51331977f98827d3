"""Drive every kernel family of libmgb200 on small grids, checking the memory the library may touch.

    [MG_LIBRARY=paper_1406_5369_b200/libmgb200_checked.so] python tools/sanitize.py [case ...]

The SURVEY §4 T4 tier.  compute-sanitizer is closed on this pool, so this runs
the CHECKED build (csrc/checked.h: guard bands around every library-owned buffer, bounded
mbarrier waits) with CUDA_LAUNCH_BLOCKING=1 (tests/test_gpu_checked.py), and works under
compute-sanitizer too where it is available (tools/round.sh `sanitize`).  Per case:
  - the caller's u and f live inside larger buffers whose guard regions and x-padding elements
    hold a sentinel: after the case they must be unchanged (the ABI: the library never writes
    padding, nor outside the arrays; in slab mode the halo planes are library scratch);
  - every level kernel runs eagerly (FLAG_NO_GRAPH | FLAG_HOST_LOOP) with pm_min_nx lowered so
    the TMA plane-marching kernels run on 33^3 .. 129^3 grids; the coarse levels run the
    cluster tail kernel; then the per-operation entry points;
  - one JSON line: a digest of the results (compared between the checked and the product
    build: the guards must not change a single bit) and the guard verdicts; with the checked
    build also mg_checked_guard_failures() (the library's own buffers).
"""
import ctypes
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1406_5369_b200 as mgb  # noqa: E402
from paper_1406_5369_b200 import workloads as wl  # noqa: E402

EAGER = mgb.FLAG_NO_GRAPH | mgb.FLAG_HOST_LOOP
GUARD = 4096  # elements of sentinel before and after each caller array
SENT = {torch.float64: 7.25, torch.float32: 7.25, torch.complex128: 7.25 + 3j, torch.complex64: 7.25 + 3j}


class Guarded:
    """A caller array of S's level-0 layout inside a sentinel-filled buffer."""

    def __init__(self, S, a, slab_halo=False):
        P, R, X = S.level_shape(0)
        n = P * R * X
        self.dtype = S.torch_dtype
        self.buf = torch.full((n + 2 * GUARD,), SENT[self.dtype], dtype=self.dtype, device="cuda")
        self.t = self.buf[GUARD: GUARD + n].view(P, R, X)
        dense = S.from_numpy(a)  # padded layout with zero padding
        nxv = S.level_cells(0)[0] + (0 if S.complex else 1)
        self.nxv = nxv
        self.t[:, :, :nxv].copy_(dense[:, :, :nxv])  # the padding keeps the sentinel
        self.slab_halo = slab_halo

    def ok(self):
        s = SENT[self.dtype]
        g = torch.cat([self.buf[:GUARD], self.buf[-GUARD:]])
        pad = self.t[:, :, self.nxv:]
        return bool((g == s).all()) and bool((pad == s).all())


def digest(*arrays):
    h = hashlib.sha1()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def poisson(dim, n, smoother, dtype, flags=0, nu=(2, 2), pm_min_nx=16, cycles=2):
    S = mgb.Solver(dim, n, smoother=smoother, dtype=dtype, nu1=nu[0], nu2=nu[1], flags=EAGER | flags,
                   pm_min_nx=pm_min_nx)
    npdt = np.float64 if dtype == "f64" else np.float32
    cells = (n - 1,) * dim
    u, f = wl.workload("W4", dim, cells, seed=7, dtype=npdt)
    gu, gf = Guarded(S, u), Guarded(S, f)
    du, df = gu.t, gf.t
    k, hist = S.solve(du, df, 0.0, cycles)
    S.vcycle(du, df)
    r = S.residual_norm(du, df)
    t, rr = S.empty(0), S.empty(0)
    S.op_smooth(0, du, df, t)
    S.op_residual(0, du, df, rr)
    fc = S.empty(1)
    S.op_restrict(0, rr, fc)
    S.op_prolong_correct(0, fc, du)
    nrm = S.op_norm(0, du, df)
    torch.cuda.synchronize()
    out = dict(digest=digest(S.to_numpy(du), S.to_numpy(t), S.to_numpy(rr), S.to_numpy(fc, 1), np.array(hist + [r, nrm])),
               caller_guards_ok=gu.ok() and gf.ok())
    S.close()
    return out


def complex_diffusion(dim, n, smoother, dtype):
    S = mgb.Solver(dim, n, smoother=smoother, omega=0.8 if smoother == "jacobi" else 1.0, dtype=dtype,
                   problem="complex_diffusion", flags=EAGER, pm_min_nx=16)
    npdt = np.complex128 if dtype == "f64" else np.complex64
    u, f = wl.cd_workload(dim, (n,) * dim, 42, npdt)
    gu, gf = Guarded(S, u), Guarded(S, f)
    k, hist = S.solve(gu.t, gf.t, 0.0, 2)
    torch.cuda.synchronize()
    out = dict(digest=digest(S.to_numpy(gu.t), np.array(hist)), caller_guards_ok=gu.ok() and gf.ok())
    S.close()
    return out


CASES = {
    "p3_33_rbgs_f64": lambda: poisson(3, 33, "rbgs", "f64"),
    "p3_65_rbgs_f64": lambda: poisson(3, 65, "rbgs", "f64"),
    "p3_65_rbgs_f32": lambda: poisson(3, 65, "rbgs", "f32"),
    "p3_65_jac_f64": lambda: poisson(3, 65, "jacobi", "f64"),
    "p3_129_rbgs_f64": lambda: poisson(3, 129, "rbgs", "f64", pm_min_nx=64),
    "p3_129_rbgs_f32": lambda: poisson(3, 129, "rbgs", "f32", pm_min_nx=64),
    "p3_97_rbgs_f64_ragged": lambda: poisson(3, 97, "rbgs", "f64"),
    "p3_65_separate_prolong_f64": lambda: poisson(3, 65, "rbgs", "f64", flags=mgb.FLAG_SEPARATE_PROLONG),
    "p3_65_baseline_f64": lambda: poisson(3, 65, "rbgs", "f64", flags=mgb.FLAG_BASELINE),
    "p3_33_lex_f64": lambda: poisson(3, 33, "gs_lex", "f64"),
    "p2_257_jac33_f32": lambda: poisson(2, 257, "jacobi", "f32", nu=(3, 3)),
    "p2_257_jac33_f64": lambda: poisson(2, 257, "jacobi", "f64", nu=(3, 3)),
    "p2_257_rbgs_f64": lambda: poisson(2, 257, "rbgs", "f64"),
    "p2_65_jac_f64": lambda: poisson(2, 65, "jacobi", "f64"),
    "cd2_128_jac_f32": lambda: complex_diffusion(2, 128, "jacobi", "f32"),
    "cd2_128_rbgs_f64": lambda: complex_diffusion(2, 128, "rbgs", "f64"),
    "cd3_64_jac_f32": lambda: complex_diffusion(3, 64, "jacobi", "f32"),
}


def main(argv):
    names = argv or list(CASES)
    torch.cuda.set_device(0)
    lib = mgb.load_library()
    checked = hasattr(lib, "mg_checked_guard_failures")
    if checked:
        lib.mg_checked_guard_failures.restype = ctypes.c_longlong
    for name in names:
        rec = dict(case=name, **CASES[name]())
        if checked:
            rec["library_guard_failures"] = int(lib.mg_checked_guard_failures())
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
