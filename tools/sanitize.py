"""Drive every kernel family of libmgb200.so on small grids, for compute-sanitizer.

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize.py [case ...]

Cases run eagerly (FLAG_NO_GRAPH | FLAG_HOST_LOOP, so every kernel is a plain launch) with
pm_min_nx lowered so the TMA plane-marching kernels run on 33^3 .. 129^3 grids; the levels below
the tail threshold run the cluster tail kernel.  Product path only (no oracle): the sanitizer's
report is the result.  Prints one line per case.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1406_5369_b200 as mgb  # noqa: E402
from paper_1406_5369_b200 import workloads as wl  # noqa: E402

EAGER = mgb.FLAG_NO_GRAPH | mgb.FLAG_HOST_LOOP


def poisson(dim, n, smoother, dtype, flags=0, nu=(2, 2), pm_min_nx=16, cycles=2):
    S = mgb.Solver(dim, n, smoother=smoother, dtype=dtype, nu1=nu[0], nu2=nu[1], flags=EAGER | flags,
                   pm_min_nx=pm_min_nx)
    npdt = np.float64 if dtype == "f64" else np.float32
    cells = (n - 1,) * dim
    u, f = wl.workload("W4", dim, cells, seed=7, dtype=npdt)
    du, df = S.from_numpy(u), S.from_numpy(f)
    k, hist = S.solve(du, df, 0.0, cycles)
    S.vcycle(du, df)
    r = S.residual_norm(du, df)
    # per-op entry points at level 0 and 1
    t, rr = S.empty(0), S.empty(0)
    S.op_smooth(0, du, df, t)
    S.op_residual(0, du, df, rr)
    fc = S.empty(1)
    S.op_restrict(0, rr, fc)
    S.op_prolong_correct(0, fc, du)
    S.op_norm(0, du, df)
    torch.cuda.synchronize()
    S.close()
    return f"k={k} r={r:.3e}"


def complex_diffusion(dim, n, smoother, dtype):
    S = mgb.Solver(dim, n, smoother=smoother, omega=0.8 if smoother == "jacobi" else 1.0, dtype=dtype,
                   problem="complex_diffusion", flags=EAGER, pm_min_nx=16)
    npdt = np.complex128 if dtype == "f64" else np.complex64
    u, f = wl.cd_workload(dim, (n,) * dim, 42, npdt)
    du, df = S.from_numpy(u), S.from_numpy(f)
    k, hist = S.solve(du, df, 0.0, 2)
    torch.cuda.synchronize()
    S.close()
    return f"k={k} r={hist[-1]:.3e}"


CASES = {
    "p3_33_rbgs_f64": lambda: poisson(3, 33, "rbgs", "f64"),
    "p3_65_rbgs_f64": lambda: poisson(3, 65, "rbgs", "f64"),
    "p3_65_rbgs_f32": lambda: poisson(3, 65, "rbgs", "f32"),
    "p3_65_jac_f64": lambda: poisson(3, 65, "jacobi", "f64"),
    "p3_129_rbgs_f64": lambda: poisson(3, 129, "rbgs", "f64", pm_min_nx=64),
    "p3_129_rbgs_f32": lambda: poisson(3, 129, "rbgs", "f32", pm_min_nx=64),
    "p3_65_fuseprolong_f64": lambda: poisson(3, 65, "rbgs", "f64", flags=mgb.FLAG_FUSE_PROLONG),
    "p3_65_slab_f64": lambda: poisson(3, 65, "rbgs", "f64", flags=mgb.FLAG_SLAB),
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
    for name in names:
        print(f"{name}: {CASES[name]()}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
