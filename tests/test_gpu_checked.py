"""SURVEY §4 tier T4 (memory and race checks).  compute-sanitizer is closed on this pool (runs
under it left GPUs needing a reset), so:
  - tools/sanitize.py drives every kernel family on small grids with the caller's arrays inside
    sentinel-guarded buffers, once through the product library and once through the CHECKED
    build (libmgb200_checked.so: guard bands around every library-owned buffer, bounded mbarrier
    waits that trap instead of hanging) with CUDA_LAUNCH_BLOCKING=1: no CUDA error, no guard or
    padding element written, the library's own guard bands intact, and bit-identical results in
    both builds;
  - races: a race-free kernel is deterministic, so full-size runs repeated in fresh solvers
    must agree bit for bit (besides every parity test's bitwise comparison with the oracle)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_1406_5369_b200", "libmgb200_checked.so")


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return {d["case"]: d for d in (json.loads(l) for l in r.stdout.splitlines() if l.startswith("{"))}


def test_checked_build_guards_and_identical_results():
    assert os.path.exists(CHECKED), "build the checked library: make checked (__graft_entry__.build())"
    prod = _run({})
    chk = _run({"MG_LIBRARY": CHECKED, "CUDA_LAUNCH_BLOCKING": "1"})
    assert set(prod) == set(chk) and len(prod) >= 15
    for name, d in chk.items():
        assert d["caller_guards_ok"], (name, "the library wrote outside the caller's arrays or into padding")
        assert d["library_guard_failures"] == 0, (name, "a kernel wrote outside a library-owned buffer")
        assert prod[name]["caller_guards_ok"], name
        assert d["digest"] == prod[name]["digest"], (name, "checked and product builds differ")


@pytest.mark.parametrize("cfg", [(3, 513, "rbgs", "f64"), (3, 513, "rbgs", "f32"), (2, 8193, "jacobi", "f32")],
                         ids=lambda c: f"{c[0]}d-{c[1]}-{c[2]}-{c[3]}")
def test_run_to_run_bitwise(cfg):
    """Determinism at full size (bench configs C3 FP64/FP32, C4): two fresh solvers, the same
    input, three cycles through the device loop -> identical iterates and norms."""
    import torch

    import paper_1406_5369_b200 as mgb
    dim, n, sm, dt = cfg
    outs = []
    for _ in range(2):
        S = mgb.Solver(dim, n, smoother=sm, dtype=dt, nu1=3 if dim == 2 else 2, nu2=3 if dim == 2 else 2)
        u, f = S.empty(), S.empty()
        S.workload_fill(u, 42)
        S.workload_fill(f, 7, -1.0, 1.0)
        k, hist = S.solve(u, f, -1.0, 3)
        torch.cuda.synchronize()
        outs.append((u.clone(), hist))
        S.close()
        del u, f
    assert torch.equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1]
