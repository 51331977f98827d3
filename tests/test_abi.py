"""Host-side checks of the C-ABI library (CPU only, no compute calls):
it loads, exports every symbol include/mg.h declares, validates configs, and
fails loudly (no CPU fallback) when there is no GPU."""
import ctypes
import os
import re

import pytest

import paper_1406_5369_b200 as mgb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "mg.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mg_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = mgb.load_library()
    syms = header_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(lib, name), name
    assert sorted(mgb.ABI_SYMBOLS) == syms


def test_library_is_sm100a_only():
    """The library carries sm_100a SASS (no PTX-JIT / other-arch fallback)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", mgb.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def _create(**kw):
    lib = mgb.load_library()
    c = mgb.MGConfig()
    lib.mg_config_default(ctypes.byref(c), kw.pop("dim", 3), kw.pop("nodes", 17))
    for k, v in kw.items():
        if k == "nodes3":
            for d in range(3):
                c.nodes[d] = v[d]
        else:
            setattr(c, k, v)
    h = ctypes.c_void_p()
    st = lib.mg_create(ctypes.byref(c), ctypes.byref(h))
    return st, h, lib.mg_error_string(None).decode()


def test_config_defaults():
    lib = mgb.load_library()
    c = mgb.MGConfig()
    lib.mg_config_default(ctypes.byref(c), 3, 513)
    assert (c.dim, list(c.nodes), c.levels, c.smoother, c.omega, c.nu1, c.nu2, c.coarse, c.ncoarse) == \
        (3, [513, 513, 513], 0, mgb.RBGS, 1.0, 2, 2, mgb.COARSE_DIRECT, 10)
    assert (c.problem, c.tau, c.kappa) == (mgb.PROBLEM_POISSON, 0.1, 2.0) and abs(c.theta - 3.141592653589793 / 30) < 1e-16


def test_complex_diffusion_config_valid_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    st, h, msg = _create(problem=1, nodes=16, coarse=1)
    assert st == 4 and "no CPU fallback" in msg


@pytest.mark.parametrize("kw,status", [
    (dict(dim=4), 1),
    (dict(omega=2.0), 1),
    (dict(omega=0.0), 1),
    (dict(nu1=-1), 1),
    (dict(smoother=7), 1),
    (dict(dtype=5), 1),
    (dict(nodes=18), 2),                          # 17 cells: not coarsenable
    (dict(nodes=17, levels=6), 2),                # 16 cells, 6 levels -> coarsest has 0 interior nodes
    (dict(nodes3=(17, 33, 10)), 2),               # 9 cells along z
    # complex diffusion (problem 1): nodes are cells; FAS needs SWEEPS; one rank; Eq. 3 parameters
    (dict(problem=1, nodes=16), 1),               # coarse = DIRECT (the default) is rejected
    (dict(problem=1, nodes=16, coarse=1, nranks=2), 1),
    (dict(problem=1, nodes=16, coarse=1, theta=2.0), 1),
    (dict(problem=1, nodes=16, coarse=1, tau=0.0), 1),
    (dict(problem=1, nodes=16, coarse=1, kappa=-1.0), 1),
    (dict(problem=1, nodes3=(16, 16, 12), coarse=1, levels=4), 2),  # 12 cells not divisible by 8
    (dict(problem=2), 1),
    (dict(smoother=2, nranks=2), 1),              # lexicographic GS is sequential: one rank only
    (dict(problem=1, nodes=16, coarse=1, smoother=2), 1),  # ... and Poisson only
])
def test_create_rejects_bad_config(kw, status):
    st, h, msg = _create(**kw)
    assert st == status, (st, msg)
    assert not h.value
    assert msg


def test_create_without_gpu_fails_loudly():
    """No CPU fallback: a valid config on a GPU-less host is MG_ERR_CUDA."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    st, h, msg = _create(nodes=17)
    assert st == 4 and "no CPU fallback" in msg
