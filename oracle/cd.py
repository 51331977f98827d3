"""ctypes wrapper of the complex-diffusion FAS oracle (oracle/cd_oracle.c).

TEST INFRASTRUCTURE ONLY (same rules as oracle/__init__.py).  Arrays are dense
unpadded complex cell arrays: 2D (ny, nx), 3D (nz, ny, nx); numpy complex128
for the FP64 build, complex64 for the FP32 build.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import lib as _lib

JACOBI, RBGS = 0, 1
# defaults recorded by SPEC: the paper gives no tau, theta, k
TAU, THETA, KAPPA = 0.1, math.pi / 30.0, 2.0


class _CdCfg(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int),
        ("n", ctypes.c_int * 3),
        ("levels", ctypes.c_int),
        ("h", ctypes.c_double * 3),
        ("smoother", ctypes.c_int),
        ("omega", ctypes.c_double),
        ("nu1", ctypes.c_int),
        ("nu2", ctypes.c_int),
        ("ncoarse", ctypes.c_int),
        ("tau", ctypes.c_double),
        ("theta", ctypes.c_double),
        ("kappa", ctypes.c_double),
    ]


@dataclass
class CDConfig:
    """Mirror of cd_config; `cells` per axis of the finest level (the unknowns)."""
    dim: int
    cells: tuple
    levels: int = 0          # 0 => paper rule: coarsest level has 2 cells (< 3 unknowns) per axis
    smoother: int = RBGS
    omega: float = 1.0
    nu1: int = 2
    nu2: int = 2
    ncoarse: int = 10
    tau: float = TAU
    theta: float = THETA
    kappa: float = KAPPA
    h: tuple = field(default=None)

    def resolved_levels(self) -> int:
        if self.levels:
            return self.levels
        return int(min(self.cells[: self.dim])).bit_length() - 1

    def level_cells(self, l: int):
        return tuple(c >> l for c in self.cells[: self.dim])

    def shape(self, l: int = 0):
        return tuple(reversed(self.level_cells(l)))

    def c_struct(self) -> _CdCfg:
        c = _CdCfg()
        c.dim = self.dim
        for d in range(3):
            c.n[d] = int(self.cells[d]) if d < self.dim else 1
            if self.h is None:
                c.h[d] = 1.0 / self.cells[d] if d < self.dim else 0.0
            else:
                c.h[d] = float(self.h[d]) if d < self.dim else 0.0
        c.levels = self.resolved_levels()
        c.smoother, c.omega = self.smoother, self.omega
        c.nu1, c.nu2, c.ncoarse = self.nu1, self.nu2, self.ncoarse
        c.tau, c.theta, c.kappa = self.tau, self.theta, self.kappa
        return c


def _bind(L):
    if getattr(L, "_cd_bound", False):
        return L
    P = ctypes.c_void_p
    C = ctypes.POINTER(_CdCfg)
    L.cd_level_cells.argtypes = [C, ctypes.c_int]
    L.cd_level_cells.restype = ctypes.c_int64
    L.cd_gfield.argtypes = [C, ctypes.c_int, P, P]
    L.cd_apply.argtypes = [C, ctypes.c_int, P, P, P, P]
    L.cd_smooth.argtypes = [C, ctypes.c_int, P, P, P]
    L.cd_restrict.argtypes = [C, ctypes.c_int, P, P]
    L.cd_prolong_add.argtypes = [C, ctypes.c_int, P, P]
    L.cd_norm.argtypes = [C, ctypes.c_int, P, P]
    L.cd_norm.restype = ctypes.c_double
    L.cd_cycle.argtypes = [C, P, P]
    L.cd_cycle.restype = ctypes.c_int
    L.cd_solve.argtypes = [C, P, P, ctypes.c_double, ctypes.c_int, P]
    L.cd_solve.restype = ctypes.c_int
    L._cd_bound = True
    return L


def _ptr(a):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)


class CDOracle:
    """FP64 (complex128) or FP32 (complex64) complex-diffusion FAS oracle."""

    def __init__(self, cfg: CDConfig, dtype=np.complex128):
        self.cfg = cfg
        self.dtype = np.dtype(dtype)
        self.real = np.float64 if self.dtype == np.complex128 else np.float32
        self.lib = _bind(_lib(self.real))
        self._c = cfg.c_struct()

    @property
    def levels(self):
        return self._c.levels

    def shape(self, l=0):
        return self.cfg.shape(l)

    def _arr(self, a, l):
        a = np.ascontiguousarray(a, dtype=self.dtype)
        assert a.shape == self.shape(l), (a.shape, self.shape(l))
        return a

    def diffusivity(self, s):
        out = np.zeros(2, self.real)
        fn = self.lib.cd_diffusivity
        fn.argtypes = [ctypes.POINTER(_CdCfg), ctypes.c_double if self.real == np.float64 else ctypes.c_float,
                       ctypes.c_void_p]
        fn(ctypes.byref(self._c), float(s), _ptr(out))
        return complex(out[0], out[1])

    def gfield(self, l, ul):
        ul = self._arr(ul, l)
        g = np.zeros_like(ul)
        self.lib.cd_gfield(ctypes.byref(self._c), l, _ptr(ul), _ptr(g))
        return g

    def apply(self, l, g, u):
        g, u = self._arr(g, l), self._arr(u, l)
        Au, diag = np.zeros_like(u), np.zeros_like(u)
        self.lib.cd_apply(ctypes.byref(self._c), l, _ptr(g), _ptr(u), _ptr(Au), _ptr(diag))
        return Au, diag

    def smooth(self, l, g, u, f):
        g, f = self._arr(g, l), self._arr(f, l)
        u = self._arr(u, l).copy()
        self.lib.cd_smooth(ctypes.byref(self._c), l, _ptr(g), _ptr(u), _ptr(f))
        return u

    def restrict(self, l, v):
        v = self._arr(v, l)
        out = np.zeros(self.shape(l + 1), self.dtype)
        self.lib.cd_restrict(ctypes.byref(self._c), l, _ptr(v), _ptr(out))
        return out

    def prolong_add(self, l, e, u):
        e = self._arr(e, l + 1)
        u = self._arr(u, l).copy()
        self.lib.cd_prolong_add(ctypes.byref(self._c), l, _ptr(e), _ptr(u))
        return u

    def norm(self, l, u, f):
        return self.lib.cd_norm(ctypes.byref(self._c), l, _ptr(self._arr(u, l)), _ptr(self._arr(f, l)))

    def cycle(self, u, f):
        u = self._arr(u, 0).copy()
        if self.lib.cd_cycle(ctypes.byref(self._c), _ptr(u), _ptr(self._arr(f, 0))) != 0:
            raise RuntimeError("cd_cycle failed")
        return u

    def solve(self, u, f, rtol, max_cycles):
        u = self._arr(u, 0).copy()
        hist = np.zeros(max_cycles + 1, np.float64)
        k = self.lib.cd_solve(ctypes.byref(self._c), _ptr(u), _ptr(self._arr(f, 0)), float(rtol), int(max_cycles),
                              _ptr(hist))
        if k < 0:
            raise RuntimeError("oracle cd_solve failed (non-finite residual)")
        return u, k, hist[: k + 1]
