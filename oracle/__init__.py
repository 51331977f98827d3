"""ctypes wrapper of the CPU oracle (oracle/mg_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  Never by the product
package.  Arrays are dense unpadded node arrays (see workloads.node_shape).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

JACOBI, RBGS, GS_LEX = 0, 1, 2
COARSE_DIRECT, COARSE_SWEEPS = 0, 1


class _Cfg(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int),
        ("n", ctypes.c_int * 3),
        ("levels", ctypes.c_int),
        ("a", ctypes.c_double * 3),
        ("h", ctypes.c_double * 3),
        ("smoother", ctypes.c_int),
        ("omega", ctypes.c_double),
        ("nu1", ctypes.c_int),
        ("nu2", ctypes.c_int),
        ("coarse", ctypes.c_int),
        ("ncoarse", ctypes.c_int),
    ]


@dataclass
class Config:
    """Mirror of or_config; `cells` are cells per axis of the finest level."""
    dim: int
    cells: tuple
    levels: int = 0          # 0 => paper rule: coarsest level has 1 interior node
    smoother: int = RBGS
    omega: float = 1.0
    nu1: int = 2
    nu2: int = 2
    coarse: int = COARSE_DIRECT
    ncoarse: int = 10
    a: tuple = (1.0, 1.0, 1.0)
    h: tuple = field(default=None)

    def resolved_levels(self) -> int:
        if self.levels:
            return self.levels
        m = min(self.cells[: self.dim])
        return int(m).bit_length() - 1  # coarsest: 2 cells = 1 interior node

    def level_cells(self, l: int):
        return tuple(c >> l for c in self.cells[: self.dim])

    def c_struct(self) -> _Cfg:
        c = _Cfg()
        c.dim = self.dim
        cells = list(self.cells) + [0] * (3 - len(self.cells))
        for d in range(3):
            c.n[d] = int(cells[d]) if d < self.dim else 0
            c.a[d] = float(self.a[d]) if d < self.dim else 0.0
            if self.h is None:
                c.h[d] = 1.0 / cells[d] if d < self.dim else 0.0
            else:
                c.h[d] = float(self.h[d]) if d < self.dim else 0.0
        c.levels = self.resolved_levels()
        c.smoother = self.smoother
        c.omega = self.omega
        c.nu1, c.nu2 = self.nu1, self.nu2
        c.coarse, c.ncoarse = self.coarse, self.ncoarse
        return c


def _load(dtype):
    name = "liboracle_f64.so" if np.dtype(dtype) == np.float64 else "liboracle_f32.so"
    path = os.path.join(_HERE, name)
    if not os.path.exists(path):
        raise RuntimeError(f"{path} missing: run `make oracle` (or __graft_entry__.build())")
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    C = ctypes.POINTER(_Cfg)
    lib.or_residual.argtypes = [C, ctypes.c_int, P, P, P]
    lib.or_jacobi.argtypes = [C, ctypes.c_int, P, P, P]
    lib.or_rbgs.argtypes = [C, ctypes.c_int, P, P]
    lib.or_gs_lex.argtypes = [C, ctypes.c_int, P, P]
    lib.or_smooth.argtypes = [C, ctypes.c_int, P, P, P]
    lib.or_restrict.argtypes = [C, ctypes.c_int, P, P]
    lib.or_prolong_correct.argtypes = [C, ctypes.c_int, P, P]
    lib.or_coarse_solve.argtypes = [C, P, P]
    lib.or_coarse_solve.restype = ctypes.c_int
    lib.or_norm.argtypes = [C, ctypes.c_int, P, P]
    lib.or_norm.restype = ctypes.c_double
    lib.or_vcycle.argtypes = [C, P, P]
    lib.or_vcycle.restype = ctypes.c_int
    lib.or_solve.argtypes = [C, P, P, ctypes.c_double, ctypes.c_int, P]
    lib.or_solve.restype = ctypes.c_int
    lib.or_coeffs.argtypes = [C, ctypes.c_int, ctypes.POINTER(ctypes.c_double * 3),
                              ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    lib.or_num_threads.restype = ctypes.c_int
    return lib


_LIBS = {}


def lib(dtype=np.float64):
    key = np.dtype(dtype).name
    if key not in _LIBS:
        _LIBS[key] = _load(dtype)
    return _LIBS[key]


def _ptr(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)


class Oracle:
    """Per-op and whole-cycle entry points on numpy arrays of one dtype."""

    def __init__(self, cfg: Config, dtype=np.float64):
        self.cfg = cfg
        self.dtype = np.dtype(dtype)
        self.lib = lib(dtype)
        self._c = cfg.c_struct()
        self.levels = self._c.levels

    def shape(self, l: int):
        cells = self.cfg.level_cells(l)
        return tuple(c + 1 for c in cells[::-1])

    def _chk(self, a, l):
        assert a.dtype == self.dtype and a.shape == self.shape(l), (a.dtype, a.shape, self.shape(l))
        return _ptr(a)

    def coeffs(self, l: int):
        c = (ctypes.c_double * 3)()
        D = ctypes.c_double()
        wd = ctypes.c_double()
        self.lib.or_coeffs(ctypes.byref(self._c), l, ctypes.byref(c), ctypes.byref(D), ctypes.byref(wd))
        return list(c), D.value, wd.value

    def residual(self, l, u, f):
        r = np.empty(self.shape(l), self.dtype)
        self.lib.or_residual(ctypes.byref(self._c), l, self._chk(u, l), self._chk(f, l), _ptr(r))
        return r

    def jacobi(self, l, u, f):
        out = np.empty(self.shape(l), self.dtype)
        self.lib.or_jacobi(ctypes.byref(self._c), l, self._chk(u, l), self._chk(f, l), _ptr(out))
        return out

    def rbgs(self, l, u, f):
        u = u.copy()
        self.lib.or_rbgs(ctypes.byref(self._c), l, self._chk(u, l), self._chk(f, l))
        return u

    def gs_lex(self, l, u, f):
        u = u.copy()
        self.lib.or_gs_lex(ctypes.byref(self._c), l, self._chk(u, l), self._chk(f, l))
        return u

    def smooth(self, l, u, f):
        if self.cfg.smoother == JACOBI:
            return self.jacobi(l, u, f)
        return self.gs_lex(l, u, f) if self.cfg.smoother == GS_LEX else self.rbgs(l, u, f)

    def restrict(self, l, r):
        fc = np.empty(self.shape(l + 1), self.dtype)
        self.lib.or_restrict(ctypes.byref(self._c), l, self._chk(r, l), _ptr(fc))
        return fc

    def prolong_correct(self, l, e, u):
        u = u.copy()
        self.lib.or_prolong_correct(ctypes.byref(self._c), l, self._chk(e, l + 1), self._chk(u, l))
        return u

    def coarse_solve(self, f):
        l = self.levels - 1
        e = np.empty(self.shape(l), self.dtype)
        rc = self.lib.or_coarse_solve(ctypes.byref(self._c), _ptr(e), self._chk(f, l))
        if rc:
            raise RuntimeError("coarse solve failed")
        return e

    def norm(self, l, u, f) -> float:
        return self.lib.or_norm(ctypes.byref(self._c), l, self._chk(u, l), self._chk(f, l))

    def vcycle(self, u, f):
        """One V-cycle; returns the new u (input untouched)."""
        u = np.ascontiguousarray(u, dtype=self.dtype).copy()
        f = np.ascontiguousarray(f, dtype=self.dtype)
        if self.lib.or_vcycle(ctypes.byref(self._c), self._chk(u, 0), self._chk(f, 0)):
            raise RuntimeError("oracle vcycle failed")
        return u

    def vcycle_inplace(self, u, f):
        if self.lib.or_vcycle(ctypes.byref(self._c), self._chk(u, 0), self._chk(f, 0)):
            raise RuntimeError("oracle vcycle failed")

    def solve(self, u, f, rtol, max_cycles):
        """Returns (u, cycles, history[0..cycles])."""
        u = np.ascontiguousarray(u, dtype=self.dtype).copy()
        f = np.ascontiguousarray(f, dtype=self.dtype)
        hist = np.zeros(max_cycles + 1, np.float64)
        k = self.lib.or_solve(ctypes.byref(self._c), self._chk(u, 0), self._chk(f, 0),
                              float(rtol), int(max_cycles), _ptr(hist))
        if k < 0:
            raise RuntimeError("oracle solve failed (non-finite residual)")
        return u, k, hist[: k + 1]


def num_threads(dtype=np.float64) -> int:
    return lib(dtype).or_num_threads()
