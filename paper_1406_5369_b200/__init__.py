"""paper_1406_5369_b200 — B200-native geometric multigrid V-cycle (arXiv:1406.5369).

Thin Python binding of the C ABI in include/mg.h (libmgb200.so, built in-tree
by `make` / __graft_entry__.build()).  This module only marshals arguments:
every step of the V-cycle runs in the library's sm_100a kernels.  There is no
CPU fallback — if the shared library or a B200 is missing, calls fail loudly.

PyTorch supplies device memory and streams: u/f are CUDA tensors of shape
Solver.shape (= [planes][rows][pitch], see mg.h); `from_numpy`/`to_numpy`
convert between the dense unpadded node arrays used by the tests and that
layout.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MG_LIBRARY selects another build of the same library (the tests' CHECKED build,
# libmgb200_checked.so: guard-banded allocations and bounded mbarrier waits); default: the product
LIB_PATH = os.environ.get("MG_LIBRARY") or os.path.join(_HERE, "libmgb200.so")

JACOBI, RBGS, GS_LEX = 0, 1, 2
FP64, FP32 = 0, 1
COARSE_DIRECT, COARSE_SWEEPS = 0, 1
FLAG_NO_GRAPH, FLAG_BASELINE, FLAG_SLAB, FLAG_SEPARATE_PROLONG, FLAG_HOST_LOOP = 1, 2, 4, 8, 16
FLAG_NO_KFUSE, FLAG_CD_KFUSE = 32, 64
PROBLEM_POISSON, PROBLEM_COMPLEX_DIFFUSION = 0, 1

# every symbol include/mg.h declares (checked by tests/test_abi.py)
ABI_SYMBOLS = [
    "mg_config_default", "mg_create", "mg_layout", "mg_level_layout", "mg_num_levels", "mg_vcycle",
    "mg_residual_norm", "mg_solve", "mg_vcycle_host", "mg_vcycle_host_batch", "mg_loopback_group_create",
    "mg_loopback_group_destroy", "mg_op_smooth", "mg_op_residual", "mg_op_restrict",
    "mg_op_prolong_correct", "mg_op_coarse_solve", "mg_op_norm", "mg_workload_fill",
    "mg_launches_per_cycle", "mg_profile_enable", "mg_profile_read", "mg_error_string", "mg_destroy",
    "mg_partition", "mg_nccl_unique_id", "mg_fault_inject",
]
FAULT_NONE, FAULT_COMM_ERROR, FAULT_HALO_CORRUPT = 0, 1, 2


class MGConfig(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int32),
        ("nodes", ctypes.c_int64 * 3),
        ("levels", ctypes.c_int32),
        ("coeff", ctypes.c_double * 3),
        ("h", ctypes.c_double * 3),
        ("smoother", ctypes.c_int32),
        ("omega", ctypes.c_double),
        ("nu1", ctypes.c_int32),
        ("nu2", ctypes.c_int32),
        ("coarse", ctypes.c_int32),
        ("ncoarse", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("nranks", ctypes.c_int32),
        ("nccl_id", ctypes.c_void_p),
        ("flags", ctypes.c_uint32),
        ("pm_min_nx", ctypes.c_int32),
        ("problem", ctypes.c_int32),
        ("tau", ctypes.c_double),
        ("theta", ctypes.c_double),
        ("kappa", ctypes.c_double),
        ("loopback", ctypes.c_void_p),
        ("comm_timeout_s", ctypes.c_double),
    ]


class MGError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"mg status {status}: {msg}")
        self.status = status


_lib = None


def load_library():
    """Load libmgb200.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `make lib` or __graft_entry__.build()")
    lib = ctypes.CDLL(LIB_PATH)
    P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    pI64 = ctypes.POINTER(ctypes.c_int64)
    pD = ctypes.POINTER(ctypes.c_double)
    lib.mg_config_default.argtypes = [ctypes.POINTER(MGConfig), I32, I64]
    lib.mg_config_default.restype = None
    lib.mg_create.argtypes = [ctypes.POINTER(MGConfig), ctypes.POINTER(P)]
    lib.mg_layout.argtypes = [P, pI64, pI64, pI64]
    lib.mg_level_layout.argtypes = [P, I32, pI64]
    lib.mg_num_levels.argtypes = [P]
    lib.mg_num_levels.restype = I32
    lib.mg_vcycle.argtypes = [P, P, P, P]
    lib.mg_residual_norm.argtypes = [P, P, P, pD, P]
    lib.mg_solve.argtypes = [P, P, P, D, I32, ctypes.POINTER(I32), pD, P]
    lib.mg_vcycle_host.argtypes = [P, P, P, I32, pD, P]
    lib.mg_loopback_group_create.argtypes = [I32, ctypes.POINTER(P)]
    lib.mg_loopback_group_destroy.argtypes = [P]
    lib.mg_loopback_group_destroy.restype = None
    lib.mg_vcycle_host_batch.argtypes = [P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P), I32, I32, pD, P]
    lib.mg_op_smooth.argtypes = [P, I32, P, P, P, P]
    lib.mg_op_residual.argtypes = [P, I32, P, P, P, P]
    lib.mg_op_restrict.argtypes = [P, I32, P, P, P]
    lib.mg_op_prolong_correct.argtypes = [P, I32, P, P, P]
    lib.mg_op_coarse_solve.argtypes = [P, P, P, P]
    lib.mg_op_norm.argtypes = [P, I32, P, P, pD, P]
    lib.mg_workload_fill.argtypes = [P, P, ctypes.c_uint64, D, D, P]
    lib.mg_launches_per_cycle.argtypes = [P]
    lib.mg_launches_per_cycle.restype = I64
    lib.mg_profile_enable.argtypes = [P, I32]
    lib.mg_profile_read.argtypes = [P, I32, ctypes.POINTER(ctypes.c_char_p), pD, pI64, pD]
    lib.mg_profile_read.restype = I32
    lib.mg_error_string.argtypes = [P]
    lib.mg_error_string.restype = ctypes.c_char_p
    lib.mg_partition.argtypes = [ctypes.POINTER(MGConfig), I32, pI64, pI64, ctypes.POINTER(I32),
                                 ctypes.POINTER(I32)]
    lib.mg_nccl_unique_id.argtypes = [P]
    lib.mg_destroy.argtypes = [P]
    lib.mg_fault_inject.argtypes = [P, I32, I32]
    lib.mg_destroy.restype = None
    for name in ABI_SYMBOLS:
        if name not in ("mg_config_default", "mg_num_levels", "mg_launches_per_cycle", "mg_profile_read",
                        "mg_error_string", "mg_destroy"):
            getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _torch():
    import torch
    return torch


def _smoother_code(smoother):
    return {"rbgs": RBGS, RBGS: RBGS, "gs_lex": GS_LEX, GS_LEX: GS_LEX}.get(smoother, JACOBI)


def _problem_code(problem):
    return PROBLEM_COMPLEX_DIFFUSION if problem in ("complex_diffusion", "cd", PROBLEM_COMPLEX_DIFFUSION) \
        else PROBLEM_POISSON


def make_config(dim, nodes, levels=0, smoother="rbgs", omega=None, nu1=2, nu2=2, coarse="direct", ncoarse=10,
                dtype="f64", device=0, coeff=(1.0, 1.0, 1.0), h=None, flags=0, rank=0, nranks=1, pm_min_nx=0,
                problem="poisson", tau=None, theta=None, kappa=None):
    """Build an mg_config (argument marshalling only)."""
    lib = load_library()
    if isinstance(nodes, int):
        nodes = (nodes,) * dim
    c = MGConfig()
    lib.mg_config_default(ctypes.byref(c), dim, int(nodes[0]))
    for d in range(3):
        c.nodes[d] = int(nodes[d]) if d < dim else 1
        c.coeff[d] = float(coeff[d])
        c.h[d] = 0.0 if h is None or d >= dim else float(h[d])
    c.levels = levels
    c.smoother = _smoother_code(smoother)
    c.omega = float(omega) if omega is not None else (0.8 if c.smoother == JACOBI else 1.0)
    c.nu1, c.nu2 = nu1, nu2
    c.coarse = COARSE_DIRECT if coarse in ("direct", COARSE_DIRECT) else COARSE_SWEEPS
    c.ncoarse = ncoarse
    c.dtype = FP64 if dtype in ("f64", FP64) else FP32
    c.device = device
    c.rank, c.nranks = rank, nranks
    c.flags = flags
    c.pm_min_nx = pm_min_nx
    c.problem = _problem_code(problem)
    if tau is not None:
        c.tau = float(tau)
    if theta is not None:
        c.theta = float(theta)
    if kappa is not None:
        c.kappa = float(kappa)
    return c


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (rank 0 creates it; broadcast it to the other ranks)."""
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    st = lib.mg_nccl_unique_id(buf)
    if st != 0:
        raise MGError(st, lib.mg_error_string(None).decode())
    return buf.raw


class LoopbackGroup:
    """mg_loopback_group_create: `nranks` solvers of this process on one device, each driven
    by its own host thread and stream, exchanging halos by device copies (tests of the
    multi-rank path on one GPU; solvers need flags=FLAG_NO_GRAPH)."""

    def __init__(self, nranks):
        self.lib = load_library()
        h = ctypes.c_void_p()
        st = self.lib.mg_loopback_group_create(int(nranks), ctypes.byref(h))
        if st != 0:
            raise MGError(st, self.lib.mg_error_string(None).decode())
        self.handle = h.value
        self.nranks = nranks

    def close(self):
        if self.handle:
            self.lib.mg_loopback_group_destroy(ctypes.c_void_p(self.handle))
            self.handle = None


def distributed_solver(dim, nodes, **kw):
    """Collective: one Solver per rank of the default torch.distributed group, z-slab
    decomposed over NCCL (the unique id is broadcast through torch.distributed)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return Solver(dim, nodes, rank=rank, nranks=world, nccl_id=obj[0], **kw)


def partition(level, **kw):
    """Host-only mg_partition: (first_plane, owned_planes, distributed, halo) of `level`."""
    lib = load_library()
    c = make_config(**kw)
    a, n = ctypes.c_int64(), ctypes.c_int64()
    d, hh = ctypes.c_int32(), ctypes.c_int32()
    st = lib.mg_partition(ctypes.byref(c), level, ctypes.byref(a), ctypes.byref(n), ctypes.byref(d), ctypes.byref(hh))
    if st != 0:
        raise MGError(st, lib.mg_error_string(None).decode())
    return a.value, n.value, bool(d.value), hh.value


class Solver:
    """Owns one mg_solver (include/mg.h).  Arguments mirror mg_config."""

    def __init__(self, dim, nodes, levels=0, smoother="rbgs", omega=None, nu1=2, nu2=2, coarse="direct",
                 ncoarse=10, dtype="f64", device=0, coeff=(1.0, 1.0, 1.0), h=None, flags=0, rank=0, nranks=1,
                 nccl_id=None, pm_min_nx=0, problem="poisson", tau=None, theta=None, kappa=None, loopback=None,
                 comm_timeout_s=0.0):
        """problem="complex_diffusion": `nodes` are CELLS per axis, arrays are complex
        (torch complex64 / complex128), coarse defaults to "sweeps" (FAS)."""
        lib = load_library()
        self.lib = lib
        if isinstance(nodes, int):
            nodes = (nodes,) * dim
        c = MGConfig()
        lib.mg_config_default(ctypes.byref(c), dim, int(nodes[0]))
        for d in range(3):
            c.nodes[d] = int(nodes[d]) if d < dim else 1
            c.coeff[d] = float(coeff[d])
            c.h[d] = 0.0 if h is None or d >= dim else float(h[d])
        c.levels = levels
        c.smoother = _smoother_code(smoother)
        c.omega = float(omega) if omega is not None else (0.8 if c.smoother == JACOBI else 1.0)
        c.nu1, c.nu2 = nu1, nu2
        c.coarse = COARSE_DIRECT if coarse in ("direct", COARSE_DIRECT) else COARSE_SWEEPS
        c.ncoarse = ncoarse
        c.dtype = FP64 if dtype in ("f64", FP64) else FP32
        c.device = device
        c.rank, c.nranks = rank, nranks
        self._nccl_id = nccl_id
        c.nccl_id = ctypes.cast(ctypes.c_char_p(nccl_id), ctypes.c_void_p) if nccl_id is not None else None
        c.flags = flags
        c.pm_min_nx = pm_min_nx
        c.problem = _problem_code(problem)
        c.loopback = loopback.handle if isinstance(loopback, LoopbackGroup) else loopback
        c.comm_timeout_s = float(comm_timeout_s)
        self._loopback = loopback  # keep the group alive while this rank exists
        self.complex = c.problem == PROBLEM_COMPLEX_DIFFUSION
        if self.complex and coarse == "direct":
            c.coarse = COARSE_SWEEPS
        if tau is not None:
            c.tau = float(tau)
        if theta is not None:
            c.theta = float(theta)
        if kappa is not None:
            c.kappa = float(kappa)
        self.cfg = c
        self.dim = dim
        self.nodes = tuple(int(n) for n in nodes[:dim])
        h_ = ctypes.c_void_p()
        st = lib.mg_create(ctypes.byref(c), ctypes.byref(h_))
        if st != 0:
            raise MGError(st, lib.mg_error_string(None).decode())
        self.h = h_
        self.levels = lib.mg_num_levels(self.h)
        torch = _torch()
        if self.complex:
            self.torch_dtype = torch.complex128 if c.dtype == FP64 else torch.complex64
            self.np_dtype = np.complex128 if c.dtype == FP64 else np.complex64
            self.first_plane, self.owned_planes, self.distributed, self.halo = 0, self.shape[0], False, 0
            return
        self.torch_dtype = torch.float64 if c.dtype == FP64 else torch.float32
        self.np_dtype = np.float64 if c.dtype == FP64 else np.float32
        self.first_plane, self.owned_planes, self.distributed, self.halo = partition(
            0, dim=dim, nodes=nodes, levels=levels, flags=flags, rank=rank, nranks=nranks)

    # ---- lifetime
    def close(self):
        if getattr(self, "h", None):
            self.lib.mg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, st):
        if st != 0:
            raise MGError(st, self.lib.mg_error_string(self.h).decode())

    @staticmethod
    def _stream(stream):
        if stream is None:
            return ctypes.c_void_p(_torch().cuda.current_stream().cuda_stream)
        return ctypes.c_void_p(getattr(stream, "cuda_stream", stream))

    @staticmethod
    def _p(t):
        return ctypes.c_void_p(t.data_ptr())

    def _dev(self, t, level=0, what="array"):
        """Device pointer of a caller array after checking what the C ABI cannot: a CUDA tensor on
        the solver's device, the solver's dtype, contiguous, of the level's layout (mg.h) — a raw
        pointer to anything else would be read and written out of bounds."""
        torch = _torch()
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{what}: expected a torch.Tensor, got {type(t).__name__}")
        if t.device.type != "cuda" or (t.device.index or 0) != self.cfg.device:
            raise ValueError(f"{what}: expected a tensor on cuda:{self.cfg.device}, got {t.device}")
        if t.dtype != self.torch_dtype:
            raise TypeError(f"{what}: expected dtype {self.torch_dtype}, got {t.dtype}")
        want = self.shape if level == 0 else self.level_shape(level)
        if tuple(t.shape) != tuple(want):
            raise ValueError(f"{what}: expected shape {tuple(want)} (level {level} layout), got {tuple(t.shape)}")
        if not t.is_contiguous():
            raise ValueError(f"{what}: expected a contiguous tensor")
        return ctypes.c_void_p(t.data_ptr())

    def _host(self, t, what="host array"):
        """Host pointer of a level-0 host array (dense layout, the solver's dtype)."""
        torch = _torch()
        if not isinstance(t, torch.Tensor) or t.device.type != "cpu":
            raise TypeError(f"{what}: expected a CPU torch.Tensor")
        if t.dtype != self.torch_dtype or tuple(t.shape) != tuple(self.shape) or not t.is_contiguous():
            raise ValueError(f"{what}: expected a contiguous {self.torch_dtype} tensor of shape {tuple(self.shape)}, "
                             f"got {t.dtype} {tuple(t.shape)}")
        return t.data_ptr()

    # ---- layout
    @property
    def shape(self):
        s = (ctypes.c_int64 * 3)()
        first, owned = ctypes.c_int64(), ctypes.c_int64()
        self._chk(self.lib.mg_layout(self.h, s, ctypes.byref(first), ctypes.byref(owned)))
        return tuple(s)

    def level_shape(self, level):
        s = (ctypes.c_int64 * 3)()
        self._chk(self.lib.mg_level_layout(self.h, level, s))
        return tuple(s)

    def level_cells(self, level):
        if self.complex:
            return tuple(n >> level for n in self.nodes)
        return tuple((n - 1) >> level for n in self.nodes)

    def empty(self, level=0):
        torch = _torch()
        return torch.zeros(self.level_shape(level), dtype=self.torch_dtype, device=f"cuda:{self.cfg.device}")

    def from_numpy(self, a, level=0):
        """Dense GLOBAL node array (2D: (ny+1,nx+1); 3D: (nz+1,ny+1,nx+1)) -> padded device
        tensor of this rank's layout (in slab mode: its planes plus halo planes)."""
        torch = _torch()
        P, R, X = self.level_shape(level)
        host = np.zeros((P, R, X), dtype=self.np_dtype)
        a = np.asarray(a, dtype=self.np_dtype)
        if self.dim == 2:
            a = a[:, None, :]
        if self.complex:  # cell array, no boundary entries
            host[:, :, : a.shape[2]] = a
            return torch.from_numpy(host).to(f"cuda:{self.cfg.device}")
        g0 = self.first_plane - self.halo if (level == 0 and self.distributed) else 0
        for i in range(P):
            gp = g0 + i
            if 0 <= gp < a.shape[0]:
                host[i, :, : a.shape[2]] = a[gp]
        return torch.from_numpy(host).to(f"cuda:{self.cfg.device}")

    def to_numpy(self, t, level=0):
        """Device tensor -> dense node array; in slab mode the rank's OWNED planes only."""
        nx = self.level_cells(level)[0] + (0 if self.complex else 1)
        a = t.detach().cpu().numpy()
        if level == 0 and self.distributed:
            a = a[self.halo: self.halo + self.owned_planes]
        return np.ascontiguousarray(a[:, 0, :nx] if self.dim == 2 else a[:, :, :nx])

    # ---- the method
    def vcycle(self, u, f, stream=None):
        self._chk(self.lib.mg_vcycle(self.h, self._dev(u, 0, "u"), self._dev(f, 0, "f"), self._stream(stream)))

    def residual_norm(self, u, f, stream=None):
        out = ctypes.c_double()
        self._chk(self.lib.mg_residual_norm(self.h, self._dev(u, 0, "u"), self._dev(f, 0, "f"), ctypes.byref(out),
                                            self._stream(stream)))
        return out.value

    def solve(self, u, f, rtol, max_cycles, stream=None):
        hist = (ctypes.c_double * (max_cycles + 1))()
        k = ctypes.c_int32()
        self._chk(self.lib.mg_solve(self.h, self._dev(u, 0, "u"), self._dev(f, 0, "f"), float(rtol), int(max_cycles), ctypes.byref(k),
                                    hist, self._stream(stream)))
        return k.value, list(hist)[: k.value + 1]

    def vcycle_host(self, u_host, f_host, ncycles=1, stream=None):
        """End-to-end through the C ABI with host (pinned) tensors; returns the residual norm."""
        out = ctypes.c_double()
        self._chk(self.lib.mg_vcycle_host(self.h, ctypes.c_void_p(self._host(u_host, "u_host")),
                                          ctypes.c_void_p(self._host(f_host, "f_host")), int(ncycles), ctypes.byref(out),
                                          self._stream(stream)))
        return out.value

    def vcycle_host_batch(self, u_in, u_out, f_in, ncycles=1, stream=None):
        """Pipelined end-to-end over independent problems held in host (pinned) tensors:
        lists u_in, u_out, f_in of equal length; returns the residual norm of each problem."""
        n = len(u_in)
        if not (len(u_out) == len(f_in) == n):
            raise ValueError("u_in, u_out and f_in must have equal lengths")
        arr = lambda ts: (ctypes.c_void_p * n)(*[self._host(t) for t in ts])
        norms = (ctypes.c_double * n)()
        self._chk(self.lib.mg_vcycle_host_batch(self.h, arr(u_in), arr(u_out), arr(f_in), n, int(ncycles), norms,
                                                self._stream(stream)))
        return list(norms)

    # ---- per-operation entry points
    def op_smooth(self, level, u_in, f, u_out, stream=None):
        self._chk(self.lib.mg_op_smooth(self.h, level, self._dev(u_in, level, "u_in"), self._dev(f, level, "f"),
                                        self._dev(u_out, level, "u_out"),
                                        self._stream(stream)))

    def op_residual(self, level, u, f, r, stream=None):
        self._chk(self.lib.mg_op_residual(self.h, level, self._dev(u, level, "u"), self._dev(f, level, "f"),
                                          self._dev(r, level, "r"), self._stream(stream)))

    def op_restrict(self, level, r, fc, stream=None):
        self._chk(self.lib.mg_op_restrict(self.h, level, self._dev(r, level, "r"), self._dev(fc, level + 1, "fc"),
                                          self._stream(stream)))

    def op_prolong_correct(self, level, e, u, stream=None):
        self._chk(self.lib.mg_op_prolong_correct(self.h, level, self._dev(e, level + 1, "e"), self._dev(u, level, "u"),
                                                 self._stream(stream)))

    def op_coarse_solve(self, f, e, stream=None):
        self._chk(self.lib.mg_op_coarse_solve(self.h, self._dev(f, self.levels - 1, "f"), self._dev(e, self.levels - 1, "e"),
                                              self._stream(stream)))

    def op_norm(self, level, u, f, stream=None):
        out = ctypes.c_double()
        self._chk(self.lib.mg_op_norm(self.h, level, self._dev(u, level, "u"), self._dev(f, level, "f"), ctypes.byref(out),
                                      self._stream(stream)))
        return out.value

    def workload_fill(self, dst, seed, lo=0.0, hi=1.0, stream=None):
        self._chk(self.lib.mg_workload_fill(self.h, self._dev(dst, 0, "dst"), ctypes.c_uint64(seed), float(lo), float(hi),
                                            self._stream(stream)))

    def fault_inject(self, kind, countdown=1):
        """mg_fault_inject (tests of the multi-rank failure path)."""
        self._chk(self.lib.mg_fault_inject(self.h, int(kind), int(countdown)))

    # ---- instrumentation
    @property
    def launches_per_cycle(self):
        return self.lib.mg_launches_per_cycle(self.h)

    def profile_enable(self, on=True):
        self._chk(self.lib.mg_profile_enable(self.h, 1 if on else 0))

    def profile_read(self):
        n = self.lib.mg_profile_read(self.h, 0, None, None, None, None)
        names = (ctypes.c_char_p * max(n, 1))()
        ms = (ctypes.c_double * max(n, 1))()
        cnt = (ctypes.c_int64 * max(n, 1))()
        by = (ctypes.c_double * max(n, 1))()
        n = self.lib.mg_profile_read(self.h, n, names, ms, cnt, by)
        return [dict(name=names[i].decode(), ms=ms[i], count=cnt[i], bytes=by[i]) for i in range(n)]
