"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the multigrid method: only the counter-based
generator and the right-hand sides / initial guesses of the paper's workloads
(DESIGN.md §4 "input recipe").  Both sides receive identical arrays from here,
or — for full-size bench grids — the CUDA library's ``mg_workload_fill``
re-implements the same counter-based generator on the device (a GPU test
checks the two bit for bit).

Workloads:
  W1  the paper's test problem: f = 0, u0 ~ U[0,1) on interior nodes,
      homogeneous Dirichlet boundary ("Function f = 0",
      "Unknown solution = initrandom", "PDEBC bc { solution = 0 }").
  W2  sine manufactured solution u* = prod sin(pi x_d), f = d pi^2 u*.
  W3  polynomial manufactured solution u* = prod x_d(1-x_d),
      f = 2 sum_d prod_{e != d} x_e(1-x_e)   (the discrete solution is exact).
  W4  generic right-hand side f ~ U[-1,1), u0 = 0.
  W5  complex diffusion: one implicit-Euler step from
      a noisy image u^n (real part U[0,1) per cell, imaginary part 0): f = u^n,
      initial guess u = u^n.  Cell arrays, complex.

Arrays are dense, unpadded node arrays including the boundary, x fastest:
shape (ny+1, nx+1) in 2D and (nz+1, ny+1, nx+1) in 3D.
"""
from __future__ import annotations

import numpy as np

# SplitMix64 constants (reading 10 of DESIGN.md §3)
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64_uniform(seed: int, idx: np.ndarray) -> np.ndarray:
    """The idx-th SplitMix64 output mapped to [0,1): (z >> 11) * 2^-53.

    z = seed + (idx+1)*0x9E3779B97F4A7C15 (mod 2^64), then the standard
    SplitMix64 finaliser.  Vectorised over ``idx`` (uint64)."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (idx + np.uint64(1)) * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def node_shape(dim: int, cells) -> tuple:
    cells = list(cells)
    if dim == 2:
        return (cells[1] + 1, cells[0] + 1)
    return (cells[2] + 1, cells[1] + 1, cells[0] + 1)


def _interior_mask(shape) -> np.ndarray:
    m = np.zeros(shape, dtype=bool)
    m[(slice(1, -1),) * len(shape)] = True
    return m


def random_interior(dim: int, cells, seed: int, dtype=np.float64, lo=0.0, hi=1.0) -> np.ndarray:
    """U[lo,hi) on interior nodes from the global node index, 0 on the boundary.
    idx = (k*(ny+1) + j)*(nx+1) + i on the unpadded global node grid."""
    shape = node_shape(dim, cells)
    n = int(np.prod(shape))
    r = splitmix64_uniform(seed, np.arange(n, dtype=np.uint64)).reshape(shape)
    if lo != 0.0 or hi != 1.0:
        r = lo + (hi - lo) * r
    r[~_interior_mask(shape)] = 0.0
    return r.astype(dtype)  # FP32: round-to-nearest of the double


def coords(dim: int, cells, h=None):
    """Node coordinates x_d = i_d * h_d (unit domain by default), broadcastable."""
    cells = list(cells)[:dim]
    if h is None:
        h = [1.0 / c for c in cells]
    axes = [np.arange(c + 1, dtype=np.float64) * hh for c, hh in zip(cells, h)]
    # returned in array-axis order (z, y, x) / (y, x)
    grids = np.meshgrid(*axes[::-1], indexing="ij")
    return grids[::-1]  # x, y[, z]


def workload(name: str, dim: int, cells, seed: int = 42, dtype=np.float64):
    """Return (u0, f) for workload W1..W4 as dense node arrays."""
    shape = node_shape(dim, cells)
    if name == "W1":
        return random_interior(dim, cells, seed, dtype), np.zeros(shape, dtype=dtype)
    if name == "W4":
        f = random_interior(dim, cells, seed, np.float64, -1.0, 1.0)
        return np.zeros(shape, dtype=dtype), f.astype(dtype)
    xs = coords(dim, cells)
    if name == "W2":
        us = np.ones(shape)
        for x in xs:
            us = us * np.sin(np.pi * x)
        f = dim * np.pi ** 2 * us
    elif name == "W3":
        f = np.zeros(shape)
        for d in range(dim):
            t = np.full(shape, 2.0)
            for e, x in enumerate(xs):
                if e != d:
                    t = t * (x * (1.0 - x))
            f = f + t
    else:
        raise ValueError(f"unknown workload {name}")
    f[~_interior_mask(shape)] = 0.0
    return np.zeros(shape, dtype=dtype), f.astype(dtype)


def cell_shape(dim: int, cells) -> tuple:
    cells = list(cells)
    return (cells[1], cells[0]) if dim == 2 else (cells[2], cells[1], cells[0])


def random_cells(dim: int, cells, seed: int, lo=0.0, hi=1.0) -> np.ndarray:
    """U[lo,hi) per cell from the global cell index idx = (k*ny + j)*nx + i (float64)."""
    shape = cell_shape(dim, cells)
    r = splitmix64_uniform(seed, np.arange(int(np.prod(shape)), dtype=np.uint64)).reshape(shape)
    if lo != 0.0 or hi != 1.0:
        r = lo + (hi - lo) * r
    return r


def cd_workload(dim: int, cells, seed: int = 42, dtype=np.complex128):
    """W5: (u0, f) = (u^n, u^n), u^n = U[0,1) + 0i per cell (a noise image)."""
    re = random_cells(dim, cells, seed).astype(np.float64 if np.dtype(dtype) == np.complex128 else np.float32)
    u = re.astype(dtype)
    return u.copy(), u


def exact_solution(name: str, dim: int, cells) -> np.ndarray:
    """Continuous solution u* of W2/W3 at the nodes (for error checks)."""
    xs = coords(dim, cells)
    u = np.ones(node_shape(dim, cells))
    for x in xs:
        u = u * (np.sin(np.pi * x) if name == "W2" else x * (1.0 - x))
    return u
