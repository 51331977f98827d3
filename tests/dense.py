"""Dense-matrix brute force of the multigrid components, written from the
definitions in the paper (not from the oracle's code): used only to PIN the
oracle on tiny grids (DESIGN.md §5 "pins").

Unknowns are the interior nodes of a level, lexicographic with x fastest:
p = (k*my + j)*mx + i (0-based over the interior), matching a C-order
reshape of the interior block of a node array (z, y, x).
"""
from __future__ import annotations

import numpy as np


def tri(m: int) -> np.ndarray:
    """1D second difference tridiag(-1, 2, -1) of size m (the 1D -Delta_h * h^2)."""
    return 2.0 * np.eye(m) - np.eye(m, k=1) - np.eye(m, k=-1)


def kron_axes(mats_xyz):
    """Kronecker product with x fastest: M = Mz (x) My (x) Mx."""
    out = np.ones((1, 1))
    for M in mats_xyz[::-1]:
        out = np.kron(out, M)
    return out


def level_cells(cells, l):
    return [c >> l for c in cells]


def coeffs(cells0, l, a=(1.0, 1.0, 1.0), h0=None, omega=1.0):
    """Re-discretised coefficients at level l: c_d = a_d / (2^l h_d)^2."""
    dim = len(cells0)
    if h0 is None:
        h0 = [1.0 / n for n in cells0]
    c = [a[d] / (2.0 ** l * h0[d]) ** 2 for d in range(dim)]
    D = 2.0 * sum(c)
    return c, D, omega / D


def assemble_A(cells, c):
    """A = -Delta_h on the interior of a level with `cells` per axis (x,y[,z]):
    sum_d c_d * (I (x) ... T_d ... (x) I), Dirichlet boundary eliminated."""
    dim = len(cells)
    m = [n - 1 for n in cells]
    A = np.zeros((int(np.prod(m)),) * 2)
    for d in range(dim):
        mats = [np.eye(m[e]) if e != d else tri(m[e]) for e in range(dim)]
        A += c[d] * kron_axes(mats)
    return A


def P1(nc: int) -> np.ndarray:
    """1D linear interpolation, coarse interior (nc-1) -> fine interior (2nc-1)."""
    mf, mc = 2 * nc - 1, nc - 1
    P = np.zeros((mf, mc))
    for I in range(1, nc):
        P[2 * I - 1, I - 1] = 1.0          # fine node 2I coincides with coarse I
        P[2 * I - 2, I - 1] = 0.5          # fine node 2I-1
        P[2 * I, I - 1] = 0.5              # fine node 2I+1
    return P


def assemble_P(cells_coarse):
    """Bi-/trilinear prolongation: tensor product of 1D P1."""
    return kron_axes([P1(n) for n in cells_coarse])


def assemble_R(cells_coarse):
    """Full weighting R = 2^-d P^T (P:227 'its transpose as restriction'; reading 7)."""
    d = len(cells_coarse)
    return assemble_P(cells_coarse).T / 2.0 ** d


def colour_masks(cells):
    """Red = even sum of global node indices (reading 8)."""
    idx = np.indices([n - 1 for n in cells[::-1]]) + 1  # (z,y,x) interior node indices
    s = idx.sum(axis=0).reshape(-1)
    return (s % 2 == 0), (s % 2 == 1)


def jacobi(A, D, omega, u, f):
    return u + omega / D * (f - A @ u)


def rbgs(A, D, omega, u, f, cells):
    red, black = colour_masks(cells)
    u = u.copy()
    for mask in (red, black):
        r = f - A @ u
        u[mask] = u[mask] + omega / D * r[mask]
    return u


def gs_lex(A, D, omega, u, f):
    """Lexicographic SOR written as a matrix iteration: with A = D - L - U (L strictly
    lower in lex order), u' = u + omega (D - omega L)^-1 (f - A u)."""
    L = -np.tril(A, -1)
    return u + omega * np.linalg.solve(np.diag(np.full(A.shape[0], D)) - omega * L, f - A @ u)


def interior(a: np.ndarray) -> np.ndarray:
    return a[(slice(1, -1),) * a.ndim].reshape(-1).astype(np.float64)


def embed(v: np.ndarray, cells) -> np.ndarray:
    shape = [n + 1 for n in cells[::-1]]
    out = np.zeros(shape)
    out[(slice(1, -1),) * len(shape)] = v.reshape([n - 1 for n in cells[::-1]])
    return out


class DenseMG:
    """Algorithm 1 in dense linear algebra on interior vectors."""

    def __init__(self, cells0, levels, smoother="rbgs", omega=1.0, nu1=2, nu2=2,
                 coarse="direct", ncoarse=10):
        self.cells0 = list(cells0)
        self.levels = levels
        self.smoother, self.omega, self.nu1, self.nu2 = smoother, omega, nu1, nu2
        self.coarse, self.ncoarse = coarse, ncoarse
        self.A, self.D, self.cells = [], [], []
        for l in range(levels):
            cl = level_cells(self.cells0, l)
            c, D, _ = coeffs(self.cells0, l, omega=omega)
            self.cells.append(cl)
            self.A.append(assemble_A(cl, c))
            self.D.append(D)
        self.P = [assemble_P(self.cells[l + 1]) for l in range(levels - 1)]
        self.R = [assemble_R(self.cells[l + 1]) for l in range(levels - 1)]

    def smooth(self, l, u, f):
        if self.smoother == "jacobi":
            return jacobi(self.A[l], self.D[l], self.omega, u, f)
        if self.smoother == "gs_lex":
            return gs_lex(self.A[l], self.D[l], self.omega, u, f)
        return rbgs(self.A[l], self.D[l], self.omega, u, f, self.cells[l])

    def vcycle(self, u, f, l=0):
        if l == self.levels - 1:
            if self.coarse == "direct":
                return np.linalg.solve(self.A[l], f) if l > 0 else u + np.linalg.solve(self.A[l], f - self.A[l] @ u)
            for _ in range(self.ncoarse):
                u = self.smooth(l, u, f)
            return u
        for _ in range(self.nu1):
            u = self.smooth(l, u, f)
        r = f - self.A[l] @ u
        fH = self.R[l] @ r
        eH = self.vcycle(np.zeros_like(fH), fH, l + 1)
        u = u + self.P[l] @ eH
        for _ in range(self.nu2):
            u = self.smooth(l, u, f)
        return u

    def error_matrix(self):
        """Error propagation matrix M_V of one cycle (f = 0)."""
        n = self.A[0].shape[0]
        return np.stack([self.vcycle(e, np.zeros(n)) for e in np.eye(n)], axis=1)
