"""CPU emulation of the slab-decomposed V-cycle schedule for the
world-size-2 gloo tests: the SAME partition (libmgb200's host-only
mg_partition), the same halo exchanges (torch.distributed send/recv), the same
agglomeration (all_gather of coarse chunks) and the same deterministic norm
(all_gather of per-rank sums, summed in rank order) as the NCCL path, with the
per-plane arithmetic written in numpy in the canonical order (DESIGN.md
reading 13).  The coarse tail below the agglomeration level is the oracle's own
V-cycle.  Test infrastructure only.

Arrays are numpy (planes, rows, nx+1) slabs of global planes [g0, g0 + planes):
3D rows = y nodes; 2D rows = 1 and the plane axis is the paper's y (as in the
library).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

import oracle as orc
import paper_1406_5369_b200 as mgb


class Level:
    def __init__(self, dim, cells, l, h0, omega, dtype):
        self.dim = dim
        self.cells = [c >> l for c in cells]       # x, y(, z)
        self.nx = self.cells[0]
        self.n = self.cells[-1]                      # plane-axis cells
        self.rows = self.cells[1] + 1 if dim == 3 else 1
        hl = [h * 2.0 ** l for h in h0]
        c = [1.0 / (hh * hh) for hh in hl]
        D = 2.0 * sum(c)
        t = dtype
        self.cx = t(c[0])
        self.cy = t(c[1]) if dim == 3 else t(0.0)
        self.cz = t(c[2] if dim == 3 else c[1])
        self.D = t(D)
        self.wd = t(omega / D)
        self.dtype = dtype


def _rows(L):
    return slice(1, -1) if L.dim == 3 else slice(0, 1)


def apply_A(L, U, k):
    """A u at the interior nodes of local plane k (canonical order)."""
    rs = _rows(L)
    C = U[k][rs, 1:-1]
    s = L.cx * (U[k][rs, :-2] + U[k][rs, 2:])
    if L.dim == 3:
        s = s + L.cy * (U[k][:-2, 1:-1] + U[k][2:, 1:-1])
    s = s + L.cz * (U[k - 1][rs, 1:-1] + U[k + 1][rs, 1:-1])
    return L.D * C - s


def colour_mask(L, gplane, colour):
    """Interior-node mask of the plane's nodes of `colour` (0 red) by global parity."""
    rows = np.arange(1, L.rows - 1) if L.dim == 3 else np.array([0])
    xs = np.arange(1, L.nx)
    par = (rows[:, None] + xs[None, :] + gplane) & 1
    return par == colour


class SlabMG:
    def __init__(self, dim, nodes, smoother, omega, nu1, nu2, levels, rank, P, dtype=np.float64):
        self.dim, self.P, self.rank = dim, P, rank
        self.cells = [nodes - 1] * dim
        self.h0 = [1.0 / c for c in self.cells]
        self.sm, self.omega, self.nu1, self.nu2 = smoother, omega, nu1, nu2
        self.dtype = dtype
        kw = dict(dim=dim, nodes=nodes, levels=levels, smoother=smoother, omega=omega, nu1=nu1, nu2=nu2,
                  nranks=P, rank=rank)
        cfg_probe = mgb.Solver.__init__  # noqa: F841  (the library is only used for mg_partition)
        self.L = levels
        self.part = [mgb.partition(l, **kw) for l in range(levels)]   # (first, owned, distributed, halo)
        self.la = next(l for l in range(levels) if not self.part[l][2])
        self.H = self.part[0][3]
        self.lv = [Level(dim, self.cells, l, self.h0, omega, dtype) for l in range(levels)]

    # ---- layout helpers
    def g0(self, l):
        first, owned, distd, H = self.part[l]
        return first - H if distd else 0

    def local_planes(self, l):
        first, owned, distd, H = self.part[l]
        return owned + 2 * H if distd else self.lv[l].n + 1

    def owned_local(self, l):
        """local plane range [lo, hi) of owned planes that hold interior nodes."""
        first, owned, distd, H = self.part[l]
        n = self.lv[l].n
        a, b = first, first + owned
        lo, hi = max(a, 1), min(b, n)
        return lo - self.g0(l), hi - self.g0(l)

    def zeros(self, l):
        L = self.lv[l]
        return np.zeros((self.local_planes(l), L.rows, L.nx + 1), self.dtype)

    def from_global(self, l, A):
        U = self.zeros(l)
        g0 = self.g0(l)
        for i in range(U.shape[0]):
            if 0 <= g0 + i < A.shape[0]:
                U[i] = A[g0 + i]
        return U

    # ---- communication (same pattern as Exec::exchange / allgather_level / norm)
    def exchange(self, l, U, h):
        first, owned, distd, H = self.part[l]
        if not distd or self.P == 1:
            return
        reqs = []
        bufs = []
        if self.rank < self.P - 1:
            top = torch.from_numpy(np.ascontiguousarray(U[H + owned - h: H + owned]))
            rbuf = torch.empty_like(top)
            reqs += [dist.isend(top, self.rank + 1), dist.irecv(rbuf, self.rank + 1)]
            bufs.append((H + owned, rbuf))
        if self.rank > 0:
            bot = torch.from_numpy(np.ascontiguousarray(U[H: H + h]))
            rbuf = torch.empty_like(bot)
            reqs += [dist.isend(bot, self.rank - 1), dist.irecv(rbuf, self.rank - 1)]
            bufs.append((H - h, rbuf))
        for r in reqs:
            r.wait()
        for at, rb in bufs:
            U[at: at + h] = rb.numpy()

    def allgather_level(self, l, Fc):
        n = self.lv[l].n
        chunk = n // self.P
        mine = torch.from_numpy(np.ascontiguousarray(Fc[self.rank * chunk: (self.rank + 1) * chunk]))
        outs = [torch.empty_like(mine) for _ in range(self.P)]
        dist.all_gather(outs, mine)
        for p, o in enumerate(outs):
            Fc[p * chunk: (p + 1) * chunk] = o.numpy()

    # ---- level operators on slabs
    def smooth(self, l, U, F):
        L = self.lv[l]
        lo, hi = self.owned_local(l)
        rs = _rows(L)
        g0 = self.g0(l)
        if self.sm == "jacobi":
            self.exchange(l, U, 1)
            V = U.copy()
            for k in range(lo, hi):
                V[k][rs, 1:-1] = U[k][rs, 1:-1] + L.wd * (F[k][rs, 1:-1] - apply_A(L, U, k))
            U[lo:hi] = V[lo:hi]
            return
        # fused RBGS semantics: 2-plane halo, red on [lo-1, hi], black on [lo, hi)
        dist_l = self.part[l][2]
        self.exchange(l, U, 2)
        V = U.copy()
        rlo, rhi = (lo - 1, hi + 1) if dist_l else (lo, hi)
        for colour, (a, b) in ((0, (rlo, rhi)), (1, (lo, hi))):
            for k in range(a, b):
                gk = g0 + k
                if not (1 <= gk <= L.n - 1):
                    continue
                m = colour_mask(L, gk, colour)
                upd = V[k][rs, 1:-1] + L.wd * (F[k][rs, 1:-1] - apply_A(L, V, k))
                blk = V[k][rs, 1:-1]
                blk[m] = upd[m]
                V[k][rs, 1:-1] = blk
        U[lo:hi] = V[lo:hi]

    def resid_restrict(self, l, U, F, Fc):
        """f_{l+1}(owned coarse planes) = FW(f - A u)."""
        L, C = self.lv[l], self.lv[l + 1]
        rs = _rows(L)
        g0f, g0c = self.g0(l), self.g0(l + 1)
        self.exchange(l, U, 2)
        R = np.zeros_like(U)
        for k in range(1, U.shape[0] - 1):
            gk = g0f + k
            if 1 <= gk <= L.n - 1:
                R[k][rs, 1:-1] = F[k][rs, 1:-1] - apply_A(L, U, k)
        # owned coarse planes (first full level: this rank's chunk)
        if self.part[l + 1][2]:
            clo, chi = self.owned_local(l + 1)
        else:
            first, owned = self.part[l + 1][0], self.part[l + 1][1]
            chunk = C.n // self.P
            a = self.rank * chunk
            b = C.n + 1 if self.rank == self.P - 1 else a + chunk
            clo, chi = max(a, 1), min(b, C.n)
        two = self.dtype(2)
        scale = self.dtype(1 / 64 if self.dim == 3 else 1 / 16)
        for K in range(clo, chi):
            gK = g0c + K
            kf = 2 * gK - g0f
            ty = []
            for dz in (-1, 0, 1):
                P_ = R[kf + dz]
                if self.dim == 3:
                    tx = [(P_[2 * np.arange(1, C.cells[1]) + dy][:, 2 * np.arange(1, C.nx) - 1]
                           + P_[2 * np.arange(1, C.cells[1]) + dy][:, 2 * np.arange(1, C.nx) + 1])
                          + two * P_[2 * np.arange(1, C.cells[1]) + dy][:, 2 * np.arange(1, C.nx)]
                          for dy in (-1, 0, 1)]
                    ty.append((tx[0] + tx[2]) + two * tx[1])
                else:
                    row = P_[0]
                    I = np.arange(1, C.nx)
                    ty.append((row[2 * I - 1] + row[2 * I + 1]) + two * row[2 * I])
            t = (ty[0] + ty[2]) + two * ty[1]
            if self.dim == 3:
                Fc[K][1:-1, 1:-1] = t * scale
            else:
                Fc[K][0, 1:-1] = t * scale

    def prolong(self, l, E, U):
        L, C = self.lv[l], self.lv[l + 1]
        lo, hi = self.owned_local(l)
        g0f, g0c = self.g0(l), self.g0(l + 1)
        half = self.dtype(0.5)
        self.exchange(l + 1, E, 1)
        i = np.arange(1, L.nx)
        I, dx = i >> 1, i & 1
        rows = np.arange(1, L.rows - 1) if self.dim == 3 else np.array([0])
        J, dy = (rows >> 1, rows & 1) if self.dim == 3 else (np.array([0]), np.array([0]))
        for k in range(lo, hi):
            gk = g0f + k
            Z, dz = gk >> 1, gk & 1

            def V(Zg):
                P_ = E[Zg - g0c]
                vx0 = np.where(dx[None, :] == 1, half * (P_[J][:, I] + P_[J][:, I + 1]), P_[J][:, I])
                if self.dim == 2:
                    return vx0
                vx1 = np.where(dx[None, :] == 1, half * (P_[J + 1][:, I] + P_[J + 1][:, I + 1]), P_[J + 1][:, I])
                return np.where(dy[:, None] == 1, half * (vx0 + vx1), vx0)
            v = half * (V(Z) + V(Z + 1)) if dz else V(Z)
            U[k][rows[:, None], i[None, :]] = U[k][rows[:, None], i[None, :]] + v

    def norm(self, U, F):
        L = self.lv[0]
        lo, hi = self.owned_local(0)
        self.exchange(0, U, 1)
        s = 0.0
        for k in range(lo, hi):
            r = (F[k][_rows(L), 1:-1] - apply_A(L, U, k)).astype(np.float64)
            s += float(np.sum(r * r))   # summation order differs from the library: compared to 1e-12
        t = torch.tensor([s], dtype=torch.float64)
        outs = [torch.empty_like(t) for _ in range(self.P)]
        dist.all_gather(outs, t)
        tot = 0.0
        for o in outs:
            tot += float(o.item())
        return tot ** 0.5

    # ---- the cycle
    def tail(self, Fc_full):
        """Levels la..L-1 held in full: the oracle's own V-cycle from a zero guess."""
        la = self.la
        L = self.lv[la]
        cells = tuple(L.cells)
        cfg = orc.Config(dim=self.dim, cells=cells, levels=self.L - la,
                         smoother=orc.RBGS if self.sm == "rbgs" else orc.JACOBI, omega=self.omega, nu1=self.nu1,
                         nu2=self.nu2, h=tuple(h * 2.0 ** la for h in self.h0))
        O = orc.Oracle(cfg, self.dtype)
        f = Fc_full[:, 0, :] if self.dim == 2 else Fc_full
        f = np.ascontiguousarray(f)
        if self.L - la == 1:
            e = O.coarse_solve(f)
        else:
            e = O.vcycle(np.zeros_like(f), f)
        return e[:, None, :] if self.dim == 2 else e

    def vcycle(self, U0, F0):
        Us, Fs = [U0], [F0]
        self.exchange(0, F0, 1)
        for l in range(self.la):
            U, F = Us[l], Fs[l]
            for k in range(self.nu1):
                self.smooth(l, U, F)
            Fc = self.zeros(l + 1)
            self.resid_restrict(l, U, F, Fc)
            if l + 1 < self.la:
                self.exchange(l + 1, Fc, 1)
                Us.append(self.zeros(l + 1))
            else:
                self.allgather_level(l + 1, Fc)
            Fs.append(Fc)
        E = self.tail(Fs[self.la])
        Us.append(E)
        for l in range(self.la - 1, -1, -1):
            self.prolong(l, Us[l + 1], Us[l])
            for k in range(self.nu2):
                self.smooth(l, Us[l], Fs[l])
        return Us[0]
