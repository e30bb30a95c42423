"""TEST INFRASTRUCTURE: the time-slab STMG algorithm on the CPU oracle kernels,
one torch.distributed (gloo) process per rank.

Each rank holds full-size numpy level vectors but owns only its slab rows (the
partition comes from the product's stmg_dist_partition); every row outside
[lo - 1, hi + 1) is poisoned with NaN after each step, so any read outside
the slab plus one ghost level per side shows up in the result.  Ghost levels
move with point-to-point sends, norms with all_reduce, the first gathered
level's right-hand side is gathered to rank 0 (which runs the tail V-cycle on
full vectors) and the correction is broadcast — the same schedule as
csrc/stmg_dist.cuh.  The iterate after every cycle must equal the
single-domain oracle's bit for bit.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def _rows(b, g):
    return int(b[g]), int(b[g + 1])


class SlabSim:
    def __init__(self, hp, dirs, shapes, bounds, lg, rank, world, nu, omega=0.5):
        self.hp, self.dirs, self.shapes = hp, list(dirs), shapes
        self.bounds, self.lg, self.rank, self.world = bounds, lg, rank, world
        self.nu, self.omega = nu, omega
        self.L = len(shapes)

    def nn(self, l):
        return self.shapes[l][0] + 1

    def nt(self, l):
        return self.shapes[l][1]

    def poison(self, l, v):
        lo, hi = _rows(self.bounds[l], self.rank)
        V = v.reshape(self.nt(l) + 1, self.nn(l))
        V[: max(lo - 1, 0)] = np.nan
        V[hi + 1:] = np.nan
        return v

    def keep_own(self, l, new, old):
        lo, hi = _rows(self.bounds[l], self.rank)
        out = old.copy().reshape(self.nt(l) + 1, self.nn(l))
        out[lo:hi] = new.reshape(self.nt(l) + 1, self.nn(l))[lo:hi]
        return self.poison(l, out.reshape(-1))

    def exchange(self, l, v):
        """first own row -> rank-1's trailing ghost, last own row -> rank+1's leading ghost"""
        g, W, nn = self.rank, self.world, self.nn(l)
        b = self.bounds[l]
        V = v.reshape(self.nt(l) + 1, nn)
        ops, recv = [], []
        if g > 0:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(V[b[g]].copy()), g - 1))
            buf = torch.empty(nn, dtype=torch.float64)
            ops.append(dist.P2POp(dist.irecv, buf, g - 1))
            recv.append((b[g] - 1, buf))
        if g < W - 1:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(V[b[g + 1] - 1].copy()), g + 1))
            buf = torch.empty(nn, dtype=torch.float64)
            ops.append(dist.P2POp(dist.irecv, buf, g + 1))
            recv.append((b[g + 1], buf))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        for row, buf in recv:
            V[row] = buf.numpy()
        return v

    def sweep(self, l, f, x):
        x = self.exchange(l, x)
        return self.keep_own(l, self.hp.sweeps(l, f, x, 1, self.omega), x)

    # ---- tail (levels >= lg) on full vectors, rank 0 only: proj/src/multigrid.cpp:184-208
    def tail_vcycle(self, l, f):
        hp = self.hp
        if l == self.L - 1:
            return hp.coarsest(f)
        x = np.zeros_like(f)
        for _ in range(self.nu):
            x = hp.sweeps(l, f, x, 1, self.omega)
        fc = hp.restrict(l, hp.residual(l, f, x))
        xc = self.tail_vcycle(l + 1, fc)
        x = hp.prolong_add(l, xc, x)
        for _ in range(self.nu):
            x = hp.sweeps(l, f, x, 1, self.omega)
        return x

    def gathered_rows(self, g):
        lg = self.lg
        b = self.bounds[lg - 1]
        if self.dirs[lg - 1] == 1:
            lo = int(b[g]) // 2
            hi = self.nt(lg) + 1 if g == self.world - 1 else int(b[g + 1]) // 2
            return lo, hi
        return int(b[g]), int(b[g + 1])

    def vcycle(self, l, f, x):
        """Distributed V-cycle at level l < lg; returns this rank's x (slab rows valid)."""
        hp = self.hp
        for _ in range(self.nu):
            x = self.sweep(l, f, x)
        x = self.exchange(l, x)
        r = hp.residual(l, f, x)
        fc_full = hp.restrict(l, r)  # only this rank's coarse rows are meaningful
        if l + 1 < self.lg:
            fc = self.keep_own(l + 1, fc_full, np.full_like(fc_full, np.nan))
            xc = self.vcycle(l + 1, fc, self.poison(l + 1, np.zeros_like(fc)))
            xc = self.exchange(l + 1, xc)
        else:
            nnc = self.nn(l + 1)
            lo, hi = self.gathered_rows(self.rank)
            mine = torch.from_numpy(fc_full.reshape(-1, nnc)[lo:hi].copy())
            if self.rank == 0:
                F = fc_full.reshape(-1, nnc).copy()
                for g in range(1, self.world):
                    glo, ghi = self.gathered_rows(g)
                    buf = torch.empty((ghi - glo) * nnc, dtype=torch.float64)
                    dist.recv(buf, g)
                    F[glo:ghi] = buf.numpy().reshape(ghi - glo, nnc)
                xc = self.tail_vcycle(l + 1, F.reshape(-1))
                t = torch.from_numpy(xc.copy())
            else:
                dist.send(mine.reshape(-1), 0)
                t = torch.empty(fc_full.size, dtype=torch.float64)
            dist.broadcast(t, 0)
            xc = t.numpy()
        x = self.keep_own(l, hp.prolong_add(l, xc, x), x)
        for _ in range(self.nu):
            x = self.sweep(l, f, x)
        return x

    def norm(self, b0, x):
        x = self.exchange(0, x)
        r = self.hp.residual(0, b0, x)
        lo, hi = _rows(self.bounds[0], self.rank)
        own = r.reshape(self.nt(0) + 1, self.nn(0))[lo:hi]
        t = torch.tensor([float(np.sum(own * own))], dtype=torch.float64)
        dist.all_reduce(t)
        return float(np.sqrt(t.item()))

    def solve(self, b, tol, max_cycles):
        x = self.poison(0, np.zeros_like(b))
        lo, hi = _rows(self.bounds[0], self.rank)
        bb = b.reshape(self.nt(0) + 1, self.nn(0))[lo:hi]
        t = torch.tensor([float(np.sum(bb * bb))], dtype=torch.float64)
        dist.all_reduce(t)
        nb = float(np.sqrt(t.item()))
        hist = [self.norm(b, x) / nb]
        cycles = 0
        iterates = []
        while hist[-1] >= tol and cycles < max_cycles:
            x = self.vcycle(0, b, x)
            cycles += 1
            iterates.append(x.copy())
            hist.append(self.norm(b, x) / nb)
        return x, hist, cycles, iterates
