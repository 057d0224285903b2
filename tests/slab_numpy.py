"""Test infrastructure: a numpy partition for `paper_1410_2788_b200.slab.run_slabs`.

It restates the slab-decomposed LOD step (include/pbg.h, pbg_slab_*) on the host with the
oracle's Thomas solver, so the multi-rank orchestration (exchange order, partition ranges,
interface algebra, divergence agreement) runs on CPU under gloo and can be checked against
the oracle's single-domain march.  Exchange block per rank: four (n1-2)*(n2-2) planes and a
divergence slot."""

from __future__ import annotations

import numpy as np
import torch

from oracle import pbs_oracle as O

NO_DIV = 2 ** 31 - 1


def interface_solve(G, Q, rank, nranks):
    """Chunk end values per line (same recurrence as k_slab_interface).
    G[r] = (g_f, g_l), Q[r] = (p_f, p_l, q_f, q_l); returns (L_{rank-1}, F_{rank+1})."""
    c = d = 0.0
    e, hh, cc, dd = [], [], [], []
    for r in range(nranks):
        gf, gl = G[r]
        pf, pl = (Q[r][0], Q[r][1]) if r > 0 else (0.0, 0.0)
        qf, ql = (Q[r][2], Q[r][3]) if r + 1 < nranks else (0.0, 0.0)
        inv = 1.0 / (1.0 - pf * d)
        e.append((gf + pf * c) * inv)
        hh.append(qf * inv)
        c, d = gl + pl * c + pl * d * e[-1], pl * d * hh[-1] + ql
        cc.append(c)
        dd.append(d)
    F = 0.0
    Lprev = Fnext = None
    for r in range(nranks - 1, -1, -1):
        Fr = e[r] + hh[r] * F
        if r == rank + 1:
            Fnext = Fr
        if r == rank - 1:
            Lprev = cc[r] + dd[r] * F
        F = Fr
    return Lprev, Fnext


class NumpySlab:
    nchunks = 1

    def phase(self, phase, chunk):  # one exchange block for every phase
        return 0, self.send.numel()

    def step_a_chunk(self, c):
        self.step_a()

    def __init__(self, p: O.OProblem, variant, dt, T, rank, nranks, first, stop, recv=None,
                 threshold=1e12):
        fam, mult, self.cn, _ = O.PLANS[variant]
        assert fam in ("lod1", "lod2")
        self.fam = fam
        self.rank, self.nranks, self.first, self.stop = rank, nranks, first, stop
        self.threshold = threshold
        g = p.grid
        n0, n1, n2 = g.shape
        sl = slice(first - 1, stop + 1)
        self.lg = O.OGrid((g.lo[0] + (first - 1) * g.h, g.lo[1], g.lo[2]), g.h,
                          (stop - first + 2, n1, n2))
        r = p.region
        self.region = O.ORegion(r.eps_node[sl], (r.eps_half[0][first - 1:stop], r.eps_half[1][sl],
                                                 r.eps_half[2][sl]), r.kappa2[sl])
        self.bvals = p.bvals[sl].copy()
        self.rho = p.rho[sl]
        self.u = p.initial[sl].copy()
        self.dta = dt / p.alpha
        self.f = mult * self.dta
        self.cn_c = mult * self.dta / g.h ** 2
        self.decay = np.exp(-self.region.kappa2 * self.dta)
        self.fac = [None] + [O.LineFactors(self.lg, self.region, self.bvals, a, self.f)
                             for a in (1, 2)]
        self.P = (n1 - 2) * (n2 - 2)
        self.send = torch.zeros(4 * self.P + 1, dtype=torch.float64)
        self.recv = recv if recv is not None else torch.zeros(nranks * (4 * self.P + 1),
                                                              dtype=torch.float64)
        self.dflag = NO_DIV
        self.step = 0
        # static responses of the chunk end rows to unit ghost values
        zero = np.zeros((self.lg.shape[0] - 2, n1 - 2, n2 - 2))
        for side in (0, 1):
            b = np.zeros(self.lg.shape)
            b[0 if side == 0 else -1] = 1.0
            x = O.LineFactors(self.lg, self.region, b, 0, self.f).solve(zero)
            self._put(2 * side, x[0])
            self._put(2 * side + 1, x[-1])
        self.send[4 * self.P] = NO_DIV

    # exchange block helpers
    def _put(self, k, plane):
        self.send[k * self.P:(k + 1) * self.P] = torch.from_numpy(np.ascontiguousarray(plane).ravel())

    def _blk(self, r, k):
        E = 4 * self.P + 1
        return self.recv[r * E + k * self.P:r * E + (k + 1) * self.P].numpy().reshape(
            self.lg.shape[1] - 2, self.lg.shape[2] - 2)

    def _flag(self, r):
        return int(self.recv[r * (4 * self.P + 1) + 4 * self.P].item())

    def setup(self):
        N = self.nranks
        self.Q = [[self._blk(r, k).copy() for k in range(4)] for r in range(N)]

    def halo_pack(self):
        self._put(0, self.u[1, 1:-1, 1:-1])
        self._put(1, self.u[-2, 1:-1, 1:-1])

    def halo_unpack(self):
        if self.rank > 0:
            self.u[0, 1:-1, 1:-1] = self._blk(self.rank - 1, 1)
        if self.rank + 1 < self.nranks:
            self.u[-1, 1:-1, 1:-1] = self._blk(self.rank + 1, 0)

    def _rhs0(self):
        if self.fam == "lod2":
            w = self.u + self.dta * self.rho
        else:
            w = O.sinh_flow(self.u, self.decay)
        rhs = w[O.INT]
        if self.cn:
            rhs = rhs + self.cn_c * O.delta2(w, self.region.eps_half[0], 0)
        return rhs

    def _ghosts(self, lo=None, hi=None):
        b = self.bvals.copy()
        if self.rank > 0:
            b[0, 1:-1, 1:-1] = 0.0 if lo is None else lo
        if self.rank + 1 < self.nranks:
            b[-1, 1:-1, 1:-1] = 0.0 if hi is None else hi
        return b

    def step_a(self):
        x = O.LineFactors(self.lg, self.region, self._ghosts(), 0, self.f).solve(self._rhs0())
        self._put(0, x[0])
        self._put(1, x[-1])
        self.send[4 * self.P] = self.dflag

    def step_b(self):
        N = self.nranks
        for r in range(N):
            self.dflag = min(self.dflag, self._flag(r))
        if self.dflag < self.step + 1:
            return  # an earlier step diverged somewhere: every rank stops
        G = [(self._blk(r, 0), self._blk(r, 1)) for r in range(N)]
        lo, hi = interface_solve(G, self.Q, self.rank, N)
        x = O.LineFactors(self.lg, self.region, self._ghosts(lo, hi), 0, self.f).solve(
            self._rhs0())
        w = np.empty(self.lg.shape)
        w[O.INT] = x
        O.apply_faces(w, self.bvals)
        for a in (1, 2):
            rhs = w[O.INT]
            if self.cn:
                rhs = rhs + self.cn_c * O.delta2(w, self.region.eps_half[a], a)
            w2 = np.empty(self.lg.shape)
            w2[O.INT] = self.fac[a].solve(rhs)
            O.apply_faces(w2, self.bvals)
            w = w2
        if self.fam == "lod2":
            w = O.sinh_flow(w, self.decay)
            O.apply_faces(w, self.bvals)
        else:
            w = w + self.dta * self.rho
        self.step += 1
        own = w[1:-1]
        amax = np.max(np.abs(own))
        if not np.isfinite(amax) or amax > self.threshold:
            self.dflag = min(self.dflag, self.step)
        # keep the ghost planes of the previous state (only CN reads them, after a halo)
        w[0], w[-1] = self.u[0], self.u[-1]
        self.u = w

    def flag_pack(self):
        self.send[4 * self.P] = self.dflag

    def finish(self):
        d = min([self.dflag] + [self._flag(r) for r in range(self.nranks)])
        taken = self.step if d == NO_DIV else min(d, self.step)
        return taken, (None if d == NO_DIV else taken), self.u
