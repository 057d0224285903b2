"""Slab-decomposed march across ranks.

The grid is split along axis 0 into contiguous slabs of interior planes, one per rank
(`slab_ranges`).  Every step runs the rank-local phase A (chunk solve of the axis-0 lines
with zero ghost values, end rows only), one all-gather of the chunk end rows, and phase B
(interface solve, axis-0 chunk sweep with the neighbours' end values, local axis-1/2
sweeps with the fused source and flow).  `include/pbg.h` (pbg_slab_*) documents the
algebra; the result equals the single-device march up to reassociation.

Exchanges are pluggable:
  * `GroupExchange`  one partition per process, `torch.distributed` all-gather (NCCL over
    NVLink on the GPU box; gloo in the CPU tests of the orchestration);
  * `LocalExchange`  several partitions in one process on one GPU, exchange by device copy
    (how the multi-rank algebra is tested with a single GPU).

The reference (pbsplit) is single-process; this module has no reference counterpart and
only the LOD variants LODIE1, LODIE2 and LODCN2 shard (AOS/MAOS/LODCN1 stay single-device).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .grid import ScalarField
from .schemes import MarchConfig, MarchReport, _resolve_alpha, device_problem, parse_variant

SLAB_SCHEMES = ("LODIE1", "LODIE2", "LODCN2")
MAX_RANKS = 16


def slab_ranges(n0: int, nranks: int, cost=None):
    """Owned global interior planes [first, stop) per rank, contiguous.  Without `cost` the
    sizes differ by <= 1.  With `cost` (one positive weight per interior plane, e.g.
    `plane_costs`) the split minimises the largest per-rank cost sum: planes through the
    molecule sweep slower (general segments, cyclic-reduction tiles, the wider flow tiers),
    so the ranks holding it take fewer planes."""
    m = int(n0) - 2
    if not (1 <= nranks <= MAX_RANKS):
        raise ValueError(f"nranks must be in 1..{MAX_RANKS}")
    if m < nranks:
        raise ValueError(f"{m} interior planes cannot be split over {nranks} ranks")
    if cost is None:
        base, extra = divmod(m, nranks)
        counts = [base + (1 if r < extra else 0) for r in range(nranks)]
    else:
        c = np.asarray(cost, dtype=np.float64)
        if c.shape != (m,) or not np.all(c > 0) or not np.all(np.isfinite(c)):
            raise ValueError("cost must hold one positive finite weight per interior plane")
        counts = _balanced_counts(c, nranks)
    out, first = [], 1
    for cnt in counts:
        out.append((first, first + cnt))
        first += cnt
    return out


def _balanced_counts(c, nranks):
    """Contiguous split of the weights c into nranks non-empty parts with the smallest
    possible largest part sum (bisection on the capacity, greedy fill)."""
    m = len(c)

    def fill(cap):
        counts, i = [], 0
        for r in range(nranks):
            left = nranks - r - 1  # parts that still need a plane each
            acc, n = 0.0, 0
            while i < m - left and (n == 0 or acc + c[i] <= cap):
                acc += c[i]
                i += 1
                n += 1
            counts.append(n)
        return counts if i == m else None

    lo, hi = float(c.max()), float(c.sum())
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if fill(mid) is None:
            lo = mid
        else:
            hi = mid
    return fill(hi)


def slab_beta():
    """Relative extra cost of a plane that is all solute, for `plane_costs` (measured on
    config 4: planes with a ~10% solute cross-section run ~1.6x slower; PBG_SLAB_BETA
    overrides, 0 = equal plane counts)."""
    import os

    return float(os.environ.get("PBG_SLAB_BETA", "6.0"))


def plane_costs(dp, beta=None):
    """Per interior plane weight 1 + beta * (solute fraction of the plane), from the device
    region codes (bit 0 = solute).  None when beta == 0."""
    beta = slab_beta() if beta is None else float(beta)
    if beta == 0.0:
        return None
    n0, n1, n2 = dp.grid.shape
    pitch, _ = nat.layout(dp.grid.shape)
    plane = n1 * pitch
    sol = (dp.codes[:n0 * plane].view(n0, plane) & 1).sum(dim=1, dtype=nat.torch_cuda().int64)
    frac = sol[1:n0 - 1].double().cpu().numpy() / float((n1 - 2) * (n2 - 2))
    return 1.0 + beta * frac


SETUP, HALO, STEP = 0, 1, 2  # exchange phases (include/pbg.h PBG_SLAB_*)


def run_slabs(parts, exchange, nsteps: int, cn: bool):
    """Drive the partitions of this process through setup, `nsteps` steps and the final flag
    agreement.  `parts` are this process's partitions (all of them for LocalExchange, one
    for GroupExchange); each exposes `send`/`recv` buffers, `phase(phase, chunk)` ->
    (offset, count) of the exchanged part of send, `nchunks`, and the phase calls.  Phase A
    runs chunk by chunk; each chunk's all-gather is issued as soon as the chunk is done, so
    (with an asynchronous exchange) it overlaps phase A of the next chunk."""
    exchange.gather(parts, *parts[0].phase(SETUP, 0))  # static responses (from creation)
    for p in parts:
        p.setup()
    nc = parts[0].nchunks
    for _ in range(nsteps):
        if cn:
            for p in parts:
                p.halo_pack()
            exchange.gather(parts, *parts[0].phase(HALO, 0))
            for p in parts:
                p.halo_unpack()
        pending = []
        for c in range(nc):
            for p in parts:
                p.step_a_chunk(c)
            pending.append(exchange.gather(parts, *parts[0].phase(STEP, c), async_op=True))
        for w in pending:
            if w is not None:
                w.wait()
        for p in parts:
            p.step_b()
    for p in parts:
        p.flag_pack()
    exchange.gather(parts, *parts[0].phase(STEP, 0))
    return [p.finish() for p in parts]


class LocalExchange:
    """All partitions live in this process and share one `recv` buffer (device copies on
    the current stream, in order)."""

    def gather(self, parts, offset, count, async_op=False):
        recv = parts[0].recv
        base = len(parts) * offset
        for r, p in enumerate(parts):
            recv[base + r * count:base + (r + 1) * count].copy_(p.send[offset:offset + count])
        return None


class GroupExchange:
    """One partition per process; all-gather over a torch.distributed group (NCCL: runs on
    the communicator's stream, ordered after the work already queued on the current stream,
    so an async gather overlaps the kernels launched after it)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.nccl = dist.get_backend(group) == "nccl"

    def gather(self, parts, offset, count, async_op=False):
        (p,) = parts
        n = self.dist.get_world_size(self.group)
        dst = p.recv[n * offset:n * (offset + count)]
        src = p.send[offset:offset + count]
        if self.nccl:
            return self.dist.all_gather_into_tensor(dst, src, group=self.group,
                                                    async_op=async_op)
        return self.dist.all_gather(list(dst.view(n, -1).unbind(0)), src, group=self.group,
                                    async_op=async_op)


class DeviceSlab:
    """One rank's slab on the device: local copies of the global buffers' planes
    [first-1, stop] (same pitched layout) and a native pbg_slab handle."""

    def __init__(self, dp, variant, dt, alpha, nsteps, threshold, rank, nranks, first, stop,
                 initial_dev, recv=None, check_divergence=True):
        torch = nat.torch_cuda()
        self.lib = nat.lib()
        g = dp.grid
        n0, n1, n2 = g.shape
        pitch, _ = nat.layout(g.shape)
        plane = n1 * pitch
        self.rank, self.nranks, self.first, self.stop = rank, nranks, first, stop
        self.plane = plane
        nl0 = stop - first + 2
        lgs = nat.PbgGrid()
        for a in range(3):
            lgs.n[a] = dp.gs.n[a]
            lgs.lo[a] = dp.gs.lo[a]
        lgs.n[0] = nl0
        lgs.lo[0] = dp.gs.lo[0] + (first - 1) * dp.gs.h
        lgs.pitch = dp.gs.pitch
        lgs.h = dp.gs.h
        self.gs = lgs
        nloc = nl0 * plane + 64
        lo, hi = (first - 1) * plane, (stop + 1) * plane

        def slab(t):
            out = torch.zeros(nloc, dtype=t.dtype, device=t.device)
            out[:hi - lo].copy_(t[lo:hi])
            return out

        self.codes = slab(dp.codes)
        self.rho = slab(dp.rho)
        self.work = (slab(dp.bnd), slab(dp.bnd))
        self.initial = slab(initial_dev)
        E = int(self.lib.pbg_slab_exchange_elems(ctypes.byref(lgs)))
        self.send = torch.empty(E, dtype=torch.float64, device="cuda")
        self.recv = recv if recv is not None else torch.empty(nranks * E, dtype=torch.float64,
                                                              device="cuda")
        d = nat.PbgMarchDesc()
        d.grid = lgs
        d.pal = dp.pal
        d.variant = nat.VARIANT_IDS[variant]
        d.aos_literal = 0
        d.dt = float(dt)
        d.alpha = float(alpha)
        d.divergence_threshold = float(threshold)
        d.nsteps = int(nsteps)
        d.check_divergence = 1 if check_divergence else 0
        d.codes = self.codes.data_ptr()
        d.rho = self.rho.data_ptr()
        d.initial = self.initial.data_ptr()
        d.work[0] = self.work[0].data_ptr()
        d.work[1] = self.work[1].data_ptr()
        self.desc = d
        self.handle = ctypes.c_void_p()
        nat.check(self.lib.pbg_slab_create(ctypes.byref(d), int(rank), int(nranks),
                                           nat.ptr(self.send), nat.ptr(self.recv),
                                           ctypes.byref(self.handle), nat.stream_ptr()))

    def _call(self, fn):
        nat.check(fn(self.handle, nat.stream_ptr()))

    def setup(self):
        self._call(self.lib.pbg_slab_setup)

    def halo_pack(self):
        self._call(self.lib.pbg_slab_halo_pack)

    def halo_unpack(self):
        self._call(self.lib.pbg_slab_halo_unpack)

    def step_a(self):
        self._call(self.lib.pbg_slab_step_a)

    def step_a_chunk(self, c):
        nat.check(self.lib.pbg_slab_step_a_chunk(self.handle, int(c), nat.stream_ptr()))

    @property
    def nchunks(self):
        return int(self.lib.pbg_slab_nchunks(self.handle))

    def phase(self, phase, chunk):
        off, cnt = ctypes.c_int64(), ctypes.c_int64()
        nat.check(self.lib.pbg_slab_phase(self.handle, int(phase), int(chunk),
                                          ctypes.byref(off), ctypes.byref(cnt)))
        return int(off.value), int(cnt.value)

    def step_b(self):
        self._call(self.lib.pbg_slab_step_b)

    def flag_pack(self):
        self._call(self.lib.pbg_slab_flag_pack)

    def finish(self):
        taken, dstep, slot = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        nat.check(self.lib.pbg_slab_finish(self.handle, ctypes.byref(taken),
                                           ctypes.byref(dstep), ctypes.byref(slot),
                                           nat.stream_ptr()))
        return taken.value, (dstep.value or None), self.work[slot.value]

    def owned(self, local_field):
        """The owned planes of a local field (flat view)."""
        return local_field[self.plane:(self.stop - self.first + 1) * self.plane]

    def close(self):
        if self.handle:
            self.lib.pbg_slab_destroy(self.handle, nat.stream_ptr())
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _check_variant(config: MarchConfig):
    v = parse_variant(config.variant).value
    if v not in SLAB_SCHEMES:
        raise NotImplementedError(f"{v} does not shard across ranks; slab schemes: "
                                  f"{', '.join(SLAB_SCHEMES)}")
    return v


def make_slabs(problem, config: MarchConfig, ranks, nranks: int, recv=None,
               initial_dev=None, beta=None):
    """DeviceSlab objects for the given ranks of an `nranks`-way split of `problem`; the
    split is cost weighted (`plane_costs`; every rank derives the same ranges from the same
    region codes)."""
    v = _check_variant(config)
    dp = device_problem(problem)
    nsteps = max(1, int(round(config.T / config.dt)))
    init = initial_dev if initial_dev is not None else problem.initial._device()
    rng = slab_ranges(problem.grid.shape[0], nranks, plane_costs(dp, beta))
    return [DeviceSlab(dp, v, config.dt, _resolve_alpha(config.alpha, problem), nsteps,
                       config.divergence_threshold, r, nranks, rng[r][0], rng[r][1], init,
                       recv=recv) for r in ranks], nsteps, v.startswith("LODCN")


def march_partitioned(problem, config: MarchConfig, nparts: int, beta=None) -> MarchReport:
    """march() with the grid split into `nparts` slabs inside this process (one GPU,
    exchange by device copy).  Same result as march() up to reassociation.  `beta`: weight
    of the cost-balanced split (`plane_costs`; 0 = equal plane counts)."""
    torch = nat.torch_cuda()
    _check_variant(config)
    g = problem.grid
    E = int(nat.lib().pbg_slab_exchange_elems(ctypes.byref(_local_gs(g, 1))))
    recv = torch.empty(nparts * E, dtype=torch.float64, device="cuda")
    parts, nsteps, cn = make_slabs(problem, config, range(nparts), nparts, recv=recv,
                                   beta=beta)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = run_slabs(parts, LocalExchange(), nsteps, cn)
    e1.record()
    torch.cuda.synchronize()
    final = device_problem(problem).bnd.clone()
    for p, (_, _, f) in zip(parts, res):
        plane = p.plane
        final[p.first * plane:p.stop * plane].copy_(p.owned(f))
    taken, dstep = res[0][0], res[0][1]
    for p in parts:
        p.close()
    diverged = dstep is not None
    return MarchReport(final=ScalarField._from_device(g, final, diverged), steps_taken=taken,
                       diverged=diverged, diverged_step=dstep,
                       wall_time=e0.elapsed_time(e1) / 1e3)


def _local_gs(grid, nl0):
    gs = nat.grid_struct(grid)
    gs.n[0] = nl0
    return gs


def march_distributed(problem, config: MarchConfig, group=None):
    """march() with one slab per torch.distributed rank (NCCL on the GPU box).  Returns
    (steps_taken, diverged_step, the rank's DeviceSlab, its final local field)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    (part,), nsteps, cn = make_slabs(problem, config, [rank], world)
    taken, dstep, final = run_slabs([part], GroupExchange(group), nsteps, cn)[0]
    return taken, dstep, part, final


__all__ = ["SLAB_SCHEMES", "slab_ranges", "plane_costs", "run_slabs", "LocalExchange", "GroupExchange",
           "DeviceSlab", "make_slabs", "march_partitioned", "march_distributed"]
