"""Batch of independent proteins (BASELINE config 5; SURVEY.md §8e "replicas only").

Proteins are distributed over ranks round-robin (protein i -> rank i % world, no data-path
collective).  On one GPU the marches of a rank run concurrently on `streams` CUDA streams
(one host thread per stream; the C ABI releases the GIL), which fills the GPU the way one
batched launch would: a 97^3 sweep alone occupies only ~1.3 waves of the 148 SMs.  Results
(per protein, per variant: steps, divergence, max|u|, optional field checksum) are gathered
on every rank with one all_gather_object at the end.
"""

from __future__ import annotations

import ctypes
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .schemes import MarchConfig, march


@dataclass
class BatchItem:
    index: int
    n_atoms: int
    variant: str
    steps_taken: int
    diverged: bool
    max_abs: float
    device_s: float


def config5_problem(index: int, n_atoms: int):
    """Device-assembled config-5 protein `index` (seeded sizes from configs.batch_sizes)."""
    import paper_1410_2788_b200 as pb
    from .configs import batch_config, cubic_box, kappa_bar, synthetic_atoms
    from .problem import assemble_on_grid

    c = batch_config(index, n_atoms)
    atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
    lo, hi = cubic_box(atoms, c.n, c.h)
    system = pb.MolecularSystem([pb.Atom(a[:3], a[3], a[4]) for a in atoms], label=c.name)
    return c, assemble_on_grid(system, pb.make_grid(lo, hi, c.h), kappa_bar(c.ionic_strength),
                               c.eps_m, c.eps_s)


def rank_indices(count: int, rank: int, world: int):
    """Proteins of `rank` in a round-robin split of `count` over `world` ranks."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("need 0 <= rank < world")
    return list(range(rank, count, world))


def _max_abs(field) -> float:
    data = field.data if hasattr(field, "data") else field
    return float(np.max(np.abs(data)))


_STREAMS = {}


def _stream_pool(torch, count: int):
    """The same `count` CUDA streams on every call (per device): the caching allocator keeps
    blocks per stream, so fresh streams per batch would miss the blocks a previous batch (or
    the warm-up) left cached and allocate again inside the batch."""
    dev = torch.cuda.current_device()
    pool = _STREAMS.setdefault(dev, [])
    while len(pool) < count:
        pool.append(torch.cuda.Stream())
    return pool[:count]


def march_many(jobs, streams: int = 8, march_fn=None):
    """Run `jobs` = [(key, problem, MarchConfig)] concurrently on `streams` CUDA streams.
    Returns {key: MarchReport}.  `march_fn` (problem, config) -> report defaults to the
    device march."""
    if march_fn is not None:  # host-side test seam: sequential, no device
        return {key: march_fn(prob, cfg) for key, prob, cfg in jobs}
    torch = nat.torch_cuda()
    fn = march
    pool = _stream_pool(torch, max(1, streams))
    local = threading.local()
    lock = threading.Lock()
    counter = [0]

    def stream_of_thread():
        if not hasattr(local, "s"):
            with lock:
                local.s = pool[counter[0] % len(pool)]
                counter[0] += 1
        return local.s

    def run(job):
        key, prob, cfg = job
        s = stream_of_thread()
        with torch.cuda.stream(s):
            rep = fn(prob, cfg)
            s.synchronize()
        return key, rep

    with ThreadPoolExecutor(max_workers=len(pool)) as ex:
        return dict(ex.map(run, jobs))


class BatchMarch:
    """Batched march of independent problems on one grid shape (config 5: SURVEY.md §8e,
    "8 proteins per GPU, batched into one launch per sweep"): the problems' device buffers
    are stacked (one pitched grid each, `stride` elements apart) and every sweep of a step
    is ONE launch over the lines of all grids (pbg_plan_create_batch / pbg_plan_run_batch);
    divergence is tracked per grid.  Plans are prepared once per (variant, dt, alpha) and
    reused, like the reference's Stepper (schemes.py:188-262).  Results equal march() on
    each problem (same kernels and arithmetic)."""

    def __init__(self, problems):
        from .schemes import device_problem

        torch = nat.torch_cuda()
        if not problems:
            raise ValueError("no problems")
        g = problems[0].grid
        for q in problems:
            if q.grid.shape != g.shape or q.grid.h != g.h:
                raise ValueError("a batched march needs problems on one grid shape and h")
        dps = [device_problem(q) for q in problems]
        pal = dps[0].pal.as_tuple()
        for dp in dps[1:]:
            if dp.pal.as_tuple() != pal:
                raise ValueError("a batched march needs one coefficient palette (eps, kappa2)")
        pitch, nelem = nat.layout(g.shape)
        self.n = len(problems)
        self.stride = -(-nelem // pitch) * pitch  # >= one pitched grid, multiple of pitch
        self.problems = problems
        self.grid = g
        self.gs = dps[0].gs
        self.pal = dps[0].pal
        n, st = self.n, self.stride

        def stack(get, dtype):
            out = torch.zeros(n * st, dtype=dtype, device="cuda")
            for b, item in enumerate(get()):
                out[b * st:b * st + item.numel()].copy_(item)
            return out

        self.codes = stack(lambda: (dp.codes for dp in dps), torch.uint8)
        self.rho = stack(lambda: (dp.rho for dp in dps), torch.float64)
        self.bnd = stack(lambda: (dp.bnd for dp in dps), torch.float64)
        self.initial = stack(lambda: (q.initial._device() for q in problems), torch.float64)
        self._plans = {}

    def plan(self, variant, dt, alpha, aos_literal, threshold):
        key = (nat.VARIANT_IDS[variant], float(dt), float(alpha), bool(aos_literal),
               float(threshold))
        h = self._plans.get(key)
        if h is None:
            d = nat.PbgMarchDesc()
            d.grid, d.pal = self.gs, self.pal
            d.variant = key[0]
            d.aos_literal = 1 if aos_literal else 0
            d.dt, d.alpha, d.divergence_threshold = key[1], key[2], key[4]
            d.nsteps, d.check_divergence = 1, 1
            d.codes, d.rho = self.codes.data_ptr(), self.rho.data_ptr()
            d.initial = d.work[0] = d.work[1] = self.bnd.data_ptr()
            h = ctypes.c_void_p()
            nat.check(nat.lib().pbg_plan_create_batch(ctypes.byref(d), self.n, self.stride,
                                                      ctypes.byref(h), nat.stream_ptr()))
            self._plans[key] = h
        return h

    def march(self, config: MarchConfig, keep_fields: bool = True):
        """Batched march(); returns one MarchReport per problem (final fields as views of
        the batch's work buffer when keep_fields, else None) and the device seconds."""
        from .grid import ScalarField
        from .schemes import MarchReport, _resolve_alpha

        alphas = {_resolve_alpha(config.alpha, q) for q in self.problems}
        if len(alphas) != 1:
            raise ValueError("a batched march needs one alpha")
        alpha = alphas.pop()
        nsteps = max(1, int(round(config.T / config.dt)))
        h = self.plan(config.variant.value, config.dt, alpha,
                      config.aos_nonlinear == "literal", config.divergence_threshold)
        w0, w1 = self.bnd.clone(), self.bnd.clone()
        arr = ctypes.c_int32 * self.n
        taken, dstep, slot = arr(), arr(), arr()
        ms = ctypes.c_float()
        nat.check(nat.lib().pbg_plan_run_batch(h, nat.ptr(self.initial), nat.ptr(w0),
                                               nat.ptr(w1), nsteps, 1, taken, dstep, slot,
                                               ctypes.byref(ms), nat.stream_ptr()))
        reps = []
        st = self.stride
        _, nelem = nat.layout(self.grid.shape)
        for b in range(self.n):
            buf = w0 if slot[b] == 0 else w1
            final = None
            if keep_fields:
                final = ScalarField._from_device(self.grid,
                                                 buf[b * st:b * st + nelem].clone(),
                                                 dstep[b] != 0)
            reps.append(MarchReport(final=final, steps_taken=int(taken[b]),
                                    diverged=dstep[b] != 0,
                                    diverged_step=int(dstep[b]) or None,
                                    wall_time=ms.value / 1e3))
        return reps, ms.value / 1e3

    def __del__(self):
        try:
            for h in self._plans.values():
                nat.load_library().pbg_plan_destroy(h, None)
            self._plans.clear()
        except Exception:
            pass


def run_config5(rank: int = 0, world: int = 1, count: int = 64, variants=("AOSIE1", "LODIE2"),
                nsteps: int = 100, streams: int = 8, group=None, march_fn=None,
                problem_fn=None, batched: bool = True):
    """Config 5 on this rank's share of the batch; returns the items of all ranks sorted by
    protein and variant (gathered with all_gather_object when world > 1).  batched: one
    BatchMarch per variant (one launch per sweep for all the rank's proteins); otherwise
    one march per protein on `streams` concurrent CUDA streams."""
    from .configs import batch_sizes

    sizes = batch_sizes(count)
    make = problem_fn or config5_problem
    mine = rank_indices(count, rank, world)
    probs = {i: make(i, sizes[i]) for i in mine}
    if batched and march_fn is None:
        bm = BatchMarch([probs[i][1] for i in mine])
        c0 = probs[mine[0]][0]
        reports = {}
        for v in variants:
            reps, _ = bm.march(MarchConfig(dt=c0.dt, T=c0.dt * nsteps, variant=v))
            reports.update({(i, v): r for i, r in zip(mine, reps)})
        return _items(reports, sizes, world, group)
    jobs = []
    for i in mine:
        c, p = probs[i]
        for v in variants:
            jobs.append(((i, v), p, MarchConfig(dt=c.dt, T=c.dt * nsteps, variant=v)))
    if march_fn is None:  # device views built once on the default stream, before the threads
        from .schemes import device_problem

        for i in mine:
            device_problem(probs[i][1])
        nat.torch_cuda().cuda.synchronize()
    reports = march_many(jobs, streams, march_fn)
    return _items(reports, sizes, world, group)


def _items(reports, sizes, world, group):
    items = []
    for (i, v), rep in sorted(reports.items()):
        items.append(BatchItem(i, sizes[i], v, rep.steps_taken, rep.diverged,
                               _max_abs(rep.final), rep.wall_time))
    if world > 1:
        import torch.distributed as dist

        gathered = [None] * world
        dist.all_gather_object(gathered, items, group=group)
        items = [it for part in gathered for it in part]
    return sorted(items, key=lambda it: (it.index, it.variant))


__all__ = ["BatchItem", "BatchMarch", "config5_problem", "rank_indices", "march_many",
           "run_config5"]
