"""Batch of independent proteins (BASELINE config 5; SURVEY.md §8e "replicas only").

Proteins are distributed over ranks round-robin (protein i -> rank i % world, no data-path
collective).  On one GPU the marches of a rank run concurrently on `streams` CUDA streams
(one host thread per stream; the C ABI releases the GIL), which fills the GPU the way one
batched launch would: a 97^3 sweep alone occupies only ~1.3 waves of the 148 SMs.  Results
(per protein, per variant: steps, divergence, max|u|, optional field checksum) are gathered
on every rank with one all_gather_object at the end.
"""

from __future__ import annotations

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


def run_config5(rank: int = 0, world: int = 1, count: int = 64, variants=("AOSIE1", "LODIE2"),
                nsteps: int = 100, streams: int = 8, group=None, march_fn=None,
                problem_fn=None):
    """Config 5 on this rank's share of the batch; returns the items of all ranks sorted by
    protein and variant (gathered with all_gather_object when world > 1)."""
    from .configs import batch_sizes

    sizes = batch_sizes(count)
    make = problem_fn or config5_problem
    mine = rank_indices(count, rank, world)
    probs = {i: make(i, sizes[i]) for i in mine}
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


__all__ = ["BatchItem", "config5_problem", "rank_indices", "march_many", "run_config5"]
