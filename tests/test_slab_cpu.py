"""Slab decomposition across ranks, CPU: the orchestration of
paper_1410_2788_b200.slab.run_slabs with numpy partitions (tests/slab_numpy.py), in one
process and over a world_size-2 gloo group, against the reference's golden marches."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1410_2788_b200.slab import GroupExchange, LocalExchange, run_slabs, slab_ranges
from tests.helpers import golden, oracle_protein
from tests.slab_numpy import NumpySlab

TOL = 1e-12


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def test_slab_ranges_cover_interior_contiguously():
    for n0 in (3, 10, 65, 513):
        for n in range(1, min(16, n0 - 2) + 1):
            rng = slab_ranges(n0, n)
            assert rng[0][0] == 1 and rng[-1][1] == n0 - 1
            assert all(a[1] == b[0] for a, b in zip(rng, rng[1:]))
            sizes = [b - a for a, b in rng]
            assert min(sizes) >= 1 and max(sizes) - min(sizes) <= 1
    assert [b - a for a, b in slab_ranges(513, 8)] == [64] * 7 + [63]
    # cost-weighted split: contiguous cover, the expensive planes end up in smaller slabs,
    # the largest per-rank cost is optimal for this small case, uniform weights = equal counts
    cost = np.ones(30)
    cost[12:18] = 5.0
    rng = slab_ranges(32, 4, cost)
    assert rng[0][0] == 1 and rng[-1][1] == 31
    assert all(rng[r][1] == rng[r + 1][0] for r in range(3))
    sums = [cost[a - 1:b - 1].sum() for a, b in rng]
    assert max(sums) <= 15.0 + 1e-9  # total 54 over 4 ranks: 13.5 is a lower bound, 15 reachable
    assert [b - a for a, b in slab_ranges(32, 4, np.ones(30))] in ([8, 8, 7, 7], [8, 7, 8, 7],
                                                                  [8, 8, 8, 6], [7, 8, 8, 7])
    assert all(b > a for a, b in slab_ranges(7, 5, np.array([9.0, 1, 1, 1, 1])))
    with pytest.raises(ValueError):
        slab_ranges(32, 4, np.ones(29))
    with pytest.raises(ValueError):
        slab_ranges(5, 4)
    with pytest.raises(ValueError):
        slab_ranges(100, 17)


def _parts_local(p, variant, dt, T, nparts, threshold=1e12):
    rng = slab_ranges(p.grid.shape[0], nparts)
    E = 4 * (p.grid.shape[1] - 2) * (p.grid.shape[2] - 2) + 1
    recv = torch.zeros(nparts * E, dtype=torch.float64)
    return [NumpySlab(p, variant, dt, T, r, nparts, a, b, recv=recv, threshold=threshold)
            for r, (a, b) in enumerate(rng)]


def _assemble(p, parts, results):
    out = p.bvals.copy()
    for part, (_, _, u) in zip(parts, results):
        out[part.first:part.stop] = u[1:-1]
    return out


@pytest.mark.parametrize("variant", ["LODIE1", "LODIE2", "LODCN2"])
@pytest.mark.parametrize("nparts", [1, 3, 4])
def test_partitioned_march_matches_reference_golden(variant, nparts):
    d = golden("march_variants")
    p = oracle_protein(d)
    dt, T = float(d["dt"]), float(d["T"])
    nsteps = max(1, int(round(T / dt)))
    parts = _parts_local(p, variant, dt, T, nparts)
    res = run_slabs(parts, LocalExchange(), nsteps, variant.startswith("LODCN"))
    assert all(r[0] == nsteps and r[1] is None for r in res)
    assert _rel(_assemble(p, parts, res), d[variant]) <= TOL


def test_partitioned_divergence_agrees_over_ranks():
    d = golden("march_variants")
    p = oracle_protein(d)
    parts = _parts_local(p, "LODIE1", 0.3, 3.0, 3, threshold=2.0e3)
    res = run_slabs(parts, LocalExchange(), 10, False)
    taken = {r[0] for r in res}
    dstep = {r[1] for r in res}
    assert taken == {int(d["div_steps"])} and dstep == {int(d["div_step"])}
    assert _rel(_assemble(p, parts, res), d["div_final"]) <= TOL


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, variant, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d = golden("march_variants")
        p = oracle_protein(d)
        dt, T = float(d["dt"]), float(d["T"])
        nsteps = max(1, int(round(T / dt)))
        a, b = slab_ranges(p.grid.shape[0], world)[rank]
        part = NumpySlab(p, variant, dt, T, rank, world, a, b)
        taken, dstep, u = run_slabs([part], GroupExchange(), nsteps,
                                    variant.startswith("LODCN"))[0]
        # gather the owned planes on every rank (the decomposition's result exchange)
        owned = torch.from_numpy(np.ascontiguousarray(u[1:-1]))
        sizes = [bb - aa for aa, bb in slab_ranges(p.grid.shape[0], world)]
        n1, n2 = p.grid.shape[1:]
        bufs = [torch.zeros((s, n1, n2), dtype=torch.float64) for s in sizes]
        dist.all_gather(bufs, owned)
        if rank == 0:
            full = p.bvals.copy()
            full[1:-1] = torch.cat(bufs).numpy()
            np.savez(os.path.join(out_dir, f"{variant}.npz"), full=full, taken=taken,
                     dstep=-1 if dstep is None else dstep)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("variant", ["LODIE2", "LODCN2"])
def test_gloo_world2_slab_march(tmp_path, variant):
    world = 2
    mp.spawn(_gloo_worker, args=(world, _free_port(), variant, str(tmp_path)), nprocs=world,
             join=True)
    d = golden("march_variants")
    r = np.load(tmp_path / f"{variant}.npz")
    assert int(r["taken"]) == max(1, int(round(float(d["T"]) / float(d["dt"]))))
    assert int(r["dstep"]) == -1
    assert _rel(r["full"], d[variant]) <= TOL


# ---------------------------------------------------------------------------------------
# Config 5 batch (replicas): round-robin assignment and the result gather over gloo, with a
# host stand-in for the march (the device path is covered by tests/test_gpu_batch.py).

def _fake_problem(i, n_atoms):
    from paper_1410_2788_b200.configs import batch_config

    return batch_config(i, n_atoms), i


def _fake_march(prob, cfg):
    from types import SimpleNamespace

    n = max(1, int(round(cfg.T / cfg.dt)))
    return SimpleNamespace(steps_taken=n, diverged=False,
                           final=np.full((2, 2, 2), float(prob) + (0.5 if cfg.variant.value == "LODIE2" else 0.0)),
                           wall_time=0.0)


def test_batch_rank_indices_partition():
    from paper_1410_2788_b200.batch import rank_indices

    for world in (1, 2, 3, 8):
        got = sorted(i for r in range(world) for i in rank_indices(64, r, world))
        assert got == list(range(64))
    with pytest.raises(ValueError):
        rank_indices(64, 2, 2)


def _batch_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1410_2788_b200.batch import run_config5

        items = run_config5(rank, world, count=10, nsteps=3, march_fn=_fake_march,
                            problem_fn=_fake_problem)
        if rank == 0:
            np.save(os.path.join(out_dir, "items.npy"),
                    np.array([(it.index, it.variant == "LODIE2", it.steps_taken, it.max_abs)
                              for it in items]))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_batch_gather(tmp_path):
    mp.spawn(_batch_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    arr = np.load(tmp_path / "items.npy")
    assert arr.shape == (20, 4)
    assert list(arr[:, 0]) == [i for i in range(10) for _ in range(2)]
    assert np.all(arr[:, 2] == 3)
    assert np.allclose(arr[:, 3], arr[:, 0] + 0.5 * arr[:, 1])
