"""Config 5 batch on one GPU: concurrent marches on several streams give the same results
as the sequential device march and the CPU oracle."""

import numpy as np
import pytest

import paper_1410_2788_b200 as pb
from oracle import pbs_oracle as O
from paper_1410_2788_b200.batch import config5_problem, march_many, run_config5
from paper_1410_2788_b200.configs import batch_sizes, batch_config, cubic_box, kappa_bar, synthetic_atoms
from tests.helpers import rel_err

pytestmark = pytest.mark.gpu


def test_concurrent_streams_match_sequential():
    sizes = batch_sizes()
    probs = [config5_problem(i, sizes[i]) for i in range(4)]
    jobs, seq = [], {}
    for i, (c, p) in enumerate(probs):
        for v in ("AOSIE1", "LODIE2"):
            cfg = pb.MarchConfig(dt=c.dt, T=c.dt * 10, variant=v)
            seq[(i, v)] = pb.march(p, cfg).final.data
            jobs.append(((i, v), p, cfg))
    got = march_many(jobs, streams=4)
    for key, rep in got.items():
        assert rep.steps_taken == 10
        assert np.array_equal(rep.final.data, seq[key])  # same kernels, same order: bitwise


def test_run_config5_small_batch_vs_oracle():
    items = run_config5(count=3, nsteps=5, streams=3)
    assert [(it.index, it.variant) for it in items] == [
        (i, v) for i in range(3) for v in ("AOSIE1", "LODIE2")]
    sizes = batch_sizes()
    c = batch_config(1, sizes[1])
    atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
    lo, hi = cubic_box(atoms, c.n, c.h)
    g = pb.make_grid(lo, hi, c.h)
    op = O.protein_on_grid(O.OGrid(g.lo, g.h, g.shape), atoms, c.eps_m, c.eps_s,
                           kappa_bar(c.ionic_strength))
    for it in items:
        if it.index != 1:
            continue
        ref = O.march(op, it.variant, c.dt, 5 * c.dt).final
        assert abs(it.max_abs - np.max(np.abs(ref))) <= 1e-9 * np.max(np.abs(ref))
        assert not it.diverged and it.steps_taken == 5


def test_stream_pool_persists_and_repeats_bitwise():
    """march_many reuses one stream pool per device (the allocator's per-stream blocks from a
    warm-up stay usable), and a repeated batch reproduces the first bit for bit."""
    from paper_1410_2788_b200 import batch as B

    sizes = batch_sizes()
    probs = [config5_problem(i, sizes[i]) for i in range(2)]
    jobs = [((i, v), p, pb.MarchConfig(dt=c.dt, T=c.dt * 4, variant=v))
            for i, (c, p) in enumerate(probs) for v in ("AOSIE1", "LODIE2")]
    first = march_many(jobs, streams=3)
    import torch

    pool = list(B._STREAMS[torch.cuda.current_device()][:3])
    second = march_many(jobs, streams=3)
    assert B._STREAMS[torch.cuda.current_device()][:3] == pool
    for key in first:
        assert np.array_equal(first[key].final.data, second[key].final.data)
