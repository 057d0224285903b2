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


def test_batched_march_matches_per_problem_marches():
    """One launch per sweep over all grids (pbg_plan_run_batch) == march() per protein, up to
    reassociation: lines of two grids can share a warp, which may pick the PCR reduced solve
    where the single-grid launch took the static inverse (same system, other rounding)."""
    from paper_1410_2788_b200.batch import BatchMarch

    sizes = batch_sizes()
    probs = [config5_problem(i, sizes[i])[1] for i in range(5)]
    bm = BatchMarch(probs)
    for v in ("AOSIE1", "LODIE2", "LODIE1", "LODCN2", "MAOSIE"):
        cfg = pb.MarchConfig(dt=0.5, T=3.0, variant=v)
        reps, secs = bm.march(cfg)
        assert secs > 0
        for p, rep in zip(probs, reps):
            want = pb.march(p, cfg)
            assert rep.steps_taken == want.steps_taken == 6 and not rep.diverged
            assert rel_err(rep.final.data, want.final.data) <= 1e-13, v


def test_batched_march_divergence_is_per_grid():
    """A grid that crosses the threshold stops at its own step (the oracle's); the others
    run to the end, each with its own final field."""
    from paper_1410_2788_b200.batch import BatchMarch

    g = pb.make_grid((0, 0, 0), (0.25 * 8, 0.25 * 9, 0.25 * 96), 0.25)  # 97-row lines
    rng = np.random.default_rng(9)
    region = pb.build_region_maps(g, pb.AnalyticSphere(0.7), 2.0, 80.0, 1.0)
    probs = []
    for scale in (1.0, 500.0, 2.0):
        rho = np.zeros(g.shape)
        rho[1:-1, 1:-1, 1:-1] = scale * rng.standard_normal(tuple(s - 2 for s in g.shape))
        p = pb.NPBProblem(grid=g, region=region, rho=pb.ScalarField(g, rho),
                          qfrac=pb.ScalarField.zeros(g),
                          boundary=pb.BoundarySpec(g, np.zeros(g.shape)), alpha=1.0,
                          initial=pb.ScalarField.zeros(g))
        probs.append(p)
    amax = [np.max(np.abs(pb.march(probs[1], pb.MarchConfig(dt=0.2, T=0.2 * k,
                                                           variant="LODIE2")).final.data))
            for k in (2, 6)]
    thr = 0.5 * (amax[0] + amax[1])
    cfg = pb.MarchConfig(dt=0.2, T=2.0, variant="LODIE2", divergence_threshold=thr)
    reps, _ = BatchMarch(probs).march(cfg)
    for p, rep in zip(probs, reps):
        want = pb.march(p, cfg)
        assert rep.steps_taken == want.steps_taken and rep.diverged == want.diverged
        assert rel_err(rep.final.data, want.final.data) <= 1e-13
    assert reps[1].diverged and 2 < reps[1].steps_taken <= 6
    assert not reps[0].diverged and reps[0].steps_taken == 10
