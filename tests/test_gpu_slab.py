"""Slab-decomposed march on one GPU: N partitions in one process with the
exchange done by device copies (NCCL cannot put two ranks on one GPU).  The partitioned
result must match the reference fixtures and the single-device march to the potential bar;
observed agreement is reassociation level (~1e-15)."""

import numpy as np
import pytest

import paper_1410_2788_b200 as pb
from paper_1410_2788_b200.slab import march_partitioned
from tests.helpers import golden, rel_err
from tests.test_gpu_parity import POT_TOL, protein_from

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def case():
    d = golden("march_variants")
    return d, protein_from(d)


@pytest.mark.parametrize("variant", ["LODIE1", "LODIE2", "LODCN2"])
@pytest.mark.parametrize("nparts", [1, 2, 3, 5])
def test_partitioned_vs_reference(case, variant, nparts):
    d, p = case
    cfg = pb.MarchConfig(dt=float(d["dt"]), T=float(d["T"]), variant=variant)
    rep = march_partitioned(p, cfg, nparts)
    assert rep.steps_taken == 5 and not rep.diverged
    assert rel_err(rep.final.data, d[variant]) <= POT_TOL
    single = pb.march(p, cfg)
    assert rel_err(rep.final.data, single.final.data) <= 1e-12


def test_partitioned_divergence(case):
    d, p = case
    cfg = pb.MarchConfig(dt=0.3, T=3.0, variant="LODIE1", divergence_threshold=2.0e3)
    rep = march_partitioned(p, cfg, 3)
    assert rep.diverged
    assert rep.steps_taken == int(d["div_steps"])
    assert rep.diverged_step == int(d["div_step"])
    assert rel_err(rep.final.data, d["div_final"]) <= POT_TOL


def test_partitioned_unsupported_variant(case):
    _, p = case
    with pytest.raises(NotImplementedError):
        march_partitioned(p, pb.MarchConfig(dt=0.3, T=0.3, variant="AOSIE1"), 2)


@pytest.mark.parametrize("variant,nparts", [("LODIE2", 8), ("LODCN2", 4), ("LODIE2", 2),
                                            ("LODCN2", 2)])
def test_partitioned_config2_vs_single(variant, nparts):
    """129^3, 500 atoms (config 2 grid): 8 slabs of 15-16 planes, 4 steps (2 slabs:
    64- and 63-row axis-0 chunks, the four-segment column shape)."""
    from paper_1410_2788_b200.configs import CONFIGS, cubic_box, kappa_bar, synthetic_atoms
    from paper_1410_2788_b200.problem import assemble_on_grid
    from tests.helpers import system_of

    c = CONFIGS["c2"]
    atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
    lo, hi = cubic_box(atoms, c.n, c.h)
    p = assemble_on_grid(system_of(atoms), pb.make_grid(lo, hi, c.h),
                         kappa_bar(c.ionic_strength), c.eps_m, c.eps_s)
    cfg = pb.MarchConfig(dt=c.dt, T=4 * c.dt, variant=variant)
    single = pb.march(p, cfg).final.data
    rep = march_partitioned(p, cfg, nparts)
    assert rep.steps_taken == 4
    assert rel_err(rep.final.data, single) <= 1e-12
    assert np.isfinite(rep.final.data).all()
    # equal plane counts and a strongly cost-weighted split give the same field
    for beta in (0.0, 40.0):
        rep = march_partitioned(p, cfg, nparts, beta=beta)
        assert rel_err(rep.final.data, single) <= 1e-12, beta


def test_cost_weighted_ranges_follow_the_molecule():
    """The ranks holding the molecule get fewer planes; beta = 0 keeps equal counts."""
    from paper_1410_2788_b200.configs import CONFIGS, cubic_box, kappa_bar, synthetic_atoms
    from paper_1410_2788_b200.problem import assemble_on_grid
    from paper_1410_2788_b200.schemes import device_problem
    from paper_1410_2788_b200.slab import plane_costs, slab_ranges
    from tests.helpers import system_of

    c = CONFIGS["c2"]
    atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
    lo, hi = cubic_box(atoms, c.n, c.h)
    p = assemble_on_grid(system_of(atoms), pb.make_grid(lo, hi, c.h),
                         kappa_bar(c.ionic_strength), c.eps_m, c.eps_s)
    dp = device_problem(p)
    assert plane_costs(dp, 0.0) is None
    cost = plane_costs(dp, 6.0)
    assert cost.shape == (c.n - 2,) and cost.min() >= 1.0 and cost.max() > 1.2
    sizes = [b - a for a, b in slab_ranges(c.n, 4, cost)]
    assert sum(sizes) == c.n - 2 and sizes[1] < sizes[0] and sizes[2] < sizes[3]
