"""Comparison schemes on the device (ADI1, ADI2, ExplicitEuler; schemes.py:240-253,
331-363) against the reference fixtures (tests/golden/comparison.npz) and the oracle."""

import numpy as np
import pytest

import paper_1410_2788_b200 as pb
from oracle import pbs_oracle as O
from tests.helpers import golden, rel_err
from tests.test_gpu_parity import POT_TOL, protein_from

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def case():
    d = golden("comparison")
    return d, protein_from(d)


@pytest.mark.parametrize("variant", ["ADI1", "ADI2"])
def test_adi_vs_reference(case, variant):
    d, p = case
    rep = pb.march(p, pb.MarchConfig(dt=0.3, T=1.5, variant=variant))
    assert rep.steps_taken == int(d[variant + "_steps"]) and not rep.diverged
    assert rel_err(rep.final.data, d[variant]) <= POT_TOL
    assert rel_err(rep.final.data, d[variant]) <= 1e-13


def test_explicit_euler_vs_reference(case):
    d, p = case
    rep = pb.march(p, pb.MarchConfig(dt=2e-4, T=2e-2, variant="ExplicitEuler"))
    assert rep.steps_taken == 100 and not rep.diverged
    assert rel_err(rep.final.data, d["Euler"]) <= 1e-13


def test_explicit_euler_divergence(case):
    d, p = case
    rep = pb.march(p, pb.MarchConfig(dt=0.01, T=1.0, variant="ExplicitEuler",
                                     divergence_threshold=1e6))
    assert rep.diverged and rep.diverged_step == int(d["Euler_div_step"])
    assert rep.steps_taken == int(d["Euler_div_steps"])
    assert rel_err(rep.final.data, d["Euler_div_final"]) <= 1e-12


@pytest.mark.parametrize("variant", ["ADI1", "ExplicitEuler"])
def test_comparison_schemes_config2_vs_oracle(variant):
    from paper_1410_2788_b200.configs import CONFIGS, cubic_box, kappa_bar, synthetic_atoms
    from paper_1410_2788_b200.problem import assemble_on_grid
    from tests.helpers import system_of

    c = CONFIGS["c2"]
    atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
    lo, hi = cubic_box(atoms, c.n, c.h)
    grid = pb.make_grid(lo, hi, c.h)
    p = assemble_on_grid(system_of(atoms), grid, kappa_bar(c.ionic_strength), c.eps_m, c.eps_s)
    dt, n = (c.dt, 3) if variant == "ADI1" else (1e-4, 20)
    rep = pb.march(p, pb.MarchConfig(dt=dt, T=dt * n, variant=variant))
    op = O.protein_on_grid(O.OGrid(grid.lo, grid.h, grid.shape), atoms, c.eps_m, c.eps_s,
                           kappa_bar(c.ionic_strength))
    orep = O.march(op, variant, dt, dt * n)
    assert rep.steps_taken == orep.steps_taken == n
    assert rel_err(rep.final.data, orep.final) <= POT_TOL
