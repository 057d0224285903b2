"""DST-I vacuum solver (pbg_vacuum_dst, cuFFT) and the Plain / RE energy variants against
the reference fixtures (tests/golden/vacuum.npz) and the scipy oracle at config-2 size."""

import numpy as np
import pytest

import paper_1410_2788_b200 as pb
from oracle import pbs_oracle as O
from tests.helpers import golden, rel_err
from tests.test_gpu_parity import DG_TOL, POT_TOL, protein_from

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def case():
    d = golden("vacuum")
    return d, protein_from(d)


def test_vacuum_potential_fast_vs_reference(case):
    d, p = case
    vac = pb.make_vacuum_problem(p)
    phi0 = pb.vacuum_potential_fast(p.rho, p.grid, p.eps_m, vac.boundary)
    assert rel_err(phi0.data, d["phi0_fast"]) <= 1e-12


@pytest.mark.parametrize("variant", ["LODIE2", "AOSIE1"])
@pytest.mark.parametrize("mode", ["Plain", "RE"])
def test_plain_re_energies_vs_reference(case, variant, mode):
    d, p = case
    res = pb.energy_pipeline(p, pb.MarchConfig(dt=0.5, T=5.0, variant=variant), mode)
    want = float(d[f"dg_{mode}_{variant}"])
    assert not res.diverged
    assert abs(res.delta_g - want) <= DG_TOL * abs(want)


def test_kirkwood_plain_energy_vs_reference():
    from paper_1410_2788_b200.configs import KIRKWOOD as kw

    d = golden("vacuum")
    sysk = pb.MolecularSystem([pb.Atom((0.0, 0.0, 0.0), 1.0, 2.0)], label="kirkwood")
    p = pb.protein_problem(sysk, h=kw["h"], padding=kw["padding"], kappa_bar=kw["kappa_bar"],
                           eps_m=kw["eps_m"], eps_s=kw["eps_s"])
    res = pb.energy_pipeline(p, pb.MarchConfig(dt=kw["dt"], T=kw["T"], variant="LODIE2"), "Plain")
    want = float(d["dg_kirkwood_plain"])
    assert abs(res.delta_g - want) <= DG_TOL * abs(want)
    plane = res.phi_0.data[res.phi_0.data.shape[0] // 2]
    assert rel_err(plane, d["kirkwood_phi0_plane"]) <= POT_TOL


def test_vacuum_potential_config2_size_vs_oracle():
    from paper_1410_2788_b200.configs import CONFIGS, cubic_box, kappa_bar, synthetic_atoms
    from paper_1410_2788_b200.problem import assemble_on_grid
    from tests.helpers import system_of

    c = CONFIGS["c2"]
    atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
    lo, hi = cubic_box(atoms, c.n, c.h)
    grid = pb.make_grid(lo, hi, c.h)
    p = assemble_on_grid(system_of(atoms), grid, kappa_bar(c.ionic_strength), c.eps_m, c.eps_s)
    vac = pb.make_vacuum_problem(p)
    got = pb.vacuum_potential_fast(p.rho, grid, p.eps_m, vac.boundary).data
    og = O.OGrid(grid.lo, grid.h, grid.shape)
    op = O.protein_on_grid(og, atoms, c.eps_m, c.eps_s, kappa_bar(c.ionic_strength))
    want = O.vacuum_potential_fast(op.rho, og, c.eps_m, O.vacuum_of(op).bvals)
    assert rel_err(got, want) <= 1e-12
    # the solve satisfies the discrete equation: residual of -eps*lap(phi) - rho
    lap = O._const_laplacian_interior(got)
    res = -(c.eps_m / grid.h ** 2) * lap - op.rho[O.INT]
    assert np.max(np.abs(res)) <= 1e-9 * np.max(np.abs(op.rho))
