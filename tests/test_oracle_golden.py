"""Pin the CPU oracle (oracle/pbs_oracle.py) against fixtures produced by the real reference.

CPU only.  Assembly must be bit-exact; marches agree to <= 1e-13 relative (same IEEE
operations in the same order; observed exactly equal).
"""

import numpy as np
import pytest

from oracle import pbs_oracle as O
from tests.helpers import atoms_of, faces, golden, ogrid, oracle_protein, rel_err


@pytest.mark.parametrize("tag", ["a40", "a60_probe"])
def test_assembly_bit_exact(tag):
    d = golden(f"assembly_{tag}")
    p = oracle_protein(d)
    r = p.region
    assert np.array_equal(r.eps_node == d["eps_m"], d["node_solute"])
    for a, key in enumerate(("hx", "hy", "hz")):
        assert np.array_equal(r.eps_half[a] == d["eps_m"], d[key])
    assert np.array_equal(r.kappa2, d["kappa2"])
    assert np.array_equal(p.qfrac, d["qfrac"])
    assert np.array_equal(p.rho, d["rho"])
    assert np.array_equal(faces(p.bvals), d["faces"])


def test_bbox_grid_rule_matches_reference():
    d = golden("assembly_a40")
    g = O.protein_bbox_grid(atoms_of(d), float(d["h"]), float(d["padding"]))
    assert g.shape == tuple(int(v) for v in d["shape"])
    assert np.array_equal(np.array(g.lo), d["lo"])


VARIANTS = ["LODIE1", "LODIE2", "LODCN1", "LODCN2", "AOSIE1", "AOSIE2", "AOSCN1", "AOSCN2",
            "MAOSIE", "MAOSCN"]


@pytest.fixture(scope="module")
def march_golden():
    d = golden("march_variants")
    return d, oracle_protein(d)


@pytest.mark.parametrize("variant", VARIANTS)
def test_march_variants(march_golden, variant):
    d, p = march_golden
    rep = O.march(p, variant, float(d["dt"]), float(d["T"]))
    assert rel_err(rep.final, d[variant]) <= 1e-13


@pytest.mark.parametrize("variant", ["AOSIE1", "AOSCN2"])
def test_aos_literal(march_golden, variant):
    d, p = march_golden
    rep = O.march(p, variant, float(d["dt"]), float(d["T"]), aos_nonlinear="literal")
    assert rel_err(rep.final, d[variant + "_literal"]) <= 1e-13


def test_alpha_override_and_divergence(march_golden):
    d, p = march_golden
    rep = O.march(p, "LODIE2", float(d["dt"]), float(d["T"]), alpha=0.5)
    assert rel_err(rep.final, d["LODIE2_alpha05"]) <= 1e-13
    rep = O.march(p, "LODIE1", 0.3, 3.0, threshold=2.0e3)
    assert rep.steps_taken == int(d["div_steps"])
    assert (rep.diverged_step or -1) == int(d["div_step"])
    assert rel_err(rep.final, d["div_final"]) <= 1e-13


def test_single_sweeps_and_flow():
    d = golden("small_api")
    g = O.grid_from_bounds((0, 0, 0), (2, 2, 2), 0.5)
    reg = O.sphere_region(g, 0.8, 1.0, 80.0, 1.0)
    for axis in range(3):
        lf = O.LineFactors(g, reg, d["sweep_bvals"], axis, 3.0 * 0.21 / 1.7)
        out = d["sweep_rhs"].copy()
        out[O.INT] = lf.solve(d["sweep_rhs"][O.INT])
        O.apply_faces(out, d["sweep_bvals"])
        assert rel_err(out, d[f"ie_{axis}"]) <= 1e-14
    w, k2 = d["flow_w"], d["flow_k2"]
    assert np.array_equal(O.sinh_flow(w, np.exp(-(0.37 / 1.3) * k2)), d["flow_out"])


def test_sphere_benchmark_march():
    d = golden("sphere")
    g = O.grid_from_bounds((-3, -3, -3), (3, 3, 3), 0.5)
    reg = O.sphere_region(g, 1.0, 1.0, 80.0, 1.0)
    p = O.OProblem(g, reg, d["rho"], np.zeros(g.shape), d["bvals"], 1.0, d["initial"])
    for v in ("LODIE1", "AOSCN2", "MAOSIE"):
        rep = O.march(p, v, 0.0125, 1.0)
        assert rel_err(rep.final, d[v]) <= 1e-13


def test_energy_replusv():
    d = golden("energy")
    p = oracle_protein(d)
    for v in ("LODIE2", "AOSIE1"):
        dg, pm, p0, div = O.energy_replusv(p, v, 0.5, 5.0)
        assert not div
        assert abs(dg - float(d[f"dg_{v}"])) <= 1e-12 * abs(float(d[f"dg_{v}"]))
        assert rel_err(pm, d[f"phim_{v}"]) <= 1e-13
        assert rel_err(p0, d[f"phi0_{v}"]) <= 1e-13


def test_kirkwood_config1():
    d = golden("kirkwood")
    atoms = [(0.0, 0.0, 0.0, 1.0, 2.0)]
    g = O.protein_bbox_grid(atoms, 0.25, 8.0)
    assert g.shape == (65, 65, 65)
    p = O.protein_on_grid(g, atoms, 1.0, 80.0, float(np.sqrt(O.KAPPA2_PER_MOLAR * 0.1)))
    for v in ("LODIE1", "LODIE2"):
        rep = O.march(p, v, 0.1, 20.0)
        u = rep.final
        assert rel_err(u[32], d[v + "_plane"]) <= 1e-13
        st = np.array([np.max(np.abs(u)), np.sum(u), np.sum(u * u)])
        assert np.allclose(st, d[v + "_stats"], rtol=1e-12, atol=0)


def test_vacuum_direct_solver_and_plain_re_energies():
    """DST-I vacuum solve and Plain / RE energies against the reference (vacuum.npz)."""
    d = golden("vacuum")
    p = oracle_protein(d)
    phi0 = O.vacuum_potential_fast(p.rho, p.grid, p.eps_m, O.vacuum_of(p).bvals)
    assert rel_err(phi0, d["phi0_fast"]) <= 1e-13
    for v in ("LODIE2", "AOSIE1"):
        for mode in ("Plain", "RE"):
            dg, _, _, div = O.energy_direct(p, v, 0.5, 5.0, mode)
            want = float(d[f"dg_{mode}_{v}"])
            assert not div and abs(dg - want) <= 1e-10 * abs(want)


def test_comparison_schemes_vs_reference():
    """ADI1 / ADI2 / ExplicitEuler (schemes.py:240-253, 331-363) against comparison.npz."""
    d = golden("comparison")
    p = oracle_protein(d)
    for v in ("ADI1", "ADI2"):
        rep = O.march(p, v, 0.3, 1.5)
        assert rep.steps_taken == int(d[v + "_steps"])
        assert rel_err(rep.final, d[v]) <= 1e-13
    rep = O.march(p, "ExplicitEuler", 2e-4, 2e-2)
    assert rep.steps_taken == int(d["Euler_steps"]) and not rep.diverged
    assert rel_err(rep.final, d["Euler"]) <= 1e-13
    rep = O.march(p, "ExplicitEuler", 0.01, 1.0, threshold=1e6)
    assert rep.diverged and rep.diverged_step == int(d["Euler_div_step"])
    assert rep.steps_taken == int(d["Euler_div_steps"])
    assert rel_err(rep.final, d["Euler_div_final"]) <= 1e-13
