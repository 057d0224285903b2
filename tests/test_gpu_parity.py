"""Device parity: libpbg.so kernels vs the reference fixtures and the CPU oracle.

Bars (north_star): potentials max|du| <= 1e-9 * max|u_ref|; energies |dG - dG_ref| <=
1e-8 |dG_ref|.  Assembly (codes, qfrac, rho) is integer/ordering work and must be
bit-exact; faces use the device exp (<= 1e-15 relative).  Observed agreement of the
marches is ~1e-15 (segmented Thomas + PCR reassociates fp64 only).
"""

import ctypes

import numpy as np
import pytest

import paper_1410_2788_b200 as pb
from oracle import pbs_oracle as O
from tests.helpers import atoms_of, faces, golden, oracle_protein, rel_err, system_of

pytestmark = pytest.mark.gpu

POT_TOL = 1e-9
DG_TOL = 1e-8
VARIANTS = ["LODIE1", "LODIE2", "LODCN1", "LODCN2", "AOSIE1", "AOSIE2", "AOSCN1", "AOSCN2",
            "MAOSIE", "MAOSCN"]


def protein_from(d, alpha=1.0):
    probe = float(d["probe"]) if "probe" in d else 0.0
    return pb.protein_problem(system_of(atoms_of(d)), h=float(d["h"]),
                              padding=float(d["padding"]), kappa_bar=float(d["kappa_bar"]),
                              eps_m=float(d["eps_m"]), eps_s=float(d["eps_s"]), alpha=alpha,
                              probe_inflation=probe)


@pytest.mark.parametrize("tag", ["a40", "a60_probe"])
def test_assembly_bit_exact(tag):
    d = golden(f"assembly_{tag}")
    p = protein_from(d)
    assert p.grid.shape == tuple(int(v) for v in d["shape"])
    r = p.region
    assert np.array_equal(r.eps_node.data == d["eps_m"], d["node_solute"])
    assert np.array_equal(r.eps_half_x == d["eps_m"], d["hx"])
    assert np.array_equal(r.eps_half_y == d["eps_m"], d["hy"])
    assert np.array_equal(r.eps_half_z == d["eps_m"], d["hz"])
    assert np.array_equal(r.kappa2.data, d["kappa2"])
    assert np.array_equal(p.qfrac.data, d["qfrac"])
    assert np.array_equal(p.rho.data, d["rho"])
    assert rel_err(faces(p.boundary.values), d["faces"]) <= 1e-15


@pytest.fixture(scope="module")
def march_case():
    d = golden("march_variants")
    return d, protein_from(d)


@pytest.mark.parametrize("variant", VARIANTS)
def test_march_variants_vs_reference(march_case, variant):
    d, p = march_case
    rep = pb.march(p, pb.MarchConfig(dt=float(d["dt"]), T=float(d["T"]), variant=variant))
    assert rep.steps_taken == 5 and not rep.diverged
    assert rel_err(rep.final.data, d[variant]) <= POT_TOL
    assert rel_err(rep.final.data, d[variant]) <= 1e-13  # observed floor, far below the bar


@pytest.mark.parametrize("variant", ["AOSIE1", "AOSCN2"])
def test_aos_literal_mode(march_case, variant):
    d, p = march_case
    rep = pb.march(p, pb.MarchConfig(dt=0.3, T=1.5, variant=variant, aos_nonlinear="literal"))
    assert rel_err(rep.final.data, d[variant + "_literal"]) <= POT_TOL


def test_alpha_override(march_case):
    d, p = march_case
    rep = pb.march(p, pb.MarchConfig(dt=0.3, T=1.5, variant="LODIE2", alpha=0.5))
    assert rel_err(rep.final.data, d["LODIE2_alpha05"]) <= POT_TOL


def test_divergence_is_data(march_case):
    d, p = march_case
    rep = pb.march(p, pb.MarchConfig(dt=0.3, T=3.0, variant="LODIE1",
                                     divergence_threshold=2.0e3))
    assert rep.diverged and rep.final.diverged
    assert rep.steps_taken == int(d["div_steps"])
    assert rep.diverged_step == int(d["div_step"])
    assert rel_err(rep.final.data, d["div_final"]) <= POT_TOL


def test_single_sweeps_vs_reference():
    d = golden("small_api")
    g = pb.make_grid((0, 0, 0), (2, 2, 2), 0.5)
    region = pb.build_region_maps(g, pb.AnalyticSphere(0.8), 1.0, 80.0, 1.0)
    b = pb.BoundarySpec(g, d["sweep_bvals"])
    rhs = pb.ScalarField(g, d["sweep_rhs"])
    for axis in range(3):
        assert rel_err(pb.ie_sweep(axis, rhs, 3.0, 0.21, 1.7, region, b).data,
                       d[f"ie_{axis}"]) <= 1e-13
        assert rel_err(pb.cn_sweep(axis, rhs, 4.0, 0.15, 0.8, region, b).data,
                       d[f"cn_{axis}"]) <= 1e-13


def test_multi_segment_sweeps_vs_reference():
    d = golden("small_api")
    atoms = atoms_of(d, "big_atoms")
    p = pb.protein_problem(system_of(atoms), h=0.5, padding=3.0, kappa_bar=1.0, eps_m=2.0,
                           eps_s=80.0)
    assert p.grid.shape == tuple(int(v) for v in d["big_shape"])
    rhs = pb.ScalarField(p.grid, np.random.default_rng(78).standard_normal(p.grid.shape))
    for axis in range(3):
        got = pb.ie_sweep(axis, rhs, 1.0, 0.5, 1.0, p.region, p.boundary).data
        assert rel_err(got, d[f"big_ie_{axis}"]) <= 1e-13
        got = pb.cn_sweep(axis, rhs, 1.0, 0.5, 1.0, p.region, p.boundary).data
        assert rel_err(got, d[f"big_cn_{axis}"]) <= 1e-13


def test_nonlinear_step_vs_reference():
    d = golden("small_api")
    w, k2 = d["flow_w"], d["flow_k2"]
    for key, kw in (("flow_out", {}), ("flow_out_pm4", {"premultiplier": 4.0}),
                    ("flow_out_rate4", {"rate": 4.0})):
        got = pb.nonlinear_step(w, k2, 0.37, 1.3, **kw)
        want = d[key]
        assert np.all(np.isfinite(got))
        assert np.max(np.abs(got - want) / np.maximum(np.abs(want), 1e-300)) <= 1e-13


def test_step_api_and_aos_order_invariance():
    d = golden("small_api")
    g = pb.make_grid((0, 0, 0), (2, 2, 2), 0.25)
    reg = pb.build_region_maps(g, pb.AnalyticSphere(1.1), 1.0, 80.0, 1.0)
    p = pb.NPBProblem(grid=g, region=reg, rho=pb.ScalarField(g, d["step_rho"]),
                      qfrac=pb.ScalarField.zeros(g), boundary=pb.BoundarySpec(g, d["step_b"]),
                      alpha=1.0, initial=pb.ScalarField(g, d["step_s"]), eps_m=1.0,
                      eps_s=80.0, kappa_bar=1.0, label="perm")
    s = pb.ScalarField(g, d["step_s"])
    for v in VARIANTS:
        out = pb.step(v, s, p, dt=0.2)
        assert not out.diverged
        assert rel_err(out.data, d[f"step_{v}"]) <= 1e-13
    for v in ("AOSIE1", "AOSCN2"):
        base = pb.step(v, s, p, dt=0.2).data
        for order in ((2, 0, 1), (1, 2, 0), (2, 1, 0)):
            other = pb.step(v, s, p, dt=0.2, aos_order=order).data
            assert np.max(np.abs(base - other)) <= 1e-13


def test_sphere_benchmark_vs_reference():
    d = golden("sphere")
    g = pb.default_sphere_grid(0.5)
    p = pb.sphere_benchmark(g, H=1.0)
    assert rel_err(p.rho.data, d["rho"]) <= 1e-15
    for v in ("LODIE1", "AOSCN2", "MAOSIE"):
        rep = pb.march(p, pb.MarchConfig(dt=0.0125, T=1.0, variant=v))
        assert rel_err(rep.final.data, d[v]) <= 1e-12


def test_energy_replusv_vs_reference():
    d = golden("energy")
    p = protein_from(d)
    for v in ("LODIE2", "AOSIE1"):
        res = pb.energy_pipeline(p, pb.MarchConfig(dt=0.5, T=5.0, variant=v), "REplusV")
        want = float(d[f"dg_{v}"])
        assert abs(res.delta_g - want) <= DG_TOL * abs(want)
        assert rel_err(res.phi_m.data, d[f"phim_{v}"]) <= POT_TOL
        assert rel_err(res.phi_0.data, d[f"phi0_{v}"]) <= POT_TOL


def test_kirkwood_config1_vs_reference():
    from paper_1410_2788_b200.configs import KIRKWOOD as kw

    d = golden("kirkwood")
    sysk = pb.MolecularSystem([pb.Atom((0.0, 0.0, 0.0), 1.0, 2.0)], label="kirkwood")
    p = pb.protein_problem(sysk, h=kw["h"], padding=kw["padding"], kappa_bar=kw["kappa_bar"],
                           eps_m=kw["eps_m"], eps_s=kw["eps_s"])
    assert p.grid.shape == (65, 65, 65)
    for v in ("LODIE1", "LODIE2"):
        rep = pb.march(p, pb.MarchConfig(dt=kw["dt"], T=kw["T"], variant=v))
        assert rep.steps_taken == 200
        u = rep.final.data
        assert rel_err(u[32], d[v + "_plane"]) <= POT_TOL
        st = np.array([np.max(np.abs(u)), np.sum(u), np.sum(u * u)])
        assert np.allclose(st, d[v + "_stats"], rtol=1e-10, atol=0)
    res = pb.energy_pipeline(p, pb.MarchConfig(dt=kw["dt"], T=kw["T"], variant="LODIE2"),
                             "REplusV")
    want = float(d["dg_replusv_lodie2"])
    assert abs(res.delta_g - want) <= DG_TOL * abs(want)


def _oracle_vs_device(cfg_atoms, n, h, eps_m, eps_s, kbar, variant, dt, steps):
    from paper_1410_2788_b200.configs import cubic_box

    lo, hi = cubic_box(cfg_atoms, n, h)
    grid = pb.make_grid(lo, hi, h)
    from paper_1410_2788_b200.problem import assemble_on_grid

    p = assemble_on_grid(system_of(cfg_atoms), grid, kbar, eps_m, eps_s)
    og = O.OGrid(grid.lo, grid.h, grid.shape)
    op = O.protein_on_grid(og, cfg_atoms, eps_m, eps_s, kbar)
    rep = pb.march(p, pb.MarchConfig(dt=dt, T=dt * steps, variant=variant))
    orep = O.march(op, variant, dt, dt * steps)
    return rep, orep, p, op


def test_config2_protein500_129_lodie2_vs_oracle():
    from paper_1410_2788_b200.configs import CONFIGS, kappa_bar, synthetic_atoms

    c = CONFIGS["c2"]
    atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
    rep, orep, p, op = _oracle_vs_device(atoms, c.n, c.h, c.eps_m, c.eps_s,
                                         kappa_bar(c.ionic_strength), "LODIE2", c.dt, c.steps)
    assert rep.steps_taken == orep.steps_taken == c.steps
    assert rel_err(rep.final.data, orep.final) <= POT_TOL


@pytest.mark.parametrize("variant", ["AOSIE1", "LODIE2"])
def test_config5_protein_97_vs_oracle(variant):
    from paper_1410_2788_b200.configs import batch_config, batch_sizes, kappa_bar, synthetic_atoms

    n_atoms = batch_sizes()[0]
    c = batch_config(0, n_atoms)
    atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
    rep, orep, _, _ = _oracle_vs_device(atoms, c.n, c.h, c.eps_m, c.eps_s,
                                        kappa_bar(c.ionic_strength), variant, c.dt, c.steps)
    assert rel_err(rep.final.data, orep.final) <= POT_TOL


def test_config3_size_short_march_vs_oracle():
    """257^3 (config 3 grid, 2,500 atoms): two LODIE2 steps against the oracle."""
    from paper_1410_2788_b200.configs import CONFIGS, kappa_bar, synthetic_atoms

    c = CONFIGS["c3"]
    atoms = synthetic_atoms(c.n_atoms, c.ball_radius, c.seed)
    rep, orep, p, op = _oracle_vs_device(atoms, c.n, c.h, c.eps_m, c.eps_s,
                                         kappa_bar(c.ionic_strength), "LODIE2", c.dt, 2)
    assert rel_err(rep.final.data, orep.final) <= POT_TOL
    # assembly bit-exact at full size (bbox-culled oracle)
    r = p.region
    assert np.array_equal(r.eps_half_x == c.eps_m, op.region.eps_half[0] == c.eps_m)
    assert np.array_equal(r.kappa2.data, op.region.kappa2)
    assert np.array_equal(p.qfrac.data, op.qfrac)


def test_march_host_c_abi_matches_device_march():
    """pbg_march_host (host buffers in/out, the FFI call) == march()."""
    from paper_1410_2788_b200 import _native as nat

    d = golden("march_variants")
    p = protein_from(d)
    rep = pb.march(p, pb.MarchConfig(dt=0.3, T=1.5, variant="LODIE2"))
    from paper_1410_2788_b200.schemes import device_problem

    dp = device_problem(p)
    codes = dp.codes.cpu().numpy()
    rho = p.rho.data
    idx = np.flatnonzero(rho).astype(np.int64)
    val = rho.ravel()[idx].copy()
    fc = np.ascontiguousarray(faces(p.boundary.values))
    out = np.empty(p.grid.shape)
    desc = nat.PbgMarchDesc()
    desc.grid = nat.grid_struct(p.grid)
    desc.pal = dp.pal
    desc.variant = nat.VARIANT_IDS["LODIE2"]
    desc.dt, desc.alpha, desc.divergence_threshold = 0.3, 1.0, 1e12
    desc.nsteps, desc.check_divergence = 5, 1
    taken, dstep = ctypes.c_int32(), ctypes.c_int32()
    ms = ctypes.c_float()
    nat.check(nat.lib().pbg_march_host(
        ctypes.byref(desc), codes.ctypes.data, len(idx), idx.ctypes.data, val.ctypes.data,
        fc.ctypes.data, None, out.ctypes.data, ctypes.byref(taken), ctypes.byref(dstep),
        ctypes.byref(ms), nat.stream_ptr()))
    assert taken.value == 5 and dstep.value == 0
    assert np.array_equal(out, rep.final.data)


def test_constant_state_steady_every_device_variant():
    g = pb.make_grid((0, 0, 0), (2, 2, 2), 0.5)
    region = pb.uniform_region(g, 1.0, 0.0)
    b = pb.BoundarySpec(g, np.full(g.shape, 1.7))
    p = pb.NPBProblem(grid=g, region=region, rho=pb.ScalarField.zeros(g),
                      qfrac=pb.ScalarField.zeros(g), boundary=b, alpha=1.0,
                      initial=pb.ScalarField(g, np.full(g.shape, 1.7)), eps_m=1.0, eps_s=1.0,
                      kappa_bar=0.0, label="constant")
    for v in VARIANTS:
        out = pb.step(v, p.initial, p, dt=0.3)
        assert np.allclose(out.data, 1.7, atol=1e-13)


def test_large_grid_linearity_property():
    """Full-size property (config-4 sized lines, m = 511): with no ions the LODIE2 step is
    affine in (rho, boundary); doubling both doubles the field."""
    n = 513
    g = pb.make_grid((0, 0, 0), (0.3 * (n - 1), 0.3 * 16, 0.3 * (n - 1)), 0.3)
    rng = np.random.default_rng(5)
    b1 = rng.standard_normal(g.shape)
    rho = np.zeros(g.shape)
    rho[1:-1, 1:-1, 1:-1] = rng.standard_normal(tuple(s - 2 for s in g.shape))
    region = pb.uniform_region(g, 2.0, 0.0)
    outs = []
    for s in (1.0, 2.0):
        p = pb.NPBProblem(grid=g, region=region, rho=pb.ScalarField(g, s * rho),
                          qfrac=pb.ScalarField.zeros(g), boundary=pb.BoundarySpec(g, s * b1),
                          alpha=1.0, initial=pb.ScalarField(g, np.zeros(g.shape)))
        outs.append(pb.march(p, pb.MarchConfig(dt=0.5, T=1.5, variant="LODIE2")).final.data)
    assert rel_err(outs[1], 2.0 * outs[0]) <= 1e-13
