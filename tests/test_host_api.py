"""Host-side API logic of the drop-in package (no device): grid contract, validation and
error behaviour mirror pbsplit (grid.py, schemes.py:49-76, problem.py, geometry.py)."""

import numpy as np
import pytest

import paper_1410_2788_b200 as pb
from paper_1410_2788_b200 import configs


def test_public_names_mirror_reference():
    names = {"C_ES", "KAPPA2_PER_MOLAR", "KCAL_PER_DIMENSIONLESS", "PhysicalConstants",
             "EnergyResult", "energy_pipeline", "recovered_surface_potential", "richardson",
             "solvation_energy", "vacuum_potential_fast", "vacuum_potential_lod",
             "AnalyticSphere", "Atom", "MolecularSystem", "Region", "RegionMap",
             "UnionOfSpheres", "build_region_maps", "classify", "parse_pqr",
             "parse_system_table", "uniform_region", "Grid3D", "NormPair", "ScalarField",
             "deposit_charges", "dump_field_csv", "make_grid", "relative_norms",
             "BoundarySpec", "NPBProblem", "coulomb_screened_boundary", "default_sphere_grid",
             "make_vacuum_problem", "parse_config", "protein_problem", "sphere_benchmark",
             "sphere_exact", "sphere_exact_field", "SCHEME_NAMES", "MarchConfig",
             "MarchReport", "SchemeVariant", "cn_sweep", "ie_sweep", "march",
             "nonlinear_step", "source_step", "step", "TriDiagSystem", "assemble_line",
             "thomas_solve"}
    assert names <= set(pb.__all__)


def test_make_grid_contract():
    g = pb.make_grid((-3, -3, -3), (3, 3, 3), 0.5)
    assert g.shape == (13, 13, 13)
    assert np.allclose(g.x, -3 + 0.5 * np.arange(13))
    with pytest.raises(ValueError, match="integer multiple"):
        pb.make_grid((0, 0, 0), (1, 1, 1), 0.3)
    with pytest.raises(ValueError):
        pb.make_grid((0, 0, 0), (-1, 1, 1), 0.5)
    g = pb.make_grid((0, 0, 0), (2, 1.5, 1), 0.5)
    i, j, k = np.meshgrid(*(np.arange(n) for n in g.shape), indexing="ij")
    flat = g.flat_index(i, j, k)
    assert np.array_equal(np.sort(flat.ravel()), np.arange(g.num_nodes))
    assert all(np.array_equal(a, b) for a, b in zip(g.unflatten(flat), (i, j, k)))


def test_march_config_validation_and_variants():
    with pytest.raises(ValueError):
        pb.MarchConfig(dt=0.0, T=1.0, variant="LODIE1")
    with pytest.raises(ValueError):
        pb.MarchConfig(dt=1.0, T=0.5, variant="LODIE1")
    with pytest.raises(ValueError):
        pb.MarchConfig(dt=0.1, T=1.0, variant="LODIE1", aos_nonlinear="other")
    with pytest.raises(ValueError, match="LODIE1"):
        pb.MarchConfig(dt=0.1, T=1.0, variant="LODXX")
    assert len(pb.SCHEME_NAMES) == 13


def test_scalar_field_host_behaviour():
    g = pb.make_grid((0, 0, 0), (1, 1, 1), 0.5)
    f = pb.ScalarField(g, np.arange(27.0).reshape(3, 3, 3))
    assert f.data.dtype == np.float64 and f.data.flags.c_contiguous
    with pytest.raises(ValueError):
        pb.ScalarField(g, np.zeros((2, 2, 2)))
    n = pb.relative_norms(f, f)
    assert n.l2 == 0.0 and n.linf == 0.0


def test_boundary_spec_from_function_and_apply():
    g = pb.make_grid((0, 0, 0), (1, 1, 1), 0.5)
    b = pb.BoundarySpec.from_function(g, lambda p: p[:, 0] + 10 * p[:, 1] + 100 * p[:, 2])
    data = np.full(g.shape, -1.0)
    b.apply(data)
    assert data[1, 1, 1] == -1.0
    assert data[0, 2, 1] == 0 + 10 * 1.0 + 100 * 0.5
    with pytest.raises(ValueError):
        pb.BoundarySpec(g, np.full(g.shape, np.inf))


def test_parsers():
    s = pb.parse_system_table("atom 0 0 0 1 1.5  # c\n\natom 1 2 3 -0.5 1.2\n")
    assert len(s) == 2 and s.total_charge() == 0.5
    with pytest.raises(ValueError):
        pb.parse_system_table("atom 0 0 0 1\n")
    q = pb.parse_pqr("REMARK x\nATOM 1 N ALA 1 1.0 2.0 3.0 -0.3 1.8\n")
    assert q.atoms[0].center == (1.0, 2.0, 3.0)
    cfg = pb.parse_config("h = 0.5\nscheme = LODIE2\ndomain = -3, 3\n")
    assert cfg == {"h": 0.5, "scheme": "LODIE2", "domain": (-3.0, 3.0)}
    with pytest.raises(ValueError, match="unknown key"):
        pb.parse_config("bogus = 1\n")


def test_thomas_and_assemble_line():
    sys_ = pb.TriDiagSystem(np.array([0., -1., -1.]), np.full(3, 2.0), np.array([-1., -1., 0.]),
                            np.array([1., 0., 1.]))
    assert np.allclose(pb.thomas_solve(sys_), 1.0)
    with pytest.raises(ValueError, match="singular"):
        pb.thomas_solve(pb.TriDiagSystem(np.array([0., 1.]), np.array([0., 1.]),
                                         np.array([1., 0.]), np.array([1., 1.])))


def test_synthetic_config_generator_pinned():
    a = configs.synthetic_atoms(500, 12.0, 1002)
    assert len(a) == 500
    assert abs(sum(x[3] for x in a) - 2.0) < 1e-12
    assert all(1.2 <= x[4] <= 2.0 for x in a)
    assert max(np.linalg.norm(x[:3]) for x in a) <= 12.0
    lo, hi = configs.cubic_box(a, 129, 0.5)
    g = pb.make_grid(lo, hi, 0.5)
    assert g.shape == (129, 129, 129)
    sizes = configs.batch_sizes()
    assert len(sizes) == 64 and min(sizes) >= 200 and max(sizes) <= 800


def test_device_entry_points_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = pb.make_grid((0, 0, 0), (1, 1, 1), 0.5)
    with pytest.raises(RuntimeError, match="CUDA"):
        pb.build_region_maps(g, pb.AnalyticSphere(0.3), 1.0, 80.0, 1.0)
