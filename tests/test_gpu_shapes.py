"""Ragged and extreme line lengths: every tile geometry (P = 4/8/16/32 segments, S from 2 to
32, padding segments, row tiles, the longest supported line m = 1024, the single-node grid)
against the CPU oracle on an off-centre dielectric sphere with a random sparse source and
random Dirichlet faces; lines longer than 1024 interior nodes are refused loudly."""

import numpy as np
import pytest

import paper_1410_2788_b200 as pb
from oracle import pbs_oracle as O
from tests.helpers import rel_err

pytestmark = pytest.mark.gpu

SHAPES = [(3, 3, 3), (4, 5, 6), (18, 19, 20), (131, 10, 9), (9, 260, 11), (7, 8, 600),
          (6, 390, 5), (1026, 5, 5), (66, 9, 20), (8, 59, 21), (50, 7, 36), (77, 8, 30), (9, 70, 19), (152, 6, 20), (7, 180, 18)]
VARIANTS = ["LODIE1", "LODCN2", "AOSCN1", "MAOSIE", "ADI2"]


def problems(shape, seed=0, faces=1.0, source=5.0):
    h = 0.25
    lo = (-0.35 * (shape[0] - 1) * h, -0.6 * (shape[1] - 1) * h, -0.45 * (shape[2] - 1) * h)
    hi = tuple(lo[a] + (shape[a] - 1) * h for a in range(3))
    g = pb.make_grid(lo, hi, h)
    assert g.shape == shape
    R = 0.3 * min(hi[a] - lo[a] for a in range(3)) + 0.3
    rng = np.random.default_rng(seed)
    bvals = faces * rng.standard_normal(shape)
    rho = np.zeros(shape)
    idx = tuple(rng.integers(1, max(2, s - 1), size=7) for s in shape)
    rho[idx] = rng.standard_normal(7) * source
    region = pb.build_region_maps(g, pb.AnalyticSphere(R), 2.0, 80.0, 1.3)
    init = np.zeros(shape)
    bspec = pb.BoundarySpec(g, bvals)
    bspec.apply(init)
    p = pb.NPBProblem(grid=g, region=region, rho=pb.ScalarField(g, rho),
                      qfrac=pb.ScalarField.zeros(g), boundary=bspec, alpha=1.0,
                      initial=pb.ScalarField(g, init), eps_m=2.0, eps_s=80.0, kappa_bar=1.14)
    og = O.OGrid(g.lo, g.h, shape)
    op = O.OProblem(og, O.sphere_region(og, R, 2.0, 80.0, 1.3), rho, np.zeros(shape), bvals,
                    1.0, init.copy(), 2.0, 80.0, 1.14)
    return p, op


@pytest.mark.parametrize("shape", SHAPES)
def test_ragged_shapes_vs_oracle(shape):
    p, op = problems(shape)
    for v in VARIANTS:
        rep = pb.march(p, pb.MarchConfig(dt=0.2, T=0.6, variant=v))
        orep = O.march(op, v, 0.2, 0.6)
        assert rep.steps_taken == orep.steps_taken == 3, v
        assert rel_err(rep.final.data, orep.final) <= 1e-12, (shape, v)


def test_line_longer_than_supported_is_refused():
    g = pb.make_grid((0, 0, 0), (0.25 * 1026, 0.75, 0.75), 0.25)  # m = 1025 along x
    p = pb.NPBProblem(grid=g, region=pb.uniform_region(g, 1.0, 0.0),
                      rho=pb.ScalarField.zeros(g), qfrac=pb.ScalarField.zeros(g),
                      boundary=pb.BoundarySpec(g, np.zeros(g.shape)), alpha=1.0,
                      initial=pb.ScalarField.zeros(g), eps_m=1.0, eps_s=1.0)
    with pytest.raises(NotImplementedError):
        pb.march(p, pb.MarchConfig(dt=0.1, T=0.1, variant="LODIE2"))


# Row-warp sweeps (axis 2 lines of 32*S - 1, 16*S - 1 or 8*S - 1 interior rows: one, two or
# four lines per warp, a line count off the multiple leaves part of a warp idle) with each
# LOD epilogue, against the oracle.
RW_SHAPES = [(5, 6, 513), (7, 9, 257), (6, 5, 129), (4, 5, 257), (5, 6, 97), (7, 9, 97)]


@pytest.mark.parametrize("shape", RW_SHAPES)
def test_row_warp_lines_vs_oracle(shape):
    p, op = problems(shape, seed=1)
    for v in ["LODIE1", "LODIE2", "ADI1", "LODCN2", "AOSIE1"]:
        rep = pb.march(p, pb.MarchConfig(dt=0.2, T=0.6, variant=v))
        orep = O.march(op, v, 0.2, 0.6)
        assert rep.steps_taken == orep.steps_taken == 3, v
        assert rel_err(rep.final.data, orep.final) <= 1e-12, (shape, v)


@pytest.mark.parametrize("shape", [(5, 6, 513), (7, 9, 257), (7, 9, 129), (7, 9, 97)])
def test_row_warp_divergence_vs_oracle(shape):
    # zero faces and a strong source: max|u| grows step by step, so a threshold between the
    # step-2 and step-6 maxima trips inside the march (the row-warp sweep raises the flag);
    # the march must stop at the oracle's step and return that step's field
    p, op = problems(shape, seed=2, faces=0.0, source=500.0)
    for v in ["LODIE2", "LODIE1", "AOSIE1"]:
        amax = [np.max(np.abs(O.march(op, v, 0.2, 0.2 * k).final)) for k in (2, 6)]
        assert amax[1] > amax[0] > 0.0
        thr = 0.5 * (amax[0] + amax[1])
        orep = O.march(op, v, 0.2, 2.0, threshold=thr)
        rep = pb.march(p, pb.MarchConfig(dt=0.2, T=2.0, variant=v, divergence_threshold=thr))
        assert orep.diverged and 2 < orep.steps_taken <= 6, v
        assert rep.diverged and rep.steps_taken == orep.steps_taken, v
        assert rel_err(rep.final.data, orep.final) <= 1e-12, (shape, v)
