"""Prepared marches (pbg_plan_*): the Stepper factors once and steps cheaply, like the
reference's Stepper (schemes.py:185-262 setup, 365-380 step); results equal march()."""

import ctypes

import numpy as np
import pytest

import paper_1410_2788_b200 as pb
from paper_1410_2788_b200 import _native as nat
from tests.helpers import golden, oracle_protein, rel_err
from oracle import pbs_oracle as O
from tests.test_gpu_parity import protein_from

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("variant", ["LODIE2", "LODIE1", "AOSIE1", "MAOSCN", "ADI1"])
def test_stepper_loop_matches_march_bitwise(variant):
    d = golden("march_variants")
    p = protein_from(d)
    cfg = pb.MarchConfig(dt=0.3, T=1.5, variant=variant)
    rep = pb.march(p, cfg)
    from paper_1410_2788_b200.schemes import Stepper

    st = Stepper(p, cfg)
    assert p.region._codes is not None  # the maps stay on the device
    u = p.initial.data.copy()
    for _ in range(5):
        u = st.step(u)
    assert p.region._codes is not None
    assert np.array_equal(u, rep.final.data)


def test_plan_reused_across_marches_and_runs():
    """Repeated marches reuse one prepared plan per (variant, dt, alpha, threshold); a plan
    run twice from the same initial field reproduces itself bit for bit."""
    d = golden("march_variants")
    p = protein_from(d)
    from paper_1410_2788_b200.schemes import device_problem

    a = pb.march(p, pb.MarchConfig(dt=0.3, T=1.5, variant="LODIE2")).final.data
    dp = device_problem(p)
    n_before = len(dp._plans)
    b = pb.march(p, pb.MarchConfig(dt=0.3, T=1.5, variant="LODIE2")).final.data
    assert len(dp._plans) == n_before
    assert np.array_equal(a, b)
    # a different dt is a different plan; the cache is bounded
    for k in range(6):
        pb.march(p, pb.MarchConfig(dt=0.1 + 0.01 * k, T=0.3, variant="LODIE2"))
    assert len(dp._plans) <= dp._MAX_PLANS


def test_plan_c_abi_run_matches_march():
    d = golden("march_variants")
    p = protein_from(d)
    from paper_1410_2788_b200.schemes import device_problem

    want = pb.march(p, pb.MarchConfig(dt=0.3, T=1.5, variant="LODIE1")).final.data
    dp = device_problem(p)
    desc = nat.PbgMarchDesc()
    desc.grid, desc.pal = dp.gs, dp.pal
    desc.variant = nat.VARIANT_IDS["LODIE1"]
    desc.dt, desc.alpha, desc.divergence_threshold = 0.3, 1.0, 1e12
    desc.nsteps, desc.check_divergence = 5, 1
    desc.codes, desc.rho = dp.codes.data_ptr(), dp.rho.data_ptr()
    w0, w1 = dp.work_pair()
    desc.initial = desc.work[0] = w0.data_ptr()
    desc.work[1] = w1.data_ptr()
    h = ctypes.c_void_p()
    lib = nat.lib()
    nat.check(lib.pbg_plan_create(ctypes.byref(desc), ctypes.byref(h), nat.stream_ptr()))
    try:
        for _ in range(2):
            w0, w1 = dp.work_pair()
            taken, dstep, slot = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
            ms = ctypes.c_float()
            nat.check(lib.pbg_plan_run(h, nat.ptr(w0), nat.ptr(w0), nat.ptr(w1), 5, 1,
                                       ctypes.byref(taken), ctypes.byref(dstep),
                                       ctypes.byref(slot), ctypes.byref(ms), nat.stream_ptr()))
            assert taken.value == 5 and dstep.value == 0
            out = pb.ScalarField._from_device(p.grid, w0 if slot.value == 0 else w1).data
            assert np.array_equal(out, want)
    finally:
        lib.pbg_plan_destroy(h, nat.stream_ptr())
    # invalid arguments are rejected, not crashed on
    assert lib.pbg_plan_run(None, None, None, None, 1, 1, None, None, None, None, None) != 0


def _region_with_values(g, values_x):
    """A user-built RegionMap whose eps_half_x takes the given values in thirds of the box."""
    n0, n1, n2 = g.shape
    ex = np.full((n0 - 1, n1, n2), values_x[0])
    ex[(n0 - 1) // 3:] = values_x[1]
    ex[2 * (n0 - 1) // 3:] = values_x[-1]
    ey = np.full((n0, n1 - 1, n2), 80.0)
    ez = np.full((n0, n1, n2 - 1), 80.0)
    k2 = np.full(g.shape, 0.5)
    return pb.RegionMap(g, pb.ScalarField(g, np.full(g.shape, 80.0)), ex, ey, ez,
                        pb.ScalarField(g, k2))


def _problem(region):
    g = region.grid
    rng = np.random.default_rng(3)
    b = rng.standard_normal(g.shape)
    rho = np.zeros(g.shape)
    rho[1:-1, 1:-1, 1:-1] = rng.standard_normal(tuple(s - 2 for s in g.shape))
    return pb.NPBProblem(grid=g, region=region, rho=pb.ScalarField(g, rho),
                         qfrac=pb.ScalarField.zeros(g), boundary=pb.BoundarySpec(g, b),
                         alpha=1.0, initial=pb.ScalarField(g, b.copy()))


def test_user_region_two_arbitrary_values_vs_oracle():
    g = pb.make_grid((0, 0, 0), (3.0, 2.5, 3.5), 0.25)
    p = _problem(_region_with_values(g, (3.0, 45.0, 45.0)))
    r = p.region
    og = O.OGrid(g.lo, g.h, g.shape)
    oreg = O.ORegion(r.eps_node.data, (r.eps_half_x, r.eps_half_y, r.eps_half_z),
                     r.kappa2.data)
    op = O.OProblem(og, oreg, p.rho.data, np.zeros(g.shape), p.boundary.values, 1.0,
                    p.initial.data)
    for v in ("LODIE2", "AOSIE1"):
        rep = pb.march(p, pb.MarchConfig(dt=0.2, T=0.6, variant=v))
        orep = O.march(op, v, 0.2, 0.6)
        assert rel_err(rep.final.data, orep.final) <= 1e-12, v


def test_user_region_more_than_two_values_fails_early_and_clearly():
    """The device encodes two values per coefficient map (build_region_maps never makes
    more); a user map with three is refused with NotImplementedError before any step."""
    from paper_1410_2788_b200.schemes import Stepper

    g = pb.make_grid((0, 0, 0), (3.0, 2.5, 3.5), 0.25)
    p = _problem(_region_with_values(g, (3.0, 45.0, 80.0)))
    cfg = pb.MarchConfig(dt=0.2, T=0.6, variant="LODIE2")
    with pytest.raises(NotImplementedError, match="more than two distinct values"):
        pb.march(p, cfg)
    with pytest.raises(NotImplementedError, match="more than two distinct values"):
        Stepper(p, cfg)
