"""CPU checks of the flow interval table and the small-argument polynomial the sweep kernels
evaluate (pbg_flow_table / pbg_flow_small, host only): the piecewise polynomial, evaluated the way the device does, against the oracle's
restatement of _apply_flow (pbsplit/schemes.py:88-103) and an extended-precision value."""

import ctypes

import mpmath as mp
import numpy as np
import pytest

from oracle import pbs_oracle as O
from paper_1410_2788_b200 import _native as nat

N = 1008


def table(decay):
    lib = nat.load_library()
    out = np.zeros(N, dtype=np.float64)
    nat.check(lib.pbg_flow_table(decay, out.ctypes.data_as(ctypes.c_void_p)))
    return out.reshape(84, 12)


def poly_eval(w, T):
    """Device evaluation (pbg_internal.cuh flow_poly) in numpy."""
    x = np.abs(w)
    hi = ((x + 1.0).view(np.int64) >> 32).astype(np.int64)
    idx = (hi >> 16) - 0x3FF0
    rows = T[idx]
    t = x - rows[:, 0]
    p = rows[:, 10]
    for q in range(9, 0, -1):
        p = p * t + rows[:, q]
    return np.copysign(p, w)


def samples(seed=0):
    rng = np.random.default_rng(seed)
    w = np.concatenate([rng.uniform(-38, 38, 20000), rng.uniform(-4, 4, 20000),
                        rng.uniform(-1e-3, 1e-3, 2000), [0.0, -0.0, 38.0, -38.0, 1e-300]])
    # interval edges in |w| + 1 = 2^e (1 + s/16), and their neighbours
    e = np.array([np.ldexp(1 + s / 16, k) - 1 for k in range(6) for s in range(16)])
    e = e[e <= 38.0]
    return np.concatenate([w, e, np.nextafter(e, 0), np.nextafter(e, 40), -e])


@pytest.mark.parametrize("decay", [0.529131809679411, 0.6541980527948197, 0.880466373414563,
                                   0.9186325916063356, 0.1, 1e-3, 0.0])
def test_flow_table_matches_reference_flow(decay):
    T = table(decay)
    w = samples()
    got = poly_eval(w, T)
    ref = O.sinh_flow(w, decay)
    # the reference's own tanh/atanh evaluation errs by up to ~1.5e-15 at d = 0.92
    assert np.max(np.abs(got - ref)) <= 4e-15
    mp.mp.dps = 30
    sub = w[::97]
    exact = np.array([float(2 * mp.atanh(decay * mp.tanh(mp.mpf(v) / 2))) for v in sub])
    assert np.max(np.abs(poly_eval(sub, T) - exact)) <= 1e-15


def test_flow_table_near_one_decay():
    # d -> 1 sharpens the knee at w ~ 2 artanh(d); the reference itself loses digits there
    decay = 0.99
    T = table(decay)
    w = samples(1)
    mp.mp.dps = 30
    sub = w[::53]
    exact = np.array([float(2 * mp.atanh(decay * mp.tanh(mp.mpf(v) / 2))) for v in sub])
    assert np.max(np.abs(poly_eval(sub, T) - exact)) <= 5e-15
    assert np.max(np.abs(poly_eval(w, T) - O.sinh_flow(w, decay))) <= 5e-14


def test_flow_table_rejects_bad_decay():
    lib = nat.load_library()
    out = np.zeros(N)
    for d in (1.0, 1.5, -0.1, float("nan")):
        assert lib.pbg_flow_table(d, out.ctypes.data_as(ctypes.c_void_p)) != 0


def small(decay):
    lib = nat.load_library()
    out = np.zeros(16, dtype=np.float64)
    nat.check(lib.pbg_flow_small(decay, out.ctypes.data_as(ctypes.c_void_p)))
    return out


def small_eval(w, g):
    """Device evaluation (pbg_internal.cuh flow_small) in numpy, |w| <= 2."""
    t = w * w - 2.0
    p = np.full_like(w, g[-1])
    for q in g[-2::-1]:
        p = p * t + q
    return w * p


@pytest.mark.parametrize("decay", [0.529131809679411, 0.6541980527948197, 0.880466373414563,
                                   0.9186325916063356, 0.99, 0.1, 1e-3, 0.0])
def test_flow_small_matches_reference_flow(decay):
    g = small(decay)
    rng = np.random.default_rng(3)
    w = np.concatenate([rng.uniform(-2, 2, 20000), rng.uniform(-1e-3, 1e-3, 2000),
                        [0.0, -0.0, 2.0, -2.0, 1e-300, np.nextafter(2.0, 0)]])
    got = small_eval(w, g)
    assert np.max(np.abs(got - O.sinh_flow(w, decay))) <= 4e-15
    mp.mp.dps = 30
    sub = w[::41]
    exact = np.array([float(2 * mp.atanh(decay * mp.tanh(mp.mpf(v) / 2))) for v in sub])
    err = np.abs(small_eval(sub, g) - exact)
    # ~1 ulp relative (numpy has no fma; the device Horner is fused)
    assert np.max(err / np.maximum(np.abs(exact), 1e-300)) <= 1e-15
    assert np.max(err) <= 1e-15
    # the small form and the table agree where both apply
    if decay > 0:
        T = table(decay)
        assert np.max(np.abs(got - poly_eval(w, T))) <= 1e-15


def test_flow_small_rejects_bad_decay():
    lib = nat.load_library()
    out = np.zeros(16)
    for d in (1.0, -0.1, float("nan")):
        assert lib.pbg_flow_small(d, out.ctypes.data_as(ctypes.c_void_p)) != 0


def tiny(decay):
    lib = nat.load_library()
    out = np.zeros(8, dtype=np.float64)
    nat.check(lib.pbg_flow_tiny(decay, out.ctypes.data_as(ctypes.c_void_p)))
    return out


def tiny_eval(w, g):
    """Device evaluation (pbg_internal.cuh flow_tiny) in numpy, |w| <= 0.5."""
    t = w * w - 0.125
    p = np.full_like(w, g[-1])
    for q in g[-2::-1]:
        p = p * t + q
    return w * p


@pytest.mark.parametrize("decay", [0.529131809679411, 0.6541980527948197, 0.880466373414563,
                                   0.9186325916063356, 0.99, 0.1, 1e-3, 0.0])
def test_flow_tiny_matches_reference_flow(decay):
    g = tiny(decay)
    rng = np.random.default_rng(4)
    w = np.concatenate([rng.uniform(-0.5, 0.5, 20000), rng.uniform(-1e-3, 1e-3, 2000),
                        [0.0, -0.0, 0.5, -0.5, 1e-300, np.nextafter(0.5, 0)]])
    got = tiny_eval(w, g)
    assert np.max(np.abs(got - O.sinh_flow(w, decay))) <= 4e-15
    mp.mp.dps = 30
    sub = w[::41]
    exact = np.array([float(2 * mp.atanh(decay * mp.tanh(mp.mpf(v) / 2))) for v in sub])
    err = np.abs(tiny_eval(sub, g) - exact)
    assert np.max(err / np.maximum(np.abs(exact), 1e-300)) <= 1e-15
    if decay > 0:  # agrees with the small-argument form where both apply
        assert np.max(np.abs(got - small_eval(w, small(decay)))) <= 1e-16


def test_flow_tiny_rejects_bad_decay():
    lib = nat.load_library()
    out = np.zeros(8)
    for d in (1.0, -0.1, float("nan")):
        assert lib.pbg_flow_tiny(d, out.ctypes.data_as(ctypes.c_void_p)) != 0
