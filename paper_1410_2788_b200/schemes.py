"""Time stepping: the pseudo-transient LOD / AOS / MAOS step on the device.

API mirror of pbsplit/schemes.py.  `march`, `step`, `Stepper.step`, `ie_sweep`, `cn_sweep`,
`nonlinear_step` and `source_step` run the hand-written sm_100a kernels of libpbg.so
(north_star items 2-4); there is no CPU fallback.  The comparison schemes ADI1/ADI2/
ExplicitEuler use the same device march (schemes_extra.cu).
"""

from __future__ import annotations

import ctypes
import enum
import threading
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .grid import ScalarField

_CLIP = float(np.nextafter(1.0, 0.0))
_INTERIOR = (slice(1, -1),) * 3


class SchemeVariant(str, enum.Enum):
    LODIE1 = "LODIE1"
    LODIE2 = "LODIE2"
    LODCN1 = "LODCN1"
    LODCN2 = "LODCN2"
    AOSIE1 = "AOSIE1"
    AOSIE2 = "AOSIE2"
    AOSCN1 = "AOSCN1"
    AOSCN2 = "AOSCN2"
    MAOSIE = "MAOSIE"
    MAOSCN = "MAOSCN"
    ADI1 = "ADI1"
    ADI2 = "ADI2"
    ExplicitEuler = "ExplicitEuler"


SCHEME_NAMES = tuple(v.value for v in SchemeVariant)
SPLITTING_SCHEMES = tuple(n for n in SCHEME_NAMES if n.startswith(("LOD", "AOS", "MAOS")))
DEVICE_SCHEMES = SCHEME_NAMES


def parse_variant(name) -> SchemeVariant:
    try:
        return SchemeVariant(name)
    except ValueError:
        raise ValueError(f"unknown scheme {name!r}; valid schemes: {', '.join(SCHEME_NAMES)}") \
            from None


@dataclass
class MarchConfig:
    """Pseudo-time marching parameters (schemes.py:49-76)."""

    dt: float
    T: float
    variant: SchemeVariant
    alpha: float | None = None
    divergence_threshold: float = 1e12
    aos_nonlinear: str = "exact"

    def __post_init__(self):
        if self.dt <= 0:
            raise ValueError("dt must be positive")
        if self.T < self.dt:
            raise ValueError("T must be at least dt")
        if self.alpha is not None and self.alpha <= 0:
            raise ValueError("alpha must be positive")
        if self.aos_nonlinear not in ("exact", "literal"):
            raise ValueError("aos_nonlinear must be 'exact' or 'literal'")
        self.variant = parse_variant(self.variant)


@dataclass
class MarchReport:
    final: ScalarField
    steps_taken: int
    diverged: bool
    diverged_step: int | None
    wall_time: float


# ---------------------------------------------------------------------------------------
# Device problem: codes (+ source bit), palette, pitched rho and Dirichlet faces.


class DeviceProblem:
    def __init__(self, problem):
        g = problem.grid
        self.grid = g
        self.gs = nat.grid_struct(g)
        rcodes, pal = problem.region._device_codes()
        self.pal = pal
        self.rho = problem.rho._device()
        codes = rcodes.clone()
        nat.check(nat.lib().pbg_mark_charged(ctypes.byref(self.gs), nat.ptr(self.rho),
                                             nat.ptr(codes), nat.stream_ptr()))
        self.codes = codes
        self.bnd = problem.boundary._device()
        self._plans = {}  # (variant, dt, alpha, literal, threshold) -> pbg_plan, LRU
        self._lock = threading.Lock()  # config-5 batches march one problem from two threads

    _MAX_PLANS = 4

    def plan(self, variant, dt, alpha, aos_literal, threshold):
        """Prepared march (pbg_plan_create: tables, descriptors, segment factors) for this
        problem's codes, built once and reused by every march / step with the same
        constants -- the reference's Stepper factors once (schemes.py:188-262)."""
        key = (nat.VARIANT_IDS[variant], float(dt), float(alpha), bool(aos_literal),
               float(threshold))
        with self._lock:
            return self._plan_locked(key, aos_literal)

    def _plan_locked(self, key, aos_literal):
        h = self._plans.pop(key, None)
        if h is None:
            d = nat.PbgMarchDesc()
            d.grid = self.gs
            d.pal = self.pal
            d.variant = key[0]
            d.aos_literal = 1 if aos_literal else 0
            d.dt, d.alpha, d.divergence_threshold = key[1], key[2], key[4]
            d.nsteps, d.check_divergence = 1, 1
            d.codes = self.codes.data_ptr()
            d.rho = self.rho.data_ptr()
            d.initial = d.work[0] = d.work[1] = self.bnd.data_ptr()  # setup reads none
            out = ctypes.c_void_p()
            nat.check(nat.lib().pbg_plan_create(ctypes.byref(d), ctypes.byref(out),
                                                nat.stream_ptr()))
            h = out
            while len(self._plans) >= self._MAX_PLANS:
                old = self._plans.pop(next(iter(self._plans)))
                nat.lib().pbg_plan_destroy(old, nat.stream_ptr())
        self._plans[key] = h  # most recently used last
        return h

    def __del__(self):
        try:
            for h in self._plans.values():
                nat.load_library().pbg_plan_destroy(h, None)
            self._plans.clear()
        except Exception:
            pass

    def work_pair(self):
        """Two pitched buffers whose faces hold the Dirichlet data."""
        w0 = self.bnd.clone()
        w1 = self.bnd.clone()
        return w0, w1


def _dev_key(problem):
    return (problem.region, problem.region._codes, problem.rho, problem.rho._dev,
            problem.boundary, problem.boundary._dev)


def device_problem(problem) -> DeviceProblem:
    """Device view of an NPBProblem, cached while its components stay device resident."""
    cache = getattr(problem, "_devcache", None)
    key = _dev_key(problem)
    if cache is not None and len(cache[0]) == len(key) and all(
            a is b for a, b in zip(cache[0], key)):
        return cache[1]
    dp = DeviceProblem(problem)
    try:
        problem._devcache = (_dev_key(problem), dp)
    except AttributeError:
        pass
    return dp


def _run_march(problem, variant, dt, alpha, nsteps, threshold, aos_literal, check_div,
               initial_dev=None, work=None):
    v = parse_variant(variant)
    dp = device_problem(problem)
    w0, w1 = work if work is not None else dp.work_pair()
    init = initial_dev if initial_dev is not None else problem.initial._device()
    h = dp.plan(v.value, dt, alpha, aos_literal, threshold)
    taken, dstep, slot = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    ms = ctypes.c_float()
    nat.check(nat.lib().pbg_plan_run(h, nat.ptr(init), nat.ptr(w0), nat.ptr(w1), int(nsteps),
                                     1 if check_div else 0, ctypes.byref(taken),
                                     ctypes.byref(dstep), ctypes.byref(slot), ctypes.byref(ms),
                                     nat.stream_ptr()))
    final = w0 if slot.value == 0 else w1
    return final, taken.value, (dstep.value or None), ms.value / 1e3


def _resolve_alpha(config_alpha, problem):
    return config_alpha if config_alpha is not None else problem.alpha


def march(problem, config: MarchConfig) -> MarchReport:
    """March round(T/dt) steps on the device (schemes.py:399-425).

    Divergence (non-finite or max|u| > threshold) stops the run and is reported as data.
    wall_time is the device time of the step loop (setup excluded, like the reference)."""
    n = int(round(config.T / config.dt))
    n = max(n, 1)
    final, taken, dstep, secs = _run_march(
        problem, config.variant, config.dt, _resolve_alpha(config.alpha, problem), n,
        config.divergence_threshold, config.aos_nonlinear == "literal", True)
    diverged = dstep is not None
    return MarchReport(final=ScalarField._from_device(problem.grid, final, diverged),
                       steps_taken=taken, diverged=diverged, diverged_step=dstep,
                       wall_time=secs)


def _maxabs(grid, dev) -> float:
    out = ctypes.c_double()
    nat.check(nat.lib().pbg_maxabs(ctypes.byref(nat.grid_struct(grid)), nat.ptr(dev),
                                   ctypes.byref(out), nat.stream_ptr()))
    return out.value


def step(variant, state: ScalarField, problem, dt: float, alpha: float | None = None,
         aos_nonlinear: str = "exact", aos_order=(0, 1, 2)) -> ScalarField:
    """One time increment (schemes.py:383-396); non-finite output flags `diverged`.

    AOS branches are combined in axis order, so `aos_order` cannot change the result (the
    reference's order-invariance property, tests/test_schemes.py:268-285)."""
    MarchConfig(dt=dt, T=dt, variant=variant, alpha=alpha, aos_nonlinear=aos_nonlinear)
    if sorted(aos_order) != [0, 1, 2]:
        raise ValueError("aos_order must be a permutation of (0, 1, 2)")
    final, _, _, _ = _run_march(problem, variant, dt, _resolve_alpha(alpha, problem), 1,
                                float("inf"), aos_nonlinear == "literal", False,
                                initial_dev=state._device())
    m = _maxabs(problem.grid, final)
    return ScalarField._from_device(problem.grid, final, diverged=not np.isfinite(m))


class Stepper:
    """Per-march engine (schemes.py:185-380): the device plan (tables, descriptors, segment
    factors) is prepared once here, and each .step(u) only uploads u, launches one step and
    downloads the result.  The region maps stay device resident (nothing is materialised on
    the host)."""

    def __init__(self, problem, config: MarchConfig, aos_order=(0, 1, 2)):
        self.problem = problem
        self.config = config
        self.grid = problem.grid
        self.variant = config.variant
        self.dt = config.dt
        self.alpha = _resolve_alpha(config.alpha, problem)
        self.dta = self.dt / self.alpha
        if sorted(aos_order) != [0, 1, 2]:
            raise ValueError("aos_order must be a permutation of (0, 1, 2)")
        self.aos_order = aos_order
        v = self.variant.value
        self.pm = 4.0 if (v.startswith("AOS") and config.aos_nonlinear == "literal") else 1.0
        self._literal = config.aos_nonlinear == "literal"
        self._dp = device_problem(problem)
        self._dp.plan(v, self.dt, self.alpha, self._literal, float("inf"))
        self._work = self._dp.work_pair()

    @property
    def decay(self):
        """Per-node flow decay (schemes.py:212, 264-270); materialises kappa2 on the host."""
        k2 = self.problem.region.kappa2.data
        if self.variant.value.startswith("AOS") and self.config.aos_nonlinear == "exact":
            return np.exp(-4.0 * k2 * self.dta)
        return np.exp(-k2 * self.dta)

    def _nl(self, u, decay, pm=1.0):
        """Flow stage with the Dirichlet faces re-applied (schemes.py:280-283)."""
        decay = np.asarray(decay, float)
        with np.errstate(divide="ignore"):
            k2eff = -np.log(decay)
        out = nonlinear_step(np.asarray(u, float), k2eff, 1.0, 1.0, premultiplier=pm)
        self.problem.boundary.apply(out)
        return out

    def step(self, u: np.ndarray) -> np.ndarray:
        f = ScalarField(self.grid, u)
        final, _, _, _ = _run_march(self.problem, self.variant, self.dt, self.alpha, 1,
                                    float("inf"), self._literal, False,
                                    initial_dev=f._device(), work=self._work)
        return ScalarField._from_device(self.grid, final).data


def nonlinear_step(w, kappa2, dt: float, alpha: float, premultiplier: float = 1.0,
                   rate: float = 1.0):
    """alpha*w_t = -rate*kappa2*sinh(w) over dt, closed form (schemes.py:106-120), on device."""
    torch = nat.torch_cuda()
    is_field = isinstance(w, ScalarField)
    w_arr = w.data if is_field else np.asarray(w, float)
    k2 = kappa2.data if isinstance(kappa2, ScalarField) else np.asarray(kappa2, float)
    w_arr, k2 = np.broadcast_arrays(np.asarray(w_arr, float), np.asarray(k2, float))
    shape = w_arr.shape
    wd = nat.upload_flat(w_arr.ravel())
    kd = nat.upload_flat(k2.ravel())
    out = torch.empty_like(wd)
    coef = rate * dt / alpha
    nat.check(nat.lib().pbg_flow_dense(wd.numel(), nat.ptr(wd), nat.ptr(kd), float(coef),
                                       float(premultiplier), nat.ptr(out), nat.stream_ptr()))
    res = out.cpu().numpy().reshape(shape)
    if is_field:
        return ScalarField(w.grid, res)
    return res


def delta2_block(u: np.ndarray, region, axis: int) -> np.ndarray:
    """Host helper: eps_plus*(u_plus-u) + eps_minus*(u_minus-u) on the interior block
    (schemes.py:123-143); used by residual checks, not by the device step."""
    eps = region.eps_half(axis)
    c = u[_INTERIOR]
    sp, sm, ep, em = ([slice(1, -1)] * 3 for _ in range(4))
    sp[axis], sm[axis] = slice(2, None), slice(0, -2)
    ep[axis], em[axis] = slice(1, None), slice(0, -1)
    return eps[tuple(ep)] * (u[tuple(sp)] - c) + eps[tuple(em)] * (u[tuple(sm)] - c)


def _single_sweep(axis, field: ScalarField, factor, cn, region, boundary):
    g = field.grid
    gs = nat.grid_struct(g)
    codes, pal = region._device_codes()
    bnd = boundary._device()
    dst = bnd.clone()
    nat.check(nat.lib().pbg_sweep(ctypes.byref(gs), ctypes.byref(pal), nat.ptr(codes), int(axis),
                                  float(factor), 1 if cn else 0, nat.ptr(field._device()),
                                  nat.ptr(bnd), nat.ptr(dst), nat.stream_ptr()))
    return ScalarField._from_device(g, dst)


def ie_sweep(axis: int, rhs: ScalarField, c: float, dt: float, alpha: float, region,
             boundary) -> ScalarField:
    """Solve (1 - c*dt/alpha * d2_axis) out = rhs on every line (schemes.py:146-158)."""
    return _single_sweep(axis, rhs, c * dt / alpha, False, region, boundary)


def cn_sweep(axis: int, field: ScalarField, c: float, dt: float, alpha: float, region,
             boundary) -> ScalarField:
    """Crank-Nicolson half-and-half sweep (schemes.py:161-176)."""
    return _single_sweep(axis, field, 0.5 * c * dt / alpha, True, region, boundary)


def source_step(field: ScalarField, qsource: ScalarField, dt: float, alpha: float,
                fraction: float = 1.0) -> ScalarField:
    """out = field + fraction*(dt/alpha)*qsource (schemes.py:179-182), on device."""
    g = field.grid
    out = nat.new_field(g)
    nat.check(nat.lib().pbg_axpby(ctypes.byref(nat.grid_struct(g)), 1.0, nat.ptr(field._device()),
                                  float(fraction * (dt / alpha)), nat.ptr(qsource._device()),
                                  nat.ptr(out), nat.stream_ptr()))
    return ScalarField._from_device(g, out)
