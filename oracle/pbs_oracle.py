"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of the reference `pbsplit` hot path (arXiv 1410.2788 time-splitting NPB
solver), written from the reference's behaviour and cited file:line by file:line
(`pbsplit/X.py` = /root/reference/pkg/src/pbsplit/X.py).  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline / `--impl reference` legs may
import it, and only as the checker or the timed CPU baseline.

Parity pinning: `tests/golden/make_golden.py` runs the real reference (importable in the
build container) on seeded inputs and stores the results as `tests/golden/*.npz`;
`tests/test_oracle_golden.py` checks this module against them (bit-exact for assembly,
<= 1e-13 relative for marches — the reference's numba Thomas and this module's numpy
Thomas perform the same IEEE operations, so they normally agree exactly).

Arithmetic order follows the reference operation by operation (e.g. `(f*e)*b` fold-ins,
`((dx*dx + dy*dy) + dz*dz)` distances), so assembly is bit-identical.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# pbsplit/constants.py:6-17
KCAL_PER_DIMENSIONLESS = 0.592183
KAPPA2_PER_MOLAR = 8.486902807
C_ES = 332.0636 / KCAL_PER_DIMENSIONLESS
FOUR_PI = 4.0 * np.pi
CLIP = float(np.nextafter(1.0, 0.0))  # pbsplit/schemes.py:16

VARIANTS = ("LODIE1", "LODIE2", "LODCN1", "LODCN2", "AOSIE1", "AOSIE2", "AOSCN1",
            "AOSCN2", "MAOSIE", "MAOSCN")


# ---------------------------------------------------------------------------------------
# Grid and geometry


@dataclass
class OGrid:
    lo: tuple
    h: float
    shape: tuple

    def coords(self, axis):  # pbsplit/grid.py:39-41
        return self.lo[axis] + self.h * np.arange(self.shape[axis])

    def half_coords(self, axis):  # pbsplit/geometry.py:117-119
        return self.coords(axis)[:-1] + 0.5 * self.h


def grid_from_bounds(lo, hi, h):
    """make_grid (pbsplit/grid.py:101-125) without the error paths."""
    lo = tuple(float(v) for v in lo)
    hi = tuple(float(v) for v in hi)
    n = tuple(int(round((hi[d] - lo[d]) / h)) + 1 for d in range(3))
    return OGrid(lo, float(h), n)


def _mesh_axes(g: OGrid, half_axis):
    return [g.half_coords(d) if d == half_axis else g.coords(d) for d in range(3)]


def union_of_spheres_mask(g: OGrid, atoms, probe, half_axis=None):
    """UnionOfSpheres.solute_mask on one mesh (pbsplit/geometry.py:78-85, 122-133).

    Bounding-box culled: each atom only tests the mesh points inside its index box, with
    the reference's exact expression d2 = ((dx*dx + dy*dy) + dz*dz) <= rr*rr.
    """
    ax = _mesh_axes(g, half_axis)
    shape = tuple(len(a) for a in ax)
    mask = np.zeros(shape, dtype=bool)
    h = g.h
    for (cx, cy, cz, _q, rad) in atoms:
        c = (cx, cy, cz)
        rr = rad + probe
        sl = []
        for d in range(3):
            i0 = max(0, int(math.floor((c[d] - rr - g.lo[d]) / h)) - 2)
            i1 = min(shape[d], int(math.ceil((c[d] + rr - g.lo[d]) / h)) + 3)
            sl.append((i0, i1))
        if any(a >= b for a, b in sl):
            continue
        dx = ax[0][sl[0][0]:sl[0][1]] - c[0]
        dy = ax[1][sl[1][0]:sl[1][1]] - c[1]
        dz = ax[2][sl[2][0]:sl[2][1]] - c[2]
        d2 = (dx[:, None, None] ** 2 + dy[None, :, None] ** 2) + dz[None, None, :] ** 2
        mask[sl[0][0]:sl[0][1], sl[1][0]:sl[1][1], sl[2][0]:sl[2][1]] |= d2 <= rr * rr
    return mask


def analytic_sphere_mask(g: OGrid, R, half_axis=None):
    """AnalyticSphere.solute_mask (pbsplit/geometry.py:58-60)."""
    ax = _mesh_axes(g, half_axis)
    r2 = (ax[0][:, None, None] ** 2 + ax[1][None, :, None] ** 2) + ax[2][None, None, :] ** 2
    return r2 <= R * R


@dataclass
class ORegion:
    eps_node: np.ndarray
    eps_half: tuple
    kappa2: np.ndarray


def region_from_masks(masks, eps_m, eps_s, kappa2_solvent):
    """build_region_maps (pbsplit/geometry.py:135-156)."""
    node, hx, hy, hz = masks
    eps_node = np.where(node, eps_m, eps_s)
    kappa2 = np.where(eps_node == eps_m, 0.0, kappa2_solvent)
    halves = tuple(np.where(mk, eps_m, eps_s) for mk in (hx, hy, hz))
    return ORegion(eps_node, halves, kappa2)


def union_region(g, atoms, eps_m, eps_s, kappa2_solvent, probe=0.0):
    masks = [union_of_spheres_mask(g, atoms, probe, ha) for ha in (None, 0, 1, 2)]
    return region_from_masks(masks, eps_m, eps_s, kappa2_solvent)


def sphere_region(g, R, eps_m, eps_s, kappa2_solvent):
    masks = [analytic_sphere_mask(g, R, ha) for ha in (None, 0, 1, 2)]
    return region_from_masks(masks, eps_m, eps_s, kappa2_solvent)


def uniform_region(g, eps, kappa2=0.0):
    """uniform_region (pbsplit/geometry.py:159-169)."""
    n0, n1, n2 = g.shape
    return ORegion(np.full(g.shape, float(eps)),
                   (np.full((n0 - 1, n1, n2), float(eps)), np.full((n0, n1 - 1, n2), float(eps)),
                    np.full((n0, n1, n2 - 1), float(eps))),
                   np.full(g.shape, float(kappa2)))


def deposit(g: OGrid, atoms, prefactor=FOUR_PI * C_ES):
    """deposit_charges (pbsplit/grid.py:205-252): returns (qfrac, rho)."""
    pos = np.array([a[:3] for a in atoms], dtype=float)
    q = np.array([a[3] for a in atoms], dtype=float)
    t = (pos - np.asarray(g.lo)) / g.h
    cell = np.floor(t).astype(np.int64)
    frac = t - cell
    snap = frac >= 1.0 - 1e-12
    cell[snap] += 1
    frac[snap] = 0.0
    n = np.asarray(g.shape)
    bad = np.any((cell < 1) | ((cell > n - 3) & ~((cell == n - 2) & (frac == 0.0))), axis=1)
    if np.any(bad):
        raise ValueError(f"atom {int(np.argmax(bad))} is not strictly inside the grid interior")
    qfrac = np.zeros(g.shape)
    for di in (0, 1):
        wx = frac[:, 0] if di else 1.0 - frac[:, 0]
        for dj in (0, 1):
            wy = frac[:, 1] if dj else 1.0 - frac[:, 1]
            for dk in (0, 1):
                wz = frac[:, 2] if dk else 1.0 - frac[:, 2]
                np.add.at(qfrac, (cell[:, 0] + di, cell[:, 1] + dj, cell[:, 2] + dk),
                          q * (wx * wy * wz))
    return qfrac, (prefactor / g.h ** 3) * qfrac


def coulomb_values(points, atoms, eps_s, kappa_bar):
    """coulomb_screened_values (pbsplit/problem.py:106-117)."""
    total = np.zeros(points.shape[0])
    damp = kappa_bar / math.sqrt(eps_s)
    for (cx, cy, cz, qa, _r) in atoms:
        d = np.sqrt(np.sum((points - np.asarray((cx, cy, cz))) ** 2, axis=-1))
        if np.any(d == 0.0):
            raise ValueError("boundary point coincides with an atom center")
        total += qa / d * np.exp(-damp * d)
    return (C_ES / eps_s) * total


def faces_from_function(g: OGrid, fn):
    """BoundarySpec.from_function (pbsplit/problem.py:44-61): grid-shaped, faces filled."""
    values = np.zeros(g.shape)
    co = [g.coords(d) for d in range(3)]
    for d in range(3):
        p0, p1 = [p for p in range(3) if p != d]
        A, B = np.meshgrid(co[p0], co[p1], indexing="ij")
        pts = np.zeros(A.shape + (3,))
        pts[..., p0] = A
        pts[..., p1] = B
        for side, c in ((0, co[d][0]), (-1, co[d][-1])):
            pts[..., d] = c
            sl = [slice(None)] * 3
            sl[d] = side
            values[tuple(sl)] = fn(pts.reshape(-1, 3)).reshape(A.shape)
    return values


def apply_faces(dst, bvals):
    """BoundarySpec.apply (pbsplit/problem.py:63-69)."""
    for d in range(3):
        for side in (0, -1):
            sl = [slice(None)] * 3
            sl[d] = side
            dst[tuple(sl)] = bvals[tuple(sl)]


@dataclass
class OProblem:
    grid: OGrid
    region: ORegion
    rho: np.ndarray
    qfrac: np.ndarray
    bvals: np.ndarray
    alpha: float
    initial: np.ndarray
    eps_m: float = 1.0
    eps_s: float = 80.0
    kappa_bar: float = 0.0
    atoms: list = field(default_factory=list)


def protein_on_grid(g: OGrid, atoms, eps_m, eps_s, kappa_bar, alpha=1.0, probe=0.0):
    """protein_problem's assembly (pbsplit/problem.py:221-234) on a given grid."""
    region = union_region(g, atoms, eps_m, eps_s, kappa_bar ** 2, probe)
    qfrac, rho = deposit(g, atoms, FOUR_PI * C_ES)
    bvals = faces_from_function(g, lambda p: coulomb_values(p, atoms, eps_s, kappa_bar))
    init = np.zeros(g.shape)
    apply_faces(init, bvals)
    return OProblem(g, region, rho, qfrac, bvals, alpha, init, eps_m, eps_s, kappa_bar,
                    list(atoms))


def protein_bbox_grid(atoms, h, padding):
    """Box rule of protein_problem (pbsplit/problem.py:206-211)."""
    pos = np.array([a[:3] for a in atoms])
    lo = pos.min(axis=0) - padding
    hi = pos.max(axis=0) + padding
    cells = np.maximum(2, np.ceil((hi - lo) / h - 1e-12).astype(int))
    hi = lo + cells * h
    return grid_from_bounds(lo, hi, h)


def vacuum_of(p: OProblem):
    """make_vacuum_problem (pbsplit/problem.py:237-257)."""
    g = p.grid
    region = uniform_region(g, p.eps_m, 0.0)
    bvals = faces_from_function(g, lambda q: coulomb_values(q, p.atoms, p.eps_m, 0.0))
    init = np.zeros(g.shape)
    apply_faces(init, bvals)
    return OProblem(g, region, p.rho, p.qfrac, bvals, p.alpha, init, p.eps_m, p.eps_m, 0.0,
                    p.atoms)


# ---------------------------------------------------------------------------------------
# Time stepping

INT = (slice(1, -1),) * 3


def sinh_flow(w, decay, pm=1.0):
    """_apply_flow (pbsplit/schemes.py:88-103)."""
    t = np.tanh(0.5 * w) * decay
    np.clip(t, -CLIP, CLIP, out=t)
    out = 2.0 * np.arctanh(t)
    ident = decay >= 1.0
    if np.any(ident):
        out = np.where(ident, w, out)
    if pm != 1.0:
        out = pm * out
    return out


def _axis_blocks(arr, axis, lo_sl, hi_sl):
    """Interior block of an eps_half array with the sweep axis sliced and moved first."""
    sl = [slice(1, -1)] * 3
    sl[axis] = slice(lo_sl, hi_sl)
    return np.moveaxis(arr[tuple(sl)], axis, 0)


class LineFactors:
    """Prefactored (1 - factor*d2_axis) over all interior lines (pbsplit/tridiag.py:158-206)."""

    def __init__(self, g: OGrid, region: ORegion, bvals, axis, factor):
        self.axis = axis
        m = g.shape[axis] - 2
        self.m = m
        f = float(factor) / g.h ** 2
        em = _axis_blocks(region.eps_half[axis], axis, 0, m)
        ep = _axis_blocks(region.eps_half[axis], axis, 1, m + 1)
        self.bshape = em.shape
        L = em.shape[1] * em.shape[2]
        em = np.ascontiguousarray(em.reshape(m, L))
        ep = np.ascontiguousarray(ep.reshape(m, L))
        diag = 1.0 + f * (ep + em)
        self.sub = -f * em
        sup = -f * ep
        self.cp = np.empty_like(diag)
        self.inv = np.empty_like(diag)
        self.inv[0] = 1.0 / diag[0]
        self.cp[0] = sup[0] * self.inv[0]
        for i in range(1, m):
            self.inv[i] = 1.0 / (diag[i] - self.sub[i] * self.cp[i - 1])
            self.cp[i] = sup[i] * self.inv[i]
        lo = [slice(1, -1)] * 3
        hi = [slice(1, -1)] * 3
        lo[axis] = 0
        hi[axis] = -1
        self.fold_lo = (f * em[0].reshape(self.bshape[1:]) * bvals[tuple(lo)]).reshape(L)
        self.fold_hi = (f * ep[-1].reshape(self.bshape[1:]) * bvals[tuple(hi)]).reshape(L)

    def solve(self, rhs_int):
        """rhs_int: interior-shaped block in grid axis order; returns the same shape."""
        m = self.m
        blk = np.moveaxis(rhs_int, self.axis, 0).reshape(m, -1).copy()
        blk[0] += self.fold_lo
        blk[-1] += self.fold_hi
        dp = np.empty_like(blk)
        dp[0] = blk[0] * self.inv[0]
        for i in range(1, m):
            dp[i] = (blk[i] - self.sub[i] * dp[i - 1]) * self.inv[i]
        out = np.empty_like(blk)
        out[m - 1] = dp[m - 1]
        for i in range(m - 2, -1, -1):
            out[i] = dp[i] - self.cp[i] * out[i + 1]
        return np.moveaxis(out.reshape(self.bshape), 0, self.axis)


def delta2(u, eps_half, axis):
    """delta2_block (pbsplit/schemes.py:123-143)."""
    c = u[INT]
    up = [slice(1, -1)] * 3
    um = [slice(1, -1)] * 3
    up[axis] = slice(2, None)
    um[axis] = slice(0, -2)
    ep = [slice(1, -1)] * 3
    em = [slice(1, -1)] * 3
    ep[axis] = slice(1, None)
    em[axis] = slice(0, -1)
    return eps_half[tuple(ep)] * (u[tuple(up)] - c) + eps_half[tuple(em)] * (u[tuple(um)] - c)


# variant -> (family, factor multiple of dta, cn, source coefficients)  schemes.py:209-262
PLANS = {
    "LODIE1": ("lod1", 1.0, False, None),
    "LODIE2": ("lod2", 1.0, False, None),
    "LODCN1": ("lod1", 0.5, True, None),
    "LODCN2": ("lod2", 0.5, True, None),
    "AOSIE1": ("aos", 4.0, False, (4.0, 0.0, 0.0)),
    "AOSIE2": ("aos", 4.0, False, (4.0 / 3.0, 4.0 / 3.0, 4.0 / 3.0)),
    "AOSCN1": ("aos", 2.0, True, (4.0, 0.0, 0.0)),
    "AOSCN2": ("aos", 2.0, True, (4.0 / 3.0, 4.0 / 3.0, 4.0 / 3.0)),
    "MAOSIE": ("maos", 3.0, False, (1.0, 1.0, 1.0)),
    "MAOSCN": ("maos", 1.5, True, (1.0, 1.0, 1.0)),
}


EXTRA_PLANS = {"ADI1": "adi1", "ADI2": "adi2", "ExplicitEuler": "euler"}


class OStepper:
    """Stepper (pbsplit/schemes.py:185-380) for the LOD/AOS/MAOS families."""

    def __init__(self, p: OProblem, variant, dt, alpha=None, aos_nonlinear="exact"):
        self.p = p
        self.variant = variant
        if variant in EXTRA_PLANS:  # comparison schemes (schemes.py:240-253)
            self._init_extra(p, variant, dt, alpha)
            return
        self.family, mult, self.cn, self.src = PLANS[variant]
        self.alpha = alpha if alpha is not None else p.alpha
        self.dta = dt / self.alpha
        self.h2 = p.grid.h ** 2
        k2 = p.region.kappa2
        self.fac = [LineFactors(p.grid, p.region, p.bvals, a, mult * self.dta) for a in range(3)]
        self.cn_f = mult * self.dta
        self.pm = 1.0
        if self.family == "aos" and aos_nonlinear == "exact":
            self.decay = np.exp(-4.0 * k2 * self.dta)
        else:
            self.decay = np.exp(-k2 * self.dta)
            if self.family == "aos":
                self.pm = 4.0
        self.rho_int = p.rho[INT]

    def _faces(self, interior):
        out = np.empty(self.p.grid.shape)
        out[INT] = interior
        apply_faces(out, self.p.bvals)
        return out

    def _nl(self, u, pm=1.0):
        out = sinh_flow(u, self.decay, pm)
        apply_faces(out, self.p.bvals)
        return out

    def _sweep(self, u, axis, extra=None):
        rhs = u[INT]
        if self.cn:
            rhs = rhs + (self.cn_f / self.h2) * delta2(u, self.p.region.eps_half[axis], axis)
        if extra is not None:
            rhs = rhs + extra
        return self._faces(self.fac[axis].solve(rhs))

    def _init_extra(self, p, variant, dt, alpha):
        self.family = EXTRA_PLANS[variant]
        self.alpha = alpha if alpha is not None else p.alpha
        self.dta = dt / self.alpha
        self.h2 = p.grid.h ** 2
        k2 = p.region.kappa2
        self.rho_int = p.rho[INT]
        self.cn = False
        if variant == "ADI1":
            self.fac = [LineFactors(p.grid, p.region, p.bvals, a, self.dta) for a in range(3)]
            self.decay = np.exp(-k2 * self.dta)
        elif variant == "ADI2":
            self.fac = [LineFactors(p.grid, p.region, p.bvals, a, 0.5 * self.dta)
                        for a in range(3)]
            self.decay = np.exp(-0.5 * k2 * self.dta)
        else:
            self.k2_int = k2[INT]
            self.ion_mask = self.k2_int > 0.0

    def _d2(self, w, axis):
        return delta2(w, self.p.region.eps_half[axis], axis) / self.h2

    def _step_extra(self, u):
        fam = self.family
        if fam == "adi1":  # schemes.py:331-342
            w = self._nl(u)
            sy, sz = self._d2(w, 1), self._d2(w, 2)
            u1 = self._faces(self.fac[0].solve(w[INT] + self.dta * (sy + sz + self.rho_int)))
            u2 = self._faces(self.fac[1].solve(u1[INT] - self.dta * sy))
            return self._faces(self.fac[2].solve(u2[INT] - self.dta * sz))
        if fam == "adi2":  # schemes.py:344-353
            w = self._nl(u)
            sx, sy, sz = self._d2(w, 0), self._d2(w, 1), self._d2(w, 2)
            rhs = w[INT] + self.dta * (0.5 * sx + sy + sz + self.rho_int)
            v1 = self._faces(self.fac[0].solve(rhs))
            v2 = self._faces(self.fac[1].solve(v1[INT] - 0.5 * self.dta * sy))
            v3 = self._faces(self.fac[2].solve(v2[INT] - 0.5 * self.dta * sz))
            return self._nl(v3)
        # explicit Euler, schemes.py:355-363
        r = self.p.region
        lap = (delta2(u, r.eps_half[0], 0) + delta2(u, r.eps_half[1], 1)
               + delta2(u, r.eps_half[2], 2)) / self.h2
        ui = u[INT]
        react = np.zeros_like(ui)
        m = self.ion_mask
        react[m] = self.k2_int[m] * np.sinh(ui[m])
        return self._faces(ui + self.dta * (lap - react + self.rho_int))

    def step(self, u):
        with np.errstate(over="ignore", invalid="ignore", under="ignore"):
            if self.variant in EXTRA_PLANS:
                return self._step_extra(u)
            fam = self.family
            if fam in ("lod1", "lod2"):  # schemes.py:301-311
                if fam == "lod2":
                    w = u + self.dta * self.p.rho
                else:
                    w = self._nl(u)
                for axis in range(3):
                    w = self._sweep(w, axis)
                return self._nl(w) if fam == "lod2" else w + self.dta * self.p.rho
            if fam == "aos":  # schemes.py:313-323
                w = self._nl(u, self.pm)
                b = []
                for axis in range(3):
                    c = self.src[axis]
                    b.append(self._sweep(u, axis, c * self.dta * self.rho_int if c else None)[INT])
                return self._faces(0.25 * (w[INT] + b[0] + b[1] + b[2]))
            w = self._nl(u)  # MAOS, schemes.py:325-329
            extra = self.dta * self.rho_int
            b = [self._sweep(w, axis, extra)[INT] for axis in range(3)]
            return self._faces((b[0] + b[1] + b[2]) / 3.0)


@dataclass
class OReport:
    final: np.ndarray
    steps_taken: int
    diverged: bool
    diverged_step: int | None


def n_steps(T, dt):
    """schemes.py:406-408."""
    return max(1, int(round(T / dt)))


def march(p: OProblem, variant, dt, T, alpha=None, threshold=1e12, aos_nonlinear="exact"):
    """march (pbsplit/schemes.py:399-425)."""
    st = OStepper(p, variant, dt, alpha, aos_nonlinear)
    u = p.initial.copy()
    for k in range(1, n_steps(T, dt) + 1):
        u = st.step(u)
        amax = np.max(np.abs(u))
        if not np.isfinite(amax) or amax > threshold:
            return OReport(u, k, True, k)
    return OReport(u, n_steps(T, dt), False, None)


def solvation_energy(qfrac, phi_m, phi_0):
    """solvation_energy (pbsplit/energy.py:31-43)."""
    return float(0.5 * np.sum(qfrac * (phi_m - phi_0)) * KCAL_PER_DIMENSIONLESS)


def richardson(phi_dt, phi_half):
    """richardson (pbsplit/energy.py:99-106)."""
    return 2.0 * phi_half - phi_dt


def energy_replusv(p: OProblem, variant, dt, T, alpha=None, aos_nonlinear="exact"):
    """energy_pipeline(variant="REplusV") (pbsplit/energy.py:109-164).

    Returns (delta_g, phi_m, phi_0, diverged)."""
    r1 = march(p, variant, dt, T, alpha, aos_nonlinear=aos_nonlinear)
    r2 = march(p, variant, 0.5 * dt, T, alpha, aos_nonlinear=aos_nonlinear)
    vac = vacuum_of(p)
    v1 = march(vac, "LODIE2", dt, T, alpha)
    v2 = march(vac, "LODIE2", 0.5 * dt, T, alpha)
    phi_m = richardson(r1.final, r2.final)
    phi_0 = richardson(v1.final, v2.final)
    div = any(r.diverged for r in (r1, r2, v1, v2))
    dg = float("nan") if div else solvation_energy(p.qfrac, phi_m, phi_0)
    return dg, phi_m, phi_0, div


def _const_laplacian_interior(u):
    """pbsplit/energy.py:46-56 (same accumulation order)."""
    c = u[INT]
    out = -6.0 * c
    out += u[2:, 1:-1, 1:-1]
    out += u[:-2, 1:-1, 1:-1]
    out += u[1:-1, 2:, 1:-1]
    out += u[1:-1, :-2, 1:-1]
    out += u[1:-1, 1:-1, 2:]
    out += u[1:-1, 1:-1, :-2]
    return out


def vacuum_potential_fast(rho, g: OGrid, eps_m, bvals):
    """vacuum_potential_fast (pbsplit/energy.py:59-85): boundary lifting, type-I DST
    diagonalisation of the 7-point operator, eigenvalue divide, inverse DST."""
    import scipy.fft

    gg = np.zeros(g.shape)
    apply_faces(gg, bvals)
    rhs = rho[INT] + (eps_m / g.h ** 2) * _const_laplacian_interior(gg)
    lam_1d = []
    for d in range(3):
        n = g.shape[d]
        m = np.arange(1, n - 1)
        lam_1d.append(4.0 * np.sin(np.pi * m / (2.0 * (n - 1))) ** 2)
    lam = (eps_m / g.h ** 2) * (lam_1d[0][:, None, None] + lam_1d[1][None, :, None]
                                + lam_1d[2][None, None, :])
    psi = scipy.fft.idstn(scipy.fft.dstn(rhs, type=1) / lam, type=1)
    out = gg
    out[INT] = psi
    return out


def energy_direct(p: OProblem, variant, dt, T, mode="Plain", alpha=None,
                  aos_nonlinear="exact"):
    """energy_pipeline(variant="Plain" | "RE") (pbsplit/energy.py:109-164): solvent march
    (or its Richardson pair) against the direct vacuum solve."""
    if mode == "Plain":
        r = march(p, variant, dt, T, alpha, aos_nonlinear=aos_nonlinear)
        phi_m, div = r.final, r.diverged
    else:
        r1 = march(p, variant, dt, T, alpha, aos_nonlinear=aos_nonlinear)
        r2 = march(p, variant, 0.5 * dt, T, alpha, aos_nonlinear=aos_nonlinear)
        phi_m, div = richardson(r1.final, r2.final), r1.diverged or r2.diverged
    phi_0 = vacuum_potential_fast(p.rho, p.grid, p.eps_m, vacuum_of(p).bvals)
    dg = float("nan") if div else solvation_energy(p.qfrac, phi_m, phi_0)
    return dg, phi_m, phi_0, div
