"""Uniform 3D grids, scalar fields, relative norms, charge deposition.

API mirror of pbsplit/grid.py.  `ScalarField` keeps the reference's fields
(`grid`, `data`, `diverged`) but may be backed by a pitched device buffer: `.data`
downloads on first host access and from then on the host array is authoritative (callers
may mutate it in place, as the reference allows).  `deposit_charges` runs on the device
(north_star item 1, pbsplit/grid.py:205-252).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .constants import C_ES

FOUR_PI = 4.0 * np.pi


@dataclass(frozen=True)
class Grid3D:
    """Uniform Cartesian grid (pbsplit/grid.py:14-98); flat index (i*ny + j)*nz + k."""

    lo: tuple
    hi: tuple
    h: float
    nx: int
    ny: int
    nz: int

    @property
    def shape(self):
        return (self.nx, self.ny, self.nz)

    @property
    def num_nodes(self):
        return self.nx * self.ny * self.nz

    def axis_coords(self, axis):
        return self.lo[axis] + self.h * np.arange(self.shape[axis])

    @property
    def x(self):
        return self.axis_coords(0)

    @property
    def y(self):
        return self.axis_coords(1)

    @property
    def z(self):
        return self.axis_coords(2)

    def node_mesh(self):
        return np.meshgrid(self.x, self.y, self.z, indexing="ij", sparse=True)

    def radii(self, floor: float = 0.0):
        X, Y, Z = self.node_mesh()
        r = np.sqrt(X * X + Y * Y + Z * Z)
        return np.maximum(r, floor) if floor > 0.0 else r

    def flat_index(self, i, j, k):
        return (np.asarray(i) * self.ny + np.asarray(j)) * self.nz + np.asarray(k)

    def unflatten(self, flat):
        flat = np.asarray(flat)
        ij, k = np.divmod(flat, self.nz)
        i, j = np.divmod(ij, self.ny)
        return i, j, k

    def origin_index(self):
        out = []
        for d in range(3):
            t = -self.lo[d] / self.h
            i = int(round(t))
            if abs(t - i) > 1e-9 or not 0 <= i < self.shape[d]:
                raise ValueError("coordinate origin is not a grid node")
            out.append(i)
        return tuple(out)

    def boundary_mask(self):
        m = np.zeros(self.shape, dtype=bool)
        m[[0, -1], :, :] = True
        m[:, [0, -1], :] = True
        m[:, :, [0, -1]] = True
        return m


def make_grid(lo, hi, h: float) -> Grid3D:
    """Grid with node coordinates lo + i*h; rejects non-commensurate bounds (grid.py:101-125)."""
    lo = tuple(float(v) for v in lo)
    hi = tuple(float(v) for v in hi)
    if h <= 0:
        raise ValueError(f"spacing must be positive, got h={h}")
    n = []
    for d in range(3):
        if hi[d] <= lo[d]:
            raise ValueError(f"axis {d}: hi={hi[d]} must exceed lo={lo[d]}")
        cells = (hi[d] - lo[d]) / h
        whole = round(cells)
        if abs(cells - whole) > 1e-9:
            raise ValueError(f"axis {d}: extent {hi[d] - lo[d]} is not an integer multiple "
                             f"of h={h} (got {cells} cells)")
        if whole < 2:
            raise ValueError(f"axis {d}: need at least 2 cells (3 nodes), got {whole}")
        n.append(int(whole) + 1)
    return Grid3D(lo, hi, h, *n)


class ScalarField:
    """Node-indexed fp64 field over a Grid3D, optionally device resident (grid.py:128-152)."""

    def __init__(self, grid: Grid3D, data=None, diverged: bool = False):
        self.grid = grid
        self.diverged = diverged
        self._dev = None
        self._host = None
        if data is not None:
            self.data = data

    # -- host view ---------------------------------------------------------------------
    @property
    def data(self) -> np.ndarray:
        if self._host is None:
            if self._dev is None:
                raise ValueError("field has no data")
            self._host = nat.download_dense(self.grid, self._dev)
        self._dev = None  # the host array is authoritative from here on
        return self._host

    @data.setter
    def data(self, value):
        arr = np.ascontiguousarray(value, dtype=np.float64)
        if arr.shape != self.grid.shape:
            raise ValueError(f"data shape {arr.shape} does not match grid {self.grid.shape}")
        self._host = arr
        self._dev = None

    # -- device view -------------------------------------------------------------------
    @classmethod
    def _from_device(cls, grid, dev, diverged=False):
        f = cls(grid, None, diverged)
        f._dev = dev
        return f

    def _device(self):
        """Pitched device buffer with the current values (uploads host data if needed)."""
        if self._dev is None:
            self._dev = nat.upload_dense(self.grid, self._host)
        return self._dev

    @property
    def _on_device(self):
        return self._dev is not None and self._host is None

    @classmethod
    def zeros(cls, grid):
        return cls(grid, np.zeros(grid.shape))

    def copy(self):
        if self._on_device:
            return ScalarField._from_device(self.grid, self._dev.clone(), self.diverged)
        return ScalarField(self.grid, self.data.copy(), self.diverged)

    def __repr__(self):
        where = "device" if self._on_device else "host"
        return f"ScalarField(grid={self.grid}, {where}, diverged={self.diverged})"


@dataclass(frozen=True)
class NormPair:
    l2: float
    linf: float


def relative_norms(exact: ScalarField, approx: ScalarField, exclude=None) -> NormPair:
    """Relative L2 / Linf of approx against exact (grid.py:161-186)."""
    if exact.grid != approx.grid:
        raise ValueError("fields live on different grids")
    e, a = exact.data, approx.data
    if exclude is not None:
        keep = ~np.asarray(exclude, dtype=bool)
        e, a = e[keep], a[keep]
    e = np.asarray(e, float)
    a = np.asarray(a, float)
    diff = e - a
    emax = np.max(np.abs(e))
    if emax == 0.0:
        raise ValueError("relative norms undefined: exact field is identically zero")
    return NormPair(float(np.sqrt(np.sum(diff * diff) / np.sum(e * e))),
                    float(np.max(np.abs(diff)) / emax))


def trilinear_weights(frac: np.ndarray):
    """((di, dj, dk), w) for the 8 cell corners (grid.py:189-202)."""
    f = [frac[..., 0], frac[..., 1], frac[..., 2]]
    for di in (0, 1):
        wx = f[0] if di else 1.0 - f[0]
        for dj in (0, 1):
            wy = f[1] if dj else 1.0 - f[1]
            for dk in (0, 1):
                wz = f[2] if dk else 1.0 - f[2]
                yield (di, dj, dk), wx * wy * wz


def _deposit_device(system, grid, prefactor, codes=None):
    """Device deposit; returns (qfrac_dev, rho_dev, atoms_dev)."""
    if not system.atoms:
        raise ValueError("system has no atoms")
    atoms_dev, atoms_host = nat.atoms_array(system)
    qf = nat.new_field(grid)
    rho = nat.new_field(grid)
    rc = nat.lib().pbg_deposit(ctypes.byref(nat.grid_struct(grid)), nat.ptr(atoms_dev),
                               len(system.atoms), float(prefactor), nat.ptr(qf), nat.ptr(rho),
                               nat.ptr(codes), nat.stream_ptr())
    if rc == -1:
        msg = nat.lib().pbg_last_error().decode()
        m = nat._ERR_RE.search(msg)
        if m:
            a = int(m.group(1))
            pos = tuple(float(v) for v in atoms_host[a, :3])
            raise ValueError(f"atom {a} at {pos} is not strictly inside the grid interior")
    nat.check(rc)
    return qf, rho, atoms_dev


def deposit_charges(system, grid: Grid3D, prefactor: float = FOUR_PI * C_ES):
    """Trilinear spreading on the device -> (qfrac, rho) ScalarFields (grid.py:205-252)."""
    qf, rho, _ = _deposit_device(system, grid, prefactor)
    q = ScalarField._from_device(grid, qf)
    r = ScalarField._from_device(grid, rho)
    q._deposit_of = system
    return q, r


def dump_field_csv(field: ScalarField, path) -> None:
    """One node per line, i,j,k,x,y,z,value with 12 significant digits (grid.py:255-267)."""
    g = field.grid
    xs, ys, zs = g.x, g.y, g.z
    data = field.data
    with open(path, "w") as fh:
        fh.write("i,j,k,x,y,z,value\n")
        for i in range(g.nx):
            for j in range(g.ny):
                for k in range(g.nz):
                    fh.write(f"{i},{j},{k},{xs[i]:.12e},{ys[j]:.12e},{zs[k]:.12e},"
                             f"{data[i, j, k]:.12e}\n")
