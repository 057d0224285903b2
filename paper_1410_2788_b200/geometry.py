"""Molecules, solute surfaces and the dielectric / ion coefficient maps.

API mirror of pbsplit/geometry.py.  `build_region_maps` classifies the node mesh and the
three half-edge meshes on the device (north_star item 1) straight into 1-byte node codes;
`RegionMap` exposes the reference's dense arrays lazily (expanded on the device and
downloaded on first host access).
"""

from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .grid import Grid3D, ScalarField


class Region(enum.Enum):
    SOLUTE = "solute"
    SOLVENT = "solvent"


@dataclass(frozen=True)
class Atom:
    """Point charge with a radius (geometry.py:13-27)."""

    center: tuple
    charge: float
    radius: float

    def __post_init__(self):
        object.__setattr__(self, "center", tuple(float(c) for c in self.center))
        if not all(np.isfinite(self.center)):
            raise ValueError("atom center must be finite")
        if not np.isfinite(self.charge):
            raise ValueError("atom charge must be finite")
        if not (self.radius > 0):
            raise ValueError(f"atom radius must be positive, got {self.radius}")


@dataclass
class MolecularSystem:
    atoms: list = field(default_factory=list)
    label: str = "system"

    def __len__(self):
        return len(self.atoms)

    def total_charge(self) -> float:
        return float(sum(a.charge for a in self.atoms))


@dataclass(frozen=True)
class AnalyticSphere:
    """Closed ball of radius R at the origin (geometry.py:48-60)."""

    R: float

    def __post_init__(self):
        if not (self.R > 0):
            raise ValueError("sphere radius must be positive")

    def solute_mask(self, pts):
        p = np.asarray(pts, float)
        return np.sum(p ** 2, axis=-1) <= self.R * self.R


@dataclass(frozen=True)
class UnionOfSpheres:
    """Union of atom balls inflated by probe_inflation (geometry.py:63-85)."""

    system: MolecularSystem
    probe_inflation: float = 0.0

    def __post_init__(self):
        if self.probe_inflation < 0:
            raise ValueError("probe_inflation must be >= 0")

    def solute_mask(self, pts):
        """Host evaluation for arbitrary points (classify / tests); the grid maps use the
        device kernel in build_region_maps."""
        p = np.asarray(pts, float)
        mask = np.zeros(p.shape[:-1], dtype=bool)
        for a in self.system.atoms:
            rr = a.radius + self.probe_inflation
            mask |= np.sum((p - np.asarray(a.center)) ** 2, axis=-1) <= rr * rr
        return mask


Surface = AnalyticSphere | UnionOfSpheres


def classify(point, surface) -> Region:
    inside = surface.solute_mask(np.asarray(point, float).reshape(1, 3))[0]
    return Region.SOLUTE if inside else Region.SOLVENT


class RegionMap:
    """eps at nodes / half-edge midpoints and nodal kappa2 (geometry.py:97-114).

    Either host arrays (reference behaviour) or device codes + two-value palettes.  Host
    arrays are produced on demand; once materialised they are authoritative, and the
    device codes are rebuilt from them (pbg_pack_region) on the next device use.
    """

    def __init__(self, grid, eps_node, eps_half_x, eps_half_y, eps_half_z, kappa2):
        self.grid = grid
        self._h = dict(eps_node=eps_node, eps_half_x=np.asarray(eps_half_x, float),
                       eps_half_y=np.asarray(eps_half_y, float),
                       eps_half_z=np.asarray(eps_half_z, float), kappa2=kappa2)
        self._codes = None
        self._pal = None
        self._node_pal = None

    @classmethod
    def _from_codes(cls, grid, codes, palette, node_pal):
        r = cls.__new__(cls)
        r.grid = grid
        r._h = None
        r._codes = codes
        r._pal = palette
        r._node_pal = tuple(float(v) for v in node_pal)
        return r

    def _materialize(self):
        if self._h is None:
            torch = nat.torch_cuda()
            g = self.grid
            n0, n1, n2 = g.shape
            mk = lambda *s: torch.empty(s, dtype=torch.float64, device="cuda")
            en, ex, ey, ez, k2 = mk(n0, n1, n2), mk(n0 - 1, n1, n2), mk(n0, n1 - 1, n2), \
                mk(n0, n1, n2 - 1), mk(n0, n1, n2)
            npal = (ctypes.c_double * 2)(*self._node_pal)
            nat.check(nat.lib().pbg_expand_region(
                ctypes.byref(nat.grid_struct(g)), nat.ptr(self._codes), ctypes.byref(self._pal),
                npal, nat.ptr(en), nat.ptr(ex), nat.ptr(ey), nat.ptr(ez), nat.ptr(k2),
                nat.stream_ptr()))
            self._h = dict(eps_node=ScalarField(g, en.cpu().numpy()), eps_half_x=ex.cpu().numpy(),
                           eps_half_y=ey.cpu().numpy(), eps_half_z=ez.cpu().numpy(),
                           kappa2=ScalarField(g, k2.cpu().numpy()))
        self._codes = None  # host is authoritative now
        return self._h

    eps_node = property(lambda self: self._materialize()["eps_node"])
    eps_half_x = property(lambda self: self._materialize()["eps_half_x"])
    eps_half_y = property(lambda self: self._materialize()["eps_half_y"])
    eps_half_z = property(lambda self: self._materialize()["eps_half_z"])
    kappa2 = property(lambda self: self._materialize()["kappa2"])

    def eps_half(self, axis: int):
        return (self.eps_half_x, self.eps_half_y, self.eps_half_z)[axis]

    def _device_codes(self):
        """(codes uint8 pitched device tensor with bits 0-3, PbgPalette)."""
        if self._codes is None:
            h = self._h
            g = self.grid
            k2 = h["kappa2"].data if isinstance(h["kappa2"], ScalarField) else h["kappa2"]
            arrs = [nat.upload_flat(np.ascontiguousarray(a, dtype=np.float64))
                    for a in (h["eps_half_x"], h["eps_half_y"], h["eps_half_z"], k2)]
            codes = nat.new_codes(g)
            pal = nat.PbgPalette()
            nat.check(nat.lib().pbg_pack_region(
                ctypes.byref(nat.grid_struct(g)), nat.ptr(arrs[0]), nat.ptr(arrs[1]),
                nat.ptr(arrs[2]), nat.ptr(arrs[3]), None, nat.ptr(codes), ctypes.byref(pal),
                nat.stream_ptr()))
            self._codes, self._pal = codes, pal
        return self._codes, self._pal


def build_region_maps(grid: Grid3D, surface, eps_m: float, eps_s: float,
                      kappa2_solvent: float) -> RegionMap:
    """Device classification of nodes and half-edge midpoints (geometry.py:135-156)."""
    if eps_m <= 0 or eps_s <= 0:
        raise ValueError("dielectric constants must be positive")
    if kappa2_solvent < 0:
        raise ValueError("kappa2_solvent must be >= 0")
    codes = nat.new_codes(grid)
    pal = nat.PbgPalette()
    gs = nat.grid_struct(grid)
    if isinstance(surface, AnalyticSphere):
        nat.check(nat.lib().pbg_classify_sphere(ctypes.byref(gs), float(surface.R), float(eps_m),
                                                float(eps_s), float(kappa2_solvent),
                                                nat.ptr(codes), ctypes.byref(pal),
                                                nat.stream_ptr()))
    elif isinstance(surface, UnionOfSpheres):
        n = len(surface.system.atoms)
        atoms = nat.atoms_array(surface.system)[0] if n else None
        nat.check(nat.lib().pbg_classify_spheres(
            ctypes.byref(gs), nat.ptr(atoms), n, float(surface.probe_inflation), float(eps_m),
            float(eps_s), float(kappa2_solvent), 0, nat.ptr(codes), ctypes.byref(pal),
            nat.stream_ptr()))
    else:
        raise TypeError(f"unsupported surface type {type(surface).__name__}")
    return RegionMap._from_codes(grid, codes, pal, (eps_s, eps_m))


def uniform_region(grid: Grid3D, eps: float, kappa2: float = 0.0) -> RegionMap:
    """Single-medium map (geometry.py:159-169), device resident (all codes zero)."""
    pal = nat.PbgPalette.make([(eps, eps)] * 3, (kappa2, kappa2))
    return RegionMap._from_codes(grid, nat.new_codes(grid), pal, (eps, eps))


def parse_pqr(text) -> MolecularSystem:
    """ATOM/HETATM records; last five fields x y z q r (geometry.py:172-196)."""
    if isinstance(text, bytes):
        text = text.decode("utf-8", errors="replace")
    atoms = []
    for lineno, line in enumerate(text.splitlines(), start=1):
        f = line.split()
        if not f or f[0] not in ("ATOM", "HETATM"):
            continue
        if len(f) < 6:
            raise ValueError(f"PQR line {lineno}: record has too few fields")
        try:
            x, y, z, q, r = (float(v) for v in f[-5:])
        except ValueError:
            raise ValueError(f"PQR line {lineno}: last five fields are not all numeric") from None
        atoms.append(Atom((x, y, z), q, r))
    if not atoms:
        raise ValueError("no atoms parsed from PQR input")
    return MolecularSystem(atoms, label="pqr")


def parse_system_table(text, label: str = "synthetic") -> MolecularSystem:
    """`atom x y z q r` lines with # comments (geometry.py:199-221)."""
    if isinstance(text, bytes):
        text = text.decode("utf-8")
    atoms = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        f = line.split()
        if f[0] != "atom" or len(f) != 6:
            raise ValueError(f"system line {lineno}: expected 'atom x y z q r'")
        try:
            x, y, z, q, r = (float(v) for v in f[1:])
        except ValueError:
            raise ValueError(f"system line {lineno}: non-numeric field") from None
        atoms.append(Atom((x, y, z), q, r))
    if not atoms:
        raise ValueError("no atoms parsed from system input")
    return MolecularSystem(atoms, label=label)
