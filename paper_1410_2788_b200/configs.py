"""Seeded synthetic inputs for BASELINE.json's five configurations.

The reference ships no generator for these configs, so they are pinned here
and used identically by the oracle, the tests and bench.py.  Pure numpy, no device work.

Generator: centres uniform in a ball of radius R (direction = normalised
N(0, I3), radius = R*U^(1/3)), radii ~ U[1.2, 2.0] A, charges ~ N(0, 0.4) e shifted to a
total of +2 e; atoms in generation order.  Grids are cubic boxes of exactly n nodes centred
on the atom bounding box (effective padding >= 10 A), built with the public make_grid.
Ionic strength -> kappa_bar = sqrt(KAPPA2_PER_MOLAR * I) with the reference's 298 K
constant (constants.py:9).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

KAPPA2_PER_MOLAR = 8.486902807


def synthetic_atoms(n_atoms: int, ball_radius: float, seed: int, q_total: float = 2.0):
    """List of (x, y, z, q, r) tuples."""
    rng = np.random.default_rng(seed)
    dirs = rng.standard_normal((n_atoms, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    rad = ball_radius * rng.uniform(size=n_atoms) ** (1.0 / 3.0)
    centres = dirs * rad[:, None]
    radii = rng.uniform(1.2, 2.0, n_atoms)
    q = rng.normal(0.0, 0.4, n_atoms)
    q = q + (q_total - q.sum()) / n_atoms
    return [(float(c[0]), float(c[1]), float(c[2]), float(qq), float(r))
            for c, qq, r in zip(centres, q, radii)]


def cubic_box(atoms, n: int, h: float):
    """(lo, hi) of a cube with n nodes per axis centred on the atom bounding box."""
    pos = np.array([a[:3] for a in atoms])
    centre = 0.5 * (pos.min(axis=0) + pos.max(axis=0))
    half = 0.5 * h * (n - 1)
    lo = tuple(float(c - half) for c in centre)
    hi = tuple(float(lo[d] + h * (n - 1)) for d in range(3))
    return lo, hi


def kappa_bar(ionic_strength: float) -> float:
    return math.sqrt(KAPPA2_PER_MOLAR * ionic_strength)


@dataclass(frozen=True)
class Config:
    name: str
    n_atoms: int
    ball_radius: float
    seed: int
    n: int
    h: float
    eps_m: float
    eps_s: float
    ionic_strength: float
    variant: str
    dt: float
    steps: int


# Config 1 (Kirkwood) is built by protein_problem with padding 8 (exactly [-8, 8]^3).
KIRKWOOD = dict(h=0.25, padding=8.0, kappa_bar=kappa_bar(0.1), eps_m=1.0, eps_s=80.0,
                dt=0.1, T=20.0)

CONFIGS = {
    "c2": Config("c2-protein500-129", 500, 12.0, 1002, 129, 0.5, 2.0, 80.0, 0.15, "LODIE2",
                 0.5, 100),
    "c3": Config("c3-protein2500-257", 2500, 20.0, 1003, 257, 0.4, 2.0, 80.0, 0.15, "LODIE2",
                 0.5, 100),
    "c4": Config("c4-protein10000-513", 10000, 32.0, 1004, 513, 0.3, 2.0, 80.0, 0.15,
                 "LODIE2", 0.5, 50),
}


def batch_sizes(count: int = 64, seed: int = 1005):
    """Config 5: seeded protein sizes U{200..800}."""
    rng = np.random.default_rng(seed)
    return [int(v) for v in rng.integers(200, 801, size=count)]


def batch_config(index: int, n_atoms: int) -> Config:
    radius = 12.0 * (n_atoms / 500.0) ** (1.0 / 3.0)
    return Config(f"c5-protein{index}", n_atoms, radius, 5000 + index, 97, 0.5, 2.0, 80.0,
                  0.15, "AOSIE1", 0.5, 100)
