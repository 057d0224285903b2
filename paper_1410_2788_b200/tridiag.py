"""Per-line tridiagonal API (pbsplit/tridiag.py:19-112).

These scalar per-line helpers are the reference's own test oracle for the batched sweep
engine (out of scope as kernels); they stay host-side.  The batched engine
(`LineSweepSolver` / `_solve_batch`, tridiag.py:115-219) is replaced by the device sweeps
behind `ie_sweep` / `cn_sweep` / `march` (csrc/sweep.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

PIVOT_FLOOR = 1e-300


@dataclass
class TriDiagSystem:
    """sub[0] and sup[n-1] are unused."""

    sub: np.ndarray
    diag: np.ndarray
    sup: np.ndarray
    rhs: np.ndarray

    def __post_init__(self):
        n = len(self.diag)
        for name in ("sub", "diag", "sup", "rhs"):
            arr = np.ascontiguousarray(getattr(self, name), dtype=np.float64)
            if arr.shape != (n,):
                raise ValueError(f"{name} must have length {n}")
            if not np.all(np.isfinite(arr)):
                raise ValueError(f"{name} contains non-finite entries")
            setattr(self, name, arr)
        if n < 1:
            raise ValueError("system must have at least one unknown")

    def dense(self):
        n = len(self.diag)
        a = np.diag(self.diag)
        if n > 1:
            a += np.diag(self.sub[1:], -1) + np.diag(self.sup[:-1], 1)
        return a


def thomas_solve(system: TriDiagSystem) -> np.ndarray:
    """Forward elimination + back substitution with a near-zero pivot check."""
    b, c, a, r = system.diag, system.sup, system.sub, system.rhs
    n = len(b)
    cp = np.empty(n)
    x = np.empty(n)
    piv = b[0]
    if abs(piv) < PIVOT_FLOOR:
        raise ValueError("singular tridiagonal system (zero pivot at row 0)")
    cp[0] = c[0] / piv if n > 1 else 0.0
    x[0] = r[0] / piv
    for i in range(1, n):
        piv = b[i] - a[i] * cp[i - 1]
        if abs(piv) < PIVOT_FLOOR:
            raise ValueError(f"singular tridiagonal system (zero pivot at row {i})")
        cp[i] = c[i] / piv if i < n - 1 else 0.0
        x[i] = (r[i] - a[i] * x[i - 1]) / piv
    for i in range(n - 2, -1, -1):
        x[i] -= cp[i] * x[i + 1]
    return x


def assemble_line(axis, line_index, region, scale, dt, alpha, rhs_line, boundary_values):
    """(1 - scale*dt/alpha * d2_axis) system of one interior line with Dirichlet folds."""
    g = region.grid
    m = g.shape[axis] - 2
    if m < 1:
        raise ValueError("line has no interior nodes")
    rhs_line = np.asarray(rhs_line, dtype=np.float64)
    if rhs_line.shape != (m,):
        raise ValueError(f"rhs_line must have length {m}")
    eps = region.eps_half(axis)
    idx = list(line_index)
    lo = idx.copy()
    hi = idx.copy()
    lo.insert(axis, slice(0, m))
    hi.insert(axis, slice(1, m + 1))
    e_m = eps[tuple(lo)]
    e_p = eps[tuple(hi)]
    f = scale * dt / (alpha * g.h ** 2)
    rhs = rhs_line.copy()
    b_lo, b_hi = boundary_values
    rhs[0] += f * e_m[0] * b_lo
    rhs[-1] += f * e_p[-1] * b_hi
    return TriDiagSystem(-f * e_m, 1.0 + f * (e_p + e_m), -f * e_p, rhs)
