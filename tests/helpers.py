"""Shared helpers: golden fixtures and matching oracle / device problems."""

from __future__ import annotations

import os

import numpy as np

from oracle import pbs_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def ogrid(d):
    lo = tuple(float(v) for v in d["lo"])
    return O.OGrid(lo, float(d["h"]), tuple(int(v) for v in d["shape"]))


def atoms_of(d, key="atoms"):
    return [tuple(float(v) for v in row) for row in d[key]]


def oracle_protein(d, alpha=1.0):
    g = ogrid(d)
    return O.protein_on_grid(g, atoms_of(d), float(d["eps_m"]), float(d["eps_s"]),
                             float(d["kappa_bar"]), alpha, float(d["probe"]) if "probe" in d
                             else 0.0)


def faces(arr):
    return np.concatenate([arr[0].ravel(), arr[-1].ravel(), arr[:, 0].ravel(),
                           arr[:, -1].ravel(), arr[:, :, 0].ravel(), arr[:, :, -1].ravel()])


def system_of(atoms, label="golden"):
    import paper_1410_2788_b200 as pb

    return pb.MolecularSystem([pb.Atom(a[:3], a[3], a[4]) for a in atoms], label=label)


def rel_err(got, want):
    """max|got - want| / max|want| (the north_star potential parity measure)."""
    got = np.asarray(got)
    want = np.asarray(want)
    scale = np.max(np.abs(want))
    return float(np.max(np.abs(got - want)) / (scale if scale > 0 else 1.0))
