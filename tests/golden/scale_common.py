"""Summaries shared by the scale fixtures (make_golden_scale.py) and the tests that read them.

Pure numpy; imports `configs.py` by file path so that callers that must not load the
package (the fixture generator, bench.py's reference arm) can use the seeded generator.
"""

from __future__ import annotations

import hashlib
import importlib.util
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
SAMPLE_SEED = 20261020
SAMPLE_N = 4096


def load_configs():
    """paper_1410_2788_b200/configs.py without importing the package (no libpbg.so)."""
    path = os.path.join(ROOT, "paper_1410_2788_b200", "configs.py")
    spec = importlib.util.spec_from_file_location("_pbg_configs", path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules.setdefault("_pbg_configs", mod)
    spec.loader.exec_module(mod)
    return mod


def mask_digest(mask) -> str:
    """sha256 of a boolean mask (shape-tagged, bit-packed)."""
    m = np.ascontiguousarray(np.asarray(mask, dtype=bool))
    h = hashlib.sha256(np.array(m.shape, dtype=np.int64).tobytes())
    h.update(np.packbits(m.ravel()).tobytes())
    return h.hexdigest()


def sample_index(shape, n=SAMPLE_N, seed=SAMPLE_SEED):
    """Seeded flat indices of interior nodes (the same for a given shape)."""
    rng = np.random.default_rng(seed)
    ijk = [rng.integers(1, s - 1, size=n) for s in shape]
    return np.ravel_multi_index(ijk, shape)


def field_stats(u) -> np.ndarray:
    """(max|u|, sum u, sum u^2) in numpy's own reduction order."""
    u = np.asarray(u)
    return np.array([np.max(np.abs(u)), np.sum(u), np.sum(u * u)])
