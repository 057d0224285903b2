"""ctypes binding of the C ABI in include/pbg.h (libpbg.so, built in-tree for sm_100a).

This is the only module that touches the native library.  There is no fallback: if the
library or a CUDA device is missing, every device entry point raises RuntimeError.
Device memory and streams come from PyTorch (plumbing only; no torch ops on the path
except allocation and host<->device copies).
"""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PBG_LIB") or os.path.join(_HERE, "_lib", "libpbg.so")  # PBG_LIB: A/B builds

PBG_OFFSET = 31
VARIANT_IDS = {"LODIE1": 0, "LODIE2": 1, "LODCN1": 2, "LODCN2": 3, "AOSIE1": 4, "AOSIE2": 5,
               "AOSCN1": 6, "AOSCN2": 7, "MAOSIE": 8, "MAOSCN": 9, "ADI1": 10, "ADI2": 11,
               "ExplicitEuler": 12}

c_int32, c_int64, c_double, c_void_p = (ctypes.c_int32, ctypes.c_int64, ctypes.c_double,
                                        ctypes.c_void_p)


class PbgGrid(ctypes.Structure):
    _fields_ = [("n", c_int32 * 3), ("pitch", c_int64), ("lo", c_double * 3), ("h", c_double)]


class PbgPalette(ctypes.Structure):
    _fields_ = [("eps", (c_double * 2) * 3), ("kappa2", c_double * 2)]

    def as_tuple(self):
        return (tuple(tuple(self.eps[a][b] for b in range(2)) for a in range(3)),
                tuple(self.kappa2[b] for b in range(2)))

    @classmethod
    def make(cls, eps, kappa2):
        p = cls()
        for a in range(3):
            for b in range(2):
                p.eps[a][b] = float(eps[a][b])
        for b in range(2):
            p.kappa2[b] = float(kappa2[b])
        return p


class PbgMarchDesc(ctypes.Structure):
    _fields_ = [("grid", PbgGrid), ("pal", PbgPalette), ("variant", c_int32),
                ("aos_literal", c_int32), ("dt", c_double), ("alpha", c_double),
                ("divergence_threshold", c_double), ("nsteps", c_int32),
                ("check_divergence", c_int32), ("codes", c_void_p), ("rho", c_void_p),
                ("initial", c_void_p), ("work", c_void_p * 2)]


_P = ctypes.POINTER
_SIGS = {
    "pbg_version": ([], ctypes.c_int),
    "pbg_last_error": ([], ctypes.c_char_p),
    "pbg_layout": ([c_int32, c_int32, c_int32, _P(c_int64), _P(c_int64)], ctypes.c_int),
    "pbg_pitch_from_dense": ([_P(PbgGrid), c_void_p, c_void_p, c_void_p], ctypes.c_int),
    "pbg_dense_from_pitched": ([_P(PbgGrid), c_void_p, c_void_p, c_void_p], ctypes.c_int),
    "pbg_copy_faces": ([_P(PbgGrid), c_void_p, c_void_p, c_void_p], ctypes.c_int),
    "pbg_unpack_faces": ([_P(PbgGrid), c_void_p, c_void_p, c_void_p, c_void_p], ctypes.c_int),
    "pbg_pack_region": ([_P(PbgGrid), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                         c_void_p, _P(PbgPalette), c_void_p], ctypes.c_int),
    "pbg_expand_region": ([_P(PbgGrid), c_void_p, _P(PbgPalette), _P(c_double), c_void_p,
                           c_void_p, c_void_p, c_void_p, c_void_p, c_void_p], ctypes.c_int),
    "pbg_classify_spheres": ([_P(PbgGrid), c_void_p, c_int32, c_double, c_double, c_double,
                              c_double, c_int32, c_void_p, _P(PbgPalette), c_void_p],
                             ctypes.c_int),
    "pbg_classify_sphere": ([_P(PbgGrid), c_double, c_double, c_double, c_double, c_void_p,
                             _P(PbgPalette), c_void_p], ctypes.c_int),
    "pbg_deposit": ([_P(PbgGrid), c_void_p, c_int32, c_double, c_void_p, c_void_p, c_void_p,
                     c_void_p], ctypes.c_int),
    "pbg_mark_charged": ([_P(PbgGrid), c_void_p, c_void_p, c_void_p], ctypes.c_int),
    "pbg_coulomb_faces": ([_P(PbgGrid), c_void_p, c_int32, c_double, c_double, c_void_p,
                           c_void_p], ctypes.c_int),
    "pbg_march": ([_P(PbgMarchDesc), _P(c_int32), _P(c_int32), _P(c_int32),
                   _P(ctypes.c_float), c_void_p], ctypes.c_int),
    "pbg_march_host": ([_P(PbgMarchDesc), c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                        c_void_p, c_void_p, _P(c_int32), _P(c_int32), _P(ctypes.c_float),
                        c_void_p], ctypes.c_int),
    "pbg_sweep": ([_P(PbgGrid), _P(PbgPalette), c_void_p, c_int32, c_double, c_int32,
                   c_void_p, c_void_p, c_void_p, c_void_p], ctypes.c_int),
    "pbg_flow_dense": ([c_int64, c_void_p, c_void_p, c_double, c_double, c_void_p, c_void_p],
                       ctypes.c_int),
    "pbg_flow_table": ([c_double, c_void_p], ctypes.c_int),
    "pbg_flow_small": ([c_double, c_void_p], ctypes.c_int),
    "pbg_flow_tiny": ([c_double, c_void_p], ctypes.c_int),
    "pbg_energy_atoms": ([_P(PbgGrid), c_void_p, c_int32, c_void_p, c_void_p, c_double,
                          c_double, c_void_p, c_void_p, c_double, c_double, c_double,
                          _P(c_double), c_void_p], ctypes.c_int),
    "pbg_energy_dense": ([_P(PbgGrid), c_void_p, c_void_p, c_void_p, c_double, _P(c_double),
                          c_void_p], ctypes.c_int),
    "pbg_axpby": ([_P(PbgGrid), c_double, c_void_p, c_double, c_void_p, c_void_p, c_void_p],
                  ctypes.c_int),
    "pbg_maxabs": ([_P(PbgGrid), c_void_p, _P(c_double), c_void_p], ctypes.c_int),
    "pbg_set_profiling": ([c_int32], ctypes.c_int),
    "pbg_get_profile": ([_P(c_double), _P(c_int64)], ctypes.c_int),
    "pbg_vacuum_dst": ([_P(PbgGrid), c_double, c_void_p, c_void_p, c_void_p, c_void_p],
                       ctypes.c_int),
    "pbg_plan_create": ([_P(PbgMarchDesc), _P(c_void_p), c_void_p], ctypes.c_int),
    "pbg_plan_run": ([c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_int32, _P(c_int32),
                      _P(c_int32), _P(c_int32), _P(ctypes.c_float), c_void_p], ctypes.c_int),
    "pbg_plan_destroy": ([c_void_p, c_void_p], ctypes.c_int),
    "pbg_plan_create_batch": ([_P(PbgMarchDesc), c_int32, c_int64, _P(c_void_p), c_void_p],
                              ctypes.c_int),
    "pbg_plan_run_batch": ([c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_int32,
                            _P(c_int32), _P(c_int32), _P(c_int32), _P(ctypes.c_float),
                            c_void_p], ctypes.c_int),
    "pbg_slab_exchange_elems": ([_P(PbgGrid)], c_int64),
    "pbg_slab_nchunks": ([c_void_p], c_int32),
    "pbg_slab_phase": ([c_void_p, c_int32, c_int32, _P(c_int64), _P(c_int64)], ctypes.c_int),
    "pbg_slab_step_a_chunk": ([c_void_p, c_int32, c_void_p], ctypes.c_int),
    "pbg_slab_create": ([_P(PbgMarchDesc), c_int32, c_int32, c_void_p, c_void_p,
                         _P(c_void_p), c_void_p], ctypes.c_int),
    "pbg_slab_setup": ([c_void_p, c_void_p], ctypes.c_int),
    "pbg_slab_halo_pack": ([c_void_p, c_void_p], ctypes.c_int),
    "pbg_slab_halo_unpack": ([c_void_p, c_void_p], ctypes.c_int),
    "pbg_slab_step_a": ([c_void_p, c_void_p], ctypes.c_int),
    "pbg_slab_step_b": ([c_void_p, c_void_p], ctypes.c_int),
    "pbg_slab_flag_pack": ([c_void_p, c_void_p], ctypes.c_int),
    "pbg_slab_finish": ([c_void_p, _P(c_int32), _P(c_int32), _P(c_int32), c_void_p],
                        ctypes.c_int),
    "pbg_slab_destroy": ([c_void_p, c_void_p], ctypes.c_int),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load_library():
    """Load libpbg.so and declare every exported signature (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"native library missing: {LIB_PATH} (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


_torch = None


def torch_cuda():
    """The torch module, after checking a CUDA device exists (no CPU fallback)."""
    global _torch
    if _torch is None:
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_1410_2788_b200 needs a CUDA (sm_100a) device; none found")
        load_library()
        _torch = torch
    return _torch


def lib():
    torch_cuda()
    return _lib


def stream_ptr():
    return c_void_p(torch_cuda().cuda.current_stream().cuda_stream)


_ERR_RE = re.compile(r"atom (\d+) is not strictly inside")


def check(rc: int):
    if rc == 0:
        return
    msg = _lib.pbg_last_error().decode(errors="replace")
    if rc == -1:
        raise ValueError(msg)
    if rc == -3:
        raise NotImplementedError(msg)
    raise RuntimeError(f"pbg CUDA error: {msg}")


def ptr(t) -> c_void_p:
    return c_void_p(0 if t is None else t.data_ptr())


def layout(shape):
    pitch = c_int64()
    nelem = c_int64()
    check(load_library().pbg_layout(int(shape[0]), int(shape[1]), int(shape[2]),
                                    ctypes.byref(pitch), ctypes.byref(nelem)))
    return int(pitch.value), int(nelem.value)


def grid_struct(grid) -> PbgGrid:
    g = PbgGrid()
    pitch, _ = layout(grid.shape)
    for a in range(3):
        g.n[a] = int(grid.shape[a])
        g.lo[a] = float(grid.lo[a])
    g.pitch = pitch
    g.h = float(grid.h)
    return g


def new_field(grid, fill=None):
    torch = torch_cuda()
    _, nelem = layout(grid.shape)
    if fill is None:
        return torch.empty(nelem, dtype=torch.float64, device="cuda")
    return torch.full((nelem,), float(fill), dtype=torch.float64, device="cuda")


def new_codes(grid):
    torch = torch_cuda()
    _, nelem = layout(grid.shape)
    return torch.zeros(nelem, dtype=torch.uint8, device="cuda")


def upload_dense(grid, arr: np.ndarray):
    """Host (n0, n1, n2) fp64 -> new pitched device field."""
    torch = torch_cuda()
    arr = np.ascontiguousarray(arr, dtype=np.float64)
    dense = torch.from_numpy(arr).to("cuda")
    out = new_field(grid, 0.0)
    check(lib().pbg_pitch_from_dense(ctypes.byref(grid_struct(grid)), ptr(dense), ptr(out),
                                     stream_ptr()))
    return out


def upload_flat(arr: np.ndarray):
    torch = torch_cuda()
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).to("cuda")


def download_dense(grid, field) -> np.ndarray:
    torch = torch_cuda()
    dense = torch.empty(tuple(int(s) for s in grid.shape), dtype=torch.float64, device="cuda")
    check(lib().pbg_dense_from_pitched(ctypes.byref(grid_struct(grid)), ptr(field), ptr(dense),
                                       stream_ptr()))
    return dense.cpu().numpy()


def atoms_array(system):
    """MolecularSystem -> device (N, 5) fp64 array (x, y, z, q, r) in atom order."""
    arr = np.array([[a.center[0], a.center[1], a.center[2], a.charge, a.radius]
                    for a in system.atoms], dtype=np.float64).reshape(-1, 5)
    return upload_flat(arr), arr
