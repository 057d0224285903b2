"""CPU checks of the drop-in boundary: libpbg.so loads without a GPU and exports exactly
the C ABI declared in include/pbg.h; pure-arithmetic entry points and error reporting."""

import ctypes
import os
import re

import pytest

from paper_1410_2788_b200 import _native as nat

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "pbg.h")).read()
    return sorted(set(re.findall(r"PBG_API\s+[\w\s\*]+?\b(pbg_\w+)\s*\(", text)))


def test_library_loads_and_exports_header_symbols():
    lib = nat.load_library()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(nat.EXPORTED)


def test_version_and_layout():
    lib = nat.load_library()
    assert lib.pbg_version() == 1
    for n, pitch in ((65, 96), (97, 128), (129, 160), (257, 288), (513, 544)):
        p, ne = nat.layout((n, n, n))
        assert p == pitch and ne == n * n * pitch + 64
        assert (1 + nat.PBG_OFFSET) % 32 == 0  # interior k=1 is 256-byte aligned


def test_invalid_arguments_report_errors():
    lib = nat.load_library()
    p = ctypes.c_int64()
    e = ctypes.c_int64()
    rc = lib.pbg_layout(2, 5, 5, ctypes.byref(p), ctypes.byref(e))
    assert rc == -1
    assert b"3 nodes" in lib.pbg_last_error()
    with pytest.raises(ValueError):
        nat.check(rc)


def test_struct_layouts_match_c():
    assert ctypes.sizeof(nat.PbgGrid) == 56
    assert ctypes.sizeof(nat.PbgPalette) == 64
    assert nat.PbgMarchDesc.codes.offset == 56 + 64 + 8 + 24 + 8
    assert ctypes.sizeof(nat.PbgMarchDesc) == 56 + 64 + 8 + 24 + 8 + 5 * 8


def test_variant_ids_follow_reference_enum_order():
    from paper_1410_2788_b200.schemes import SCHEME_NAMES

    assert [nat.VARIANT_IDS[n] for n in SCHEME_NAMES] == list(range(13))
