"""Experiment CLI on the device path against CSV reports of the reference CLI
(tests/golden/cli/*.csv, written by tests/golden/make_golden.py cli): same columns, same
non-numeric fields, numbers within the parity bar (wall-clock column excluded)."""

import math
import os

import pytest

from paper_1410_2788_b200.cli import main
from tests.golden.make_golden_cases import CLI_CASES

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")


def _rows(path):
    lines = open(path).read().splitlines()
    return lines[0].split(","), [ln.split(",") for ln in lines[1:]]


@pytest.mark.parametrize("name", sorted(CLI_CASES))
def test_cli_report_matches_reference(tmp_path, name):
    argv = [os.path.join(HERE, "mini.sys") if a == "SYS" else a for a in CLI_CASES[name]]
    out = tmp_path / f"{name}.csv"
    assert main(argv + ["--out", str(out)]) == 0
    hdr, got = _rows(out)
    want_hdr, want = _rows(os.path.join(HERE, name + ".csv"))
    assert hdr == want_hdr and len(got) == len(want)
    for g, w in zip(got, want):
        for col, a, b in zip(hdr, g, w):
            if col == "wall_time_s":
                continue
            try:
                fa, fb = float(a), float(b)
            except ValueError:
                assert a == b, (col, a, b)
                continue
            if math.isnan(fb):
                assert math.isnan(fa), (col, a, b)
            else:
                assert abs(fa - fb) <= 1e-8 * max(1.0, abs(fb)), (col, a, b)
