"""CLI argument handling and exit codes (no device work reached): cli.py:19-21, 440-463."""

import pytest

from paper_1410_2788_b200.cli import (EXIT_CONFIG, EXIT_IO, ExperimentSpec, _fit_order,
                                      _rung_order, _stable_range, main, report_lines)


def test_exit_codes(tmp_path):
    assert main(["protein"]) == EXIT_CONFIG                       # no molecular system
    assert main(["sphere-spatial"]) == EXIT_CONFIG                # empty h ladder
    assert main(["stability", "--h", "0.5"]) == EXIT_CONFIG       # empty dt ladder
    assert main(["vacuum-check", "--system", str(tmp_path / "missing.sys")]) == EXIT_IO
    assert main(["sphere-spatial", "--config", str(tmp_path / "none.cfg")]) == EXIT_IO
    assert main(["sphere-spatial", "--h", "0.5", "--domain", "1,2,3"]) == EXIT_CONFIG
    assert main(["sphere-spatial", "--h", "0.5", "--scheme", "LOD"]) == EXIT_CONFIG
    with pytest.raises(SystemExit):
        main(["no-such-command"])


def test_ladders_sorted_coarse_to_fine():
    s = ExperimentSpec(kind="SphereTemporal", schemes=("LODIE1",), dt_values=(0.1, 0.4, 0.2))
    assert s.dt_values == (0.4, 0.2, 0.1)


def test_orders_and_ranges():
    assert abs(_rung_order(4.0, 1.0, 0.2, 0.1) - 2.0) < 1e-15
    assert _rung_order(0.0, 1.0, 0.2, 0.1) != _rung_order(0.0, 1.0, 0.2, 0.1)  # NaN
    assert abs(_fit_order([0.4, 0.2, 0.1], [16.0, 4.0, 1.0]) - 2.0) < 1e-12
    assert _stable_range([0.01, 0.1, 1.0], {0.01: True, 0.1: True, 1.0: False}) == "[0.01,0.1]"
    assert _stable_range([0.01, 0.1], {0.01: False, 0.1: False}) == "[]"
    lines = report_lines([{"a": True, "b": 3, "c": 0.5, "d": "x"}], ["a", "b", "c", "d"])
    assert lines == ["a,b,c,d", "true,3,5.000000000000e-01,x"]
