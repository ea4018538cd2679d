"""The paper's printed performance numbers (tests/golden/paper_numbers.json, each
with its PAPER.md line) against paper_1410_1387_b200.perfmodel."""
import json
import os

import pytest

from paper_1410_1387_b200 import perfmodel as PM

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_numbers.json")))


def test_flops_per_point_92():
    g = GOLD["flops_per_point"]
    assert PM.flops_per_point(g["r_xy"], g["r_z"]) == g["value"]


def test_ci_optimistic_3_3():
    g = GOLD["ci_optimistic"]
    assert PM.ci_optimistic(12, 8) == pytest.approx(g["value"], abs=g["tol"])
    assert PM.ci_optimistic(12, 8) == pytest.approx(92 / 28)


def test_ci_pessimistic_0_4():
    g = GOLD["ci_pessimistic"]
    assert PM.ci_pessimistic(12, 8) == pytest.approx(g["value"], abs=g["tol"])
    assert PM.ci_pessimistic(12, 8) == pytest.approx(23 / 64)


def test_cpu_peak_fraction_47_percent_needs_gib():
    g = GOLD["cpu_peak_fraction"]
    assert PM.peak_fraction(12, 8, g["peak_gflops"], g["bw_gbs"], gib=True) == pytest.approx(g["value"], abs=g["tol"])
    assert PM.peak_fraction(12, 8, g["peak_gflops"], g["bw_gbs"]) == pytest.approx(0.505, abs=0.001)


def test_table1_peak_column_is_mpts_times_92_flops():
    g = GOLD["table1_occa_compact_16"]
    frac = g["mpts"] * 1e6 * PM.flops_per_point(12, 8) / 666e9
    assert round(100 * frac) == g["peak_pct"]


def test_byte_model():
    assert PM.bytes_per_point(32) == 36 and PM.bytes_per_point(64) == 72
    assert PM.step_flops_per_point(4, 4) > PM.flops_per_point(4, 4)
