"""CPU checks of bench.py's roofline object (no GPU, no compute calls).

The reported roofline is the issue-slot one whenever the config has an ncu
capture in profiles/ncu_traffic.json; the BASELINE's naive int-op roofline
(exceeded by bit-slicing) is carried under ``naive_alu``.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _ncu():
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
        return json.load(f)


def test_issue_roofline_uses_ncu_instruction_count():
    info = _ncu()["c2"]
    naive = {"bound": "alu", "frac": 6.4}
    r = bench._roofline(info, info["duration_s"] * 1e3, 1965.0, "measured", info["dram_bytes_per_launch"], naive)
    assert r["bound"] == "issue"
    assert abs(r["peak"] - 148 * 4 * 1965e6 / 1e12) < 1e-9
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    # timed at ncu's own launch duration, the fraction is ncu's issue-active share
    assert abs(r["frac"] * 100 - info["issue_active_pct"]) < 5.0
    assert 0 < r["frac"] <= 1.0
    assert r["naive_alu"] is naive


def test_roofline_without_capture_falls_back_to_naive():
    naive = {"bound": "alu", "frac": 0.3}
    assert bench._roofline(None, 10.0, 1965.0, "measured", None, naive) is naive
