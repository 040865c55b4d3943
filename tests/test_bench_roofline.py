"""CPU checks of the algorithmic roofline (paper_2403_06777_b200/roofline.py) that
bench.py reports: the minimum instruction / POPC counts of the bit-sliced
algorithm for a table's own row and term mix (no GPU, no compute calls).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2403_06777_b200 as P  # noqa: E402
from paper_2403_06777_b200 import gen_slice_ops as G  # noqa: E402
from paper_2403_06777_b200 import roofline as RL  # noqa: E402
from paper_2403_06777_b200 import synth  # noqa: E402


def test_row_minimum_per_class_is_pinned():
    # op = class * 2 + single; class (0,0) two-parity: V(4p,4q) = 2 * w^(4pq) -> ONE lop3
    assert len(G.case_body(0, False, True)) == 1
    # class (2,2) two-parity: J += 6pq (2-bit ripple) and Z |= p ^ q
    assert len(G.case_body(2 * 18, False, True)) == 5
    # class (1,4) two-parity: V = 2 w^(x[q]) over x = 1 + 4p -> a 3-bit ripple add
    assert len(G.case_body(2 * 12, False, True)) == 7
    ops = np.zeros(129)
    ops[0] = 10      # 10 two-parity rows: 1 LDS + 2 x 4 parity + 1 body = 10 each
    ops[37] = 5      # 5 single-parity rows of class (2,2): 1 + 4 + 1 = 6 each
    kinds = np.array([1, 2, 3])  # epilogue minimum 32 x (3, 4, 6) per term and warp
    c = RL.min_counts(ops, kinds, 1024)
    assert c["warp_instructions"] == 10 * 10 + 5 * 6 + 32 * (3 + 2 * 4 + 3 * 6)
    assert c["warp_popc"] == 10 * 2 + 5 * 1
    # the sorted kernel forms each parity from G table words: 2G + 3 per parity
    c4 = RL.min_counts(ops, kinds, 1024, "sorted", 4)
    assert c4["warp_instructions"] == 10 * (1 + 2 * 11 + 1) + 5 * (1 + 11 + 1) + 32 * 29


def test_c1_table_minimum_regression():
    cfg = synth.CONFIGS["c1s"]
    h = P.HostTable(synth.generate_config(cfg))
    ops, kinds = h.slice_stats()
    assert int(ops.sum()) == h.n_rows and int(kinds.sum()) == h.n_terms
    c = RL.min_counts(ops, kinds, cfg.n_assign)
    assert c["warp_instructions"] == 83135.0
    assert abs(c["per_row_per_warp"] - 11.259) < 1e-3


def test_frac_is_bounded_and_shard_invariant():
    cfg = synth.CONFIGS["c1s"]
    h = P.HostTable(synth.generate_config(cfg))
    ops, kinds = h.slice_stats()
    c = RL.min_counts(ops, kinds, 1 << 20)
    t_min = max(c["warp_instructions"] / (148 * 4 * 1965e6), c["warp_popc"] * 32 / (148 * 16 * 1965e6))
    # a launch can never beat the minimum: at t = t_min the fraction is exactly 1
    r = RL.roofline(ops, kinds, 1 << 20, t_min, 1965.0)
    assert abs(r["frac"] - 1.0) < 1e-9
    slow = RL.roofline(ops, kinds, 1 << 20, 3 * t_min, 1965.0)
    assert abs(slow["frac"] - 1 / 3) < 1e-9
    # an 8-way assignment shard: each rank does 1/8 of the work in 1/8 of the time
    shard = RL.roofline(ops, kinds, (1 << 20) // 8, 3 * t_min / 8, 1965.0)
    assert abs(shard["frac"] - slow["frac"]) < 1e-9
