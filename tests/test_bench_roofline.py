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
    # ALU pipe: per parity AND + LOP3->P + SEL, plus the body
    assert c["warp_alu"] == 10 * (2 * 3 + 1) + 5 * (3 + 1)
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
    t_min = max(c["warp_instructions"] / (148 * 4 * 1965e6), c["warp_alu"] / (148 * 2 * 1965e6),
                c["warp_popc"] * 32 / (148 * 16 * 1965e6))
    # a launch can never beat the minimum: at t = t_min the fraction is exactly 1
    r = RL.roofline(ops, kinds, 1 << 20, t_min, 1965.0)
    assert abs(r["frac"] - 1.0) < 1e-9
    slow = RL.roofline(ops, kinds, 1 << 20, 3 * t_min, 1965.0)
    assert abs(slow["frac"] - 1 / 3) < 1e-9
    # an 8-way assignment shard: each rank does 1/8 of the work in 1/8 of the time
    shard = RL.roofline(ops, kinds, (1 << 20) // 8, 3 * t_min / 8, 1965.0)
    assert abs(shard["frac"] - slow["frac"]) < 1e-9


def test_page_minimum_by_family_and_class():
    # C, G (all in the class split), D, dropped, L | S2, S6, E0, E2, G1, G3
    fam = [10, 40, 2, 5, 4, 8, 2, 10, 10, 6, 4]
    d_ops = np.zeros(129)
    d_ops[0] = 2  # class (0,0) two-parity: body 1
    c = RL.min_counts_page(fam, d_ops, np.array([1, 0, 0]), 1024)
    rows = 10 + 40 + 2 + 4
    pre = rows * 12 / 32
    assert abs(c["warp_instructions"] - (pre + 5 * 10 + 6 * 10 + 7 * 10 + 9 * 10 + 11 * 10 + 11 * 4
                                         + 2 * 8 + 32 * 3)) < 1e-9
    assert abs(c["warp_alu"] - (rows * 6 / 32 + 3 * 10 + 4 * 10 + 5 * 10 + 7 * 10 + 9 * 10 + 9 * 4
                                + 2 * 5)) < 1e-9
    # a layout without the class split counts every G row as GG
    old = RL.min_counts_page(fam[:5], d_ops, np.array([1, 0, 0]), 1024)
    assert old["warp_alu"] > c["warp_alu"]


def test_headline_table_bound_and_classes_cover_g():
    h = P.HostTable(synth.generate_config(synth.CONFIGS["c2"]))
    fam, d_ops = h.page_stats()
    assert int(fam[5:].sum()) == int(fam[1])
    ops, kinds = h.slice_stats()
    r = RL.roofline(ops, kinds, 1 << 20, 0.2, 1965.0, "page", page_stats=(fam, d_ops))
    assert r["bound"] in ("alu pipe", "issue") and 0 < r["frac"] < 1
    # the two minima are within a few % of each other for this table (the binding one is reported)
    assert 0.8 < r["min_time_alu_s"] / r["min_time_issue_s"] < 1.25


def test_page_smem_floor_is_informational_and_pinned():
    fam = [10, 40, 2, 5, 4, 8, 2, 10, 10, 6, 4]   # C, G, D, dropped, L | S2, S6, E0, E2, G1, G3
    kinds = np.array([1, 2, 3])
    wf = RL.smem_floor_page(fam, kinds, 1024)
    want = 3 * 10 + 2 * 10 + 3 * 30 + 3 * 4 + 5 * 2 + 32 * (4 * 1 + 5.5 * 2 + 5.5 * 3)
    assert abs(wf - want) < 1e-9
    d_ops = np.zeros(129)
    r = RL.roofline(np.zeros(129), kinds, 1024, 1e-3, 1965.0, "page", page_stats=(fam, d_ops))
    assert "smem_floor" in r and r["smem_floor"]["frac"] > 0
    assert r["frac"] == r["achieved"] / r["peak"]            # the reported frac is unchanged
