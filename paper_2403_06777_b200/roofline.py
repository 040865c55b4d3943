"""Algorithmic roofline of the bit-sliced evaluators.

The BASELINE's naive int-op count (8 ops per row-eval) is not a bound for a
bit-sliced kernel: one 32-bit LOP3 updates a row for 32 assignments at once.
The roofline reported instead is the MINIMUM instruction count of the
bit-sliced algorithm itself, derived from the generated per-class LOP3 chains
(gen_slice_ops.case_body) and the table's own row / term mix
(pzx_table_slice_stats), against the two sm_100 resources it can saturate:

* issue slots: 148 SMs x 4 schedulers x 1 warp-instruction / clk;
* the ALU pipe (LOP3, SEL, LOP3->P, PRMT, IADD3, SHF): 16 lanes / clk / SMSP,
  i.e. one warp-instruction per 2 clk per scheduler (B300_MICROARCH "Pipe
  rates": alu rt_SMSP = 2; ncu's sm__inst_executed_pipe_alu peak agrees: the
  round-2 C2 capture shows the ALU pipe at 63 % of its peak at 62 % issue
  utilisation). The bit-sliced row updates are almost all ALU work, so this
  pipe, not the issue slots, binds the minimum;
* the XU pipe (POPC): 16 lanes / clk / SM (profiles/r01/microbench.json).

Per row and warp (one warp = 32 threads x 32 assignments = 1024 assignments):

    1 LDS (the row record)  +  per parity vector (1 or 2) the enumerated kernels'
    X = W ^ -parity(mask & base):  AND + POPC + LOP3->P + SEL  (4, one POPC)
    +  the class's LOP3 chain (len(case_body(op)): phase counter ripple add,
       zero / lambda / pi / pi' indicators)

Per term and warp (the epilogue, 32 assignments per thread), per assignment:

    kind-free term: 1 LDS (C w^j) + 2 DADD            = 3
    lambda-only   : 2 LDS + 2 DFMA (real (sqrt2-1)^s)  = 4
    with pi / pi' : 2 LDS + 4 DFMA (complex factor)    = 6

For word-list batches the sorted kernel forms each parity vector from G
Four-Russians table words: G LDS + G XOR + AND + POPC + 1 = 2G + 3 per parity
(G = 4 dense, 6 sparse batches).

The page kernel (enumerated batches, page layout) resolves the high-bit
parities once per row and WARP in a pre-pass (2 POPC per row, spread over the
lanes: (1 LDS + 2 x (index, LDS, AND, POPC, XOR) + 1 STS) / 32 per row and
warp), then per row and warp:
                                                                       issue   ALU
    C row: 2 LDS (record, lane word) + LOP3->P + SEL + OR                  5      3
    G rows by update class (page_term):
      S2/S6 (single parity, J += 2q / 6q): 2 LDS + LOP3->P + SEL + 2 LOP3   6      4
      E0 (J2 ^= X & Y): 2 LDS + 2 x (LOP3->P + SEL) + 1 LOP3                7      5
      E2 (J += 2Y + 4XY): 2 LDS + 2 x (LOP3->P + SEL) + 3 LOP3              9      7
      G1/G3 (odd k): 2 LDS + 2 x (LOP3->P + SEL) + 5 LOP3                  11      9
    L row (k in {0, 4}): 2 LDS + LOP3->P + SEL + 7 LOP3 (lambda ripple)    11      9
    D row: 3 LDS + 2 x (LOP3->P + SEL) + the class's LOP3 chain       7 + body  4 + body
Loop control, row prefetch, TMA waits, counter decode, TMEM traffic and the
chunk reduction are implementation overhead and are NOT in the minimum, so
frac <= 1 by construction.
"""
from __future__ import annotations

from functools import lru_cache

import numpy as np

N_SM = 148
ISSUE_PER_SM = 4        # warp-instructions / clk / SM (one per scheduler)
ALU_PER_SM = 2          # ALU-pipe warp-instructions / clk / SM (16 lanes / clk / SMSP)
POPC_LANES_PER_SM = 16  # XU lanes / clk / SM (measured 15.9, profiles/r01/microbench.json)
EPI_PER_ASSIGN = (3, 4, 6)  # kind-free, lambda-only, pi: minimum instructions per (term, assignment)


@lru_cache(maxsize=None)
def _op_table():
    from . import gen_slice_ops as G
    body = np.array([len(G.case_body(op, False, True)) for op in range(129)], np.int64)
    par = np.array([0 if op >= 128 else (1 if op & 1 else 2) for op in range(129)], np.int64)
    return body, par


def min_counts(op_rows, term_kinds, n_assign: int, kernel: str = "slice", sorted_groups: int = 4) -> dict:
    """Minimum warp-instructions and warp-POPCs of one evaluation launch."""
    body, par = _op_table()
    op_rows = np.asarray(op_rows, np.float64)
    kinds = np.asarray(term_kinds, np.float64)
    per_parity = 4 if kernel != "sorted" else 2 * sorted_groups + 3
    alu_parity = 3 if kernel != "sorted" else sorted_groups + 2  # AND, LOP3->P, SEL (+ the table XORs)
    row_inst = float(np.sum(op_rows * (1 + per_parity * par + body)))
    row_alu = float(np.sum(op_rows * (alu_parity * par + body)))
    popc = float(np.sum(op_rows * par))
    term_inst = float(np.sum(kinds * 32 * np.array(EPI_PER_ASSIGN)))
    warps = n_assign / 1024.0
    return {"warp_instructions": warps * (row_inst + term_inst), "warp_alu": warps * row_alu,
            "warp_popc": warps * popc,
            "row_share": row_inst / max(row_inst + term_inst, 1.0),
            "per_row_per_warp": row_inst / max(float(np.sum(op_rows)), 1.0),
            "per_term_per_warp": term_inst / max(float(np.sum(kinds)), 1.0)}


def min_counts_page(family_rows, d_op_rows, term_kinds, n_assign: int) -> dict:
    """Minimum warp-instructions / warp-POPCs of one page-kernel launch."""
    body, _ = _op_table()
    fr = [float(x) for x in family_rows]
    fr += [0.0] * (11 - len(fr))
    c, g, d, _dropped, l_ = fr[:5]  # family_rows: C, G, D, dropped, L, G by class S2, S6, E0, E2, G1, G3
    s_, e0, e2 = fr[5] + fr[6], fr[7], fr[8]
    gg = g - s_ - e0 - e2          # G1 + G3 (a layout without the class split: every G row is odd-k)
    d_ops = np.asarray(d_op_rows, np.float64)
    rows = c + g + d + l_
    pre = rows * (1 + 2 * 5 + 1) / 32.0
    row_inst = (pre + 5 * c + 6 * s_ + 7 * e0 + 9 * e2 + 11 * gg + 11 * l_ +
                float(np.sum(d_ops * (3 + 4 + body))))
    row_alu = (rows * 6 / 32.0 + 3 * c + 4 * s_ + 5 * e0 + 7 * e2 + 9 * gg + 9 * l_ +
               float(np.sum(d_ops * (4 + body))))
    kinds = np.asarray(term_kinds, np.float64)
    term_inst = float(np.sum(kinds * 32 * np.array(EPI_PER_ASSIGN)))
    warps = n_assign / 1024.0
    return {"warp_instructions": warps * (row_inst + term_inst), "warp_alu": warps * row_alu,
            "warp_popc": warps * rows * 2 / 32.0,
            "row_share": row_inst / max(row_inst + term_inst, 1.0),
            "per_row_per_warp": row_inst / max(rows, 1.0),
            "per_term_per_warp": term_inst / max(float(np.sum(kinds)), 1.0)}


# Shared-memory wavefronts (1 / clk / SM) of the page kernel's own data movement:
# a warp-wide 128-bit load with per-lane addresses costs >= 4 wavefronts (one per
# quarter-warp), a uniform one 2, 64- / 32-bit loads 1-2 (tools/micro/lds128_bcast.cu).
PAGE_WF_ROW = {"c": 3.0, "s": 2.0, "e": 3.0, "g": 3.0, "l": 3.0, "d": 5.0}  # record + lane word per row-warp
PAGE_WF_ASSIGN = (4.0, 5.5, 5.5)  # per (term, assignment-warp): crot | crot + uz | T + uz


def smem_floor_page(family_rows, term_kinds, n_assign: int) -> float:
    """Minimum shared-memory wavefronts of one page-kernel launch: the row
    loops' record / lane-word loads and the epilogue's per-lane table lookups
    at their conflict-free cost (no pre-pass, no bank conflicts)."""
    fr = [float(x) for x in family_rows] + [0.0] * 11
    c, g, d, _dropped, l_ = fr[:5]
    s_ = fr[5] + fr[6]
    W = PAGE_WF_ROW
    rows = W["c"] * c + W["s"] * s_ + W["g"] * (g - s_) + W["l"] * l_ + W["d"] * d
    kinds = np.asarray(term_kinds, np.float64)
    terms = float(np.sum(kinds * 32 * np.array(PAGE_WF_ASSIGN)))
    return n_assign / 1024.0 * (rows + terms)


def roofline(op_rows, term_kinds, n_assign: int, seconds: float, f_mhz: float, kernel: str = "slice",
             sorted_groups: int = 4, page_stats=None) -> dict:
    """The bench's `roofline` object: the binding resource of the algorithm's
    minimum work (issue slots or the POPC pipe) against the measured launch time."""
    if kernel == "page" and page_stats is not None:
        c = min_counts_page(page_stats[0], page_stats[1], term_kinds, n_assign)
    else:
        c = min_counts(op_rows, term_kinds, n_assign, kernel, sorted_groups)
    hz = f_mhz * 1e6
    t_issue = c["warp_instructions"] / (N_SM * ISSUE_PER_SM * hz)
    t_alu = c["warp_alu"] / (N_SM * ALU_PER_SM * hz)
    t_xu = c["warp_popc"] * 32 / (N_SM * POPC_LANES_PER_SM * hz)
    t_max = max(t_issue, t_alu, t_xu)
    if t_alu == t_max:
        out = {"bound": "alu pipe", "achieved": c["warp_alu"] / seconds / 1e12,
               "peak": N_SM * ALU_PER_SM * hz / 1e12, "unit": "T ALU warp-instructions/s (algorithmic minimum)"}
    elif t_issue == t_max:
        out = {"bound": "issue", "achieved": c["warp_instructions"] / seconds / 1e12,
               "peak": N_SM * ISSUE_PER_SM * hz / 1e12, "unit": "T warp-instructions/s (algorithmic minimum)"}
    else:
        out = {"bound": "xu (POPC)", "achieved": c["warp_popc"] * 32 / seconds / 1e12,
               "peak": N_SM * POPC_LANES_PER_SM * hz / 1e12, "unit": "T POPC lane-ops/s (algorithmic minimum)"}
    out["frac"] = out["achieved"] / out["peak"]
    out.update({"min_warp_instructions": c["warp_instructions"], "min_warp_alu": c["warp_alu"],
                "min_warp_popc": c["warp_popc"],
                "min_time_issue_s": t_issue, "min_time_alu_s": t_alu, "min_time_popc_s": t_xu,
                "min_per_row_per_warp": c["per_row_per_warp"], "min_per_term_per_warp": c["per_term_per_warp"],
                "kernel_model": kernel if kernel != "sorted" else f"sorted (G={sorted_groups})"})
    if kernel == "page" and page_stats is not None:
        # informational: the page kernel against the floor of its own shared-memory
        # traffic (the pipe ncu shows closest to saturation); frac stays the
        # conservative instruction minimum above
        wf = smem_floor_page(page_stats[0], term_kinds, n_assign)
        t_smem = wf / (N_SM * hz)
        out["smem_floor"] = {"wavefronts": wf, "time_s": t_smem, "frac": t_smem / seconds,
                             "note": "conflict-free shared-memory wavefronts of the row loads and epilogue "
                                     "lookups at 1 / clk / SM; not the reported frac"}
    return out
