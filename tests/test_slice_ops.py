"""CPU checks of the bit-sliced kernel's generated per-row PTX (no GPU needed).

* the op table the generator derives (Python, exact Z[w]) equals the C++
  constexpr table the host compiler uses (pzx_slice_op_table), and the
  generated .inc in the tree is up to date;
* every one of the 129 generated LOP3 chains is executed by a tiny PTX-subset
  interpreter on all (p, q) parities and all 3-bit starting counters: the new
  (J2 J1 J0) must equal old + w'(p, q) mod 8, Z must OR in the zero
  indicator, and the lambda / pi / pi' indicator outputs must match;
* jbase + w' reproduces the exact exponent j of every non-zero variant.
"""
import re

import numpy as np
import pytest

import paper_2403_06777_b200 as P
from paper_2403_06777_b200 import gen_slice_ops as G
from zw_exact import ZQ, pair_value, SQRT2, LAMBDA, MU, PI, PIP, ONE


def test_generated_table_matches_cxx_constexpr():
    cxx = P.slice_op_table()
    for op in range(129):
        jb, w, z, lam, pi, pip, lm = G.slice_op(op)
        assert list(cxx[op]) == [jb, *w, z, lam, pi, pip, lm], op


def test_generated_include_is_current():
    assert open(G.OUT).read() == G.generate()


def _bodies(p64=False, name=None):
    text = G.generate()
    name = name or ("PZX_SLICE_DISPATCH_ASM_P64" if p64 else "PZX_SLICE_DISPATCH_ASM_P32")
    block = text[text.index(name + " "):]
    block = block[:block.index("\n\n")]
    lines = re.findall(r'"(.*?)\\n"', block)
    table = next(ln for ln in lines if ".branchtargets" in ln)
    targets = [int(x.strip().split("_")[0][1:]) for x in table.split(".branchtargets")[1].rstrip(";").split(",")]
    bodies, cur = {}, None
    for ln in lines:
        m = re.match(r"L(\d+)_%=:", ln)
        if m:
            cur = int(m.group(1))
            bodies[cur] = []
        elif ln.startswith("bra.uni") or ln.startswith("D%="):
            cur = None
        elif cur is not None:
            bodies[cur].append(ln)
    return {op: bodies[targets[op]] for op in range(len(targets))}


def _run(body, regs):
    """Interpret the generated PTX subset on 1-bit lanes."""
    r = dict(regs)

    def val(tok):
        return int(tok, 0) & 1 if tok[0].isdigit() else r[tok]
    for ins in body:
        m = re.match(r"(lop3\.b32|and\.b32|xor\.b32|popc\.b32|neg\.s32) (.*);", ins)
        assert m, ins
        ops = [o.strip() for o in m.group(2).split(",")]
        kind = m.group(1)
        if kind == "lop3.b32":
            d, a, b, c, imm = ops
            i = (val(a) << 2) | (val(b) << 1) | val(c)
            r[d] = (int(imm, 16) >> i) & 1
        elif kind == "and.b32":
            r[ops[0]] = val(ops[1]) & val(ops[2])
        elif kind == "xor.b32":
            r[ops[0]] = val(ops[1]) ^ val(ops[2])
        elif kind == "popc.b32":
            r[ops[0]] = val(ops[1])          # 1-bit lane: popcount parity == the bit
        else:
            r[ops[0]] = val(ops[1])          # -x on one bit is x (all-ones mask)
    return r


@pytest.mark.parametrize("p64", [False, True])
def test_every_generated_chain_is_a_correct_mod8_add(p64):
    bodies = _bodies(p64)
    assert len(bodies) == 129
    for op in range(129):
        jb, w, z, lam, pi, pip, _ = G.slice_op(op)
        single = op < 128 and (op & 1)
        for v in range(4):
            p, q = v & 1, v >> 1
            if single and q:
                continue
            for j0 in range(8):
                for zin in (0, 1):
                    # Y = Walsh(phi) ^ -parity(phi & base): phi = 1, base = q, Walsh = 0 -> q
                    regs = {"%0": j0 & 1, "%1": (j0 >> 1) & 1, "%2": (j0 >> 2) & 1, "%3": zin,
                            "%4": 0, "%5": 0, "%6": 0, "%7": p, "%9": 1, "%10": 0, "%11": q,
                            "%12": 0, "%13": 0}
                    out = _run(bodies[op], regs)
                    jn = out["%0"] | (out["%1"] << 1) | (out["%2"] << 2)
                    if not (z >> v) & 1:
                        assert jn == (j0 + w[v]) % 8, (op, v, j0)
                    assert out["%3"] == (zin | ((z >> v) & 1)), (op, v)
                    assert out["%4"] == (lam >> v) & 1
                    assert out["%5"] == (pi >> v) & 1
                    assert out["%6"] == (pip >> v) & 1


def test_jbase_plus_w_is_the_exact_exponent():
    gens = {G.KNONE: ONE, G.KLAMBDA: LAMBDA, G.KMU: MU, G.KPI: PI, G.KPIP: PIP}
    for op in range(128):
        jb, w, z, lam, pi, pip, lm = G.slice_op(op)
        cls, single = op >> 1, op & 1
        ka, kb = cls >> 3, cls & 7
        for v in range(4):
            p, q = v & 1, v >> 1
            if single and q:
                continue
            want = pair_value(ka + 4 * p, kb + 4 * q)
            if (z >> v) & 1:
                assert want == ZQ((0, 0, 0, 0))
                continue
            kind, j, e = G.factor_pair(ka + 4 * p, kb + 4 * q)
            assert (jb + w[v]) % 8 == j
            assert ZQ.w(j) * SQRT2 ** e * gens[kind] == want
            assert bool((lam >> v) & 1) == (kind == G.KLAMBDA)
            assert bool((pi >> v) & 1) == (kind == G.KPI)
            assert bool((pip >> v) & 1) == (kind == G.KPIP)


def test_two_slice_chains_are_two_independent_mod8_adds():
    """XY2 (two-slice kernel): slice a and slice b updated independently, each
    exactly like the one-slice chain, from their own X / Y."""
    bodies = _bodies(name="PZX_SLICE_DISPATCH_ASM_XY2")
    assert len(bodies) == 129
    for op in range(129):
        jb, w, z, lam, pi, pip, _ = G.slice_op(op)
        single = op < 128 and (op & 1)
        for va in range(4):
            for vb in range(4):
                pa, qa, pb, qb = va & 1, va >> 1, vb & 1, vb >> 1
                if single and (qa or qb):
                    continue
                for ja in (0, 5):
                    for jbv in (3, 6):
                        regs = {"%0": ja & 1, "%1": (ja >> 1) & 1, "%2": (ja >> 2) & 1, "%3": 0,
                                "%4": jbv & 1, "%5": (jbv >> 1) & 1, "%6": (jbv >> 2) & 1, "%7": 1,
                                "%8": 0, "%9": 0, "%10": 0, "%11": 0, "%12": 0, "%13": 0,
                                "%14": pa, "%15": qa, "%16": pb, "%17": qb}
                        out = _run(bodies[op], regs)
                        for (v, j0, J, Zr, Zin, L, PI, PIP) in (
                                (va, ja, ("%0", "%1", "%2"), "%3", 0, "%8", "%9", "%10"),
                                (vb, jbv, ("%4", "%5", "%6"), "%7", 1, "%11", "%12", "%13")):
                            jn = out[J[0]] | (out[J[1]] << 1) | (out[J[2]] << 2)
                            if not (z >> v) & 1:
                                assert jn == (j0 + w[v]) % 8, (op, v)
                            assert out[Zr] == (Zin | ((z >> v) & 1))
                            assert out[L] == (lam >> v) & 1
                            assert out[PI] == (pi >> v) & 1
                            assert out[PIP] == (pip >> v) & 1


@pytest.mark.parametrize("name", ["PZX_SLICE_ROWLOOP_P32", "PZX_SLICE_ROWLOOP_P64"])
def test_fused_row_loop_bodies(name):
    """The fused row loop's class bodies (operands renumbered: %1-%4 J0 J1 J2 Z,
    %5-%7 vl vpi vpip, X / Y in xx / yv) are the same mod-8 chains, and every
    body ends by looping back to the head or leaving the block."""
    text = G.generate()
    block = text[text.index("#define " + name + " "):]
    block = block[:block.index("\n\n")]
    lines = re.findall(r'"(.*?)\\n"', block)
    table = next(ln for ln in lines if ".branchtargets" in ln)
    targets = [int(x.strip().split("_")[0][1:]) for x in table.split(".branchtargets")[1].rstrip(";").split(",")]
    bodies, cur = {}, None
    for ln in lines:
        m = re.match(r"L(\d+)_%=:", ln)
        if m:
            cur = int(m.group(1))
            bodies[cur] = []
        elif cur is not None and ln.startswith("@cont bra.uni H%="):
            cur = None
        elif cur is not None:
            bodies[cur].append(ln)
    assert len(targets) == 129 and set(targets) <= set(bodies)
    assert block.count("@cont bra.uni H%=;") == len(bodies) and block.count("bra.uni X%=;") == len(bodies)
    for op in range(129):
        jb, w, z, lam, pi, pip, _ = G.slice_op(op)
        single = op < 128 and (op & 1)
        body = [ln.replace("xx", "%14").replace("yv", "%15") for ln in bodies[targets[op]]]
        for v in range(4):
            p, q = v & 1, v >> 1
            if single and q:
                continue
            for j0 in range(8):
                regs = {"%1": j0 & 1, "%2": (j0 >> 1) & 1, "%3": (j0 >> 2) & 1, "%4": 0,
                        "%5": 0, "%6": 0, "%7": 0, "%14": p, "%15": q}
                out = _run(body, regs)
                jn = out["%1"] | (out["%2"] << 1) | (out["%3"] << 2)
                if not (z >> v) & 1:
                    assert jn == (j0 + w[v]) % 8, (op, v, j0)
                assert out["%4"] == ((z >> v) & 1)
                assert out["%5"] == (lam >> v) & 1 and out["%6"] == (pi >> v) & 1 and out["%7"] == (pip >> v) & 1
