"""CPU emulation of the page kernel's row families (pzx_table_page_layout):
every record of the page layout is interpreted exactly as k_eval_page does
(X = parity ? ~W : W via the record words, then C: Z |= X; G: J += (k + 4p)q~;
L: J += k p, S += p ^ inv; D: the class op's w'(p, q) / zero / lambda / pi /
pi' tables) and the per-term
exponent codes, with the term's folded j offset, must reconstruct the
reference's instantiate_diagram value (diagram.cpp:149-165) bit for bit.
No GPU: this pins the host classification the GPU tests then exercise."""
import numpy as np
import pytest

import oracle_py as O
import paper_2403_06777_b200 as P
from paper_2403_06777_b200 import synth
from zw_exact import ZQ, term_from_code

PAGE = 256
OPS = None


def par(x):
    return bin(int(x)).count("1") & 1


def vec(w0, w1, mask, a):
    """The kernel's X for assignment a: bit (a % 32) of (parity(mask & a_hi) ? w1 : w0)."""
    hi = int(a) & ~31
    return ((int(w1) if par(int(mask) & hi) else int(w0)) >> (int(a) & 31)) & 1


def emulate_term(slots, hdr, a):
    global OPS
    if OPS is None:
        OPS = P.slice_op_table()
    cnt = int(slots[hdr, 4])
    nc, ng, nd = cnt & 0xFF, (cnt >> 8) & 0xFF, (cnt >> 16) & 0xFF
    nl = (int(slots[hdr, 5]) & 0xFF) + (int(slots[hdr, 5]) >> 8)  # L0 + L4
    ng += sum((int(slots[hdr, 6]) >> (8 * i)) & 0xFF for i in range(4)) + int(slots[hdr, 7])  # + S2..E2, G3
    j = z = s1 = pa = pb = 0
    q = hdr + 1
    for _ in range(nc):
        w = slots[q]
        z |= vec(w[0], w[1], w[6], a)
        q += 1
    cls = [0] * 4 + [ng, int(slots[hdr, 7])]
    for i in range(4):
        cls[i] = (int(slots[hdr, 6]) >> (8 * i)) & 0xFF
        cls[4] -= cls[i]
    cls[4] -= cls[5]
    for c, n_c in enumerate(cls):          # S2, S6, E0, E2, G1, G3: the kernel's per-class updates
        for _ in range(n_c):
            w = slots[q]
            X = vec(w[0], w[1], w[6], a)
            Y = vec(w[2], w[3], w[7], a)
            k = (1 if w[4] else 0) + (2 if w[5] else 0)
            if c == 0:
                assert w[6] == 0 and k == 2 and w[0] == 0
                j += 2 * Y
            elif c == 1:
                assert w[6] == 0 and k == 2 and w[0] == 0xFFFFFFFF
                j += 6 * Y
            elif c == 2:
                assert k == 0
                j += 4 * (X & Y)
            elif c == 3:
                assert k == 2
                j += 2 * Y + 4 * (X & Y)
            elif c == 4:
                assert k == 1
                j += Y + 4 * (X & Y)        # X = p ^ K2: v2 = Y & X carries k's bit 2
            else:
                assert k == 3
                j += -Y + 4 * (X & Y)       # X stored complemented: 3Y + 4(~X)Y = -Y + 4XY (mod 8)
            q += 1
    for i_l in range(nl):
        w = slots[q]
        lam = vec(w[0], w[1], w[6], a)      # Lambda = p ^ inv, from the x parity word
        p_ = vec(w[2], w[3], w[6], a)
        k = (1 if w[4] else 0) + (2 if w[5] else 0) + (4 if w[7] else 0)
        assert k == (0 if i_l < (int(slots[hdr, 5]) & 0xFF) else 4)   # L0 rows, then L4 rows
        j += k * p_
        s1 += lam
        q += 1
    for _ in range(nd):
        w = slots[q]
        p_ = vec(w[0], w[1], w[6], a)
        q_ = vec(w[2], w[3], w[7], a)
        op = int(w[5])
        jb, w0, w1, w2, w3, ztt, ltt, ptt, pptt, _ = OPS[op]
        v = p_ | (q_ << 1)
        if (ztt >> v) & 1:
            z = 1
        j += (w0, w1, w2, w3)[v]
        s1 += (ltt >> v) & 1
        pa += (ptt >> v) & 1
        pb += (pptt >> v) & 1
        q += 1
    return j & 7, z, s1, pa, pb


@pytest.mark.parametrize("case", ["p8", "p20", "p31", "clifford", "c1", "simplify"])
def test_page_layout_reconstructs_reference_terms(case):
    if case == "c1":
        e = synth.generate_config(synth.CONFIGS["c1"])
    elif case == "clifford":
        e = synth.generate(12, 80, 0, 40, 31, mix="clifford")
    elif case == "simplify":
        e = synth.generate(6, 80, 2, 30, 32)
    else:
        Pn = int(case[1:])
        e = synth.generate(Pn, 120, 0, 60, 700 + Pn)
    h = P.HostTable(e)
    lay = h.page_layout()
    assert lay is not None
    slots, tslot, jfold, fam = lay
    assert slots.shape[0] % PAGE == 0 and int(fam[:5].sum()) == h.n_rows and fam[5:].sum() == fam[1]
    assert len(fam) == 11
    # no term straddles a page; the last term of every used page is flagged
    for t in range(h.n_terms):
        cnt = int(slots[tslot[t], 4])
        n = 1 + (cnt & 0xFF) + ((cnt >> 8) & 0xFF) + ((cnt >> 16) & 0xFF) + (int(slots[tslot[t], 5]) & 0xFF)
        n += int(slots[tslot[t], 5]) >> 8
        n += sum((int(slots[tslot[t], 6]) >> (8 * i)) & 0xFF for i in range(4)) + int(slots[tslot[t], 7])
        assert tslot[t] // PAGE == (tslot[t] + n - 1) // PAGE
        nxt = tslot[t + 1] if t + 1 < h.n_terms else None
        if nxt is not None and nxt // PAGE != tslot[t] // PAGE:
            assert (cnt >> 24) & 1
    oe = O.OExpr(e)
    impl = "ref" if O.have_ref() else "port"
    rng = np.random.default_rng(5)
    words = rng.integers(0, 1 << e.n_params, 6, dtype=np.uint64)
    for t in range(min(h.n_terms, 60)):
        coef, E, nlm = h.term_info(t)
        for w in words:
            j, z, s1, a, b = emulate_term(slots, int(tslot[t]), int(w))
            got = term_from_code(coef.as_tuple(), E, nlm, (j + int(jfold[t])) & 7, z, s1, a, b)
            assert got == ZQ.from_quad(O.term_value(oe, t, int(w), impl=impl)), (case, t, int(w))


def test_page_families_on_the_headline_table():
    """C2's rows: the generic (branch-free) family carries the bulk."""
    h = P.HostTable(synth.generate_config(synth.CONFIGS["c2"]))
    _, _, _, fam = h.page_layout()
    c, g, d, dropped, l_ = (int(x) for x in fam[:5])
    assert c + g + d + dropped + l_ == h.n_rows
    assert g > 0.7 * h.n_rows and c > 0 and d > 0
