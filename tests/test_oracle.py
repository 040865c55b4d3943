"""Pin the CPU oracle (oracle/pzx_oracle.c) before trusting it.

1. SPEC known-answer examples and the golden 8x8 pair table of SURVEY §8c.
2. Golden fixtures generated from the reference itself (tests/golden/, made by
   tests/golden/make_golden.py through oracle/_ref).
3. Where oracle/_ref is built (this container; it also travels to the GPU
   box), random expressions are evaluated by both and compared exactly,
   including the error class when the reference throws.
"""
import glob
import json
import math
import os

import numpy as np
import pytest

import oracle_py as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
KATS = json.load(open(os.path.join(GOLD, "kats.json")))

# SURVEY.md §8c golden pair table (a, b, c, d), exp = 0, row = k_alpha
SURVEY_PAIR = """
(2,0,0,0) (2,0,0,0)   (2,0,0,0)   (2,0,0,0)   (2,0,0,0)  (2,0,0,0)   (2,0,0,0)   (2,0,0,0)
(2,0,0,0) (1,1,-1,1)  (1,1,1,0)   (2,0,0,1)   (0,1,0,1)  (1,0,1,0)   (1,0,-1,1)  (0,1,0,0)
(2,0,0,0) (1,1,1,0)   (2,0,2,0)   (1,0,1,1)   (0,0,2,0)  (1,-1,1,0)  (0,0,0,0)   (1,0,1,-1)
(2,0,0,0) (2,0,0,1)   (1,0,1,1)   (1,-1,1,1)  (0,-1,0,1) (0,-1,0,0)  (1,-1,-1,0) (1,0,-1,0)
(2,0,0,0) (0,1,0,1)   (0,0,2,0)   (0,-1,0,1)  (-2,0,0,0) (0,-1,0,-1) (0,0,-2,0)  (0,1,0,-1)
(2,0,0,0) (1,0,1,0)   (1,-1,1,0)  (0,-1,0,0)  (0,-1,0,-1)(1,-1,-1,-1)(1,0,-1,-1) (2,0,0,-1)
(2,0,0,0) (1,0,-1,1)  (0,0,0,0)   (1,-1,-1,0) (0,0,-2,0) (1,0,-1,-1) (2,0,-2,0)  (1,1,-1,0)
(2,0,0,0) (0,1,0,0)   (1,0,1,-1)  (1,0,-1,0)  (0,1,0,-1) (2,0,0,-1)  (1,1,-1,0)  (1,1,1,-1)
"""


def _survey_pairs():
    rows = []
    for line in SURVEY_PAIR.strip().splitlines():
        cells = line.replace(")(", ") (").split()
        rows.append([tuple(int(v) for v in c.strip("()").split(",")) for c in cells])
    return rows


def test_pair_table_matches_survey_and_reference_golden():
    sp = _survey_pairs()
    for a in range(8):
        for b in range(8):
            v = O.pair_value(a, b)
            assert v[:4] == sp[a][b] and v[4] == 0
            assert list(v) == KATS["pair_table"][a][b]


def test_spec_ring_kats():
    # S:348-350
    assert O.ring_add((1, 0, 0, 0, 0), (1, 0, 0, 0, 0)) == (2, 0, 0, 0, 0)
    x = O.make(3, -2, 5, 1, 2)
    assert O.ring_add(x, (0, 0, 0, 0, 0)) == x
    assert O.ring_add((0, 1, 0, 1, 1), (0, 1, 0, -1, 1)) == (0, 1, 0, 0, 0)  # = sqrt2 canonical
    # S:357-359
    assert O.ring_mul((1, 1, 0, 0, 0), (1, 1, 0, 0, 0)) == (3, 2, 0, 0, 0)
    assert O.ring_mul(x, (1, 0, 0, 0, 0)) == x
    assert O.ring_mul((0, 0, 1, 0, 0), (0, 0, 1, 0, 0)) == (-1, 0, 0, 0, 0)
    # S:363 phase_to_ring table; S:407 w^j w^k = w^(j+k)
    table = [(1, 0, 0, 0, 0), (0, 1, 0, 1, 1), (0, 0, 1, 0, 0), (0, -1, 0, 1, 1),
             (-1, 0, 0, 0, 0), (0, -1, 0, -1, 1), (0, 0, -1, 0, 0), (0, 1, 0, -1, 1)]
    for k in range(8):
        assert O.omega(k) == table[k]
        for j in range(8):
            assert O.ring_mul(O.omega(j), O.omega(k)) == O.omega((j + k) % 8)
    with pytest.raises(O.OracleError):
        O.omega(8)


def test_spec_phase_kats():
    # S:64-66 (p1 = bit 0, p2 = bit 1)
    assert O.instantiate_phase(1, 0b11, 0b11, 2) == 1
    assert O.instantiate_phase(1, 0b11, 0b01, 2) == 5
    assert O.instantiate_phase(6, 0, 0b11, 2) == 6
    # bits above n_params are dropped by ParamAssignment::total (phase.hpp:18-23)
    assert O.instantiate_phase(0, 0b1, 0b10, 1) == 0
    # MissingParameter: mask beyond the declared parameters
    with pytest.raises(O.OracleError) as e:
        O.instantiate_phase(0, 0b100, 0, 2)
    assert e.value.status == O.E_MISSING


def test_spec_normalize_and_eval_kats():
    # S:375-377 pi_pair Psi=(1,{}), Phi=(0,{}): value 1; Phi=(4,{}): value w
    c, pair = O.normalize(3, 1, 0, 0, 0)
    assert c == (1, 0, 0, 0, 0) and pair is None
    c, pair = O.normalize(3, 1, 0, 4, 0)
    assert c == O.omega(1) and pair is None
    # node (0, {}) -> 2
    assert O.normalize(0, 0, 0)[0] == (2, 0, 0, 0, 0)
    # pair(1, 4) = 2w = (0,1,0,1,0)
    assert O.pair_value(1, 4) == (0, 1, 0, 1, 0)
    # pair((0,{p1}), (0,{p1})) at p1 = 1 -> -2
    assert O.subterm_value(1, 0, 1, 0, 1, 1, 1) == (-2, 0, 0, 0, 0)


def test_bss_target_value():
    # ((1 + w)/2)^6 = (-7 - 5 sqrt2 + i(7 + 5 sqrt2)) / 2^5
    x = O.ring_mul(O.ring_add((1, 0, 0, 0, 0), O.omega(1)), (1, 0, 0, 0, 1))
    v = (1, 0, 0, 0, 0)
    for _ in range(6):
        v = O.ring_mul(v, x)
    assert v == (-7, -5, 7, 5, 5)
    z = O.to_complex(v)
    assert z == complex(-0.43972086912079611, 0.43972086912079611) or abs(z - complex(-0.4397208691207961, 0.4397208691207961)) < 1e-16


def test_reduce_strided_worked_example():
    # App. E worked example: sum of 0..9 = 45 in the exact ring
    tot = (0, 0, 0, 0, 0)
    for i in range(10):
        tot = O.ring_add(tot, (i, 0, 0, 0, 0))
    assert tot == (45, 0, 0, 0, 0)


def test_kats_json_from_reference():
    for r in KATS["ring"]:
        assert list(O.ring_add(tuple(r["x"]), tuple(r["y"]))) == r["add"]
        assert list(O.ring_mul(tuple(r["x"]), tuple(r["y"]))) == r["mul"]
        c = O.to_complex(tuple(r["x"]))
        assert (c.real, c.imag) == tuple(r["cx"])
    for k, mask, word, P, want in KATS["instantiate_phase"]:
        assert O.instantiate_phase(k, mask, word, P) == want


def test_normalize_exhaustive_against_reference_golden():
    """Exhaustive normalize_subterm + subterm_value check."""
    n = 0
    for rec in KATS["normalize"]:
        kind, pk, pm, fk, fm = rec["s"]
        if "norm_err" in rec:
            with pytest.raises(O.OracleError) as e:
                O.normalize(kind, pk, pm, fk, fm)
            assert e.value.status == rec["norm_err"]
        else:
            c, pair = O.normalize(kind, pk, pm, fk, fm)
            assert [list(c), list(pair) if pair else None] == rec["norm"]
        for word, want in enumerate(rec["val"]):
            if isinstance(want, int):
                with pytest.raises(O.OracleError) as e:
                    O.subterm_value(kind, pk, pm, fk, fm, word, 2)
                assert e.value.status == -want
            else:
                got = O.subterm_value(kind, pk, pm, fk, fm, word, 2)
                assert list(got) == want
                # the normalised form reproduces the value at every assignment (Lemmas 3-5)
                if "norm" in rec:
                    c, pair = rec["norm"]
                    v = tuple(c)
                    if pair:
                        kp = O.instantiate_phase(pair[0], pair[1], word, 2)
                        kf = O.instantiate_phase(pair[2], pair[3], word, 2)
                        v = O.ring_mul(v, O.pair_value(kp, kf))
                    assert list(v) == want
                    n += 1
    assert n > 3000


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "expr_*.npz"))))
def test_expression_goldens(path):
    z = np.load(path)
    e = type("E", (), {k: z[k] for k in z.files})
    ex, amp = O.eval_batch(e, z["words"], 4)
    assert (ex == z["exact"]).all()
    assert np.array_equal(amp, z["amp"])


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built here")
@pytest.mark.parametrize("seed", range(6))
def test_port_equals_reference_random(seed):
    from paper_2403_06777_b200 import synth
    rng = np.random.default_rng(seed)
    P = int(rng.integers(1, 65))
    e = synth.generate(P, int(rng.integers(1, 40)), 1, 20, 1000 + seed, "general" if seed % 2 else "clifford")
    words = rng.integers(0, 2**64, 64, dtype=np.uint64)
    try:
        ex_r, amp_r = O.eval_batch(e, words, 2, impl="ref")
    except O.OracleError as err:
        with pytest.raises(O.OracleError) as e2:
            O.eval_batch(e, words, 2)
        assert e2.value.status == err.status
        return
    ex_p, amp_p = O.eval_batch(e, words, 2)
    assert (ex_p == ex_r).all() and np.array_equal(amp_p, amp_r)
    # per-term values against the literal instantiate_diagram
    for t in range(min(e.n_terms, 5)):
        assert O.term_value(e, t, int(words[0])) == O.term_value(e, t, int(words[0]), impl="ref")


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built here")
def test_port_error_classes_match_reference():
    # HalfPi outside {2,6}: DomainError; PiPair selector not Pauli: DomainError
    assert O.normalize(2, 2, 1) and True
    for args in [(2, 3, 1), (3, 1, 1, 2, 1)]:
        with pytest.raises(O.OracleError) as a:
            O.normalize(*args)
        with pytest.raises(O.OracleError) as b:
            O.normalize(*args, impl="ref")
        assert a.value.status == b.value.status == O.E_DOMAIN


def test_to_complex_no_fma():
    v = (3, 7, -5, 11, 3)
    s2 = math.sqrt(2.0)
    want = complex((3.0 + 7.0 * s2) * 0.125, (-5.0 + 11.0 * s2) * 0.125)
    assert O.to_complex(v) == want
