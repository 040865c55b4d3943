"""PZX1 table codec (SPEC "External Interfaces" and serialize/deserialize,
S:396-403): the binary form of a normalised table, its JSON mirror, and the
codec laws -- decode(encode(x)) == x, encode(decode(b)) == b byte for byte,
explicit decode errors (no partial value) on malformed input. CPU only; the
GPU test uploads a PZX1 blob and compares with the expression path."""
import struct

import numpy as np
import pytest

import oracle_py as O
import paper_2403_06777_b200 as P
from paper_2403_06777_b200 import synth


@pytest.mark.parametrize("seed,P_", [(1, 8), (2, 20), (3, 33), (4, 64)])
def test_round_trip_and_oracle_normalisation(seed, P_):
    e = synth.generate(P_, 200, 0, 30, 4000 + seed, "general" if seed % 2 else "clifford")
    b = P.encode_pzx1(e)
    t = P.decode_pzx1(b)
    assert P.encode_pzx1(t) == b                       # byte-identical after a round trip
    # the stored table is the oracle's normalize_subterm output (constants folded)
    f, offs, (ka, psi, kb, phi) = O.normalize_expr(e)
    assert np.array_equal(t.term_coef, f)
    assert np.array_equal(t.term_row_offset, offs)
    assert np.array_equal(t.k_alpha, ka) and np.array_equal(t.k_beta, kb)
    assert np.array_equal(t.psi_mask, psi) and np.array_equal(t.phi_mask, phi)
    # header and size: 32 + 40 m + 19 R with R = m * n_max
    magic, n, m, n_max, R = struct.unpack_from("<4sIQQQ", b, 0)
    sizes = np.diff(offs.astype(np.int64))
    assert magic == b"PZX1" and n == P_ and m == e.n_terms and n_max == sizes.max() and R == m * n_max
    assert len(b) == 32 + 40 * m + 19 * R
    # JSON mirror
    assert P.pzx1_from_json(P.pzx1_to_json(b)) == b


def test_padding_rule_and_empty():
    one = P.RingQuad.one()
    pp = P.Subterm.phase_pair(P.ParamPhase(1, 1), P.ParamPhase(0, 2))
    e = P.ScalarExpression.from_terms(2, [(one, [pp, pp, pp]), (one, [pp])])
    b = P.encode_pzx1(e)
    _, _, m, n_max, R = struct.unpack_from("<4sIQQQ", b, 0)
    assert (m, n_max, R) == (2, 3, 6)                   # SPEC: sizes (3, 1) -> R = 6, 2 dummies
    flags = np.frombuffer(b, np.uint8, R, 32 + 40 * m)
    assert flags.tolist() == [0, 0, 0, 0, 1, 1]
    empty = P.encode_pzx1(P.ScalarExpression.from_terms(4, []))
    assert len(empty) == 32 and P.decode_pzx1(empty).n_terms == 0


def test_decode_errors_are_explicit():
    e = synth.generate(10, 20, 1, 8, 77)
    b = P.encode_pzx1(e)
    for bad in (b[:-1], b[:20], b"", b"PZX2" + b[4:], b + b"\0"):
        with pytest.raises(P.ParseError):
            P.decode_pzx1(bad)
    # a real row after padding is malformed
    _, _, m, n_max, R = struct.unpack_from("<4sIQQQ", b, 0)
    flags_at = 32 + 40 * m
    fl = bytearray(b)
    first_dummy = next(i for i in range(R) if fl[flags_at + i] == 1)
    if (first_dummy + 1) % n_max:
        fl[flags_at + first_dummy + 1] = 0
        with pytest.raises(P.ParseError):
            P.decode_pzx1(bytes(fl))
    with pytest.raises(P.ParseError):
        P.pzx1_from_json('{"magic": "PZX2"}')


@pytest.mark.gpu
def test_upload_pzx1_matches_expression_path():
    ctx = P.Context(0)
    e = synth.generate(20, 500, 1, 40, 4242)
    t1 = ctx.compile_bit_table(e)
    t2 = ctx.upload_pzx1(P.encode_pzx1(e))
    n = 1 << 12
    assert np.array_equal(ctx.evaluate_range(t1, 0, n), ctx.evaluate_range(t2, 0, n))
    words = np.random.default_rng(1).integers(0, 2**20, 777, dtype=np.uint64)
    assert np.array_equal(ctx.evaluate_batch(t1, words), ctx.evaluate_batch(t2, words))
    with pytest.raises(P.ParseError):
        ctx.upload_pzx1(P.encode_pzx1(e)[:-3])
