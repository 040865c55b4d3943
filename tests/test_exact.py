"""Exact evaluation (pzx_evaluate_exact): the SPEC's integer-ring backend
contract -- "any two conforming backends produce identical RingQuad outputs"
(S:444), "data-parallel output = reference output, component-for-component
exactly". Bar: bit-identical canonical RingQuads (a, b, c, d, exp)
against the oracle's sequential fold (ring_add over instantiate_diagram values,
diagram.cpp:149-165; the oracle is pinned to the reference in test_oracle.py),
and OverflowError exactly where the value leaves int64."""
import glob
import os

import numpy as np
import pytest

import oracle_py as O
import paper_2403_06777_b200 as P
from paper_2403_06777_b200 import synth

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
GOLDENS = sorted(glob.glob(os.path.join(GOLD, "expr_*.npz")))


@pytest.fixture(scope="module")
def ctx():
    c = P.Context(0)
    yield c
    c.close()


def load(path):
    z = np.load(path)
    e = P.ScalarExpression(int(z["n_params"]), z["term_offset"], z["term_scalar"], z["kind"], z["psi_k"],
                           z["psi_mask"], z["phi_k"], z["phi_mask"])
    return e, z


def exact_oracle(e, words):
    return O.eval_batch(e, words, 8)[0]


def to_complex(q):
    s2 = np.sqrt(2.0)
    sc = np.ldexp(1.0, -q[:, 4])
    return (q[:, 0] + q[:, 1] * s2) * sc + 1j * (q[:, 2] + q[:, 3] * s2) * sc


@pytest.mark.parametrize("path", GOLDENS)
def test_exact_vs_oracle_goldens(ctx, path):
    e, z = load(path)
    t = ctx.compile_bit_table(e)
    words = z["words"]
    got = ctx.evaluate_exact(t, words)
    assert np.array_equal(got, exact_oracle(e, words))
    # the exact values round to the golden amplitudes the reference produced
    amp = to_complex(got)
    assert np.allclose(amp, z["amp"], rtol=1e-12, atol=1e-12 * np.sqrt(np.mean(np.abs(z["amp"]) ** 2)))


@pytest.mark.parametrize("P_,mix,lo,hi", [(8, "clifford", 0, 20), (12, "general", 1, 40), (20, "general", 2, 32),
                                           (33, "general", 1, 24), (64, "general", 1, 16)])
def test_exact_random_tables(ctx, P_, mix, lo, hi):
    e = synth.generate(P_, 700, lo, hi, 5100 + P_, mix)
    t = ctx.compile_bit_table(e)
    rng = np.random.default_rng(P_)
    words = rng.integers(0, 2 ** min(P_, 63), 300, dtype=np.uint64)
    try:
        want = exact_oracle(e, words)
    except O.OracleError:
        pytest.skip("oracle fold overflows on this table")
    assert np.array_equal(ctx.evaluate_exact(t, words), want)


def test_exact_range_chunking_and_long_terms(ctx):
    # enumerated range == the same words as a list; small n -> many term chunks
    e = synth.generate(10, 3000, 1, 24, 5300)
    t = ctx.compile_bit_table(e)
    words = np.arange(1024, dtype=np.uint64)
    want = exact_oracle(e, words)
    assert np.array_equal(ctx.evaluate_exact_range(t, 0, 1024), want)
    assert np.array_equal(ctx.evaluate_exact(t, words[:7]), want[:7])      # 1 CTA, chunked
    assert np.array_equal(ctx.evaluate_exact(t, words[::-1]), want[::-1])
    # terms longer than the SWAR segment (> 127 rows)
    path = [p for p in GOLDENS if "long" in p][0]
    e2, z = load(path)
    t2 = ctx.compile_bit_table(e2)
    assert t2.max_term_rows > 127
    assert np.array_equal(ctx.evaluate_exact(t2, z["words"]), exact_oracle(e2, z["words"]))


def test_exact_edge_cases(ctx):
    R = P.RingQuad
    # empty expression: canonical zero
    t = ctx.compile_bit_table(P.ScalarExpression.from_terms(4, []))
    assert np.array_equal(ctx.evaluate_exact_range(t, 0, 4), np.zeros((4, 5), np.int64))
    assert ctx.evaluate_exact(t, []).shape == (0, 5)
    # parameter-free term: its folded constant, canonical (1/2 -> exp 1)
    t = ctx.compile_bit_table(P.ScalarExpression.from_terms(0, [(R.make(1, 0, 0, 0, 1), [])]))
    assert ctx.evaluate_exact(t, [0, 3]).tolist() == [[1, 0, 0, 0, 1]] * 2
    # V(0,0) = 2, V(4,4) = -2
    pp = P.Subterm.phase_pair(P.ParamPhase(0, 1), P.ParamPhase(0, 1))
    t = ctx.compile_bit_table(P.ScalarExpression.from_terms(1, [(R.one(), [pp])]))
    assert ctx.evaluate_exact(t, [0, 1]).tolist() == [[2, 0, 0, 0, 0], [-2, 0, 0, 0, 0]]
    # cancellation to exact zero: C and -C
    e = synth.generate(6, 40, 1, 8, 5400)
    ts = e.term_scalar.reshape(-1, 5)
    neg = ts.copy()
    neg[:, :4] *= -1
    e2 = P.ScalarExpression(6, np.concatenate([e.term_offset, e.term_offset[1:] + e.term_offset[-1]]),
                            np.concatenate([ts, neg]), np.tile(e.kind, 2), np.tile(e.psi_k, 2),
                            np.tile(e.psi_mask, 2), np.tile(e.phi_k, 2), np.tile(e.phi_mask, 2))
    t = ctx.compile_bit_table(e2)
    assert np.array_equal(ctx.evaluate_exact_range(t, 0, 64), np.zeros((64, 5), np.int64))


def test_exact_overflow_is_explicit(ctx):
    R = P.RingQuad
    big = R.make(1 << 62, 0, 0, 0, 0)
    # 2^62 + 2^62 = 2^63: out of int64 -> OverflowError (the oracle's fold throws too)
    e = P.ScalarExpression.from_terms(2, [(big, []), (big, [])])
    with pytest.raises(O.OracleError):
        exact_oracle(e, np.arange(2, dtype=np.uint64))
    t = ctx.compile_bit_table(e)
    with pytest.raises(P.OverflowError):
        ctx.evaluate_exact(t, [0, 1])
    out = ctx.evaluate_exact(t, [0, 1], allow_overflow=True)
    assert (out[:, 4] == -1).all()
    # a value that fits after cancellation is fine: 2^62 - 2^62 + 3
    e = P.ScalarExpression.from_terms(2, [(big, []), (R.make(-(1 << 62), 0, 0, 0, 0), []), (R.make(3, 0, 0, 0, 0), [])])
    assert ctx.evaluate_exact(ctx.compile_bit_table(e), [0]).tolist() == [[3, 0, 0, 0, 0]]


@pytest.mark.parametrize("cid", ["c2", "c3"])
def test_exact_full_size_tables_vs_float_kernels(ctx, cid):
    """BASELINE tables at full size (C2: 2^17 terms / 4.2e6 rows; C3: 2^18
    terms, P = 30): the integer-ring kernel and the fp64 bit-sliced / sorted
    kernels are independent implementations of the same sum; on a sample of
    assignments the exact values, rounded once, equal the fp64 amplitudes to
    1e-12 relative (batch-RMS floor), and the integer kernel is shard- and
    order-invariant bit for bit."""
    cfg = synth.CONFIGS[cid]
    e = synth.generate_config(cfg)
    t = ctx.compile_bit_table(e)
    rng = np.random.default_rng(7)
    words = rng.integers(0, 2 ** cfg.n_params, 4096, dtype=np.uint64)
    ex = ctx.evaluate_exact(t, words)
    amp = ctx.evaluate_batch(t, words)
    ref = to_complex(ex)
    floor = np.sqrt(np.mean(np.abs(ref) ** 2))
    assert np.all(np.abs(amp - ref) <= 1e-12 * np.maximum(np.abs(ref), floor))
    assert np.array_equal(ctx.evaluate_exact(t, words[:100]), ex[:100])
    assert np.array_equal(ctx.evaluate_exact(t, words[::-1]), ex[::-1])
    # oracle spot check at full size
    assert np.array_equal(ex[:4], O.eval_batch(e, words[:4], 8)[0])


@pytest.mark.parametrize("G", [1, 2, 5])
def test_ringquad_sum_term_split(ctx, G):
    """pzx_ringquad_sum: exact partials of G row-balanced term ranges (the term
    split) summed on the device equal the whole table's values."""
    from paper_2403_06777_b200 import dist as D
    e = synth.generate(16, 300, 2, 40, 11 + G)
    words = np.random.default_rng(G).integers(0, 1 << 16, 2000, dtype=np.uint64)
    full = ctx.evaluate_exact(ctx.compile_bit_table(e), words)
    parts = []
    for t0, t1 in D.term_ranges(e.term_offset, G):
        t = ctx.compile_bit_table(e.slice_terms(t0, t1))
        parts.append(ctx.evaluate_exact(t, words))
        t.free()
    got = ctx.ringquad_sum(np.stack(parts))
    assert np.array_equal(got, full)
    assert np.array_equal(got, exact_oracle(e, words))
    # the device-pointer path used by dist.gpu_exact_sum_fn
    import torch
    dev = torch.from_numpy(np.stack(parts)).cuda()
    got_d = D.gpu_exact_sum_fn(ctx)(dev).cpu().numpy()
    assert np.array_equal(got_d, full)


def test_ringquad_sum_vs_oracle_ring_add(ctx):
    """Random canonical RingQuads (mixed exponents, cancellations, zeros): the
    device sum equals the reference's ring_add fold (ring.cpp:57-70)."""
    rng = np.random.default_rng(5)
    G, n = 4, 3000
    parts = np.zeros((G, n, 5), np.int64)
    for r in range(G):
        for i in range(n):
            v = rng.integers(-2**20, 2**20, 4) if rng.random() < 0.8 else np.zeros(4, np.int64)
            parts[r, i] = O.make(*(int(x) for x in v), int(rng.integers(0, 30)))[:5]
    parts[1, :100, :4] = -parts[0, :100, :4]  # exact cancellation -> canonical zero
    parts[1, :100, 4] = parts[0, :100, 4]
    parts[2:, :100] = 0
    got = ctx.ringquad_sum(parts)
    for i in range(n):
        acc = tuple(int(x) for x in parts[0, i])
        for r in range(1, G):
            acc = O.ring_add(acc, tuple(int(x) for x in parts[r, i]))
        assert tuple(got[i]) == acc[:5], i
    assert not got[:100].any()


def test_ringquad_sum_overflow_is_explicit(ctx):
    big = np.array([[[2**62, 0, 0, 0, 0]], [[2**62, 0, 0, 0, 0]]], np.int64)
    with pytest.raises(P.OverflowError):
        ctx.ringquad_sum(big)
    got = ctx.ringquad_sum(big, allow_overflow=True)
    assert got[0, 4] == -1
    flagged = np.array([[[1, 0, 0, 0, 0]], [[0, 0, 0, 0, -1]]], np.int64)  # an overflowed partial
    assert ctx.ringquad_sum(flagged, allow_overflow=True)[0, 4] == -1
    assert np.array_equal(ctx.ringquad_sum(np.zeros((3, 0, 5), np.int64)), np.zeros((0, 5), np.int64))
