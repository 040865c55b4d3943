"""GPU parity: the sm_100a path against the CPU oracle (pinned to the reference).

Bars (north_star): phase indices bit-exact; per-term products bit-exact (exact
exponent codes, reconstructed with big integers); amplitudes within

    |amp_gpu - amp_ref| <= 1e-12 * max(|amp_ref|, rms(amp_ref over the batch))

i.e. 1e-12 relative, with the batch RMS as the floor for amplitudes that
cancel to (near) zero. Every call goes through the C ABI (ctypes).
"""
import glob
import os

import numpy as np
import pytest

import oracle_py as O
import paper_2403_06777_b200 as P
from paper_2403_06777_b200 import synth
from zw_exact import ZQ, term_from_code

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
GOLDENS = sorted(glob.glob(os.path.join(GOLD, "expr_*.npz")))
TOL = 1e-12


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


def assert_close(got, want, tol=TOL):
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape
    floor = np.sqrt(np.mean(np.abs(want) ** 2)) if want.size else 0.0
    scale = np.maximum(np.abs(want), floor)
    err = np.abs(got - want)
    bad = err > tol * scale + 1e-300
    assert not bad.any(), f"max rel err {np.max(err / np.maximum(scale, 1e-300)):.3e} at {np.argmax(bad)}"
    return float(np.max(err / np.maximum(scale, 1e-300))) if want.size else 0.0


@pytest.mark.parametrize("path", GOLDENS)
def test_phase_indices_bit_exact(ctx, path):
    e, z = load(path)
    t = ctx.compile_bit_table(e)
    words = z["words"][:32]
    got = ctx.debug_phase_indices(t, words)
    want = O.phase_indices(e, words)
    assert got.shape == want.shape
    assert np.array_equal(got, want)


@pytest.mark.parametrize("path", GOLDENS)
def test_term_products_bit_exact(ctx, path):
    e, z = load(path)
    t = ctx.compile_bit_table(e)
    words = z["words"][:8]
    codes = ctx.debug_term_codes(t, words)
    for term in range(min(t.n_terms, 40)):
        coef, E, nlm = t.term_info(term)
        for wi, w in enumerate(words):
            j, zz, s1, a, b = (int(v) for v in codes[term, wi])
            got = term_from_code(coef.as_tuple(), E, nlm, j, zz, s1, a, b)
            assert got == ZQ.from_quad(O.term_value(e, term, int(w))), (term, int(w))


@pytest.mark.parametrize("path", GOLDENS)
@pytest.mark.parametrize("kernel", ["auto", "general"])
def test_amplitudes_vs_reference_goldens(ctx, path, kernel):
    e, z = load(path)
    t = ctx.compile_bit_table(e)
    flags = P.KERNEL_GENERAL if kernel == "general" else 0
    amp, prob = ctx.evaluate_batch(t, z["words"], prob=True, flags=flags)
    assert_close(amp, z["amp"])
    assert_close(prob, np.abs(z["amp"]) ** 2, 1e-11)


@pytest.mark.parametrize("path", [p for p in GOLDENS if "p8" in p])
def test_enumerated_range_kernels(ctx, path):
    e, z = load(path)
    t = ctx.compile_bit_table(e)
    n = len(z["words"])
    a_gray = ctx.evaluate_range(t, 0, n, flags=P.KERNEL_GRAY)
    a_gen = ctx.evaluate_range(t, 0, n, flags=P.KERNEL_GENERAL)
    a_slice = ctx.evaluate_range(t, 0, n, flags=P.KERNEL_SLICE)
    a_slice2 = ctx.evaluate_range(t, 0, n, flags=P.KERNEL_SLICE2)
    assert_close(a_gray, z["amp"])
    assert_close(a_gen, z["amp"])
    assert_close(a_slice, z["amp"])
    assert_close(a_slice2, z["amp"])
    # explicit contiguous word list (what pzx_evaluate sees from a user sweep)
    assert_close(ctx.evaluate_batch(t, np.arange(n, dtype=np.uint64)), z["amp"])
    # unaligned start (general kernel) and ragged length
    assert_close(ctx.evaluate_range(t, 3, n - 7), z["amp"][3:n - 4])


@pytest.mark.parametrize("P_", [3, 5, 12, 20, 33, 64])
def test_slice_kernel_vs_oracle(ctx, P_):
    """Bit-sliced kernel on enumerated batches, against the reference oracle."""
    e = synth.generate(P_, 700, 1, 40, 300 + P_)
    t = ctx.compile_bit_table(e)
    n = 1 << min(P_, 11)
    first = 0 if P_ <= 11 else 32 * 12345
    amp = ctx.evaluate_range(t, first, n, flags=P.KERNEL_SLICE)
    words = np.arange(first, first + n, dtype=np.uint64)
    idx = np.random.default_rng(P_).choice(n, min(n, 96), replace=False)
    _, want = O.eval_batch(e, words[idx], 8, impl="ref" if O.have_ref() else "port")
    assert_close(amp[idx], want)
    assert_close(amp, ctx.evaluate_range(t, first, n, flags=P.KERNEL_GENERAL), 1e-13)


@pytest.mark.parametrize("P_", [10, 14, 20, 27, 32])
def test_page_kernel_vs_oracle(ctx, P_):
    """Page-layout kernel (C / G / D row families, lane-parity pre-pass, zero
    skip) on enumerated batches: against the reference oracle and the
    round-1 bit-sliced kernel, both row mixes, ragged batch ends, term chunks."""
    for mix in ("general", "clifford"):
        e = synth.generate(P_, 900, 0, 60, 1700 + P_, mix, exp_cap=40)  # keeps the reference's int64 ring_add in range
        t = ctx.compile_bit_table(e)
        n = (1 << min(P_, 16)) - 77
        first = 0 if P_ <= 16 else 1024 * 37
        amp = ctx.evaluate_range(t, first, n, flags=P.KERNEL_PAGE)
        assert ctx.last_kernel()["kernel"] == "page"
        words = np.arange(first, first + n, dtype=np.uint64)
        idx = np.random.default_rng(P_).choice(n, 64, replace=False)
        _, want = O.eval_batch(e, words[idx], 8, impl="ref" if O.have_ref() else "port")
        assert_close(amp[idx], want)
        assert_close(amp, ctx.evaluate_range(t, first, n, flags=P.KERNEL_SLICE), 1e-13)
        assert_close(ctx.evaluate_range(t, first, n), amp, 1e-13)   # auto


def test_page_kernel_zero_skip(ctx):
    """Terms whose constraint rows kill every assignment of a warp are skipped
    (the skip is exact: the skipped terms are zero there)."""
    R = P.RingQuad
    nd = lambda k, m: P.Subterm.node(P.ParamPhase(k, m))  # noqa: E731
    pp = lambda a, m1, b, m2: P.Subterm.phase_pair(P.ParamPhase(a, m1), P.ParamPhase(b, m2))  # noqa: E731
    terms = []
    for i in range(300):
        # (1 + (-1)^{a_15}) kills every assignment with bit 15 set; bits 10..14 vary per warp
        rows = [nd(0, 1 << 15), pp(1, (i % 7 + 1) << 3, 3, 0b101), nd(1, 0b11 | 1 << (10 + i % 5))]
        terms.append((R.make(i % 5 + 1, 1, 0, 0, 2), rows))
    e = P.ScalarExpression.from_terms(16, terms)
    t = ctx.compile_bit_table(e)
    amp = ctx.evaluate_range(t, 0, 1 << 16, flags=P.KERNEL_PAGE)
    assert np.all(amp[1 << 15:] == 0)
    assert_close(amp, ctx.evaluate_range(t, 0, 1 << 16, flags=P.KERNEL_GENERAL), 1e-13)


@pytest.mark.parametrize("P_", [3, 6, 12, 20, 33, 64])
def test_slice2_kernel_vs_oracle(ctx, P_):
    """Two-slice (64 assignments / thread, TMEM accumulators) enumerated kernel."""
    e = synth.generate(P_, 700, 1, 40, 900 + P_)
    t = ctx.compile_bit_table(e)
    n = 1 << min(P_, 13)
    first = 0 if P_ <= 13 else 64 * 4321
    amp = ctx.evaluate_range(t, first, n, flags=P.KERNEL_SLICE2)
    words = np.arange(first, first + n, dtype=np.uint64)
    idx = np.random.default_rng(P_).choice(n, min(n, 96), replace=False)
    _, want = O.eval_batch(e, words[idx], 8, impl="ref" if O.have_ref() else "port")
    assert_close(amp[idx], want)
    assert_close(amp, ctx.evaluate_range(t, first, n, flags=P.KERNEL_GENERAL), 1e-13)
    # term-chunked grid (partials + fixed-order reduction) on a long batch
    amp2 = ctx.evaluate_range(t, first, 1 << 16, flags=P.KERNEL_SLICE2)
    assert_close(amp2[:n], amp, 1e-13)


@pytest.mark.parametrize("P_", [7, 20, 32, 33, 64])
def test_slice_rand_kernel_vs_oracle(ctx, P_):
    """Bit-sliced kernel on arbitrary word lists (transposed parameter planes)."""
    e = synth.generate(P_, 600, 1, 40, 500 + P_)
    t = ctx.compile_bit_table(e)
    words = np.random.default_rng(P_).integers(0, 2**64, 3000, dtype=np.uint64)  # high bits ignored
    amp = ctx.evaluate_batch(t, words, flags=P.KERNEL_SLICE_RAND)
    idx = np.random.default_rng(1).choice(words.size, 64, replace=False)
    _, want = O.eval_batch(e, words[idx], 8, impl="ref" if O.have_ref() else "port")
    assert_close(amp[idx], want)
    assert_close(amp, ctx.evaluate_batch(t, words, flags=P.KERNEL_GENERAL), 1e-13)


@pytest.mark.parametrize("P_", [12, 20, 30, 32])
def test_sorted_kernel_vs_oracle(ctx, P_):
    """Sort + Four-Russians bit-sliced kernel on dense random batches (C3-like)."""
    e = synth.generate(P_, 500, 1, 40, 700 + P_)
    t = ctx.compile_bit_table(e)
    n = min(1 << P_, 1 << 16) + 77                        # ragged tail, duplicates when P_ is small
    rng = np.random.default_rng(P_)
    words = rng.integers(0, 2**64, n, dtype=np.uint64)
    if P_ >= 20:   # a dense window (density ~1/64 like C3): 32-word groups span < 2^16
        lo = 1 << (P_ - 3)
        words = np.uint64(lo) + (words & np.uint64((1 << min(22, P_ - 3)) - 1))
        words |= np.uint64(7) << np.uint64(P_ + 3)  # bits above n_params must be ignored
    amp = ctx.evaluate_batch(t, words, flags=P.KERNEL_SORTED)
    idx = rng.choice(n, 64, replace=False)
    _, want = O.eval_batch(e, words[idx], 8, impl="ref" if O.have_ref() else "port")
    assert_close(amp[idx], want)
    assert_close(amp, ctx.evaluate_batch(t, words, flags=P.KERNEL_GENERAL), 1e-13)
    # auto choice on the same batch agrees
    assert_close(ctx.evaluate_batch(t, words), amp, 1e-13)


@pytest.mark.parametrize("P_,n", [(28, 4096 + 5), (32, (1 << 16) + 33)])
def test_sorted_kernel_wide_tables(ctx, P_, n):
    """Sparse batches (C5-like: 2^16 random 32-bit words): 32-word groups span
    2^16..2^24, so the sorted kernel uses 6 Four-Russians groups (24 bits)."""
    e = synth.generate(P_, 300, 1, 40, 1100 + P_)
    t = ctx.compile_bit_table(e)
    rng = np.random.default_rng(P_)
    words = rng.integers(0, 2**64, n, dtype=np.uint64)
    amp = ctx.evaluate_batch(t, words, flags=P.KERNEL_SORTED)
    idx = rng.choice(n, 48, replace=False)
    _, want = O.eval_batch(e, words[idx], 8, impl="ref" if O.have_ref() else "port")
    assert_close(amp[idx], want)
    assert_close(amp, ctx.evaluate_batch(t, words, flags=P.KERNEL_GENERAL), 1e-13)
    assert_close(ctx.evaluate_batch(t, words), amp, 1e-13)


def test_sorted_kernel_rejects_sparse_batches(ctx):
    e = synth.generate(32, 64, 1, 20, 9)
    t = ctx.compile_bit_table(e)
    words = np.random.default_rng(3).integers(0, 2**32, 1024, dtype=np.uint64)  # ~4 words per 2^24 window
    with pytest.raises(P.Error):
        ctx.evaluate_batch(t, words, flags=P.KERNEL_SORTED)
    # auto falls back to the POPC kernel
    _, want = O.eval_batch(e, words[:16], 8)
    assert_close(ctx.evaluate_batch(t, words)[:16], want)


def test_random_assignments_mid_size(ctx):
    e = synth.generate(20, 4096, 16, 48, 77)
    t = ctx.compile_bit_table(e)
    rng = np.random.default_rng(3)
    words = rng.integers(0, 2**64, 4096, dtype=np.uint64)
    amp = ctx.evaluate_batch(t, words)
    idx = rng.choice(len(words), 48, replace=False)
    _, want = O.eval_batch(e, words[idx], 8, impl="ref" if O.have_ref() else "port")
    assert_close(amp[idx], want)


def test_p64_and_high_bits(ctx):
    e = synth.generate(64, 256, 4, 20, 5)
    t = ctx.compile_bit_table(e)
    words = np.random.default_rng(9).integers(0, 2**64, 300, dtype=np.uint64)
    _, want = O.eval_batch(e, words, 8)
    assert_close(ctx.evaluate_batch(t, words), want)
    # P < 64: bits >= P are ignored (ParamAssignment::total, phase.hpp:18-23)
    e2 = synth.generate(12, 128, 4, 20, 6)
    t2 = ctx.compile_bit_table(e2)
    lo = words & np.uint64(0xFFF)
    assert np.array_equal(ctx.evaluate_batch(t2, words), ctx.evaluate_batch(t2, lo))


def test_edge_cases(ctx):
    one = P.RingQuad.one()
    # empty expression: S = 0
    t = ctx.compile_bit_table(P.ScalarExpression.from_terms(4, []))
    assert np.all(ctx.evaluate_range(t, 0, 16) == 0)
    # a term without assignment-dependent rows is its constant (BSS target S:474)
    half = P.RingQuad.make(1, 0, 0, 0, 1)
    node = P.Subterm.node(P.ParamPhase(1, 0))  # (1 + w), parameter-free -> folded
    t = ctx.compile_bit_table(P.ScalarExpression.from_terms(3, [(P.RingQuad.make(1, 0, 0, 0, 6), [node] * 6)]))
    v = ctx.evaluate_range(t, 0, 8)
    assert_close(v, np.full(8, complex(-0.4397208691207961, 0.4397208691207961)))
    # single row, S:455-456 examples through the whole path
    pp = P.Subterm.phase_pair(P.ParamPhase(0, 1), P.ParamPhase(0, 1))
    t = ctx.compile_bit_table(P.ScalarExpression.from_terms(1, [(one, [pp])]))
    assert_close(ctx.evaluate_batch(t, [0, 1]), np.array([2.0, -2.0]))
    # Clifford-only table, C = 1/2
    t = ctx.compile_bit_table(P.ScalarExpression.from_terms(0, [(half, [])]))
    assert_close(ctx.evaluate_batch(t, [0, 5]), np.array([0.5, 0.5]))
    # n = 0 and n = 1
    assert ctx.evaluate_batch(t, []).size == 0
    # Re(value) output for doubled diagrams
    _, pr = ctx.evaluate_range(t, 0, 4, prob_real=True)
    assert np.allclose(pr, 0.5, rtol=0, atol=1e-15)
    # validation at upload
    with pytest.raises(P.MissingParameter):
        ctx.compile_bit_table(P.ScalarExpression.from_terms(2, [(one, [P.Subterm.node(P.ParamPhase(1, 4))])]))


def test_long_terms_segment_path(ctx):
    path = [p for p in GOLDENS if "long" in p][0]
    e, z = load(path)
    t = ctx.compile_bit_table(e)
    assert t.max_term_rows > 127
    assert_close(ctx.evaluate_batch(t, z["words"]), z["amp"])
    assert_close(ctx.evaluate_batch(t, z["words"], flags=P.KERNEL_GENERAL), z["amp"])


@pytest.mark.parametrize("m", [0, 3, 11, 13])
def test_marginal_sum(ctx, m):
    """Marginal summing: sum of |amp|^2 (or Re amp) over the
    2^m settings of the low m parameters, against per-assignment evaluation."""
    P_ = 18
    e = synth.generate(P_, 400, 1, 30, 1300 + m)
    t = ctx.compile_bit_table(e)
    rng = np.random.default_rng(m)
    fixed = (rng.integers(0, 1 << (P_ - m), 5, dtype=np.uint64) << np.uint64(m)).astype(np.uint64)
    got = ctx.marginal_sum(t, fixed, m)
    for i, f in enumerate(fixed):
        amp = ctx.evaluate_range(t, int(f), 1 << m)
        want = float(np.sum(np.abs(amp) ** 2))
        assert abs(got[i] - want) <= 1e-12 * max(want, 1e-300), (i, got[i], want)
    got_re = ctx.marginal_sum(t, fixed[:2], m, prob_real=True)
    for i, f in enumerate(fixed[:2]):
        want = float(np.sum(ctx.evaluate_range(t, int(f), 1 << m).real))
        assert abs(got_re[i] - want) <= 1e-12 * max(abs(want), np.sqrt(np.sum(np.abs(want) ** 2)), 1e-300) + 1e-12
    # deterministic, and the oracle agrees on a small case
    assert np.array_equal(ctx.marginal_sum(t, fixed, m), got)
    if m <= 3:
        words = (fixed[0] | np.arange(1 << m, dtype=np.uint64)).astype(np.uint64)
        _, want = O.eval_batch(e, words, 8, impl="ref" if O.have_ref() else "port")
        assert abs(got[0] - np.sum(np.abs(want) ** 2)) <= 1e-12 * np.sum(np.abs(want) ** 2)
    with pytest.raises(P.Error):
        ctx.marginal_sum(t, fixed | np.uint64(1), max(m, 1))


def test_device_pointer_api_and_term_split(ctx):
    torch = pytest.importorskip("torch")
    e = synth.generate(10, 3000, 16, 40, 21)
    t = ctx.compile_bit_table(e)
    n = 1024
    full = ctx.evaluate_range(t, 0, n)
    amp = torch.zeros(2 * n, dtype=torch.float64, device="cuda:0")
    part = torch.zeros(2 * n, dtype=torch.float64, device="cuda:0")
    cut = 1234
    st = torch.cuda.current_stream().cuda_stream
    ctx.evaluate_device(t, n, first=0, term_begin=0, term_end=cut, d_amp=amp.data_ptr(), stream=st)
    ctx.evaluate_device(t, n, first=0, term_begin=cut, d_amp=part.data_ptr(), stream=st)
    torch.cuda.synchronize()
    s = (amp + part).cpu().numpy().view(np.complex128)
    assert_close(s, full, 1e-13)
    # PZX_ACCUMULATE: the second range adds into the first one's amplitudes
    acc = torch.zeros(2 * n, dtype=torch.float64, device="cuda:0")
    ctx.evaluate_device(t, n, first=0, term_begin=0, term_end=cut, d_amp=acc.data_ptr(), stream=st)
    ctx.evaluate_device(t, n, first=0, term_begin=cut, d_amp=acc.data_ptr(), flags=P.ACCUMULATE, stream=st)
    torch.cuda.synchronize()
    assert_close(acc.cpu().numpy().view(np.complex128), full, 1e-13)
    prob = torch.empty(n, dtype=torch.float64, device="cuda:0")
    both = amp + part
    ctx.amp_to_prob_device(both.data_ptr(), n, prob.data_ptr(), stream=st)
    torch.cuda.synchronize()
    assert_close(prob.cpu().numpy(), np.abs(full) ** 2, 1e-12)


def test_full_size_c2_properties(ctx):
    """BASELINE config C2 at full size: enumerated 2^20 assignments, 2^17 terms."""
    cfg = synth.CONFIGS["c2"]
    e = synth.generate_config(cfg)
    t = ctx.compile_bit_table(e)
    N = cfg.n_assign
    amp = ctx.evaluate_range(t, 0, N)
    # shard invariance (what the multi-GPU assignment split relies on)
    half = ctx.evaluate_range(t, N // 2, N // 2)
    assert_close(half, amp[N // 2:], 1e-13)
    # the other enumerated kernels agree (auto picks the bit-sliced one here)
    assert_close(ctx.evaluate_range(t, 0, N, flags=P.KERNEL_GRAY), amp, 1e-13)
    # general kernel on a random subset of the same words
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(N, 2048, replace=False)).astype(np.uint64)
    assert_close(ctx.evaluate_batch(t, idx, flags=P.KERNEL_GENERAL), amp[idx.astype(np.int64)], 1e-13)
    # oracle spot check (reference implementation where built, else the port)
    pick = idx[:16]
    _, want = O.eval_batch(e, pick, os.cpu_count() or 8, impl="ref" if O.have_ref() else "port")
    assert_close(amp[pick.astype(np.int64)], want)


def product_marginal_tables(s):
    """Doubled-marginal tables of a product distribution over len(s) bits,
    p_j(0) = (1 + s_j) / 2 with dyadic s_j: P_k(a) = prod_{j<k} p_j(a_j)
    = sum over subsets S of [k] of prod_{j in S} s_j / 2^k * (-1)^{parity(S & a)};
    (-1)^parity as the pair row V(4 parity, 4) / 2 = PhasePair((0, S), (4, {}))/2."""
    exprs = []
    for k in range(1, len(s) + 1):
        terms = []
        for S in range(1 << k):
            sign, den = 1, k
            for j in range(k):
                if S >> j & 1:
                    num, d = s[j]
                    sign *= num
                    den += d
            if S == 0:
                terms.append((P.RingQuad.make(1, 0, 0, 0, k), []))
            else:
                pp = P.Subterm.phase_pair(P.ParamPhase(0, S), P.ParamPhase(4, 0))
                terms.append((P.RingQuad.make(sign, 0, 0, 0, den + 1), [pp]))
        exprs.append(P.ScalarExpression.from_terms(k, terms))
    return exprs


def test_weak_sample_product_distribution(ctx):
    """Repeated weak simulation (PAPER App. F Alg. 2) on tables whose marginals
    are known in closed form: bit frequencies and a joint frequency within
    6 sigma of the product distribution, reproducible per seed."""
    s = [(1, 1), (-1, 1), (1, 1), (1, 2), (-1, 2), (0, 0)]   # s_j = num / 2^d: 1/2, -1/2, 1/2, 1/4, -1/4, 0
    exprs = product_marginal_tables(s)
    # the tables are the marginals (oracle check of the construction)
    for k, e in enumerate(exprs[:3], 1):
        words = np.arange(1 << k, dtype=np.uint64)
        _, v = O.eval_batch(e, words, 4)
        p0 = [(1 + (n / 2 ** d)) / 2 for n, d in s]
        want = [np.prod([p0[j] if not (w >> j) & 1 else 1 - p0[j] for j in range(k)]) for w in range(1 << k)]
        assert np.allclose(v.real, want, rtol=0, atol=1e-15) and np.allclose(v.imag, 0, atol=1e-15)
    tables = [ctx.compile_bit_table(e) for e in exprs]
    N = 1 << 16
    w = ctx.weak_sample(tables, N, seed=7)
    assert w.dtype == np.uint64 and np.all(w < (1 << len(s)))
    p0 = np.array([(1 + (n / 2 ** d)) / 2 for n, d in s])
    f0 = np.array([np.mean(((w >> np.uint64(j)) & np.uint64(1)) == 0) for j in range(len(s))])
    sig = np.sqrt(p0 * (1 - p0) / N)
    assert np.all(np.abs(f0 - p0) <= 6 * sig + 1e-12), (f0, p0)
    both = np.mean((w & np.uint64(3)) == 0)
    pj = p0[0] * p0[1]
    assert abs(both - pj) <= 6 * np.sqrt(pj * (1 - pj) / N)
    assert np.array_equal(ctx.weak_sample(tables, N, seed=7), w)
    assert not np.array_equal(ctx.weak_sample(tables, N, seed=8), w)
    # deterministic distribution: s = +1 -> always 0, s = -1 -> always 1
    det = [ctx.compile_bit_table(e) for e in product_marginal_tables([(1, 0), (-1, 0), (1, 0)])]
    assert np.all(ctx.weak_sample(det, 1000, seed=1) == 0b010)
    with pytest.raises(P.Error):   # table k must take k + 1 parameters
        ctx.weak_sample([tables[1], tables[0]], 10)


def test_backend_contract(ctx):
    c = ctx.backend_contract()
    assert c["max_params"] == 64 and c["deterministic"] == 1 and c["exact"] == 0
    assert c["max_rows_per_term"] == 127 and c["n_sm"] > 0 and c["preferred_batch"] > 0


@pytest.mark.parametrize("mode", ["replicate", "split_terms"])
def test_group_api_two_contexts(ctx, mode):
    """pzx_group_* with two contexts on the one GPU of the box: the sharding /
    term-split logic and the ordered partial sum, against one context."""
    e = synth.generate(16, 900, 4, 40, 1500)
    t = ctx.compile_bit_table(e)
    g = P.Group([0, 0])
    gt = g.upload(e, P.REPLICATE if mode == "replicate" else P.SPLIT_TERMS)
    n = 1 << 14
    assert_close(g.evaluate_range(gt, 0, n), ctx.evaluate_range(t, 0, n), 1e-13)
    words = np.random.default_rng(5).integers(0, 1 << 16, 3001, dtype=np.uint64)
    assert_close(g.evaluate_batch(gt, words), ctx.evaluate_batch(t, words), 1e-13)
    gt.free()
    g.close()


@pytest.mark.parametrize("seed", range(6))
def test_fuzz_kernels_against_oracle(ctx, seed):
    """Random shapes through every kernel the library can pick: random P, term
    lengths up to 120 rows, both row mixes; the forced and automatic choices
    agree with each other and with the reference oracle on a sample."""
    rng = np.random.default_rng(7000 + seed)
    P_ = int(rng.choice([5, 9, 14, 20, 27, 32, 40, 64]))
    mix = "general" if seed % 2 else "clifford"
    e = synth.generate(P_, int(rng.integers(50, 400)), 0, int(rng.integers(8, 121)), 7100 + seed, mix)
    t = ctx.compile_bit_table(e)
    n = int(rng.integers(40, 5000))
    first = 0 if P_ <= 12 else int(rng.integers(0, 1 << min(P_, 40)) // 64 * 64)
    ref = ctx.evaluate_range(t, first, n, flags=P.KERNEL_GENERAL)
    for fl in (0, P.KERNEL_GRAY, P.KERNEL_SLICE, P.KERNEL_SLICE2):
        assert_close(ctx.evaluate_range(t, first, n, flags=fl), ref, 1e-13)
    words = rng.integers(0, 2**64, n, dtype=np.uint64)
    gen = ctx.evaluate_batch(t, words, flags=P.KERNEL_GENERAL)
    assert_close(ctx.evaluate_batch(t, words), gen, 1e-13)            # auto (sorted where it applies)
    assert_close(ctx.evaluate_batch(t, words, flags=P.KERNEL_SLICE_RAND), gen, 1e-13)
    idx = rng.choice(n, 24, replace=False)
    try:
        _, want = O.eval_batch(e, words[idx], 8, impl="ref" if O.have_ref() else "port")
    except O.OracleError:  # the reference's int64 RingQuad overflows on long random terms (ring.cpp:61-63)
        return
    assert_close(gen[idx], want)


def test_simplify_pairwise_node_cancellation(ctx):
    """PZX_COMPILE_SIMPLIFY (PAPER "Conclusions"): Node rows on one mask whose
    constants differ by pi fold into the term constant, 0/pi pairs zero the
    term; values equal the unsimplified table and the oracle."""
    R = P.RingQuad
    nd = lambda k, m: P.Subterm.node(P.ParamPhase(k, m))  # noqa: E731
    pp = lambda a, m1, b, m2: P.Subterm.phase_pair(P.ParamPhase(a, m1), P.ParamPhase(b, m2))  # noqa: E731
    terms = [
        (R.make(1, 0, 0, 0, 1), [nd(2, 0b011), nd(6, 0b011), pp(1, 0b100, 3, 0b010)]),     # (1+i)(1-i) = 2 folds
        (R.make(3, 1, 0, 0, 2), [nd(0, 0b101), nd(4, 0b101), pp(1, 0b001, 1, 0b010)]),     # 0 / pi pair: zero term
        (R.make(1, 0, 1, 0, 1), [nd(1, 0b110), nd(5, 0b110), nd(3, 0b110), nd(7, 0b110)]),  # two pairs
        (R.make(-2, 0, 0, 1, 0), [pp(1, 0b111, 2, 0b001), nd(1, 0b010)]),                  # nothing to fold
    ]
    e = P.ScalarExpression.from_terms(3, terms)
    plain = ctx.compile_bit_table(e)
    simp = ctx.compile_bit_table(e, simplify=True)
    assert simp.n_rows < plain.n_rows
    words = np.arange(8, dtype=np.uint64)
    _, want = O.eval_batch(e, words, 4)
    assert_close(ctx.evaluate_batch(simp, words), want)
    assert_close(ctx.evaluate_batch(plain, words), want)
    # random tables over few parameters (many shared masks): identical values on every kernel
    for seed in range(3):
        e2 = synth.generate(4, 600, 2, 30, 4400 + seed)
        t1, t2 = ctx.compile_bit_table(e2), ctx.compile_bit_table(e2, simplify=True)
        assert t2.n_rows <= t1.n_rows
        a1 = ctx.evaluate_range(t1, 0, 16, flags=P.KERNEL_GENERAL)
        for fl in (0, P.KERNEL_GENERAL, P.KERNEL_SLICE):
            assert_close(ctx.evaluate_range(t2, 0, 16, flags=fl), a1, 1e-12)


@pytest.mark.parametrize("P_", [33, 64])
def test_wide_params_tmem_slice_path(ctx, P_):
    """P > 32 through the 128-thread TMEM bit-sliced kernel (batches >= 16K)
    and the warp-chunk kernel (small batches), against the POPC kernel and the
    oracle; bits above the parameter count are ignored."""
    e = synth.generate(P_, 300, 1, 40, 5200 + P_)
    t = ctx.compile_bit_table(e)
    first = (1 << (P_ - 2)) + 64 * 977
    n = 1 << 15
    amp = ctx.evaluate_range(t, first, n)
    assert_close(amp, ctx.evaluate_range(t, first, n, flags=P.KERNEL_GENERAL), 1e-13)
    small = ctx.evaluate_range(t, first, 2048)
    assert_close(small, amp[:2048], 1e-13)
    idx = np.random.default_rng(P_).choice(n, 24, replace=False)
    _, want = O.eval_batch(e, (np.uint64(first) + idx.astype(np.uint64)), 8, impl="ref" if O.have_ref() else "port")
    assert_close(amp[idx], want)


def test_sorted_kernel_sub_batches(ctx):
    """Word lists above the sorted kernel's 2^26 batch cap run as independent
    sorted sub-batches (bounded scratch); results in the caller's order."""
    e = synth.generate(24, 64, 1, 12, 5300)
    t = ctx.compile_bit_table(e)
    n = (1 << 26) + 1000
    words = np.random.default_rng(1).integers(0, 1 << 24, n, dtype=np.uint64)
    amp = ctx.evaluate_batch(t, words)
    idx = np.random.default_rng(2).choice(n, 4096, replace=False)
    idx[:2] = [n - 1, (1 << 26) - 1]
    assert_close(amp[idx], ctx.evaluate_batch(t, words[idx], flags=P.KERNEL_GENERAL), 1e-13)
