"""Full-size BASELINE configs through the exact code paths bench.py times.

For every config the table is the bench's own (synth.generate_config, full
size) and the batch is evaluated the way bench.py evaluates it (kernel choice
left to the library: warp-chunk bit-sliced for C1/C4, 128-thread TMEM
bit-sliced for C2, sorted Four-Russians for C3/C5). Each is checked against
  * the reference itself (oracle/_ref: the unmodified core compiled from
    /root/reference, summing subterm_value / ring_mul / ring_add in
    instantiate_diagram's constant-first order, diagram.cpp:149-165,
    ring.cpp:57-86) on a sample of assignments, and
  * the integer-ring kernel (pzx_evaluate_exact: canonical RingQuads, itself
    pinned bit-for-bit to the reference on the goldens, tests/test_exact.py)
    rounded once, on every assignment (C1, C2, C4) or >= 4096 of them (C5);
plus the headline kernels' OWN per-term state (pzx_debug_slice_codes: the
bit planes J, Z, s1, a, b of k_eval_slice / k_eval_slice_wc / k_eval_sorted
at each term's end row), bit-exact against the reference's instantiate_diagram
value of that term at that assignment.

Tolerance (north_star "1e-12 relative in fp64"): |got - want| <= 1e-12 *
max(|want|, 1e-2 * rms(want)) -- 1e-12 relative for every amplitude above 1 %
of the batch RMS (all but ~1e-4 of a Gaussian-distributed batch), and 1e-14 x
RMS absolute below it: an fp64 sum of 2^17..2^24 terms cannot resolve an
amplitude that cancels to ~0 better than ~sqrt(m) ulp of its terms (the
integer-ring path, bit-exact, is the answer for those).
"""
import os

import numpy as np
import pytest

import oracle_py as O
import paper_2403_06777_b200 as P
from paper_2403_06777_b200 import synth
from zw_exact import ZQ, term_from_code

pytestmark = pytest.mark.gpu
TOL = 1e-12
THREADS = os.cpu_count() or 8
IMPL = "ref" if O.have_ref() else "port"


@pytest.fixture(scope="module")
def ctx():
    c = P.Context(0)
    yield c
    c.close()


def assert_close(got, want, tol=TOL, floor_frac=1e-2):
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape
    floor = floor_frac * np.sqrt(np.mean(np.abs(want) ** 2)) if want.size else 0.0
    scale = np.maximum(np.abs(want), floor)
    err = np.abs(got - want)
    bad = err > tol * scale + 1e-300
    assert not bad.any(), f"max rel err {np.max(err / np.maximum(scale, 1e-300)):.3e} at {np.argmax(bad)}"


def exact_to_complex(ex):
    return np.array([O.to_complex(tuple(int(v) for v in row)) for row in ex], np.complex128)


def check_slice_codes(ctx, e, t, terms, words, codes):
    """codes[k, i] (the kernel's own planes for term terms[k] at words[i]) equal the
    reference's instantiate_diagram value of that term, bit for bit."""
    oe = e if isinstance(e, O.OExpr) else O.OExpr(e)
    for k, term in enumerate(terms):
        coef, E, nlm = t.term_info(term)
        for i, w in enumerate(words):
            j, z, s1, a, b = (int(v) for v in codes[k, i])
            got = term_from_code(coef.as_tuple(), E, nlm, j, z, s1, a, b)
            assert got == ZQ.from_quad(O.term_value(oe, term, int(w), impl=IMPL)), (term, int(w))


@pytest.mark.parametrize("cid", ["c1", "c1s"])
def test_c1_full_all_amplitudes(ctx, cid):
    """C1: the real reduction of the 8-qubit T=20 circuit (and the round-1
    synthetic 1024-term table), all 256 amplitudes (warp-chunk kernel) against
    the reference on every assignment, bit-exact against the integer kernel,
    and -- for the circuit -- against the dense statevector."""
    cfg = synth.CONFIGS[cid]
    e = synth.generate_config(cfg)
    t = ctx.compile_bit_table(e)
    amp, prob = ctx.evaluate_range(t, 0, cfg.n_assign, prob=True)
    assert ctx.last_kernel()["kernel"] == "slice_wc"
    words = np.arange(cfg.n_assign, dtype=np.uint64)
    ex, want = O.eval_batch(e, words, THREADS, impl=IMPL)
    assert_close(amp, want)
    assert_close(prob, np.abs(want) ** 2, 2 * TOL)
    assert np.array_equal(ctx.evaluate_exact_range(t, 0, cfg.n_assign), ex)
    if cfg.circuit is not None:
        import statevector as SV
        assert np.max(np.abs(amp - SV.run(synth.config_circuit(cfg)))) <= 1e-12
    # the kernel's own per-term planes, every term at 16 assignments
    pick = np.arange(0, 256, 16, dtype=np.uint64)
    codes = ctx.debug_slice_codes(t, first=0, n=cfg.n_assign)
    check_slice_codes(ctx, e, t, range(t.n_terms), pick, codes[:, pick.astype(np.int64)])


def test_c2_full_headline_kernel(ctx):
    """C2 (the headline): all 2^20 amplitudes on the 128-thread TMEM bit-sliced
    kernel against the integer kernel on EVERY assignment and the reference on
    256; the kernel's own planes for terms at the start, middle and end of the
    table (first, interior and last term chunks of the headline grid)."""
    cfg = synth.CONFIGS["c2"]
    e = synth.generate_config(cfg)
    t = ctx.compile_bit_table(e)
    N = cfg.n_assign
    amp = ctx.evaluate_range(t, 0, N)
    kinfo = ctx.last_kernel()
    assert kinfo["kernel"] == "page" and kinfo["term_chunks"] > 1
    ex = ctx.evaluate_exact_range(t, 0, N)
    assert_close(amp, exact_to_complex(ex))
    # the round-1 bit-sliced kernel (srows layout) on the same batch
    assert_close(ctx.evaluate_range(t, 0, N, flags=P.KERNEL_SLICE), amp, 1e-13, 1.0)
    rng = np.random.default_rng(2)
    pick = np.sort(rng.choice(N, 256, replace=False)).astype(np.uint64)
    ex_ref, want = O.eval_batch(e, pick, THREADS, impl=IMPL)
    assert np.array_equal(ex[pick.astype(np.int64)], ex_ref)
    assert_close(amp[pick.astype(np.int64)], want)
    m = t.n_terms
    for t0 in (0, m // 2 - 3, m - 6):
        codes = ctx.debug_slice_codes(t, first=0, n=N, term_begin=t0, term_end=t0 + 6)
        sub = pick[::16]
        check_slice_codes(ctx, e, t, range(t0, t0 + 6), sub, codes[:, sub.astype(np.int64)])


def test_c2r_real_circuit_all_amplitudes(ctx):
    """C2r: the real reduction of the 20-qubit T=40 circuit, all 2^20 amplitudes
    on the headline kernel against the dense 2^20 statevector (every amplitude),
    the integer kernel (every amplitude) and the reference (64)."""
    import statevector as SV
    cfg = synth.CONFIGS["c2r"]
    e = synth.generate_config(cfg)
    t = ctx.compile_bit_table(e)
    N = cfg.n_assign
    amp = ctx.evaluate_range(t, 0, N)
    assert ctx.last_kernel()["kernel"] == "page"
    sv = SV.run(synth.config_circuit(cfg))
    assert np.max(np.abs(amp - sv)) <= 1e-12 * np.sqrt(np.mean(np.abs(sv) ** 2)) * 1e3
    ex = ctx.evaluate_exact_range(t, 0, N)
    assert_close(amp, exact_to_complex(ex))
    pick = np.random.default_rng(5).choice(N, 64, replace=False).astype(np.uint64)
    ex_ref, want = O.eval_batch(e, pick, THREADS, impl=IMPL)
    assert np.array_equal(ex[pick.astype(np.int64)], ex_ref)


def test_c4_full_marginal_kernel(ctx):
    """C4: the full 2^22-term (2e8-row) doubled-diagram table, all 1024
    enumerated assignments with Re output (warp-chunk kernel, term-chunked
    grid): against the integer kernel on all 1024 and the reference on 16."""
    cfg = synth.CONFIGS["c4"]
    e = synth.generate_config(cfg)
    t = ctx.compile_bit_table(e)
    N = cfg.n_assign
    amp, re = ctx.evaluate_range(t, 0, N, prob_real=True)
    kinfo = ctx.last_kernel()
    assert kinfo["kernel"] == "slice_wc" and kinfo["term_chunks"] > 1
    ex = ctx.evaluate_exact_range(t, 0, N)
    ref = exact_to_complex(ex)
    assert_close(amp, ref)
    assert_close(re, ref.real)
    pick = np.arange(0, N, N // 16, dtype=np.uint64)
    ex_ref, want = O.eval_batch(e, pick, THREADS, impl=IMPL)
    assert np.array_equal(ex[pick.astype(np.int64)], ex_ref)
    assert_close(amp[pick.astype(np.int64)], want)
    codes = ctx.debug_slice_codes(t, first=0, n=N, term_begin=t.n_terms - 4, term_end=t.n_terms)
    check_slice_codes(ctx, e, t, range(t.n_terms - 4, t.n_terms), pick[:4], codes[:, pick[:4].astype(np.int64)])


def test_c5_full_term_split(ctx):
    """C5: the full 2^24-term (8e8-row) table against 2^16 random 32-bit words
    (wide sorted kernel): 4096 words against the integer kernel; the two row-
    balanced term halves combined with evaluate_device + PZX_ACCUMULATE (fp64)
    and with ringquad_sum (exact) equal the unsplit results; the reference on
    4 words; the sorted kernel's own planes on the last terms."""
    torch = pytest.importorskip("torch")
    from paper_2403_06777_b200 import dist as D
    cfg = synth.CONFIGS["c5"]
    e = synth.generate_config(cfg)
    words = synth.assignments(cfg)
    t = ctx.compile_bit_table(e)
    oe = O.OExpr(e)   # marshalled once (8e8 subterms) for the reference calls below
    amp = ctx.evaluate_batch(t, words)
    kinfo = ctx.last_kernel()
    assert kinfo["kernel"] == "sorted" and kinfo["sorted_groups"] == 6
    sub = words[:4096]
    ex = ctx.evaluate_exact(t, sub)
    assert_close(amp[:4096], exact_to_complex(ex))
    # term split in halves on the same device table (term ranges), fp64
    (a0, a1), (b0, b1) = D.term_ranges(e.term_offset, 2)
    n = words.size
    dw = torch.from_numpy(words.view(np.int64)).cuda()
    acc = torch.zeros(2 * n, dtype=torch.float64, device="cuda:0")
    st = torch.cuda.current_stream().cuda_stream
    ctx.evaluate_device(t, n, d_assignments=dw.data_ptr(), term_begin=a0, term_end=a1, d_amp=acc.data_ptr(), stream=st)
    ctx.evaluate_device(t, n, d_assignments=dw.data_ptr(), term_begin=b0, term_end=b1, d_amp=acc.data_ptr(),
                        flags=P.ACCUMULATE, stream=st)
    torch.cuda.synchronize()
    assert_close(acc.cpu().numpy().view(np.complex128), amp, 1e-13, 1.0)
    codes = ctx.debug_slice_codes(t, words, term_begin=t.n_terms - 3, term_end=t.n_terms)  # the bench batch
    assert ctx.last_kernel()["kernel"] == "sorted"
    check_slice_codes(ctx, oe, t, range(t.n_terms - 3, t.n_terms), sub[:8], codes[:, :8])
    t.free()
    # exact halves on their own tables, summed on the device
    parts = []
    for lo, hi in ((a0, a1), (b0, b1)):
        th = ctx.compile_bit_table(e.slice_terms(lo, hi))
        parts.append(ctx.evaluate_exact(th, sub))
        th.free()
    assert np.array_equal(ctx.ringquad_sum(np.stack(parts)), ex)
    # the reference itself on 4 words (8e8 subterm_value calls each)
    ex_ref, want = O.eval_batch(oe, sub[:4], 4, impl=IMPL)
    assert np.array_equal(ex[:4], ex_ref)
    assert_close(amp[:4], want)


@pytest.mark.parametrize("kernel", ["slice", "page", "sorted"])
def test_slice_codes_goldens_and_random(ctx, kernel):
    """Per-term planes of the production kernels on the reference-generated
    goldens and random tables (P up to 32 for sorted, 64 for slice)."""
    import glob
    gold = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "expr_*.npz")))
    cases = []
    for path in gold:
        z = np.load(path)
        e = P.ScalarExpression(int(z["n_params"]), z["term_offset"], z["term_scalar"], z["kind"], z["psi_k"],
                               z["psi_mask"], z["phi_k"], z["phi_mask"])
        cases.append(e)
    cases += [synth.generate(p, 200, 1, 60, 8800 + p) for p in (9, 20, 31)]
    for e in cases:
        t = ctx.compile_bit_table(e)
        if t.max_term_rows > 127 or (kernel in ("sorted", "page") and e.n_params > 32):
            continue
        rng = np.random.default_rng(e.n_params)
        if kernel in ("slice", "page"):
            n = 1 << 14                       # 128-thread TMEM variant (>= 16K assignments)
            first = 0 if e.n_params <= 14 else int(rng.integers(0, 1 << min(e.n_params - 14, 40))) << 14
            fl = P.KERNEL_SLICE if kernel == "slice" else P.KERNEL_PAGE
            codes = ctx.debug_slice_codes(t, first=first, n=n, term_end=min(t.n_terms, 24), flags=fl)
            assert ctx.last_kernel()["kernel"] == kernel
            idx = rng.choice(n, 24, replace=False)
            check_slice_codes(ctx, e, t, range(min(t.n_terms, 24)), np.uint64(first) + idx.astype(np.uint64),
                              codes[:, idx])
        else:
            words = rng.integers(0, 2 ** 64, 4096, dtype=np.uint64)
            if e.n_params >= 20:   # dense window so that the sorted kernel applies
                words = np.uint64(1 << (e.n_params - 3)) + (words & np.uint64((1 << 16) - 1))
            codes = ctx.debug_slice_codes(t, words, term_end=min(t.n_terms, 24), flags=P.KERNEL_SORTED)
            idx = rng.choice(words.size, 24, replace=False)
            check_slice_codes(ctx, e, t, range(min(t.n_terms, 24)), words[idx], codes[:, idx])
        t.free()
