"""CPU tests of the product's native library (no GPU needed).

* libpzx_gpu.so loads and exports every symbol include/pzx_gpu.h declares;
* the host table compiler (pzx_table_compile_host) folds exactly the
  constants the oracle's normalize_subterm restatement folds;
* the per-class variant codes the kernels add, combined with the per-term
  constants, reproduce the oracle's exact per-term value at every assignment
  (big-integer check of the factorisation) -- this is the same
  arithmetic the CUDA kernels perform, emulated exactly on the host;
* no evaluation path exists without the CUDA device (fails loudly).
"""
import ctypes
import glob
import os
import re

import numpy as np
import pytest

import oracle_py as O
import paper_2403_06777_b200 as P
from paper_2403_06777_b200 import _native as N
from paper_2403_06777_b200 import synth
from zw_exact import ZQ, pair_value, term_from_code

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def header_symbols():
    text = open(os.path.join(ROOT, "include", "pzx_gpu.h")).read()
    return sorted(set(re.findall(r"\b(pzx_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(N.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(N.EXPORTS)


def test_status_strings_and_version():
    L = N.lib()
    assert L.pzx_status_string(0) == b"ok"
    assert L.pzx_status_string(3) == b"missing parameter"
    assert b"sm_100a" in L.pzx_version()


def test_class_table_matches_exact_factorisation():
    codes, e, lm = P.class_table()
    for ka in range(8):
        for kb in range(8):
            for v in range(4):
                p, q = v & 1, v >> 1
                want = pair_value(ka + 4 * p, kb + 4 * q)
                c = int(codes[ka * 8 + kb, v])
                z, s1, a, b, j = c & 127, (c >> 7) & 127, (c >> 14) & 127, (c >> 21) & 127, c >> 29
                got = term_from_code((1, 0, 0, 0, 0), int(e[ka * 8 + kb]), int(lm[ka * 8 + kb]), j, z, s1, a, b)
                assert got == want, (ka, kb, p, q)
    # 32 classes are monomial-under-flips; here: e=2 for k in {0,4}, e=3 for {2,6}^2
    assert sorted(np.bincount(e, minlength=4).tolist()) == [0, 4, 28, 32]


def _emulate_codes(expr, words):
    """Host emulation of what the kernels accumulate: per (term, word) codes."""
    codes, _, _ = P.class_table()
    folded, offs, (ka, psi, kb, phi) = O.normalize_expr(expr)
    m = len(offs) - 1
    out = np.zeros((m, len(words), 5), np.int64)
    pr = lambda x: bin(int(x)).count("1") & 1  # noqa: E731
    for t in range(m):
        for wi, w in enumerate(words):
            acc = [0, 0, 0, 0, 0]
            for r in range(int(offs[t]), int(offs[t + 1])):
                p, q = pr(int(psi[r]) & int(w)), pr(int(phi[r]) & int(w))
                c = int(codes[int(ka[r]) * 8 + int(kb[r]), p | (q << 1)])
                acc[0] += c >> 29
                acc[1] += c & 127
                acc[2] += (c >> 7) & 127
                acc[3] += (c >> 14) & 127
                acc[4] += (c >> 21) & 127
            out[t, wi] = acc
    return folded, offs, out


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "expr_*.npz"))))
def test_host_compile_matches_oracle_normalisation(path):
    z = np.load(path)
    e = P.ScalarExpression(int(z["n_params"]), z["term_offset"], z["term_scalar"], z["kind"], z["psi_k"],
                           z["psi_mask"], z["phi_k"], z["phi_mask"])
    h = P.HostTable(e)
    folded, offs, _ = O.normalize_expr(e)
    assert h.n_terms == e.n_terms and h.n_rows == int(offs[-1])
    for t in range(e.n_terms):
        c, _, _ = h.term_info(t)
        assert c.as_tuple() == tuple(int(v) for v in folded[t])


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "expr_*.npz")))[:4])
def test_exponent_codes_reproduce_exact_term_values(path):
    z = np.load(path)
    e = P.ScalarExpression(int(z["n_params"]), z["term_offset"], z["term_scalar"], z["kind"], z["psi_k"],
                           z["psi_mask"], z["phi_k"], z["phi_mask"])
    h = P.HostTable(e)
    words = [int(w) for w in z["words"][:6]]
    _, offs, codes = _emulate_codes(e, words)
    for t in range(min(e.n_terms, 24)):
        coef, E, nlm = h.term_info(t)
        for wi, w in enumerate(words):
            j, zz, s1, a, b = (int(v) for v in codes[t, wi])
            got = term_from_code(coef.as_tuple(), E, nlm, j % 8, zz, s1, a, b)
            want = ZQ.from_quad(O.term_value(e, t, w))
            assert got == want, (t, w)


def test_host_compile_validation_errors():
    ok = P.ScalarExpression.from_terms(3, [(P.RingQuad.one(), [P.Subterm.node(P.ParamPhase(1, 0b101))])])
    P.HostTable(ok)
    bad_mask = P.ScalarExpression.from_terms(2, [(P.RingQuad.one(), [P.Subterm.node(P.ParamPhase(1, 0b100))])])
    with pytest.raises(P.MissingParameter):
        P.HostTable(bad_mask)
    bad_half = P.ScalarExpression.from_terms(2, [(P.RingQuad.one(), [P.Subterm(P.SubtermKind.HalfPi, P.ParamPhase(3, 1))])])
    with pytest.raises(P.DomainError):
        P.HostTable(bad_half)
    bad_pi = P.ScalarExpression.from_terms(2, [(P.RingQuad.one(), [P.Subterm(P.SubtermKind.PiPair, P.ParamPhase(1, 1), P.ParamPhase(2, 2))])])
    with pytest.raises(P.DomainError):
        P.HostTable(bad_pi)
    with pytest.raises(P.DomainError):
        P.ScalarExpression.from_terms(65, [])
    long_term = P.ScalarExpression.from_terms(2, [(P.RingQuad.one(), [P.Subterm.node(P.ParamPhase(0, 1))] * 5000)])
    with pytest.raises(P.DomainError):  # capacity (PZX_E_CAPACITY) maps to DomainError
        P.HostTable(long_term)


def test_subterm_constructors_mirror_reference():
    s = P.Subterm.pi_pair(P.ParamPhase(4, 1), P.ParamPhase(1, 2))  # phi not Pauli -> swapped
    assert s.phi.k == 4 and s.psi.k == 1
    with pytest.raises(P.DomainError):
        P.Subterm.pi_pair(P.ParamPhase(1, 1), P.ParamPhase(3, 2))
    with pytest.raises(P.DomainError):
        P.Subterm.half_pi(P.ParamPhase(1, 1))
    assert P.ParamPhase(-1).k == 7
    assert P.phase_add(P.ParamPhase(4, 1), P.ParamPhase(4, 1)) == P.ParamPhase(0, 0)


def test_ringquad_python_mirror_matches_oracle():
    rng = np.random.default_rng(1)
    for _ in range(200):
        x = P.RingQuad.make(*[int(v) for v in rng.integers(-40, 41, 4)], int(rng.integers(0, 5)))
        y = P.RingQuad.make(*[int(v) for v in rng.integers(-40, 41, 4)], int(rng.integers(0, 5)))
        assert (x * y).as_tuple() == O.ring_mul(x.as_tuple(), y.as_tuple())
        assert (x + y).as_tuple() == O.ring_add(x.as_tuple(), y.as_tuple())
        assert x.to_complex() == O.to_complex(x.as_tuple())


def test_no_device_means_no_evaluation():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(P.CudaError):
        P.Context(0)


def test_synth_is_deterministic_and_within_invariants():
    cfg = synth.CONFIGS["c1s"]
    a = synth.generate_config(cfg)
    b = synth.generate_config(cfg)
    for f in ("term_offset", "term_scalar", "kind", "psi_k", "psi_mask", "phi_k", "phi_mask"):
        assert np.array_equal(getattr(a, f), getattr(b, f))
    assert a.n_terms == cfg.n_terms
    n = np.diff(a.term_offset.astype(np.int64))
    assert n.min() >= cfg.n_lo and n.max() <= cfg.n_hi
    assert (a.psi_mask < (1 << cfg.n_params)).all() and (a.psi_mask != 0).all()
    half = a.kind == 2
    assert np.isin(a.psi_k[half], [2, 6]).all()
    assert np.isin(a.phi_k[a.kind == 3], [0, 4]).all()
    assert (a.phi_mask[(a.kind == 0) | half] == 0).all()
    assert (a.term_scalar[:, :4] != 0).any(axis=1).all()
