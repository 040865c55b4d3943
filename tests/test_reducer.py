"""The host parametric reducer (csrc/pzx_reduce.cpp) against a dense statevector.

SPEC acceptance #1: for >= 50 random Clifford+T circuits (<= 6
qubits, <= 40 gates, T <= 16, <= 4 parameters) every assignment of the
parametric pipeline's value equals the dense statevector amplitude within
1e-9. The pipeline here is reducer -> leaf-term expression -> the reference's
own evaluator (oracle/_ref where built, else the pinned C port) -- the GPU path
is checked against the same expressions in the -m gpu tests. Plus the SPEC's
examples, the doubled marginals (summing = doubling =
statevector, completeness), non-parametric == parametric bit for bit, the
term-count bound and parametric inputs. CPU only.
"""
import numpy as np
import pytest

import oracle_py as O
import statevector as SV
from paper_2403_06777_b200 import circuit as CI
from paper_2403_06777_b200 import synth

IMPL = "ref" if O.have_ref() else "port"


def values(red, words):
    ex, amp = O.eval_batch(red.expr, np.asarray(words, np.uint64), 4, impl=IMPL)
    return ex, amp


def all_outputs(n):
    return [CI.param(q) for q in range(n)]


def test_spec_examples():
    # empty circuit <0|I|0> = 1; <0|H|0> = 1/sqrt2; CNOT |10> -> |11>
    assert values(CI.reduce_amplitudes(CI.Circuit(1), [0]), [0])[1][0] == 1
    v = values(CI.reduce_amplitudes(CI.Circuit(1).add("h", 0), [0]), [0])[0][0]
    assert tuple(v) == (0, 1, 0, 0, 1)                     # sqrt2 / 2, exactly
    c = CI.Circuit(2).add("cx", 0, 1)
    assert values(CI.reduce_amplitudes(c, [1, 1], in_spec=[1, 0]), [0])[1][0] == 1
    assert values(CI.reduce_amplitudes(c, [1, 0], in_spec=[1, 0]), [0])[1].size == 1
    # <1|H|0> = 1/sqrt2; identity doubled, a = 0 -> 1, a = 1 -> 0
    assert abs(values(CI.reduce_amplitudes(CI.Circuit(1).add("h", 0), [1]), [0])[1][0] - 2 ** -0.5) < 1e-15
    d = CI.reduce_doubled(CI.Circuit(1), [CI.param(0)])
    assert np.allclose(values(d, [0, 1])[1], [1, 0])
    # 1-qubit H, a parametric: P = 1/2 at both assignments
    d = CI.reduce_doubled(CI.Circuit(1).add("h", 0), [CI.param(0)])
    assert np.allclose(values(d, [0, 1])[1], [0.5, 0.5])
    # the doubled diagram carries twice the T-count
    c = CI.random_clifford_t(3, 5, seed=1)
    assert CI.reduce_doubled(c, [CI.param(0), CI.TRACED, 0]).t_count == 2 * c.t_count()


@pytest.mark.parametrize("seed", range(60))
def test_acceptance_1_random_circuits_vs_statevector(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 7))
    t = int(rng.integers(0, 17))
    c = CI.random_clifford_t(n, t, n_clifford=int(rng.integers(4, max(5, 40 - t))), seed=seed)
    assert len(c.gates) <= 40 + n and c.t_count() == t
    k = min(n, 4)                                  # <= 4 parameters: outputs 0..k-1, the rest fixed
    rest = [int(b) for b in rng.integers(0, 2, n - k)]
    red = CI.reduce_amplitudes(c, all_outputs(k) + rest)
    words = np.arange(1 << k, dtype=np.uint64)
    ex, amp = values(red, words)
    sv = SV.run(c)
    idx = words.astype(np.int64) | sum(b << (k + i) for i, b in enumerate(rest))
    assert np.max(np.abs(amp - sv[idx])) <= 1e-9
    # non-parametric path (every bit fixed, one reduction per assignment) gives
    # the same exact value, bit for bit
    for w in rng.choice(1 << k, min(4, 1 << k), replace=False):
        fixed = [int(w >> q) & 1 for q in range(k)] + rest
        exf, _ = values(CI.reduce_amplitudes(c, fixed), [0])
        want = ex[int(w)] if exf.size else np.zeros(5, np.int64)
        got = exf[0] if exf.size else np.zeros(5, np.int64)
        assert np.array_equal(got, want) or (not got[:4].any() and not want[:4].any())


@pytest.mark.parametrize("seed", range(12))
def test_all_amplitudes_and_parametric_inputs(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 8))
    c = CI.random_circuit(n, int(rng.integers(2, 14)), seed=seed)
    inb = int(rng.integers(0, 1 << n))
    red = CI.reduce_amplitudes(c, all_outputs(n), in_spec=[CI.param(n + q) for q in range(n)])
    words = np.arange(1 << n, dtype=np.uint64) | np.uint64(inb << n)
    _, amp = values(red, words)
    sv = SV.run(c, [(inb >> q) & 1 for q in range(n)])
    assert np.max(np.abs(amp - sv)) <= 1e-9


@pytest.mark.parametrize("seed", range(10))
def test_marginals_summing_doubling_statevector(seed):
    rng = np.random.default_rng(200 + seed)
    n = int(rng.integers(2, 6))
    c = CI.random_clifford_t(n, int(rng.integers(0, 9)), seed=300 + seed)
    k = int(rng.integers(1, n + 1))
    prob = np.abs(SV.run(c)) ** 2
    marg = np.array([prob[(np.arange(1 << n) % (1 << k)) == w].sum() for w in range(1 << k)])
    d = CI.reduce_doubled(c, [CI.param(q) if q < k else CI.TRACED for q in range(n)])
    _, dv = values(d, np.arange(1 << k, dtype=np.uint64))
    assert np.max(np.abs(dv.imag)) <= 1e-12
    assert np.max(np.abs(dv.real - marg)) <= 1e-9
    assert abs(dv.real.sum() - 1) <= 1e-9                      # completeness
    # summing: the low k outputs fixed per pattern, the other n - k summed
    s = CI.reduce_amplitudes(c, all_outputs(n))
    _, amp = values(s, np.arange(1 << n, dtype=np.uint64))
    summed = np.array([np.sum(np.abs(amp[(np.arange(1 << n) % (1 << k)) == w]) ** 2) for w in range(1 << k)])
    assert np.max(np.abs(summed - dv.real)) <= 1e-9


def test_bell_marginals():
    c = CI.Circuit(2).add("h", 0).add("cx", 0, 1)
    d = CI.reduce_doubled(c, [CI.param(0), CI.TRACED])
    assert np.allclose(values(d, [0, 1])[1], [0.5, 0.5])
    d2 = CI.reduce_doubled(c, [CI.param(0), CI.param(1)])
    assert np.allclose(values(d2, [0, 1, 2, 3])[1], [0.5, 0, 0, 0.5])


def test_term_count_bound_and_config_tables():
    # SPEC S:287 / acceptance #3: m <= 7^ceil(t/6) * 2^5 with t the T-count after
    # Clifford simplification (the T-pair decomposition gives <= 2^ceil(t/2))
    for seed in range(8):
        c = CI.random_circuit(8, 12 + 2 * seed, seed=seed)
        red = CI.reduce_amplitudes(c, all_outputs(8))
        t = red.t_after_simp
        assert red.expr.n_terms <= 7 ** -(-t // 6) * 2 ** 5
        assert red.expr.n_terms <= 2 ** -(-t // 2)
    # the C1 config table is a real reduction, checked amplitude by amplitude
    cfg = synth.CONFIGS["c1"]
    red = synth.circuit_reduction(cfg)
    assert red.t_count == 20 and red.expr.n_params == 8
    _, amp = values(red, np.arange(256, dtype=np.uint64))
    assert np.max(np.abs(amp - SV.run(synth.config_circuit(cfg)))) <= 1e-12


def test_reducer_validation():
    import paper_2403_06777_b200 as P
    with pytest.raises(P.Error):
        CI.reduce_amplitudes(CI.Circuit(2).add("cx", 0, 0), [0, 0])      # control == target
    with pytest.raises(ValueError):
        CI.reduce_amplitudes(CI.Circuit(2), [0])                          # spec length
    with pytest.raises(P.Error):
        CI.reduce_amplitudes(CI.Circuit(2), [0, CI.TRACED])               # traced needs doubled mode
