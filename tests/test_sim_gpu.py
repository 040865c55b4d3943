"""Sim-driver workflows end to end on the GPU: reducer ->
table -> B200 kernels, against the dense statevector and the non-parametric
path (acceptance #7 and #8 of SPEC S:615-616)."""
import numpy as np
import pytest

import statevector as SV
import paper_2403_06777_b200 as P
from paper_2403_06777_b200 import circuit as CI
from paper_2403_06777_b200 import sim

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = P.Context(0)
    yield c
    c.close()


def test_amplitudes_strong_and_nonparametric_agree(ctx):
    c = CI.random_circuit(10, 18, seed=3)
    amp, red, t = sim.amplitudes(ctx, c)
    sv = SV.run(c)
    assert np.max(np.abs(amp - sv)) <= 1e-12
    for w in (0, 5, 1023):
        assert abs(sim.strong_amplitude(c, [(w >> q) & 1 for q in range(10)]) - amp[w]) <= 1e-13
    t.free()


def test_marginals_summing_doubling_and_sampling(ctx):
    c = CI.random_clifford_t(6, 8, seed=11)
    prob = np.abs(SV.run(c)) ** 2
    # P(q1 = 1, q4 = 0) by summing and by doubling
    mask = ((np.arange(64) >> 1) & 1 == 1) & ((np.arange(64) >> 4) & 1 == 0)
    want = prob[mask].sum()
    assert abs(sim.marginal_summing(ctx, c, {1: 1, 4: 0}) - want) <= 1e-9
    pd = sim.marginal_doubling(ctx, c, [1, 4], [0b01])        # bit0 -> q1 = 1, bit1 -> q4 = 0
    assert abs(pd[0] - want) <= 1e-9
    # completeness over all patterns of 3 measured qubits
    allp = sim.marginal_doubling(ctx, c, [0, 2, 5], np.arange(8))
    assert abs(allp.sum() - 1) <= 1e-9
    # weak sampling: Bell pair -> 00 / 11 only, each ~1/2
    bell = CI.Circuit(2).add("h", 0).add("cx", 0, 1)
    s = sim.weak_sample(ctx, bell, 100000, seed=3)
    assert set(np.unique(s).tolist()) <= {0, 3}
    assert abs(np.mean(s == 0) - 0.5) <= 0.01


def test_speedup_benchmark_sigmoid(ctx):
    """SPEC acceptance #8 shape: S_N monotone over the schedule and the
    sigmoid fit; both paths return equal values."""
    c = CI.random_circuit(12, 30, seed=7)
    r = sim.speedup_benchmark(ctx, c, schedule=(1, 16, 256, 4096), baseline_seconds=3.0)
    assert r["max_abs_diff_param_vs_nonparam"] <= 1e-12
    assert r["monotone"]
    assert r["R2"] >= 0.9
    assert r["schedule"][-1]["S_N"] >= 10
