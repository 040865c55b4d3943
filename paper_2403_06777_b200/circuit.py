"""Clifford+T circuits and the host parametric reducer.

``Circuit`` is the SPEC's circuit type (H, X, Z, S, S^dag, T, T^dag,
CNOT, CZ, RZ(k pi/4)). ``reduce_amplitudes`` / ``reduce_doubled`` run the
native reducer (``pzx_circuit_reduce``, csrc/pzx_reduce.cpp): circuit ->
closed polar-parameterised ZX diagram -> Clifford simplification ->
stabiliser decomposition -> the leaf-term ``ScalarExpression`` that
``Context.compile_bit_table`` uploads. Output bits (or inputs) given as
``param(p)`` become boolean parameters, so ONE reduction yields every
amplitude <a|U|in> (SPEC strong_amplitude / marginal_summing) or
every doubled marginal P(a) (marginal_doubling).

``random_clifford_t`` draws the synthetic random Clifford+T circuits of the
BASELINE configs (seeded, exact T-count).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .pzx import ScalarExpression, _check

OPS = {"h": 0, "x": 1, "z": 2, "s": 3, "sdg": 4, "t": 5, "tdg": 6, "cx": 7, "cnot": 7, "cz": 8, "rz": 9}
AMPLITUDE, DOUBLED = 0, 1
TRACED = -1


def param(p: int) -> int:
    """out_spec / in_spec entry: parameter p (bit p of the assignment word)."""
    return 2 + p


@dataclass
class Circuit:
    n_qubits: int
    gates: list = field(default_factory=list)  # (name, q0[, q1]) or ("rz", q, k)

    def add(self, name: str, *qs) -> "Circuit":
        self.gates.append((name.lower(),) + tuple(int(q) for q in qs))
        return self

    def t_count(self) -> int:
        return sum(1 for g in self.gates if g[0] in ("t", "tdg") or (g[0] == "rz" and g[2] % 2))

    def encoded(self) -> np.ndarray:
        a = np.zeros((max(len(self.gates), 1), 4), np.uint8)
        for i, g in enumerate(self.gates):
            op = OPS[g[0]]
            a[i, 0] = op
            a[i, 1] = g[1]
            if op in (7, 8):
                a[i, 2] = g[2]
            if op == 9:
                a[i, 3] = g[2] % 8
        return a


class Reduction:
    """The reducer's output: the leaf-term expression plus its statistics."""

    def __init__(self, expr: ScalarExpression, t_count: int, t_after_simp: int, seconds: float):
        self.expr, self.t_count, self.t_after_simp, self.seconds = expr, t_count, t_after_simp, seconds


def _reduce(circ: Circuit, out_spec, in_spec, mode: int, max_terms: int) -> Reduction:
    n = circ.n_qubits
    gates = circ.encoded()
    outs = np.ascontiguousarray(np.asarray(out_spec, np.int32))
    ins = None if in_spec is None else np.ascontiguousarray(np.asarray(in_spec, np.int32))
    if outs.size != n or (ins is not None and ins.size != n):
        raise ValueError("bit specs must have one entry per qubit")
    L = N.lib()
    h = C.c_void_p()
    _check(L.pzx_circuit_reduce(n, gates.ctypes.data_as(C.c_void_p), len(circ.gates), N.ptr(ins, C.c_int32),
                                N.ptr(outs, C.c_int32), mode, max_terms, C.byref(h)))
    try:
        v = N.ExprView()
        _check(L.pzx_expr_get_view(h, C.byref(v)))
        m = int(v.n_terms)
        off = np.ctypeslib.as_array(v.term_offset, (m + 1,)).copy()
        S = int(off[-1])
        scal = (np.ctypeslib.as_array(v.term_scalar, (5 * m,)).reshape(m, 5).copy() if m
                else np.zeros((0, 5), np.int64))

        def arr(p, dt):
            return np.ctypeslib.as_array(p, (max(S, 1),))[:S].astype(dt) if S else np.zeros(0, dt)
        expr = ScalarExpression(int(v.n_params), off, scal, arr(v.kind, np.uint8), arr(v.psi_k, np.uint8),
                                arr(v.psi_mask, np.uint64), arr(v.phi_k, np.uint8), arr(v.phi_mask, np.uint64))
        t, ta, sec = C.c_uint32(), C.c_uint32(), C.c_double()
        _check(L.pzx_expr_info(h, C.byref(t), C.byref(ta), C.byref(sec)))
        return Reduction(expr, t.value, ta.value, sec.value)
    finally:
        L.pzx_expr_free(h)


def reduce_amplitudes(circ: Circuit, out_spec, in_spec=None, max_terms: int = 0) -> Reduction:
    """<out|U|in> as a parametric expression (parameters where the spec says param(p))."""
    return _reduce(circ, out_spec, in_spec, AMPLITUDE, max_terms)


def reduce_doubled(circ: Circuit, meas_spec, in_spec=None, max_terms: int = 0) -> Reduction:
    """P(measured qubits = a) = <in|U^dag (|a><a| (x) I) U|in>; meas_spec: 0/1,
    param(p), or TRACED per qubit. Evaluate with Re output (PZX_PROB_REAL)."""
    return _reduce(circ, meas_spec, in_spec, DOUBLED, max_terms)


def random_circuit(n_qubits: int, t_count: int, seed: int, p_cnot: float = 0.5, p_h: float = 0.3,
                   p_s: float = 0.1) -> Circuit:
    """The BASELINE configs' "random Clifford+T circuit, n qubits, T-count t":
    H on every qubit, then gates drawn i.i.d. (CNOT on a random pair with
    p_cnot, H with p_h, S with p_s, else T / T^dag) until exactly t T-gates,
    then H on every qubit. MT19937(seed). CNOT-heavy, so the Clifford
    simplification removes only ~15-25 % of the T-count (pzx_expr_info)."""
    rng = np.random.Generator(np.random.MT19937(seed))
    c = Circuit(n_qubits)
    for q in range(n_qubits):
        c.add("h", q)
    nt = 0
    while nt < t_count:
        r = rng.random()
        if r < p_cnot and n_qubits > 1:
            a, b = rng.choice(n_qubits, 2, replace=False)
            c.add("cx", int(a), int(b))
        elif r < p_cnot + p_h:
            c.add("h", int(rng.integers(n_qubits)))
        elif r < p_cnot + p_h + p_s:
            c.add("s", int(rng.integers(n_qubits)))
        elif r >= p_cnot + p_h + p_s:
            c.add("t" if rng.random() < 0.5 else "tdg", int(rng.integers(n_qubits)))
            nt += 1
    for q in range(n_qubits):
        c.add("h", q)
    return c


def random_clifford_t(n_qubits: int, t_count: int, n_clifford: int | None = None, seed: int = 0,
                      two_qubit_frac: float = 0.35) -> Circuit:
    """Seeded random Clifford+T circuit with exactly `t_count` T / T^dag gates
    interleaved with ~n_clifford random Clifford gates (H, S, S^dag, X, Z,
    CNOT, CZ); an H layer first so the T gates act on superpositions."""
    rng = np.random.Generator(np.random.MT19937(seed))
    n_c = 4 * t_count + 2 * n_qubits if n_clifford is None else n_clifford
    c = Circuit(n_qubits)
    for q in range(n_qubits):
        c.add("h", q)
    slots = np.sort(rng.choice(n_c + t_count, t_count, replace=False)) if t_count else np.zeros(0, int)
    ts = set(int(x) for x in slots)
    for i in range(n_c + t_count):
        if i in ts:
            c.add("t" if rng.random() < 0.5 else "tdg", int(rng.integers(n_qubits)))
        elif n_qubits > 1 and rng.random() < two_qubit_frac:
            a, b = rng.choice(n_qubits, 2, replace=False)
            c.add("cx" if rng.random() < 0.6 else "cz", int(a), int(b))
        else:
            c.add(["h", "s", "sdg", "x", "z", "h"][int(rng.integers(6))], int(rng.integers(n_qubits)))
    return c
