"""Dense statevector simulator -- TEST INFRASTRUCTURE (the reducer's oracle).

SPEC acceptance #1 and the sim-driver examples check the
parametric pipeline against a dense statevector; the reference declares such
an oracle (dense.hpp:29, dense_semantics) but never defines it, so this is a
plain numpy restatement of the gate set of SPEC Circuit. Only tests
and bench.py's baselines may import it.
"""
from __future__ import annotations

import numpy as np

_S2 = 1 / np.sqrt(2)
_W = np.exp(1j * np.pi / 4)
ONE_Q = {
    "h": np.array([[_S2, _S2], [_S2, -_S2]], np.complex128),
    "x": np.array([[0, 1], [1, 0]], np.complex128),
    "z": np.diag([1, -1]).astype(np.complex128),
    "s": np.diag([1, 1j]),
    "sdg": np.diag([1, -1j]),
    "t": np.diag([1, _W]),
    "tdg": np.diag([1, np.conj(_W)]),
}


def _apply1(psi, n, q, U):
    psi = psi.reshape((2,) * n)
    psi = np.moveaxis(np.tensordot(U, psi, axes=([1], [n - 1 - q])), 0, n - 1 - q)
    return psi.reshape(-1)


def apply_gate(psi, n, g):
    name = g[0]
    if name in ONE_Q:
        return _apply1(psi, n, g[1], ONE_Q[name])
    if name == "rz":
        return _apply1(psi, n, g[1], np.diag([1, _W ** (g[2] % 8)]))
    idx = np.arange(psi.size)
    if name in ("cx", "cnot"):
        c, t = g[1], g[2]
        src = np.where((idx >> c) & 1, idx ^ (1 << t), idx)
        return psi[src]
    if name == "cz":
        a, b = g[1], g[2]
        return psi * np.where(((idx >> a) & 1) & ((idx >> b) & 1), -1, 1)
    raise ValueError(name)


def run(circ, in_bits=None) -> np.ndarray:
    """U|in> as a vector indexed by the output bitstring (bit q = qubit q)."""
    n = circ.n_qubits
    psi = np.zeros(1 << n, np.complex128)
    b = 0 if in_bits is None else sum(int(v) << q for q, v in enumerate(in_bits))
    psi[b] = 1
    for g in circ.gates:
        psi = apply_gate(psi, n, g)
    return psi
