"""Generate the golden fixtures under tests/golden/ from the REFERENCE ITSELF.

Run here (where /root/reference exists and oracle/_ref/libpzx_ref.so was built
from it by oracle/Makefile):

    python tests/golden/make_golden.py

Every number in the fixtures is produced by the reference's own functions
(phase_pair_value, normalize_subterm, subterm_value, instantiate_phase,
instantiate_diagram / ring_mul / ring_add, to_complex) through the C shim
oracle/ref_shim.cpp. The fixtures travel with the repo so the oracle
restatement and the GPU path are checked against the reference on machines
without /root/reference.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle_py as O  # noqa: E402
from paper_2403_06777_b200 import synth  # noqa: E402  (seeded input generator only)

# (name, n_params, n_terms, n_lo, n_hi, seed, mix, n_assign, enumerated[, kind_p])
LONG_P = (0.02, 0.03, 0.35, 0.6)  # few Node rows: long terms that do not vanish / overflow
EXPRS = [
    ("p8_general", 8, 96, 8, 24, 11, "general", 256, True),
    ("p8_clifford", 8, 64, 8, 24, 12, "clifford", 256, True),
    ("p20_general", 20, 128, 16, 48, 13, "general", 96, False),
    ("p30_long", 30, 24, 100, 140, 14, "clifford", 48, False, LONG_P, 24),
    ("p40_general", 40, 64, 8, 32, 15, "general", 64, False),
    ("p64_general", 64, 48, 8, 32, 16, "general", 64, False),
]


def pair_table():
    return [[list(O.pair_value(a, b, impl="ref")) for b in range(8)] for a in range(8)]


def normalize_exhaustive():
    """kind x psi.k x phi.k x masks in {{}, {p0}, {p1}, {p0,p1}}^2, 2 parameters."""
    recs = []
    for kind in range(4):
        for pk in range(8):
            for fk in range(8):
                for pm in range(4):
                    for fm in range(4):
                        if kind in (0, 2) and (fk or fm):
                            continue  # phi unused for Node / HalfPi
                        rec = {"s": [kind, pk, pm, fk, fm]}
                        try:
                            c, pair = O.normalize(kind, pk, pm, fk, fm, impl="ref")
                            rec["norm"] = [list(c), list(pair) if pair else None]
                        except O.OracleError as e:
                            rec["norm_err"] = e.status
                        vals = []
                        for word in range(4):
                            try:
                                vals.append(list(O.subterm_value(kind, pk, pm, fk, fm, word, 2, impl="ref")))
                            except O.OracleError as e:
                                vals.append(-e.status)
                        rec["val"] = vals
                        recs.append(rec)
    return recs


def ring_kats():
    rng = np.random.default_rng(5)
    out = []
    for _ in range(400):
        x = O.make(*[int(v) for v in rng.integers(-50, 51, 4)], int(rng.integers(0, 6)), impl="ref")
        y = O.make(*[int(v) for v in rng.integers(-50, 51, 4)], int(rng.integers(0, 6)), impl="ref")
        out.append({"x": list(x), "y": list(y), "add": list(O.ring_add(x, y, impl="ref")),
                    "mul": list(O.ring_mul(x, y, impl="ref")), "cx": [O.to_complex(x, impl="ref").real,
                                                                      O.to_complex(x, impl="ref").imag]})
    return out


def phase_kats():
    rng = np.random.default_rng(6)
    out = []
    for _ in range(300):
        P = int(rng.integers(1, 65))
        full = (1 << P) - 1
        k = int(rng.integers(0, 8))
        mask = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2)) & full
        word = int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2))
        out.append([k, mask, word, P, O.instantiate_phase(k, mask, word, P, impl="ref")])
    return out


def main():
    O.build()
    assert O.have_ref(), "oracle/_ref/libpzx_ref.so missing (needs /root/reference)"
    with open(os.path.join(HERE, "kats.json"), "w") as f:
        json.dump({"pair_table": pair_table(), "normalize": normalize_exhaustive(), "ring": ring_kats(),
                   "instantiate_phase": phase_kats()}, f, separators=(",", ":"))
    for name, P, m, lo, hi, seed, mix, n, enum, *kp in EXPRS:
        e = synth.generate(P, m, lo, hi, seed, mix, *kp)
        if enum:
            words = np.arange(n, dtype=np.uint64)
        else:
            rng = np.random.default_rng(seed)
            words = rng.integers(0, 2**64, n, dtype=np.uint64)  # includes bits >= P (must be ignored)
        ex0, amp0 = O.eval_batch(e, words, 8, impl="ref", mode=0)
        ex1, amp1 = O.eval_batch(e, words, 8, impl="ref", mode=1)
        assert (ex0 == ex1).all() and np.array_equal(amp0, amp1)
        np.savez_compressed(os.path.join(HERE, f"expr_{name}.npz"), n_params=P, seed=seed, term_offset=e.term_offset,
                            term_scalar=e.term_scalar, kind=e.kind, psi_k=e.psi_k, psi_mask=e.psi_mask,
                            phi_k=e.phi_k, phi_mask=e.phi_mask, words=words, exact=ex0, amp=amp0)
        print(name, "terms", m, "subterms", int(e.term_offset[-1]), "max|amp|", float(np.abs(amp0).max()))


if __name__ == "__main__":
    main()
