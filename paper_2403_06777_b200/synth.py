"""Seeded synthetic leaf-term lists for the BASELINE configs.

The reference ships no circuits and no reducer, so the term
tables are synthetic with the statistics SURVEY §8(d) fixes:

* raw subterm kinds PiPair 0.5 / HalfPi 0.2 / Node 0.2 / PhasePair 0.1;
* phase constants drawn inside each kind's invariant (subterm.cpp:5-21):
  HalfPi k in {2, 6}; PiPair phi.k in {0, 4}; "general" mix allows odd k
  (T-like) everywhere else, "clifford" mix only even k;
* every mask bit set i.i.d. with rho = 0.25 over the P parameters, a mask is
  never empty (an all-empty subterm would have been folded by push_subterm,
  diagram.cpp:114-120);
* n_t ~ U[n_lo, n_hi] subterms per term;
* C_t = RingQuad::make(U[-8, 8]^4, exp = n_t), never zero (C3-C5 cap exp at 40:
  the reference's ring_add throws when term exponents differ by > 62,
  ring.cpp:61-63, which long terms would otherwise hit);
* bit generator MT19937 seeded with 20261018 + config id.

Everything is plain numpy; the same arrays feed the GPU path and both CPU
baselines, so every arm sees identical inputs.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .pzx import ScalarExpression


@dataclass(frozen=True)
class Config:
    cid: int
    name: str
    n_params: int
    n_terms: int
    n_lo: int
    n_hi: int
    n_assign: int
    enumerated: bool
    prob_real: bool = False
    mix: str = "general"
    exp_cap: int | None = None  # cap on the scalar's 2^-exp: keeps the reference's int64 ring_add in range
    # (n_qubits, T-count, seed): the table is the host reducer's output for
    # circuit.random_circuit (every output bit a parameter) instead of a
    # synthetic term list; n_terms / n_lo / n_hi are then unused
    circuit: tuple | None = None


CONFIGS = {
    # C1 (BASELINE configs[0]): the real reduction of an 8-qubit, T-count-20
    # random circuit; all 2^8 amplitudes
    "c1": Config(1, "C1: 8-qubit T=20 random Clifford+T circuit, all 2^8 amplitudes via parametric reduction",
                 8, 0, 0, 0, 1 << 8, True, circuit=(8, 20, 20261018 + 1)),
    "c2": Config(2, "C2: P=20, all 2^20 amplitudes (20 qubits, T=40)", 20, 1 << 17, 16, 48, 1 << 20, True),
    # C2 on the real reduction of a 20-qubit, T-count-40 random circuit
    "c2r": Config(12, "C2r: 20-qubit T=40 random Clifford+T circuit, all 2^20 amplitudes via parametric reduction",
                  20, 0, 0, 0, 1 << 20, True, circuit=(20, 40, 20261018 + 2)),
    # the round-1 synthetic C1-shaped table (kept for the kernel tests)
    "c1s": Config(1, "C1s: P=8 synthetic 1024-term table, all 2^8 amplitudes", 8, 1 << 10, 8, 24, 1 << 8, True),
    "c3": Config(3, "C3: P=30, 2^24 sampled probabilities (30 qubits, T=60)", 30, 1 << 18, 24, 56, 1 << 24, False,
                 exp_cap=40),
    "c4": Config(4, "C4: P=10 doubled-diagram marginals, 2^10 params (term split)", 10, 1 << 22, 32, 64, 1 << 10,
                 True, prob_real=True, exp_cap=40),
    "c5": Config(5, "C5: P=32, T>=100 term-split table (> L2)", 32, 1 << 24, 32, 64, 1 << 16, False, exp_cap=40),
}

KIND_P = (0.2, 0.1, 0.2, 0.5)  # Node, PhasePair, HalfPi, PiPair  (SubtermKind order)


def _masks(rng: np.random.Generator, n: int, P: int) -> np.ndarray:
    full = np.uint64((1 << P) - 1) if P < 64 else np.uint64(2**64 - 1)
    m = (rng.integers(0, 2**64, n, dtype=np.uint64, endpoint=False)
         & rng.integers(0, 2**64, n, dtype=np.uint64, endpoint=False)) & full
    empty = m == 0
    if empty.any():
        m[empty] = np.left_shift(np.uint64(1), rng.integers(0, P, int(empty.sum())).astype(np.uint64))
    return m


def _canon_scalars(vals: np.ndarray, exps: np.ndarray) -> np.ndarray:
    """RingQuad::make canonical form (ring.cpp:20-48) on int64 rows."""
    v = vals.astype(np.int64).copy()
    e = exps.astype(np.int64).copy()
    while True:
        even = ((v[:, 0] | v[:, 1] | v[:, 2] | v[:, 3]) & 1) == 0
        sel = even & (e > 0)
        if not sel.any():
            break
        v[sel] //= 2
        e[sel] -= 1
    return np.concatenate([v, e[:, None]], axis=1)


def generate(n_params: int, n_terms: int, n_lo: int, n_hi: int, seed: int, mix: str = "general",
             kind_p=KIND_P, exp_cap: int | None = None) -> ScalarExpression:
    rng = np.random.Generator(np.random.MT19937(seed))
    P = n_params
    n = rng.integers(n_lo, n_hi + 1, n_terms)
    off = np.zeros(n_terms + 1, np.uint64)
    np.cumsum(n, out=off[1:])
    S = int(off[-1])
    kind = rng.choice(4, size=S, p=kind_p).astype(np.uint8)
    psi_k = rng.integers(0, 8, S).astype(np.uint8)
    phi_k = rng.integers(0, 8, S).astype(np.uint8)
    if mix == "clifford":
        psi_k &= np.uint8(6)
        phi_k &= np.uint8(6)
    half = kind == 2
    psi_k[half] = np.where(rng.integers(0, 2, int(half.sum())) == 0, 2, 6).astype(np.uint8)
    pip = kind == 3
    phi_k[pip] = np.where(rng.integers(0, 2, int(pip.sum())) == 0, 0, 4).astype(np.uint8)
    single = (kind == 0) | half
    phi_k[single] = 0
    psi_mask = _masks(rng, S, P)
    phi_mask = _masks(rng, S, P)
    phi_mask[single] = 0
    vals = rng.integers(-8, 9, (n_terms, 4))
    zero = ~vals.any(axis=1)
    while zero.any():
        vals[zero] = rng.integers(-8, 9, (int(zero.sum()), 4))
        zero = ~vals.any(axis=1)
    scal = _canon_scalars(vals, n if exp_cap is None else np.minimum(n, exp_cap))
    return ScalarExpression(P, off, scal, kind, psi_k, psi_mask, phi_k, phi_mask)


CHUNK_TERMS = 1 << 20   # configs above this are generated as independently seeded term chunks


def n_chunks(cfg: Config, n_terms: int | None = None) -> int:
    n = cfg.n_terms if n_terms is None else n_terms
    return max(1, -(-n // CHUNK_TERMS))


def concat(parts: list[ScalarExpression]) -> ScalarExpression:
    """Term lists back to back (offsets rebased)."""
    if len(parts) == 1:
        return parts[0]
    offs, base = [np.zeros(1, np.uint64)], np.uint64(0)
    for e in parts:
        offs.append(e.term_offset[1:] + base)
        base += e.term_offset[-1]
    cat = lambda name: np.concatenate([getattr(e, name) for e in parts])  # noqa: E731
    return ScalarExpression(parts[0].n_params, np.concatenate(offs), np.concatenate([e.term_scalar for e in parts]),
                            cat("kind"), cat("psi_k"), cat("psi_mask"), cat("phi_k"), cat("phi_mask"))


def generate_config(cfg: Config, n_terms: int | None = None, chunks: range | None = None,
                    workers: int | None = None) -> ScalarExpression:
    """The config's term list. Above CHUNK_TERMS terms it is the concatenation of
    chunks seeded (seed, chunk index), so a term-split rank can generate just its
    own chunks (`chunks`) and big tables generate on several threads. Circuit
    configs run the host reducer (circuit.py) on their random circuit."""
    if cfg.circuit is not None:
        return circuit_reduction(cfg).expr
    n = cfg.n_terms if n_terms is None else n_terms
    seed = 20261018 + cfg.cid
    if n <= CHUNK_TERMS and chunks is None:
        return generate(cfg.n_params, n, cfg.n_lo, cfg.n_hi, seed, cfg.mix, exp_cap=cfg.exp_cap)
    nc = n_chunks(cfg, n)
    chunks = range(nc) if chunks is None else chunks

    def one(c):
        m = min(CHUNK_TERMS, n - c * CHUNK_TERMS)
        return generate(cfg.n_params, m, cfg.n_lo, cfg.n_hi, seed * 4099 + c, cfg.mix, exp_cap=cfg.exp_cap)
    import concurrent.futures as cf
    import os
    with cf.ThreadPoolExecutor(workers or min(len(chunks), os.cpu_count() or 1, 32)) as ex:
        parts = list(ex.map(one, chunks))
    return concat(parts)


def config_circuit(cfg: Config):
    from .circuit import random_circuit
    n, t, seed = cfg.circuit
    return random_circuit(n, t, seed)


_REDUCTIONS: dict = {}


def circuit_reduction(cfg: Config):
    """The parametric reduction of a circuit config (cached per process): every
    output bit q is parameter q, so the table yields all 2^n amplitudes."""
    from .circuit import param, reduce_amplitudes
    if cfg.name not in _REDUCTIONS:
        c = config_circuit(cfg)
        _REDUCTIONS[cfg.name] = reduce_amplitudes(c, [param(q) for q in range(c.n_qubits)])
    return _REDUCTIONS[cfg.name]


def term_row_offsets(cfg: Config) -> np.ndarray:
    """Subterm offsets [m + 1] of the whole config table without generating it:
    the term sizes are the first draw of every (chunk) generator, so this is
    cheap even for C5's 2^24 terms. Used to cut row-balanced term ranges
    (dist.term_ranges) for the term split before any rank builds its table."""
    if cfg.circuit is not None:
        return np.asarray(generate_config(cfg).term_offset, np.uint64) - np.uint64(0)
    seed = 20261018 + cfg.cid
    n = cfg.n_terms
    if n <= CHUNK_TERMS:
        sizes = [np.random.Generator(np.random.MT19937(seed)).integers(cfg.n_lo, cfg.n_hi + 1, n)]
    else:
        sizes = [np.random.Generator(np.random.MT19937(seed * 4099 + c)).integers(
                     cfg.n_lo, cfg.n_hi + 1, min(CHUNK_TERMS, n - c * CHUNK_TERMS)) for c in range(n_chunks(cfg))]
    off = np.zeros(n + 1, np.uint64)
    np.cumsum(np.concatenate(sizes), out=off[1:])
    return off


def generate_config_terms(cfg: Config, t0: int, t1: int) -> ScalarExpression:
    """Terms [t0, t1) of the config table (only the chunks that overlap the
    range are generated), rebased so the slice starts at subterm 0."""
    if cfg.circuit is not None or cfg.n_terms <= CHUNK_TERMS:
        full = generate_config(cfg)
        c0 = 0
    else:
        c0, c1 = t0 // CHUNK_TERMS, max(t0, t1 - 1) // CHUNK_TERMS + 1
        full = generate_config(cfg, chunks=range(c0, c1))
        c0 *= CHUNK_TERMS
    a, b = t0 - c0, t1 - c0
    off = full.term_offset
    s0, s1 = int(off[a]), int(off[b])
    return ScalarExpression(full.n_params, off[a:b + 1] - np.uint64(s0), full.term_scalar[a:b],
                            full.kind[s0:s1], full.psi_k[s0:s1], full.psi_mask[s0:s1], full.phi_k[s0:s1],
                            full.phi_mask[s0:s1])


def assignments(cfg: Config, n: int | None = None, seed_offset: int = 0) -> np.ndarray:
    """The config's assignment batch: enumerated 0..N-1 or seeded uniform P-bit words."""
    N = cfg.n_assign if n is None else n
    if cfg.enumerated:
        return np.arange(N, dtype=np.uint64)
    rng = np.random.Generator(np.random.MT19937(20261018 + 100 * cfg.cid + seed_offset))
    full = (1 << cfg.n_params) - 1 if cfg.n_params < 64 else 2**64 - 1
    return rng.integers(0, 2**64, N, dtype=np.uint64) & np.uint64(full)
