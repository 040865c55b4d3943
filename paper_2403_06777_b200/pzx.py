"""Host-side mirror of the reference's evaluate-on-assignments interface.

Names, argument meanings and error classes follow the reference
(/root/reference/proj/core/include/pzx/*.hpp and SPEC.md):

=====================  =====================================================
this module            reference
=====================  =====================================================
``Error`` ...          ``pzx::Error`` hierarchy, common.hpp:13-48
``kMaxParams``         common.hpp:11
``ParamAssignment``    phase.hpp:14-29 (``total``: bits >= n are dropped)
``ParamPhase``         phase.hpp:34-52 (k mod 8 + XOR mask)
``SubtermKind``        subterm.hpp:19
``Subterm``            subterm.hpp:21-36 (``half_pi``/``pi_pair`` validate
                       and orient exactly like subterm.cpp:5-21)
``RingQuad``           ring.hpp:17-38 (exact; canonical form ring.cpp:20-48)
``ScalarExpression``   SPEC ScalarExpression as a leaf-term list
                       (scalar_ + pending_ of ZXDiagram, diagram.hpp:70-77)
``compile_bit_table``  SPEC compile_bit_table + upload
``Context.evaluate_batch``  SPEC evaluate_batch
``Context.evaluate``   SPEC evaluate
=====================  =====================================================

Amplitudes come back as complex128 (the value the reference's ``to_complex``
produces from its exact RingQuad, ring.cpp:131-136). All evaluation runs in
the sm_100a kernels of ``libpzx_gpu.so``; nothing here computes amplitudes.
"""
from __future__ import annotations

import builtins
import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import _native as N

kMaxParams = 64


# ---------------------------------------------------------------- errors ----
class Error(RuntimeError):
    """pzx::Error (common.hpp:14-17)."""


class ParseError(Error):
    """pzx::ParseError (common.hpp:20-23)."""


class DomainError(Error):
    """pzx::DomainError (common.hpp:26-29)."""


class Lemma1Violation(DomainError):
    """pzx::Lemma1Violation (common.hpp:33-36)."""


class OverflowError(Error):  # noqa: A001 -- the reference's name (common.hpp:39-42)
    """pzx::OverflowError: exact arithmetic left its range."""


class MissingParameter(DomainError):
    """pzx::MissingParameter (common.hpp:45-48)."""


class CudaError(Error):
    """Device-side failure (no reference analogue)."""


_STATUS = {1: ParseError, 2: DomainError, 3: MissingParameter, 4: OverflowError,
           5: Error, 6: DomainError, 10: CudaError, 11: CudaError, 12: CudaError}


def _check(st: int, ctx=None) -> None:
    if st == 0:
        return
    lib = N.lib()
    msg = lib.pzx_status_string(st).decode()
    if ctx is not None:
        detail = lib.pzx_last_error(ctx).decode()
        if detail:
            msg = f"{msg}: {detail}"
    raise _STATUS.get(st, Error)(msg)


# ------------------------------------------------------- phases, subterms ----
@dataclass(frozen=True)
class ParamAssignment:
    """Total assignment (phase.hpp:14-29)."""

    bits: int = 0
    defined: int = 0

    @staticmethod
    def total(bits: int, n_params: int) -> "ParamAssignment":
        if n_params >= 64:
            return ParamAssignment(bits & (2**64 - 1), 2**64 - 1)
        m = (1 << n_params) - 1
        return ParamAssignment(bits & m, m)

    def covers(self, mask: int) -> bool:
        return (mask & ~self.defined) == 0


@dataclass(frozen=True)
class ParamPhase:
    """k*pi/4 + pi * XOR(params in mask) (phase.hpp:34-52)."""

    k: int = 0
    mask: int = 0

    def __post_init__(self):
        object.__setattr__(self, "k", self.k % 8)

    def parametric(self) -> bool:
        return self.mask != 0

    def pauli_image(self) -> bool:
        return self.k in (0, 4)

    def proper_clifford_image(self) -> bool:
        return self.k in (2, 6)


def phase_add(a: ParamPhase, b: ParamPhase) -> ParamPhase:
    """phase.hpp:55-60."""
    return ParamPhase((a.k + b.k) & 7, a.mask ^ b.mask)


class SubtermKind(enum.IntEnum):
    Node = 0
    PhasePair = 1
    HalfPi = 2
    PiPair = 3


@dataclass(frozen=True)
class Subterm:
    kind: SubtermKind
    psi: ParamPhase
    phi: ParamPhase = ParamPhase()

    @staticmethod
    def node(psi: ParamPhase) -> "Subterm":
        return Subterm(SubtermKind.Node, psi)

    @staticmethod
    def phase_pair(psi: ParamPhase, phi: ParamPhase) -> "Subterm":
        return Subterm(SubtermKind.PhasePair, psi, phi)

    @staticmethod
    def half_pi(psi: ParamPhase) -> "Subterm":
        if not psi.proper_clifford_image():  # subterm.cpp:5-10
            raise DomainError("half-pi subterm needs Image(psi) in {pi/2, 3pi/2}")
        return Subterm(SubtermKind.HalfPi, psi)

    @staticmethod
    def pi_pair(psi: ParamPhase, phi: ParamPhase) -> "Subterm":
        if phi.pauli_image():  # subterm.cpp:12-21
            return Subterm(SubtermKind.PiPair, psi, phi)
        if psi.pauli_image():
            return Subterm(SubtermKind.PiPair, phi, psi)
        raise DomainError("pi-pair subterm needs a phase with image in {0, pi}")

    def param_mask(self) -> int:
        return self.psi.mask | self.phi.mask


# -------------------------------------------------------------- RingQuad ----
@dataclass(frozen=True)
class RingQuad:
    """(a + b*sqrt2 + i(c + d*sqrt2)) / 2^exp, canonical (ring.cpp:20-48)."""

    a: int = 0
    b: int = 0
    c: int = 0
    d: int = 0
    exp: int = 0

    @staticmethod
    def make(a: int, b: int, c: int, d: int, exp: int) -> "RingQuad":
        while exp < 0:
            a, b, c, d, exp = 2 * a, 2 * b, 2 * c, 2 * d, exp + 1
        if a == b == c == d == 0:
            return RingQuad()
        while exp > 0 and not ((a | b | c | d) & 1):
            a, b, c, d, exp = a >> 1, b >> 1, c >> 1, d >> 1, exp - 1
        for v in (a, b, c, d):
            if not (-(2**63) <= v < 2**63):
                raise OverflowError("ring coefficient out of 64-bit range")
        return RingQuad(a, b, c, d, exp)

    @staticmethod
    def one() -> "RingQuad":
        return RingQuad(1, 0, 0, 0, 0)

    def __mul__(self, o: "RingQuad") -> "RingQuad":
        x, y = self, o
        return RingQuad.make(x.a * y.a + 2 * x.b * y.b - x.c * y.c - 2 * x.d * y.d,
                             x.a * y.b + x.b * y.a - x.c * y.d - x.d * y.c,
                             x.a * y.c + 2 * x.b * y.d + x.c * y.a + 2 * x.d * y.b,
                             x.a * y.d + x.b * y.c + x.c * y.b + x.d * y.a, x.exp + y.exp)

    def __add__(self, o: "RingQuad") -> "RingQuad":
        e = max(self.exp, o.exp)
        sx, sy = e - self.exp, e - o.exp
        return RingQuad.make(self.a * 2**sx + o.a * 2**sy, self.b * 2**sx + o.b * 2**sy,
                             self.c * 2**sx + o.c * 2**sy, self.d * 2**sx + o.d * 2**sy, e)

    def to_complex(self) -> complex:
        s2 = 2.0 ** 0.5
        sc = 2.0 ** -self.exp
        return complex((float(self.a) + float(self.b) * s2) * sc, (float(self.c) + float(self.d) * s2) * sc)

    def as_tuple(self) -> tuple:
        return (self.a, self.b, self.c, self.d, self.exp)


# ------------------------------------------------------ ScalarExpression ----
@dataclass
class ScalarExpression:
    """Leaf-term list: value(a) = sum_t C_t * prod_j subterm_value(S_tj, a).

    Stored structure-of-arrays (numpy) so that million-term synthetic tables
    and small hand-written ones share one path to the C ABI.
    """

    n_params: int
    term_offset: np.ndarray = field(default_factory=lambda: np.zeros(1, np.uint64))
    term_scalar: np.ndarray = field(default_factory=lambda: np.zeros((0, 5), np.int64))
    kind: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    psi_k: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    psi_mask: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    phi_k: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    phi_mask: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))

    @staticmethod
    def from_terms(n_params: int, terms: Iterable[tuple[RingQuad, Sequence[Subterm]]]) -> "ScalarExpression":
        if n_params > kMaxParams:
            raise DomainError("parameter capacity (64) exceeded")
        off, sc, kd, pk, pm, fk, fm = [0], [], [], [], [], [], []
        for c, subs in terms:
            sc.append(c.as_tuple())
            for s in subs:
                kd.append(int(s.kind)); pk.append(s.psi.k); pm.append(s.psi.mask)
                fk.append(s.phi.k); fm.append(s.phi.mask)
            off.append(len(kd))
        return ScalarExpression(
            n_params, np.asarray(off, np.uint64), np.asarray(sc, np.int64).reshape(-1, 5),
            np.asarray(kd, np.uint8), np.asarray(pk, np.uint8), np.asarray(pm, np.uint64),
            np.asarray(fk, np.uint8), np.asarray(fm, np.uint64))

    @property
    def n_terms(self) -> int:
        return len(self.term_offset) - 1

    @property
    def n_subterms(self) -> int:
        return int(self.term_offset[-1]) if len(self.term_offset) else 0

    def terms(self):
        """Iterate (RingQuad, [Subterm]) -- for small expressions / tests."""
        for t in range(self.n_terms):
            subs = []
            for j in range(int(self.term_offset[t]), int(self.term_offset[t + 1])):
                subs.append(Subterm(SubtermKind(int(self.kind[j])),
                                    ParamPhase(int(self.psi_k[j]), int(self.psi_mask[j])),
                                    ParamPhase(int(self.phi_k[j]), int(self.phi_mask[j]))))
            yield RingQuad(*map(int, self.term_scalar[t])), subs

    def slice_terms(self, t0: int, t1: int) -> "ScalarExpression":
        """Contiguous term range (absolute subterm indices are kept)."""
        return ScalarExpression(self.n_params, self.term_offset[t0:t1 + 1], self.term_scalar[t0:t1],
                                self.kind, self.psi_k, self.psi_mask, self.phi_k, self.phi_mask)

    def _arrays(self):
        a = [np.ascontiguousarray(self.term_offset, np.uint64),
             np.ascontiguousarray(self.term_scalar, np.int64).reshape(-1),
             np.ascontiguousarray(self.kind, np.uint8), np.ascontiguousarray(self.psi_k, np.uint8),
             np.ascontiguousarray(self.psi_mask, np.uint64), np.ascontiguousarray(self.phi_k, np.uint8),
             np.ascontiguousarray(self.phi_mask, np.uint64)]
        return [x if x.size else np.zeros(1, x.dtype) for x in a]

    def view(self):
        arrs = self._arrays()
        v = N.ExprView(self.n_params, self.n_terms, N.ptr(arrs[0], C.c_uint64), N.ptr(arrs[1], C.c_int64),
                       N.ptr(arrs[2], C.c_uint8), N.ptr(arrs[3], C.c_uint8), N.ptr(arrs[4], C.c_uint64),
                       N.ptr(arrs[5], C.c_uint8), N.ptr(arrs[6], C.c_uint64))
        return v, arrs  # keep arrays alive while the view is used


# ---------------------------------------------------------------- device ----
PROB_ABS2 = 1
PROB_REAL = 2
KERNEL_GENERAL = 1 << 8
KERNEL_GRAY = 1 << 9
KERNEL_SLICE = 1 << 10
KERNEL_SLICE_RAND = 1 << 11
ACCUMULATE = 1 << 2
KERNEL_SORTED = 1 << 12
KERNEL_SLICE2 = 1 << 13
KERNEL_PAGE = 1 << 14


class DeviceTable:
    """Device-resident compiled table (immutable; SPEC BitTable S:336-339)."""

    def __init__(self, ctx: "Context", handle: C.c_void_p):
        self._ctx = ctx
        self.handle = handle
        L = N.lib()
        p, m, r, mx = C.c_uint32(), C.c_uint64(), C.c_uint64(), C.c_uint32()
        _check(L.pzx_table_shape(handle, C.byref(p), C.byref(m), C.byref(r), C.byref(mx)))
        self.n_params, self.n_terms, self.n_rows, self.max_term_rows = p.value, m.value, r.value, mx.value

    def term_info(self, t: int):
        coef = np.zeros(5, np.int64)
        e, lm = C.c_int32(), C.c_int32()
        _check(N.lib().pzx_table_term_info(self.handle, t, N.ptr(coef, C.c_int64), C.byref(e), C.byref(lm)))
        return RingQuad(*map(int, coef)), e.value, lm.value

    def slice_stats(self):
        """(op_rows[129], term_kinds[3]): rows per bit-sliced op and terms per
        epilogue kind (kind-free, lambda-only, with pi) -- the work counts behind
        the algorithmic roofline (roofline.py)."""
        ops = np.zeros(129, np.uint64)
        kinds = np.zeros(3, np.uint64)
        _check(N.lib().pzx_table_slice_stats(self.handle, N.ptr(ops, C.c_uint64), N.ptr(kinds, C.c_uint64)))
        return ops, kinds

    def page_stats(self):
        """(family_rows [C, G, D, dropped, L, then G by class S2, S6, E0, E2, G1, G3],
        dispatch rows per op [129]) of the page layout, or None when the table
        has none (pzx_table_page_stats)."""
        fam = np.zeros(11, np.uint64)
        ops = np.zeros(129, np.uint64)
        st = N.lib().pzx_table_page_stats(self.handle, N.ptr(fam, C.c_uint64), N.ptr(ops, C.c_uint64))
        if st == 6:
            return None
        _check(st)
        return fam, ops

    def free(self) -> None:
        if self.handle:
            N.lib().pzx_table_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Context:
    """One device, one stream (pzx_ctx). Not thread-safe."""

    def __init__(self, device: int = 0):
        L = N.lib()
        h = C.c_void_p()
        _check(L.pzx_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    def close(self) -> None:
        if self.handle:
            N.lib().pzx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def launch_count(self) -> int:
        return int(N.lib().pzx_launch_count(self.handle))

    KERNEL_NAMES = {1: "popc", 2: "gray", 3: "slice", 4: "slice_rand", 5: "sorted", 6: "slice2", 7: "slice_wc", 8: "page"}

    def last_kernel(self) -> dict:
        """The evaluation kernel the last evaluate* call chose (pzx_last_kernel)."""
        k, g, c = C.c_int32(), C.c_int32(), C.c_int32()
        _check(N.lib().pzx_last_kernel(self.handle, C.byref(k), C.byref(g), C.byref(c)), self.handle)
        return {"kernel": self.KERNEL_NAMES.get(k.value, str(k.value)), "sorted_groups": g.value,
                "term_chunks": c.value}

    # -- compile + upload ---------------------------------------------------
    def compile_bit_table(self, expr: ScalarExpression, simplify: bool = False) -> DeviceTable:
        """SPEC compile_bit_table; simplify=True folds assignment-independent row
        groups (pairwise node cancellation, PZX_COMPILE_SIMPLIFY)."""
        v, keep = expr.view()
        h = C.c_void_p()
        _check(N.lib().pzx_table_upload_expr_ex(self.handle, C.byref(v), 1 if simplify else 0, C.byref(h)),
               self.handle)
        del keep
        return DeviceTable(self, h)

    def upload_rows(self, n_params, term_row_offset, term_coef, psi_mask, phi_mask, k_alpha, k_beta) -> DeviceTable:
        arrs = [np.ascontiguousarray(term_row_offset, np.uint64), np.ascontiguousarray(term_coef, np.int64).reshape(-1),
                np.ascontiguousarray(psi_mask, np.uint64), np.ascontiguousarray(phi_mask, np.uint64),
                np.ascontiguousarray(k_alpha, np.uint8), np.ascontiguousarray(k_beta, np.uint8)]
        arrs = [x if x.size else np.zeros(1, x.dtype) for x in arrs]
        v = N.TableView(n_params, len(term_row_offset) - 1, N.ptr(arrs[0], C.c_uint64), N.ptr(arrs[1], C.c_int64),
                        N.ptr(arrs[2], C.c_uint64), N.ptr(arrs[3], C.c_uint64), N.ptr(arrs[4], C.c_uint8),
                        N.ptr(arrs[5], C.c_uint8))
        h = C.c_void_p()
        _check(N.lib().pzx_table_upload(self.handle, C.byref(v), C.byref(h)), self.handle)
        return DeviceTable(self, h)

    def backend_contract(self) -> dict:
        """SPEC BackendContract: this backend's capabilities."""
        c = N.BackendContract()
        _check(N.lib().pzx_backend_contract_get(self.handle, C.byref(c)), self.handle)
        return {k: getattr(c, k) for k, _ in N.BackendContract._fields_}

    def upload_pzx1(self, data: bytes) -> DeviceTable:
        """Upload a PZX1-encoded table (see encode_pzx1)."""
        buf = np.frombuffer(bytes(data), np.uint8) if len(data) else np.zeros(1, np.uint8)
        h = C.c_void_p()
        _check(N.lib().pzx_table_upload_pzx1(self.handle, N.ptr(buf, C.c_uint8), len(data), C.byref(h)),
               self.handle)
        return DeviceTable(self, h)

    # -- evaluation -----------------------------------------------------------
    def evaluate_batch(self, table: DeviceTable, assignments, *, prob: bool = False,
                       prob_real: bool = False, flags: int = 0):
        """Amplitudes (complex128) at assignment words, input order kept."""
        a = np.ascontiguousarray(np.asarray(assignments, dtype=np.uint64))
        n = a.size
        amp = np.empty(n, np.complex128)
        pr = np.empty(n, np.float64) if (prob or prob_real) else None
        fl = flags | (PROB_REAL if prob_real else PROB_ABS2)
        if n:
            _check(N.lib().pzx_evaluate(self.handle, table.handle, N.ptr(a, C.c_uint64), n,
                                        amp.ctypes.data_as(N.dblp), N.ptr(pr, C.c_double), fl), self.handle)
        return (amp, pr) if pr is not None else amp

    def evaluate(self, table: DeviceTable, word: int) -> complex:
        return complex(self.evaluate_batch(table, [word])[0])

    def evaluate_range(self, table: DeviceTable, first: int, n: int, *, prob: bool = False,
                       prob_real: bool = False, flags: int = 0):
        amp = np.empty(n, np.complex128)
        pr = np.empty(n, np.float64) if (prob or prob_real) else None
        fl = flags | (PROB_REAL if prob_real else PROB_ABS2)
        if n:
            _check(N.lib().pzx_evaluate_range(self.handle, table.handle, first, n, amp.ctypes.data_as(N.dblp),
                                              N.ptr(pr, C.c_double), fl), self.handle)
        return (amp, pr) if pr is not None else amp

    def evaluate_exact(self, table: DeviceTable, assignments, *, allow_overflow: bool = False) -> np.ndarray:
        """Exact S(a) per assignment as canonical RingQuads, int64 [n, 5] =
        (a, b, c, d, exp) -- the SPEC's integer backend, the same
        layout as oracle_py.eval_batch's exact output. OverflowError when a
        value leaves int64 (allow_overflow: return with exp = -1 there)."""
        a = np.ascontiguousarray(np.asarray(assignments, dtype=np.uint64))
        out = np.zeros((a.size, 5), np.int64)
        if a.size:
            st = N.lib().pzx_evaluate_exact(self.handle, table.handle, a.ctypes.data_as(N.u64p), a.size,
                                            out.ctypes.data_as(N.i64p))
            if not (allow_overflow and st == 4):
                _check(st, self.handle)
        return out

    def evaluate_exact_range(self, table: DeviceTable, first: int, n: int, *,
                             allow_overflow: bool = False) -> np.ndarray:
        out = np.zeros((n, 5), np.int64)
        if n:
            st = N.lib().pzx_evaluate_exact_range(self.handle, table.handle, first, n, out.ctypes.data_as(N.i64p))
            if not (allow_overflow and st == 4):
                _check(st, self.handle)
        return out

    def ringquad_sum(self, parts, *, allow_overflow: bool = False) -> np.ndarray:
        """Exact sum over axis 0 of canonical RingQuads, int64 [G, n, 5] -> [n, 5]
        (the term split's combine; order-free, canonical).
        OverflowError when a sum leaves int64 (allow_overflow: exp = -1 there)."""
        p = np.ascontiguousarray(np.asarray(parts, dtype=np.int64))
        if p.ndim != 3 or p.shape[2] != 5:
            raise ValueError("ringquad_sum: parts must be int64 [G, n, 5]")
        out = np.zeros((p.shape[1], 5), np.int64)
        if p.shape[1]:
            st = N.lib().pzx_ringquad_sum(self.handle, p.ctypes.data_as(N.i64p), p.shape[0], p.shape[1],
                                          out.ctypes.data_as(N.i64p))
            if not (allow_overflow and st == 4):
                _check(st, self.handle)
        return out

    def ringquad_sum_device(self, d_parts: int, n_parts: int, n: int, d_out: int, stream: int = 0) -> None:
        """Async device-pointer form of ringquad_sum (raw CUDA pointers as ints)."""
        _check(N.lib().pzx_ringquad_sum_device(self.handle, d_parts or None, n_parts, n, d_out or None,
                                               stream or None), self.handle)

    def evaluate_device(self, table: DeviceTable, n: int, *, d_assignments: int = 0, first: int = 0,
                        term_begin: int = 0, term_end: int = 2**64 - 1, d_amp: int = 0, d_prob: int = 0,
                        flags: int = PROB_ABS2, stream: int = 0) -> None:
        """Async device-pointer form (raw CUDA pointers as ints, e.g. torch data_ptr())."""
        _check(N.lib().pzx_evaluate_device(self.handle, table.handle, d_assignments or None, first, n,
                                           term_begin, term_end, d_amp or None, d_prob or None, flags,
                                           stream or None), self.handle)

    def amp_to_prob_device(self, d_amp: int, n: int, d_prob: int, flags: int = PROB_ABS2, stream: int = 0):
        _check(N.lib().pzx_amp_to_prob_device(self.handle, d_amp, n, d_prob, flags, stream or None), self.handle)

    def synchronize(self) -> None:
        _check(N.lib().pzx_synchronize(self.handle), self.handle)

    def weak_sample(self, tables, n_samples: int, seed: int = 0, abs2: bool = False, flags: int = 0) -> np.ndarray:
        """Repeated weak simulation (PAPER App. F Alg. 2): tables[k] is the
        doubled marginal over parameters a_1..a_{k+1}; returns n_samples
        words whose bit k is the sampled output bit k."""
        hs = (C.c_void_p * max(1, len(tables)))(*[t.handle for t in tables])
        out = np.zeros(n_samples, np.uint64)
        flags = (flags & ~(PROB_ABS2 | PROB_REAL)) | (PROB_ABS2 if abs2 else PROB_REAL)
        if n_samples:
            _check(N.lib().pzx_weak_sample(self.handle, hs, len(tables), n_samples, seed & (2**64 - 1), flags,
                                           N.ptr(out, C.c_uint64)), self.handle)
        return out

    def marginal_sum(self, table: DeviceTable, fixed, m: int, prob_real: bool = False,
                     flags: int = 0) -> np.ndarray:
        """Marginal summing (sim-driver): for every fixed word,
        the sum over the 2^m settings of the low m parameters (the don't-care
        outputs) of |amp|^2 -- or of Re(amp) for doubled diagrams."""
        f = np.ascontiguousarray(np.asarray(fixed, dtype=np.uint64))
        out = np.empty(f.size, np.float64)
        if f.size:
            flags = (flags & ~(PROB_ABS2 | PROB_REAL)) | (PROB_REAL if prob_real else PROB_ABS2)
            _check(N.lib().pzx_marginal_sum(self.handle, table.handle, N.ptr(f, C.c_uint64), f.size, m, flags,
                                            N.ptr(out, C.c_double)), self.handle)
        return out

    # -- debug / parity hooks -------------------------------------------------
    def debug_phase_indices(self, table: DeviceTable, assignments) -> np.ndarray:
        a = np.ascontiguousarray(np.asarray(assignments, dtype=np.uint64))
        out = np.empty((table.n_rows, a.size), np.uint8)
        if out.size:
            _check(N.lib().pzx_debug_phase_indices(self.handle, table.handle, N.ptr(a, C.c_uint64), a.size,
                                                   N.ptr(out, C.c_uint8)), self.handle)
        return out

    def debug_term_codes(self, table: DeviceTable, assignments) -> np.ndarray:
        a = np.ascontiguousarray(np.asarray(assignments, dtype=np.uint64))
        out = np.zeros((table.n_terms, a.size, 5), np.uint32)
        if out.size:
            _check(N.lib().pzx_debug_term_codes(self.handle, table.handle, N.ptr(a, C.c_uint64), a.size,
                                                out.ctypes.data_as(C.POINTER(N.TermCode))), self.handle)
        return out


def _debug_slice_codes(self, table, assignments=None, first: int = 0, n: int | None = None, term_begin: int = 0,
                       term_end: int | None = None, flags: int = 0):
    """The production bit-sliced kernel's own per-term codes (pzx_debug_slice_codes):
    uint32 [terms, n, 5] = {j, z (flag), s1, a, b} for terms [term_begin, term_end)."""
    a = None
    if assignments is not None:
        a = np.ascontiguousarray(np.asarray(assignments, dtype=np.uint64))
        n = a.size
    te = table.n_terms if term_end is None else term_end
    out = np.zeros((max(te - term_begin, 0), n, 5), np.uint32)
    if out.size:
        _check(N.lib().pzx_debug_slice_codes(self.handle, table.handle, N.ptr(a, C.c_uint64), first, n, term_begin,
                                             te, flags, out.ctypes.data_as(C.POINTER(N.TermCode))), self.handle)
    return out


Context.debug_slice_codes = _debug_slice_codes


class HostTable:
    """Host-only compiled table (pzx_table_compile_host): inspection and CPU tests."""

    def __init__(self, expr: ScalarExpression):
        v, keep = expr.view()
        h = C.c_void_p()
        _check(N.lib().pzx_table_compile_host(C.byref(v), C.byref(h)))
        del keep
        self.handle = h
        L = N.lib()
        p, m, r, mx = C.c_uint32(), C.c_uint64(), C.c_uint64(), C.c_uint32()
        _check(L.pzx_table_shape(h, C.byref(p), C.byref(m), C.byref(r), C.byref(mx)))
        self.n_params, self.n_terms, self.n_rows, self.max_term_rows = p.value, m.value, r.value, mx.value

    term_info = DeviceTable.term_info
    slice_stats = DeviceTable.slice_stats
    page_stats = DeviceTable.page_stats

    def page_layout(self):
        """(slots uint32 [n, 8], term_slot [m], jfold [m], family_rows [11]) of the
        page kernel's layout (pzx_table_page_layout), or None without one."""
        L = N.lib()
        n = C.c_uint64()
        fam = np.zeros(11, np.uint64)
        st = L.pzx_table_page_layout(self.handle, None, C.byref(n), None, None, N.ptr(fam, C.c_uint64))
        if st == 6:
            return None
        _check(st)
        slots = np.zeros((max(n.value, 1), 8), np.uint32)
        ts = np.zeros(max(self.n_terms, 1), np.uint32)
        jf = np.zeros(max(self.n_terms, 1), np.uint8)
        _check(L.pzx_table_page_layout(self.handle, slots.ctypes.data_as(C.POINTER(C.c_uint32)), C.byref(n),
                                       ts.ctypes.data_as(C.POINTER(C.c_uint32)), N.ptr(jf, C.c_uint8), None))
        return slots[:n.value], ts[:self.n_terms], jf[:self.n_terms], fam
    free = DeviceTable.free
    __del__ = DeviceTable.__del__


def class_table():
    """(codes[64,4] uint32, e[64], lm[64]) -- the kernels' per-class variant codes."""
    codes = np.zeros(256, np.uint32)
    e = np.zeros(64, np.int32)
    lm = np.zeros(64, np.int32)
    _check(N.lib().pzx_class_table(N.ptr(codes, C.c_uint32), N.ptr(e, C.c_int32), N.ptr(lm, C.c_int32)))
    return codes.reshape(64, 4), e, lm


def slice_op_table() -> np.ndarray:
    """[129, 10] int32: the bit-sliced kernel's row ops (pzx_slice_op_table)."""
    out = np.zeros(129 * 10, np.int32)
    _check(N.lib().pzx_slice_op_table(N.ptr(out, C.c_int32)))
    return out.reshape(129, 10)


# ------------------------------------------------------------ multi-GPU ----
REPLICATE, SPLIT_TERMS = 0, 1


class Group:
    """Several GPUs driven from this thread through the C ABI (pzx_group_*):
    REPLICATE shards batches across devices, SPLIT_TERMS splits the table and
    sums partial amplitudes on the first device (peer copies, device order)."""

    def __init__(self, devices: Sequence[int]):
        arr = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _check(N.lib().pzx_group_create(arr, len(devices), C.byref(h)))
        self.handle = h
        self.devices = list(devices)

    def _check(self, st: int) -> None:
        if st:
            lib = N.lib()
            raise _STATUS.get(st, Error)(f"{lib.pzx_status_string(st).decode()}: "
                                         f"{lib.pzx_group_last_error(self.handle).decode()}")

    def upload(self, expr: ScalarExpression, mode: int = REPLICATE) -> "GroupTable":
        v, keep = expr.view()
        h = C.c_void_p()
        self._check(N.lib().pzx_group_upload_expr(self.handle, C.byref(v), mode, C.byref(h)))
        del keep
        return GroupTable(h)

    def evaluate_batch(self, table: "GroupTable", assignments, prob_real: bool = False) -> np.ndarray:
        a = np.ascontiguousarray(np.asarray(assignments, dtype=np.uint64))
        amp = np.empty(a.size, np.complex128)
        if a.size:
            self._check(N.lib().pzx_group_evaluate(self.handle, table.handle, N.ptr(a, C.c_uint64), 0, a.size,
                                                   N.ptr(amp.view(np.float64), C.c_double), None,
                                                   PROB_REAL if prob_real else PROB_ABS2))
        return amp

    def evaluate_range(self, table: "GroupTable", first: int, n: int) -> np.ndarray:
        amp = np.empty(n, np.complex128)
        if n:
            self._check(N.lib().pzx_group_evaluate(self.handle, table.handle, None, first, n,
                                                   N.ptr(amp.view(np.float64), C.c_double), None, PROB_ABS2))
        return amp

    def close(self) -> None:
        if self.handle:
            N.lib().pzx_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GroupTable:
    def __init__(self, handle):
        self.handle = handle

    def free(self) -> None:
        if self.handle:
            N.lib().pzx_group_table_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# ---------------------------------------------------------------- PZX1 ----
@dataclass
class PhaseTable:
    """A normalised table (SPEC ScalarExpression after Eq. 4): term t is
    C_t * prod of pair rows term_row_offset[t] .. term_row_offset[t+1]-1."""

    n_params: int
    term_row_offset: np.ndarray
    term_coef: np.ndarray      # [m, 5] RingQuad a, b, c, d, exp
    psi_mask: np.ndarray
    phi_mask: np.ndarray
    k_alpha: np.ndarray
    k_beta: np.ndarray

    @property
    def n_terms(self) -> int:
        return len(self.term_row_offset) - 1

    def view(self):
        arrs = [np.ascontiguousarray(self.term_row_offset, np.uint64),
                np.ascontiguousarray(self.term_coef, np.int64).reshape(-1),
                np.ascontiguousarray(self.psi_mask, np.uint64), np.ascontiguousarray(self.phi_mask, np.uint64),
                np.ascontiguousarray(self.k_alpha, np.uint8), np.ascontiguousarray(self.k_beta, np.uint8)]
        arrs = [x if x.size else np.zeros(1, x.dtype) for x in arrs]
        v = N.TableView(self.n_params, self.n_terms, N.ptr(arrs[0], C.c_uint64), N.ptr(arrs[1], C.c_int64),
                        N.ptr(arrs[2], C.c_uint64), N.ptr(arrs[3], C.c_uint64), N.ptr(arrs[4], C.c_uint8),
                        N.ptr(arrs[5], C.c_uint8))
        return v, arrs


def _encode(fn, view) -> bytes:
    n = C.c_uint64()
    _check(fn(C.byref(view), None, 0, C.byref(n)))
    buf = np.empty(max(1, n.value), np.uint8)
    _check(fn(C.byref(view), N.ptr(buf, C.c_uint8), n.value, C.byref(n)))
    return buf[:n.value].tobytes()


def encode_pzx1(obj) -> bytes:
    """PZX1 binary codec (SPEC "External Interfaces"): a ScalarExpression is
    normalised first (normalize_subterm, constants folded); a PhaseTable is
    written as is."""
    L = N.lib()
    if isinstance(obj, ScalarExpression):
        v, keep = obj.view()
        out = _encode(L.pzx_pzx1_encode_expr, v)
        del keep
        return out
    v, keep = obj.view()
    out = _encode(L.pzx_pzx1_encode, v)
    del keep
    return out


def decode_pzx1(data: bytes) -> PhaseTable:
    L = N.lib()
    buf = np.frombuffer(bytes(data), np.uint8) if len(data) else np.zeros(1, np.uint8)
    p, m, r = C.c_uint32(), C.c_uint64(), C.c_uint64()
    _check(L.pzx_pzx1_info(N.ptr(buf, C.c_uint8), len(data), C.byref(p), C.byref(m), C.byref(r)))
    off = np.empty(m.value + 1, np.uint64)
    coef = np.empty(max(1, 5 * m.value), np.int64)
    R = max(1, r.value)
    psi, phi = np.empty(R, np.uint64), np.empty(R, np.uint64)
    ka, kb = np.empty(R, np.uint8), np.empty(R, np.uint8)
    _check(L.pzx_pzx1_decode(N.ptr(buf, C.c_uint8), len(data), N.ptr(off, C.c_uint64), N.ptr(coef, C.c_int64),
                             N.ptr(psi, C.c_uint64), N.ptr(phi, C.c_uint64), N.ptr(ka, C.c_uint8),
                             N.ptr(kb, C.c_uint8)))
    n = r.value
    return PhaseTable(p.value, off, coef[:5 * m.value].reshape(-1, 5), psi[:n], phi[:n], ka[:n], kb[:n])


def pzx1_to_json(data: bytes) -> str:
    """JSON mirror of a PZX1 blob (same fields, padded rows included)."""
    import json
    import struct
    if len(data) < 32 or data[:4] != b"PZX1":
        raise ParseError("PZX1: bad magic / truncated header")
    n, m, n_max, R = struct.unpack_from("<IQQQ", data, 4)
    t = decode_pzx1(data)
    flags, ka, kb, psi, phi = [], [], [], [], []
    for i in range(m):
        a, b = int(t.term_row_offset[i]), int(t.term_row_offset[i + 1])
        for j in range(n_max):
            real = a + j < b
            flags.append(0 if real else 1)
            ka.append(int(t.k_alpha[a + j]) if real else 0)
            kb.append(int(t.k_beta[a + j]) if real else 0)
            psi.append(int(t.psi_mask[a + j]) if real else 0)
            phi.append(int(t.phi_mask[a + j]) if real else 0)
    return json.dumps({"magic": "PZX1", "n_params": n, "m": m, "n_max": n_max, "R": R,
                       "constants": t.term_coef.tolist(), "flags": flags, "k_alpha": ka, "psi": psi,
                       "k_beta": kb, "phi": phi}, separators=(",", ":"))


def pzx1_from_json(text: str) -> bytes:
    import json
    import struct
    d = json.loads(text)
    if d.get("magic") != "PZX1":
        raise ParseError("PZX1 JSON: bad magic")
    m, n_max, R = d["m"], d["n_max"], d["R"]
    if R != m * n_max or any(len(d[k]) != R for k in ("flags", "k_alpha", "psi", "k_beta", "phi")) \
            or len(d["constants"]) != m:
        raise ParseError("PZX1 JSON: inconsistent shape")
    out = bytearray(b"PZX1" + struct.pack("<IQQQ", d["n_params"], m, n_max, R))
    out += np.asarray(d["constants"], np.int64).reshape(-1).astype("<i8").tobytes()
    out += np.asarray(d["flags"], np.uint8).tobytes() + np.asarray(d["k_alpha"], np.uint8).tobytes()
    out += np.asarray(d["psi"], np.uint64).astype("<u8").tobytes()
    out += np.asarray(d["k_beta"], np.uint8).tobytes() + np.asarray(d["phi"], np.uint64).astype("<u8").tobytes()
    decode_pzx1(bytes(out))  # validate
    return bytes(out)


def compile_bit_table(expr: ScalarExpression, ctx: Context) -> DeviceTable:
    """SPEC compile_bit_table: normalise, classify, upload."""
    return ctx.compile_bit_table(expr)


def evaluate_batch(ctx: Context, table: DeviceTable, assignments) -> np.ndarray:
    """SPEC evaluate_batch; output order equals input order."""
    return ctx.evaluate_batch(table, assignments)


def evaluate(ctx: Context, table: DeviceTable, word: int) -> complex:
    """SPEC evaluate."""
    return ctx.evaluate(table, word)


__all__ = [
    "Error", "ParseError", "DomainError", "Lemma1Violation", "OverflowError", "MissingParameter", "CudaError",
    "kMaxParams", "ParamAssignment", "ParamPhase", "phase_add", "SubtermKind", "Subterm", "RingQuad",
    "ScalarExpression", "DeviceTable", "HostTable", "class_table", "Context", "compile_bit_table", "evaluate_batch", "evaluate",
    "Group", "GroupTable", "REPLICATE", "SPLIT_TERMS", "PhaseTable", "encode_pzx1", "decode_pzx1", "pzx1_to_json", "pzx1_from_json",
    "PROB_ABS2", "PROB_REAL", "ACCUMULATE", "KERNEL_GENERAL", "KERNEL_GRAY", "KERNEL_SLICE", "KERNEL_SLICE_RAND", "KERNEL_SORTED", "KERNEL_SLICE2", "KERNEL_PAGE", "slice_op_table",
]
_ = builtins
