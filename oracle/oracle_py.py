"""ctypes front-end for the CPU ORACLES (test infrastructure only).

Loads
  * ``oracle/lib/libpzx_oracle.so`` -- the plain-C restatement (pzx_oracle.c), and
  * ``oracle/_ref/libpzx_ref.so``   -- the UNMODIFIED reference core compiled
    from /root/reference by oracle/Makefile (present wherever it was built; it
    travels to the GPU box with the snapshot).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module; the product never does.
Expressions are duck-typed: any object with the ScalarExpression SoA fields
(n_params, term_offset, term_scalar, kind, psi_k, psi_mask, phi_k, phi_mask).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "lib", "libpzx_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libpzx_ref.so")

OK, E_PARSE, E_DOMAIN, E_MISSING, E_OVERFLOW = 0, 1, 2, 3, 4


class Quad(C.Structure):
    _fields_ = [("a", C.c_int64), ("b", C.c_int64), ("c", C.c_int64), ("d", C.c_int64),
                ("exp", C.c_int32), ("pad_", C.c_int32)]

    def tup(self):
        return (self.a, self.b, self.c, self.d, self.exp)


class Sub(C.Structure):
    _fields_ = [("kind", C.c_uint8), ("psi_k", C.c_uint8), ("phi_k", C.c_uint8), ("pad_", C.c_uint8 * 5),
                ("psi_mask", C.c_uint64), ("phi_mask", C.c_uint64)]


class Expr(C.Structure):
    _fields_ = [("n_params", C.c_uint32), ("n_terms", C.c_uint64), ("term_offset", C.POINTER(C.c_uint64)),
                ("scalars", C.POINTER(Quad)), ("subterms", C.POINTER(Sub))]


QUAD_DT = np.dtype([("a", "<i8"), ("b", "<i8"), ("c", "<i8"), ("d", "<i8"), ("exp", "<i4"), ("pad", "<i4")])
SUB_DT = np.dtype([("kind", "u1"), ("psi_k", "u1"), ("phi_k", "u1"), ("pad", "u1", 5),
                   ("psi_mask", "<u8"), ("phi_mask", "<u8")])
assert QUAD_DT.itemsize == C.sizeof(Quad) and SUB_DT.itemsize == C.sizeof(Sub)


def build() -> None:
    """Build the restatement (always) and oracle/_ref (where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "-f", os.path.join(HERE, "Makefile")], check=True)


_port = None
_ref = None


def _proto(L, ref: bool):
    qp, sp, ep = C.POINTER(Quad), C.POINTER(Sub), C.POINTER(Expr)
    u64p, dblp = C.POINTER(C.c_uint64), C.POINTER(C.c_double)
    if ref:
        L.ref_eval_batch.argtypes = [ep, u64p, C.c_uint64, C.c_int, C.c_int, qp, dblp]
        L.ref_term_value.argtypes = [ep, C.c_uint64, C.c_uint64, qp]
        L.ref_normalize.argtypes = [sp, qp, C.POINTER(C.c_int), sp]
        L.ref_subterm_value.argtypes = [sp, C.c_uint64, C.c_uint32, qp]
        L.ref_pair_value.argtypes = [C.c_int, C.c_int, qp]
        L.ref_instantiate_phase.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint32, C.POINTER(C.c_int)]
        L.ref_ring_add.argtypes = [qp, qp, qp]
        L.ref_ring_mul.argtypes = [qp, qp, qp]
        L.ref_make.argtypes = [C.c_int64] * 4 + [C.c_int32, qp]
        L.ref_to_complex.argtypes = [qp, dblp, dblp]
        L.ref_to_complex.restype = None
        L.ref_prepare.argtypes = [ep, C.c_int, C.POINTER(C.c_int)]
        L.ref_prepare.restype = C.c_void_p
        L.ref_eval_prepared.argtypes = [C.c_void_p, u64p, C.c_uint64, C.c_int, qp, dblp]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_free.restype = None
    else:
        L.oq_make.argtypes = [C.c_int64] * 4 + [C.c_int32, qp]
        L.oq_add.argtypes = [qp, qp, qp]
        L.oq_sub.argtypes = [qp, qp, qp]
        L.oq_mul.argtypes = [qp, qp, qp]
        L.oq_omega.argtypes = [C.c_int, qp]
        L.oq_to_complex.argtypes = [qp, dblp, dblp]
        L.oq_to_complex.restype = None
        L.oq_instantiate_phase.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_int)]
        L.oq_pair_value.argtypes = [C.c_int, C.c_int, qp]
        L.oq_subterm_value.argtypes = [sp, C.c_uint64, C.c_uint64, qp]
        L.oq_normalize.argtypes = [sp, qp, C.POINTER(C.c_int), sp]
        L.oq_term_value.argtypes = [ep, C.c_uint64, C.c_uint64, C.c_uint64, qp]
        L.oq_eval_one.argtypes = [ep, C.c_uint64, qp]
        L.oq_eval_batch.argtypes = [ep, u64p, C.c_uint64, C.c_int, qp, dblp]
        L.oq_normalize_expr.argtypes = [ep, qp, u64p, sp, u64p]
        L.oq_phase_indices.argtypes = [ep, u64p, C.c_uint64, C.POINTER(C.c_uint8)]
    return L


def port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_LIB):
            build()
        _port = _proto(C.CDLL(PORT_LIB), False)
    return _port


def have_ref() -> bool:
    return os.path.exists(REF_LIB)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_LIB):
            raise FileNotFoundError(REF_LIB + " (build oracle/_ref where /root/reference exists)")
        _ref = _proto(C.CDLL(REF_LIB), True)
    return _ref


class OExpr:
    """An expression marshalled into the oracle's C structs (arrays kept alive)."""

    def __init__(self, e):
        self.n_params = int(e.n_params)
        self.off = np.ascontiguousarray(e.term_offset, np.uint64)
        m = len(self.off) - 1
        sc = np.asarray(e.term_scalar, np.int64).reshape(-1, 5)[:m]
        self.scal = np.zeros(max(m, 1), QUAD_DT)
        for i, f in enumerate(("a", "b", "c", "d", "exp")):
            self.scal[f][:m] = sc[:, i]
        S = int(self.off[-1]) if m else 0
        self.subs = np.zeros(max(S, 1), SUB_DT)
        if S:
            self.subs["kind"][:S] = np.asarray(e.kind)[:S]
            self.subs["psi_k"][:S] = np.asarray(e.psi_k)[:S]
            self.subs["phi_k"][:S] = np.asarray(e.phi_k)[:S]
            self.subs["psi_mask"][:S] = np.asarray(e.psi_mask)[:S]
            self.subs["phi_mask"][:S] = np.asarray(e.phi_mask)[:S]
        self.c = Expr(self.n_params, m, self.off.ctypes.data_as(C.POINTER(C.c_uint64)),
                      self.scal.ctypes.data_as(C.POINTER(Quad)), self.subs.ctypes.data_as(C.POINTER(Sub)))
        self.n_terms = m


class OracleError(RuntimeError):
    def __init__(self, status):
        super().__init__(f"oracle status {status}")
        self.status = status


def eval_batch(expr, words, threads: int = 1, impl: str = "port", mode: int = 0):
    """Exact values (int64 [n,5]: a,b,c,d,exp) and complex128 amplitudes."""
    oe = expr if isinstance(expr, OExpr) else OExpr(expr)
    w = np.ascontiguousarray(np.asarray(words, np.uint64))
    n = w.size
    ex = np.zeros(max(n, 1), QUAD_DT)
    amp = np.zeros(max(n, 1), np.complex128)
    args = (C.byref(oe.c), w.ctypes.data_as(C.POINTER(C.c_uint64)), n, threads)
    outs = (ex.ctypes.data_as(C.POINTER(Quad)), amp.ctypes.data_as(C.POINTER(C.c_double)))
    st = ref().ref_eval_batch(*args, mode, *outs) if impl == "ref" else port().oq_eval_batch(*args, *outs)
    if st:
        raise OracleError(st)
    exact = np.stack([ex[f][:n].astype(np.int64) for f in ("a", "b", "c", "d", "exp")], axis=1)
    return exact, amp[:n]


class RefPrepared:
    """The reference's own evaluator with the term list converted to its value
    types once (ref_prepare), so that timing covers only the evaluation path."""

    def __init__(self, expr, mode: int = 0):
        self.oe = expr if isinstance(expr, OExpr) else OExpr(expr)
        st = C.c_int()
        self.h = ref().ref_prepare(C.byref(self.oe.c), mode, C.byref(st))
        if not self.h:
            raise OracleError(st.value)

    def eval(self, words, threads: int = 1, want_exact: bool = True):
        w = np.ascontiguousarray(np.asarray(words, np.uint64))
        n = w.size
        ex = np.zeros(max(n, 1), QUAD_DT)
        amp = np.zeros(max(n, 1), np.complex128)
        st = ref().ref_eval_prepared(self.h, w.ctypes.data_as(C.POINTER(C.c_uint64)), n, threads,
                                     ex.ctypes.data_as(C.POINTER(Quad)) if want_exact else None,
                                     amp.ctypes.data_as(C.POINTER(C.c_double)))
        if st:
            raise OracleError(st)
        exact = np.stack([ex[f][:n].astype(np.int64) for f in ("a", "b", "c", "d", "exp")], axis=1)
        return exact, amp[:n]

    def close(self):
        if self.h:
            ref().ref_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def term_value(expr, t: int, word: int, impl: str = "port"):
    oe = expr if isinstance(expr, OExpr) else OExpr(expr)
    q = Quad()
    if impl == "ref":
        st = ref().ref_term_value(C.byref(oe.c), t, word, C.byref(q))
    else:
        P = oe.n_params
        m = (1 << P) - 1 if P < 64 else 2**64 - 1
        st = port().oq_term_value(C.byref(oe.c), t, word & m, m, C.byref(q))
    if st:
        raise OracleError(st)
    return q.tup()


def normalize_expr(expr):
    """Folded constants [m,5], row offsets [m+1], rows (k_alpha, psi, k_beta, phi)."""
    oe = expr if isinstance(expr, OExpr) else OExpr(expr)
    nrows = C.c_uint64()
    L = port()
    st = L.oq_normalize_expr(C.byref(oe.c), None, None, None, C.byref(nrows))
    if st:
        raise OracleError(st)
    R = nrows.value
    folded = np.zeros(max(oe.n_terms, 1), QUAD_DT)
    offs = np.zeros(oe.n_terms + 1, np.uint64)
    rows = np.zeros(max(R, 1), SUB_DT)
    st = L.oq_normalize_expr(C.byref(oe.c), folded.ctypes.data_as(C.POINTER(Quad)),
                             offs.ctypes.data_as(C.POINTER(C.c_uint64)), rows.ctypes.data_as(C.POINTER(Sub)),
                             C.byref(nrows))
    if st:
        raise OracleError(st)
    f = np.stack([folded[k][:oe.n_terms].astype(np.int64) for k in ("a", "b", "c", "d", "exp")], axis=1)
    r = rows[:R]
    return f, offs, (r["psi_k"].copy(), r["psi_mask"].copy(), r["phi_k"].copy(), r["phi_mask"].copy())


def phase_indices(expr, words):
    oe = expr if isinstance(expr, OExpr) else OExpr(expr)
    w = np.ascontiguousarray(np.asarray(words, np.uint64))
    _, offs, _ = normalize_expr(oe)
    R = int(offs[-1])
    out = np.zeros((max(R, 1), max(w.size, 1)), np.uint8)
    st = port().oq_phase_indices(C.byref(oe.c), w.ctypes.data_as(C.POINTER(C.c_uint64)), w.size,
                                 out.ctypes.data_as(C.POINTER(C.c_uint8)))
    if st:
        raise OracleError(st)
    return out[:R, :w.size]


# -- scalar helpers for known-answer tests ------------------------------------
def _q(t):
    return Quad(int(t[0]), int(t[1]), int(t[2]), int(t[3]), int(t[4]), 0)


def make(a, b, c, d, e, impl="port"):
    q = Quad()
    st = (ref().ref_make if impl == "ref" else port().oq_make)(a, b, c, d, e, C.byref(q))
    if st:
        raise OracleError(st)
    return q.tup()


def ring_add(x, y, impl="port"):
    q = Quad()
    st = (ref().ref_ring_add if impl == "ref" else port().oq_add)(C.byref(_q(x)), C.byref(_q(y)), C.byref(q))
    if st:
        raise OracleError(st)
    return q.tup()


def ring_mul(x, y, impl="port"):
    q = Quad()
    st = (ref().ref_ring_mul if impl == "ref" else port().oq_mul)(C.byref(_q(x)), C.byref(_q(y)), C.byref(q))
    if st:
        raise OracleError(st)
    return q.tup()


def pair_value(ka, kb, impl="port"):
    q = Quad()
    st = (ref().ref_pair_value if impl == "ref" else port().oq_pair_value)(ka, kb, C.byref(q))
    if st:
        raise OracleError(st)
    return q.tup()


def omega(k):
    q = Quad()
    st = port().oq_omega(k, C.byref(q))
    if st:
        raise OracleError(st)
    return q.tup()


def instantiate_phase(k, mask, word, n_params, impl="port"):
    out = C.c_int()
    if impl == "ref":
        st = ref().ref_instantiate_phase(k, mask, word, n_params, C.byref(out))
    else:
        m = (1 << n_params) - 1 if n_params < 64 else 2**64 - 1
        st = port().oq_instantiate_phase(k, mask, word & m, m, C.byref(out))
    if st:
        raise OracleError(st)
    return out.value


def _sub(kind, psi_k, psi_mask, phi_k=0, phi_mask=0):
    s = Sub()
    s.kind, s.psi_k, s.phi_k, s.psi_mask, s.phi_mask = kind, psi_k, phi_k, psi_mask, phi_mask
    return s


def subterm_value(kind, psi_k, psi_mask, phi_k, phi_mask, word, n_params, impl="port"):
    s = _sub(kind, psi_k, psi_mask, phi_k, phi_mask)
    q = Quad()
    if impl == "ref":
        st = ref().ref_subterm_value(C.byref(s), word, n_params, C.byref(q))
    else:
        m = (1 << n_params) - 1 if n_params < 64 else 2**64 - 1
        st = port().oq_subterm_value(C.byref(s), word & m, m, C.byref(q))
    if st:
        raise OracleError(st)
    return q.tup()


def normalize(kind, psi_k, psi_mask, phi_k=0, phi_mask=0, impl="port"):
    s = _sub(kind, psi_k, psi_mask, phi_k, phi_mask)
    q, has, pr = Quad(), C.c_int(), Sub()
    st = (ref().ref_normalize if impl == "ref" else port().oq_normalize)(C.byref(s), C.byref(q), C.byref(has),
                                                                          C.byref(pr))
    if st:
        raise OracleError(st)
    pair = (pr.psi_k, pr.psi_mask, pr.phi_k, pr.phi_mask) if has.value else None
    return q.tup(), pair


def to_complex(x, impl="port"):
    re, im = C.c_double(), C.c_double()
    (ref().ref_to_complex if impl == "ref" else port().oq_to_complex)(C.byref(_q(x)), C.byref(re), C.byref(im))
    return complex(re.value, im.value)
