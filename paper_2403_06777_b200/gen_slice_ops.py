"""Generate csrc/pzx_slice_dispatch.inc: the bit-sliced kernel's per-row
update as ONE inline-PTX block with a jump table (brx.idx -> SASS BRX).

Each of the 129 slice ops (op = class * 2 + single, 128 = unit row;
pzx_classes.h) gets a straight-line LOP3 chain with compile-time truth tables:

  (J2 J1 J0) += w'(X, Y)  mod 8     ripple carry over the three bit planes
  Z          |= zero(X, Y)           parity-constraint rows
  vl / vpi / vpip = lambda / pi / pi' indicator vectors (consumed in C++)

X (Y) holds parity(psi & a) (parity(phi & a)) for the thread's 32 assignments.
The op table is re-derived here by exact Z[w] factorisation; tests compare it
with the constexpr table the C++ side uses (pzx_slice_op_table).
"""
from __future__ import annotations

import os

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "csrc", "pzx_slice_dispatch.inc")

# ---------------------------------------------------------------- Z[w] ----


def wpow(k):
    k %= 8
    c = [0, 0, 0, 0]
    if k < 4:
        c[k] = 1
    else:
        c[k - 4] = -1
    return tuple(c)


def mul(x, y):
    t = [0] * 8
    for i in range(4):
        for j in range(4):
            t[i + j] += x[i] * y[j]
    return tuple(t[i] - t[i + 4] for i in range(4))


def add(x, y):
    return tuple(a + b for a, b in zip(x, y))


def sigma(x, s):
    r = (0, 0, 0, 0)
    for i, c in enumerate(x):
        r = add(r, tuple(c * v for v in wpow(s * i)))
    return r


def norm(x):
    return mul(mul(x, sigma(x, 3)), mul(sigma(x, 5), sigma(x, 7)))[0]


def div(x, y):
    co = mul(mul(sigma(y, 3), sigma(y, 5)), sigma(y, 7))
    n = norm(y)
    t = mul(x, co)
    if all(v % n == 0 for v in t):
        return tuple(v // n for v in t)
    return None


KNONE, KLAMBDA, KMU, KPI, KPIP, KZERO = range(6)
GEN = {KNONE: (1, 0, 0, 0), KLAMBDA: (1, -1, 0, 0), KMU: (1, 1, 0, 0), KPI: (1, 1, 0, 1), KPIP: (1, -1, 0, -1)}
SQRT2 = (0, 1, 0, -1)


def factor_pair(x, y):
    v = add(add(add((1, 0, 0, 0), wpow(x)), wpow(y)), tuple(-c for c in wpow(x + y)))
    if v == (0, 0, 0, 0):
        return (KZERO, 0, 0)
    for kind in (KNONE, KLAMBDA, KMU, KPI, KPIP):
        q = div(v, GEN[kind])
        if q is None:
            continue
        p = (1, 0, 0, 0)
        for e in range(7):
            for j in range(8):
                if mul(p, wpow(j)) == q:
                    return (kind, j, e)
            p = mul(p, SQRT2)
    raise AssertionError((x, y))


def slice_op(op):
    """(jbase, w[4], zero_tt, lam_tt, pi_tt, pip_tt, lm) -- mirrors pzx_classes.h."""
    if op >= 128:
        return (0, [0, 0, 0, 0], 0, 0, 0, 0, 0)
    cls, single = op >> 1, op & 1
    ka, kb = cls >> 3, cls & 7
    reach = [True, True, not single, not single]
    var = [factor_pair(ka + 4 * (v & 1), kb + 4 * (v >> 1)) for v in range(4)]
    first = next((v for v in range(4) if reach[v] and var[v][0] != KZERO), None)
    jbase = var[first][1] if first is not None else 0
    w = [0, 0, 0, 0]
    z = lam = pi = pip = lm = 0
    for v in range(4):
        if not reach[v]:
            continue
        k = var[v][0]
        if k == KZERO:
            z |= 1 << v
            continue
        w[v] = (var[v][1] - jbase) % 8
        if k == KLAMBDA:
            lam |= 1 << v
        if k == KPI:
            pi |= 1 << v
        if k == KPIP:
            pip |= 1 << v
        if k in (KLAMBDA, KMU):
            lm = 1
    return (jbase, w, z, lam, pi, pip, lm)


# -------------------------------------------------------- LOP3 immediates ----
def tt_bit(f, p, q):
    return (f >> (p | (q << 1))) & 1


def imm(fn):
    """lop3 immLut of fn(a, b, c) with a = 0xF0, b = 0xCC, c = 0xAA."""
    r = 0
    for i in range(8):
        r |= (fn((i >> 2) & 1, (i >> 1) & 1, i & 1) & 1) << i
    return r


def imm_f(f):            # f(b = X, c = Y)
    return imm(lambda a, b, c: tt_bit(f, b, c))


def imm_af(f, op):       # a OP f(b = X, c = Y)
    ops = {"and": lambda x, y: x & y, "xor": lambda x, y: x ^ y, "or": lambda x, y: x | y}
    return imm(lambda a, b, c: ops[op](a, tt_bit(f, b, c)))


def imm_fxc(f):          # f(a = X, b = Y) ^ c
    return imm(lambda a, b, c: tt_bit(f, a, b) ^ c)


MAJ, XOR3 = 0xE8, 0x96

# operands: %0 J0, %1 J1, %2 J2, %3 Z, %4 vl, %5 vpi, %6 vpip, %7 X, %8 op,
#           %9 phi, %10 Walsh32(phi), %11 base_lo [, %12 phi_hi, %13 base_hi]
# Double-parity cases compute Y = Walsh32(phi) ^ -parity(phi & base) into the
# local register yy themselves; single-parity cases never read it (their
# truth tables are made independent of the q input).


def _single_tables(op):
    """Truth tables of single-parity ops copied from the q = 0 column to q = 1."""
    jb, w, z, lam, pi, pip, lm = slice_op(op)
    if op < 128 and (op & 1):
        w = [w[0], w[1], w[0], w[1]]
        dup = lambda t: (t & 3) | ((t & 3) << 2)  # noqa: E731
        z, lam, pi, pip = dup(z), dup(lam), dup(pi), dup(pip)
    return jb, w, z, lam, pi, pip, lm


def case_body(op, p64=False, y_in=False):
    """y_in: Y arrives as operand %9 (random-batch kernel) instead of being formed here."""
    _, w, z, lam, pi, pip, _ = _single_tables(op)
    t = [sum(((w[v] >> b) & 1) << v for v in range(4)) for b in range(3)]
    L = []
    double = op < 128 and not (op & 1)
    Y = ("%9" if y_in else "yy") if double else "%7"
    if double and not y_in and (any(t) or bool(z | lam | pi | pip)):
        if p64:
            L.append("and.b32 yy, %9, %11;")
            L.append("and.b32 c0, %12, %13;")
            L.append("xor.b32 yy, yy, c0;")
        else:
            L.append("and.b32 yy, %9, %11;")
        L.append("popc.b32 yy, yy;")
        L.append("and.b32 yy, yy, 1;")
        L.append("neg.s32 yy, yy;")
        L.append("xor.b32 yy, yy, %10;")
    c0 = c1 = False
    if t[0]:
        L.append(f"lop3.b32 c0, %0, %7, {Y}, {imm_af(t[0], 'and'):#04x};")
        L.append(f"lop3.b32 %0, %0, %7, {Y}, {imm_af(t[0], 'xor'):#04x};")
        c0 = True
    if t[1] and c0:
        L.append(f"lop3.b32 w1, %7, %7, {Y}, {imm_f(t[1]):#04x};")
        L.append(f"lop3.b32 c1, %1, w1, c0, {MAJ:#04x};")
        L.append(f"lop3.b32 %1, %1, w1, c0, {XOR3:#04x};")
        c1 = True
    elif t[1]:
        L.append(f"lop3.b32 c1, %1, %7, {Y}, {imm_af(t[1], 'and'):#04x};")
        L.append(f"lop3.b32 %1, %1, %7, {Y}, {imm_af(t[1], 'xor'):#04x};")
        c1 = True
    elif c0:
        L.append("and.b32 c1, %1, c0;")
        L.append("xor.b32 %1, %1, c0;")
        c1 = True
    if t[2] and c1:
        L.append(f"lop3.b32 w1, %7, {Y}, c1, {imm_fxc(t[2]):#04x};")
        L.append("xor.b32 %2, %2, w1;")
    elif t[2]:
        L.append(f"lop3.b32 %2, %2, %7, {Y}, {imm_af(t[2], 'xor'):#04x};")
    elif c1:
        L.append("xor.b32 %2, %2, c1;")
    if z:
        L.append(f"lop3.b32 %3, %3, %7, {Y}, {imm_af(z, 'or'):#04x};")
    if lam:
        L.append(f"lop3.b32 %4, %7, %7, {Y}, {imm_f(lam):#04x};")
    if pi:
        L.append(f"lop3.b32 %5, %7, %7, {Y}, {imm_f(pi):#04x};")
    if pip:
        L.append(f"lop3.b32 %6, %7, %7, {Y}, {imm_f(pip):#04x};")
    return L


def _rename(line, mp):
    """Substitute operand / temp names (whole tokens) in one PTX line."""
    import re
    return re.sub(r"%\d+|\b(?:c0|c1|w1|yy)\b", lambda m: mp.get(m.group(0), m.group(0)), line)


# two-slice variant: 64 assignments per thread, slices a and b share X/Y-free
# row data and the jump; operands
#   %0-%3 J0 J1 J2 Z (a), %4-%7 (b), %8-%10 vl vpi vpip (a), %11-%13 (b),
#   %14 Xa, %15 Ya, %16 Xb, %17 Yb, %18 op
_DUAL_A = {"%4": "%8", "%5": "%9", "%6": "%10", "%7": "%14", "%9": "%15"}
_DUAL_B = {"%0": "%4", "%1": "%5", "%2": "%6", "%3": "%7", "%4": "%11", "%5": "%12", "%6": "%13",
           "%7": "%16", "%9": "%17", "c0": "d0", "c1": "d1", "w1": "x1"}


def case_body_dual(op):
    a = [_rename(ln, _DUAL_A) for ln in case_body(op, False, True)]
    b = [_rename(ln, _DUAL_B) for ln in case_body(op, False, True)]
    out = []
    for i in range(max(len(a), len(b))):  # interleave the two independent chains
        if i < len(a):
            out.append(a[i])
        if i < len(b):
            out.append(b[i])
    return out


# ------------------------------------------------------- fused row loop ----
# The whole plain-row loop of the enumerated bit-sliced kernel as one inline
# PTX block: per row, the head forms X / Y (AND + POPC + predicate + SEL on
# the row's Walsh / ~Walsh words; P64: XOR form), tests the row's kind / end
# flags, advances, prefetches the next row into the same registers and jumps
# (BRX) into the class body, which ends with ONE branch straight back to the
# head -- two taken branches per row instead of four. The block returns to
# C++ after a flagged row (bumps / epilogue) or at the tile end.
# operands (outputs first, as inline asm numbers them):
#   %0 ad (in/out), %1-%4 J0 J1 J2 Z, %5-%7 vl vpi vpip (out), %8 code of the
#   last row (out), %9-%16 row registers r0..r7 (in/out: current row in, next
#   row out), %17 aend, %18 blo, %19 bhi
_LOOP_MAP = {"%0": "%1", "%1": "%2", "%2": "%3", "%3": "%4", "%4": "%5", "%5": "%6", "%6": "%7",
             "%7": "xx", "%9": "yv"}
ROW_FLAG_MASK = (1 << 8) | (1 << 9) | (1 << 10) | (1 << 31)


def _loop_block(name, p64):
    n = 129
    bodies, label_of = {}, []
    for i in range(n):
        key = tuple(_rename(ln, _LOOP_MAP) for ln in case_body(i, False, True))
        if key not in bodies:
            bodies[key] = len(bodies)
        label_of.append(bodies[key])
    b = ["{", ".reg .b32 c0, c1, w1, yy, xx, yv, tq, opi, nc;", ".reg .pred q1, q2, pl, mo, cont;",
         "ts%=: .branchtargets " + ", ".join(f"L{label_of[i]}_%=" for i in range(n)) + ";",
         "H%=:",
         # the next row's code word first: its consumer (the next head's flag
         # test, which the compiler runs on the uniform datapath) then waits on
         # a load issued a whole head earlier
         "ld.shared.u32 nc, [%0+40];"]
    if p64:  # rows {psi, phi, code, W(psi)}, {W(phi), psi_hi, phi_hi, op}
        b += ["and.b32 tq, %9, %18;", "and.b32 c0, %14, %19;", "xor.b32 tq, tq, c0;", "popc.b32 tq, tq;",
              "and.b32 tq, tq, 1;", "neg.s32 tq, tq;", "xor.b32 xx, %12, tq;",
              "and.b32 tq, %10, %18;", "and.b32 c0, %15, %19;", "xor.b32 tq, tq, c0;", "popc.b32 tq, tq;",
              "and.b32 tq, tq, 1;", "neg.s32 tq, tq;", "xor.b32 yv, %13, tq;"]
    else:    # rows {psi, phi, code, W(psi)}, {W(phi), ~W(psi), ~W(phi), op}
        b += ["and.b32 tq, %9, %18;", "popc.b32 tq, tq;", "and.b32 tq, tq, 1;", "setp.ne.b32 q1, tq, 0;",
              "selp.b32 xx, %14, %12, q1;",
              "and.b32 tq, %10, %18;", "popc.b32 tq, tq;", "and.b32 tq, tq, 1;", "setp.ne.b32 q2, tq, 0;",
              "selp.b32 yv, %15, %13, q2;"]
    b += ["mov.b32 opi, %16;", "mov.b32 %8, %11;",
          f"and.b32 tq, %11, {ROW_FLAG_MASK:#x};", "setp.eq.b32 pl, tq, 0;",
          "add.u32 %0, %0, 32;", "setp.lt.u32 mo, %0, %17;", "and.pred cont, pl, mo;",
          "ld.shared.v4.u32 {%9, %10, %11, %12}, [%0];", "ld.shared.v4.u32 {%13, %14, %15, %16}, [%0+16];",
          "mov.b32 %11, nc;",
          "brx.idx.uni opi, ts%=;"]
    for key, lab in sorted(bodies.items(), key=lambda kv: kv[1]):
        b.append(f"L{lab}_%=:")
        b.extend(key)
        b.append("@cont bra.uni H%=;")
        b.append("bra.uni X%=;")
    b += ["X%=:", "}"]
    lines = [f"#define {name} \\"] + [f'    "{x}\\n" \\' for x in b] + [""]
    return lines


# sorted-batch kernel's fused loop. Rows {psi, phi, code, op}, {psi offsets
# 0|1, 2|3, phi offsets 0|1, 2|3} (16-bit byte offsets into the thread's
# Four-Russians tables); X = XOR of G table words (groups 4.. computed from
# the mask) ^ -parity(psi & H0): the host regroups the sorted words so that a
# thread's 32 words share their high part H0. Y likewise, its loads
# predicated off for one-parity rows (phi == 0 -> Y = 0).
# operands: %0 ad, %1-%4 J0 J1 J2 Z, %5-%7 vl vpi vpip, %8 code (out),
#   %9-%16 row registers, %17 aend, %18 tab (this thread's table address), %19 H0
def _sorted_par(out, mask, o01, o23, G, pred=None, shift=9):
    """X = XOR of the G table words ^ -parity(mask & H0); the row carries the
    byte offsets (k * 16 + nibble_k) * 512 of groups 0..3 (128-thread tables),
    shifted once more for 256-thread CTAs (shift = log2(4 x CTA threads))."""
    pp = f"@{pred} " if pred else ""
    L = []
    for i, (src, sh) in enumerate(((o01, False), (o01, True), (o23, False), (o23, True))):
        L.append(f"{'shr.b32' if sh else 'and.b32'} ta, {src}, {'16' if sh else '0xFFFF'};")
        if shift > 9:  # the row's byte offsets assume 128-thread tables
            L.append(f"shl.b32 ta, ta, {shift - 9};")
        L.append("add.u32 ta, ta, %18;")
        L.append(f"{pp}ld.shared.u32 t{i}, [ta];")
    for k in range(4, G):
        L.append(f"shr.b32 ta, {mask}, {4 * k};")
        L.append("and.b32 ta, ta, 15;")
        L.append(f"shl.b32 ta, ta, {shift};")
        L.append("add.u32 ta, ta, %18;")
        L.append(f"{pp}ld.shared.u32 t{k}, [ta+{16 * k << shift}];")
    L.append(f"and.b32 ta, {mask}, %19;")
    L.append("popc.b32 ta, ta;")
    L.append("and.b32 ta, ta, 1;")
    L.append("neg.s32 ta, ta;")
    for i in range(G):
        L.append(f"xor.b32 ta, ta, t{i};")
    L.append(f"mov.b32 {out}, ta;" if not pred else f"selp.b32 {out}, ta, 0, {pred};")
    return L


def _sorted_loop_block(name, G, shift=9):
    n = 129
    bodies, label_of = {}, []
    for i in range(n):
        key = tuple(_rename(ln, _LOOP_MAP) for ln in case_body(i, False, True))
        if key not in bodies:
            bodies[key] = len(bodies)
        label_of.append(bodies[key])
    regs = ", ".join(f"t{i}" for i in range(G))
    b = ["{", f".reg .b32 c0, c1, w1, yy, xx, yv, tq, opi, ta, {regs};",
         ".reg .pred pl, mo, cont, hp;",
         "ts%=: .branchtargets " + ", ".join(f"L{label_of[i]}_%=" for i in range(n)) + ";",
         "H%=:"]
    b += _sorted_par("xx", "%9", "%13", "%14", G, shift=shift)
    # one-parity rows (phi == 0, ~40 %) jump over the Y lookups (a uniform branch)
    b += ["setp.eq.b32 hp, %10, 0;", "mov.b32 yv, 0;", "@hp bra.uni NY%=;"]
    b += _sorted_par("yv", "%10", "%15", "%16", G, shift=shift)
    b += ["NY%=:"]
    b += ["mov.b32 opi, %12;", "mov.b32 %8, %11;",
          f"and.b32 tq, %11, {ROW_FLAG_MASK:#x};", "setp.eq.b32 pl, tq, 0;",
          "add.u32 %0, %0, 32;", "setp.lt.u32 mo, %0, %17;", "and.pred cont, pl, mo;",
          "ld.shared.v4.u32 {%9, %10, %11, %12}, [%0];", "ld.shared.v4.u32 {%13, %14, %15, %16}, [%0+16];",
          "brx.idx.uni opi, ts%=;"]
    for key, lab in sorted(bodies.items(), key=lambda kv: kv[1]):
        b.append(f"L{lab}_%=:")
        b.extend(key)
        b.append("@cont bra.uni H%=;")
        b.append("bra.uni X%=;")
    b += ["X%=:", "}"]
    return [f"#define {name} \\"] + [f'    "{x}\\n" \\' for x in b] + [""]


def kind_flags(op):
    """Row code-word flag bits the C++ side reads: bit 8 lambda, 9 pi, 10 pi'."""
    _, _, _, lam, pi, pip, _ = slice_op(op)
    return (1 << 8 if lam else 0) | (1 << 9 if pi else 0) | (1 << 10 if pip else 0)


def _asm_block(name, p64, y_in=False, dual=False):
    n = 129
    # identical case bodies share one label (smaller code, fewer I-cache misses)
    bodies, label_of = {}, []
    for i in range(n):
        key = tuple(case_body_dual(i) if dual else case_body(i, p64, y_in))
        if key not in bodies:
            bodies[key] = len(bodies)
        label_of.append(bodies[key])
    lines = [f"#define {name} \\"]
    body = ["{", ".reg .b32 c0, c1, w1, yy, d0, d1, x1;" if dual else ".reg .b32 c0, c1, w1, yy;",
            "ts%=: .branchtargets " + ", ".join(f"L{label_of[i]}_%=" for i in range(n)) + ";",
            f"brx.idx.uni {'%18' if dual else '%8'}, ts%=;"]
    for key, lab in sorted(bodies.items(), key=lambda kv: kv[1]):
        body.append(f"L{lab}_%=:")
        body.extend(key)
        body.append("bra.uni D%=;")
    body.append("D%=:")
    body.append("}")
    for b in body:
        lines.append(f'    "{b}\\n" \\')
    lines.append("")
    return lines, len(bodies)


def generate() -> str:
    n = 129
    lines = ["// GENERATED by paper_2403_06777_b200/gen_slice_ops.py -- do not edit.",
             "// Bit-sliced per-row update, one jump-table dispatch (brx.idx) per row.",
             "// operands: %0 J0, %1 J1, %2 J2, %3 Z, %4 vl, %5 vpi, %6 vpip, %7 X, %8 op,",
             "//           %9 phi, %10 Walsh32(phi), %11 base_lo [, %12 phi_hi, %13 base_hi]"]
    b32, n32 = _asm_block("PZX_SLICE_DISPATCH_ASM_P32", False)
    b64, _ = _asm_block("PZX_SLICE_DISPATCH_ASM_P64", True)
    bxy, _ = _asm_block("PZX_SLICE_DISPATCH_ASM_XY", False, True)
    bxy2, _ = _asm_block("PZX_SLICE_DISPATCH_ASM_XY2", False, True, dual=True)
    lines += [f"// {n32} distinct case bodies",
              "// _XY variant: operand %9 is Y itself",
              "// _XY2 variant (two slices): %0-%3 J0 J1 J2 Z (a), %4-%7 (b), %8-%10 vl vpi vpip (a),",
              "//   %11-%13 (b), %14 Xa, %15 Ya, %16 Xb, %17 Yb, %18 op"] + b32 + b64 + bxy + bxy2
    lines += ["// fused plain-row loop (enumerated kernel): %0 ad, %1-%4 J0 J1 J2 Z, %5-%7 vl vpi vpip,",
              "//   %8 code (out), %9-%16 row registers, %17 aend, %18 blo, %19 bhi"]
    lines += _loop_block("PZX_SLICE_ROWLOOP_P32", False) + _loop_block("PZX_SLICE_ROWLOOP_P64", True)
    lines += ["// fused loop of the sorted-batch kernel (G = 4 / 6 table groups): %0 ad, %1-%4 J0 J1 J2 Z,",
              "//   %5-%7 vl vpi vpip, %8 code, %9-%16 row registers, %17 aend, %18 table, %19 H0"]
    # table rows are 4 B x CTA threads apart: 128 threads -> shift 9, 256 -> 10
    lines += (_sorted_loop_block("PZX_SORTED_ROWLOOP_G4", 4, 9) + _sorted_loop_block("PZX_SORTED_ROWLOOP_G6", 6, 9) +
              _sorted_loop_block("PZX_SORTED_ROWLOOP_G6_256", 6, 10))
    lines.append("// per-op row code-word flags (bit 8 lambda, 9 pi, 10 pi')")
    lines.append("#define PZX_SLICE_KIND_FLAGS { " + ", ".join(str(kind_flags(i)) for i in range(n)) + " }")
    lines.append("#define PZX_SLICE_JBASE { " + ", ".join(str(slice_op(i)[0]) for i in range(n)) + " }")
    return "\n".join(lines) + "\n"


def main() -> str:
    text = generate()
    old = open(OUT).read() if os.path.exists(OUT) else None
    if old != text:
        with open(OUT, "w") as f:
            f.write(text)
    return OUT


if __name__ == "__main__":
    print(main())
