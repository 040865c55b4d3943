"""Exact arithmetic in Z[w][1/2], w = e^{i pi/4} (test helper, Python ints).

Used to turn the GPU's per-term exponent codes (pzx_debug_term_codes) back
into exact values and compare them bit-for-bit with the oracle's RingQuads.
"""
from __future__ import annotations


class ZQ:
    """(c0 + c1 w + c2 w^2 + c3 w^3) / 2^s, with w^4 = -1."""

    __slots__ = ("c", "s")

    def __init__(self, c, s=0):
        c = [int(x) for x in c]
        s = int(s)
        while s > 0 and all(x % 2 == 0 for x in c):
            c = [x // 2 for x in c]
            s -= 1
        while s < 0:
            c = [2 * x for x in c]
            s += 1
        if not any(c):
            s = 0
        self.c, self.s = tuple(c), s

    @staticmethod
    def from_quad(q):
        """RingQuad (a + b sqrt2 + i(c + d sqrt2)) / 2^e; sqrt2 = w - w^3, i = w^2."""
        a, b, c, d, e = (int(x) for x in q)
        return ZQ((a, b + d, c, d - b), e)

    @staticmethod
    def w(k):
        k %= 8
        c = [0, 0, 0, 0]
        if k < 4:
            c[k] = 1
        else:
            c[k - 4] = -1
        return ZQ(c)

    def __mul__(self, o):
        t = [0] * 8
        for i in range(4):
            for j in range(4):
                t[i + j] += self.c[i] * o.c[j]
        return ZQ([t[i] - t[i + 4] for i in range(4)], self.s + o.s)

    def __add__(self, o):
        s = max(self.s, o.s)
        return ZQ([x * 2 ** (s - self.s) + y * 2 ** (s - o.s) for x, y in zip(self.c, o.c)], s)

    def __pow__(self, n):
        r = ZQ((1, 0, 0, 0))
        for _ in range(n):
            r = r * self
        return r

    def __eq__(self, o):
        return self.c == o.c and self.s == o.s

    def __repr__(self):
        return f"ZQ({self.c}, /2^{self.s})"

    def to_complex(self):
        import cmath
        w = cmath.exp(1j * cmath.pi / 4)
        return sum(x * w**i for i, x in enumerate(self.c)) / 2**self.s


ONE = ZQ((1, 0, 0, 0))
SQRT2 = ZQ((0, 1, 0, -1))
LAMBDA = ZQ((1, -1, 0, 0))
MU = ZQ((1, 1, 0, 0))
PI = ZQ((1, 1, 0, 1))
PIP = ZQ((1, -1, 0, -1))
ZERO = ZQ((0, 0, 0, 0))


def pair_value(x, y):
    """V(x, y) = 1 + w^x + w^y - w^(x+y)."""
    return ONE + ZQ.w(x) + ZQ.w(y) + ZQ.w(x + y) * ZQ((-1, 0, 0, 0))


def term_from_code(coef, e_sqrt2, n_lm, j, z, s1, a, b):
    """Exact product the kernel encodes (include/pzx_gpu.h pzx_term_code)."""
    if z:
        return ZERO
    return (ZQ.from_quad(coef) * SQRT2 ** e_sqrt2 * ZQ.w(j) * LAMBDA ** s1 * MU ** (n_lm - s1)
            * PI ** a * PIP ** b)
