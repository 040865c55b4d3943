// pzx_math.hpp -- host-side exact arithmetic for the table compiler.
//
// Two number systems, both exact:
//   Quad : the reference's RingQuad value domain (ring.hpp:17-38),
//          (a + b*sqrt2 + i(c + d*sqrt2)) / 2^e, int64 coefficients, the same
//          canonical form (ring.cpp:20-48) so folded constants compare
//          bit-for-bit with the reference.
//   Zw   : the cyclotomic integers Z[w], w = e^{i pi/4}, in the power basis
//          (1, w, w^2, w^3) with w^4 = -1. Every row value of the paper's
//          phase-pair subterm, V(x,y) = 1 + w^x + w^y - w^(x+y) (P:164-198,
//          subterm.cpp:23-27), is 0 or  w^j * sqrt2^e * g  with
//          g in {1, lambda=1-w, mu=1+w, pi=1+w+w^3, pi'=1-w-w^3}
//          (Z[w] is a UFD; 2 ramifies as (lambda)^4 and the norm-9 primes above
//          3 are pi, pi'). The factorisation is computed here, once, by exact
//          division -- see DESIGN.md §2.
// __float128 is used only to round derived constants (powers of units and
// primes) to the nearest double.
#pragma once

#include <cstdint>
#include <cstring>

namespace pzxb {

using i128 = __int128;
using f128 = __float128;

// ---------------------------------------------------------------- Quad ----
struct Quad {
    int64_t a = 0, b = 0, c = 0, d = 0;
    int32_t e = 0;
};

// canonical form of ring.cpp:20-48; returns false on int64 overflow.
inline bool quad_canon(i128 a, i128 b, i128 c, i128 d, int64_t e, Quad& out) {
    while (e < 0) {
        a *= 2; b *= 2; c *= 2; d *= 2; ++e;
        const i128 lim = i128(1) << 100;
        if (a > lim || a < -lim) return false;
    }
    if (a == 0 && b == 0 && c == 0 && d == 0) { out = Quad{}; return true; }
    while (e > 0 && ((a | b | c | d) & 1) == 0) { a /= 2; b /= 2; c /= 2; d /= 2; --e; }
    const i128 hi = INT64_MAX, lo = INT64_MIN;
    auto ok = [&](i128 v) { return v <= hi && v >= lo; };
    if (!ok(a) || !ok(b) || !ok(c) || !ok(d) || e > INT32_MAX) return false;
    out.a = int64_t(a); out.b = int64_t(b); out.c = int64_t(c); out.d = int64_t(d);
    out.e = int32_t(e);
    return true;
}

// product (Lemma 8); false on overflow
inline bool quad_mul(const Quad& x, const Quad& y, Quad& out) {
    const i128 re0 = i128(x.a) * y.a + 2 * i128(x.b) * y.b - i128(x.c) * y.c - 2 * i128(x.d) * y.d;
    const i128 re1 = i128(x.a) * y.b + i128(x.b) * y.a - i128(x.c) * y.d - i128(x.d) * y.c;
    const i128 im0 = i128(x.a) * y.c + 2 * i128(x.b) * y.d + i128(x.c) * y.a + 2 * i128(x.d) * y.b;
    const i128 im1 = i128(x.a) * y.d + i128(x.b) * y.c + i128(x.c) * y.b + i128(x.d) * y.a;
    return quad_canon(re0, re1, im0, im1, int64_t(x.e) + y.e, out);
}

inline f128 f128_sqrt2() { return 1.41421356237309504880168872420969807857Q; }

inline void quad_to_f128(const Quad& q, f128& re, f128& im) {
    f128 scale = 1;
    for (int i = 0; i < q.e; ++i) scale /= 2;
    re = (f128(q.a) + f128(q.b) * f128_sqrt2()) * scale;
    im = (f128(q.c) + f128(q.d) * f128_sqrt2()) * scale;
}

// ------------------------------------------------------------------ Zw ----
struct Zw {
    int64_t c[4] = {0, 0, 0, 0};
    bool zero() const { return !c[0] && !c[1] && !c[2] && !c[3]; }
    bool operator==(const Zw& o) const { return !std::memcmp(c, o.c, sizeof c); }
};

inline Zw zw(int64_t a, int64_t b, int64_t c, int64_t d) { Zw z; z.c[0] = a; z.c[1] = b; z.c[2] = c; z.c[3] = d; return z; }

inline Zw zw_pow_w(int k) {           // w^k
    k &= 7;
    Zw z;
    if (k < 4) z.c[k] = 1; else z.c[k - 4] = -1;
    return z;
}
inline Zw zw_add(const Zw& x, const Zw& y) { Zw r; for (int i = 0; i < 4; ++i) r.c[i] = x.c[i] + y.c[i]; return r; }
inline Zw zw_sub(const Zw& x, const Zw& y) { Zw r; for (int i = 0; i < 4; ++i) r.c[i] = x.c[i] - y.c[i]; return r; }
inline Zw zw_mul(const Zw& x, const Zw& y) {
    int64_t t[8] = {0};
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) t[i + j] += x.c[i] * y.c[j];
    Zw r;
    for (int i = 0; i < 4; ++i) r.c[i] = t[i] - t[i + 4];
    return r;
}
// Galois automorphism w -> w^s (s odd)
inline Zw zw_sigma(const Zw& x, int s) {
    Zw r;
    for (int i = 0; i < 4; ++i) {
        Zw t = zw_pow_w(s * i);
        for (int k = 0; k < 4; ++k) r.c[k] += x.c[i] * t.c[k];
    }
    return r;
}
inline int64_t zw_norm(const Zw& x) {  // absolute norm, an integer
    Zw p = zw_mul(zw_mul(x, zw_sigma(x, 3)), zw_mul(zw_sigma(x, 5), zw_sigma(x, 7)));
    return p.c[0];
}
// exact division; false when y does not divide x in Z[w]
inline bool zw_div(const Zw& x, const Zw& y, Zw& q) {
    const Zw co = zw_mul(zw_mul(zw_sigma(y, 3), zw_sigma(y, 5)), zw_sigma(y, 7));
    const int64_t n = zw_norm(y);
    const Zw t = zw_mul(x, co);
    for (int i = 0; i < 4; ++i)
        if (t.c[i] % n) return false;
    for (int i = 0; i < 4; ++i) q.c[i] = t.c[i] / n;
    return true;
}
// Z[w] -> RingQuad: w = (sqrt2/2)(1+i), w^3 = (sqrt2/2)(-1+i)
inline bool zw_to_quad(const Zw& z, Quad& out) {
    return quad_canon(i128(2) * z.c[0], i128(z.c[1]) - z.c[3], i128(2) * z.c[2],
                      i128(z.c[1]) + z.c[3], 1, out);
}
// V(x, y) = 1 + w^x + w^y - w^(x+y)   (phase_pair_value, subterm.cpp:23-27)
inline Zw zw_pair_value(int x, int y) {
    return zw_sub(zw_add(zw_add(zw(1, 0, 0, 0), zw_pow_w(x)), zw_pow_w(y)), zw_pow_w(x + y));
}

// Factor kinds.
enum Kind : int { K_NONE = 0, K_LAMBDA = 1, K_MU = 2, K_PI = 3, K_PIP = 4, K_ZERO = 5 };

inline Zw zw_generator(int kind) {
    switch (kind) {
    case K_LAMBDA: return zw(1, -1, 0, 0);
    case K_MU: return zw(1, 1, 0, 0);
    case K_PI: return zw(1, 1, 0, 1);
    case K_PIP: return zw(1, -1, 0, -1);
    default: return zw(1, 0, 0, 0);
    }
}

struct Factor { int kind, j, e; };

// v = w^j * sqrt2^e * generator(kind), or kind = K_ZERO
inline bool zw_factor(const Zw& v, Factor& f) {
    if (v.zero()) { f = {K_ZERO, 0, 0}; return true; }
    const Zw s2 = zw(0, 1, 0, -1);  // sqrt2 = w - w^3
    for (int kind = K_NONE; kind <= K_PIP; ++kind) {
        Zw q;
        if (!zw_div(v, zw_generator(kind), q)) continue;
        Zw p = zw(1, 0, 0, 0);
        for (int e = 0; e <= 6; ++e) {
            for (int j = 0; j < 8; ++j)
                if (zw_mul(p, zw_pow_w(j)) == q) { f = {kind, j, e}; return true; }
            p = zw_mul(p, s2);
        }
    }
    return false;
}

// --------------------------------------------------------- f128 complex ----
struct C128 { f128 re = 0, im = 0; };
inline C128 cmul(const C128& x, const C128& y) { return {x.re * y.re - x.im * y.im, x.re * y.im + x.im * y.re}; }
inline C128 zw_to_c128(const Zw& z) {
    const f128 h = f128_sqrt2() / 2;
    return {f128(z.c[0]) + h * f128(z.c[1]) - h * f128(z.c[3]),
            f128(z.c[2]) + h * f128(z.c[1]) + h * f128(z.c[3])};
}

}  // namespace pzxb
