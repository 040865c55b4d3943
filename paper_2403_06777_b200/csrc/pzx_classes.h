// pzx_classes.h -- compile-time (constexpr, host + device) factorisation of the
// 64 phase-pair row classes, and the per-row "slice ops" of the bit-sliced
// kernel. DESIGN.md §2 explains the algebra; pzx_math.hpp holds the runtime
// twin used by the table compiler, and tests compare the two.
//
// Row class (ka, kb): value at parities (p, q) is V(ka + 4p, kb + 4q) =
//   0  or  w^j * sqrt2^e * g,  g in {1, lambda, mu, pi, pi'}.
// A slice op is a class plus whether the row has one parity (q == 0) or two.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define PZX_HD __host__ __device__
#else
#define PZX_HD
#endif

namespace pzxb {
namespace cx {

struct Z4 {
    long long c[4];
};

PZX_HD constexpr Z4 z4(long long a, long long b, long long c, long long d) { return Z4{{a, b, c, d}}; }

PZX_HD constexpr Z4 wpow(int k) {
    k &= 7;
    Z4 z = z4(0, 0, 0, 0);
    if (k < 4) z.c[k] = 1;
    else z.c[k - 4] = -1;
    return z;
}

PZX_HD constexpr Z4 add(Z4 x, Z4 y) { return z4(x.c[0] + y.c[0], x.c[1] + y.c[1], x.c[2] + y.c[2], x.c[3] + y.c[3]); }
PZX_HD constexpr Z4 sub(Z4 x, Z4 y) { return z4(x.c[0] - y.c[0], x.c[1] - y.c[1], x.c[2] - y.c[2], x.c[3] - y.c[3]); }

PZX_HD constexpr Z4 mul(Z4 x, Z4 y) {
    long long t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) t[i + j] += x.c[i] * y.c[j];
    return z4(t[0] - t[4], t[1] - t[5], t[2] - t[6], t[3] - t[7]);
}

PZX_HD constexpr Z4 sigma(Z4 x, int s) {
    Z4 r = z4(0, 0, 0, 0);
    for (int i = 0; i < 4; ++i) {
        const Z4 t = wpow(s * i);
        for (int k = 0; k < 4; ++k) r.c[k] += x.c[i] * t.c[k];
    }
    return r;
}

PZX_HD constexpr long long norm(Z4 x) { return mul(mul(x, sigma(x, 3)), mul(sigma(x, 5), sigma(x, 7))).c[0]; }

PZX_HD constexpr bool divides(Z4 x, Z4 y, Z4& q) {
    const Z4 co = mul(mul(sigma(y, 3), sigma(y, 5)), sigma(y, 7));
    const long long n = norm(y);
    const Z4 t = mul(x, co);
    for (int i = 0; i < 4; ++i)
        if (t.c[i] % n) return false;
    q = z4(t.c[0] / n, t.c[1] / n, t.c[2] / n, t.c[3] / n);
    return true;
}

PZX_HD constexpr bool eq(Z4 x, Z4 y) {
    return x.c[0] == y.c[0] && x.c[1] == y.c[1] && x.c[2] == y.c[2] && x.c[3] == y.c[3];
}

enum { KNONE = 0, KLAMBDA = 1, KMU = 2, KPI = 3, KPIP = 4, KZERO = 5 };

PZX_HD constexpr Z4 generator(int kind) {
    return kind == KLAMBDA ? z4(1, -1, 0, 0)
         : kind == KMU     ? z4(1, 1, 0, 0)
         : kind == KPI     ? z4(1, 1, 0, 1)
         : kind == KPIP    ? z4(1, -1, 0, -1)
                           : z4(1, 0, 0, 0);
}

struct Var {
    int kind, j, e;
};

// V(x, y) = 1 + w^x + w^y - w^(x+y) factored as w^j sqrt2^e g
PZX_HD constexpr Var factor_pair(int x, int y) {
    const Z4 v = sub(add(add(z4(1, 0, 0, 0), wpow(x)), wpow(y)), wpow(x + y));
    if (v.c[0] == 0 && v.c[1] == 0 && v.c[2] == 0 && v.c[3] == 0) return Var{KZERO, 0, 0};
    const Z4 s2 = z4(0, 1, 0, -1);
    for (int kind = KNONE; kind <= KPIP; ++kind) {
        Z4 q = z4(0, 0, 0, 0);
        if (!divides(v, generator(kind), q)) continue;
        Z4 p = z4(1, 0, 0, 0);
        for (int e = 0; e <= 6; ++e) {
            for (int j = 0; j < 8; ++j)
                if (eq(mul(p, wpow(j)), q)) return Var{kind, j, e};
            p = mul(p, s2);
        }
    }
    return Var{-1, 0, 0};
}

}  // namespace cx

// ---------------------------------------------------------------- slice ops --
constexpr int kSliceOps = 129;    // op = cls * 2 + single, 128 = unit (row-less term)
constexpr int kSliceUnitOp = 128;
// slice row code word: op (bits 0..7) | kind flags | kEndFlag (bit 31)
constexpr uint32_t kSliceLamFlag = 1u << 8;
constexpr uint32_t kSlicePiFlag = 1u << 9;
constexpr uint32_t kSlicePipFlag = 1u << 10;

// Truth tables are 4-bit, indexed by v = p | (q << 1).
struct SliceOp {
    int jbase;    // j of the first nonzero reachable variant (folded into the term constant)
    int w[4];     // (j(v) - jbase) mod 8 for nonzero reachable variants, else 0
    int zero_tt;  // variant is zero
    int lam_tt;   // variant carries lambda (class is a lambda/mu class)
    int pi_tt;    // variant carries pi
    int pip_tt;   // variant carries pi'
    int lm;       // class is a lambda/mu class (every nonzero variant is lambda or mu)
};

PZX_HD constexpr SliceOp slice_op(int op) {
    SliceOp s{0, {0, 0, 0, 0}, 0, 0, 0, 0, 0};
    if (op >= kSliceUnitOp) return s;
    const int cls = op >> 1, single = op & 1;
    const int ka = cls >> 3, kb = cls & 7;
    cx::Var var[4] = {cx::Var{0, 0, 0}, cx::Var{0, 0, 0}, cx::Var{0, 0, 0}, cx::Var{0, 0, 0}};
    bool reach[4] = {true, true, !single, !single};
    int first = -1;
    for (int v = 0; v < 4; ++v) {
        var[v] = cx::factor_pair(ka + 4 * (v & 1), kb + 4 * (v >> 1));
        if (reach[v] && var[v].kind != cx::KZERO && first < 0) first = v;
    }
    s.jbase = first >= 0 ? var[first].j : 0;
    for (int v = 0; v < 4; ++v) {
        if (!reach[v]) continue;
        const int k = var[v].kind;
        if (k == cx::KZERO) { s.zero_tt |= 1 << v; continue; }
        s.w[v] = (var[v].j - s.jbase) & 7;
        if (k == cx::KLAMBDA) s.lam_tt |= 1 << v;
        if (k == cx::KPI) s.pi_tt |= 1 << v;
        if (k == cx::KPIP) s.pip_tt |= 1 << v;
        if (k == cx::KLAMBDA || k == cx::KMU) s.lm = 1;
    }
    return s;
}

}  // namespace pzxb
