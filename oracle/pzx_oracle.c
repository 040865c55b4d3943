/*
 * pzx_oracle.c -- CPU ORACLE (test infrastructure, NOT product code).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load this library, and only as the checker or the timed CPU
 * baseline. The product path (paper_2403_06777_b200/) never links it.
 *
 * What it is: a plain-C restatement of the reference's exact evaluator for the
 * parametric scalar  S(a) = sum_i C_i * prod_j S_ij(a)  as the reference's own
 * API composes it:
 *
 *   for each assignment a:            ParamAssignment::total   phase.hpp:18-23
 *     total = 0
 *     for each leaf term i:           instantiate_diagram      diagram.cpp:149-165
 *       covers(used mask) else MissingParameter                diagram.cpp:150-152
 *       s = C_i   (constant FIRST)                             diagram.cpp:158
 *       for each pending subterm:     subterm_value            subterm.cpp:29-49
 *         s = ring_mul(s, value)                               diagram.cpp:160
 *     total = ring_add(total, s)      ring_add                 ring.cpp:57-70
 *   amplitude = to_complex(total)                              ring.cpp:131-136
 *
 * Every arithmetic primitive cites the reference function it restates. The
 * value domain is the reference's RingQuad (a + b*sqrt2 + i(c + d*sqrt2))/2^exp
 * with int64 coefficients, __int128 intermediates and the same canonical form,
 * so results are bit-identical to the reference whenever the reference does not
 * throw, and the same error class is reported when it does.
 *
 * Pinning: tests/test_oracle.py checks this restatement against (1) the SPEC
 * known-answer examples and the golden 8x8 pair table and
 * (2) the reference itself, compiled from /root/reference by oracle/Makefile
 * into oracle/_ref/ (fixtures committed under tests/golden/).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "pzx_oracle.h"

typedef __int128 i128;

/* ---- exact ring: ring.cpp ------------------------------------------------ */

/* canonical(): ring.cpp:20-48. Negative exponents are folded into the
 * coefficients (with the reference's overflow guard on `a` only, :25-30), zero
 * has exp 0 (:32-34), and common factors of two are divided out while exp > 0
 * (:35-38). Narrowing to int64 is checked (:13-18, :42-45). */
static int oq_canon(i128 a, i128 b, i128 c, i128 d, int64_t e, oq_quad* out) {
    const i128 lim = ((i128)1) << 100;
    while (e < 0) {
        a *= 2; b *= 2; c *= 2; d *= 2; ++e;
        if (a > lim || a < -lim) return OQ_E_OVERFLOW;
    }
    if (a == 0 && b == 0 && c == 0 && d == 0) {
        memset(out, 0, sizeof *out);
        return OQ_OK;
    }
    while (e > 0 && ((a | b | c | d) & 1) == 0) {
        a /= 2; b /= 2; c /= 2; d /= 2; --e;
    }
    if (e > INT32_MAX) return OQ_E_OVERFLOW;
    const i128 hi = (i128)INT64_MAX, lo = (i128)INT64_MIN;
    if (a > hi || a < lo || b > hi || b < lo || c > hi || c < lo || d > hi || d < lo)
        return OQ_E_OVERFLOW;
    out->a = (int64_t)a; out->b = (int64_t)b; out->c = (int64_t)c; out->d = (int64_t)d;
    out->exp = (int32_t)e;
    return OQ_OK;
}

int oq_make(int64_t a, int64_t b, int64_t c, int64_t d, int32_t e, oq_quad* out) {
    return oq_canon(a, b, c, d, e, out);      /* RingQuad::make ring.cpp:52-55 */
}

/* ring_add: ring.cpp:57-70 (exponent alignment, spread > 62 is an overflow). */
int oq_add(const oq_quad* x, const oq_quad* y, oq_quad* out) {
    const int32_t e = x->exp > y->exp ? x->exp : y->exp;
    const int sx = e - x->exp, sy = e - y->exp;
    if (sx > 62 || sy > 62) return OQ_E_OVERFLOW;
    const i128 fx = ((i128)1) << sx, fy = ((i128)1) << sy;
    return oq_canon((i128)x->a * fx + (i128)y->a * fy, (i128)x->b * fx + (i128)y->b * fy,
                    (i128)x->c * fx + (i128)y->c * fy, (i128)x->d * fx + (i128)y->d * fy, e, out);
}

static oq_quad oq_negate(oq_quad x) {       /* ring_neg ring.cpp:88-92 */
    x.a = -x.a; x.b = -x.b; x.c = -x.c; x.d = -x.d;
    return x;
}

int oq_sub(const oq_quad* x, const oq_quad* y, oq_quad* out) {   /* ring.cpp:72-74 */
    oq_quad ny = oq_negate(*y);
    return oq_add(x, &ny, out);
}

/* ring_mul: ring.cpp:76-86 (Lemma 8). */
int oq_mul(const oq_quad* x, const oq_quad* y, oq_quad* out) {
    const i128 xa = x->a, xb = x->b, xc = x->c, xd = x->d;
    const i128 ya = y->a, yb = y->b, yc = y->c, yd = y->d;
    const i128 re0 = xa * ya + 2 * xb * yb - xc * yc - 2 * xd * yd;
    const i128 re1 = xa * yb + xb * ya - xc * yd - xd * yc;
    const i128 im0 = xa * yc + 2 * xb * yd + xc * ya + 2 * xd * yb;
    const i128 im1 = xa * yd + xb * yc + xc * yb + xd * ya;
    return oq_canon(re0, re1, im0, im1, (int64_t)x->exp + y->exp, out);
}

/* phase_to_ring: ring.cpp:114-129 (omega^k, omega = e^{i pi/4}); the
 * coefficient table is the SPEC's. */
int oq_omega(int k, oq_quad* out) {
    static const int8_t tab[8][5] = {
        {1, 0, 0, 0, 0}, {0, 1, 0, 1, 1}, {0, 0, 1, 0, 0}, {0, -1, 0, 1, 1},
        {-1, 0, 0, 0, 0}, {0, -1, 0, -1, 1}, {0, 0, -1, 0, 0}, {0, 1, 0, -1, 1}};
    if (k < 0 || k > 7) return OQ_E_DOMAIN;
    out->a = tab[k][0]; out->b = tab[k][1]; out->c = tab[k][2]; out->d = tab[k][3];
    out->exp = tab[k][4];
    return OQ_OK;
}

/* to_complex: ring.cpp:131-136 -- (double(a) + double(b)*sqrt2) * 2^-exp,
 * evaluated without FMA contraction (this file is built -ffp-contract=off). */
void oq_to_complex(const oq_quad* x, double* re, double* im) {
    const double s2 = sqrt(2.0);
    const double scale = ldexp(1.0, -x->exp);
    *re = ((double)x->a + (double)x->b * s2) * scale;
    *im = ((double)x->c + (double)x->d * s2) * scale;
}

/* ---- phases and assignments: phase.hpp ----------------------------------- */

/* ParamAssignment::total: phase.hpp:18-23. */
static void oq_total(uint64_t bits, unsigned n, uint64_t* b, uint64_t* defined) {
    if (n >= 64) { *b = bits; *defined = ~(uint64_t)0; return; }
    const uint64_t m = (((uint64_t)1) << n) - 1;
    *b = bits & m; *defined = m;
}

/* instantiate_phase: phase.hpp:71-77 -- (k + 4*parity(mask & bits)) & 7. */
int oq_instantiate_phase(int k, uint64_t mask, uint64_t bits, uint64_t defined, int* out) {
    if (mask & ~defined) return OQ_E_MISSING;        /* covers(): phase.hpp:25 */
    const int parity = __builtin_popcountll(mask & bits) & 1;
    *out = (k + 4 * parity) & 7;
    return OQ_OK;
}

/* ---- subterms: subterm.cpp ------------------------------------------------ */

/* phase_pair_value: subterm.cpp:23-27 -- 1 + w^a + w^b - w^(a+b). */
int oq_pair_value(int ka, int kb, oq_quad* out) {
    oq_quad one, wa, wb, wab, t, u;
    int st;
    oq_make(1, 0, 0, 0, 0, &one);
    oq_omega(ka & 7, &wa); oq_omega(kb & 7, &wb); oq_omega((ka + kb) & 7, &wab);
    if ((st = oq_add(&one, &wa, &t))) return st;
    if ((st = oq_add(&t, &wb, &u))) return st;
    return oq_sub(&u, &wab, out);
}

/* subterm_value: subterm.cpp:29-49. Order of instantiation follows the
 * reference (PiPair resolves its selector phi first, :42-46). */
int oq_subterm_value(const oq_subterm* s, uint64_t bits, uint64_t defined, oq_quad* out) {
    int st, kp, kf;
    oq_quad one, w;
    switch (s->kind) {
    case OQ_NODE:
        if ((st = oq_instantiate_phase(s->psi_k, s->psi_mask, bits, defined, &kp))) return st;
        oq_make(1, 0, 0, 0, 0, &one);
        oq_omega(kp, &w);
        return oq_add(&one, &w, out);
    case OQ_PHASE_PAIR:
        if ((st = oq_instantiate_phase(s->psi_k, s->psi_mask, bits, defined, &kp))) return st;
        if ((st = oq_instantiate_phase(s->phi_k, s->phi_mask, bits, defined, &kf))) return st;
        return oq_pair_value(kp, kf, out);
    case OQ_HALF_PI:
        if ((st = oq_instantiate_phase(s->psi_k, s->psi_mask, bits, defined, &kp))) return st;
        if (kp == 2) return oq_omega(1, out);
        if (kp == 6) return oq_omega(7, out);
        return OQ_E_DOMAIN;
    case OQ_PI_PAIR:
        if ((st = oq_instantiate_phase(s->phi_k, s->phi_mask, bits, defined, &kf))) return st;
        if (kf == 0) return oq_make(1, 0, 0, 0, 0, out);
        if (kf == 4) {
            if ((st = oq_instantiate_phase(s->psi_k, s->psi_mask, bits, defined, &kp))) return st;
            return oq_omega(kp, out);
        }
        return OQ_E_DOMAIN;
    }
    return OQ_E_DOMAIN;
}

static int pauli_image(int k) { return k == 0 || k == 4; }          /* phase.hpp:47 */
static int proper_clifford_image(int k) { return k == 2 || k == 6; } /* phase.hpp:49 */

/* normalize_subterm: subterm.cpp:51-96 (Lemmas 3-5). Writes the constant and,
 * when the subterm depends on the assignment, the phase-pair row
 * (k_alpha, psi mask, k_beta, phi mask); *has_pair says which. */
int oq_normalize(const oq_subterm* s, oq_quad* constant, int* has_pair, oq_subterm* pair) {
    int st;
    *has_pair = 0;
    memset(pair, 0, sizeof *pair);
    pair->kind = OQ_PHASE_PAIR;
    switch (s->kind) {
    case OQ_PHASE_PAIR:                                               /* :54-58 */
        if (!s->psi_mask && !s->phi_mask) return oq_pair_value(s->psi_k, s->phi_k, constant);
        oq_make(1, 0, 0, 0, 0, constant);
        *pair = *s; pair->psi_k &= 7; pair->phi_k &= 7;
        *has_pair = 1;
        return OQ_OK;
    case OQ_NODE: {                                                   /* :59-66 */
        if (!s->psi_mask) {
            oq_quad one, w;
            oq_make(1, 0, 0, 0, 0, &one);
            if ((st = oq_omega(s->psi_k & 7, &w))) return st;
            return oq_add(&one, &w, constant);
        }
        /* (1 + e^{i psi}) = (1-i)/2 * pair(psi + pi/2, pi/2) */
        oq_make(1, 0, -1, 0, 1, constant);
        pair->psi_k = (uint8_t)((s->psi_k + 2) & 7); pair->psi_mask = s->psi_mask;
        pair->phi_k = 2; pair->phi_mask = 0;
        *has_pair = 1;
        return OQ_OK;
    }
    case OQ_PI_PAIR: {                                                /* :67-77 */
        if (!pauli_image(s->phi_k)) return OQ_E_DOMAIN;
        if (!s->phi_mask && !s->psi_mask) {
            if (s->phi_k == 4) return oq_omega(s->psi_k & 7, constant);
            return oq_make(1, 0, 0, 0, 0, constant);
        }
        oq_make(1, 0, 0, 0, 1, constant);                             /* 1/2 */
        pair->psi_k = s->psi_k & 7; pair->psi_mask = s->psi_mask;
        pair->phi_k = s->phi_k & 7; pair->phi_mask = s->phi_mask;
        *has_pair = 1;
        return OQ_OK;
    }
    case OQ_HALF_PI: {                                                /* :78-93 */
        if (!proper_clifford_image(s->psi_k)) return OQ_E_DOMAIN;
        oq_quad c;
        oq_omega(s->psi_k == 2 ? 1 : 7, &c);
        if (!s->psi_mask) { *constant = c; return OQ_OK; }
        /* change of variable: pi_pair(base=(8-k, {}), selector=(0, mask)); the
         * selector has Pauli image so it stays in the phi slot (subterm.cpp:12-21),
         * and its normalisation is 1/2 * pair(base, selector). */
        oq_quad half;
        oq_make(1, 0, 0, 0, 1, &half);
        if ((st = oq_mul(&c, &half, constant))) return st;
        pair->psi_k = (uint8_t)((8 - s->psi_k) & 7); pair->psi_mask = 0;
        pair->phi_k = 0; pair->phi_mask = s->psi_mask;
        *has_pair = 1;
        return OQ_OK;
    }
    }
    return OQ_E_DOMAIN;
}

/* ---- whole-expression evaluation ----------------- */

static uint64_t subterm_param_mask(const oq_subterm* s) {   /* subterm.hpp:34 */
    return s->psi_mask | s->phi_mask;
}

/* One leaf term at one assignment: instantiate_diagram's scalar fold,
 * diagram.cpp:149-165 (coverage check, then constant-first product). */
int oq_term_value(const oq_expr* e, uint64_t t, uint64_t bits, uint64_t defined, oq_quad* out) {
    uint64_t used = 0;
    for (uint64_t j = e->term_offset[t]; j < e->term_offset[t + 1]; ++j)
        used |= subterm_param_mask(&e->subterms[j]);
    if (used & ~defined) return OQ_E_MISSING;
    oq_quad s = e->scalars[t], v, tmp;
    int st;
    for (uint64_t j = e->term_offset[t]; j < e->term_offset[t + 1]; ++j) {
        if ((st = oq_subterm_value(&e->subterms[j], bits, defined, &v))) return st;
        if ((st = oq_mul(&s, &v, &tmp))) return st;
        s = tmp;
    }
    *out = s;
    return OQ_OK;
}

int oq_eval_one(const oq_expr* e, uint64_t word, oq_quad* out) {
    uint64_t bits, defined;
    oq_total(word, e->n_params, &bits, &defined);
    oq_quad total, tv, tmp;
    memset(&total, 0, sizeof total);
    int st;
    for (uint64_t t = 0; t < e->n_terms; ++t) {
        if ((st = oq_term_value(e, t, bits, defined, &tv))) return st;
        if ((st = oq_add(&total, &tv, &tmp))) return st;
        total = tmp;
    }
    *out = total;
    return OQ_OK;
}

typedef struct {
    const oq_expr* e;
    const uint64_t* words;
    uint64_t begin, end;
    oq_quad* exact;
    double* amp;
    int status;
} oq_job;

static void* oq_worker(void* p) {
    oq_job* j = (oq_job*)p;
    j->status = OQ_OK;
    for (uint64_t i = j->begin; i < j->end; ++i) {
        oq_quad q;
        int st = oq_eval_one(j->e, j->words[i], &q);
        if (st) { j->status = st; return NULL; }
        if (j->exact) j->exact[i] = q;
        if (j->amp) oq_to_complex(&q, &j->amp[2 * i], &j->amp[2 * i + 1]);
    }
    return NULL;
}

/* evaluate_batch over assignment words, parallel over assignments
 * like the SPEC's chunked CPU backend. Output order = input order. */
int oq_eval_batch(const oq_expr* e, const uint64_t* words, uint64_t n, int n_threads,
                  oq_quad* exact, double* amp) {
    if (n_threads < 1) n_threads = 1;
    if ((uint64_t)n_threads > n) n_threads = n ? (int)n : 1;
    oq_job* jobs = (oq_job*)calloc((size_t)n_threads, sizeof(oq_job));
    pthread_t* th = (pthread_t*)calloc((size_t)n_threads, sizeof(pthread_t));
    for (int t = 0; t < n_threads; ++t) {
        jobs[t].e = e; jobs[t].words = words; jobs[t].exact = exact; jobs[t].amp = amp;
        jobs[t].begin = n * (uint64_t)t / (uint64_t)n_threads;
        jobs[t].end = n * (uint64_t)(t + 1) / (uint64_t)n_threads;
    }
    for (int t = 1; t < n_threads; ++t) pthread_create(&th[t], NULL, oq_worker, &jobs[t]);
    oq_worker(&jobs[0]);
    int st = OQ_OK;
    for (int t = 0; t < n_threads; ++t) {
        if (t) pthread_join(th[t], NULL);
        if (jobs[t].status && !st) st = jobs[t].status;
    }
    free(jobs); free(th);
    return st;
}

/* Normalised-row view of an expression (the table compiler's contract,
 * S:387-395 with constants folded per term): row r of term t is the phase
 * pair of the r-th assignment-dependent subterm; folded constant C_t' =
 * C_t * prod K_j. Rows are written in subterm order. Returns the row count via
 * *n_rows when rows == NULL. */
int oq_normalize_expr(const oq_expr* e, oq_quad* folded, uint64_t* row_offset,
                      oq_subterm* rows, uint64_t* n_rows) {
    uint64_t r = 0;
    int st;
    for (uint64_t t = 0; t < e->n_terms; ++t) {
        oq_quad c = e->scalars[t], k, tmp;
        if (row_offset) row_offset[t] = r;
        for (uint64_t j = e->term_offset[t]; j < e->term_offset[t + 1]; ++j) {
            oq_subterm pair;
            int has;
            if ((st = oq_normalize(&e->subterms[j], &k, &has, &pair))) return st;
            if ((st = oq_mul(&c, &k, &tmp))) return st;
            c = tmp;
            if (has) { if (rows) rows[r] = pair; ++r; }
        }
        if (folded) folded[t] = c;
    }
    if (row_offset) row_offset[e->n_terms] = r;
    *n_rows = r;
    return OQ_OK;
}

/* E3 oracle: per (row, assignment) phase indices of the normalised rows,
 * idx_psi*8 + idx_phi, row-major over rows then assignments. */
int oq_phase_indices(const oq_expr* e, const uint64_t* words, uint64_t n, uint8_t* out) {
    uint64_t n_rows = 0;
    int st = oq_normalize_expr(e, NULL, NULL, NULL, &n_rows);
    if (st) return st;
    oq_subterm* rows = (oq_subterm*)malloc(sizeof(oq_subterm) * (n_rows ? n_rows : 1));
    st = oq_normalize_expr(e, NULL, NULL, rows, &n_rows);
    for (uint64_t r = 0; !st && r < n_rows; ++r) {
        for (uint64_t i = 0; i < n; ++i) {
            uint64_t bits, defined;
            int kp, kf;
            oq_total(words[i], e->n_params, &bits, &defined);
            if ((st = oq_instantiate_phase(rows[r].psi_k, rows[r].psi_mask, bits, defined, &kp))) break;
            if ((st = oq_instantiate_phase(rows[r].phi_k, rows[r].phi_mask, bits, defined, &kf))) break;
            out[r * n + i] = (uint8_t)(kp * 8 + kf);
        }
    }
    free(rows);
    return st;
}
