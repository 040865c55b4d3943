/* pzx_oracle.h -- CPU ORACLE interface (test infrastructure only; see
 * pzx_oracle.c). Restates the reference's exact evaluator
 * (/root/reference/proj/core: ring.cpp, subterm.cpp, diagram.cpp:149-165). */
#ifndef PZX_ORACLE_H
#define PZX_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error classes of common.hpp:13-48, as status codes. */
enum { OQ_OK = 0, OQ_E_PARSE = 1, OQ_E_DOMAIN = 2, OQ_E_MISSING = 3, OQ_E_OVERFLOW = 4 };

/* SubtermKind, subterm.hpp:19. */
enum { OQ_NODE = 0, OQ_PHASE_PAIR = 1, OQ_HALF_PI = 2, OQ_PI_PAIR = 3 };

/* RingQuad, ring.hpp:17-38. */
typedef struct { int64_t a, b, c, d; int32_t exp; int32_t pad_; } oq_quad;

/* Subterm, subterm.hpp:21-36 (ParamPhase psi/phi as (k in [0,7], XOR mask)). */
typedef struct {
    uint8_t kind, psi_k, phi_k, pad_[5];
    uint64_t psi_mask, phi_mask;
} oq_subterm;

/* A leaf-term list: term t = scalars[t] * prod subterms[term_offset[t] ..
 * term_offset[t+1]) -- the scalar_/pending_ pair of a leaf ZXDiagram
 * (diagram.hpp:91-92). */
typedef struct {
    uint32_t n_params;
    uint64_t n_terms;
    const uint64_t* term_offset; /* [n_terms + 1], absolute indices into subterms */
    const oq_quad* scalars;      /* [n_terms] */
    const oq_subterm* subterms;
} oq_expr;

int oq_make(int64_t a, int64_t b, int64_t c, int64_t d, int32_t e, oq_quad* out);
int oq_add(const oq_quad* x, const oq_quad* y, oq_quad* out);
int oq_sub(const oq_quad* x, const oq_quad* y, oq_quad* out);
int oq_mul(const oq_quad* x, const oq_quad* y, oq_quad* out);
int oq_omega(int k, oq_quad* out);
void oq_to_complex(const oq_quad* x, double* re, double* im);
int oq_instantiate_phase(int k, uint64_t mask, uint64_t bits, uint64_t defined, int* out);
int oq_pair_value(int ka, int kb, oq_quad* out);
int oq_subterm_value(const oq_subterm* s, uint64_t bits, uint64_t defined, oq_quad* out);
int oq_normalize(const oq_subterm* s, oq_quad* constant, int* has_pair, oq_subterm* pair);
int oq_term_value(const oq_expr* e, uint64_t t, uint64_t bits, uint64_t defined, oq_quad* out);
int oq_eval_one(const oq_expr* e, uint64_t word, oq_quad* out);
int oq_eval_batch(const oq_expr* e, const uint64_t* words, uint64_t n, int n_threads,
                  oq_quad* exact, double* amp);
int oq_normalize_expr(const oq_expr* e, oq_quad* folded, uint64_t* row_offset,
                      oq_subterm* rows, uint64_t* n_rows);
int oq_phase_indices(const oq_expr* e, const uint64_t* words, uint64_t n, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif
