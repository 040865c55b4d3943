/*
 * pzx_gpu.h -- C ABI of the B200 evaluator for the parametric sum-over-Cliffords
 * scalar of arXiv 2403.06777:
 *
 *     S(a) = sum_i C_i * prod_j S_ij(a)            (PAPER Eq. 3)
 *
 * evaluated at many boolean parameter assignments a (output bitstrings,
 * marginals, samples). This is the drop-in boundary for the reference's
 * evaluate-on-assignments path; the entry points replace:
 *
 *   pzx_table_upload_expr  <- ZXDiagram leaf list (scalar_ + pending_ subterms,
 *                             diagram.hpp:70-77, diagram.cpp:114-120) run
 *                             through normalize_subterm (subterm.cpp:51-96) and
 *                             SPEC compile_bit_table
 *   pzx_table_upload       <- SPEC BitTable upload: already
 *                             normalised phase-pair rows
 *   pzx_evaluate           <- SPEC evaluate_batch(BitTable, AssignmentBatch)
 *                             (S:475-483); per element it equals
 *                             sum_i instantiate_diagram(leaf_i, a).scalar()
 *                             (diagram.cpp:149-165) through to_complex
 *                             (ring.cpp:131-136)
 *   pzx_evaluate_range     <- the same over the enumerated batch first..first+n-1
 *                             ("all 2^P amplitudes", strong_amplitude /
 *                             marginal_summing sweeps)
 *   pzx_debug_phase_indices<- instantiate_phase (phase.hpp:71-77) per (row, a)
 *   pzx_debug_term_codes   <- the per-term product of subterm_value factors
 *                             (diagram.cpp:158-161) in exact exponent form
 *
 * Conventions: no exceptions cross the ABI -- every call
 * returns a pzx_status whose codes map the reference's pzx::Error hierarchy
 * (common.hpp:13-48); validation happens at upload (k in [0,7], masks within
 * the declared n_params <= 64 = kMaxParams, common.hpp:11); tables are
 * immutable after upload; a context is driven by one host thread at a time;
 * evaluation is a pure function of (table, assignments); output order equals
 * input order. Assignment words follow ParamAssignment::total (phase.hpp:18-23):
 * bit i = parameter i, bits >= n_params ignored.
 *
 * Plain pointers and sizes only; no CUDA or torch types in the signatures
 * (streams are passed as void* = cudaStream_t and used as given: NULL is the
 * CUDA legacy default stream; the synchronous host entry points use the
 * context's own stream). The asynchronous *_device calls take their per-call
 * scratch (sort buffers, term-chunk bounds and partials) from a stream-ordered
 * pool on the caller's stream, so calls in flight on different streams of one
 * context do not share buffers; the host thread rule above still applies.
 */
#ifndef PZX_GPU_H
#define PZX_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PZX_OK = 0,
    PZX_E_PARSE = 1,          /* pzx::ParseError        common.hpp:20-23 */
    PZX_E_DOMAIN = 2,         /* pzx::DomainError       common.hpp:26-29 */
    PZX_E_MISSING_PARAM = 3,  /* pzx::MissingParameter  common.hpp:45-48 */
    PZX_E_OVERFLOW = 4,       /* pzx::OverflowError     common.hpp:39-42 */
    PZX_E_INVALID = 5,        /* bad handle / argument (no reference analogue) */
    PZX_E_CAPACITY = 6,       /* table shape outside what this build supports */
    PZX_E_CUDA = 10,
    PZX_E_NCCL = 11,
    PZX_E_OOM = 12
} pzx_status;

/* SubtermKind, subterm.hpp:19 */
enum { PZX_NODE = 0, PZX_PHASE_PAIR = 1, PZX_HALF_PI = 2, PZX_PI_PAIR = 3 };

/* pzx_evaluate flags */
enum {
    PZX_PROB_ABS2 = 1u << 0,  /* prob[i] = |amp_i|^2 (Born rule)            */
    PZX_PROB_REAL = 1u << 1,  /* prob[i] = Re(amp_i) (doubled diagram)      */
    PZX_ACCUMULATE = 1u << 2, /* pzx_evaluate_device: add into d_amp (term ranges)  */
    PZX_KERNEL_GENERAL = 1u << 8, /* force the per-assignment POPC kernel          */
    PZX_KERNEL_GRAY = 1u << 9,    /* force the enumerated (low-bit Walsh) kernel   */
    PZX_KERNEL_SLICE = 1u << 10,  /* force the bit-sliced enumerated kernel        */
    PZX_KERNEL_SLICE_RAND = 1u << 11, /* force the plane-XOR bit-sliced kernel for any word list */
    PZX_KERNEL_SORTED = 1u << 12, /* force sort + bit-sliced Four-Russians kernel (any word list) */
    PZX_KERNEL_SLICE2 = 1u << 13, /* force the two-slice (64 assignments / thread) enumerated kernel */
    PZX_KERNEL_PAGE = 1u << 14    /* force the page-layout enumerated kernel (branch-free row families) */
};

typedef struct pzx_ctx pzx_ctx;
typedef struct pzx_table pzx_table;

/* Leaf-term list, i.e. what parametric reduction leaves behind: for term t the
 * exact constant C_t (RingQuad a,b,c,d,exp; ring.hpp:17-38, value
 * (a + b*sqrt2 + i(c + d*sqrt2)) * 2^-exp) times the product of the raw
 * subterms [term_offset[t], term_offset[t+1]) of any of the four kinds
 * (subterm.hpp:21-36). term_offset holds ABSOLUTE indices into the subterm
 * arrays, so a contiguous term range of a bigger list is a valid view (used
 * for the multi-GPU term split). */
typedef struct {
    uint32_t n_params;            /* <= 64 */
    uint64_t n_terms;
    const uint64_t* term_offset;  /* [n_terms + 1] */
    const int64_t* term_scalar;   /* [n_terms * 5]: a, b, c, d, exp */
    const uint8_t* kind;          /* PZX_NODE .. PZX_PI_PAIR */
    const uint8_t* psi_k;         /* [0,7] */
    const uint64_t* psi_mask;
    const uint8_t* phi_k;         /* [0,7]; ignored for Node / HalfPi */
    const uint64_t* phi_mask;
} pzx_expr_view;

/* Already-normalised phase-pair rows (SPEC ScalarExpression after Eq. 4,
 * S:332-335): row r contributes 1 + w^x + w^y - w^(x+y) with
 * x = k_alpha[r] + 4*parity(psi_mask[r] & a), y = k_beta[r] + 4*parity(phi_mask[r] & a).
 * No dummy padding is needed (CSR offsets), unlike the paper's padded
 * m x n_max matrix. */
typedef struct {
    uint32_t n_params;
    uint64_t n_terms;
    const uint64_t* term_row_offset;  /* [n_terms + 1], absolute */
    const int64_t* term_coef;         /* [n_terms * 5] exact C_t */
    const uint64_t* psi_mask;
    const uint64_t* phi_mask;
    const uint8_t* k_alpha;
    const uint8_t* k_beta;
} pzx_table_view;

/* Per-term debug record of pzx_debug_term_codes: the exact product of the
 * term's row values at one assignment is
 *   C'_t * sqrt2^E_t * mu^nLM_t * w^j * (lambda/mu)^s1 * pi^a * pi'^b   (z == 0)
 * and 0 when z > 0, with w = e^{i pi/4}, lambda = 1 - w, mu = 1 + w,
 * pi = 1 + w + w^3, pi' = 1 - w - w^3 (E_t, nLM_t, C'_t from
 * pzx_table_term_info). DESIGN.md §2 derives this factorisation. */
typedef struct { uint32_t j, z, s1, a, b; } pzx_term_code;

const char* pzx_status_string(pzx_status s);
const char* pzx_version(void);

pzx_status pzx_create(int device, pzx_ctx** out);
void pzx_destroy(pzx_ctx* ctx);
const char* pzx_last_error(const pzx_ctx* ctx);
/* Number of kernel launches issued by this context since creation. */
uint64_t pzx_launch_count(const pzx_ctx* ctx);
/* The evaluation kernel the last pzx_evaluate* call of this context chose:
 * 1 POPC, 2 gray, 3 bit-sliced, 4 bit-sliced word list, 5 sorted, 6 two-slice,
 * 7 warp-chunk bit-sliced; the sorted kernel's table groups (4 or 6) and the
 * term-chunk count of the grid. For reports (bench.py's roofline). */
pzx_status pzx_last_kernel(const pzx_ctx* ctx, int32_t* kernel, int32_t* sorted_groups, int32_t* term_chunks);

pzx_status pzx_table_upload_expr(pzx_ctx* ctx, const pzx_expr_view* expr, pzx_table** out);
pzx_status pzx_table_upload(pzx_ctx* ctx, const pzx_table_view* view, pzx_table** out);
void pzx_table_free(pzx_table* t);
/* Host-only compile (no device, no context): normalisation + classification
 * exactly as pzx_table_upload_expr, for inspection (shape / term_info) and
 * CPU tests. Evaluating such a table returns PZX_E_INVALID. */
pzx_status pzx_table_compile_host(const pzx_expr_view* expr, pzx_table** out);
/* Host-only: the per-class variant codes [64 classes][4 variants], sqrt2
 * exponent e[64] and lambda/mu flag lm[64] the kernels use. */
pzx_status pzx_class_table(uint32_t codes[256], int32_t e[64], int32_t lm[64]);
/* Host-only: the bit-sliced kernel's 129 row ops (class * 2 + single, 128 =
 * unit row): per op {jbase, w'[4], zero_tt, lambda_tt, pi_tt, pi'_tt, lm}
 * (pzx_classes.h); returns PZX_E_DOMAIN if it disagrees with the generated
 * PTX tables (pzx_slice_dispatch.inc). */
pzx_status pzx_slice_op_table(int32_t out[129 * 10]);
/* shape: n_params, n_terms, n_rows (genuine rows), max rows in one term */
pzx_status pzx_table_shape(const pzx_table* t, uint32_t* n_params, uint64_t* n_terms,
                           uint64_t* n_rows, uint32_t* max_term_rows);
/* Work statistics behind bench.py's algorithmic roofline:
 * op_rows[op] = rows of bit-sliced op (class * 2 + single-parity, 128 = unit
 * row), term_kinds = terms whose epilogue is kind-free / lambda-only / with a
 * pi or pi' row. Either pointer may be NULL. */
pzx_status pzx_table_slice_stats(const pzx_table* t, uint64_t op_rows[129], uint64_t term_kinds[3]);
/* Rows per page family: {constraint, generic, dispatch, dropped, lambda} and
 * the generic rows by update class {S2, S6, E0, E2, G1, G3} (pzx_host.cpp,
 * page_term) -- PZX_PAGE_FAMILIES counts -- and the dispatch rows per op
 * (bench.py's roofline of the page kernel); any table with a page layout,
 * PZX_E_CAPACITY otherwise. */
#define PZX_PAGE_FAMILIES 11
pzx_status pzx_table_page_stats(const pzx_table* t, uint64_t family_rows[PZX_PAGE_FAMILIES], uint64_t d_op_rows[129]);
/* Host-only tables (pzx_table_compile_host): the page layout of the
 * enumerated page kernel -- *n_slots 32-byte records (8 x u32 each; slots may
 * be NULL to query the size), the header slot of every term, the w^j folded
 * into each term's page constant, and the rows per family (as
 * pzx_table_page_stats). PZX_E_CAPACITY: the table has no page layout. */
pzx_status pzx_table_page_layout(const pzx_table* t, uint32_t* slots, uint64_t* n_slots, uint32_t* term_slot,
                                 uint8_t* jfold, uint64_t family_rows[PZX_PAGE_FAMILIES]);
/* Folded exact constant C'_t (a,b,c,d,exp), sqrt2 exponent E_t and the count
 * nLM_t of lambda/mu rows of term t (see pzx_term_code). */
pzx_status pzx_table_term_info(const pzx_table* t, uint64_t term, int64_t coef[5],
                               int32_t* e_sqrt2, int32_t* n_lm);

/* Synchronous evaluation from HOST buffers: assignments[n] -> amp[2n]
 * (re,im interleaved; may be NULL) and prob[n] (may be NULL). A small call
 * (n <= 65536, pinned host buffers, an enumerated or contiguous batch)
 * repeated with the same arguments is captured into a CUDA graph on its
 * second occurrence and replayed from the third (the word contents are read
 * at every replay); PZX_NO_GRAPHS=1 disables this. */
pzx_status pzx_evaluate(pzx_ctx* ctx, const pzx_table* t, const uint64_t* assignments,
                        uint64_t n, double* amp, double* prob, uint32_t flags);
/* Enumerated batch first, first+1, ..., first+n-1 (generated on device). */
pzx_status pzx_evaluate_range(pzx_ctx* ctx, const pzx_table* t, uint64_t first, uint64_t n,
                              double* amp, double* prob, uint32_t flags);

/* Exact evaluation -- the SPEC's integer-ring backend contract (S:441-498:
 * "identical RingQuad outputs", "no floats in the kernel path"): out[5n] gets
 * the canonical RingQuad {a, b, c, d, exp} (ring.hpp:17-38, ring.cpp:20-48) of
 * S(a) per assignment, bit-identical to the reference's sequential fold
 * (ring_add over instantiate_diagram values, diagram.cpp:149-165; replaces
 * ParamScalarExpression::evaluate with exact output). Returns PZX_E_OVERFLOW
 * (pzx::OverflowError, ring.cpp:13-18) when a value or an intermediate term
 * product leaves int64; those entries get exp = -1 and the rest are written.
 * The reference may overflow earlier on intermediates of its own fold order. */
pzx_status pzx_evaluate_exact(pzx_ctx* ctx, const pzx_table* t, const uint64_t* assignments, uint64_t n,
                              int64_t* out);
pzx_status pzx_evaluate_exact_range(pzx_ctx* ctx, const pzx_table* t, uint64_t first, uint64_t n, int64_t* out);


/* Exact combine of the term split: out[i] = sum over r < n_parts of
 * parts[r][i], every entry a canonical RingQuad {a, b, c, d, exp} (int64 [n_parts][n][5],
 * part-major, e.g. the all-gathered pzx_evaluate_exact results of disjoint term
 * ranges); replaces the ring_add fold over terms (ring.cpp:57-70) across ranks.
 * The result is canonical and order-free. An input with exp = -1 (overflowed)
 * or a sum outside int64 gives exp = -1 and PZX_E_OVERFLOW (host form). The
 * _device form is asynchronous on `stream` (NULL = default) and reports
 * overflow only through exp = -1. */
pzx_status pzx_ringquad_sum(pzx_ctx* ctx, const int64_t* parts, uint32_t n_parts, uint64_t n, int64_t* out);
pzx_status pzx_ringquad_sum_device(pzx_ctx* ctx, const int64_t* d_parts, uint32_t n_parts, uint64_t n,
                                   int64_t* d_out, void* stream);
/* Asynchronous DEVICE-pointer variants on `stream` (used as given, NULL = default stream):
 * d_assignments may be NULL for the enumerated batch starting at `first`.
 * Term range [term_begin, term_end) of the table (term_end = UINT64_MAX: all)
 * gives partial amplitudes for the term split; d_amp receives 2n doubles,
 * d_prob n doubles (either may be NULL). With PZX_ACCUMULATE the amplitudes are
 * added into d_amp (and d_prob is computed from the sum); d_amp must then be
 * given (PZX_E_INVALID otherwise). */
pzx_status pzx_evaluate_device(pzx_ctx* ctx, const pzx_table* t, const uint64_t* d_assignments,
                               uint64_t first, uint64_t n, uint64_t term_begin,
                               uint64_t term_end, double* d_amp, double* d_prob,
                               uint32_t flags, void* stream);
/* Upload with compile options. PZX_COMPILE_SIMPLIFY: post-reduction table
 * simplification (PAPER "Conclusions") -- rows of a term with
 * identical masks whose product is assignment-independent are folded into the
 * term constant (pairwise node cancellation; a zero product drops the term's
 * rows and zeroes it). Values are unchanged; row order / counts then differ
 * from the plain normalisation (the debug hooks index the compiled rows). */
enum { PZX_COMPILE_SIMPLIFY = 1u << 0 };
pzx_status pzx_table_upload_expr_ex(pzx_ctx* ctx, const pzx_expr_view* expr, uint32_t compile_flags,
                                    pzx_table** out);

/* Several GPUs from one host thread. REPLICATE: the table
 * on every device, a batch cut into contiguous per-device slices evaluated
 * concurrently (no inter-GPU traffic). SPLIT_TERMS: row-balanced term ranges
 * per device, the whole batch everywhere, partial amplitudes copied peer to
 * peer to the first device and summed in device order (deterministic). */
enum { PZX_REPLICATE = 0, PZX_SPLIT_TERMS = 1 };
typedef struct pzx_group pzx_group;
typedef struct pzx_group_table pzx_group_table;
pzx_status pzx_group_create(const int* devices, int n_devices, pzx_group** out);
void pzx_group_destroy(pzx_group* g);
const char* pzx_group_last_error(const pzx_group* g);
pzx_status pzx_group_upload_expr(pzx_group* g, const pzx_expr_view* expr, uint32_t mode, pzx_group_table** out);
void pzx_group_table_free(pzx_group_table* t);
/* assignments == NULL: the enumerated batch first .. first+n-1 */
pzx_status pzx_group_evaluate(pzx_group* g, const pzx_group_table* t, const uint64_t* assignments, uint64_t first,
                              uint64_t n, double* amp, double* prob, uint32_t flags);

/* Pipe-rate microbenchmark behind the roofline denominators:
 * which = 0 int32 LOP3, 1 POPC, 2 fp64 FMA, 3 LDS.32; thread-instructions/s. */
pzx_status pzx_microbench(int device, int which, double* ops_per_s);

/* SPEC BackendContract: capability descriptor of this backend. */
typedef struct {
    uint32_t max_params;          /* 64 */
    uint32_t max_rows_per_term;   /* of the bit-sliced kernels (longer terms use the POPC / gray kernels) */
    uint64_t max_rows_in_flight;  /* table rows staged in shared memory per CTA (TMA tiles) */
    uint64_t preferred_batch;     /* assignments per call that fill the GPU */
    uint32_t exact;               /* 0: fp64 amplitudes (1e-12 relative); phase indices are exact */
    uint32_t deterministic;       /* 1: fixed-order reductions, run-to-run identical */
    uint32_t n_sm;
    uint32_t tmem_accumulators;   /* 1 when the bit-sliced kernels keep accumulators in TMEM */
} pzx_backend_contract;
pzx_status pzx_backend_contract_get(pzx_ctx* ctx, pzx_backend_contract* out);

/* PZX1 binary table codec (SPEC "External Interfaces"): the
 * normalised table as header {"PZX1", u32 n_params, u64 m, u64 n_max, u64 R =
 * m*n_max}, i64 constants[m][5], then field-major padded rows u8 flags[R] (1 =
 * dummy), u8 k_alpha[R], u64 psi[R], u8 k_beta[R], u64 phi[R], little-endian.
 * Encoders with buf == NULL report the size in *len; decode errors are
 * PZX_E_PARSE (bad magic, truncation, inconsistent shape) and never leave a
 * partial value. decode(encode(x)) == x and encode(decode(b)) == b byte for byte. */
pzx_status pzx_pzx1_encode(const pzx_table_view* view, uint8_t* buf, uint64_t cap, uint64_t* len);
pzx_status pzx_pzx1_encode_expr(const pzx_expr_view* expr, uint8_t* buf, uint64_t cap, uint64_t* len);
pzx_status pzx_pzx1_info(const uint8_t* buf, uint64_t len, uint32_t* n_params, uint64_t* n_terms,
                         uint64_t* n_rows);
pzx_status pzx_pzx1_decode(const uint8_t* buf, uint64_t len, uint64_t* term_row_offset, int64_t* term_coef,
                           uint64_t* psi_mask, uint64_t* phi_mask, uint8_t* k_alpha, uint8_t* k_beta);
pzx_status pzx_table_upload_pzx1(pzx_ctx* ctx, const uint8_t* buf, uint64_t len, pzx_table** out);

/* Marginal summing (sim-driver): out[i] = sum over b < 2^m of
 * prob(fixed[i] | b), the don't-care outputs being the low m parameters
 * (fixed[i] must have them clear); prob = |amp|^2, or Re(amp) with
 * PZX_PROB_REAL. Deterministic (fixed-order reductions). Kernel flags apply. */
pzx_status pzx_marginal_sum(pzx_ctx* ctx, const pzx_table* t, const uint64_t* fixed, uint64_t n_fixed,
                            uint32_t m, uint32_t flags, double* out);
/* Repeated weak simulation (PAPER App. F Alg. 2): tables[k]
 * is the compiled doubled marginal P(a_1..a_{k+1}) (parameter j = bit j of
 * the sample word); out[i] receives n_bits sampled bits per sample. prob =
 * Re(value) by default (doubled diagrams), |value|^2 with PZX_PROB_ABS2.
 * Draws use a counter-based RNG of (seed, bit, sample): reproducible. */
pzx_status pzx_weak_sample(pzx_ctx* ctx, const pzx_table* const* tables, uint32_t n_bits, uint64_t n_samples,
                           uint64_t seed, uint32_t flags, uint64_t* out);
/* prob from amplitudes on device (after a cross-GPU sum of partials). */
pzx_status pzx_amp_to_prob_device(pzx_ctx* ctx, const double* d_amp, uint64_t n,
                                  double* d_prob, uint32_t flags, void* stream);
pzx_status pzx_synchronize(pzx_ctx* ctx);

/* E3 debug: phase indices idx_psi*8 + idx_phi per (row, assignment), rows in
 * the canonical normalised order (term-major, subterm order), row-major
 * [n_rows][n]. */
pzx_status pzx_debug_phase_indices(pzx_ctx* ctx, const pzx_table* t,
                                   const uint64_t* assignments, uint64_t n, uint8_t* idx_out);
/* Per (term, assignment) exact product codes, [n_terms][n]. */
pzx_status pzx_debug_term_codes(pzx_ctx* ctx, const pzx_table* t, const uint64_t* assignments,
                                uint64_t n, pzx_term_code* out);
/* The PRODUCTION bit-sliced kernels' own per-term state (k_eval_slice,
 * k_eval_slice_wc, k_eval_sorted -- whichever the batch and `flags` select,
 * PZX_E_INVALID otherwise): the batch is evaluated as pzx_evaluate
 * (assignments != NULL) or pzx_evaluate_range (first, n) would, and for terms
 * [term_begin, term_end) every assignment's {j, z, s1, a, b} is read from the
 * kernel's bit planes at the term's end row and written to
 * out[(term - term_begin) * n + i] (z is a flag here; j includes the rows'
 * base exponents folded into the term constant). Compare with
 * instantiate_diagram (diagram.cpp:149-165) through pzx_table_term_info. */
pzx_status pzx_debug_slice_codes(pzx_ctx* ctx, const pzx_table* t, const uint64_t* assignments, uint64_t first,
                                 uint64_t n, uint64_t term_begin, uint64_t term_end, uint32_t flags,
                                 pzx_term_code* out);

/* ---- host parametric reducer (SPEC zx-core S:67-84,
 * rewrite-engine S:131-244, decomposer S:246-317) ------------------------
 * A Clifford+T circuit (gate set of SPEC Circuit) is turned into a
 * closed polar-parameterised ZX diagram, Clifford-simplified (local
 * complementation, pivoting, state copy, identity removal -- parameter-
 * agnostic, emitting Node / PhasePair / HalfPi / PiPair subterms) and
 * stabiliser-decomposed into the leaf-term list pzx_table_upload_expr takes:
 * the reference's leaf form (diagram.hpp:70-77: scalar_ x pending_). Runs on
 * all host threads; the term order is deterministic. */
enum { PZX_G_H = 0, PZX_G_X, PZX_G_Z, PZX_G_S, PZX_G_SDG, PZX_G_T, PZX_G_TDG, PZX_G_CNOT, PZX_G_CZ,
       PZX_G_RZ /* k * pi/4 */ };
typedef struct { uint8_t op, q0, q1, k; } pzx_gate;
/* mode: PZX_REDUCE_AMPLITUDE: <out| U |in>; PZX_REDUCE_DOUBLED: the doubled
 * marginal <in| U^dag (|a><a| (x) I) U |in> (SPEC double_diagram).
 * in_spec / out_spec per qubit: 0 / 1 a fixed bit, 2 + p parameter p (bit p
 * of the assignment word), -1 (out_spec, doubled mode only) an unmeasured
 * (traced) qubit; in_spec NULL = |0...0>. max_terms: PZX_E_CAPACITY beyond
 * (0 = 2^26). Without parameters the leaves are summed exactly into ONE
 * constant term (the non-parametric path: one amplitude per reduction). */
enum { PZX_REDUCE_AMPLITUDE = 0, PZX_REDUCE_DOUBLED = 1 };
typedef struct pzx_expr pzx_expr;
pzx_status pzx_circuit_reduce(uint32_t n_qubits, const pzx_gate* gates, uint64_t n_gates, const int32_t* in_spec,
                              const int32_t* out_spec, uint32_t mode, uint64_t max_terms, pzx_expr** out);
/* the expression as a pzx_expr_view; the pointers stay valid until pzx_expr_free */
pzx_status pzx_expr_get_view(const pzx_expr* e, pzx_expr_view* view);
/* T-count of the input, T-like spiders left after the first Clifford
 * simplification, wall seconds of the reduction */
pzx_status pzx_expr_info(const pzx_expr* e, uint32_t* t_count, uint32_t* t_after_simp, double* seconds);
void pzx_expr_free(pzx_expr* e);

#ifdef __cplusplus
}
#endif
#endif /* PZX_GPU_H */
