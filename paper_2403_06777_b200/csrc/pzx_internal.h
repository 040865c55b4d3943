// pzx_internal.h -- layout contract between the host table compiler
// (pzx_host.cpp) and the sm_100a kernels (pzx_kernels.cu). DESIGN.md §3.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pzxb {

// ---- per-variant code word (one 32-bit SWAR add per row-eval) ------------
// A row of class (k_alpha, k_beta) evaluates, at parities (p, q), to
//   V = w^j * sqrt2^e * g,   g in {1, lambda, mu, pi, pi'}   or 0.
// e and "g in {lambda, mu}" depend on the class only (folded into the term
// constant at compile time); what varies per assignment is packed here:
constexpr uint32_t kZShift = 0;   // 7 bits: number of zero factors
constexpr uint32_t kS1Shift = 7;  // 7 bits: number of lambda factors
constexpr uint32_t kAShift = 14;  // 7 bits: number of pi factors
constexpr uint32_t kBShift = 21;  // 7 bits: number of pi' factors
constexpr uint32_t kJShift = 29;  // 3 bits: sum of j mod 8 (wraps off the top)
constexpr uint32_t kField = 0x7F;
constexpr int kSegRows = 127;     // rows one SWAR accumulator can absorb
// Flags in the row's code word (bits 0..10 hold the class byte offset cls*16)
constexpr uint32_t kCodeMask = 0x7FFu;
constexpr uint32_t kSegFlag = 1u << 30;  // flush the SWAR fields after this row
constexpr uint32_t kEndFlag = 1u << 31;  // last row of its term
constexpr int kUnitClass = 64;           // placeholder row of a row-less term (all-zero codes)
constexpr int kCodeClasses = 65;
constexpr int kMaxTermRows = 4095;

// Rows per thread-owned block of the enumerated (Walsh / "gray") kernel:
// thread owns assignments base + g, g in [0, 2^kGrayBits).
constexpr int kGrayBits = 4;
constexpr int kGray = 1 << kGrayBits;

// LUT blob (global memory, copied to shared memory by every CTA)
struct LutLayout {
    uint32_t codes_off;  // uint32 codes[kCodeClasses][4 variants]
    uint32_t om_off;     // double2 w^j, j = 0..7
    uint32_t u_off;      // double (sqrt2 - 1)^s, s = 0..max_rows
    uint32_t p3_off;     // double 3^m, m = 0..max_rows/2
    uint32_t pd_off;     // double2 pi^d (d > 0) / pi'^-d (d < 0), d = -max_rows..max_rows
    uint32_t sab_off;    // double2 (sqrt2-1)^s pi^a pi'^b, s < 16, a, b < 4, index s | a << 4 | b << 6
                         // (bit-sliced kernels' epilogue fast path)
    uint32_t uz_off;     // double uz[s | z << 4] = (sqrt2 - 1)^s (z = 0), 0 (z = 1); s < 16 (page kernel)
    uint32_t bytes;
    int32_t max_rows;
};

// Device table: ONE flat row stream in term order (every term owns >= 1 row).
// Row record for n_params <= 32 (rows32):
//   x = psi mask, y = phi mask, z = code word: class byte offset into codes
//   (cls * 16) | kSegFlag | kEndFlag,
//   w = Walsh pattern of the low kGrayBits parameters:
//       bit 2g   = parity(psi & g), bit 2g+1 = parity(phi & g)
// For n_params > 32 a row is TWO uint4: {psi_lo, psi_hi, phi_lo, phi_hi},
// {code word, pattern, 0, 0}.
struct DevTable {
    const uint4* rows = nullptr;
    const uint64_t* term_row = nullptr;  // [n_terms + 1], term_row[0] == 0
    const double2* term_c = nullptr;     // C''_t = C'_t * sqrt2^E_t * mu^nLM_t
    const unsigned char* lut = nullptr;
    LutLayout lut_layout{};
    uint64_t n_terms = 0, n_rows = 0;
    uint32_t n_params = 0, max_rows = 0;
    int p64 = 0;
    // bit-sliced kernel (only when every term has <= kSegRows rows):
    // rows as 2 x uint4 {psi, phi, op | kind flags | kEndFlag, Walsh32(psi)}, {Walsh32(phi), psi_hi, phi_hi, op}
    // (n_params <= 32: {Walsh32(phi), ~Walsh32(psi), ~Walsh32(phi), op})
    // (op = class * 2 + single, pzx_classes.h), constants C''_t * w^(sum of row jbase)
    const uint4* srows = nullptr;
    const double2* sterm_c = nullptr;
    int slice_ok = 0;
    // sorted-batch bit-sliced kernel (arbitrary word lists, n_params <= 32):
    // rows as 2 x uint4 {psi, phi, op | flags, op}, {psi offsets 0|1, psi offsets 2|3,
    // phi offsets 0|1, phi offsets 2|3}; offset k = (k * 16 + nibble_k(mask)) * 512,
    // 16-bit byte offsets into the per-thread Four-Russians tables ([row][thread])
    // of a 128-thread CTA (256-thread CTAs double them)
    const uint4* qrows = nullptr;
    int sorted_ok = 0;
    // page layout: pages of kPageSlots x 32 B records (terms never straddle a
    // page) and the header slot of every term (pzx_host.cpp, page_term)
    const uint4* prows = nullptr;
    const uint32_t* term_slot = nullptr;
    uint64_t n_pages = 0;
    int page_ok = 0;
};

// page layout (enumerated page kernel): pages of kPageSlots 32-byte records
constexpr int kPageSlots = 256;
constexpr uint32_t kNoSyncFlag = 1u << 30;  // internal: enqueue without the final stream sync (graph capture)
constexpr int kPageGClasses = 6;  // page-layout G rows by update class: S2, S6, E0, E2, G1, G3

constexpr int kSortedGroups = 4;              // 4-bit groups: parameters 0..15 via tables (dense batches)
constexpr int kSortedGroupsWide = 6;          // parameters 0..23 via tables (sparse batches, e.g. 2^16 of 2^32)
constexpr int kSortedLowBits = 4 * kSortedGroups;

enum KernelChoice { KC_AUTO = 0, KC_GENERAL = 1, KC_GRAY = 2, KC_SLICE = 3, KC_SLICER = 4, KC_SORTED = 5, KC_SLICE2 = 6,
                    KC_SLICEWC = 7 /* small enumerated batches: 4 warps x 4 term chunks per CTA (auto only) */,
                    KC_PAGE = 8 /* enumerated batches on the page layout (C / G / D row families) */ };
constexpr int kWarpChunksHost = 4;  // term chunks per CTA of the warp-chunk kernel

struct LaunchReq {
    const uint64_t* d_asg = nullptr;  // nullptr: enumerated first .. first + n - 1
    uint64_t first = 0, n = 0;
    uint64_t term_begin = 0, term_end = 0;
    double2* d_amp = nullptr;         // may be nullptr if only prob is wanted
    double* d_prob = nullptr;
    int prob_mode = 0;                // 0 none, 1 |amp|^2, 2 Re(amp)
    int accumulate = 0;               // add into d_amp instead of overwriting
    KernelChoice kernel = KC_AUTO;
    int words_contiguous = 0;         // host verified d_asg[i] == first + i (i < n)
    cudaStream_t stream = 0;
    // scratch owned by the context
    double2* d_partial = nullptr;     // [n_chunks][n] when n_chunks > 1
    const uint64_t* d_chunk_terms = nullptr;  // [n_chunks + 1] term boundaries
    int n_chunks = 1;
    // KC_SORTED: the batch sorted by (masked) word; results go to d_perm[i]
    const uint64_t* d_sorted = nullptr;
    int sorted_groups = kSortedGroups;  // Four-Russians table groups of the sorted kernel (4 or 6)
    const uint32_t* d_perm = nullptr;
    // debug (pzx_debug_slice_codes): the bit-sliced kernels write their own
    // per-term planes {J (before the 6 s1 fold), Z, s1, a, b} for terms
    // [dbg_t0, dbg_t1) at [term - dbg_t0][caller position < dbg_n][5]
    uint32_t* d_dbg5 = nullptr;
    uint64_t dbg_t0 = 0, dbg_t1 = 0, dbg_n = 0;
};

// Sort an arbitrary word list (masked to n_params bits) with its positions:
// scratch must hold sort_scratch_bytes(n) bytes; outputs live inside scratch.
size_t sort_scratch_bytes(uint64_t n);
// max over 32-word groups of (last - first) of the sorted batch (device -> host)
cudaError_t group_sorted(const uint64_t* d_sorted, const uint32_t* d_perm, uint64_t n, uint32_t low, void* scratch,
                         const uint64_t** d_pw, const uint32_t** d_pp, uint64_t* n_slots, cudaStream_t s,
                         uint64_t* launches);
cudaError_t group_slots(const uint64_t* d_sorted, uint64_t n, uint32_t low, void* scratch, uint64_t* n_slots,
                        cudaStream_t s, uint64_t* launches);
size_t sort_base_bytes(uint64_t n);
cudaError_t sort_words(const uint64_t* d_words, uint64_t n, uint32_t n_params, void* scratch,
                       const uint64_t** d_sorted, const uint32_t** d_perm, cudaStream_t s,
                       uint64_t* launches);

// Grid policy helpers (host)
int grid_assign_blocks(const DevTable& t, const LaunchReq& r, KernelChoice kc);
KernelChoice choose_kernel(const DevTable& t, const LaunchReq& r);
bool tmem_accumulators();
int resident_ctas_per_sm(const DevTable& t, KernelChoice kc, int nt, int sorted_groups = kSortedGroups);
int sorted_threads(int sorted_groups);  // CTA width of the sorted kernel (256 for the wide tables with TMEM)
int slice_threads(const LaunchReq& r);
bool kernel_supported(const DevTable& t, const LaunchReq& r, KernelChoice kc);

// Launchers; each returns the CUDA error of the launch and adds the number of
// kernel launches to *launches.
cudaError_t launch_evaluate(const DevTable& t, const LaunchReq& r, KernelChoice kc,
                            uint64_t* launches);
cudaError_t launch_amp_to_prob(const double2* amp, uint64_t n, double* prob, int mode,
                               cudaStream_t s, uint64_t* launches);
cudaError_t launch_debug_phase(const DevTable& t, const uint64_t* d_asg, uint64_t n,
                               uint8_t* d_out, cudaStream_t s, uint64_t* launches);
cudaError_t launch_sample_step(uint64_t* d_words, double* d_pprev, const double* d_p0, uint64_t n, uint32_t k,
                               uint64_t seed, unsigned int* d_err, cudaStream_t s, uint64_t* launches);
// sum of n_parts partial amplitude arrays [part][n] in part order (deterministic), then prob
cudaError_t launch_sum_partials(const double2* parts, int n_parts, uint64_t n, double2* amp, double* prob,
                                int prob_mode, cudaStream_t s, uint64_t* launches);
cudaError_t launch_expand_words(const uint64_t* d_fixed, uint64_t n_fixed, uint32_t m, uint64_t* d_words,
                                cudaStream_t s, uint64_t* launches);
cudaError_t launch_segment_sum(const double* d_in, uint64_t len, uint64_t n_seg, double* d_out, int accumulate,
                               cudaStream_t s, uint64_t* launches);
cudaError_t launch_debug_codes(const DevTable& t, const uint64_t* d_asg, uint64_t n,
                               uint32_t* d_out5, cudaStream_t s, uint64_t* launches);

// Exact (integer-ring) evaluation tables, built per table on first use
// (pzx_evaluate_exact). All Z[w] elements in the power basis (1, w, w^2, w^3);
// powers of 2 are kept out of the numerators (binary exponents), as the
// reference's canonical RingQuad does (ring.cpp:20-48).
struct ExactDev {
    const int64_t* ft = nullptr;    // [n_terms * 4] F_t: C'_t * sqrt2^E_t = F_t * 2^fx_t
    const int32_t* fx = nullptr;    // [n_terms] fx_t (INT32_MIN: the constant is not representable)
    const uint32_t* nlm = nullptr;  // [n_terms] nLM_t
    const int64_t* lam = nullptr;   // [lam_n * 4] lambda^r / 2^(r/4)
    const int64_t* mu = nullptr;    // [mu_n * 4] mu^r / 2^(r/4)
    const int64_t* pd = nullptr;    // [(2 pd_n - 1) * 4] centred at pd_n - 1: pi^d (d >= 0), pi'^-d (d < 0)
    const int64_t* p3 = nullptr;    // [p3_n] 3^m
    uint32_t lam_n = 0, mu_n = 0, pd_n = 0, p3_n = 0;  // valid entries (a larger index: OVERFLOW)
};
constexpr int kExactThreads = 128;
constexpr int kExactK = 2;  // assignments per thread, exact kernel (default; 1, 2 or 4 via PZX_EXACT_K)
// d_partial: n_chunks * n * (4 int128 + int32 exponent) when n_chunks > 1; d_pflag: n uint32, zeroed by the caller;
// d_out: n * 5 int64 {a, b, c, d, exp} (exp = -1: overflow)
cudaError_t launch_exact(const DevTable& t, const ExactDev& x, const uint64_t* d_asg, uint64_t first, uint64_t n,
                         const uint64_t* d_chunk_terms, int n_chunks, void* d_partial, uint32_t* d_pflag,
                         int64_t* d_out, cudaStream_t s, uint64_t* launches, int kx);

// d_parts: g * n canonical RingQuads (rank-major), d_out: n * 5 int64 (exp = -1: overflow)
cudaError_t launch_ringquad_sum(const int64_t* d_parts, uint32_t g, uint64_t n, int64_t* d_out, cudaStream_t s,
                                uint64_t* launches);

constexpr int kThreads = 256;
constexpr int kGeneralK = 4;  // assignments per thread, general kernel

}  // namespace pzxb
