// pzx_host.cpp -- host side of the C ABI (include/pzx_gpu.h): table compiler
// (normalisation, classification, SoA/AoS device layout, LUT construction),
// device memory, launch policy and the synchronous / asynchronous entry points.
//
// The table compiler is the SPEC's compile_bit_table re-designed
// for a thread-per-assignment kernel: rows are stored per term in CSR order
// (no dummy padding, P:200-223 is not needed when all lanes walk the same
// term), every row is reduced to a class byte offset + masks + a 4-parameter
// Walsh pattern, and each term carries one fp64 constant that already contains
// every assignment-independent factor.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <thread>
#include <type_traits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <tuple>
#include <string>
#include <vector>

#include "pzx_gpu.h"
#include "pzx_classes.h"
#include "pzx_internal.h"
#include "pzx_slice_dispatch.inc"
#include "pzx_math.hpp"
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges cost nothing unless a tool (nsys / ncu) is attached

using namespace pzxb;

namespace {
// NVTX range scoped to a C-ABI call (SURVEY §5 tracing: upload / evaluate /
// exact / reduce phases show up by name on an nsys or ncu timeline)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

// ------------------------------------------------------------ class table ----
namespace {

struct ClassInfo {
    uint32_t code[4];  // variant (p | q << 1)
    int e;             // sqrt2 exponent, constant over the class's variants
    int lm;            // 1 if every nonzero variant carries lambda or mu
    bool ok;
};

struct Classes {
    ClassInfo c[64];
    bool ok = true;
    Classes() {
        for (int ka = 0; ka < 8; ++ka)
            for (int kb = 0; kb < 8; ++kb) {
                ClassInfo& ci = c[ka * 8 + kb];
                ci.e = -1; ci.lm = -1; ci.ok = true;
                for (int v = 0; v < 4; ++v) {
                    const int p = v & 1, q = v >> 1;
                    Factor f;
                    if (!zw_factor(zw_pair_value(ka + 4 * p, kb + 4 * q), f)) { ci.ok = ok = false; continue; }
                    uint32_t code = 0;
                    if (f.kind == K_ZERO) {
                        code = 1u << kZShift;
                    } else {
                        code = uint32_t(f.j) << kJShift;
                        if (f.kind == K_LAMBDA) code |= 1u << kS1Shift;
                        if (f.kind == K_PI) code |= 1u << kAShift;
                        if (f.kind == K_PIP) code |= 1u << kBShift;
                        const int lm = (f.kind == K_LAMBDA || f.kind == K_MU) ? 1 : 0;
                        // e and lambda/mu membership are class constants
                        if (ci.e < 0) ci.e = f.e; else if (ci.e != f.e) ci.ok = ok = false;
                        if (ci.lm < 0) ci.lm = lm; else if (ci.lm != lm) ci.ok = ok = false;
                    }
                    ci.code[v] = code;
                }
                if (ci.e < 0) { ci.e = 0; ci.lm = 0; }
            }
    }
};

// slice-op tables as the generated PTX sees them (pzx_slice_dispatch.inc)
const int kSliceJbase[kSliceOps] = PZX_SLICE_JBASE;
const int kSliceKindFlags[kSliceOps] = PZX_SLICE_KIND_FLAGS;

bool slice_tables_ok() {
    static const bool ok = [] {
        for (int op = 0; op < kSliceOps; ++op) {
            const SliceOp so = slice_op(op);
            const int flags = (so.lam_tt ? int(kSliceLamFlag) : 0) | (so.pi_tt ? int(kSlicePiFlag) : 0) |
                              (so.pip_tt ? int(kSlicePipFlag) : 0);
            if (so.jbase != kSliceJbase[op] || flags != kSliceKindFlags[op]) return false;
        }
        return true;
    }();
    return ok;
}

const Classes& classes() {
    static const Classes k;
    return k;
}

// ---------------------------------------------------------- normalisation ----
struct PairRow { uint8_t ka, kb; uint64_t psi, phi; };

Quad quad_omega(int k) {
    Quad q;
    zw_to_quad(zw_pow_w(k), q);
    return q;
}

// normalize_subterm, subterm.cpp:51-96 (Lemmas 3-5); returns a pzx_status.
int normalize(uint8_t kind, int psik, uint64_t psim, int phik, uint64_t phim, Quad& constant,
              bool& has_pair, PairRow& row) {
    has_pair = false;
    switch (kind) {
    case PZX_PHASE_PAIR:
        if (!psim && !phim) {
            return zw_to_quad(zw_pair_value(psik, phik), constant) ? PZX_OK : PZX_E_OVERFLOW;
        }
        constant = Quad{1, 0, 0, 0, 0};
        row = {uint8_t(psik), uint8_t(phik), psim, phim};
        has_pair = true;
        return PZX_OK;
    case PZX_NODE:
        if (!psim) return zw_to_quad(zw_add(zw(1, 0, 0, 0), zw_pow_w(psik)), constant) ? PZX_OK : PZX_E_OVERFLOW;
        constant = Quad{1, 0, -1, 0, 1};                     // (1 - i)/2
        row = {uint8_t((psik + 2) & 7), 2, psim, 0};         // pair(psi + pi/2, pi/2)
        has_pair = true;
        return PZX_OK;
    case PZX_PI_PAIR:
        if (phik != 0 && phik != 4) return PZX_E_DOMAIN;     // pauli_image(phi)
        if (!phim && !psim) {
            constant = phik == 4 ? quad_omega(psik) : Quad{1, 0, 0, 0, 0};
            return PZX_OK;
        }
        constant = Quad{1, 0, 0, 0, 1};                      // 1/2
        row = {uint8_t(psik), uint8_t(phik), psim, phim};
        has_pair = true;
        return PZX_OK;
    case PZX_HALF_PI: {
        if (psik != 2 && psik != 6) return PZX_E_DOMAIN;     // proper_clifford_image
        const Quad c = quad_omega(psik == 2 ? 1 : 7);
        if (!psim) { constant = c; return PZX_OK; }
        // pi_pair(base = (8-k, {}), selector = (0, mask)) -> 1/2 pair(base, selector)
        if (!quad_mul(c, Quad{1, 0, 0, 0, 1}, constant)) return PZX_E_OVERFLOW;
        row = {uint8_t((8 - psik) & 7), 0, 0, psim};
        has_pair = true;
        return PZX_OK;
    }
    }
    return PZX_E_DOMAIN;
}

// ---------------------------------------------------------- host table ----
struct HostTable {
    uint32_t n_params = 0;
    std::vector<uint64_t> term_row{0};
    std::vector<Quad> coef;                 // C'_t (exact, normalisation folded)
    std::vector<int32_t> e_t, nlm_t;
    std::vector<double> term_c;             // 2 per term
    std::vector<uint4> rows;                // P <= 32: {psi, phi, code, pat}; P > 32: 2 records per row
    std::vector<uint8_t> swapped;           // row stored with psi/phi exchanged
    std::vector<uint8_t> unit;              // placeholder row of a row-less term
    std::vector<uint4> srows;               // bit-sliced kernel rows (2 per row)
    std::vector<uint4> qrows;               // sorted-batch kernel rows (2 per row, n_params <= 32)
    std::vector<double> sterm_c;            // its term constants (2 per term)
    std::vector<uint8_t> jb_t;              // per term: sum of the rows' slice jbase mod 8 (folded into sterm_c)
    int jb_term = 0;                        // running sum of slice jbase in the open term
    uint32_t kinds_term = 0;                // OR of the open term's row kind flags
    // work statistics behind the algorithmic roofline (pzx_table_slice_stats)
    uint64_t op_rows[kSliceOps] = {};       // rows per bit-sliced op
    uint64_t term_kinds[3] = {};            // terms by epilogue: kind-free, lambda only, with pi / pi'
    bool want_srows = true;                 // build the bit-sliced layout (enumerated batches)
    bool want_qrows = true;                 // build the sorted-batch layout (word lists, n_params <= 32)
    // page layout of the enumerated page kernel (n_params <= 32):
    // kPageSlots-slot pages of 32-byte records, terms never straddle a page
    bool want_prows = true;
    std::vector<uint4> prows;               // 2 x uint4 per slot
    std::vector<uint32_t> term_slot;        // header slot of every term
    std::vector<uint8_t> jp_t;              // per term: the j offset folded into its page constant
    struct PendRow { uint64_t psi, phi; uint32_t op; };
    std::vector<PendRow> pend;              // rows of the open term
    uint32_t page_fill = 0;                 // slots used in the open page
    int64_t last_hdr = -1;                  // slot of the last header written
    uint64_t page_rows[5] = {};             // rows by family: constraint, G, dispatch, dropped, L
    uint64_t page_gsub[kPageGClasses] = {};  // G rows by update class: S2, S6, E0, E2, G1, G3
    uint64_t page_d_ops[kSliceOps] = {};    // dispatch-family rows per op (the roofline's D bodies)
    bool simplify = false;                  // PZX_COMPILE_SIMPLIFY: fold assignment-independent row groups
    uint64_t n_dev_rows() const { return unit.size(); }
    uint64_t genuine_rows() const { return unit.size() - uint64_t(std::count(unit.begin(), unit.end(), 1)); }
    uint32_t max_rows = 0;
};

// Walsh patterns depend only on the low mask bits: tabulated once.
struct WalshTables {
    uint32_t w16[16][2];  // interleaved 2-bit pattern contribution of psi (slot 0) / phi (slot 1)
    uint32_t w32[32];     // bit g = parity(m & g), g < 32
    WalshTables() {
        for (int m = 0; m < 16; ++m) {
            uint32_t a = 0, b = 0;
            for (int g = 0; g < kGray; ++g) {
                a |= uint32_t(__builtin_parity(unsigned(m & g))) << (2 * g);
                b |= uint32_t(__builtin_parity(unsigned(m & g))) << (2 * g + 1);
            }
            w16[m][0] = a;
            w16[m][1] = b;
        }
        for (int m = 0; m < 32; ++m) {
            uint32_t w = 0;
            for (int g = 0; g < 32; ++g) w |= uint32_t(__builtin_parity(unsigned(m & g))) << g;
            w32[m] = w;
        }
    }
};
const WalshTables& walsh() {
    static const WalshTables t;
    return t;
}

uint32_t walsh_pattern(uint64_t psi, uint64_t phi) {
    return walsh().w16[psi & 15][0] | walsh().w16[phi & 15][1];
}

uint32_t walsh32(uint64_t m) { return walsh().w32[m & 31]; }

// Which row layouts a table carries besides the base one (POPC / gray kernels).
// Each bit-sliced layout costs 32 B per row on top of the base 16 (or 32) B:
// PZX_LAYOUTS = base | slice | sorted | all picks them; by default tables up
// to 2^28 rows get all, bigger ones only the sorted-batch layout (random word
// lists are what such tables are evaluated on, and it halves host + HBM use).
void choose_layouts(HostTable& h, uint64_t rows_est) {
    const char* e = std::getenv("PZX_LAYOUTS");
    const std::string s = e ? e : "";
    bool sl, so;
    if (s == "base") sl = so = false;
    else if (s == "slice") sl = true, so = false;
    else if (s == "sorted") sl = false, so = true;
    else if (s == "all") sl = so = true;
    else sl = rows_est <= (uint64_t(1) << 28), so = true;
    h.want_srows = sl;
    h.want_qrows = so && h.n_params <= 32;
    h.want_prows = sl && h.n_params <= 32 && std::getenv("PZX_NO_PAGES") == nullptr;
}

void push_device_row(HostTable& h, uint64_t psi, uint64_t phi, uint32_t code, uint32_t pat, uint8_t sw,
                     uint8_t unit) {
    if (h.n_params <= 32) {
        h.rows.push_back(make_uint4(uint32_t(psi), uint32_t(phi), code, pat));
    } else {  // 32-byte record: masks, then {code, pattern}
        h.rows.push_back(make_uint4(uint32_t(psi), uint32_t(psi >> 32), uint32_t(phi), uint32_t(phi >> 32)));
        h.rows.push_back(make_uint4(code, pat, 0, 0));
    }
    h.swapped.push_back(sw);
    h.unit.push_back(unit);
    const uint32_t cls = (code & kCodeMask) >> 4;
    const uint32_t op = unit ? uint32_t(kSliceUnitOp) : cls * 2u + (phi == 0 ? 1u : 0u);
    h.jb_term += kSliceJbase[op];
    h.op_rows[op] += 1;
    if (h.want_prows && !unit) h.pend.push_back(HostTable::PendRow{psi, phi, op});
    h.kinds_term |= uint32_t(kSliceKindFlags[op]);
    const uint32_t scode = op | uint32_t(kSliceKindFlags[op]);
    if (h.want_srows) {
        h.srows.push_back(make_uint4(uint32_t(psi), uint32_t(phi), scode, walsh32(psi)));
        // P <= 32: the high-mask words carry ~Walsh32 instead, so the kernel
        // forms X = parity ? ~W : W with one predicate + one SEL
        if (h.n_params <= 32)
            h.srows.push_back(make_uint4(walsh32(phi), ~walsh32(psi), ~walsh32(phi), op));
        else
            h.srows.push_back(make_uint4(walsh32(phi), uint32_t(psi >> 32), uint32_t(phi >> 32), op));
    }
    if (h.want_qrows) {
        auto offs = [](uint64_t m, uint32_t k) {  // byte offset of table row (k, nibble k of m), 128-thread stride
            return uint32_t((k * 16 + ((m >> (4 * k)) & 15)) * 512u);
        };
        h.qrows.push_back(make_uint4(uint32_t(psi), uint32_t(phi), scode, op));
        h.qrows.push_back(make_uint4(offs(psi, 0) | (offs(psi, 1) << 16), offs(psi, 2) | (offs(psi, 3) << 16),
                                     offs(phi, 0) | (offs(phi, 1) << 16), offs(phi, 2) | (offs(phi, 3) << 16)));
    }
}

void push_row(HostTable& h, PairRow pr, int& e, int& lm) {
    uint8_t sw = 0;
    if (pr.psi == 0 && pr.phi != 0) {  // V(x,y) = V(y,x): keep a lone parity in psi
        std::swap(pr.ka, pr.kb);
        std::swap(pr.psi, pr.phi);
        sw = 1;
    }
    const int cls = pr.ka * 8 + pr.kb;
    const ClassInfo& ci = classes().c[cls];
    e += ci.e;
    lm += ci.lm;
    push_device_row(h, pr.psi, pr.phi, uint32_t(cls) * 16u, walsh_pattern(pr.psi, pr.phi), sw, 0);
}

// ---- page layout (enumerated page kernel) -------------------
// Every row of a term is put in one of three families by the values of its
// reachable variants (p, q) = parities of (psi, phi) (pzx_classes.h):
//   C (constraint): one parity, one variant zero           -> Z |= X
//   G (generic monomial): value w^(c0 + (k + 4p')(q' ^ inv)) sqrt2^e g, g constant
//       (every class with ka or kb in {0,4}: 28 of 64, ~83 % of the rows of the
//       BASELINE tables)                                   -> branch-free J += (k + 4p')q~
//   L (lambda): one parity, no zero, exactly one lambda/mu variant, k in {0, 4}
//       (terms with < 16 lambda-capable rows)              -> J += k p, S += p ^ inv (L0 then L4)
//   D (dispatch): zero-pair / lambda / pi / pi' rows       -> the generated class bodies
// and rows whose reachable variants are equal are dropped (their w^j goes
// into the term constant like every c0; their sqrt2^e and mu are already in
// E_t / nLM_t). Records (8 x u32), in the order header, C, G, L, D:
//   header: {C_page (double2), nc | n_g1 << 8 | nd << 16 | last_in_page << 24, n_l0 | n_l4 << 8,
//            n_s2 | n_s6 << 8 | n_e0 << 16 | n_e2 << 24, n_g3}
// with the G rows in the order S2, S6, E0, E2, G1, G3 (page_term: by update cost)
//   C: {W ^ zc, ~(W ^ zc), 0, 0, 0, 0, psi, 0}
//   G: {A = W(x) ^ K2, ~A, B = W(y) ^ INV, ~B, K0, K1, x-mask, y-mask}
//   L: {W ^ INV, ~(W ^ INV), W, ~W, K0, K1, psi, K2}
//   D: {W(psi), ~W(psi), W(phi), ~W(phi), op | kind flags, op, psi, phi}
// W = Walsh32 of the mask (bit g = parity(mask & g)); Kc = all ones when bit c of k is set.
struct PageRec { int fam; uint32_t w[8]; int jfold; uint32_t dw[8]; int djfold; };  // dw / djfold: the D form of an L row

PageRec classify_page_row(uint64_t psi, uint64_t phi, uint32_t op) {
    PageRec r{3, {0, 0, 0, 0, 0, 0, 0, 0}, 0, {0, 0, 0, 0, 0, 0, 0, 0}, 0};
    const SliceOp so = slice_op(int(op));
    const bool single = phi == 0;
    const int kinds = so.lam_tt | so.pi_tt | so.pip_tt;
    auto jv = [&](int v) { return (so.jbase + so.w[v]) & 7; };
    const uint32_t Wp = walsh32(psi), Wq = walsh32(phi);
    auto dispatch = [&] {
        r.fam = 3;
        r.w[0] = Wp; r.w[1] = ~Wp; r.w[2] = Wq; r.w[3] = ~Wq;
        r.w[4] = op | uint32_t(kSliceKindFlags[op]); r.w[5] = op; r.w[6] = uint32_t(psi); r.w[7] = uint32_t(phi);
        r.jfold = so.jbase;
        return r;
    };
    // L (single-parity lambda/mu row, one lambda variant, k in {0, 4}): J2 ^= (k/4) p, S += p ^ inv
    if (single && so.lam_tt && !so.pi_tt && !so.pip_tt && !(so.zero_tt & 3) && (so.lam_tt & 3) != 3 &&
        ((jv(1) - jv(0)) & 3) == 0) {
        dispatch();  // keep the D form: the term may have too many lambda rows for the fast counters
        std::memcpy(r.dw, r.w, sizeof r.w);
        r.djfold = r.jfold;
        const int k = (jv(1) - jv(0)) & 7;
        const uint32_t INV = (so.lam_tt & 1) ? ~0u : 0u;  // variant 0 is the lambda one: Lambda = ~p
        r.fam = 5;
        r.w[0] = Wp ^ INV; r.w[1] = ~(Wp ^ INV); r.w[2] = Wp; r.w[3] = ~Wp;
        r.w[4] = (k & 1) ? ~0u : 0u; r.w[5] = (k & 2) ? ~0u : 0u; r.w[6] = uint32_t(psi);
        r.w[7] = (k & 4) ? ~0u : 0u;
        r.jfold = jv(0);
        return r;
    }
    if (kinds) return dispatch();
    if (single) {
        const int z = so.zero_tt & 3;
        if (z == 1 || z == 2) {  // the other variant survives: its w^j is a constant
            const uint32_t zc = z == 2 ? 0u : ~0u;  // Z |= X (variant 1 zero) or ~X (variant 0 zero)
            r.fam = 0;
            r.w[0] = Wp ^ zc; r.w[1] = ~(Wp ^ zc); r.w[6] = uint32_t(psi);
            r.jfold = jv(z == 2 ? 0 : 1);
            return r;
        }
        if (z) return dispatch();
        if (jv(0) == jv(1)) { r.fam = 4; r.jfold = jv(0); return r; }  // assignment-independent
        const int k = (jv(1) - jv(0)) & 7;  // J += k * p: a G row with x = 0, q~ = p
        r.fam = 1;
        const uint32_t K2 = (k & 4) ? ~0u : 0u;
        r.w[0] = K2; r.w[1] = K2; r.w[2] = Wp; r.w[3] = ~Wp;
        r.w[4] = (k & 1) ? ~0u : 0u; r.w[5] = (k & 2) ? ~0u : 0u; r.w[6] = 0; r.w[7] = uint32_t(psi);
        r.jfold = jv(0);
        return r;
    }
    if (so.zero_tt) return dispatch();
    // j(p, q) = c0 + (k + 4p')(q' ^ inv), (p', q') = swap ? (q, p) : (p, q)
    for (int sw = 0; sw < 2; ++sw)
        for (int inv = 0; inv < 2; ++inv)
            for (int k = 0; k < 8; ++k) {
                const int c0 = (jv(0) - k * inv) & 7;  // (p, q) = (0, 0): p' = 0, q' = 0
                bool ok = true;
                for (int v = 0; v < 4 && ok; ++v) {
                    const int p = v & 1, q = v >> 1;
                    const int pp = sw ? q : p, qq = (sw ? p : q) ^ inv;
                    ok = jv(v) == ((c0 + (k + 4 * pp) * qq) & 7);
                }
                if (!ok) continue;
                const uint64_t xm = sw ? phi : psi, ym = sw ? psi : phi;
                const uint32_t K2 = (k & 4) ? ~0u : 0u, INV = inv ? ~0u : 0u;
                r.fam = 1;
                r.w[0] = walsh32(xm) ^ K2; r.w[1] = ~r.w[0];
                r.w[2] = walsh32(ym) ^ INV; r.w[3] = ~r.w[2];
                r.w[4] = (k & 1) ? ~0u : 0u; r.w[5] = (k & 2) ? ~0u : 0u;
                r.w[6] = uint32_t(xm); r.w[7] = uint32_t(ym);
                r.jfold = c0;
                return r;
            }
    return dispatch();
}

void page_pad(HostTable& h) {
    if (h.page_fill == 0) return;
    if (h.last_hdr >= 0) h.prows[2 * size_t(h.last_hdr) + 1].x |= 1u << 24;  // last term of its page
    while (h.page_fill < uint32_t(kPageSlots)) {
        h.prows.push_back(make_uint4(0, 0, 0, 0));
        h.prows.push_back(make_uint4(0, 0, 0, 0));
        ++h.page_fill;
    }
    h.page_fill = 0;
}

// the open term's rows -> one header + C, G, D records; returns its j fold
int page_term(HostTable& h, const C128& cpp) {
    // families in record order: 0 C, 1 G, 2 L, 3 D
    std::vector<PageRec> recs;
    recs.reserve(h.pend.size());
    int n_lam = 0;  // rows that can bump the lambda counter
    for (const auto& pr : h.pend) {
        recs.push_back(classify_page_row(pr.psi, pr.phi, pr.op));
        n_lam += (kSliceKindFlags[pr.op] & int(kSliceLamFlag)) != 0;
    }
    // the L loop keeps the lambda counter in its 4 register planes: a term
    // with >= 16 lambda-capable rows sends its L rows to the dispatch loop
    const bool l_ok = n_lam < 16;
    std::vector<PageRec> fam[4];
    int jf = 0;
    for (size_t i = 0; i < recs.size(); ++i) {
        PageRec r = recs[i];
        if (r.fam == 5 && !l_ok) {
            std::memcpy(r.w, r.dw, sizeof r.w);
            r.jfold = r.djfold;
            r.fam = 3;
        }
        jf += r.jfold;
        if (r.fam == 4) { h.page_rows[3] += 1; continue; }
        const int f = r.fam == 0 ? 0 : r.fam == 1 ? 1 : r.fam == 5 ? 2 : 3;
        h.page_rows[f == 2 ? 4 : f == 3 ? 2 : f] += 1;  // stats order: C, G, D, dropped, L
        if (f == 3) h.page_d_ops[h.pend[i].op] += 1;
        fam[f].push_back(r);
    }
    h.pend.clear();
    // G rows by update cost (k = the record's K0 | K1 << 1; single rows have x-mask 0, X = K2):
    //   0 S2: single, J += 2q        1 S6: single, J += 6q        (J2 ^= q & J1 (~J1); J1 ^= q)
    //   2 E0: k = 0 (and single J += 4q)  J2 ^= X & Y
    //   3 E2: k = 2                       J2 ^= Y & (J1 ^ X); J1 ^= Y
    //   4 G1: k = 1                       J += Y + 4XY (5 LOP3)
    //   5 G3: k = 3, stored with X' = ~X  J -= Y, J += 4X'Y: the G1 update on ~J
    std::vector<PageRec> gsub[kPageGClasses];
    for (PageRec r : fam[1]) {
        const int k = (r.w[4] ? 1 : 0) | (r.w[5] ? 2 : 0);
        const bool single = r.w[6] == 0;
        const int sc = (single && k == 2) ? (r.w[0] ? 1 : 0) : k == 0 ? 2 : k == 2 ? 3 : k == 1 ? 4 : 5;
        if (sc == 5) std::swap(r.w[0], r.w[1]);  // X' = ~X
        gsub[sc].push_back(r);
        h.page_gsub[sc] += 1;
    }
    std::vector<PageRec> lsub[2];  // L rows: k = 0 (S only), k = 4 (J2 ^= p)
    for (const PageRec& r : fam[2]) lsub[r.w[7] ? 1 : 0].push_back(r);
    const uint32_t n = uint32_t(1 + fam[0].size() + fam[1].size() + fam[2].size() + fam[3].size());
    if (n > uint32_t(kPageSlots)) {  // a term must fit one page: no page layout for this table
        h.want_prows = false;
        std::vector<uint4>().swap(h.prows);
        std::vector<uint32_t>().swap(h.term_slot);
        return jf & 7;
    }
    if (h.page_fill + n > uint32_t(kPageSlots)) page_pad(h);
    const C128 wj = zw_to_c128(zw_pow_w(jf & 7));
    const C128 c = cmul(cpp, wj);
    const double re = double(c.re), im = double(c.im);
    uint32_t q[4];
    std::memcpy(q, &re, 8);
    std::memcpy(q + 2, &im, 8);
    h.term_slot.push_back(uint32_t(h.prows.size() / 2));
    h.last_hdr = int64_t(h.prows.size() / 2);
    h.prows.push_back(make_uint4(q[0], q[1], q[2], q[3]));
    h.prows.push_back(make_uint4(uint32_t(fam[0].size()) | uint32_t(gsub[4].size()) << 8 |
                                     uint32_t(fam[3].size()) << 16,
                                 uint32_t(lsub[0].size()) | uint32_t(lsub[1].size()) << 8,
                                 uint32_t(gsub[0].size()) | uint32_t(gsub[1].size()) << 8 |
                                     uint32_t(gsub[2].size()) << 16 | uint32_t(gsub[3].size()) << 24,
                                 uint32_t(gsub[5].size())));
    auto put = [&](const std::vector<PageRec>& v) {
        for (const PageRec& r : v) {
            h.prows.push_back(make_uint4(r.w[0], r.w[1], r.w[2], r.w[3]));
            h.prows.push_back(make_uint4(r.w[4], r.w[5], r.w[6], r.w[7]));
        }
    };
    put(fam[0]);
    for (int sc = 0; sc < kPageGClasses; ++sc) put(gsub[sc]);
    put(lsub[0]);
    put(lsub[1]);
    put(fam[3]);
    h.page_fill += n;
    if (h.page_fill == uint32_t(kPageSlots)) page_pad(h);
    return jf & 7;
}

uint32_t& code_word(HostTable& h, uint64_t i) { return h.n_params <= 32 ? h.rows[i].z : h.rows[2 * i + 1].x; }

// Close a term: a term without assignment-dependent rows gets one unit row
// (class kUnitClass, all-zero codes) so that every term owns >= 1 row of the
// flat row stream; the last row carries kEndFlag and every kSegRows-th row of
// a long term kSegFlag (the kernels flush their 7-bit SWAR fields there).
int finish_term(HostTable& h, const Quad& c, int e, int lm, uint64_t row0) {
    uint64_t n_rows_term = h.n_dev_rows() - row0;
    if (n_rows_term > uint64_t(kMaxTermRows)) return PZX_E_CAPACITY;
    if (n_rows_term == 0) {
        push_device_row(h, 0, 0, uint32_t(kUnitClass) * 16u, 0, 0, 1);
        n_rows_term = 1;
    }
    for (uint64_t i = 0; i + 1 < n_rows_term; ++i)
        if ((i + 1) % kSegRows == 0) code_word(h, row0 + i) |= kSegFlag;
    code_word(h, row0 + n_rows_term - 1) |= kEndFlag;
    if (!h.srows.empty()) h.srows[2 * (row0 + n_rows_term - 1)].z |= kEndFlag;
    if (!h.qrows.empty()) h.qrows[2 * (row0 + n_rows_term - 1)].z |= kEndFlag;
    h.max_rows = std::max<uint32_t>(h.max_rows, uint32_t(n_rows_term));
    h.coef.push_back(c);
    h.e_t.push_back(e);
    h.nlm_t.push_back(lm);
    // C'' = C' * sqrt2^E * mu^nLM, rounded once to double
    f128 re, im;
    quad_to_f128(c, re, im);
    C128 v{re, im};
    for (int i = 0; i < e; ++i) { v.re *= f128_sqrt2(); v.im *= f128_sqrt2(); }
    const C128 mu = zw_to_c128(zw(1, 1, 0, 0));
    for (int i = 0; i < lm; ++i) v = cmul(v, mu);
    h.term_c.push_back(double(v.re));
    h.term_c.push_back(double(v.im));
    h.jb_t.push_back(uint8_t(h.jb_term & 7));
    if (h.want_prows) h.jp_t.push_back(uint8_t(page_term(h, v)));
    const C128 wj = zw_to_c128(zw_pow_w(h.jb_term & 7));  // slice kernel: w^(sum of row jbase)
    const C128 vs = cmul(v, wj);
    h.sterm_c.push_back(double(vs.re));
    h.sterm_c.push_back(double(vs.im));
    h.jb_term = 0;
    h.term_kinds[(h.kinds_term & (kSlicePiFlag | kSlicePipFlag)) ? 2 : (h.kinds_term & kSliceLamFlag) ? 1 : 0] += 1;
    h.kinds_term = 0;
    h.term_row.push_back(h.n_dev_rows());
    return PZX_OK;
}

uint64_t param_mask(uint32_t n) { return n >= 64 ? ~uint64_t(0) : ((uint64_t(1) << n) - 1); }

bool canon_input(const int64_t* q, Quad& out) {
    if (q[4] < INT32_MIN || q[4] > INT32_MAX) return false;
    return quad_canon(q[0], q[1], q[2], q[3], q[4], out);
}

// Post-reduction table simplification (PAPER "Conclusions": pairwise node
// cancellation). Rows of one term that share their (psi, phi)
// masks see the same parities, so a set of them whose product takes the same
// value at every reachable (p, q) is a constant: it is folded into C_t
// exactly, and a zero constant zeroes the whole term. The paper's example
// (1 + w^(k + 4x))(1 + w^(k + 4 + 4x)) = 1 - w^(2k) is the two-row case; k = 0
// with k = 4 gives 0. Greedy: the whole group first, then pairs.
void simplify_term(std::vector<PairRow>& rows, Quad& c, bool& zero_term) {
    zero_term = false;
    if (rows.size() < 2) return;
    auto canon = [](PairRow r) {  // lone parity in psi (V(x,y) = V(y,x))
        if (r.psi == 0 && r.phi != 0) { std::swap(r.ka, r.kb); std::swap(r.psi, r.phi); }
        return r;
    };
    for (auto& r : rows) r = canon(r);
    // value of a row set at (p, q); false on int64 growth (large groups are left alone)
    auto product = [&](const std::vector<size_t>& idx, int p, int q, Zw& out) {
        Zw v = zw(1, 0, 0, 0);
        for (size_t i : idx) {
            v = zw_mul(v, zw_pair_value(rows[i].ka + 4 * p, rows[i].kb + 4 * q));
            for (int k = 0; k < 4; ++k)
                if (v.c[k] > (int64_t(1) << 40) || v.c[k] < -(int64_t(1) << 40)) return false;
        }
        out = v;
        return true;
    };
    auto constant_of = [&](const std::vector<size_t>& idx, Zw& k) {
        const PairRow& r = rows[idx[0]];
        const int np = r.psi ? 2 : 1, nq = r.phi ? 2 : 1;
        if (!product(idx, 0, 0, k)) return false;
        for (int p = 0; p < np; ++p)
            for (int q = 0; q < nq; ++q) {
                Zw v;
                if (!product(idx, p, q, v) || !(v == k)) return false;
            }
        return true;
    };
    std::vector<char> gone(rows.size(), 0);
    auto fold = [&](const std::vector<size_t>& idx, const Zw& k) {
        if (k.zero()) { zero_term = true; return; }
        Quad kq, nc;
        if (!zw_to_quad(k, kq) || !quad_mul(c, kq, nc)) return;  // leave it unfolded on overflow
        c = nc;
        for (size_t i : idx) gone[i] = 1;
    };
    std::vector<size_t> order(rows.size());
    for (size_t i = 0; i < rows.size(); ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
        return rows[a].psi != rows[b].psi ? rows[a].psi < rows[b].psi : rows[a].phi < rows[b].phi;
    });
    for (size_t s = 0; s < order.size() && !zero_term;) {
        size_t e = s + 1;
        while (e < order.size() && rows[order[e]].psi == rows[order[s]].psi && rows[order[e]].phi == rows[order[s]].phi) ++e;
        if (e - s >= 2 && e - s <= 24) {
            std::vector<size_t> grp(order.begin() + long(s), order.begin() + long(e));
            Zw k;
            if (constant_of(grp, k)) {
                fold(grp, k);
            } else {
                for (size_t a = 0; a < grp.size() && !zero_term; ++a)
                    for (size_t b = a + 1; b < grp.size() && !gone[grp[a]]; ++b) {
                        if (gone[grp[b]]) continue;
                        const std::vector<size_t> pr{grp[a], grp[b]};
                        if (constant_of(pr, k)) fold(pr, k);
                    }
            }
        }
        s = e;
    }
    if (zero_term) { rows.clear(); c = Quad{}; return; }
    std::vector<PairRow> kept;
    for (size_t i = 0; i < rows.size(); ++i)
        if (!gone[i]) kept.push_back(rows[i]);
    rows.swap(kept);
}

int compile_expr_range(const pzx_expr_view* v, uint64_t t_begin, uint64_t t_end, HostTable& h,
                       std::string& err) {
    h.n_params = v->n_params;
    const uint64_t allowed = param_mask(v->n_params);
    std::vector<PairRow> pend;
    for (uint64_t t = t_begin; t < t_end; ++t) {
        Quad c;
        if (!canon_input(v->term_scalar + 5 * t, c)) { err = "term scalar out of range"; return PZX_E_OVERFLOW; }
        int e = 0, lm = 0;
        const uint64_t row0 = h.n_dev_rows();
        for (uint64_t j = v->term_offset[t]; j < v->term_offset[t + 1]; ++j) {
            const uint8_t kind = v->kind[j];
            const int psik = v->psi_k[j], phik = v->phi_k ? v->phi_k[j] : 0;
            const uint64_t psim = v->psi_mask[j];
            uint64_t phim = v->phi_mask ? v->phi_mask[j] : 0;
            if (kind > PZX_PI_PAIR || psik > 7 || phik > 7) { err = "subterm kind or phase out of range"; return PZX_E_DOMAIN; }
            if (kind == PZX_NODE || kind == PZX_HALF_PI) phim = 0;  // phi unused (subterm.hpp:25)
            if ((psim | phim) & ~allowed) { err = "subterm mask uses a parameter >= n_params"; return PZX_E_MISSING_PARAM; }
            Quad k;
            bool has = false;
            PairRow pr{};
            int st = normalize(kind, psik, psim, phik, phim, k, has, pr);
            if (st) { err = "normalize_subterm: kind invariant violated"; return st; }
            Quad nc;
            if (!quad_mul(c, k, nc)) { err = "term constant overflow"; return PZX_E_OVERFLOW; }
            c = nc;
            if (has) {
                if (h.simplify) pend.push_back(pr);
                else push_row(h, pr, e, lm);
            }
        }
        if (h.simplify) {
            bool zero_term = false;
            simplify_term(pend, c, zero_term);
            for (const PairRow& pr : pend) push_row(h, pr, e, lm);
            pend.clear();
        }
        int st = finish_term(h, c, e, lm, row0);
        if (st) { err = "term has more rows than supported"; return st; }
    }
    return PZX_OK;
}

// Append part (compiled with term_row starting at 0) to h.
void merge_into(HostTable& h, HostTable& part) {
    const uint64_t base = h.n_dev_rows();
    for (size_t i = 1; i < part.term_row.size(); ++i) h.term_row.push_back(base + part.term_row[i]);
    auto app = [](auto& dst, auto& src) {
        dst.insert(dst.end(), src.begin(), src.end());
        std::vector<typename std::decay_t<decltype(src)>::value_type>().swap(src);
    };
    app(h.coef, part.coef);
    app(h.e_t, part.e_t);
    app(h.nlm_t, part.nlm_t);
    app(h.term_c, part.term_c);
    app(h.sterm_c, part.sterm_c);
    app(h.jb_t, part.jb_t);
    app(h.rows, part.rows);
    app(h.srows, part.srows);
    app(h.qrows, part.qrows);
    app(h.swapped, part.swapped);
    app(h.unit, part.unit);
    h.max_rows = std::max(h.max_rows, part.max_rows);
    for (int i = 0; i < kSliceOps; ++i) h.op_rows[i] += part.op_rows[i];
    // pages: both sides padded to whole pages, the part's slots rebased
    if (h.want_prows && part.want_prows) {
        page_pad(h);
        page_pad(part);
        const uint32_t base_slot = uint32_t(h.prows.size() / 2);
        for (uint32_t ts : part.term_slot) h.term_slot.push_back(base_slot + ts);
        app(h.prows, part.prows);
        app(h.jp_t, part.jp_t);
        if (part.last_hdr >= 0) h.last_hdr = int64_t(base_slot) + part.last_hdr;
        for (int i = 0; i < 5; ++i) h.page_rows[i] += part.page_rows[i];
        for (int i = 0; i < kPageGClasses; ++i) h.page_gsub[i] += part.page_gsub[i];
        for (int i = 0; i < kSliceOps; ++i) h.page_d_ops[i] += part.page_d_ops[i];
    } else if (h.want_prows) {
        h.want_prows = false;
        std::vector<uint4>().swap(h.prows);
        std::vector<uint32_t>().swap(h.term_slot);
    }
    for (int i = 0; i < 3; ++i) h.term_kinds[i] += part.term_kinds[i];
}

// compile_bit_table over term ranges in parallel (terms are independent),
// merged in term order: the table is identical to a serial compile.
int compile_expr(const pzx_expr_view* v, HostTable& h, std::string& err) {
    if (v->n_params > 64) { err = "parameter capacity (64) exceeded"; return PZX_E_DOMAIN; }
    h.n_params = v->n_params;
    const uint64_t m = v->n_terms;
    const uint64_t rows_est = m ? v->term_offset[m] - v->term_offset[0] + m : 0;
    choose_layouts(h, rows_est);
    unsigned nth = std::max(1u, std::thread::hardware_concurrency());
    nth = unsigned(std::min<uint64_t>(nth, std::max<uint64_t>(1, m / 2048)));
    if (nth <= 1) {
        const int st = compile_expr_range(v, 0, m, h, err);
        if (!st && h.want_prows) page_pad(h);
        return st;
    }
    std::vector<HostTable> parts(nth);
    std::vector<int> st(nth, PZX_OK);
    std::vector<std::string> errs(nth);
    std::vector<std::thread> th;
    for (unsigned i = 0; i < nth; ++i) {
        parts[i].n_params = h.n_params;
        parts[i].want_srows = h.want_srows;
        parts[i].want_qrows = h.want_qrows;
        parts[i].want_prows = h.want_prows;
        parts[i].simplify = h.simplify;
        th.emplace_back([&, i] {
            st[i] = compile_expr_range(v, m * i / nth, m * (i + 1) / nth, parts[i], errs[i]);
        });
    }
    for (auto& x : th) x.join();
    for (unsigned i = 0; i < nth; ++i)
        if (st[i]) { err = errs[i]; return st[i]; }
    for (unsigned i = 0; i < nth; ++i) {
        if (i == 0) h.want_prows = parts[0].want_prows;
        merge_into(h, parts[i]);
    }
    if (h.want_prows) page_pad(h);
    return PZX_OK;
}

int compile_rows(const pzx_table_view* v, HostTable& h, std::string& err) {
    if (v->n_params > 64) { err = "parameter capacity (64) exceeded"; return PZX_E_DOMAIN; }
    h.n_params = v->n_params;
    choose_layouts(h, v->n_terms ? v->term_row_offset[v->n_terms] - v->term_row_offset[0] + v->n_terms : 0);
    const uint64_t allowed = param_mask(v->n_params);
    for (uint64_t t = 0; t < v->n_terms; ++t) {
        Quad c;
        if (!canon_input(v->term_coef + 5 * t, c)) { err = "term coefficient out of range"; return PZX_E_OVERFLOW; }
        int e = 0, lm = 0;
        const uint64_t row0 = h.n_dev_rows();
        for (uint64_t r = v->term_row_offset[t]; r < v->term_row_offset[t + 1]; ++r) {
            if (v->k_alpha[r] > 7 || v->k_beta[r] > 7) { err = "phase index out of [0,7]"; return PZX_E_DOMAIN; }
            if ((v->psi_mask[r] | v->phi_mask[r]) & ~allowed) { err = "row mask uses a parameter >= n_params"; return PZX_E_MISSING_PARAM; }
            PairRow pr{v->k_alpha[r], v->k_beta[r], v->psi_mask[r], v->phi_mask[r]};
            if (!pr.psi && !pr.phi) {  // assignment independent: fold (push_subterm, diagram.cpp:114-120)
                Quad k, nc;
                if (!zw_to_quad(zw_pair_value(pr.ka, pr.kb), k) || !quad_mul(c, k, nc)) { err = "term constant overflow"; return PZX_E_OVERFLOW; }
                c = nc;
                continue;
            }
            push_row(h, pr, e, lm);
        }
        int st = finish_term(h, c, e, lm, row0);
        if (st) { err = "term has more rows than supported"; return st; }
    }
    if (h.want_prows) page_pad(h);
    return PZX_OK;
}

std::vector<unsigned char> build_lut(uint32_t max_rows, LutLayout& L) {
    const int M = int(std::max<uint32_t>(max_rows, 1));
    auto align16 = [](uint32_t x) { return (x + 15u) & ~15u; };
    L.max_rows = M;
    L.codes_off = 0;
    L.om_off = align16(L.codes_off + kCodeClasses * 4 * 4);
    L.u_off = align16(L.om_off + 8 * 16);
    L.p3_off = align16(L.u_off + 8 * (M + 1));
    L.pd_off = align16(L.p3_off + 8 * (M / 2 + 1));
    L.sab_off = align16(L.pd_off + 16 * (2 * M + 1));
    L.uz_off = align16(L.sab_off + 16 * 256);
    L.bytes = align16(L.uz_off + 8 * 32);
    std::vector<unsigned char> blob(L.bytes, 0);
    uint32_t* codes = reinterpret_cast<uint32_t*>(blob.data() + L.codes_off);
    for (int c = 0; c < 64; ++c)
        for (int v = 0; v < 4; ++v) codes[c * 4 + v] = classes().c[c].code[v];
    for (int v = 0; v < 4; ++v) codes[kUnitClass * 4 + v] = 0;  // unit row: value 1
    double* om = reinterpret_cast<double*>(blob.data() + L.om_off);
    for (int j = 0; j < 8; ++j) {
        const C128 w = zw_to_c128(zw_pow_w(j));
        om[2 * j] = double(w.re);
        om[2 * j + 1] = double(w.im);
    }
    double* u = reinterpret_cast<double*>(blob.data() + L.u_off);
    f128 x = 1;
    for (int s = 0; s <= M; ++s) { u[s] = double(x); x *= (f128_sqrt2() - 1); }
    double* p3 = reinterpret_cast<double*>(blob.data() + L.p3_off);
    x = 1;
    for (int m = 0; m <= M / 2; ++m) { p3[m] = double(x); x *= 3; }
    double* pd = reinterpret_cast<double*>(blob.data() + L.pd_off);
    const C128 pi = zw_to_c128(zw_generator(K_PI)), pip = zw_to_c128(zw_generator(K_PIP));
    C128 a{1, 0}, b{1, 0};
    for (int d = 0; d <= M; ++d) {
        pd[2 * (M + d)] = double(a.re); pd[2 * (M + d) + 1] = double(a.im);
        pd[2 * (M - d)] = double(b.re); pd[2 * (M - d) + 1] = double(b.im);
        a = cmul(a, pi);
        b = cmul(b, pip);
    }
    // (sqrt2-1)^s pi^a pi'^b for s < 16, a, b < 4 (slice-kernel fast path),
    // each rounded once from f128, at index sab_index(s, a, b): the low three
    // bits of s XOR (a | b0 << 2), so that assignments with the same s but
    // different pi counts read different shared-memory bank groups (the
    // kernels form that index for free by XOR-ing the bit planes); a = b = 0
    // keeps index s
    double* sab = reinterpret_cast<double*>(blob.data() + L.sab_off);
    for (int is = 0; is < 16; ++is)
        for (int ia = 0; ia < 4; ++ia)
            for (int ib = 0; ib < 4; ++ib) {
                C128 v{1, 0};
                for (int k = 0; k < ia; ++k) v = cmul(v, pi);
                for (int k = 0; k < ib; ++k) v = cmul(v, pip);
                for (int k = 0; k < is; ++k) v = cmul(v, C128{f128_sqrt2() - 1, 0});
                const int i = ((is & 7) ^ (ia | ((ib & 1) << 2))) | (is & 8) | (ia << 4) | (ib << 6);
                sab[2 * i] = double(v.re);
                sab[2 * i + 1] = double(v.im);
            }
    // (sqrt2-1)^s for s < 16 at s, zeros at 16..31 (Z-marked assignments: index s | 16)
    double* uz = reinterpret_cast<double*>(blob.data() + L.uz_off);
    x = 1;
    for (int is = 0; is < 16; ++is) { uz[is] = double(x); x *= (f128_sqrt2() - 1); }
    return blob;
}

}  // namespace

// ---------------------------------------------------------------- handles ----
struct pzx_ctx {
    int device = 0;
    int n_sm = 148;
    cudaStream_t stream = nullptr;
    std::string err;
    uint64_t launches = 0;
    // scratch (grown on demand, freed with the context)
    void* d_asg = nullptr; size_t asg_cap = 0;
    void* d_amp = nullptr; size_t amp_cap = 0;
    void* d_prob = nullptr; size_t prob_cap = 0;
    void* d_partial = nullptr; size_t partial_cap = 0;
    void* d_chunks = nullptr; size_t chunks_cap = 0;
    void* d_xout = nullptr; size_t xout_cap = 0;  // exact outputs + overflow flags
    void* d_dbg = nullptr; size_t dbg_cap = 0;
    void* d_sort = nullptr; size_t sort_cap = 0;
    // per-call scratch of the evaluation kernels (sort buffers, chunk bounds,
    // term-chunk partials): stream-ordered allocations from this pool on the
    // call's stream, so concurrent pzx_evaluate_device calls on different
    // streams never share a buffer (memory is recycled once the freeing
    // stream has passed the free)
    cudaMemPool_t pool = nullptr;
    // what the last evaluation launched (pzx_last_kernel; bench.py's roofline)
    int last_kernel = 0, last_groups = 0, last_chunks = 0;
    // small host-buffer calls repeated with the same arguments replay one CUDA
    // graph (H2D + kernels + D2H) instead of re-issuing every API call
    struct GraphEntry {
        cudaGraphExec_t exec = nullptr;
        uint64_t launches = 0;  // this library's kernels per replay
        int kernel = 0, groups = 0, chunks = 0;
        void *d_asg = nullptr, *d_amp = nullptr, *d_prob = nullptr;  // scratch the graph was captured on
        int seen = 0;
    };
    std::map<std::vector<uint64_t>, GraphEntry> graphs;
};

std::atomic<uint64_t> g_table_gen{1};

struct pzx_table {
    pzx_ctx* ctx = nullptr;
    int device = 0;
    uint64_t gen = g_table_gen.fetch_add(1);  // unique per table object (graph-cache keys)
    DevTable dev;
    HostTable host;
    void* d_rows = nullptr;
    void* d_term_row = nullptr;
    void* d_term_c = nullptr;
    void* d_lut = nullptr;
    void* d_srows = nullptr;
    void* d_sterm_c = nullptr;
    void* d_qrows = nullptr;
    void* d_prows = nullptr;
    void* d_term_slot = nullptr;
    void* d_exact = nullptr;  // exact-evaluation tables (built on first pzx_evaluate_exact)
    ExactDev exact;
    // device copies of term-chunk bounds, keyed by (term range, chunk count):
    // immutable once written, so any stream may read them; saves a pageable
    // H2D copy per call (it dominates small, launch-bound batches)
    std::mutex chunk_mu;
    std::map<std::tuple<uint64_t, uint64_t, int>, void*> chunk_cache;
};

namespace {

pzx_status set_err(pzx_ctx* ctx, int st, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return pzx_status(st);
}

pzx_status cuda_err(pzx_ctx* ctx, cudaError_t e, const char* where) {
    if (e == cudaSuccess) return PZX_OK;
    return set_err(ctx, e == cudaErrorMemoryAllocation ? PZX_E_OOM : PZX_E_CUDA,
                   std::string(where) + ": " + cudaGetErrorString(e));
}

cudaError_t grow(void** p, size_t* cap, size_t need) {
    if (need <= *cap) return cudaSuccess;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    cudaError_t e = cudaMalloc(p, need);
    if (e == cudaSuccess) *cap = need;
    return e;
}

template <class T>
cudaError_t upload_vec(void** dst, const std::vector<T>& v) {
    const size_t bytes = std::max<size_t>(v.size() * sizeof(T), 16);
    cudaError_t e = cudaMalloc(dst, bytes);
    if (e != cudaSuccess) return e;
    if (!v.empty()) e = cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
    return e;
}

pzx_status finish_upload(pzx_ctx* ctx, std::unique_ptr<pzx_table>& t, pzx_table** out) {
    NvtxRange nv("pzx.table_upload");
    HostTable& h = t->host;
    pzx_status st;
    if ((st = cuda_err(ctx, cudaSetDevice(ctx->device), "cudaSetDevice"))) return st;
    if ((st = cuda_err(ctx, upload_vec(&t->d_rows, h.rows), "upload rows"))) return st;
    if ((st = cuda_err(ctx, upload_vec(&t->d_term_row, h.term_row), "upload term offsets"))) return st;
    if ((st = cuda_err(ctx, upload_vec(&t->d_term_c, h.term_c), "upload term constants"))) return st;
    const bool seg_ok = h.max_rows <= uint32_t(kSegRows) && slice_tables_ok();
    const bool slice_ok = seg_ok && h.want_srows;
    const bool sorted_ok = seg_ok && h.want_qrows && h.n_params <= 32;
    if (slice_ok && (st = cuda_err(ctx, upload_vec(&t->d_srows, h.srows), "upload slice rows"))) return st;
    if ((slice_ok || sorted_ok) &&
        (st = cuda_err(ctx, upload_vec(&t->d_sterm_c, h.sterm_c), "upload slice constants"))) return st;
    if (sorted_ok && (st = cuda_err(ctx, upload_vec(&t->d_qrows, h.qrows), "upload sorted-kernel rows"))) return st;
    const bool page_ok = slice_ok && h.want_prows && !h.prows.empty() && h.term_slot.size() == h.coef.size();
    if (page_ok && (st = cuda_err(ctx, upload_vec(&t->d_prows, h.prows), "upload page rows"))) return st;
    if (page_ok && (st = cuda_err(ctx, upload_vec(&t->d_term_slot, h.term_slot), "upload term slots"))) return st;
    LutLayout L;
    std::vector<unsigned char> blob = build_lut(h.max_rows, L);
    if ((st = cuda_err(ctx, upload_vec(&t->d_lut, blob), "upload lut"))) return st;
    DevTable& d = t->dev;
    d.rows = static_cast<const uint4*>(t->d_rows);
    d.term_row = static_cast<const uint64_t*>(t->d_term_row);
    d.term_c = static_cast<const double2*>(t->d_term_c);
    d.lut = static_cast<const unsigned char*>(t->d_lut);
    d.lut_layout = L;
    d.n_terms = h.coef.size();
    d.n_rows = h.n_dev_rows();
    d.n_params = h.n_params;
    d.max_rows = h.max_rows;
    d.p64 = h.n_params > 32;
    d.slice_ok = slice_ok ? 1 : 0;
    d.srows = static_cast<const uint4*>(t->d_srows);
    d.sterm_c = static_cast<const double2*>(t->d_sterm_c);
    d.sorted_ok = sorted_ok ? 1 : 0;
    d.qrows = static_cast<const uint4*>(t->d_qrows);
    d.page_ok = page_ok ? 1 : 0;
    d.prows = static_cast<const uint4*>(t->d_prows);
    d.term_slot = static_cast<const uint32_t*>(t->d_term_slot);
    d.n_pages = page_ok ? h.prows.size() / (2 * size_t(kPageSlots)) : 0;
    t->ctx = ctx;
    t->device = ctx->device;
    // the device owns the row layouts now; keep only what host-side queries use
    std::vector<uint4>().swap(h.rows);
    std::vector<uint4>().swap(h.srows);
    std::vector<uint4>().swap(h.qrows);
    std::vector<uint4>().swap(h.prows);
    std::vector<double>().swap(h.term_c);
    std::vector<double>().swap(h.sterm_c);
    *out = t.release();
    return PZX_OK;
}

// term-split chunk boundaries balanced by row count
void chunk_bounds(const HostTable& h, uint64_t tb, uint64_t te, int chunks, std::vector<uint64_t>& b) {
    b.assign(size_t(chunks) + 1, te);
    b[0] = tb;
    const uint64_t r0 = h.term_row[tb], r1 = h.term_row[te];
    for (int c = 1; c < chunks; ++c) {
        const uint64_t target = r0 + (r1 - r0) * uint64_t(c) / uint64_t(chunks);
        auto it = std::lower_bound(h.term_row.begin() + tb, h.term_row.begin() + te, target);
        uint64_t k = uint64_t(it - h.term_row.begin());
        b[c] = std::max(b[c - 1], std::min(k, te));
    }
}

// grid waves the term-chunk policy aims for, in units of n_sm x
// resident_ctas_per_sm (tuning knob PZX_WAVES). Measured on C2 / C3
// (profiles/r01/waves*.log): 8 -> 64 is +9 % / +5 % (C2: grid 256 x 5 ->
// 256 x 37 CTAs, i.e. ~2 -> ~16 waves of the 4 TMEM CTAs an SM holds: the
// last-wave tail shrinks), while the warp-chunk kernel (C4) loses 35 % with
// more chunks and keeps 8.
// target grid size in waves of resident CTAs (term chunks x assignment blocks);
// the page kernel's CTAs vary more in duration (warp-level zero skips), so its
// grid is finer: C2 37 -> 74 term chunks, 190.8 -> 188.3 ms (PZX_WAVES sweep,
// profiles/README.md r02)
int grid_waves(int kc) {
    static const int v = [] {
        const char* e = std::getenv("PZX_WAVES");
        return e ? std::max(1, std::atoi(e)) : 0;
    }();
    if (kc == KC_SLICEWC) return 8;
    if (v) return v;
    return kc == KC_PAGE ? 128 : 64;
}

// chunk-partial scratch bound (bytes); tuning knob PZX_PARTIAL_MIB
uint64_t partial_cap() {
    static const uint64_t v = [] {
        const char* e = std::getenv("PZX_PARTIAL_MIB");
        return (e ? std::max<uint64_t>(1, std::strtoull(e, nullptr, 10)) : uint64_t(2048)) << 20;
    }();
    return v;
}

uint64_t min_chunk_rows() {
    static const uint64_t v = [] {
        const char* e = std::getenv("PZX_MIN_CHUNK_ROWS");
        return e ? std::max<uint64_t>(1, std::strtoull(e, nullptr, 10)) : uint64_t(512);
    }();
    return v;
}

// Stream-ordered scratch of one evaluation call: every buffer comes from the
// context's pool on the call's stream and is released with cudaFreeAsync on
// the same stream when the call returns (after its kernels are enqueued), so
// the memory cannot be handed to another stream before those kernels finish.
struct CallScratch {
    pzx_ctx* ctx;
    cudaStream_t s;
    std::vector<void*> bufs;
    CallScratch(pzx_ctx* c, cudaStream_t st) : ctx(c), s(st) {}
    CallScratch(const CallScratch&) = delete;
    CallScratch& operator=(const CallScratch&) = delete;
    pzx_status alloc(size_t bytes, void** p) {
        *p = nullptr;
        cudaError_t e = cudaMallocFromPoolAsync(p, std::max<size_t>(bytes, 16), ctx->pool, s);
        if (e != cudaSuccess) return cuda_err(ctx, e, "stream-ordered scratch");
        bufs.push_back(*p);
        return PZX_OK;
    }
    ~CallScratch() {
        for (void* p : bufs) cudaFreeAsync(p, s);
    }
};

pzx_status run_eval(pzx_ctx* ctx, const pzx_table* t, LaunchReq& r, uint32_t flags) {
    NvtxRange nv("pzx.evaluate");
    if (!ctx || !t) return PZX_E_INVALID;
    if (t->device < 0) return set_err(ctx, PZX_E_INVALID, "host-only table (pzx_table_compile_host)");
    if (t->device != ctx->device) return set_err(ctx, PZX_E_INVALID, "table belongs to another device");
    if (r.term_end > t->dev.n_terms) r.term_end = t->dev.n_terms;
    if (r.term_begin > r.term_end) return set_err(ctx, PZX_E_INVALID, "bad term range");
    r.kernel = (flags & PZX_KERNEL_GENERAL) ? KC_GENERAL
             : (flags & PZX_KERNEL_GRAY)    ? KC_GRAY
             : (flags & PZX_KERNEL_SLICE)   ? KC_SLICE
             : (flags & PZX_KERNEL_SLICE_RAND) ? KC_SLICER
             : (flags & PZX_KERNEL_SORTED)  ? KC_SORTED
             : (flags & PZX_KERNEL_SLICE2)  ? KC_SLICE2
             : (flags & PZX_KERNEL_PAGE)    ? KC_PAGE
                                            : KC_AUTO;
    if (r.kernel != KC_AUTO && !kernel_supported(t->dev, r, r.kernel))
        return set_err(ctx, PZX_E_INVALID, "requested kernel does not support this batch / table "
                                           "(enumerated kernels need a contiguous batch starting at a multiple "
                                           "of 16 (gray), 32 (slice) or 64 (slice2); slice needs terms of <= 127 rows)");
    if (r.accumulate && !r.d_amp)
        return set_err(ctx, PZX_E_INVALID, "PZX_ACCUMULATE needs an amplitude buffer (d_amp)");
    KernelChoice kc = choose_kernel(t->dev, r);
    pzx_status st;
    if ((st = cuda_err(ctx, cudaSetDevice(ctx->device), "cudaSetDevice"))) return st;
    CallScratch scratch(ctx, r.stream);  // freed (stream-ordered) when this call returns
    void* sort_buf = nullptr;
    constexpr uint64_t kSortedMaxBatch = uint64_t(1) << 26;  // bounds the sort / regroup scratch (~70 B per word)
    if (kc == KC_SORTED && r.n > kSortedMaxBatch) {
        // huge word lists: independent sub-batches (each sorted on its own)
        const LaunchReq whole = r;
        for (uint64_t o = 0; o < whole.n; o += kSortedMaxBatch) {
            LaunchReq s = whole;
            s.n = std::min(kSortedMaxBatch, whole.n - o);
            s.d_asg = whole.d_asg + o;
            s.d_amp = whole.d_amp ? whole.d_amp + o : nullptr;
            s.d_prob = whole.d_prob ? whole.d_prob + o : nullptr;
            if ((st = run_eval(ctx, t, s, flags))) return st;
        }
        return PZX_OK;
    }
    if (kc == KC_SORTED) {  // sort word|position pairs; results are scattered back by position
        if (!r.d_asg) return set_err(ctx, PZX_E_INVALID, "sorted kernel needs an explicit word list");
        if ((st = scratch.alloc(sort_scratch_bytes(r.n) + 256, &sort_buf))) return st;
        if ((st = cuda_err(ctx, sort_words(r.d_asg, r.n, t->dev.n_params, sort_buf, &r.d_sorted, &r.d_perm,
                                           r.stream, &ctx->launches), "sort words"))) return st;
        // regroup: every thread's 32 words must share their high part (bits >= 4 G);
        // 16 table bits for dense batches, 24 (wide tables) when 16 would pad by
        // more than 25 % (sparse batches such as 2^16 random 32-bit words)
        void* gs = static_cast<unsigned char*>(sort_buf) + sort_base_bytes(r.n);
        uint64_t slots = 0;
        int groups = kSortedGroups;
        if ((st = cuda_err(ctx, group_slots(r.d_sorted, r.n, 4 * kSortedGroups, gs, &slots, r.stream, &ctx->launches), "group"))) return st;
        if (slots > r.n + r.n / 4 + 32) {
            groups = kSortedGroupsWide;
            if ((st = cuda_err(ctx, group_slots(r.d_sorted, r.n, 4 * kSortedGroupsWide, gs, &slots, r.stream, &ctx->launches), "group"))) return st;
        }
        if (slots > 2 * r.n + 32) {  // sparser than half-filled groups: the POPC kernel is faster
            if (r.kernel == KC_SORTED)
                return set_err(ctx, PZX_E_INVALID, "sorted kernel: batch too sparse (high-part groups under half full)");
            kc = KC_GENERAL;
            r.d_sorted = nullptr;
            r.d_perm = nullptr;
        } else {
            const uint64_t* pw = nullptr;
            const uint32_t* pp = nullptr;
            if ((st = cuda_err(ctx, group_sorted(r.d_sorted, r.d_perm, r.n, 4 * groups, gs, &pw, &pp, &slots, r.stream, &ctx->launches), "group words"))) return st;
            r.d_sorted = pw;
            r.d_perm = pp;
            r.n = slots;  // the kernel and the chunk reduction run over the padded slots
            r.sorted_groups = groups;
        }
    }
    // grid policy: split the terms into chunks so that the grid is >= kWaves
    // full waves of resident CTAs (keeps the last-wave tail small); chunk
    // partials are bounded by partial_cap() (2 GiB by default, PZX_PARTIAL_MIB)
    const int ablocks = grid_assign_blocks(t->dev, r, kc);
    const uint64_t nterms = r.term_end - r.term_begin;
    int chunks = 1;
    const int kWaves = grid_waves(kc);
    const int wave = ctx->n_sm * resident_ctas_per_sm(t->dev, kc, slice_threads(r), r.sorted_groups);
    const int target = kWaves * wave;
    if (ablocks < target && nterms > 1) {
        uint64_t c = (uint64_t(target) + ablocks - 1) / ablocks;
        c = std::min<uint64_t>(c, kc == KC_SLICEWC ? std::max<uint64_t>(1, nterms / kWarpChunksHost) : nterms);
        c = std::min<uint64_t>(c, std::max<uint64_t>(1, partial_cap() / (r.n * 16 + 1)));
        // small tables: a chunk below kMinChunkRows rows costs more in per-CTA setup
        // (table staging, TMEM allocation, the partial it writes) than it saves
        const uint64_t total_rows = t->host.term_row.size() > r.term_end
                                        ? t->host.term_row[r.term_end] - t->host.term_row[r.term_begin]
                                        : t->dev.n_rows;
        const uint64_t per = (kc == KC_SLICEWC ? uint64_t(kWarpChunksHost) : uint64_t(1)) * min_chunk_rows();
        c = std::min<uint64_t>(c, std::max<uint64_t>(1, total_rows / per));
        chunks = int(std::min<uint64_t>(c, 65535));
        // round the grid up to whole waves when that does not need more chunks than terms
        const uint64_t total = uint64_t(chunks) * ablocks;
        if (total % wave) {
            const uint64_t want = (total / wave + 1) * wave;
            const uint64_t c2 = (want + ablocks - 1) / ablocks;
            if (c2 <= nterms && c2 <= 65535 && c2 * (r.n * 16) <= partial_cap()) chunks = int(c2);
        }
    }
    if (kc == KC_SLICEWC) chunks *= kWarpChunksHost;  // 4 warp chunks per CTA row, always partials
    r.n_chunks = chunks;
    if (chunks > 1) {
        void* d_b = nullptr;
        void* d_p = nullptr;
        {
            pzx_table* mt = const_cast<pzx_table*>(t);
            std::lock_guard<std::mutex> lock(mt->chunk_mu);
            const auto key = std::make_tuple(r.term_begin, r.term_end, chunks);
            auto it = mt->chunk_cache.find(key);
            if (it != mt->chunk_cache.end()) {
                d_b = it->second;
            } else {
                std::vector<uint64_t> b;
                chunk_bounds(t->host, r.term_begin, r.term_end, chunks, b);
                if ((st = cuda_err(ctx, cudaMalloc(&d_b, b.size() * 8), "alloc chunks"))) return st;
                if ((st = cuda_err(ctx, cudaMemcpy(d_b, b.data(), b.size() * 8, cudaMemcpyHostToDevice), "copy chunks"))) {
                    cudaFree(d_b);
                    return st;
                }
                if (mt->chunk_cache.size() >= 64) {  // bounded: term ranges vary in split runs
                    cudaDeviceSynchronize();  // no call in flight may still read an evicted bound
                    for (auto& kv : mt->chunk_cache) cudaFree(kv.second);
                    mt->chunk_cache.clear();
                }
                mt->chunk_cache.emplace(key, d_b);
            }
        }
        if ((st = scratch.alloc(size_t(chunks) * r.n * 16, &d_p))) return st;
        r.d_chunk_terms = static_cast<const uint64_t*>(d_b);
        r.d_partial = static_cast<double2*>(d_p);
    }
    if (t->dev.lut_layout.bytes > 200 * 1024) return set_err(ctx, PZX_E_CAPACITY, "LUT exceeds 200 KiB");
    ctx->last_kernel = int(kc);
    ctx->last_groups = kc == KC_SORTED ? r.sorted_groups : 0;
    ctx->last_chunks = chunks;
    if ((st = cuda_err(ctx, launch_evaluate(t->dev, r, kc, &ctx->launches), "evaluate kernel"))) return st;
    return PZX_OK;
}

// --------------------------------------------------- exact evaluation ----
// Z[w] products with the device kernel's operand rule (x within 62 bits, every
// product coefficient within int64), so a table entry the host accepts is one
// the kernel can multiply.
bool zw_fits62(const Zw& z) {
    for (int i = 0; i < 4; ++i)
        if (z.c[i] >= (int64_t(1) << 62) || z.c[i] <= -(int64_t(1) << 62)) return false;
    return true;
}
bool zw_mul_chk(const Zw& x, const Zw& y, Zw& out) {
    if (!zw_fits62(x)) return false;
    i128 t[4] = {0, 0, 0, 0};
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            const i128 p = i128(x.c[i]) * y.c[j];
            if (i + j < 4) t[i + j] += p; else t[i + j - 4] -= p;
        }
    for (int k = 0; k < 4; ++k) {
        if (t[k] > INT64_MAX || t[k] < INT64_MIN) return false;
        out.c[k] = int64_t(t[k]);
    }
    return true;
}

// Per-term constants C'_t * sqrt2^E_t = F_t * 2^fx_t (F_t in Z[w], divided by
// 2 while even), nLM_t, and the power tables of the assignment-dependent factors.
pzx_status build_exact(pzx_ctx* ctx, pzx_table* t) {
    const HostTable& h = t->host;
    const uint64_t m = h.coef.size();
    const uint32_t M = std::max<uint32_t>(h.max_rows, 1);
    std::vector<int64_t> ft(4 * m, 0);
    std::vector<int32_t> fx(m, 0);
    std::vector<uint32_t> nlm(m, 0);
    const Zw s2 = zw(0, 1, 0, -1);
    for (uint64_t i = 0; i < m; ++i) {
        const Quad& c = h.coef[i];
        // a + b sqrt2 + i(c + d sqrt2) = a + (b + d) w + c w^2 + (d - b) w^3
        const i128 c1 = i128(c.b) + c.d, c3 = i128(c.d) - c.b;
        bool ok = c1 <= INT64_MAX && c1 >= INT64_MIN && c3 <= INT64_MAX && c3 >= INT64_MIN;
        Zw f = ok ? zw(c.a, int64_t(c1), c.c, int64_t(c3)) : Zw{};
        int64_t e = -int64_t(c.e) + h.e_t[i] / 2;  // sqrt2^(2q) = 2^q
        if (ok && (h.e_t[i] & 1)) ok = zw_mul_chk(s2, f, f);
        while (ok && !f.zero() && ((f.c[0] | f.c[1] | f.c[2] | f.c[3]) & 1) == 0) {
            for (int k = 0; k < 4; ++k) f.c[k] /= 2;
            ++e;
        }
        if (ok && f.zero()) e = 0;
        ok = ok && e > INT32_MIN / 2 && e < INT32_MAX / 2;
        for (int k = 0; k < 4; ++k) ft[4 * i + k] = ok ? f.c[k] : 0;
        fx[i] = ok ? int32_t(e) : INT32_MIN;
        nlm[i] = uint32_t(h.nlm_t[i]);
    }
    std::vector<Zw> lam, mu, pp, pm;
    // g^r / 2^(r/4) (lambda, mu) and g^r (pi, pi'), r = 0, 1, ... while the
    // entry can be a kernel multiply's x operand
    auto qpowers = [M](const Zw& g, std::vector<Zw>& out) {
        Zw x = zw(1, 0, 0, 0);
        for (uint32_t r = 0; r <= M && zw_fits62(x); ++r) {
            out.push_back(x);
            if (!zw_mul_chk(x, g, x)) break;
            if ((r + 1) % 4 == 0)
                for (int k = 0; k < 4; ++k) x.c[k] /= 2;  // exact: g^4 = 2 * unit for g = lambda, mu
        }
    };
    auto ipowers = [M](const Zw& g, std::vector<Zw>& out) {
        Zw x = zw(1, 0, 0, 0);
        for (uint32_t r = 0; r <= M && zw_fits62(x); ++r) {
            out.push_back(x);
            if (!zw_mul_chk(x, g, x)) break;
        }
    };
    qpowers(zw_generator(K_LAMBDA), lam);
    qpowers(zw_generator(K_MU), mu);
    ipowers(zw_generator(K_PI), pp);
    ipowers(zw_generator(K_PIP), pm);
    const uint32_t pd_n = uint32_t(std::min(pp.size(), pm.size()));
    std::vector<int64_t> vl, vm, pd, p3;
    for (const Zw& z : lam) for (int k = 0; k < 4; ++k) vl.push_back(z.c[k]);
    for (const Zw& z : mu) for (int k = 0; k < 4; ++k) vm.push_back(z.c[k]);
    for (uint32_t i = 0; i < 2 * pd_n - 1; ++i) {
        const int d = int(i) - int(pd_n - 1);
        const Zw& z = d >= 0 ? pp[size_t(d)] : pm[size_t(-d)];
        for (int k = 0; k < 4; ++k) pd.push_back(z.c[k]);
    }
    int64_t v3 = 1;
    for (uint32_t k = 0; k <= M / 2 + 1; ++k) {
        p3.push_back(v3);
        if (v3 > (int64_t(1) << 61) / 3) break;
        v3 *= 3;
    }
    // one allocation: ft | lam | mu | pd | p3 | fx | nlm
    const size_t o_l = ft.size() * 8, o_m = o_l + vl.size() * 8, o_pd = o_m + vm.size() * 8,
                 o_p3 = o_pd + pd.size() * 8, o_fx = o_p3 + p3.size() * 8, o_n = o_fx + fx.size() * 4,
                 bytes = o_n + nlm.size() * 4 + 16;
    std::vector<unsigned char> blob(bytes, 0);
    std::memcpy(blob.data(), ft.data(), ft.size() * 8);
    std::memcpy(blob.data() + o_l, vl.data(), vl.size() * 8);
    std::memcpy(blob.data() + o_m, vm.data(), vm.size() * 8);
    std::memcpy(blob.data() + o_pd, pd.data(), pd.size() * 8);
    std::memcpy(blob.data() + o_p3, p3.data(), p3.size() * 8);
    std::memcpy(blob.data() + o_fx, fx.data(), fx.size() * 4);
    std::memcpy(blob.data() + o_n, nlm.data(), nlm.size() * 4);
    pzx_status st;
    if ((st = cuda_err(ctx, upload_vec(&t->d_exact, blob), "upload exact tables"))) return st;
    const unsigned char* base = static_cast<const unsigned char*>(t->d_exact);
    ExactDev& X = t->exact;
    X.ft = reinterpret_cast<const int64_t*>(base);
    X.lam = reinterpret_cast<const int64_t*>(base + o_l);
    X.mu = reinterpret_cast<const int64_t*>(base + o_m);
    X.pd = reinterpret_cast<const int64_t*>(base + o_pd);
    X.p3 = reinterpret_cast<const int64_t*>(base + o_p3);
    X.fx = reinterpret_cast<const int32_t*>(base + o_fx);
    X.nlm = reinterpret_cast<const uint32_t*>(base + o_n);
    X.lam_n = uint32_t(lam.size());
    X.mu_n = uint32_t(mu.size());
    X.pd_n = pd_n;
    X.p3_n = uint32_t(p3.size());
    return PZX_OK;
}

pzx_status exact_host(pzx_ctx* ctx, pzx_table* t, const uint64_t* asg, uint64_t first, uint64_t n, int64_t* out) {
    NvtxRange nv("pzx.evaluate_exact");
    if (!ctx || !t || (n && !out)) return PZX_E_INVALID;
    if (t->device < 0 || !t->dev.rows) return set_err(ctx, PZX_E_INVALID, "evaluate_exact: host-only table");
    if (n == 0) return PZX_OK;
    pzx_status st;
    if ((st = cuda_err(ctx, cudaSetDevice(ctx->device), "cudaSetDevice"))) return st;
    if (!t->d_exact && (st = build_exact(ctx, t))) return st;
    const uint64_t m = t->dev.n_terms;
    const uint64_t* d_asg = nullptr;
    if (asg) {
        if ((st = cuda_err(ctx, grow(&ctx->d_asg, &ctx->asg_cap, n * 8), "alloc assignments"))) return st;
        if ((st = cuda_err(ctx, cudaMemcpyAsync(ctx->d_asg, asg, n * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D assignments"))) return st;
        d_asg = static_cast<const uint64_t*>(ctx->d_asg);
    }
    // grid: >= 32 waves of 4 resident CTAs per SM via row-balanced term chunks
    const char* ek = std::getenv("PZX_EXACT_K");  // tuning knob: assignments per thread
    const int kx = ek && (std::atoi(ek) == 1 || std::atoi(ek) == 4) ? std::atoi(ek) : kExactK;
    const uint64_t blocks = (n + kExactThreads * kx - 1) / (kExactThreads * kx);
    const char* ew = std::getenv("PZX_EXACT_WAVES");  // tuning knob
    const uint64_t target = uint64_t(ctx->n_sm) * 4 * uint64_t(ew ? std::max(1, std::atoi(ew)) : 32);  // 8 -> 32: +3.5 % on C2 (profiles/r01/exact_c2.log)
    uint64_t chunks = blocks >= target ? 1 : (target + blocks - 1) / blocks;
    chunks = std::min<uint64_t>(chunks, std::max<uint64_t>(1, m));
    chunks = std::min<uint64_t>(chunks, std::max<uint64_t>(1, t->dev.n_rows / min_chunk_rows()));
    chunks = std::min<uint64_t>(chunks, std::max<uint64_t>(1, (uint64_t(1) << 30) / (n * 80 + 1)));
    chunks = std::min<uint64_t>(chunks, 65535);
    const uint64_t* d_chunks = nullptr;
    if (chunks > 1) {
        std::vector<uint64_t> b;
        chunk_bounds(t->host, 0, m, int(chunks), b);
        if ((st = cuda_err(ctx, grow(&ctx->d_chunks, &ctx->chunks_cap, b.size() * 8), "alloc chunks"))) return st;
        if ((st = cuda_err(ctx, cudaMemcpyAsync(ctx->d_chunks, b.data(), b.size() * 8, cudaMemcpyHostToDevice, ctx->stream), "copy chunks"))) return st;
        if ((st = cuda_err(ctx, grow(&ctx->d_partial, &ctx->partial_cap, size_t(chunks) * n * 80), "alloc partials"))) return st;
        d_chunks = static_cast<const uint64_t*>(ctx->d_chunks);
    }
    if ((st = cuda_err(ctx, grow(&ctx->d_xout, &ctx->xout_cap, n * 44 + 16), "alloc exact outputs"))) return st;
    int64_t* d_out = static_cast<int64_t*>(ctx->d_xout);
    uint32_t* d_flag = reinterpret_cast<uint32_t*>(d_out + 5 * n);
    if ((st = cuda_err(ctx, cudaMemsetAsync(d_flag, 0, n * 4, ctx->stream), "clear flags"))) return st;
    if ((st = cuda_err(ctx, launch_exact(t->dev, t->exact, d_asg, first, n, d_chunks, int(chunks), ctx->d_partial, d_flag,
                                         d_out, ctx->stream, &ctx->launches, kx), "exact kernel"))) return st;
    if ((st = cuda_err(ctx, cudaMemcpyAsync(out, d_out, n * 40, cudaMemcpyDeviceToHost, ctx->stream), "D2H exact"))) return st;
    if ((st = cuda_err(ctx, cudaStreamSynchronize(ctx->stream), "evaluate_exact"))) return st;
    for (uint64_t i = 0; i < n; ++i)
        if (out[5 * i + 4] < 0) return set_err(ctx, PZX_E_OVERFLOW, "evaluate_exact: ring coefficient out of 64-bit range");
    return PZX_OK;
}

int prob_mode_of(uint32_t flags) {
    return (flags & PZX_PROB_REAL) ? 2 : (flags & PZX_PROB_ABS2) ? 1 : 1;
}

}  // namespace

// ------------------------------------------------------------------ C ABI ----
extern "C" {

const char* pzx_status_string(pzx_status s) {
    switch (s) {
    case PZX_OK: return "ok";
    case PZX_E_PARSE: return "parse error";
    case PZX_E_DOMAIN: return "domain error";
    case PZX_E_MISSING_PARAM: return "missing parameter";
    case PZX_E_OVERFLOW: return "overflow";
    case PZX_E_INVALID: return "invalid argument";
    case PZX_E_CAPACITY: return "capacity exceeded";
    case PZX_E_CUDA: return "cuda error";
    case PZX_E_NCCL: return "nccl error";
    case PZX_E_OOM: return "out of device memory";
    }
    return "unknown";
}

const char* pzx_version(void) { return "pzx-b200 0.1 (sm_100a)"; }

pzx_status pzx_create(int device, pzx_ctx** out) {
    if (!out) return PZX_E_INVALID;
    *out = nullptr;
    if (!classes().ok) return PZX_E_DOMAIN;
    std::unique_ptr<pzx_ctx> c(new (std::nothrow) pzx_ctx);
    if (!c) return PZX_E_OOM;
    c->device = device;
    pzx_status st;
    if ((st = cuda_err(c.get(), cudaSetDevice(device), "cudaSetDevice"))) return st;
    int nsm = 0;
    if ((st = cuda_err(c.get(), cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device), "device query"))) return st;
    c->n_sm = nsm > 0 ? nsm : 148;
    if ((st = cuda_err(c.get(), cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream"))) return st;
    cudaMemPoolProps pp{};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.handleTypes = cudaMemHandleTypeNone;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = device;
    if ((st = cuda_err(c.get(), cudaMemPoolCreate(&c->pool, &pp), "scratch pool"))) {
        cudaStreamDestroy(c->stream);
        return st;
    }
    // keep freed scratch in the pool across synchronisations (a C2 call takes
    // ~0.6 GB of term-chunk partials; re-mapping it every call would cost ms)
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &keep);
    *out = c.release();
    return PZX_OK;
}

void pzx_destroy(pzx_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (void* p : {ctx->d_asg, ctx->d_amp, ctx->d_prob, ctx->d_partial, ctx->d_chunks, ctx->d_dbg, ctx->d_sort, ctx->d_xout})
        if (p) cudaFree(p);
    for (auto& g : ctx->graphs)
        if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
    cudaStreamDestroy(ctx->stream);
    // pending stream-ordered frees on callers' streams: the driver releases
    // the pool once they have completed
    if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
    delete ctx;
}

const char* pzx_last_error(const pzx_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }

uint64_t pzx_launch_count(const pzx_ctx* ctx) { return ctx ? ctx->launches : 0; }

pzx_status pzx_last_kernel(const pzx_ctx* ctx, int32_t* kernel, int32_t* sorted_groups, int32_t* term_chunks) {
    if (!ctx) return PZX_E_INVALID;
    if (kernel) *kernel = ctx->last_kernel;
    if (sorted_groups) *sorted_groups = ctx->last_groups;
    if (term_chunks) *term_chunks = ctx->last_chunks;
    return PZX_OK;
}

pzx_status pzx_table_upload_expr(pzx_ctx* ctx, const pzx_expr_view* expr, pzx_table** out) {
    return pzx_table_upload_expr_ex(ctx, expr, 0, out);
}

pzx_status pzx_table_upload_expr_ex(pzx_ctx* ctx, const pzx_expr_view* expr, uint32_t compile_flags,
                                    pzx_table** out) {
    if (!ctx || !expr || !out || (expr->n_terms && (!expr->term_offset || !expr->term_scalar)))
        return PZX_E_INVALID;
    std::unique_ptr<pzx_table> t(new (std::nothrow) pzx_table);
    if (!t) return PZX_E_OOM;
    t->host.simplify = (compile_flags & PZX_COMPILE_SIMPLIFY) != 0;
    std::string err;
    int st = compile_expr(expr, t->host, err);
    if (st) return set_err(ctx, st, err);
    return finish_upload(ctx, t, out);
}

pzx_status pzx_table_upload(pzx_ctx* ctx, const pzx_table_view* view, pzx_table** out) {
    if (!ctx || !view || !out || (view->n_terms && (!view->term_row_offset || !view->term_coef)))
        return PZX_E_INVALID;
    std::unique_ptr<pzx_table> t(new (std::nothrow) pzx_table);
    if (!t) return PZX_E_OOM;
    std::string err;
    int st = compile_rows(view, t->host, err);
    if (st) return set_err(ctx, st, err);
    return finish_upload(ctx, t, out);
}

pzx_status pzx_table_compile_host(const pzx_expr_view* expr, pzx_table** out) {
    if (!expr || !out || (expr->n_terms && (!expr->term_offset || !expr->term_scalar)))
        return PZX_E_INVALID;
    std::unique_ptr<pzx_table> t(new (std::nothrow) pzx_table);
    if (!t) return PZX_E_OOM;
    std::string err;
    int st = compile_expr(expr, t->host, err);
    if (st) return pzx_status(st);
    t->device = -1;
    t->dev.n_terms = t->host.coef.size();
    t->dev.n_rows = t->host.n_dev_rows();
    t->dev.n_params = t->host.n_params;
    t->dev.max_rows = t->host.max_rows;
    *out = t.release();
    return PZX_OK;
}

// ---------------------------------------------------------------- PZX1 ----
// Binary table codec (SPEC "External Interfaces": header {magic "PZX1", n,
// m, n_max, R}, constants as 5 x i64, field-major padded table). Layout,
// little-endian:
//   char magic[4] = "PZX1"; u32 n_params; u64 m; u64 n_max; u64 R = m * n_max
//   i64 constants[m][5]                      RingQuad a, b, c, d, exp (canonical)
//   u8 flags[R] (1 = dummy padding row), u8 k_alpha[R], u64 psi[R], u8 k_beta[R], u64 phi[R]
// Row r = t * n_max + i is row i of term t (real rows first, dummies all-zero).
extern "C++" {
namespace {

constexpr uint64_t kPzx1Header = 4 + 4 + 8 + 8 + 8;

struct Rows {  // normalised table (CSR, no padding)
    uint32_t n_params = 0;
    std::vector<uint64_t> off{0};
    std::vector<int64_t> coef;
    std::vector<uint64_t> psi, phi;
    std::vector<uint8_t> ka, kb;
};

// normalize_subterm (subterm.cpp:51-96) over a raw expression, constants folded
// into C_t exactly as the compiler does (constant-first, diagram.cpp:158-161)
int normalize_rows(const pzx_expr_view* v, Rows& out, std::string& err) {
    if (v->n_params > 64) { err = "parameter capacity (64) exceeded"; return PZX_E_DOMAIN; }
    out.n_params = v->n_params;
    const uint64_t allowed = param_mask(v->n_params);
    for (uint64_t t = 0; t < v->n_terms; ++t) {
        Quad c;
        if (!canon_input(v->term_scalar + 5 * t, c)) { err = "term scalar out of range"; return PZX_E_OVERFLOW; }
        for (uint64_t j = v->term_offset[t]; j < v->term_offset[t + 1]; ++j) {
            const uint8_t kind = v->kind[j];
            const int psik = v->psi_k[j], phik = v->phi_k ? v->phi_k[j] : 0;
            const uint64_t psim = v->psi_mask[j];
            uint64_t phim = v->phi_mask ? v->phi_mask[j] : 0;
            if (kind > PZX_PI_PAIR || psik > 7 || phik > 7) { err = "subterm kind or phase out of range"; return PZX_E_DOMAIN; }
            if (kind == PZX_NODE || kind == PZX_HALF_PI) phim = 0;
            if ((psim | phim) & ~allowed) { err = "subterm mask uses a parameter >= n_params"; return PZX_E_MISSING_PARAM; }
            Quad k, nc;
            bool has = false;
            PairRow pr{};
            if (normalize(kind, psik, psim, phik, phim, k, has, pr)) { err = "normalize_subterm: kind invariant violated"; return PZX_E_DOMAIN; }
            if (!quad_mul(c, k, nc)) { err = "term constant overflow"; return PZX_E_OVERFLOW; }
            c = nc;
            if (has) {
                out.ka.push_back(pr.ka);
                out.kb.push_back(pr.kb);
                out.psi.push_back(pr.psi);
                out.phi.push_back(pr.phi);
            }
        }
        const int64_t q[5] = {c.a, c.b, c.c, c.d, c.e};
        out.coef.insert(out.coef.end(), q, q + 5);
        out.off.push_back(out.ka.size());
    }
    return PZX_OK;
}

template <typename T>
void put(uint8_t*& p, T v) {
    std::memcpy(p, &v, sizeof(T));  // little-endian host (x86-64 / aarch64)
    p += sizeof(T);
}
template <typename T>
T get(const uint8_t*& p) {
    T v;
    std::memcpy(&v, p, sizeof(T));
    p += sizeof(T);
    return v;
}

pzx_status encode_view(const pzx_table_view* v, uint8_t* buf, uint64_t cap, uint64_t* len) {
    if (!v || !len || (v->n_terms && (!v->term_row_offset || !v->term_coef))) return PZX_E_INVALID;
    const uint64_t m = v->n_terms;
    uint64_t n_max = 0;
    for (uint64_t t = 0; t < m; ++t) n_max = std::max(n_max, v->term_row_offset[t + 1] - v->term_row_offset[t]);
    const uint64_t R = m * n_max;
    const uint64_t need = kPzx1Header + 40 * m + 19 * R;
    *len = need;
    if (!buf) return PZX_OK;
    if (cap < need) return PZX_E_CAPACITY;
    uint8_t* p = buf;
    std::memcpy(p, "PZX1", 4);
    p += 4;
    put<uint32_t>(p, v->n_params);
    put<uint64_t>(p, m);
    put<uint64_t>(p, n_max);
    put<uint64_t>(p, R);
    for (uint64_t i = 0; i < 5 * m; ++i) put<int64_t>(p, v->term_coef[i]);
    uint8_t* f_flag = p;
    uint8_t* f_ka = f_flag + R;
    uint8_t* f_psi = f_ka + R;
    uint8_t* f_kb = f_psi + 8 * R;
    uint8_t* f_phi = f_kb + R;
    std::memset(f_flag, 0, 19 * R);
    for (uint64_t t = 0; t < m; ++t) {
        const uint64_t r0 = v->term_row_offset[t], n = v->term_row_offset[t + 1] - r0;
        for (uint64_t i = 0; i < n_max; ++i) {
            const uint64_t r = t * n_max + i;
            if (i >= n) { f_flag[r] = 1; continue; }
            f_ka[r] = v->k_alpha[r0 + i];
            f_kb[r] = v->k_beta[r0 + i];
            std::memcpy(f_psi + 8 * r, &v->psi_mask[r0 + i], 8);
            std::memcpy(f_phi + 8 * r, &v->phi_mask[r0 + i], 8);
        }
    }
    return PZX_OK;
}

pzx_status decode_rows(const uint8_t* buf, uint64_t len, Rows& out, std::string& err) {
    if (!buf || len < kPzx1Header) { err = "PZX1: truncated header"; return PZX_E_PARSE; }
    const uint8_t* p = buf;
    if (std::memcmp(p, "PZX1", 4) != 0) { err = "PZX1: bad magic / version"; return PZX_E_PARSE; }
    p += 4;
    out.n_params = get<uint32_t>(p);
    const uint64_t m = get<uint64_t>(p), n_max = get<uint64_t>(p), R = get<uint64_t>(p);
    if (out.n_params > 64) { err = "PZX1: n_params > 64"; return PZX_E_PARSE; }
    if (n_max > (uint64_t(1) << 32) || m > (uint64_t(1) << 40) || R != m * n_max) { err = "PZX1: inconsistent shape"; return PZX_E_PARSE; }
    const uint64_t need = kPzx1Header + 40 * m + 19 * R;
    if (len != need) { err = len < need ? "PZX1: truncated body" : "PZX1: trailing bytes"; return PZX_E_PARSE; }
    out.coef.resize(5 * m);
    for (uint64_t i = 0; i < 5 * m; ++i) out.coef[i] = get<int64_t>(p);
    const uint8_t* f_flag = p;
    const uint8_t* f_ka = f_flag + R;
    const uint8_t* f_psi = f_ka + R;
    const uint8_t* f_kb = f_psi + 8 * R;
    const uint8_t* f_phi = f_kb + R;
    out.off.assign(1, 0);
    for (uint64_t t = 0; t < m; ++t) {
        bool dummy = false;
        for (uint64_t i = 0; i < n_max; ++i) {
            const uint64_t r = t * n_max + i;
            if (f_flag[r] > 1) { err = "PZX1: bad row flag"; return PZX_E_PARSE; }
            if (f_flag[r]) { dummy = true; continue; }
            if (dummy) { err = "PZX1: real row after padding"; return PZX_E_PARSE; }
            uint64_t a, b;
            std::memcpy(&a, f_psi + 8 * r, 8);
            std::memcpy(&b, f_phi + 8 * r, 8);
            out.ka.push_back(f_ka[r]);
            out.kb.push_back(f_kb[r]);
            out.psi.push_back(a);
            out.phi.push_back(b);
        }
        out.off.push_back(out.ka.size());
    }
    return PZX_OK;
}

pzx_table_view view_of(const Rows& r) {
    pzx_table_view v{};
    v.n_params = r.n_params;
    v.n_terms = r.off.size() - 1;
    v.term_row_offset = r.off.data();
    v.term_coef = r.coef.data();
    v.psi_mask = r.psi.data();
    v.phi_mask = r.phi.data();
    v.k_alpha = r.ka.data();
    v.k_beta = r.kb.data();
    return v;
}

}  // namespace
}  // extern "C++"

pzx_status pzx_backend_contract_get(pzx_ctx* ctx, pzx_backend_contract* out) {
    if (!ctx || !out) return PZX_E_INVALID;
    out->max_params = 64;
    out->max_rows_per_term = uint32_t(kSegRows);
    out->max_rows_in_flight = 2 * 64;  // two 64-row TMA tiles per CTA (per warp for small batches)
    out->preferred_batch = uint64_t(ctx->n_sm) * 4 * 128 * 32;
    out->exact = 0;
    out->deterministic = 1;
    out->n_sm = uint32_t(ctx->n_sm);
    out->tmem_accumulators = tmem_accumulators() ? 1u : 0u;
    return PZX_OK;
}

pzx_status pzx_pzx1_encode(const pzx_table_view* view, uint8_t* buf, uint64_t cap, uint64_t* len) {
    return encode_view(view, buf, cap, len);
}

pzx_status pzx_pzx1_encode_expr(const pzx_expr_view* expr, uint8_t* buf, uint64_t cap, uint64_t* len) {
    if (!expr || !len || (expr->n_terms && (!expr->term_offset || !expr->term_scalar))) return PZX_E_INVALID;
    Rows r;
    std::string err;
    const int st = normalize_rows(expr, r, err);
    if (st) return pzx_status(st);
    const pzx_table_view v = view_of(r);
    return encode_view(&v, buf, cap, len);
}

pzx_status pzx_pzx1_info(const uint8_t* buf, uint64_t len, uint32_t* n_params, uint64_t* n_terms, uint64_t* n_rows) {
    Rows r;
    std::string err;
    const pzx_status st = decode_rows(buf, len, r, err);
    if (st) return st;
    if (n_params) *n_params = r.n_params;
    if (n_terms) *n_terms = r.off.size() - 1;
    if (n_rows) *n_rows = r.ka.size();
    return PZX_OK;
}

pzx_status pzx_pzx1_decode(const uint8_t* buf, uint64_t len, uint64_t* term_row_offset, int64_t* term_coef,
                           uint64_t* psi_mask, uint64_t* phi_mask, uint8_t* k_alpha, uint8_t* k_beta) {
    Rows r;
    std::string err;
    const pzx_status st = decode_rows(buf, len, r, err);
    if (st) return st;
    if (!term_row_offset || !term_coef || (!r.ka.empty() && (!psi_mask || !phi_mask || !k_alpha || !k_beta)))
        return PZX_E_INVALID;
    std::memcpy(term_row_offset, r.off.data(), r.off.size() * 8);
    std::memcpy(term_coef, r.coef.data(), r.coef.size() * 8);
    if (!r.ka.empty()) {
        std::memcpy(psi_mask, r.psi.data(), r.psi.size() * 8);
        std::memcpy(phi_mask, r.phi.data(), r.phi.size() * 8);
        std::memcpy(k_alpha, r.ka.data(), r.ka.size());
        std::memcpy(k_beta, r.kb.data(), r.kb.size());
    }
    return PZX_OK;
}

pzx_status pzx_table_upload_pzx1(pzx_ctx* ctx, const uint8_t* buf, uint64_t len, pzx_table** out) {
    if (!ctx || !out) return PZX_E_INVALID;
    Rows r;
    std::string err;
    const pzx_status st = decode_rows(buf, len, r, err);
    if (st) return set_err(ctx, st, err);
    const pzx_table_view v = view_of(r);
    return pzx_table_upload(ctx, &v, out);
}

pzx_status pzx_slice_op_table(int32_t out[129 * 10]) {
    if (!out) return PZX_E_INVALID;
    for (int op = 0; op < kSliceOps; ++op) {
        const SliceOp so = slice_op(op);
        int32_t* o = out + op * 10;
        o[0] = so.jbase;
        for (int v = 0; v < 4; ++v) o[1 + v] = so.w[v];
        o[5] = so.zero_tt; o[6] = so.lam_tt; o[7] = so.pi_tt; o[8] = so.pip_tt; o[9] = so.lm;
    }
    return slice_tables_ok() ? PZX_OK : PZX_E_DOMAIN;
}

pzx_status pzx_class_table(uint32_t codes[256], int32_t e[64], int32_t lm[64]) {
    const Classes& k = classes();
    if (!k.ok) return PZX_E_DOMAIN;
    for (int c = 0; c < 64; ++c) {
        for (int v = 0; v < 4; ++v)
            if (codes) codes[c * 4 + v] = k.c[c].code[v];
        if (e) e[c] = k.c[c].e;
        if (lm) lm[c] = k.c[c].lm;
    }
    return PZX_OK;
}

void pzx_table_free(pzx_table* t) {
    if (!t) return;
    if (t->device < 0) { delete t; return; }
    cudaSetDevice(t->device);
    for (void* p : {t->d_rows, t->d_term_row, t->d_term_c, t->d_lut, t->d_srows, t->d_sterm_c, t->d_qrows, t->d_exact,
                    t->d_prows, t->d_term_slot})
        if (p) cudaFree(p);
    for (auto& kv : t->chunk_cache) cudaFree(kv.second);
    delete t;
}

pzx_status pzx_table_shape(const pzx_table* t, uint32_t* n_params, uint64_t* n_terms,
                           uint64_t* n_rows, uint32_t* max_term_rows) {
    if (!t) return PZX_E_INVALID;
    if (n_params) *n_params = t->host.n_params;
    if (n_terms) *n_terms = t->dev.n_terms;
    if (n_rows) *n_rows = t->host.genuine_rows();
    if (max_term_rows) *max_term_rows = t->host.max_rows;
    return PZX_OK;
}

pzx_status pzx_table_page_layout(const pzx_table* t, uint32_t* slots, uint64_t* n_slots, uint32_t* term_slot,
                                 uint8_t* jfold, uint64_t family_rows[PZX_PAGE_FAMILIES]) {
    if (!t || !n_slots) return PZX_E_INVALID;
    const HostTable& h = t->host;
    if (!h.want_prows || h.term_slot.size() != h.coef.size()) { *n_slots = 0; return PZX_E_CAPACITY; }
    if (family_rows) {
        for (int i = 0; i < 5; ++i) family_rows[i] = h.page_rows[i];
        for (int i = 0; i < kPageGClasses; ++i) family_rows[5 + i] = h.page_gsub[i];
    }
    if (h.prows.empty() && t->device >= 0) { *n_slots = 0; return PZX_E_INVALID; }  // uploaded: host copy released
    *n_slots = h.prows.size() / 2;
    if (slots) std::memcpy(slots, h.prows.data(), h.prows.size() * 16);
    if (term_slot) std::memcpy(term_slot, h.term_slot.data(), h.term_slot.size() * 4);
    if (jfold) std::memcpy(jfold, h.jp_t.data(), h.jp_t.size());
    return PZX_OK;
}

pzx_status pzx_table_page_stats(const pzx_table* t, uint64_t family_rows[PZX_PAGE_FAMILIES], uint64_t d_op_rows[129]) {
    if (!t) return PZX_E_INVALID;
    const HostTable& h = t->host;
    if (!h.want_prows || h.term_slot.size() != h.coef.size()) return PZX_E_CAPACITY;
    if (family_rows) {
        for (int i = 0; i < 5; ++i) family_rows[i] = h.page_rows[i];
        for (int i = 0; i < kPageGClasses; ++i) family_rows[5 + i] = h.page_gsub[i];
    }
    if (d_op_rows)
        for (int i = 0; i < kSliceOps; ++i) d_op_rows[i] = h.page_d_ops[i];
    return PZX_OK;
}

pzx_status pzx_table_slice_stats(const pzx_table* t, uint64_t op_rows[129], uint64_t term_kinds[3]) {
    if (!t) return PZX_E_INVALID;
    if (op_rows)
        for (int i = 0; i < kSliceOps; ++i) op_rows[i] = t->host.op_rows[i];
    if (term_kinds)
        for (int i = 0; i < 3; ++i) term_kinds[i] = t->host.term_kinds[i];
    return PZX_OK;
}

pzx_status pzx_table_term_info(const pzx_table* t, uint64_t term, int64_t coef[5],
                               int32_t* e_sqrt2, int32_t* n_lm) {
    if (!t || term >= t->dev.n_terms) return PZX_E_INVALID;
    const Quad& q = t->host.coef[term];
    if (coef) { coef[0] = q.a; coef[1] = q.b; coef[2] = q.c; coef[3] = q.d; coef[4] = q.e; }
    if (e_sqrt2) *e_sqrt2 = t->host.e_t[term];
    if (n_lm) *n_lm = t->host.nlm_t[term];
    return PZX_OK;
}

static pzx_status eval_host_impl(pzx_ctx* ctx, const pzx_table* t, const uint64_t* asg, uint64_t first,
                                 uint64_t n, double* amp, double* prob, uint32_t flags);
static pzx_status eval_host_graph(pzx_ctx* ctx, const pzx_table* t, const uint64_t* asg, uint64_t first,
                                  uint64_t n, double* amp, double* prob, uint32_t flags, bool* handled);
static pzx_status eval_host(pzx_ctx* ctx, const pzx_table* t, const uint64_t* asg, uint64_t first,
                            uint64_t n, double* amp, double* prob, uint32_t flags) {
    NvtxRange nv("pzx.evaluate_host (H2D + kernels + D2H)");
    if (!ctx || !t) return PZX_E_INVALID;
    if (flags & kNoSyncFlag) return set_err(ctx, PZX_E_INVALID, "evaluate: unknown flag bit");
    if (t->device >= 0 && t->device == ctx->device) {
        bool handled = false;
        const pzx_status st = eval_host_graph(ctx, t, asg, first, n, amp, prob, flags, &handled);
        if (st || handled) return st;
    }
    return eval_host_impl(ctx, t, asg, first, n, amp, prob, flags);
}
static pzx_status eval_host_impl(pzx_ctx* ctx, const pzx_table* t, const uint64_t* asg, uint64_t first,
                            uint64_t n, double* amp, double* prob, uint32_t flags) {
    if (!ctx || !t) return PZX_E_INVALID;
    if (n == 0) return PZX_OK;
    pzx_status st;
    if ((st = cuda_err(ctx, cudaSetDevice(ctx->device), "cudaSetDevice"))) return st;
    LaunchReq r;
    r.stream = ctx->stream;
    r.first = first;
    r.n = n;
    r.term_begin = 0;
    r.term_end = t->dev.n_terms;
    r.prob_mode = prob_mode_of(flags);
    if (asg) {
        if ((st = cuda_err(ctx, grow(&ctx->d_asg, &ctx->asg_cap, n * 8), "alloc assignments"))) return st;
        if ((st = cuda_err(ctx, cudaMemcpyAsync(ctx->d_asg, asg, n * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D assignments"))) return st;
        r.d_asg = static_cast<const uint64_t*>(ctx->d_asg);
        // a contiguous, 16-aligned word list (a sweep over output bitstrings)
        // can use the enumerated kernel; the kernel still reads its base words
        bool contig = n >= uint64_t(kGray);
        for (uint64_t i = 1; contig && i < n; ++i) contig = asg[i] == asg[0] + i;
        if (contig) { r.words_contiguous = 1; r.first = asg[0]; }
    }
    if (amp) {
        if ((st = cuda_err(ctx, grow(&ctx->d_amp, &ctx->amp_cap, n * 16), "alloc amplitudes"))) return st;
        r.d_amp = static_cast<double2*>(ctx->d_amp);
    }
    if (prob) {
        if ((st = cuda_err(ctx, grow(&ctx->d_prob, &ctx->prob_cap, n * 8), "alloc probabilities"))) return st;
        r.d_prob = static_cast<double*>(ctx->d_prob);
    }
    if (!amp && !prob) return PZX_OK;
    auto enqueue_rest = [&]() -> pzx_status {  // kernels + D2H (the H2D is already enqueued)
        pzx_status s2;
        if ((s2 = run_eval(ctx, t, r, flags))) return s2;
        if (amp && (s2 = cuda_err(ctx, cudaMemcpyAsync(amp, ctx->d_amp, n * 16, cudaMemcpyDeviceToHost, ctx->stream), "D2H amplitudes"))) return s2;
        if (prob && (s2 = cuda_err(ctx, cudaMemcpyAsync(prob, ctx->d_prob, n * 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H probabilities"))) return s2;
        return PZX_OK;
    };
    if ((st = enqueue_rest())) return st;
    if (flags & kNoSyncFlag) return PZX_OK;  // (graph capture)
    return cuda_err(ctx, cudaStreamSynchronize(ctx->stream), "evaluate");
}

// Small, repeated host-buffer calls (a sampling loop, bench.py's e2e leg):
// the second identical call (same table object, words / buffers, batch and
// flags, pinned host memory, enumerated or contiguous-word batch) is captured
// into a CUDA graph -- H2D, kernels (their stream-ordered scratch as graph
// allocation nodes), D2H -- and later identical calls replay it: one
// cudaGraphLaunch instead of every API call. Word CONTENTS may change between
// calls (the H2D node reads them at replay); the kernel choice depends only on
// the key. PZX_NO_GRAPHS=1 turns this off.
bool graphs_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PZX_NO_GRAPHS");
        return !(e && std::string(e) == "1");
    }();
    return on;
}

bool host_pinned(const void* p) {
    if (!p) return true;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
    return a.type == cudaMemoryTypeHost;
}

static pzx_status eval_host_graph(pzx_ctx* ctx, const pzx_table* t, const uint64_t* asg, uint64_t first,
                                  uint64_t n, double* amp, double* prob, uint32_t flags, bool* handled) {
    *handled = false;
    constexpr uint64_t kGraphMaxBatch = uint64_t(1) << 16;
    if (!graphs_enabled() || n == 0 || n > kGraphMaxBatch || (!amp && !prob)) return PZX_OK;
    if (!host_pinned(asg) || !host_pinned(amp) || !host_pinned(prob)) return PZX_OK;
    bool contig = true;  // word lists: only contiguous ones (their kernel choice is fixed by asg[0])
    if (asg)
        for (uint64_t i = 1; contig && i < n; ++i) contig = asg[i] == asg[0] + i;
    if (!contig) return PZX_OK;
    const std::vector<uint64_t> key = {t->gen, uint64_t(reinterpret_cast<uintptr_t>(asg)), asg ? asg[0] : first, n,
                                       uint64_t(reinterpret_cast<uintptr_t>(amp)),
                                       uint64_t(reinterpret_cast<uintptr_t>(prob)), flags};
    auto& g = ctx->graphs[key];
    pzx_status st;
    // the device scratch the graph uses (grown first, so a replay sees the same buffers)
    if (asg && (st = cuda_err(ctx, grow(&ctx->d_asg, &ctx->asg_cap, n * 8), "alloc assignments"))) return st;
    if (amp && (st = cuda_err(ctx, grow(&ctx->d_amp, &ctx->amp_cap, n * 16), "alloc amplitudes"))) return st;
    if (prob && (st = cuda_err(ctx, grow(&ctx->d_prob, &ctx->prob_cap, n * 8), "alloc probabilities"))) return st;
    if (g.exec && (g.d_asg != (asg ? ctx->d_asg : nullptr) || g.d_amp != (amp ? ctx->d_amp : nullptr) ||
                   g.d_prob != (prob ? ctx->d_prob : nullptr))) {
        cudaGraphExecDestroy(g.exec);  // a scratch buffer moved since the capture
        g.exec = nullptr;
    }
    if (!g.exec) {
        if (++g.seen < 2) return PZX_OK;  // capture from the second identical call on
        if (ctx->graphs.size() > 64) return PZX_OK;
        const uint64_t l0 = ctx->launches;
        if ((st = cuda_err(ctx, cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal), "graph capture")))
            return PZX_OK;
        pzx_status cst = eval_host_impl(ctx, t, asg, first, n, amp, prob, flags | kNoSyncFlag);
        cudaGraph_t graph = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(ctx->stream, &graph);
        cudaGraphExec_t exec = nullptr;
        if (cst == PZX_OK && ce == cudaSuccess && graph &&
            cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess) {
            g.exec = exec;
            g.launches = ctx->launches - l0;
            g.kernel = ctx->last_kernel; g.groups = ctx->last_groups; g.chunks = ctx->last_chunks;
            g.d_asg = asg ? ctx->d_asg : nullptr;
            g.d_amp = amp ? ctx->d_amp : nullptr;
            g.d_prob = prob ? ctx->d_prob : nullptr;
            ctx->launches = l0;  // counted when the graph runs
        } else {
            ctx->launches = l0;
            cudaGetLastError();
        }
        if (graph) cudaGraphDestroy(graph);
        if (!g.exec) return PZX_OK;  // not capturable: the plain path runs
    }
    if ((st = cuda_err(ctx, cudaGraphLaunch(g.exec, ctx->stream), "graph launch"))) return st;
    ctx->launches += g.launches;
    ctx->last_kernel = g.kernel; ctx->last_groups = g.groups; ctx->last_chunks = g.chunks;
    *handled = true;
    return cuda_err(ctx, cudaStreamSynchronize(ctx->stream), "evaluate");
}

pzx_status pzx_evaluate(pzx_ctx* ctx, const pzx_table* t, const uint64_t* assignments,
                        uint64_t n, double* amp, double* prob, uint32_t flags) {
    if (n && !assignments) return PZX_E_INVALID;
    return eval_host(ctx, t, assignments, 0, n, amp, prob, flags);
}

pzx_status pzx_evaluate_range(pzx_ctx* ctx, const pzx_table* t, uint64_t first, uint64_t n,
                              double* amp, double* prob, uint32_t flags) {
    return eval_host(ctx, t, nullptr, first, n, amp, prob, flags);
}

pzx_status pzx_evaluate_exact(pzx_ctx* ctx, const pzx_table* t, const uint64_t* assignments, uint64_t n, int64_t* out) {
    if (n && !assignments) return PZX_E_INVALID;
    return exact_host(ctx, const_cast<pzx_table*>(t), assignments, 0, n, out);
}

pzx_status pzx_evaluate_exact_range(pzx_ctx* ctx, const pzx_table* t, uint64_t first, uint64_t n, int64_t* out) {
    return exact_host(ctx, const_cast<pzx_table*>(t), nullptr, first, n, out);
}

pzx_status pzx_ringquad_sum_device(pzx_ctx* ctx, const int64_t* d_parts, uint32_t n_parts, uint64_t n,
                                   int64_t* d_out, void* stream) {
    if (!ctx || (n && (!d_out || (n_parts && !d_parts)))) return PZX_E_INVALID;
    if (n == 0) return PZX_OK;
    pzx_status st;
    if ((st = cuda_err(ctx, cudaSetDevice(ctx->device), "cudaSetDevice"))) return st;
    return cuda_err(ctx, launch_ringquad_sum(d_parts, n_parts, n, d_out, static_cast<cudaStream_t>(stream),
                                             &ctx->launches), "ringquad_sum");
}

pzx_status pzx_ringquad_sum(pzx_ctx* ctx, const int64_t* parts, uint32_t n_parts, uint64_t n, int64_t* out) {
    if (!ctx || (n && (!out || (n_parts && !parts)))) return PZX_E_INVALID;
    if (n == 0) return PZX_OK;
    pzx_status st;
    if ((st = cuda_err(ctx, cudaSetDevice(ctx->device), "cudaSetDevice"))) return st;
    const size_t in_b = size_t(n_parts) * n * 40, out_b = size_t(n) * 40;
    void* d = nullptr;
    if ((st = cuda_err(ctx, cudaMallocAsync(&d, in_b + out_b, ctx->stream), "alloc ringquad_sum"))) return st;
    int64_t* d_in = static_cast<int64_t*>(d);
    int64_t* d_out = d_in + size_t(n_parts) * n * 5;
    st = cuda_err(ctx, cudaMemcpyAsync(d_in, parts, in_b, cudaMemcpyHostToDevice, ctx->stream), "H2D ringquad parts");
    if (!st) st = pzx_ringquad_sum_device(ctx, d_in, n_parts, n, d_out, ctx->stream);
    if (!st) st = cuda_err(ctx, cudaMemcpyAsync(out, d_out, out_b, cudaMemcpyDeviceToHost, ctx->stream), "D2H ringquad sum");
    cudaFreeAsync(d, ctx->stream);
    if (!st) st = cuda_err(ctx, cudaStreamSynchronize(ctx->stream), "ringquad_sum");
    if (st) return st;
    for (uint64_t i = 0; i < n; ++i)
        if (out[5 * i + 4] < 0) return set_err(ctx, PZX_E_OVERFLOW, "ringquad_sum: ring coefficient out of 64-bit range");
    return PZX_OK;
}

// Marginal summing: out[i] = sum over b < 2^m of prob(fixed[i] | b),
// prob = |amp|^2 (default) or Re(amp) (PZX_PROB_REAL). The don't-care outputs
// are the low m parameters. Large groups run as enumerated ranges (bit-sliced
// kernel); small groups are expanded into one word list per block of
// patterns. Every reduction is fixed-order (deterministic).
pzx_status pzx_marginal_sum(pzx_ctx* ctx, const pzx_table* t, const uint64_t* fixed, uint64_t n_fixed, uint32_t m,
                            uint32_t flags, double* out) {
    if (!ctx || !t || (n_fixed && (!fixed || !out))) return PZX_E_INVALID;
    if (m > 40) return set_err(ctx, PZX_E_CAPACITY, "marginal_sum: more than 2^40 summed assignments per pattern");
    if (n_fixed == 0) return PZX_OK;
    const uint64_t G = uint64_t(1) << m, low = G - 1;
    for (uint64_t i = 0; i < n_fixed; ++i)
        if (fixed[i] & low) return set_err(ctx, PZX_E_INVALID, "marginal_sum: fixed words must have the low m bits clear");
    if (flags & PZX_PROB_ABS2 && flags & PZX_PROB_REAL) return set_err(ctx, PZX_E_INVALID, "marginal_sum: one prob mode");
    const uint32_t pf = (flags & PZX_PROB_REAL) ? PZX_PROB_REAL : PZX_PROB_ABS2;
    const uint32_t kflags = (flags & ~(PZX_PROB_ABS2 | PZX_PROB_REAL)) | pf;
    pzx_status st;
    if ((st = cuda_err(ctx, cudaSetDevice(ctx->device), "cudaSetDevice"))) return st;
    constexpr uint64_t kBlock = uint64_t(1) << 22;  // assignments per evaluation launch
    double* d_out = nullptr;
    if ((st = cuda_err(ctx, cudaMalloc(reinterpret_cast<void**>(&d_out), n_fixed * 8), "alloc marginals"))) return st;
    auto fail = [&](pzx_status s) { cudaFree(d_out); return s; };
    if ((st = cuda_err(ctx, grow(&ctx->d_prob, &ctx->prob_cap, std::min(G, kBlock) * std::max<uint64_t>(1, kBlock / std::max(G, uint64_t(1))) * 8 + 8), "alloc prob"))) return fail(st);
    double* d_prob = static_cast<double*>(ctx->d_prob);
    LaunchReq r;
    r.stream = ctx->stream;
    r.term_begin = 0;
    r.term_end = t->dev.n_terms;
    r.prob_mode = prob_mode_of(pf);
    r.d_prob = d_prob;
    if (G >= uint64_t(1) << 12) {
        // per pattern: enumerated sub-ranges of <= kBlock words, partial sums accumulated in order
        for (uint64_t i = 0; i < n_fixed; ++i) {
            for (uint64_t b0 = 0; b0 < G; b0 += kBlock) {
                r.first = fixed[i] + b0;
                r.n = std::min(kBlock, G - b0);
                r.d_asg = nullptr;
                r.d_amp = nullptr;
                if ((st = run_eval(ctx, t, r, kflags))) return fail(st);
                if ((st = cuda_err(ctx, launch_segment_sum(d_prob, r.n, 1, d_out + i, b0 > 0, ctx->stream, &ctx->launches), "segment sum"))) return fail(st);
            }
        }
    } else {
        const uint64_t per = kBlock >> m;  // patterns per block
        if ((st = cuda_err(ctx, grow(&ctx->d_asg, &ctx->asg_cap, (per << m) * 8 + per * 8), "alloc words"))) return fail(st);
        uint64_t* d_words = static_cast<uint64_t*>(ctx->d_asg);
        uint64_t* d_fix = d_words + (per << m);
        for (uint64_t p0 = 0; p0 < n_fixed; p0 += per) {
            const uint64_t np = std::min(per, n_fixed - p0);
            if ((st = cuda_err(ctx, cudaMemcpyAsync(d_fix, fixed + p0, np * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D patterns"))) return fail(st);
            if ((st = cuda_err(ctx, launch_expand_words(d_fix, np, m, d_words, ctx->stream, &ctx->launches), "expand"))) return fail(st);
            r.first = 0;
            r.n = np << m;
            r.d_asg = d_words;
            r.d_amp = nullptr;
            r.words_contiguous = 0;
            if ((st = run_eval(ctx, t, r, kflags))) return fail(st);
            if ((st = cuda_err(ctx, launch_segment_sum(d_prob, G, np, d_out + p0, 0, ctx->stream, &ctx->launches), "segment sum"))) return fail(st);
        }
    }
    st = cuda_err(ctx, cudaMemcpyAsync(out, d_out, n_fixed * 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H marginals");
    if (!st) st = cuda_err(ctx, cudaStreamSynchronize(ctx->stream), "marginal_sum");
    cudaFree(d_out);
    return st;
}

// Repeated weak simulation (PAPER App. F Alg. 2): tables[k] is
// the compiled doubled marginal P(a_1 .. a_{k+1}) (parameter j = bit j of the
// sample word). Round k evaluates P(B_i || 0) for every sample on the device
// and draws bit k from P(B_i || 0) / P(B_i); the samples never leave the GPU
// until the end. n_bits tables -> n_bits compilations for any n_samples.
pzx_status pzx_weak_sample(pzx_ctx* ctx, const pzx_table* const* tables, uint32_t n_bits, uint64_t n_samples,
                           uint64_t seed, uint32_t flags, uint64_t* out) {
    if (!ctx || (n_bits && !tables) || (n_samples && !out)) return PZX_E_INVALID;
    if (n_bits > 64) return set_err(ctx, PZX_E_DOMAIN, "weak_sample: more than 64 output bits");
    for (uint32_t k = 0; k < n_bits; ++k) {
        if (!tables[k]) return set_err(ctx, PZX_E_INVALID, "weak_sample: null table");
        if (tables[k]->dev.n_params < k + 1)
            return set_err(ctx, PZX_E_MISSING_PARAM, "weak_sample: table k must take parameters a_1 .. a_{k+1}");
    }
    if (n_samples == 0) return PZX_OK;
    if (flags & PZX_PROB_ABS2 && flags & PZX_PROB_REAL) return set_err(ctx, PZX_E_INVALID, "weak_sample: one prob mode");
    const uint32_t pf = (flags & PZX_PROB_ABS2) ? PZX_PROB_ABS2 : PZX_PROB_REAL;  // doubled diagrams: Re
    const uint32_t kflags = (flags & ~(PZX_PROB_ABS2 | PZX_PROB_REAL)) | pf;
    pzx_status st;
    if ((st = cuda_err(ctx, cudaSetDevice(ctx->device), "cudaSetDevice"))) return st;
    const uint64_t n = n_samples;
    void* buf = nullptr;
    const size_t bytes = n * 8 * 3 + 256;
    if ((st = cuda_err(ctx, cudaMalloc(&buf, bytes), "alloc samples"))) return st;
    uint64_t* d_words = static_cast<uint64_t*>(buf);
    double* d_pprev = reinterpret_cast<double*>(d_words + n);
    double* d_p0 = d_pprev + n;
    unsigned int* d_err = reinterpret_cast<unsigned int*>(d_p0 + n);
    auto done = [&](pzx_status s) { cudaFree(buf); return s; };
    std::vector<double> ones(n, 1.0);  // P(empty prefix) = 1
    if ((st = cuda_err(ctx, cudaMemsetAsync(d_words, 0, n * 8, ctx->stream), "init words"))) return done(st);
    if ((st = cuda_err(ctx, cudaMemsetAsync(d_err, 0, 4, ctx->stream), "init err"))) return done(st);
    if ((st = cuda_err(ctx, cudaMemcpyAsync(d_pprev, ones.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream), "init P"))) return done(st);
    for (uint32_t k = 0; k < n_bits; ++k) {
        LaunchReq r;
        r.stream = ctx->stream;
        r.d_asg = d_words;
        r.n = n;
        r.term_begin = 0;
        r.term_end = tables[k]->dev.n_terms;
        r.prob_mode = prob_mode_of(pf);
        r.d_prob = d_p0;
        if ((st = run_eval(ctx, tables[k], r, kflags))) return done(st);
        if ((st = cuda_err(ctx, launch_sample_step(d_words, d_pprev, d_p0, n, k, seed, d_err, ctx->stream, &ctx->launches), "sample step"))) return done(st);
    }
    unsigned int err = 0;
    if ((st = cuda_err(ctx, cudaMemcpyAsync(out, d_words, n * 8, cudaMemcpyDeviceToHost, ctx->stream), "D2H samples"))) return done(st);
    if ((st = cuda_err(ctx, cudaMemcpyAsync(&err, d_err, 4, cudaMemcpyDeviceToHost, ctx->stream), "D2H err"))) return done(st);
    if ((st = cuda_err(ctx, cudaStreamSynchronize(ctx->stream), "weak_sample"))) return done(st);
    if (err) return done(set_err(ctx, PZX_E_DOMAIN, "weak_sample: zero-probability prefix encountered"));
    return done(PZX_OK);
}

pzx_status pzx_evaluate_device(pzx_ctx* ctx, const pzx_table* t, const uint64_t* d_assignments,
                               uint64_t first, uint64_t n, uint64_t term_begin,
                               uint64_t term_end, double* d_amp, double* d_prob,
                               uint32_t flags, void* stream) {
    if (!ctx || !t) return PZX_E_INVALID;
    if (n == 0) return PZX_OK;
    LaunchReq r;
    r.stream = static_cast<cudaStream_t>(stream);
    r.d_asg = d_assignments;
    r.first = first;
    r.n = n;
    r.term_begin = term_begin;
    r.term_end = term_end;
    r.d_amp = reinterpret_cast<double2*>(d_amp);
    r.d_prob = d_prob;
    r.prob_mode = prob_mode_of(flags);
    r.accumulate = (flags & PZX_ACCUMULATE) ? 1 : 0;
    if (!d_amp && !d_prob) return PZX_OK;
    return run_eval(ctx, t, r, flags);
}

pzx_status pzx_amp_to_prob_device(pzx_ctx* ctx, const double* d_amp, uint64_t n, double* d_prob,
                                  uint32_t flags, void* stream) {
    if (!ctx || (n && (!d_amp || !d_prob))) return PZX_E_INVALID;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return cuda_err(ctx, launch_amp_to_prob(reinterpret_cast<const double2*>(d_amp), n, d_prob,
                                            prob_mode_of(flags), s, &ctx->launches), "amp_to_prob");
}

pzx_status pzx_synchronize(pzx_ctx* ctx) {
    if (!ctx) return PZX_E_INVALID;
    return cuda_err(ctx, cudaStreamSynchronize(ctx->stream), "synchronize");
}

pzx_status pzx_debug_phase_indices(pzx_ctx* ctx, const pzx_table* t, const uint64_t* assignments,
                                   uint64_t n, uint8_t* idx_out) {
    if (!ctx || !t || (n && (!assignments || !idx_out))) return PZX_E_INVALID;
    if (t->device < 0) return set_err(ctx, PZX_E_INVALID, "host-only table");
    const uint64_t R = t->dev.n_rows;  // device rows incl. unit placeholders
    if (!n || !R) return PZX_OK;
    pzx_status st;
    if ((st = cuda_err(ctx, cudaSetDevice(ctx->device), "cudaSetDevice"))) return st;
    if ((st = cuda_err(ctx, grow(&ctx->d_asg, &ctx->asg_cap, n * 8), "alloc"))) return st;
    if ((st = cuda_err(ctx, grow(&ctx->d_dbg, &ctx->dbg_cap, R * n), "alloc"))) return st;
    cudaMemcpyAsync(ctx->d_asg, assignments, n * 8, cudaMemcpyHostToDevice, ctx->stream);
    if ((st = cuda_err(ctx, launch_debug_phase(t->dev, static_cast<const uint64_t*>(ctx->d_asg), n,
                                               static_cast<uint8_t*>(ctx->d_dbg), ctx->stream, &ctx->launches), "debug phase"))) return st;
    std::vector<uint8_t> all(R * n);
    if ((st = cuda_err(ctx, cudaMemcpyAsync(all.data(), ctx->d_dbg, R * n, cudaMemcpyDeviceToHost, ctx->stream), "D2H"))) return st;
    if ((st = cuda_err(ctx, cudaStreamSynchronize(ctx->stream), "debug phase"))) return st;
    // drop unit placeholder rows; un-swap rows stored as (phi, psi) so that
    // idx = idx_psi*8 + idx_phi in the caller's canonical row order
    uint64_t o = 0;
    for (uint64_t r = 0; r < R; ++r) {
        if (t->host.unit[r]) continue;
        const uint8_t* src = all.data() + r * n;
        uint8_t* dst = idx_out + o * n;
        if (t->host.swapped[r])
            for (uint64_t i = 0; i < n; ++i) dst[i] = uint8_t(((src[i] & 7) << 3) | (src[i] >> 3));
        else
            std::memcpy(dst, src, n);
        ++o;
    }
    return PZX_OK;
}

pzx_status pzx_debug_slice_codes(pzx_ctx* ctx, const pzx_table* t, const uint64_t* assignments, uint64_t first,
                                 uint64_t n, uint64_t term_begin, uint64_t term_end, uint32_t flags,
                                 pzx_term_code* out) {
    if (!ctx || !t || (n && !out)) return PZX_E_INVALID;
    if (t->device < 0) return set_err(ctx, PZX_E_INVALID, "host-only table");
    term_end = std::min<uint64_t>(term_end, t->dev.n_terms);
    if (term_begin > term_end) return set_err(ctx, PZX_E_INVALID, "bad debug term range");
    const uint64_t M = term_end - term_begin;
    if (!n || !M) return PZX_OK;
    pzx_status st;
    if ((st = cuda_err(ctx, cudaSetDevice(ctx->device), "cudaSetDevice"))) return st;
    LaunchReq r;
    r.stream = ctx->stream;
    r.first = first;
    r.n = n;
    r.term_begin = 0;
    r.term_end = t->dev.n_terms;
    r.prob_mode = 1;
    if (assignments) {
        if ((st = cuda_err(ctx, grow(&ctx->d_asg, &ctx->asg_cap, n * 8), "alloc assignments"))) return st;
        if ((st = cuda_err(ctx, cudaMemcpyAsync(ctx->d_asg, assignments, n * 8, cudaMemcpyHostToDevice, ctx->stream), "H2D assignments"))) return st;
        r.d_asg = static_cast<const uint64_t*>(ctx->d_asg);
        bool contig = n >= uint64_t(kGray);
        for (uint64_t i = 1; contig && i < n; ++i) contig = assignments[i] == assignments[0] + i;
        if (contig) { r.words_contiguous = 1; r.first = assignments[0]; }
    }
    if ((st = cuda_err(ctx, grow(&ctx->d_amp, &ctx->amp_cap, n * 16), "alloc amplitudes"))) return st;
    r.d_amp = static_cast<double2*>(ctx->d_amp);
    if ((st = cuda_err(ctx, grow(&ctx->d_dbg, &ctx->dbg_cap, M * n * 20), "alloc debug"))) return st;
    if ((st = cuda_err(ctx, cudaMemsetAsync(ctx->d_dbg, 0xFF, M * n * 20, ctx->stream), "clear debug"))) return st;
    r.d_dbg5 = static_cast<uint32_t*>(ctx->d_dbg);
    r.dbg_t0 = term_begin;
    r.dbg_t1 = term_end;
    r.dbg_n = n;
    if ((st = run_eval(ctx, t, r, flags))) return st;
    const int k = ctx->last_kernel;
    if (k != KC_SLICE && k != KC_SLICER && k != KC_SLICEWC && k != KC_SORTED && k != KC_PAGE)
        return set_err(ctx, PZX_E_INVALID, "debug_slice_codes: the batch did not run on a bit-sliced kernel");
    const std::vector<uint8_t>& jfold = k == KC_PAGE ? t->host.jp_t : t->host.jb_t;
    if ((st = cuda_err(ctx, cudaMemcpyAsync(out, ctx->d_dbg, M * n * 20, cudaMemcpyDeviceToHost, ctx->stream), "D2H"))) return st;
    if ((st = cuda_err(ctx, cudaStreamSynchronize(ctx->stream), "debug slice codes"))) return st;
    for (uint64_t tt = 0; tt < M; ++tt) {  // the slice kernels count w' relative to each row's jbase
        const uint32_t jb = jfold[term_begin + tt];
        for (uint64_t i = 0; i < n; ++i) {
            pzx_term_code& c = out[tt * n + i];
            if (c.j != 0xFFFFFFFFu) c.j = (c.j + jb) & 7u;
        }
    }
    return PZX_OK;
}

pzx_status pzx_debug_term_codes(pzx_ctx* ctx, const pzx_table* t, const uint64_t* assignments,
                                uint64_t n, pzx_term_code* out) {
    if (!ctx || !t || (n && (!assignments || !out))) return PZX_E_INVALID;
    if (t->device < 0) return set_err(ctx, PZX_E_INVALID, "host-only table");
    const uint64_t M = t->dev.n_terms;
    if (!n || !M) return PZX_OK;
    pzx_status st;
    if ((st = cuda_err(ctx, cudaSetDevice(ctx->device), "cudaSetDevice"))) return st;
    if ((st = cuda_err(ctx, grow(&ctx->d_asg, &ctx->asg_cap, n * 8), "alloc"))) return st;
    if ((st = cuda_err(ctx, grow(&ctx->d_dbg, &ctx->dbg_cap, M * n * 20), "alloc"))) return st;
    cudaMemcpyAsync(ctx->d_asg, assignments, n * 8, cudaMemcpyHostToDevice, ctx->stream);
    if ((st = cuda_err(ctx, launch_debug_codes(t->dev, static_cast<const uint64_t*>(ctx->d_asg), n,
                                               static_cast<uint32_t*>(ctx->d_dbg), ctx->stream, &ctx->launches), "debug codes"))) return st;
    if ((st = cuda_err(ctx, cudaMemcpyAsync(out, ctx->d_dbg, M * n * 20, cudaMemcpyDeviceToHost, ctx->stream), "D2H"))) return st;
    return cuda_err(ctx, cudaStreamSynchronize(ctx->stream), "debug codes");
}

}  // extern "C"
