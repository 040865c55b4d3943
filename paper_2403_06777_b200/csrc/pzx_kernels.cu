// pzx_kernels.cu -- sm_100a evaluation kernels for the parametric scalar
//   S(a) = sum_t C_t prod_r V(k_alpha_r + 4 p_r(a), k_beta_r + 4 q_r(a)),
//   p_r(a) = parity(psi_r & a), q_r(a) = parity(phi_r & a)
// (PAPER §3.3 steps 1-7; SPEC eval_row / evaluate S:448-474).
//
// Design:
//  * a thread owns assignments; all threads of a CTA walk the SAME flat row
//    stream (no divergence, no dummy padding, no per-row global loads):
//    tiles of kTileRows rows are staged into shared memory by the TMA bulk
//    engine (cp.async.bulk + mbarrier, double buffered) and read back as
//    broadcast LDS.128;
//  * the term product is accumulated EXACTLY in exponent form: one 32-bit
//    SWAR add per row-eval of a per-(class, parity) code word
//    (pzx_internal.h), flags in the row's code word mark term ends and
//    7-bit-field flushes;
//  * each term is converted once per assignment to fp64 through small
//    shared-memory tables and accumulated into the amplitude.
//
//   k_eval_general<P64, K, LONG> : any assignment batch; AND + POPC parity per
//                                  (row, assignment), K assignments per thread.
//   k_eval_gray<P64, GB, LONG>   : enumerated batches; a thread owns 2^GB
//                                  assignments differing only in the low GB
//                                  bits: per row 2 POPCs serve all of them, the
//                                  low-bit parities come from the row's
//                                  host-precomputed Walsh pattern.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "pzx_classes.h"
#include "pzx_internal.h"
#include "pzx_slice_dispatch.inc"

#include <map>
#include <mutex>
#include <tuple>

namespace {
// Per-launch host overhead matters for small batches (C1: ~0.1 ms steps), so
// the two driver queries every launch used to make are cached per device:
// the dynamic shared-memory opt-in (cudaFuncSetAttribute only when a kernel
// needs more than it was last granted) and the occupancy per (kernel, block
// size, shared memory).
std::mutex g_attr_mu;
std::map<std::tuple<int, const void*>, size_t> g_smem_set;
std::map<std::tuple<int, const void*, int, size_t>, int> g_occ;

int cur_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

template <class K>
cudaError_t set_max_smem(K* kern, size_t smem) {
    const auto key = std::make_tuple(cur_device(), reinterpret_cast<const void*>(kern));
    std::lock_guard<std::mutex> lock(g_attr_mu);
    auto it = g_smem_set.find(key);
    if (it != g_smem_set.end() && it->second >= smem) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e == cudaSuccess) g_smem_set[key] = smem;
    return e;
}

template <class K>
cudaError_t cached_occupancy(int* nb, K* kern, int threads, size_t smem) {
    const auto key = std::make_tuple(cur_device(), reinterpret_cast<const void*>(kern), threads, smem);
    {
        std::lock_guard<std::mutex> lock(g_attr_mu);
        auto it = g_occ.find(key);
        if (it != g_occ.end()) { *nb = it->second; return cudaSuccess; }
    }
    cudaError_t e = set_max_smem(kern, smem);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(nb, kern, threads, smem);
    if (e == cudaSuccess) {
        std::lock_guard<std::mutex> lock(g_attr_mu);
        g_occ[key] = *nb;
    }
    return e;
}
}  // namespace

namespace pzxb {

// PZX_ACC=smem keeps the accumulators in shared memory (A/B comparisons)
bool tmem_accumulators() {
    static const bool on = [] {
        const char* e = std::getenv("PZX_ACC");
        return !(e && std::string(e) == "smem");
    }();
    return on;
}

namespace {

constexpr int kTileRows = 256;

// Term epilogue decode: 1 = byte-lane bit transposes (slice_epilogue_tr), 0 =
// the round-1 nibble-spread decode (A/B builds: -DPZX_EPI_TRANSPOSE=0)
#ifndef PZX_EPI_TRANSPOSE
#define PZX_EPI_TRANSPOSE 1
#endif
// page kernel: pi terms through the per-warp T[j, a, b] table (page_epilogue_pi)
#ifndef PZX_PI_TAB
#define PZX_PI_TAB 1
#endif
// page kernel: the lane-parity pre-pass split over the CTA's four warps
#ifndef PZX_CTA_PREPASS
#define PZX_CTA_PREPASS 1
#endif
// lambda-term epilogue: TMEM loads one group ahead
#ifndef PZX_EPI_TMEM_PIPE
#define PZX_EPI_TMEM_PIPE 1
#endif

// ------------------------------------------------------------- PTX glue ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// ------------------------------------------------------------ LUT + math ----
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

struct SmemLut {
    const uint32_t* codes;
    uint32_t codes_s;  // shared-window address of codes (16-aligned)
    const double2* om;
    const double* u;
    const double* p3;
    const double2* pd;  // centred: pd[d], d in [-max_rows, max_rows]
    const double2* sab;  // (sqrt2-1)^s pi^a pi'^b, s < 16, a, b < 4, index s | a << 4 | b << 6
    const double* uz;    // (sqrt2-1)^s at s < 16, 0 at s | 16 (page kernel, pi terms)
};

__device__ __forceinline__ SmemLut stage_lut(const DevTable& t, unsigned char* dst_bytes) {
    const uint4* src = reinterpret_cast<const uint4*>(t.lut);
    uint4* dst = reinterpret_cast<uint4*>(dst_bytes);
    const uint32_t n16 = t.lut_layout.bytes / 16;
    for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = __ldg(src + i);
    SmemLut L;
    L.codes = reinterpret_cast<const uint32_t*>(dst_bytes + t.lut_layout.codes_off);
    L.codes_s = smem_u32(L.codes);
    L.om = reinterpret_cast<const double2*>(dst_bytes + t.lut_layout.om_off);
    L.u = reinterpret_cast<const double*>(dst_bytes + t.lut_layout.u_off);
    L.p3 = reinterpret_cast<const double*>(dst_bytes + t.lut_layout.p3_off);
    L.pd = reinterpret_cast<const double2*>(dst_bytes + t.lut_layout.pd_off) + t.lut_layout.max_rows;
    L.sab = reinterpret_cast<const double2*>(dst_bytes + t.lut_layout.sab_off);
    L.uz = reinterpret_cast<const double*>(dst_bytes + t.lut_layout.uz_off);
    return L;
}

// One term at one assignment: amp += C * w^(j + 6 s1) * (sqrt2-1)^s1 * pi^a pi'^b
// (C already carries sqrt2^E and mu^nLM; lambda^s1 mu^(nLM-s1) =
//  mu^nLM (w^6 (sqrt2-1))^s1; pi^a pi'^b = 3^min(a,b) * pi^(a-b) or pi'^(b-a)).
__device__ __forceinline__ void term_epilogue(uint32_t jraw, uint32_t z, uint32_t s1, uint32_t a,
                                              uint32_t b, const double2 C, const SmemLut& L,
                                              double2& amp) {
    if (z != 0) return;
    const uint32_t j = (jraw + 6u * s1) & 7u;
    double2 w = L.om[j];
    if (s1 | a | b) {  // non-monomial factors present
        double r = L.u[s1];
        if (a | b) {
            const uint32_t mn = a < b ? a : b;
            r *= L.p3[mn];
            const double2 pd = L.pd[int(a) - int(b)];
            const double wr = w.x * pd.x - w.y * pd.y;
            const double wi = w.x * pd.y + w.y * pd.x;
            w.x = wr;
            w.y = wi;
        }
        w.x *= r;
        w.y *= r;
    }
    amp.x += C.x * w.x - C.y * w.y;
    amp.y += C.x * w.y + C.y * w.x;
}

__device__ __forceinline__ void epilogue_packed(uint32_t acc, const double2 C, const SmemLut& L,
                                                double2& amp) {
    term_epilogue(acc >> kJShift, acc & kField, (acc >> kS1Shift) & kField, (acc >> kAShift) & kField,
                  (acc >> kBShift) & kField, C, L, amp);
}

struct Wide {
    uint32_t j, z, s1, a, b;
};

__device__ __forceinline__ void widen(Wide& w, uint32_t acc) {
    w.j += acc >> kJShift;
    w.z += acc & kField;
    w.s1 += (acc >> kS1Shift) & kField;
    w.a += (acc >> kAShift) & kField;
    w.b += (acc >> kBShift) & kField;
}

// ------------------------------------------------------------ row stream ----
template <bool P64>
struct Row;

template <>
struct Row<false> {
    uint32_t psi, phi, code, pat;
    static constexpr int kWords = 1;  // uint4 per row
    __device__ __forceinline__ void load(const uint4* p) {
        const uint4 w = *p;
        psi = w.x; phi = w.y; code = w.z; pat = w.w;
    }
    // from a shared-window address (no generic-to-shared conversion per row)
    __device__ __forceinline__ void load_s(uint32_t a) {
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(psi), "=r"(phi), "=r"(code), "=r"(pat) : "r"(a));
    }
    __device__ __forceinline__ uint32_t p(uint64_t a) const { return __popc(psi & uint32_t(a)) & 1u; }
    __device__ __forceinline__ uint32_t q(uint64_t a) const { return __popc(phi & uint32_t(a)) & 1u; }
};

template <>
struct Row<true> {
    uint32_t psi_lo, psi_hi, phi_lo, phi_hi, code, pat;
    static constexpr int kWords = 2;
    __device__ __forceinline__ void load(const uint4* p) {
        const uint4 w = p[0];
        const uint4 x = p[1];
        psi_lo = w.x; psi_hi = w.y; phi_lo = w.z; phi_hi = w.w; code = x.x; pat = x.y;
    }
    __device__ __forceinline__ void load_s(uint32_t a) {
        uint32_t z0, z1;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(psi_lo), "=r"(psi_hi), "=r"(phi_lo), "=r"(phi_hi) : "r"(a));
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(code), "=r"(pat), "=r"(z0), "=r"(z1) : "r"(a + 16u));
    }
    __device__ __forceinline__ uint32_t p(uint64_t a) const {
        return __popc((psi_lo & uint32_t(a)) ^ (psi_hi & uint32_t(a >> 32))) & 1u;
    }
    __device__ __forceinline__ uint32_t q(uint64_t a) const {
        return __popc((phi_lo & uint32_t(a)) ^ (phi_hi & uint32_t(a >> 32))) & 1u;
    }
};

template <int RW>
__host__ __device__ constexpr uint32_t tile_bytes_w() {
    return uint32_t(kTileRows) * RW * 16u;
}
template <bool P64>
__host__ __device__ constexpr uint32_t tile_bytes() {
    return tile_bytes_w<Row<P64>::kWords>();
}

// Shared memory: [tile 0][tile 1][2 mbarriers][LUT]
template <bool P64>
__host__ __device__ constexpr uint32_t smem_lut_offset() {
    return 2 * tile_bytes<P64>() + 16;
}

// Walk the flat row stream of terms [tb, te) -- staged by TMA bulk copies --
// calling cons.row(row) per row, cons.end_term(C) at term ends and
// cons.flush() at 7-bit-field flush points (long terms only).
template <class RowT, bool LONG, class Cons>
__device__ __forceinline__ void stream_rows(const DevTable& t, const uint4* rows, const double2* term_c,
                                            uint64_t tb, uint64_t te, unsigned char* smem, Cons& cons) {
    constexpr int RW = RowT::kWords;
    uint4* tiles = reinterpret_cast<uint4*>(smem);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * tile_bytes_w<RW>());
    const uint64_t R0 = t.term_row[tb], R1 = t.term_row[te];
    const uint32_t ntiles = uint32_t((R1 - R0 + kTileRows - 1) / kTileRows);
    auto issue = [&](uint32_t tile) {
        const uint64_t r = R0 + uint64_t(tile) * kTileRows;
        const uint64_t n = (R1 - r) < uint64_t(kTileRows) ? (R1 - r) : uint64_t(kTileRows);
        const uint32_t bytes = uint32_t(n) * RW * 16u;
        uint64_t* bar = &bars[tile & 1];
        mbar_expect_tx(bar, bytes);
        tma_load_1d(tiles + (tile & 1) * kTileRows * RW, rows + r * RW, bytes, bar);
    };
    if (threadIdx.x == 0) {
        if (ntiles > 0) issue(0);
        if (ntiles > 1) issue(1);
    }
    uint64_t term = tb;
    double2 C = __ldg(term_c + tb);
    double2 Cn = (tb + 1 < te) ? __ldg(term_c + tb + 1) : make_double2(0.0, 0.0);
    for (uint32_t i = 0; i < ntiles; ++i) {
        const uint32_t sbuf = smem_u32(tiles) + (i & 1) * uint32_t(kTileRows) * RW * 16u;
        mbar_wait(&bars[i & 1], (i >> 1) & 1u);
        const uint64_t rem = R1 - R0 - uint64_t(i) * kTileRows;
        const uint32_t n = rem < uint64_t(kTileRows) ? uint32_t(rem) : uint32_t(kTileRows);
        for (uint32_t k = 0; k < n; ++k) {
            RowT row;
            row.load_s(sbuf + k * RW * 16u);
            cons.row(row);
            if (row.code & kEndFlag) {
                cons.end_term(C);
                C = Cn;
                ++term;
                Cn = (term + 1 < te) ? __ldg(term_c + term + 1) : make_double2(0.0, 0.0);
            } else if (LONG && (row.code & kSegFlag)) {
                cons.flush();
            }
        }
        __syncthreads();  // every thread is done with buffer (i & 1)
        if (threadIdx.x == 0 && i + 2 < ntiles) {
            fence_proxy_async();
            issue(i + 2);
        }
    }
}

__device__ __forceinline__ void term_range(const LaunchReq& r, uint64_t& tb, uint64_t& te) {
    if (r.n_chunks > 1) {
        tb = r.d_chunk_terms[blockIdx.y];
        te = r.d_chunk_terms[blockIdx.y + 1];
    } else {
        tb = r.term_begin;
        te = r.term_end;
    }
}

__device__ __forceinline__ void store_result(const LaunchReq& r, uint64_t idx, double2 amp) {
    if (idx >= r.n) return;
    if (r.n_chunks > 1) {
        r.d_partial[uint64_t(blockIdx.y) * r.n + idx] = amp;
        return;
    }
    if (r.d_perm) {  // sorted batch: back to the caller's order (~0: a padding slot)
        idx = r.d_perm[idx];
        if (idx == 0xFFFFFFFFu) return;
    }
    if (r.accumulate) {
        const double2 o = r.d_amp[idx];
        amp.x += o.x;
        amp.y += o.y;
    }
    if (r.d_amp) r.d_amp[idx] = amp;
    if (r.d_prob) r.d_prob[idx] = r.prob_mode == 2 ? amp.x : amp.x * amp.x + amp.y * amp.y;
}

__device__ __forceinline__ SmemLut kernel_prologue(const DevTable& t, unsigned char* smem, uint32_t lut_off) {
    const SmemLut L = stage_lut(t, smem + lut_off);
    if (threadIdx.x == 0) {
        uint64_t* bars = reinterpret_cast<uint64_t*>(smem + lut_off - 16);
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    return L;
}

// ------------------------------------------------------- general kernel ----
template <bool P64, int K, bool LONG>
struct GeneralCons {
    const SmemLut& L;
    uint64_t a[K];
    uint32_t acc[K];
    Wide w[LONG ? K : 1];
    double2 amp[K];
    __device__ __forceinline__ explicit GeneralCons(const SmemLut& l) : L(l) {}
    __device__ __forceinline__ void row(const Row<P64>& v) {
        const uint32_t cb = L.codes_s + (v.code & kCodeMask);
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] += lds_u32(cb | (v.p(a[k]) << 2) | (v.q(a[k]) << 3));
    }
    __device__ __forceinline__ void flush() {
        if constexpr (LONG) {
#pragma unroll
            for (int k = 0; k < K; ++k) { widen(w[k], acc[k]); acc[k] = 0; }
        }
    }
    __device__ __forceinline__ void end_term(const double2 C) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if constexpr (LONG) {
                widen(w[k], acc[k]);
                term_epilogue(w[k].j, w[k].z, w[k].s1, w[k].a, w[k].b, C, L, amp[k]);
                w[k] = Wide{0, 0, 0, 0, 0};
            } else {
                epilogue_packed(acc[k], C, L, amp[k]);
            }
            acc[k] = 0;
        }
    }
};

template <bool P64, int K, bool LONG>
__global__ void __launch_bounds__(kThreads) k_eval_general(const DevTable t, const LaunchReq r) {
    extern __shared__ __align__(128) unsigned char smem[];
    const SmemLut L = kernel_prologue(t, smem, smem_lut_offset<P64>());
    uint64_t tb, te;
    term_range(r, tb, te);
    GeneralCons<P64, K, LONG> c(L);
    const uint64_t idx0 = uint64_t(blockIdx.x) * (kThreads * K) + threadIdx.x;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint64_t idx = idx0 + uint64_t(k) * kThreads;
        c.a[k] = idx < r.n ? (r.d_asg ? r.d_asg[idx] : r.first + idx) : 0;
        c.acc[k] = 0;
        c.amp[k] = make_double2(0.0, 0.0);
        if constexpr (LONG) c.w[k] = Wide{0, 0, 0, 0, 0};
    }
    if (tb < te) stream_rows<Row<P64>, LONG>(t, t.rows, t.term_c, tb, te, smem, c);
#pragma unroll
    for (int k = 0; k < K; ++k) store_result(r, idx0 + uint64_t(k) * kThreads, c.amp[k]);
}

// ---------------------------------------------------------- gray kernel ----
// parity(m & (base | g)) = parity(m & base) ^ parity(m_low & g); the second
// term, for all g at once, is the row's Walsh pattern.
template <bool P64, int GB, bool LONG>
struct GrayCons {
    static constexpr int G = 1 << GB;
    const SmemLut& L;
    uint64_t base;
    uint32_t acc[G];
    Wide w[LONG ? G : 1];
    double2 amp[G];
    __device__ __forceinline__ explicit GrayCons(const SmemLut& l) : L(l) {}
    __device__ __forceinline__ void row(const Row<P64>& v) {
        const uint32_t xi = v.pat ^ (0x55555555u * v.p(base)) ^ (0xAAAAAAAAu * v.q(base));
        // shared address of the row's class (16-aligned) OR the variant's byte
        // offset (idx * 4): one shift + one LOP3 + one LDS + one IADD per row-eval
        const uint32_t cb = L.codes_s + (v.code & kCodeMask);
#pragma unroll
        for (int g = 0; g < G; ++g) {
            // xi >> (2g - 2) as a multiply-high: keeps the shift on the FMA pipe
            // (IMAD.HI) so the ALU pipe only carries the LOP3 and half the adds
            const uint32_t sh = g == 0 ? (xi << 2) : g == 1 ? xi : __umulhi(xi, 1u << (34 - 2 * g));
            acc[g] += lds_u32(cb | (sh & 0xCu));
        }
    }
    __device__ __forceinline__ void flush() {
        if constexpr (LONG) {
#pragma unroll
            for (int g = 0; g < G; ++g) { widen(w[g], acc[g]); acc[g] = 0; }
        }
    }
    __device__ __forceinline__ void end_term(const double2 C) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
            if constexpr (LONG) {
                widen(w[g], acc[g]);
                term_epilogue(w[g].j, w[g].z, w[g].s1, w[g].a, w[g].b, C, L, amp[g]);
                w[g] = Wide{0, 0, 0, 0, 0};
            } else {
                epilogue_packed(acc[g], C, L, amp[g]);
            }
            acc[g] = 0;
        }
    }
};

template <bool P64, int GB, bool LONG>
__global__ void __launch_bounds__(kThreads) k_eval_gray(const DevTable t, const LaunchReq r) {
    constexpr int G = 1 << GB;
    extern __shared__ __align__(128) unsigned char smem[];
    const SmemLut L = kernel_prologue(t, smem, smem_lut_offset<P64>());
    uint64_t tb, te;
    term_range(r, tb, te);
    GrayCons<P64, GB, LONG> c(L);
    const uint64_t off = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) * G;
    // explicit word lists reach this kernel only when the host verified that
    // they are contiguous and 16-aligned: the thread's first word is its base
    c.base = r.d_asg ? (off < r.n ? r.d_asg[off] : 0) : r.first + off;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        c.acc[g] = 0;
        c.amp[g] = make_double2(0.0, 0.0);
        if constexpr (LONG) c.w[g] = Wide{0, 0, 0, 0, 0};
    }
    if (tb < te) stream_rows<Row<P64>, LONG>(t, t.rows, t.term_c, tb, te, smem, c);
#pragma unroll
    for (int g = 0; g < G; ++g) store_result(r, off + g, c.amp[g]);
}

// --------------------------------------------------------- slice kernel ----
// Bit-sliced evaluation of enumerated / contiguous batches:
// a thread owns 32 assignments base + g; each 32-bit register holds one bit
// of a per-assignment quantity for all 32 of them. Per row:
//   X = Walsh32(psi) ^ -(parity(psi & base)),  Y likewise   (bit g = p_g, q_g)
// then a class-specialised LOP3 chain (truth tables are compile-time
// constants of the row's class, see pzx_classes.h) adds the row's phase
// exponent w'(p,q) into the mod-8 counter (J2 J1 J0), ORs zero indicators
// into Z, and bumps bit-sliced lambda / pi / pi' counters. One warp-uniform
// indirect branch per row selects the chain.

constexpr int kSliceThreads = 128;
constexpr int kSliceBits = 5;
constexpr int kSliceG = 1 << kSliceBits;  // 32 assignments per thread, one bit each
constexpr int kSliceTile = 512;           // rows (32 B each) per TMA-staged tile
constexpr int kPlanes = 7;                // bit-sliced counters up to 127 (terms <= kSegRows rows)

__device__ __forceinline__ double2 lds_d2(uint32_t addr) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ double lds_d(uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr));
    return v;
}

// Bit-sliced lambda / pi / pi' counters (one bit per assignment per plane,
// up to kPlanes planes = counts < 128). The planes the epilogue fast path reads
// (s1 < 16, a, b < 4) stay in registers; the rarely reached high planes live
// in shared memory ([plane][NT], conflict-free) so they cost no registers.
constexpr int kLoS = 4, kLoAB = 2;
constexpr int kHiPlanes = (kPlanes - kLoS) + 2 * (kPlanes - kLoAB);  // 14 shared planes per thread

template <int NT, bool LOCAL = false>
struct KindCounters {
    static constexpr uint32_t stride = LOCAL ? 1u : uint32_t(NT);  // planes [kHiPlanes][stride]
    uint32_t S[kLoS], A[kLoAB], B[kLoAB];
    uint32_t nS, nA, nB;
    uint32_t* hi;  // this thread's column of the shared planes, or its local array (LOCAL)

    __device__ __forceinline__ uint32_t* hs(int i) { return hi + (i - kLoS) * stride; }
    __device__ __forceinline__ uint32_t* ha(int i) { return hi + (kPlanes - kLoS + i - kLoAB) * stride; }
    __device__ __forceinline__ uint32_t* hb(int i) { return hi + (2 * kPlanes - kLoS - kLoAB + i - kLoAB) * stride; }

    __device__ __forceinline__ void init(uint32_t* h) {
        hi = h;
#pragma unroll
        for (int i = 0; i < kLoS; ++i) S[i] = 0;
#pragma unroll
        for (int i = 0; i < kLoAB; ++i) A[i] = B[i] = 0;
        nS = nA = nB = 0;
#pragma unroll
        for (int i = 0; i < kHiPlanes; ++i) hi[i * stride] = 0;
    }
    // counter += v; n = rows that could have bumped it so far (warp-uniform),
    // so only planes below bit_length(n) move
    template <int LO, typename HiPlane>
    __device__ __forceinline__ static void bump(uint32_t (&P)[LO], uint32_t n, uint32_t v, HiPlane hp) {
        uint32_t t = v;
#pragma unroll
        for (int i = 0; i < LO; ++i) {
            if (i > 0 && (n >> i) == 0) return;
            const uint32_t u = P[i] & t;
            P[i] ^= t;
            t = u;
        }
        for (int i = LO; i < kPlanes; ++i) {
            if ((n >> i) == 0) return;
            uint32_t* q = hp(i);
            const uint32_t p = *q;
            *q = p ^ t;
            t &= p;
        }
    }
    __device__ __forceinline__ void bump_s(uint32_t v) { bump<kLoS>(S, ++nS, v, [&](int i) { return hs(i); }); }
    __device__ __forceinline__ void bump_a(uint32_t v) { bump<kLoAB>(A, ++nA, v, [&](int i) { return ha(i); }); }
    __device__ __forceinline__ void bump_b(uint32_t v) { bump<kLoAB>(B, ++nB, v, [&](int i) { return hb(i); }); }

    template <int LO, typename HiPlane>
    __device__ __forceinline__ static uint32_t decode(const uint32_t (&P)[LO], uint32_t n, int g, HiPlane hp) {
        uint32_t x = 0;
#pragma unroll
        for (int i = 0; i < LO; ++i) x |= ((P[i] >> g) & 1u) << i;
        for (int i = LO; i < kPlanes; ++i) {
            if ((n >> i) == 0) break;
            x |= ((*hp(i) >> g) & 1u) << i;
        }
        return x;
    }
    __device__ __forceinline__ uint32_t s_of(int g) { return decode<kLoS>(S, nS, g, [&](int i) { return hs(i); }); }
    __device__ __forceinline__ uint32_t a_of(int g) { return decode<kLoAB>(A, nA, g, [&](int i) { return ha(i); }); }
    __device__ __forceinline__ uint32_t b_of(int g) { return decode<kLoAB>(B, nB, g, [&](int i) { return hb(i); }); }

    __device__ __forceinline__ bool any() const { return (nS | nA | nB) != 0; }
    __device__ __forceinline__ bool fits_fast() const { return nS < 16 && nA < 4 && nB < 4; }
    __device__ __forceinline__ bool has_pi() const { return (nA | nB) != 0; }
    __device__ __forceinline__ void reset() {
        for (int i = kLoS; i < kPlanes && (nS >> i); ++i) *hs(i) = 0;
        for (int i = kLoAB; i < kPlanes && (nA >> i); ++i) *ha(i) = 0;
        for (int i = kLoAB; i < kPlanes && (nB >> i); ++i) *hb(i) = 0;
#pragma unroll
        for (int i = 0; i < kLoS; ++i) S[i] = 0;
#pragma unroll
        for (int i = 0; i < kLoAB; ++i) A[i] = B[i] = 0;
        nS = nA = nB = 0;
    }
};

template <bool P64>
__host__ __device__ constexpr uint32_t slice_lut_offset() {
    return 2 * kSliceTile * 32 + 16;
}

// ---- tensor memory (TMEM) accumulators --------------------------------------
// The bit-sliced kernels keep 32 fp64 complex accumulators per thread. In TMEM
// (128 lanes x 512 columns x 32 bit per SM) a 128-thread CTA holds them in 128
// columns: thread (warp w, lane l) owns TMEM lane 32 w + l, assignment g at
// columns 4g .. 4g+3 (re lo/hi, im lo/hi). That frees the 64 KB of shared
// memory per CTA the accumulators would otherwise take: 4 CTAs (16 warps) per
// SM instead of 3 (slice) or 2 (sorted).
constexpr uint32_t kTmemCols = 128;
constexpr size_t kTmemCtaSmem = 51200;  // dynamic smem floor: at most 4 CTAs/SM (= 512 TMEM columns)

// PZX_SLICE2=1 sends large enumerated batches to the two-slice kernel (default off)
bool slice2_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PZX_SLICE2");
        return e && std::string(e) == "1";  // measured slower than 16 warps x one slice
    }();
    return on;
}


__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
                 ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
                 ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_sync_fence() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// warp 0 allocates COLS columns; returns this thread's address: its warp's lane
// quarter, and for CTAs of more than 4 warps the 128-column block of its warp
// group (warps 4..7 use columns 128..255)
template <uint32_t COLS = kTmemCols>
__device__ __forceinline__ uint32_t tmem_alloc_cta(uint32_t* base_s) {
    if ((threadIdx.x >> 5) == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(base_s)),
                     "n"(COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tmem_sync_fence();
    return *base_s + ((((threadIdx.x >> 5) & 3u) * 32u) << 16) + (threadIdx.x >> 7) * kTmemCols;
}
__device__ __forceinline__ uint32_t tmem_base_of(uint32_t taddr) { return taddr & 0x0000FFFFu; }
template <uint32_t COLS = kTmemCols>
__device__ __forceinline__ void tmem_free_cta(uint32_t base) {
    tmem_sync_fence();
    if ((threadIdx.x >> 5) == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(COLS) : "memory");
}
__device__ __forceinline__ double2 v2d(const uint32_t* v) {
    return make_double2(__hiloint2double(int(v[1]), int(v[0])), __hiloint2double(int(v[3]), int(v[2])));
}
__device__ __forceinline__ void d2v(double2 d, uint32_t* v) {
    v[0] = uint32_t(__double2loint(d.x));
    v[1] = uint32_t(__double2hiint(d.x));
    v[2] = uint32_t(__double2loint(d.y));
    v[3] = uint32_t(__double2hiint(d.y));
}

// Accumulator home of a bit-sliced kernel thread: shared memory ([g][NT]) or TMEM.
template <int NT, bool TM>
struct SliceAcc {
    double2* amp_s;  // !TM
    uint32_t taddr;  // TM: this thread's lane, column 0
    __device__ __forceinline__ void zero() {
        if constexpr (TM) {
            uint32_t v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0u;
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_st32(taddr + 32u * c, v);
            tmem_wait_st();
        } else {
#pragma unroll
            for (int g = 0; g < kSliceG; ++g) amp_s[g * NT + threadIdx.x] = make_double2(0.0, 0.0);
        }
    }
};

// Term constants reach the epilogue through two per-warp shared slots filled
// by cp.async one term ahead (no registers live across the row loop).
struct TermC {
    double2* slot;   // this warp's 2 slots
    uint64_t next;   // index of the next constant to prefetch
    uint64_t end;
};
__device__ __forceinline__ void termc_fetch(TermC& tc, const double2* src) {
    const uint32_t k = uint32_t(tc.next & 1u);  // term i lives in slot i & 1
    // one commit group per call (empty past the end) keeps "wait_group 1" exact
    if ((threadIdx.x & 31u) == 0) {
        if (tc.next < tc.end)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(tc.slot + k)),
                         "l"(src + tc.next));
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    ++tc.next;
}
__device__ __forceinline__ void termc_init(TermC& tc, double2* slot, const double2* src, uint64_t tb, uint64_t te) {
    tc.slot = slot;
    tc.next = tb;
    tc.end = te;
    termc_fetch(tc, src);
    termc_fetch(tc, src);
}
// C of term (tc.next - 2); then refill its slot with term tc.next
__device__ __forceinline__ double2 termc_take(TermC& tc, const double2* src) {
    const uint32_t k = uint32_t(tc.next & 1u);  // == (tc.next - 2) & 1
    if ((threadIdx.x & 31u) == 0) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncwarp();
    const double2 C = tc.slot[k];
    __syncwarp();
    termc_fetch(tc, src);
    return C;
}

constexpr int kCrot = 16;  // per-warp phase table: C * w^j for j < 8, zeros for Z-marked (dead) assignments
constexpr int kWarpScratch = kCrot + 2;  // + the two TermC slots (double2 units per warp)

// Fixed-width decode of bit-sliced counters, 4 assignments at a time:
// nibble m of plane P (bits 4m..4m+3, pre-split into Q = P & 0x0F0F0F0F and
// Q' = (P >> 4) & 0x0F0F0F0F so one PRMT isolates it) is spread to bit k of
// bytes 0..3 by one multiply: bit i * (1 + 2^7 + 2^14 + 2^21) lands on 8i for
// i < 4, and no two partial products overlap below 2^25, so masking the
// product keeps exactly bit i -> byte i.
struct Nib {
    uint32_t lo, hi;
};
__device__ __forceinline__ Nib nib_split(uint32_t p) { return Nib{p & 0x0F0F0F0Fu, (p >> 4) & 0x0F0F0F0Fu}; }

// m (group of 4 assignments) may be a runtime value; k is a compile-time constant
__device__ __forceinline__ uint32_t nib_spread(const Nib& q, int m, int k) {
    const uint32_t n = __byte_perm((m & 1) ? q.hi : q.lo, 0u, 0x4440u | uint32_t(m >> 1));
    return (n * (0x00204081u << k)) & (0x01010101u << k);
}

// Term epilogue shared by the bit-sliced kernels: fold 6*s1 into J, build
// the warp's C * w^j table, and add every live assignment's term value into its
// fp64 accumulator; resets the per-term state. Fast path (every counter fits
// its field: s1 < 16, a, b < 4): per group of 4 assignments two byte-keys
// words are built by nib_spread -- (j | Z << 3) and (s1 | a << 4 | b << 6) --
// then each assignment is 2 table loads + 4 DFMA into its accumulator, no
// branches (Z-marked assignments read a zero entry).
// KINDS: some lambda / pi / pi' rows (the (sqrt2-1)^s pi^a pi'^b table is
// read); AB: planes of the pi / pi' counters to decode (0: pi-free term, 1: a,
// b < 2, 2: a, b < 4) -- known-zero planes are skipped
template <int NT, bool TM, bool KINDS, bool ROLL, int AB = 2, bool LC = false>
__device__ __forceinline__ void slice_epilogue_fast(const SmemLut& L, const double2* crot, SliceAcc<NT, TM>& acc,
                                                    uint32_t J0, uint32_t J1, uint32_t J2, uint32_t Z,
                                                    const KindCounters<NT, LC>& K) {
    const uint32_t(&S)[kLoS] = K.S;
    const uint32_t(&A)[kLoAB] = K.A;
    const uint32_t(&B)[kLoAB] = K.B;
    const Nib j0 = nib_split(J0), j1 = nib_split(J1), j2 = nib_split(J2), z = nib_split(Z);
    Nib s0{}, s1{}, s2{}, s3{}, a0{}, a1{}, b0{}, b1{};
    if constexpr (KINDS) {
        s0 = nib_split(S[0]); s1 = nib_split(S[1]); s2 = nib_split(S[2]); s3 = nib_split(S[3]);
        if constexpr (AB >= 1) {
            a0 = nib_split(A[0]);
            b0 = nib_split(B[0]);
        }
        if constexpr (AB >= 2) {
            a1 = nib_split(A[1]);
            b1 = nib_split(B[1]);
        }
    }
    auto mac = [&](double2& o, const double2 c, const double2 f) {
        if constexpr (KINDS && AB > 0) {
            o.x = fma(c.x, f.x, o.x);
            o.y = fma(c.x, f.y, o.y);
            o.x = fma(-c.y, f.y, o.x);
            o.y = fma(c.y, f.x, o.y);
        } else if constexpr (KINDS) {  // pi-free term: the table entry (sqrt2-1)^s is real
            o.x = fma(c.x, f.x, o.x);
            o.y = fma(c.y, f.x, o.y);
        } else {
            o.x += c.x;
            o.y += c.y;
        }
    };
    // the term values of group m (4 assignments): c[r] * f[r]
    auto group = [&](int m, double2 (&c)[4], double2 (&f)[4]) {
        const uint32_t kj = nib_spread(j0, m, 0) | nib_spread(j1, m, 1) | nib_spread(j2, m, 2) | nib_spread(z, m, 3);
        uint32_t ks = 0;  // s | a << 4 | b << 6
        if constexpr (KINDS) {
            ks = nib_spread(s0, m, 0) | nib_spread(s1, m, 1) | nib_spread(s2, m, 2) | nib_spread(s3, m, 3);
            if constexpr (AB >= 1) ks |= nib_spread(a0, m, 4) | nib_spread(b0, m, 6);
            if constexpr (AB >= 2) ks |= nib_spread(a1, m, 5) | nib_spread(b1, m, 7);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            c[r] = crot[__byte_perm(kj, 0u, 0x4440u | uint32_t(r))];
            if constexpr (KINDS && AB > 0) {
                const uint32_t k = __byte_perm(ks, 0u, 0x4440u | uint32_t(r));
                f[r] = L.sab[k ^ ((k >> 4) & 3u) ^ (((k >> 6) & 1u) << 2)];  // the table's bank swizzle
            } else if constexpr (KINDS) {
                f[r].x = reinterpret_cast<const double*>(L.sab)[2 * __byte_perm(ks, 0u, 0x4440u | uint32_t(r))];
                f[r].y = 0.0;
            }
        }
    };
    if constexpr (TM) {
        // 8 groups of 4 assignments = 16 TMEM columns each; the load of group
        // m + 1 is in flight while group m is computed (wait::ld waits for all)
        // (ROLL: a rolled loop over pairs of groups keeps the epilogue's code
        // small -- the row loop and its jump targets stay in the I-cache)
        tmem_wait_st();  // the previous term's stores have landed
        auto pair = [&](int m2) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int m = m2 + h;
                double2 c[4], f[4];
                uint32_t v[16];
                tmem_ld16(acc.taddr + 16u * m, v);
                group(m, c, f);
                tmem_wait_ld();
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    double2 o = v2d(v + 4 * r);
                    mac(o, c[r], f[r]);
                    d2v(o, v + 4 * r);
                }
                tmem_st16(acc.taddr + 16u * m, v);
            }
        };
        if constexpr (ROLL) {
#pragma unroll 1
            for (int m2 = 0; m2 < 8; m2 += 2) pair(m2);
        } else {
#pragma unroll
            for (int m2 = 0; m2 < 8; m2 += 2) pair(m2);
        }
    } else {
        double2* ap = acc.amp_s + threadIdx.x;
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            // all loads of the group first: the accumulator stores below may alias
            // them as far as the compiler knows, so this order is what buys ILP
            double2 c[4], f[4], o[4];
            group(m, c, f);
#pragma unroll
            for (int r = 0; r < 4; ++r) o[r] = ap[(4 * m + r) * NT];
#pragma unroll
            for (int r = 0; r < 4; ++r) mac(o[r], c[r], f[r]);
#pragma unroll
            for (int r = 0; r < 4; ++r) ap[(4 * m + r) * NT] = o[r];
        }
    }
}

// 8 bit planes -> per-assignment keys: an 8 x 8 bit transpose inside every
// byte lane (three delta-swap stages). Before: P[c] bit (8m + k) = plane c of
// assignment 8m + k. After: P[k] byte m bit c = plane c of assignment 8m + k,
// i.e. byte m of P[k] is assignment 8m + k's 8-bit key. ~60 LOP3/SHF for all
// 32 assignments x 8 planes (the nibble-spread decode it replaces took 0.75
// instructions per plane and assignment, i.e. 192).
__device__ __forceinline__ void transpose8_bytes(uint32_t (&P)[8]) {
#pragma unroll
    for (int s = 4; s > 0; s >>= 1) {
        const uint32_t m = s == 4 ? 0x0F0F0F0Fu : s == 2 ? 0x33333333u : 0x55555555u;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (c & s) continue;
            const uint32_t t = ((P[c] >> s) ^ P[c + s]) & m;
            P[c + s] ^= t;
            P[c] ^= t << s;
        }
    }
}

// Epilogue of a term with lambda / mu rows only (fast counters; every TMEM kernel):
// acc += crot[j] * uz[s | 16 z]. Two byte-lane transposes of mostly-zero
// planes put j at bits 4..6 (the crot byte offset) and s | 16 z at bits 3..7
// (the uz byte offset): no LEA, and dead assignments read crot[j] -- entries
// 0..7 fill the 32 banks exactly, so no bank conflict -- times uz[31] = 0
// (slice_epilogue_tr KIND 1 sends them to one zero entry that conflicts with
// the live j = 7 reads).
template <int NT, bool LC>
__device__ __forceinline__ void page_epilogue_lam(const SmemLut& L, uint32_t crot_s, SliceAcc<NT, true>& acc,
                                                  uint32_t J0, uint32_t J1, uint32_t J2, uint32_t Z,
                                                  const KindCounters<NT, LC>& K) {
    uint32_t R[8] = {0u, 0u, 0u, 0u, J0, J1, J2, 0u};
    transpose8_bytes(R);
    uint32_t Q[8] = {0u, 0u, 0u, K.S[0] | Z, K.S[1] | Z, K.S[2] | Z, K.S[3] | Z, Z};
    transpose8_bytes(Q);
    const uint32_t uz_s = smem_u32(L.uz);
    tmem_wait_st();
#if PZX_EPI_TMEM_PIPE
    // TMEM loads one group of 4 assignments ahead: group k+1's tcgen05.ld is in
    // flight while group k is looked up and accumulated (two register sets)
    uint32_t va[16], vb[16];
    tmem_ld16(acc.taddr, va);
    auto group = [&](int k, uint32_t (&v)[16], uint32_t (&vn)[16]) {
        const uint32_t sel = 0x4440u | uint32_t(k >> 1);
        const int h = k & 1;
        double2 c[4];
        double f[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            c[r] = lds_d2(crot_s + __byte_perm(R[4 * h + r], 0u, sel));
            f[r] = lds_d(uz_s + __byte_perm(Q[4 * h + r], 0u, sel));
        }
        tmem_wait_ld();
        if (k < 7) tmem_ld16(acc.taddr + 16u * uint32_t(k + 1), vn);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            double2 o = v2d(v + 4 * r);
            o.x = fma(c[r].x, f[r], o.x);
            o.y = fma(c[r].y, f[r], o.y);
            d2v(o, v + 4 * r);
        }
        tmem_st16(acc.taddr + 16u * uint32_t(k), v);
    };
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
        group(k, va, vb);
        group(k + 1, vb, va);
    }
#else
#pragma unroll 1
    for (int m = 0; m < 4; ++m) {
        const uint32_t sel = 0x4440u | uint32_t(m);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint32_t v[16];
            tmem_ld16(acc.taddr + 16u * uint32_t(2 * m + h), v);
            double2 c[4];
            double f[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                c[r] = lds_d2(crot_s + __byte_perm(R[4 * h + r], 0u, sel));
                f[r] = lds_d(uz_s + __byte_perm(Q[4 * h + r], 0u, sel));
            }
            tmem_wait_ld();
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                double2 o = v2d(v + 4 * r);
                o.x = fma(c[r].x, f[r], o.x);
                o.y = fma(c[r].y, f[r], o.y);
                d2v(o, v + 4 * r);
            }
            tmem_st16(acc.taddr + 16u * uint32_t(2 * m + h), v);
        }
    }
#endif
}

// Term epilogue fast path, TMEM accumulators, transposed decode.
// The planes are grouped so that each transposed byte IS a table index:
//   KIND 0 (kind-free term):  {J0 J1 J2 Z}         -> crot[j | z << 3]              acc += C w^j
//   KIND 1 (lambda rows only): {J0 J1 J2 Z S0..S3} -> crot[b & 15], u[b >> 4]       acc += C w^j (sqrt2-1)^s
//   KIND 2 (pi / pi' rows):    {J0 J1 J2 Z}, {S0..S3 A0 A1 B0 B1}
//                              -> crot[b1], sab[b2 = s | a << 4 | b << 6]         acc += C w^j (sqrt2-1)^s pi^a pi'^b
// (crot: the warp's C * w^j table with zeros for Z-marked assignments.) A
// byte is picked with one PRMT and turned into an address with one LEA;
// groups of 4 consecutive assignments (16 TMEM columns) are loaded / stored
// together; assignment 8m + 4h + r is byte m of key word 4h + r.
template <int NT, int KIND, bool LC>
__device__ __forceinline__ void slice_epilogue_tr(const SmemLut& L, const double2* crot, SliceAcc<NT, true>& acc,
                                                  uint32_t J0, uint32_t J1, uint32_t J2, uint32_t Z,
                                                  const KindCounters<NT, LC>& K) {
    // Z-marked assignments all read crot[15] (zero): OR-ing Z into the j planes
    // keeps the dead lanes off the live entries' bank groups
    uint32_t Q[8] = {J0 | Z, J1 | Z, J2 | Z, Z, 0u, 0u, 0u, 0u};
    if constexpr (KIND == 1) {
        Q[4] = K.S[0]; Q[5] = K.S[1]; Q[6] = K.S[2]; Q[7] = K.S[3];
    }
    if constexpr (KIND == 1) {
        page_epilogue_lam<NT, LC>(L, smem_u32(crot), acc, J0, J1, J2, Z, K);
        return;
    }
    transpose8_bytes(Q);
    uint32_t R[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    if constexpr (KIND == 2) {  // key = sab_index(s, a, b): low s bits XOR (a | b0 << 2), the table's swizzle
        R[0] = K.S[0] ^ K.A[0]; R[1] = K.S[1] ^ K.A[1]; R[2] = K.S[2] ^ K.B[0]; R[3] = K.S[3];
        R[4] = K.A[0]; R[5] = K.A[1]; R[6] = K.B[0]; R[7] = K.B[1];
        transpose8_bytes(R);
    }
    const uint32_t crot_s = smem_u32(crot);
    const uint32_t u_s = smem_u32(L.u), sab_s = smem_u32(L.sab);
    tmem_wait_st();  // the previous term's stores have landed
#pragma unroll 1
    for (int m = 0; m < 4; ++m) {
        const uint32_t sel = 0x4440u | uint32_t(m);  // PRMT: byte m -> byte 0, zeros above
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint32_t v[16];
            tmem_ld16(acc.taddr + 16u * uint32_t(2 * m + h), v);
            double2 c[4];
            double2 f[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const uint32_t b = __byte_perm(Q[4 * h + r], 0u, sel);
                if constexpr (KIND == 1) {
                    c[r] = lds_d2(crot_s + ((b & 15u) << 4));
                    f[r].x = lds_d(u_s + ((b >> 4) << 3));
                } else {
                    c[r] = lds_d2(crot_s + (b << 4));
                    if constexpr (KIND == 2) f[r] = lds_d2(sab_s + (__byte_perm(R[4 * h + r], 0u, sel) << 4));
                }
            }
            tmem_wait_ld();
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                double2 o = v2d(v + 4 * r);
                if constexpr (KIND == 0) {
                    o.x += c[r].x;
                    o.y += c[r].y;
                } else if constexpr (KIND == 1) {
                    o.x = fma(c[r].x, f[r].x, o.x);
                    o.y = fma(c[r].y, f[r].x, o.y);
                } else {
                    o.x = fma(c[r].x, f[r].x, o.x);
                    o.y = fma(c[r].x, f[r].y, o.y);
                    o.x = fma(-c[r].y, f[r].y, o.x);
                    o.y = fma(c[r].y, f[r].x, o.y);
                }
                d2v(o, v + 4 * r);
            }
            tmem_st16(acc.taddr + 16u * uint32_t(2 * m + h), v);
        }
    }
}

// Any counter widths: one assignment's term value (0 when Z-marked).
template <int NT, bool LC = false>
__device__ __forceinline__ double2 slice_value_slow(const SmemLut& L, const double2* crot, uint32_t J0, uint32_t J1,
                                                    uint32_t J2, uint32_t Z, KindCounters<NT, LC>& K, int g) {
    if ((Z >> g) & 1u) return make_double2(0.0, 0.0);
    const uint32_t j = ((J0 >> g) & 1u) | (((J1 >> g) & 1u) << 1) | (((J2 >> g) & 1u) << 2);
    double2 v = crot[j];
    const uint32_t s1 = K.s_of(g);
    const uint32_t a = K.a_of(g);
    const uint32_t b = K.b_of(g);
    double rr = L.u[s1];
    if (a | b) {
        const uint32_t mn = a < b ? a : b;
        rr *= L.p3[mn];
        const double2 pd = L.pd[int(a) - int(b)];
        const double vr = v.x * pd.x - v.y * pd.y;
        v.y = v.x * pd.y + v.y * pd.x;
        v.x = vr;
    }
    v.x *= rr;
    v.y *= rr;
    return v;
}

// Term epilogue, part 1 (once per warp and term): C from its cp.async slot,
// the warp's C * w^j table (zeros for Z-marked assignments at 8..15).
__device__ __forceinline__ void slice_epilogue_begin(TermC& tc, const double2* src, const SmemLut& L,
                                                     double2* crot) {
    const uint32_t lane = threadIdx.x & 31u;
    const double2 C = termc_take(tc, src);
    if (lane < uint32_t(kCrot)) {
        double2 v = make_double2(0.0, 0.0);
        if (lane < 8) {
            const double2 w = L.om[lane];
            v = make_double2(C.x * w.x - C.y * w.y, C.x * w.y + C.y * w.x);
        }
        crot[lane] = v;
    }
    __syncwarp();
}

// Term epilogue, part 2 (per 32-assignment slice): fold 6*s1 into J, add
// every live assignment's term value into its accumulator, reset the state.
template <int NT, bool TM, bool ROLL = false, bool LC = false>
__device__ __forceinline__ void slice_epilogue_apply(const SmemLut& L, const double2* crot, SliceAcc<NT, TM>& acc,
                                                     uint32_t& J0, uint32_t& J1, uint32_t& J2, uint32_t& Z,
                                                     KindCounters<NT, LC>& K) {
    if (K.nS) {  // (lambda/mu)^s1 = mu^.. * w^(6 s1) * (sqrt2-1)^s1: add 6*s1 mod 8 to J
        const uint32_t w1 = K.S[0], w2 = K.S[0] ^ K.S[1];
        const uint32_t c1 = J1 & w1;
        J1 ^= w1;
        J2 ^= w2 ^ c1;
    }
    const bool kinds = K.any();
#if PZX_EPI_TRANSPOSE
    if constexpr (TM) {
        if (!kinds) {
            slice_epilogue_tr<NT, 0, LC>(L, crot, acc, J0, J1, J2, Z, K);
            J0 = J1 = J2 = Z = 0;
            return;
        }
        if (K.fits_fast()) {
            if (!K.has_pi()) slice_epilogue_tr<NT, 1, LC>(L, crot, acc, J0, J1, J2, Z, K);
            else slice_epilogue_tr<NT, 2, LC>(L, crot, acc, J0, J1, J2, Z, K);
            J0 = J1 = J2 = Z = 0;
            K.reset();
            return;
        }
    }
#endif
    if (!kinds) {
        slice_epilogue_fast<NT, TM, false, ROLL, 2, LC>(L, crot, acc, J0, J1, J2, Z, K);
    } else if (K.fits_fast()) {
        if (!K.has_pi()) slice_epilogue_fast<NT, TM, true, ROLL, 0, LC>(L, crot, acc, J0, J1, J2, Z, K);
        else if (K.nA < 2 && K.nB < 2) slice_epilogue_fast<NT, TM, true, ROLL, 1, LC>(L, crot, acc, J0, J1, J2, Z, K);
        else slice_epilogue_fast<NT, TM, true, ROLL, 2, LC>(L, crot, acc, J0, J1, J2, Z, K);
    } else if constexpr (TM) {
        tmem_wait_st();
#pragma unroll 1
        for (int ch = 0; ch < 4; ++ch) {
            uint32_t v[32];
            tmem_ld32(acc.taddr + 32u * ch, v);
            tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const double2 d = slice_value_slow<NT, LC>(L, crot, J0, J1, J2, Z, K, 8 * ch + q);
                double2 o = v2d(v + 4 * q);
                o.x += d.x;
                o.y += d.y;
                d2v(o, v + 4 * q);
            }
            tmem_st32(acc.taddr + 32u * ch, v);
        }
    } else {
        uint32_t alive = ~Z;
        while (alive) {
            const int g = __ffs(alive) - 1;
            alive &= alive - 1;
            const double2 d = slice_value_slow<NT, LC>(L, crot, J0, J1, J2, Z, K, g);
            double2* ap = acc.amp_s + g * NT + threadIdx.x;
            double2 o = *ap;
            o.x += d.x;
            o.y += d.y;
            *ap = o;
        }
    }
    J0 = J1 = J2 = Z = 0;
    if (kinds) K.reset();
}

// Debug hook (LaunchReq::d_dbg5): the kernel's own per-term state for each of
// the thread's 32 assignments, read from the bit planes exactly as the
// epilogue sees them (before the 6 s1 fold into J). `term` = index of the
// term whose end row was just consumed. Sorted batches map the slot back to
// the caller's position (padding slots are skipped).
template <int NT, bool LC>
__device__ __noinline__ void debug_dump_codes(const LaunchReq& r, uint64_t term, uint64_t off, uint32_t J0,
                                              uint32_t J1, uint32_t J2, uint32_t Z, KindCounters<NT, LC>& K) {
    if (term < r.dbg_t0 || term >= r.dbg_t1) return;
    for (int g = 0; g < 32; ++g) {
        uint64_t idx = off + uint64_t(g);
        if (idx >= r.n) break;
        if (r.d_perm) {
            idx = r.d_perm[idx];
            if (idx == 0xFFFFFFFFu) continue;
        }
        if (idx >= r.dbg_n) continue;
        uint32_t* o = r.d_dbg5 + ((term - r.dbg_t0) * r.dbg_n + idx) * 5;
        o[0] = ((J0 >> g) & 1u) | (((J1 >> g) & 1u) << 1) | (((J2 >> g) & 1u) << 2);
        o[1] = (Z >> g) & 1u;
        o[2] = K.s_of(g);
        o[3] = K.a_of(g);
        o[4] = K.b_of(g);
    }
}

template <int NT, bool TM, bool ROLL = false, bool LC = false>
__device__ __forceinline__ void slice_term_epilogue(TermC& tc, const double2* src, const SmemLut& L, double2* crot,
                                                    SliceAcc<NT, TM>& acc, uint32_t& J0, uint32_t& J1,
                                                    uint32_t& J2, uint32_t& Z, KindCounters<NT, LC>& K) {
    slice_epilogue_begin(tc, src, L, crot);
    slice_epilogue_apply<NT, TM, ROLL, LC>(L, crot, acc, J0, J1, J2, Z, K);
}


// Random batches: the thread's 32 words are transposed into bit planes
// (plane i, bit g = bit i of word g) kept in shared memory [i][thread].
template <bool P64, bool RAND, int NT, bool TM = false>
size_t slice_smem_bytes(const DevTable& t) {
    const uint32_t amp_off = (slice_lut_offset<P64>() + t.lut_layout.bytes + 127u) & ~127u;
    const size_t planes = RAND ? size_t(P64 ? 64 : 32) * NT * 4 : 0;
    const size_t b = amp_off + (TM ? 0 : size_t(kSliceG) * NT * 16) + (NT / 32) * kWarpScratch * 16 + planes +
                     size_t(kHiPlanes) * NT * 4;
    return TM ? (b > kTmemCtaSmem ? b : kTmemCtaSmem) : b;
}

template <int NT, bool TM, bool FREE = true>
__device__ __forceinline__ void slice_store_results(const LaunchReq& r, uint64_t off, SliceAcc<NT, TM>& acc) {
    constexpr uint32_t kCols = NT > 128 ? 2 * kTmemCols : kTmemCols;
    if constexpr (TM) {
        tmem_wait_st();
#pragma unroll 1
        for (int ch = 0; ch < 4; ++ch) {
            uint32_t v[32];
            tmem_ld32(acc.taddr + 32u * ch, v);
            tmem_wait_ld();
#pragma unroll
            for (int q = 0; q < 8; ++q) store_result(r, off + 8 * ch + q, v2d(v + 4 * q));
        }
        if constexpr (FREE) tmem_free_cta<kCols>(tmem_base_of(acc.taddr) - (threadIdx.x >> 7) * kTmemCols);
    } else {
#pragma unroll 4
        for (int g = 0; g < kSliceG; ++g) store_result(r, off + g, acc.amp_s[g * NT + threadIdx.x]);
    }
}

// 32 x 32 bit-matrix transpose: afterwards a[i] bit g = (old a[g]) bit i.
__device__ __forceinline__ void transpose32(uint32_t (&a)[32]) {
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
        const uint32_t m = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu
                         : j == 2  ? 0x33333333u : 0x55555555u;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            if ((k & j) == 0) {
                const uint32_t tt = ((a[k] >> j) ^ a[k + j]) & m;
                a[k + j] ^= tt;
                a[k] ^= tt << j;
            }
        }
    }
}

// X = XOR of the planes of the parameters set in mask (uniform loop over set bits)
template <int NT>
__device__ __forceinline__ uint32_t planes_parity(uint32_t mask, uint32_t plane_addr) {
    uint32_t x = 0;
    while (mask) {
        const int i = __ffs(mask) - 1;
        mask &= mask - 1;
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(plane_addr + uint32_t(i) * (NT * 4)));
        x ^= v;
    }
    return x;
}

// Bit-sliced evaluation of enumerated / contiguous batches.
// A thread owns 32 assignments base + g (base % 32 == 0); register bit g of
// every accumulator belongs to assignment g:
//   J2 J1 J0 : sum of phase exponents mod 8      Z : some factor was zero
//   S / A / B: lambda / pi / pi' counts (bit-sliced, 7 planes)
// Per row: X = Walsh32(psi) ^ -parity(psi & base) in C++, then ONE generated
// inline-PTX block (pzx_slice_dispatch.inc) jumps (BRX) to the row class's
// LOP3 chain, which also forms Y for two-parity rows. Per term: the phase
// table C * w^j (8 entries) is built once per warp, then every live
// assignment adds C * w^j' * (stuff from S, A, B) into its fp64 accumulator in
// shared memory.
template <bool P64, bool RAND, int NT, bool TM = false, bool DBG = false>
__global__ void __launch_bounds__(NT, TM ? 4 : 1) k_eval_slice(const DevTable t, const LaunchReq r) {
    static_assert(!TM || NT == 128, "TMEM accumulators: one warp per TMEM lane quarter");
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint32_t tmem_base_s;
    const SmemLut L = kernel_prologue(t, smem, slice_lut_offset<P64>());
    const uint32_t amp_off = (slice_lut_offset<P64>() + t.lut_layout.bytes + 127u) & ~127u;
    double2* amp_s = reinterpret_cast<double2*>(smem + amp_off);
    double2* crot = amp_s + (TM ? 0 : kSliceG * NT) + (threadIdx.x >> 5) * kWarpScratch;
    uint32_t* hi_planes = reinterpret_cast<uint32_t*>(amp_s + (TM ? 0 : kSliceG * NT) + (NT / 32) * kWarpScratch) +
                          (RAND ? (P64 ? 64 : 32) * NT : 0);
    SliceAcc<NT, TM> acc{amp_s, 0u};
    if constexpr (TM) acc.taddr = tmem_alloc_cta(&tmem_base_s);
    acc.zero();

    uint64_t tb, te;
    term_range(r, tb, te);
    const uint64_t off = (uint64_t(blockIdx.x) * NT + threadIdx.x) * kSliceG;
    uint64_t base = 0;
    uint32_t planes_s = 0;  // shared address of this thread's plane 0 (RAND)
    if constexpr (RAND) {
        // thread owns the 32 arbitrary words off .. off+31: transpose into planes
        uint32_t* planes = reinterpret_cast<uint32_t*>(crot + (NT / 32 - (threadIdx.x >> 5)) * kWarpScratch);
        planes_s = smem_u32(planes) + threadIdx.x * 4;
        uint32_t w[32];
#pragma unroll
        for (int h = 0; h < (P64 ? 2 : 1); ++h) {
#pragma unroll
            for (int g = 0; g < 32; ++g) {
                const uint64_t idx = off + g;
                const uint64_t word = idx < r.n ? (r.d_asg ? r.d_asg[idx] : r.first + idx) : 0;
                w[g] = uint32_t(word >> (32 * h));
            }
            transpose32(w);
#pragma unroll
            for (int i = 0; i < 32; ++i) planes[(32 * h + i) * NT + threadIdx.x] = w[i];
        }
    } else {
        base = r.d_asg ? (off < r.n ? r.d_asg[off] : 0) : r.first + off;
    }
    const uint32_t blo = uint32_t(base), bhi = uint32_t(base >> 32);

    uint32_t J0 = 0, J1 = 0, J2 = 0, Z = 0;
    KindCounters<NT> K;
    K.init(hi_planes + threadIdx.x);

    if (tb < te) {
        uint4* tiles = reinterpret_cast<uint4*>(smem);
        uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kSliceTile * 32);
        const uint32_t tiles_s = smem_u32(tiles);
        const uint64_t R0 = t.term_row[tb], R1 = t.term_row[te];
        const uint32_t ntiles = uint32_t((R1 - R0 + kSliceTile - 1) / kSliceTile);
        auto issue = [&](uint32_t tile) {
            const uint64_t rr = R0 + uint64_t(tile) * kSliceTile;
            const uint64_t n = (R1 - rr) < uint64_t(kSliceTile) ? (R1 - rr) : uint64_t(kSliceTile);
            const uint32_t bytes = uint32_t(n) * 32u;
            uint64_t* bar = &bars[tile & 1];
            mbar_expect_tx(bar, bytes);
            tma_load_1d(tiles + (tile & 1) * kSliceTile * 2, t.srows + rr * 2, bytes, bar);
        };
        if (threadIdx.x == 0) {
            if (ntiles > 0) issue(0);
            if (ntiles > 1) issue(1);
        }
        TermC tc;
        termc_init(tc, crot + kCrot, t.sterm_c, tb, te);
        for (uint32_t i = 0; i < ntiles; ++i) {
            mbar_wait(&bars[i & 1], (i >> 1) & 1u);
            const uint64_t rem = R1 - R0 - uint64_t(i) * kSliceTile;
            const uint32_t n = rem < uint64_t(kSliceTile) ? uint32_t(rem) : uint32_t(kSliceTile);
            const uint32_t a0 = tiles_s + (i & 1) * kSliceTile * 32;
            const uint32_t aend = a0 + n * 32;
            if constexpr (!RAND) {
                // fused row loop (generated PTX, pzx_slice_dispatch.inc): plain rows
                // never leave it; it returns after a flagged row or at the tile end.
                // Rows are prefetched one ahead into r[] (the read past the last
                // row stays inside the CTA's shared window and is never used).
                uint4 ra = lds128(a0), rb = lds128(a0 + 16);
                uint32_t ad = a0;
                while (ad < aend) {
                    uint32_t vl, vpi, vpip, code;
                    if constexpr (P64) {
                        asm volatile(PZX_SLICE_ROWLOOP_P64
                                     : "+r"(ad), "+r"(J0), "+r"(J1), "+r"(J2), "+r"(Z), "=r"(vl), "=r"(vpi),
                                       "=r"(vpip), "=r"(code), "+r"(ra.x), "+r"(ra.y), "+r"(ra.z), "+r"(ra.w),
                                       "+r"(rb.x), "+r"(rb.y), "+r"(rb.z), "+r"(rb.w)
                                     : "r"(aend), "r"(blo), "r"(bhi)
                                     : "memory");
                    } else {
                        asm volatile(PZX_SLICE_ROWLOOP_P32
                                     : "+r"(ad), "+r"(J0), "+r"(J1), "+r"(J2), "+r"(Z), "=r"(vl), "=r"(vpi),
                                       "=r"(vpip), "=r"(code), "+r"(ra.x), "+r"(ra.y), "+r"(ra.z), "+r"(ra.w),
                                       "+r"(rb.x), "+r"(rb.y), "+r"(rb.z), "+r"(rb.w)
                                     : "r"(aend), "r"(blo), "r"(bhi)
                                     : "memory");
                    }
                    if (code & (kSliceLamFlag | kSlicePiFlag | kSlicePipFlag | kEndFlag)) {
                        if (code & kSliceLamFlag) K.bump_s(vl);
                        if (code & kSlicePiFlag) K.bump_a(vpi);
                        if (code & kSlicePipFlag) K.bump_b(vpip);
                        if (code & kEndFlag) {
                            if constexpr (DBG) debug_dump_codes<NT, false>(r, tc.next - 2, off, J0, J1, J2, Z, K);
                            slice_term_epilogue<NT, TM, TM>(tc, t.sterm_c, L, crot, acc, J0, J1, J2, Z, K);
                        }
                    }
                }
            } else {
            // rows software-pipelined one ahead (the read past the last row
                // stays inside the CTA's shared window and is never used). Both
                // parity vectors are formed before the jump, so nothing of the
                // current row is live across it and the next row's loads need no
                // register copies.
                uint4 na = lds128(a0), nb = lds128(a0 + 16);
                for (uint32_t ad = a0; ad < aend; ad += 32) {
                    const uint32_t code = na.z;  // op | kind flags | end
                    const uint32_t op = nb.w;    // jump-table index (the op again, own word: no masking)
                    uint32_t X = planes_parity<NT>(na.x, planes_s);
                    uint32_t Y = na.y ? planes_parity<NT>(na.y, planes_s) : 0u;
                    if constexpr (P64) {
                        X ^= planes_parity<NT>(nb.y, planes_s + 32 * NT * 4);
                        if (nb.z) Y ^= planes_parity<NT>(nb.z, planes_s + 32 * NT * 4);
                    }
                    na = lds128(ad + 32);
                    nb = lds128(ad + 48);
                    uint32_t vl, vpi, vpip;  // written only by rows whose kind flags are set
                    asm(PZX_SLICE_DISPATCH_ASM_XY
                        : "+r"(J0), "+r"(J1), "+r"(J2), "+r"(Z), "=r"(vl), "=r"(vpi), "=r"(vpip)
                        : "r"(X), "r"(op), "r"(Y));
                    if (code & (kSliceLamFlag | kSlicePiFlag | kSlicePipFlag | kEndFlag)) {
                        if (code & kSliceLamFlag) K.bump_s(vl);
                        if (code & kSlicePiFlag) K.bump_a(vpi);
                        if (code & kSlicePipFlag) K.bump_b(vpip);
                        if (code & kEndFlag) {
                            if constexpr (DBG) debug_dump_codes<NT, false>(r, tc.next - 2, off, J0, J1, J2, Z, K);
                            slice_term_epilogue<NT, TM>(tc, t.sterm_c, L, crot, acc, J0, J1, J2, Z, K);
                        }
                    }
                }
            }
            __syncthreads();  // every thread is done with buffer (i & 1)
            if (threadIdx.x == 0 && i + 2 < ntiles) {
                fence_proxy_async();
                issue(i + 2);
            }
        }
    }
    slice_store_results<NT, TM>(r, off, acc);
}

// ------------------------------------------------- warp-chunk kernel ----
// Small enumerated batches (a few thousand assignments, e.g. C4's 2^10
// marginal parameters against 2e8 rows): all 4 warps of a CTA own the SAME
// 32 x 32 assignments and walk 4 different term chunks (chunk = 4 blockIdx.y
// + warp), each with its own TMA row pipeline, so the CTA keeps 128 threads
// with TMEM accumulators (16 warps / SM) instead of 1-warp CTAs with shared-
// memory accumulators. Every warp's partial amplitudes go to its own chunk
// slot; the fixed-order chunk reduction sums them.
constexpr int kWarpChunks = kSliceThreads / 32;
constexpr int kWcTile = 128;  // rows per per-warp TMA tile (the row streams come from HBM)
static_assert(kWarpChunks == kWarpChunksHost, "warp-chunk count shared with the host");

template <bool P64>
__host__ __device__ constexpr uint32_t slicewc_lut_offset() {
    return kWarpChunks * 2 * kWcTile * 32 + kWarpChunks * 16 + 16;
}

template <bool P64>
size_t slicewc_smem_bytes(const DevTable& t) {
    const uint32_t amp_off = (slicewc_lut_offset<P64>() + t.lut_layout.bytes + 127u) & ~127u;
    const size_t b = amp_off + (kSliceThreads / 32) * kWarpScratch * 16 + size_t(kHiPlanes) * kSliceThreads * 4;
    return b > kTmemCtaSmem ? b : kTmemCtaSmem;
}

template <bool P64, bool DBG = false>
__global__ void __launch_bounds__(kSliceThreads, 4) k_eval_slice_wc(const DevTable t, const LaunchReq r) {
    constexpr int NT = kSliceThreads;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint32_t tmem_base_s;
    // the warp index through a lane-0 shuffle: provably warp-uniform, so the
    // row loop's branches stay uniform (no divergence bookkeeping)
    const uint32_t warp = __shfl_sync(0xFFFFFFFFu, threadIdx.x >> 5, 0), lane = threadIdx.x & 31u;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kWarpChunks * 2 * kWcTile * 32) + 2 * warp;
    if (lane == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    const SmemLut L = stage_lut(t, smem + slicewc_lut_offset<P64>());
    __syncthreads();
    const uint32_t amp_off = (slicewc_lut_offset<P64>() + t.lut_layout.bytes + 127u) & ~127u;
    double2* crot = reinterpret_cast<double2*>(smem + amp_off) + warp * kWarpScratch;
    uint32_t* hi_planes = reinterpret_cast<uint32_t*>(smem + amp_off + (NT / 32) * kWarpScratch * 16);
    SliceAcc<NT, true> acc{nullptr, 0u};
    acc.taddr = tmem_alloc_cta(&tmem_base_s);
    acc.zero();

    const uint32_t chunk = blockIdx.y * kWarpChunks + warp;
    const uint64_t tb = r.d_chunk_terms[chunk], te = r.d_chunk_terms[chunk + 1];
    const uint64_t off = (uint64_t(blockIdx.x) * 32 + lane) * kSliceG;
    const uint64_t base = r.d_asg ? (off < r.n ? r.d_asg[off] : 0) : r.first + off;
    const uint32_t blo = uint32_t(base), bhi = uint32_t(base >> 32);

    uint32_t J0 = 0, J1 = 0, J2 = 0, Z = 0;
    KindCounters<NT> K;
    K.init(hi_planes + threadIdx.x);

    if (tb < te) {
        uint4* tiles = reinterpret_cast<uint4*>(smem) + warp * (2 * kWcTile * 2);
        const uint32_t tiles_s = smem_u32(tiles);
        const uint64_t R0 = t.term_row[tb], R1 = t.term_row[te];
        const uint32_t ntiles = uint32_t((R1 - R0 + kWcTile - 1) / kWcTile);
        auto issue = [&](uint32_t tile) {
            const uint64_t rr = R0 + uint64_t(tile) * kWcTile;
            const uint64_t n = (R1 - rr) < uint64_t(kWcTile) ? (R1 - rr) : uint64_t(kWcTile);
            const uint32_t bytes = uint32_t(n) * 32u;
            uint64_t* bar = &bars[tile & 1];
            mbar_expect_tx(bar, bytes);
            tma_load_1d(tiles + (tile & 1) * kWcTile * 2, t.srows + rr * 2, bytes, bar);
        };
        if (lane == 0) {
            if (ntiles > 0) issue(0);
            if (ntiles > 1) issue(1);
        }
        TermC tc;
        termc_init(tc, crot + kCrot, t.sterm_c, tb, te);
        for (uint32_t i = 0; i < ntiles; ++i) {
            mbar_wait(&bars[i & 1], (i >> 1) & 1u);
            const uint64_t rem = R1 - R0 - uint64_t(i) * kWcTile;
            const uint32_t n = rem < uint64_t(kWcTile) ? uint32_t(rem) : uint32_t(kWcTile);
            const uint32_t a0 = tiles_s + (i & 1) * kWcTile * 32;
            const uint32_t aend = a0 + n * 32;
            uint4 ra = lds128(a0), rb = lds128(a0 + 16);
            uint32_t ad = a0;
            while (ad < aend) {
                uint32_t vl, vpi, vpip, code;
                if constexpr (P64) {
                    asm volatile(PZX_SLICE_ROWLOOP_P64
                                 : "+r"(ad), "+r"(J0), "+r"(J1), "+r"(J2), "+r"(Z), "=r"(vl), "=r"(vpi), "=r"(vpip),
                                   "=r"(code), "+r"(ra.x), "+r"(ra.y), "+r"(ra.z), "+r"(ra.w), "+r"(rb.x),
                                   "+r"(rb.y), "+r"(rb.z), "+r"(rb.w)
                                 : "r"(aend), "r"(blo), "r"(bhi)
                                 : "memory");
                } else {
                    asm volatile(PZX_SLICE_ROWLOOP_P32
                                 : "+r"(ad), "+r"(J0), "+r"(J1), "+r"(J2), "+r"(Z), "=r"(vl), "=r"(vpi), "=r"(vpip),
                                   "=r"(code), "+r"(ra.x), "+r"(ra.y), "+r"(ra.z), "+r"(ra.w), "+r"(rb.x),
                                   "+r"(rb.y), "+r"(rb.z), "+r"(rb.w)
                                 : "r"(aend), "r"(blo), "r"(bhi)
                                 : "memory");
                }
                if (code & (kSliceLamFlag | kSlicePiFlag | kSlicePipFlag | kEndFlag)) {
                    if (code & kSliceLamFlag) K.bump_s(vl);
                    if (code & kSlicePiFlag) K.bump_a(vpi);
                    if (code & kSlicePipFlag) K.bump_b(vpip);
                    if (code & kEndFlag) {
                        if constexpr (DBG) debug_dump_codes<NT, false>(r, tc.next - 2, off, J0, J1, J2, Z, K);
                        slice_term_epilogue<NT, true, true>(tc, t.sterm_c, L, crot, acc, J0, J1, J2, Z, K);
                    }
                }
            }
            __syncwarp();  // the warp is done with buffer (i & 1)
            if (lane == 0 && i + 2 < ntiles) {
                fence_proxy_async();
                issue(i + 2);
            }
        }
    }
    // this warp's partial amplitudes -> chunk slot `chunk`
    tmem_wait_st();
#pragma unroll 1
    for (int ch = 0; ch < 4; ++ch) {
        uint32_t v[32];
        tmem_ld32(acc.taddr + 32u * ch, v);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint64_t idx = off + 8 * ch + q;
            if (idx < r.n) r.d_partial[uint64_t(chunk) * r.n + idx] = v2d(v + 4 * q);
        }
    }
    tmem_free_cta(tmem_base_of(acc.taddr));
}

// ---------------------------------------------------------- page kernel ----
// Enumerated batches (all 2^P amplitudes, contiguous sweeps; n_params <= 32) on
// the PAGE layout (pzx_host.cpp, page_term): pages of
// kPageSlots 32-byte records, terms never straddling a page, each term a
// header (its constant) + constraint (C), generic (G, by update class), lambda
// (L) and dispatch (D) rows. A thread owns 32 assignments (bit-sliced as in
// k_eval_slice), a warp 1024 consecutive ones, base_w + 32 lane + g. Per page,
// a pre-pass (split over the CTA's warps) resolves the parity of every row mask
// against each warp's high bits ONCE per row and warp into a lane word
//   M = LW(mask bits 5..9) ^ -parity(mask & base_w)     (bit l: lane l's parity)
// so the row loops form X = parity ? ~W : W with a predicate test of M and a
// SEL -- no per-thread POPC. Per row and warp:
//   C: Z |= X                                            (6 instructions)
//   G: J += (k + 4p)q~, one loop per update class        (~5.5-12, no jump)
//   L: J += k p (k in {0, 4}), S += p ^ inv               (~13, no jump)
//   D: the generated class body through the jump table   (the slice kernel's)
// After a term's C rows a warp whose 1024 assignments are all zero skips the
// rest of the term (constraint-first order, PAPER "Conclusions"). Epilogues:
// pi terms through the warp's T[j, a, b] table (page_epilogue_pi), lambda-only
// terms through crot[j] * uz (page_epilogue_lam), the rest slice_epilogue_apply.
// Knobs (A/B builds): -DPZX_PI_TAB=0, -DPZX_CTA_PREPASS=0.
__host__ __device__ constexpr uint32_t page_lut_offset() { return 2 * kPageSlots * 32 + 16; }

// Page-kernel epilogue of a term with pi / pi' rows (fast counters): the warp
// has built T[pi_tab_index(j, a, b)] = C w^j pi^a pi'^b for the term, so each
// assignment reads ONE complex entry and one real (sqrt2-1)^s (uz, zero for
// Z-marked assignments) -- 2 DFMA -- instead of C w^j and (sqrt2-1)^s pi^a pi'^b
// (two complex lookups, 4 DFMA; slice_epilogue_tr KIND 2). Index bytes from
// two byte-lane transposes: {J0^A0, J1^A1, J2^B0, A0, A1, B0, B1} (dead
// assignments masked to entry 0, which the live (j, a, b) = 0 lanes of its bank
// group share) and {S0..S3, Z} at bits 3..7 (= the uz byte offset, no LEA).
template <int NT, bool LC>
__device__ __forceinline__ void page_epilogue_pi(const SmemLut& L, uint32_t tab_s, SliceAcc<NT, true>& acc,
                                                 uint32_t J0, uint32_t J1, uint32_t J2, uint32_t Z,
                                                 const KindCounters<NT, LC>& K) {
    // dead assignments read T[0, 0, 0] (the entry most live lanes of its bank group read)
    const uint32_t A0 = K.A[0] & ~Z, A1 = K.A[1] & ~Z, B0 = K.B[0] & ~Z, B1 = K.B[1] & ~Z;
    uint32_t R[8] = {(J0 & ~Z) ^ A0, (J1 & ~Z) ^ A1, (J2 & ~Z) ^ B0, A0, A1, B0, B1, 0u};
    transpose8_bytes(R);
    // dead assignments: s = 15 | 16 -> uz[31] = 0, off the banks of the common small s
    uint32_t Q[8] = {0u, 0u, 0u, K.S[0] | Z, K.S[1] | Z, K.S[2] | Z, K.S[3] | Z, Z};
    transpose8_bytes(Q);
    const uint32_t uz_s = smem_u32(L.uz);
    tmem_wait_st();
#pragma unroll 1
    for (int m = 0; m < 4; ++m) {
        const uint32_t sel = 0x4440u | uint32_t(m);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint32_t v[16];
            tmem_ld16(acc.taddr + 16u * uint32_t(2 * m + h), v);
            double2 c[4];
            double f[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                c[r] = lds_d2(tab_s + (__byte_perm(R[4 * h + r], 0u, sel) << 4));
                f[r] = lds_d(uz_s + __byte_perm(Q[4 * h + r], 0u, sel));
            }
            tmem_wait_ld();
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                double2 o = v2d(v + 4 * r);
                o.x = fma(c[r].x, f[r], o.x);
                o.y = fma(c[r].y, f[r], o.y);
                d2v(o, v + 4 * r);
            }
            tmem_st16(acc.taddr + 16u * uint32_t(2 * m + h), v);
        }
    }
}

__device__ __forceinline__ uint2 lds64(uint32_t addr) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}

// (J2 J1 J0) += Y & K0 + 2 (Y & K1) + 4 (Y & X)  mod 8, bit-sliced: 7 LOP3
__device__ __forceinline__ void g_row(uint32_t& J0, uint32_t& J1, uint32_t& J2, uint32_t X, uint32_t Y, uint32_t K0,
                                      uint32_t K1) {
    asm("{\n"
        ".reg .b32 c0, v1, c1, v2;\n"
        "lop3.b32 c0, %0, %3, %5, 0x80;\n"   // J0 & Y & K0
        "lop3.b32 %0, %0, %3, %5, 0x78;\n"   // J0 ^ (Y & K0)
        "and.b32 v1, %3, %6;\n"               // Y & K1
        "lop3.b32 c1, %1, v1, c0, 0xe8;\n"   // maj(J1, v1, c0)
        "lop3.b32 %1, %1, v1, c0, 0x96;\n"   // J1 ^ v1 ^ c0
        "and.b32 v2, %3, %4;\n"               // Y & X
        "lop3.b32 %2, %2, v2, c1, 0x96;\n"   // J2 ^ v2 ^ c1
        "}\n"
        : "+r"(J0), "+r"(J1), "+r"(J2)
        : "r"(Y), "r"(X), "r"(K0), "r"(K1));
}

// (J2 J1 J0) += (H2 H1 H0) mod 8
__device__ __forceinline__ void add3(uint32_t& J0, uint32_t& J1, uint32_t& J2, uint32_t H0, uint32_t H1, uint32_t H2) {
    const uint32_t c0 = J0 & H0;
    J0 ^= H0;
    const uint32_t c1 = (J1 & H1) | (c0 & (J1 ^ H1));
    J1 ^= H1 ^ c0;
    J2 ^= H2 ^ c1;
}

// One class of G rows (records at shared address ra, lane words at rm; both
// advanced past the n rows), software-pipelined one pair ahead: the next
// pair's shared loads are in flight while this pair computes (two register
// sets alternate, no copies on the back edge; the read past the last pair stays
// inside the CTA's shared window and is never used). Per row, X / Y = the
// record's word or its complement by this lane's parity bit:
//   kGS : Y only;  J2 ^= Y & J1, J1 ^= Y                   (J += 2Y)
//   kGE0: J2 ^= X & Y                                       (J += 4XY)
//   kGE2: J2 ^= Y & (J1 ^ X), J1 ^= Y                       (J += 2Y + 4XY)
//   kG1 : J2 ^= (J1 & J0 & Y) ^ (X & Y), J1 ^= J0 & Y,
//         J0 ^= Y                                           (J += Y + 4XY, 5 LOP3)
//   kGG : g_row                                             (J += (k + 4X) Y, 7 LOP3)
constexpr int kGS = 0, kGE0 = 1, kGE2 = 2, kGG = 3, kG1 = 4;

template <int V>
struct GRow {
    uint4 a;
    uint2 b, m;
};

template <int V>
__device__ __forceinline__ void g_load(GRow<V>& r, uint32_t ra, uint32_t rm) {
    if constexpr (V == kGS) {
        const uint2 t = lds64(ra + 8);
        r.a.z = t.x;
        r.a.w = t.y;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r.m.y) : "r"(rm + 4));
    } else {
        r.a = lds128(ra);
        r.m = lds64(rm);
        if constexpr (V == kGG) r.b = lds64(ra + 16);
    }
}

template <int V>
__device__ __forceinline__ void g_apply(const GRow<V>& r, uint32_t lanebit, uint32_t& J0, uint32_t& J1,
                                        uint32_t& J2) {
    const uint32_t Y = (r.m.y & lanebit) ? r.a.w : r.a.z;
    if constexpr (V == kGS) {
        J2 ^= Y & J1;
        J1 ^= Y;
    } else {
        const uint32_t X = (r.m.x & lanebit) ? r.a.y : r.a.x;
        if constexpr (V == kGE0) {
            J2 ^= X & Y;
        } else if constexpr (V == kGE2) {
            J2 ^= Y & (J1 ^ X);
            J1 ^= Y;
        } else if constexpr (V == kG1) {
            J2 ^= (J1 & J0 & Y) ^ (X & Y);
            J1 ^= J0 & Y;
            J0 ^= Y;
        } else {
            g_row(J0, J1, J2, X, Y, r.b.x, r.b.y);
        }
    }
}

template <int V>
__device__ __forceinline__ void g_loop(uint32_t& ra, uint32_t& rm, uint32_t n, uint32_t lanebit, uint32_t& J0,
                                       uint32_t& J1, uint32_t& J2, uint32_t& H0, uint32_t& H1, uint32_t& H2) {
    const uint32_t e2 = ra + 32u * (n & ~1u);
    if (ra < e2) {
        GRow<V> P0[2], P1[2];
        g_load(P0[0], ra, rm);
        g_load(P0[1], ra + 32, rm + 8);
#pragma unroll 1
        for (;;) {
            g_load(P1[0], ra + 64, rm + 16);
            g_load(P1[1], ra + 96, rm + 24);
            g_apply(P0[0], lanebit, J0, J1, J2);
            g_apply(P0[1], lanebit, H0, H1, H2);
            ra += 64; rm += 16;
            if (ra >= e2) break;
            g_load(P0[0], ra + 64, rm + 16);
            g_load(P0[1], ra + 96, rm + 24);
            g_apply(P1[0], lanebit, J0, J1, J2);
            g_apply(P1[1], lanebit, H0, H1, H2);
            ra += 64; rm += 16;
            if (ra >= e2) break;
        }
    }
    if (n & 1u) {
        GRow<V> r;
        g_load(r, ra, rm);
        g_apply(r, lanebit, J0, J1, J2);
        ra += 32; rm += 8;
    }
}

// per-warp pi-term table T[j, a, b] = C w^j pi^a pi'^b (page_epilogue_pi)
constexpr int kPiTab = 128;
__host__ __device__ constexpr uint32_t pi_tab_index(uint32_t j, uint32_t a, uint32_t b) {
    return (j ^ (a | ((b & 1u) << 2))) | (a << 3) | (b << 5);
}

size_t page_smem_bytes(const DevTable& t) {
    const uint32_t amp_off = (page_lut_offset() + t.lut_layout.bytes + 127u) & ~127u;
    const size_t b = amp_off + 4 * kCrot * 16 + 4 * size_t(kPageSlots) * 8 + size_t(kHiPlanes) * kSliceThreads * 4;
    constexpr size_t floor = kTmemCtaSmem - 4 * size_t(kPiTab) * 16;  // + the static pi tables: <= 4 CTAs / SM
    return b > floor ? b : floor;
}

template <bool DBG = false>
__global__ void __launch_bounds__(kSliceThreads, 4) k_eval_page(const DevTable t, const LaunchReq r) {
    constexpr int NT = kSliceThreads;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint32_t tmem_base_s;
    __shared__ uint32_t lw_s[32];  // lw_s[v] bit l = parity(v & l): lane bits 5..9 of the assignment
    if (threadIdx.x < 32) {
        uint32_t w = 0;
        for (uint32_t l = 0; l < 32; ++l) w |= uint32_t(__popc(threadIdx.x & l) & 1) << l;
        lw_s[threadIdx.x] = w;
    }
    const SmemLut L = kernel_prologue(t, smem, page_lut_offset());  // (its __syncthreads covers lw_s)
    // the warp index through a lane-0 shuffle: provably warp-uniform (uniform
    // datapath addressing of the warp's lane words and crot table)
    const uint32_t warp = __shfl_sync(0xFFFFFFFFu, threadIdx.x >> 5, 0), lane = threadIdx.x & 31u;
    const uint32_t amp_off = (page_lut_offset() + t.lut_layout.bytes + 127u) & ~127u;
    double2* crot = reinterpret_cast<double2*>(smem + amp_off) + warp * kCrot;
    uint2* Mw = reinterpret_cast<uint2*>(smem + amp_off + 4 * kCrot * 16) + warp * kPageSlots;
    uint32_t* hi_planes = reinterpret_cast<uint32_t*>(smem + amp_off + 4 * kCrot * 16 + 4 * kPageSlots * 8);
    // the warp's pi-term table in STATIC shared memory: its address is a link-time
    // constant + warp * 2 KB, independent of the dynamic layout (a table addressed
    // from the dynamic base shares subexpressions with the row loops' addresses and
    // costs them their uniform-datapath addressing)
    __shared__ __align__(16) double2 pitab_all[4 * kPiTab];
    double2* pitab = pitab_all + warp * kPiTab;
    for (uint32_t i = lane; i < uint32_t(kPiTab); i += 32) pitab[i] = make_double2(0.0, 0.0);  // finite for dead lanes
    SliceAcc<NT, true> acc{nullptr, 0u};
    acc.taddr = tmem_alloc_cta(&tmem_base_s);
    acc.zero();

    uint64_t tb, te;
    term_range(r, tb, te);
    const uint64_t off = (uint64_t(blockIdx.x) * NT + threadIdx.x) * kSliceG;
    const uint32_t wbase = uint32_t(r.first + (uint64_t(blockIdx.x) * NT + warp * 32u) * kSliceG);
    const uint32_t lanebit = 1u << lane;
    uint32_t J0 = 0, J1 = 0, J2 = 0, Z = 0;
    KindCounters<NT> K;
    K.init(hi_planes + threadIdx.x);

    if (tb < te) {
        uint4* pages = reinterpret_cast<uint4*>(smem);
        uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kPageSlots * 32);
        const uint32_t s0 = t.term_slot[tb];
        const uint32_t p0 = s0 / uint32_t(kPageSlots), np = t.term_slot[te - 1] / uint32_t(kPageSlots) - p0 + 1;
        auto issue = [&](uint32_t i) {
            uint64_t* bar = &bars[i & 1];
            mbar_expect_tx(bar, kPageSlots * 32);
            tma_load_1d(pages + (i & 1) * kPageSlots * 2, t.prows + uint64_t(p0 + i) * kPageSlots * 2,
                        kPageSlots * 32, bar);
        };
        if (threadIdx.x == 0) {
            issue(0);
            if (np > 1) issue(1);
        }
        uint64_t term = tb;
        uint32_t s = s0 % uint32_t(kPageSlots);
        for (uint32_t i = 0; i < np; ++i) {
            mbar_wait(&bars[i & 1], (i >> 1) & 1u);
            const uint4* pg = pages + (i & 1) * kPageSlots * 2;
#if PZX_CTA_PREPASS
            // pre-pass, split over the CTA: warp w reads the masks of slots [64 w, 64 w + 64)
            // ONCE (their 8-byte reads at a 32-byte stride are 4-way bank-conflicted) and
            // writes the lane-parity words of all four warps
            {
                const uint32_t cbase = wbase - warp * 1024u;  // the CTA's first assignment
                uint2* M0 = Mw - warp * uint32_t(kPageSlots);
#pragma unroll
                for (uint32_t k = 0; k < 2; ++k) {
                    const uint32_t q = warp * 64u + lane + 32u * k;
                    const uint4 rec = pg[2 * q + 1];
                    const uint32_t lx = lw_s[(rec.z >> 5) & 31u], ly = lw_s[(rec.w >> 5) & 31u];
#pragma unroll
                    for (uint32_t w = 0; w < 4; ++w) {
                        const uint32_t b = cbase + w * 1024u;
                        M0[w * kPageSlots + q] = make_uint2(lx ^ (0u - (uint32_t(__popc(rec.z & b)) & 1u)),
                                                            ly ^ (0u - (uint32_t(__popc(rec.w & b)) & 1u)));
                    }
                }
            }
            __syncthreads();
#else
            // pre-pass: this warp's lane-parity words of every slot of the page
#pragma unroll 4
            for (uint32_t q = lane; q < uint32_t(kPageSlots); q += 32) {
                const uint4 rec = pg[2 * q + 1];
                const uint32_t mx = lw_s[(rec.z >> 5) & 31u] ^ (0u - (uint32_t(__popc(rec.z & wbase)) & 1u));
                const uint32_t my = lw_s[(rec.w >> 5) & 31u] ^ (0u - (uint32_t(__popc(rec.w & wbase)) & 1u));
                Mw[q] = make_uint2(mx, my);
            }
            __syncwarp();
#endif
            while (term < te) {
                const uint4 h0 = pg[2 * s], h1 = pg[2 * s + 1];
                const uint32_t nc = h1.x & 0xFFu, ng = (h1.x >> 8) & 0xFFu, nd = (h1.x >> 16) & 0xFFu;
                const uint32_t nl0 = h1.y & 0xFFu, nl4 = h1.y >> 8, nl = nl0 + nl4;
                uint32_t q = s + 1;
                // C rows: parity constraints
                for (const uint32_t e = q + nc; q < e; ++q) {
                    const uint4 a = pg[2 * q];
                    Z |= (Mw[q].x & lanebit) ? a.y : a.x;
                }
                const bool dead = nc != 0 && __all_sync(0xFFFFFFFFu, Z == 0xFFFFFFFFu);
                if (dead) {
                    q += ng + nl + nd + (h1.z & 0xFFu) + ((h1.z >> 8) & 0xFFu) + ((h1.z >> 16) & 0xFFu) + (h1.z >> 24) +
                         h1.w;
                } else {
                    // G rows, by update class (page_term): S2 / S6 (single parity, J += 2q / 6q),
                    // E0 (J2 ^= X & Y), E2 (J += 2Y + 4XY), G1 / G3 (J += Y / 3Y + 4XY). Pairs of
                    // rows go to two counters (J, H) so consecutive rows do not wait on each
                    // other's carries; H is added into J once, after the G rows.
                    {
                        uint32_t H0 = 0, H1 = 0, H2 = 0;
                        uint32_t ra = smem_u32(pg + 2 * q), rm = smem_u32(Mw + q);
                        const uint32_t ns2 = h1.z & 0xFFu, ns6 = (h1.z >> 8) & 0xFFu, ne0 = (h1.z >> 16) & 0xFFu,
                                       ne2 = h1.z >> 24;
                        g_loop<kGS>(ra, rm, ns2, lanebit, J0, J1, J2, H0, H1, H2);
                        if (ns6) {  // J += 6q: the S update on ~J1
                            J1 = ~J1; H1 = ~H1;
                            g_loop<kGS>(ra, rm, ns6, lanebit, J0, J1, J2, H0, H1, H2);
                            J1 = ~J1; H1 = ~H1;
                        }
                        g_loop<kGE0>(ra, rm, ne0, lanebit, J0, J1, J2, H0, H1, H2);
                        g_loop<kGE2>(ra, rm, ne2, lanebit, J0, J1, J2, H0, H1, H2);
                        g_loop<kG1>(ra, rm, ng, lanebit, J0, J1, J2, H0, H1, H2);
                        if (h1.w) {  // J += 3Y + 4XY = ~(~J + Y + 4X'Y): the G1 update on ~J (X' stored)
                            J0 = ~J0; J1 = ~J1; J2 = ~J2; H0 = ~H0; H1 = ~H1; H2 = ~H2;
                            g_loop<kG1>(ra, rm, h1.w, lanebit, J0, J1, J2, H0, H1, H2);
                            J0 = ~J0; J1 = ~J1; J2 = ~J2; H0 = ~H0; H1 = ~H1; H2 = ~H2;
                        }
                        add3(J0, J1, J2, H0, H1, H2);
                        q += ns2 + ns6 + ne0 + ne2 + ng + h1.w;
                    }
                    // L rows (single-parity lambda / mu rows with k in {0, 4}; the host sends
                    // them here only when the term has < 16 lambda-capable rows, so S fits its
                    // 4 register planes): S += Lambda, Lambda = p ^ inv, and for L4 rows
                    // J2 ^= p -- both from the x parity word and one 16-byte record load
                    if (nl) {
                        auto lrow = [&](uint32_t qq, bool k4) {
                            const uint4 a = pg[2 * qq];
                            const bool px = Mw[qq].x & lanebit;
                            const uint32_t lam = px ? a.y : a.x;
                            if (k4) J2 ^= px ? a.w : a.z;
                            const uint32_t c0 = K.S[0] & lam;
                            K.S[0] ^= lam;
                            const uint32_t c1 = K.S[1] & c0;
                            K.S[1] ^= c0;
                            const uint32_t c2 = K.S[2] & c1;
                            K.S[2] ^= c1;
                            K.S[3] ^= c2;
                        };
#pragma unroll 2
                        for (const uint32_t e = q + nl0; q < e; ++q) lrow(q, false);
#pragma unroll 2
                        for (const uint32_t e = q + nl4; q < e; ++q) lrow(q, true);
                        K.nS = nl;
                    }
                    // D rows: the class bodies of the bit-sliced kernels (generated PTX)
                    for (const uint32_t e = q + nd; q < e; ++q) {
                        const uint4 a = pg[2 * q], b = pg[2 * q + 1];
                        const uint2 m = Mw[q];
                        const uint32_t X = (m.x & lanebit) ? a.y : a.x;
                        const uint32_t Y = (m.y & lanebit) ? a.w : a.z;
                        const uint32_t code = b.x, op = b.y;
                        uint32_t vl, vpi, vpip;
                        asm(PZX_SLICE_DISPATCH_ASM_XY
                            : "+r"(J0), "+r"(J1), "+r"(J2), "+r"(Z), "=r"(vl), "=r"(vpi), "=r"(vpip)
                            : "r"(X), "r"(op), "r"(Y));
                        if (code & (kSliceLamFlag | kSlicePiFlag | kSlicePipFlag)) {
                            if (code & kSliceLamFlag) K.bump_s(vl);
                            if (code & kSlicePiFlag) K.bump_a(vpi);
                            if (code & kSlicePipFlag) K.bump_b(vpip);
                        }
                    }
                }
                if constexpr (DBG) debug_dump_codes<NT, false>(r, term, off, J0, J1, J2, Z, K);
                if (!dead) {
                    __syncwarp();  // the previous term's epilogue is done with crot / pitab
                    const double2 C = make_double2(__hiloint2double(int(h0.y), int(h0.x)),
                                                   __hiloint2double(int(h0.w), int(h0.z)));
                    if (PZX_PI_TAB && K.has_pi() && K.fits_fast()) {
                        // T[j, a, b] = C w^j pi^a pi'^b for b <= nB: lane -> (j, a), one b per pass
                        // (every lane writes: the entries with a > nA are finite and never read
                        // by a live assignment)
                        const uint32_t j = lane & 7u, a = lane >> 3;
                        const double2 w = L.om[j];
                        const double2 cw = make_double2(C.x * w.x - C.y * w.y, C.x * w.y + C.y * w.x);
                        for (uint32_t b = 0; b <= K.nB; ++b) {
                            const double2 p = L.sab[(a | ((b & 1u) << 2)) | (a << 4) | (b << 6)];  // s = 0
                            pitab[pi_tab_index(j, a, b)] =
                                make_double2(cw.x * p.x - cw.y * p.y, cw.x * p.y + cw.y * p.x);
                        }
                        __syncwarp();
                        if (K.nS) {  // (lambda/mu)^s1 = mu^.. w^(6 s1) (sqrt2-1)^s1: J += 6 s1
                            const uint32_t w1 = K.S[0], w2 = K.S[0] ^ K.S[1];
                            const uint32_t c1 = J1 & w1;
                            J1 ^= w1;
                            J2 ^= w2 ^ c1;
                        }
                        page_epilogue_pi<NT, false>(L, smem_u32(pitab), acc, J0, J1, J2, Z, K);
                        J0 = J1 = J2 = Z = 0;
                        K.reset();
                    } else {
                        if (lane < uint32_t(kCrot)) {
                            double2 v = make_double2(0.0, 0.0);
                            if (lane < 8) {
                                const double2 w = L.om[lane];
                                v = make_double2(C.x * w.x - C.y * w.y, C.x * w.y + C.y * w.x);
                            }
                            crot[lane] = v;
                        }
                        __syncwarp();
                        if (PZX_PI_TAB && K.any() && K.fits_fast()) {  // lambda / mu rows only
                            const uint32_t w1 = K.S[0], w2 = K.S[0] ^ K.S[1];  // J += 6 s1
                            const uint32_t c1 = J1 & w1;
                            J1 ^= w1;
                            J2 ^= w2 ^ c1;
                            page_epilogue_lam<NT, false>(L, smem_u32(crot), acc, J0, J1, J2, Z, K);
                            J0 = J1 = J2 = Z = 0;
                            K.reset();
                        } else {
                            slice_epilogue_apply<NT, true, true>(L, crot, acc, J0, J1, J2, Z, K);
                        }
                    }
                } else {
                    J0 = J1 = J2 = Z = 0;
                    if (K.any()) K.reset();
                }
                ++term;
                s = q;
                if ((h1.x >> 24) & 1u) {  // last term of this page
                    s = 0;
                    break;
                }
            }
            __syncthreads();  // every warp is done with buffer (i & 1)
            if (threadIdx.x == 0 && i + 2 < np) {
                fence_proxy_async();
                issue(i + 2);
            }
        }
    }
    slice_store_results<NT, true>(r, off, acc);
}

// ---------------------------------------------------- two-slice kernel ----
// Enumerated batches, 64 assignments per thread: slice a = base + g, slice b
// = base + 32 + g (base % 64 == 0). Both slices share the row load, the
// parity POPCs (X_b = X_a ^ -(psi bit 5)), the jump and the flag tests, and
// the generated XY2 bodies run the two LOP3 chains interleaved (ILP 2), so the
// per-row overhead is paid once per 64 assignments. Accumulators: 256 TMEM
// columns per 128-thread CTA (2 CTAs = 8 warps per SM, each with twice the
// independent work of the one-slice kernel).
constexpr uint32_t kTmemCols2 = 256;
constexpr size_t kTmemCtaSmem2 = 80 * 1024;  // dynamic smem floor: at most 2 CTAs/SM (= 512 TMEM columns)

template <bool P64>
size_t slice2_smem_bytes(const DevTable& t) {
    const uint32_t amp_off = (slice_lut_offset<P64>() + t.lut_layout.bytes + 127u) & ~127u;
    const size_t b = amp_off + (kSliceThreads / 32) * kWarpScratch * 16 + 2 * size_t(kHiPlanes) * kSliceThreads * 4;
    return b > kTmemCtaSmem2 ? b : kTmemCtaSmem2;
}

template <bool P64>
__global__ void __launch_bounds__(kSliceThreads, 2) k_eval_slice2(const DevTable t, const LaunchReq r) {
    constexpr int NT = kSliceThreads;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint32_t tmem_base_s;
    const SmemLut L = kernel_prologue(t, smem, slice_lut_offset<P64>());
    const uint32_t amp_off = (slice_lut_offset<P64>() + t.lut_layout.bytes + 127u) & ~127u;
    double2* crot = reinterpret_cast<double2*>(smem + amp_off) + (threadIdx.x >> 5) * kWarpScratch;
    uint32_t* hi_planes = reinterpret_cast<uint32_t*>(smem + amp_off + (NT / 32) * kWarpScratch * 16);
    SliceAcc<NT, true> acc_a{nullptr, 0u}, acc_b{nullptr, 0u};
    acc_a.taddr = tmem_alloc_cta<kTmemCols2>(&tmem_base_s);
    acc_b.taddr = acc_a.taddr + kTmemCols;
    acc_a.zero();
    acc_b.zero();

    uint64_t tb, te;
    term_range(r, tb, te);
    const uint64_t off = (uint64_t(blockIdx.x) * NT + threadIdx.x) * (2 * kSliceG);
    const uint64_t base = r.d_asg ? (off < r.n ? r.d_asg[off] : 0) : r.first + off;
    const uint32_t blo = uint32_t(base), bhi = uint32_t(base >> 32);

    uint32_t Ja0 = 0, Ja1 = 0, Ja2 = 0, Za = 0, Jb0 = 0, Jb1 = 0, Jb2 = 0, Zb = 0;
    KindCounters<NT> Ka, Kb;
    Ka.init(hi_planes + threadIdx.x);
    Kb.init(hi_planes + kHiPlanes * NT + threadIdx.x);

    if (tb < te) {
        uint4* tiles = reinterpret_cast<uint4*>(smem);
        uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kSliceTile * 32);
        const uint32_t tiles_s = smem_u32(tiles);
        const uint64_t R0 = t.term_row[tb], R1 = t.term_row[te];
        const uint32_t ntiles = uint32_t((R1 - R0 + kSliceTile - 1) / kSliceTile);
        auto issue = [&](uint32_t tile) {
            const uint64_t rr = R0 + uint64_t(tile) * kSliceTile;
            const uint64_t n = (R1 - rr) < uint64_t(kSliceTile) ? (R1 - rr) : uint64_t(kSliceTile);
            const uint32_t bytes = uint32_t(n) * 32u;
            uint64_t* bar = &bars[tile & 1];
            mbar_expect_tx(bar, bytes);
            tma_load_1d(tiles + (tile & 1) * kSliceTile * 2, t.srows + rr * 2, bytes, bar);
        };
        if (threadIdx.x == 0) {
            if (ntiles > 0) issue(0);
            if (ntiles > 1) issue(1);
        }
        TermC tc;
        termc_init(tc, crot + kCrot, t.sterm_c, tb, te);
        for (uint32_t i = 0; i < ntiles; ++i) {
            mbar_wait(&bars[i & 1], (i >> 1) & 1u);
            const uint64_t rem = R1 - R0 - uint64_t(i) * kSliceTile;
            const uint32_t n = rem < uint64_t(kSliceTile) ? uint32_t(rem) : uint32_t(kSliceTile);
            const uint32_t a0 = tiles_s + (i & 1) * kSliceTile * 32;
            const uint32_t aend = a0 + n * 32;
            uint4 na = lds128(a0), nb = lds128(a0 + 16);
            for (uint32_t ad = a0; ad < aend; ad += 32) {
                const uint32_t code = na.z;
                const uint32_t op = nb.w;
                uint32_t px, py;
                if constexpr (P64) {
                    px = __popc((na.x & blo) ^ (nb.y & bhi));
                    py = __popc((na.y & blo) ^ (nb.z & bhi));
                } else {
                    px = __popc(na.x & blo);
                    py = __popc(na.y & blo);
                }
                const uint32_t m5x = 0u - ((na.x >> 5) & 1u), m5y = 0u - ((na.y >> 5) & 1u);
                const uint32_t Xa = na.w ^ (0u - (px & 1u)), Ya = nb.x ^ (0u - (py & 1u));
                const uint32_t Xb = Xa ^ m5x, Yb = Ya ^ m5y;
                na = lds128(ad + 32);
                nb = lds128(ad + 48);
                uint32_t vla, vpia, vpipa, vlb, vpib, vpipb;
                asm(PZX_SLICE_DISPATCH_ASM_XY2
                    : "+r"(Ja0), "+r"(Ja1), "+r"(Ja2), "+r"(Za), "+r"(Jb0), "+r"(Jb1), "+r"(Jb2), "+r"(Zb),
                      "=r"(vla), "=r"(vpia), "=r"(vpipa), "=r"(vlb), "=r"(vpib), "=r"(vpipb)
                    : "r"(Xa), "r"(Ya), "r"(Xb), "r"(Yb), "r"(op));
                if (code & (kSliceLamFlag | kSlicePiFlag | kSlicePipFlag | kEndFlag)) {
                    if (code & kSliceLamFlag) { Ka.bump_s(vla); Kb.bump_s(vlb); }
                    if (code & kSlicePiFlag) { Ka.bump_a(vpia); Kb.bump_a(vpib); }
                    if (code & kSlicePipFlag) { Ka.bump_b(vpipa); Kb.bump_b(vpipb); }
                    if (code & kEndFlag) {
                        slice_epilogue_begin(tc, t.sterm_c, L, crot);
                        slice_epilogue_apply<NT, true>(L, crot, acc_a, Ja0, Ja1, Ja2, Za, Ka);
                        slice_epilogue_apply<NT, true>(L, crot, acc_b, Jb0, Jb1, Jb2, Zb, Kb);
                    }
                }
            }
            __syncthreads();  // every thread is done with buffer (i & 1)
            if (threadIdx.x == 0 && i + 2 < ntiles) {
                fence_proxy_async();
                issue(i + 2);
            }
        }
    }
    slice_store_results<NT, true, false>(r, off, acc_a);
    slice_store_results<NT, true, false>(r, off + kSliceG, acc_b);
    tmem_free_cta<kTmemCols2>(tmem_base_of(acc_a.taddr));
}

// ------------------------------------------------------ sorted kernel ----
// Bit-sliced evaluation of an ARBITRARY word list after sorting it (host side
// sorts word|position pairs with cub and checks that every group of 32
// consecutive sorted words spans < 2^16). A thread owns 32 consecutive sorted
// words, so their high parts (bits >= 16) take at most two values H0, H0 + 1:
//   X = parity(psi & a_g) for g < 32
//     = XOR_k T_k[nibble_k(psi)]                 (parameters 0..4G-1: per-thread
//                                                  Four-Russians tables, G x 16 words)
//     ^ -parity(psi & H0)                          (the group's shared high part)
// with the tables built once per thread from its transposed low-bit planes.
// The rest (dispatch, counters, epilogue) is the slice kernel's.
// row tiles: 128 rows, 64 for the 256-thread wide-table variant (its 96 KB of
// tables must leave room for two CTAs per SM)
template <int NT = kSliceThreads>
__host__ __device__ constexpr int sorted_tile() {
    return NT > 128 ? 64 : 128;
}
template <int NT = kSliceThreads>
__host__ __device__ constexpr uint32_t sorted_lut_offset() {
    return 2 * sorted_tile<NT>() * 32 + 16;
}

template <bool TM = false, int G = kSortedGroups, int NT = kSliceThreads>
size_t sorted_smem_bytes(const DevTable& t) {
    const uint32_t amp_off = (sorted_lut_offset<NT>() + t.lut_layout.bytes + 127u) & ~127u;
    // (256-thread CTAs keep the rarely used high counter planes in local memory)
    const size_t b = amp_off + (TM ? 0 : size_t(kSliceG) * NT * 16) + (NT / 32) * kWarpScratch * 16 +
                     size_t(G) * 16 * NT * 4 + (NT > 128 ? 0 : size_t(kHiPlanes) * NT * 4);
    return TM ? (b > kTmemCtaSmem ? b : kTmemCtaSmem) : b;
}


template <bool TM = false, int G = kSortedGroups, int NT = kSliceThreads, bool DBG = false>
__global__ void __launch_bounds__(NT, TM ? (NT > 128 ? 2 : (G > 4 ? 3 : 4)) : 1) k_eval_sorted(const DevTable t,
                                                                                             const LaunchReq r) {
    static_assert(!TM || NT == 128 || NT == 256, "TMEM: 4 or 8 warps per CTA");
    constexpr int ST = sorted_tile<NT>();
    constexpr int kLow = 4 * G;  // parameters 0 .. kLow-1 through the per-thread tables
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint32_t tmem_base_s;
    const SmemLut L = kernel_prologue(t, smem, sorted_lut_offset<NT>());
    const uint32_t amp_off = (sorted_lut_offset<NT>() + t.lut_layout.bytes + 127u) & ~127u;
    double2* amp_s = reinterpret_cast<double2*>(smem + amp_off);
    double2* crot = amp_s + (TM ? 0 : kSliceG * NT) + (threadIdx.x >> 5) * kWarpScratch;
    uint32_t* tab = reinterpret_cast<uint32_t*>(amp_s + (TM ? 0 : kSliceG * NT) +
                                                (NT / 32) * kWarpScratch);
    uint32_t* hi_planes = tab + G * 16 * NT;
    SliceAcc<NT, TM> acc{amp_s, 0u};
    if constexpr (TM) acc.taddr = tmem_alloc_cta<(NT > 128 ? 2 * kTmemCols : kTmemCols)>(&tmem_base_s);
    acc.zero();

    uint64_t tb, te;
    term_range(r, tb, te);
    const uint64_t off = (uint64_t(blockIdx.x) * NT + threadIdx.x) * kSliceG;
    // ---- this thread's 32 sorted words -> planes -> Four-Russians tables ----
    uint32_t w[32];
#pragma unroll
    for (int g = 0; g < 32; ++g) {
        const uint64_t idx = off + g < r.n ? off + g : r.n - 1;  // pad with the last word (keeps order)
        w[g] = uint32_t(r.d_sorted[idx]);
    }
    // the host padded the sorted words into groups of 32 sharing one high part
    const uint32_t H0 = w[0] & ~((1u << kLow) - 1u);
    transpose32(w);  // w[i] = plane i (bit g = bit i of word g)
#pragma unroll
    for (int k = 0; k < G; ++k) {
        uint32_t e[16];
        e[0] = 0;
#pragma unroll
        for (int v = 1; v < 16; ++v) e[v] = e[v & (v - 1)] ^ w[4 * k + ((v & 1) ? 0 : (v & 2) ? 1 : (v & 4) ? 2 : 3)];
#pragma unroll
        for (int v = 0; v < 16; ++v) tab[(k * 16 + v) * NT + threadIdx.x] = e[v];
    }
    const uint32_t tab_s = smem_u32(tab) + threadIdx.x * 4;
    // per row (PZX_SORTED_ROWLOOP_G*): X = XOR_k T_k[nibble_k(psi)] ^ -parity(psi & H0)

    uint32_t J0 = 0, J1 = 0, J2 = 0, Z = 0;
    // 256-thread CTAs keep the rarely used high counter planes in local memory
    KindCounters<NT, (NT > 128)> K;
    uint32_t hi_local[NT > 128 ? kHiPlanes : 1];
    if constexpr (NT > 128) K.init(hi_local);
    else K.init(hi_planes + threadIdx.x);
    __syncwarp();

    if (tb < te) {
        uint4* tiles = reinterpret_cast<uint4*>(smem);
        uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * ST * 32);
        const uint32_t tiles_s = smem_u32(tiles);
        const uint64_t R0 = t.term_row[tb], R1 = t.term_row[te];
        const uint32_t ntiles = uint32_t((R1 - R0 + ST - 1) / ST);
        auto issue = [&](uint32_t tile) {
            const uint64_t rr = R0 + uint64_t(tile) * ST;
            const uint64_t n = (R1 - rr) < uint64_t(ST) ? (R1 - rr) : uint64_t(ST);
            const uint32_t bytes = uint32_t(n) * 32u;
            uint64_t* bar = &bars[tile & 1];
            mbar_expect_tx(bar, bytes);
            tma_load_1d(tiles + (tile & 1) * ST * 2, t.qrows + rr * 2, bytes, bar);
        };
        if (threadIdx.x == 0) {
            if (ntiles > 0) issue(0);
            if (ntiles > 1) issue(1);
        }
        TermC tc;
        termc_init(tc, crot + kCrot, t.sterm_c, tb, te);
        for (uint32_t i = 0; i < ntiles; ++i) {
            mbar_wait(&bars[i & 1], (i >> 1) & 1u);
            const uint64_t rem = R1 - R0 - uint64_t(i) * ST;
            const uint32_t n = rem < uint64_t(ST) ? uint32_t(rem) : uint32_t(ST);
            const uint32_t a0 = tiles_s + (i & 1) * ST * 32;
            const uint32_t aend = a0 + n * 32;
            // fused row loop (generated PTX): rows prefetched one ahead in ra / rb
            uint4 ra = lds128(a0), rb = lds128(a0 + 16);
            uint32_t ad = a0;
            while (ad < aend) {
                uint32_t vl, vpi, vpip, code;
                if constexpr (G > 4 && NT > 128) {
                    asm volatile(PZX_SORTED_ROWLOOP_G6_256
                                 : "+r"(ad), "+r"(J0), "+r"(J1), "+r"(J2), "+r"(Z), "=r"(vl), "=r"(vpi), "=r"(vpip),
                                   "=r"(code), "+r"(ra.x), "+r"(ra.y), "+r"(ra.z), "+r"(ra.w), "+r"(rb.x),
                                   "+r"(rb.y), "+r"(rb.z), "+r"(rb.w)
                                 : "r"(aend), "r"(tab_s), "r"(H0)
                                 : "memory");
                } else if constexpr (G > 4) {
                    asm volatile(PZX_SORTED_ROWLOOP_G6
                                 : "+r"(ad), "+r"(J0), "+r"(J1), "+r"(J2), "+r"(Z), "=r"(vl), "=r"(vpi), "=r"(vpip),
                                   "=r"(code), "+r"(ra.x), "+r"(ra.y), "+r"(ra.z), "+r"(ra.w), "+r"(rb.x),
                                   "+r"(rb.y), "+r"(rb.z), "+r"(rb.w)
                                 : "r"(aend), "r"(tab_s), "r"(H0)
                                 : "memory");
                } else {
                    asm volatile(PZX_SORTED_ROWLOOP_G4
                                 : "+r"(ad), "+r"(J0), "+r"(J1), "+r"(J2), "+r"(Z), "=r"(vl), "=r"(vpi), "=r"(vpip),
                                   "=r"(code), "+r"(ra.x), "+r"(ra.y), "+r"(ra.z), "+r"(ra.w), "+r"(rb.x),
                                   "+r"(rb.y), "+r"(rb.z), "+r"(rb.w)
                                 : "r"(aend), "r"(tab_s), "r"(H0)
                                 : "memory");
                }
                if (code & (kSliceLamFlag | kSlicePiFlag | kSlicePipFlag | kEndFlag)) {
                    if (code & kSliceLamFlag) K.bump_s(vl);
                    if (code & kSlicePiFlag) K.bump_a(vpi);
                    if (code & kSlicePipFlag) K.bump_b(vpip);
                    if (code & kEndFlag) {
                        if constexpr (DBG) debug_dump_codes<NT, (NT > 128)>(r, tc.next - 2, off, J0, J1, J2, Z, K);
                        slice_term_epilogue<NT, TM, true, (NT > 128)>(tc, t.sterm_c, L, crot, acc, J0, J1, J2, Z, K);
                    }
                }
            }
            __syncthreads();
            if (threadIdx.x == 0 && i + 2 < ntiles) {
                fence_proxy_async();
                issue(i + 2);
            }
        }
    }
    slice_store_results<NT, TM>(r, off, acc);
}


__global__ void k_mask_iota(const uint64_t* __restrict__ in, uint64_t n, uint64_t mask, uint64_t* keys,
                            uint32_t* vals) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[i] = in[i] & mask;
    vals[i] = uint32_t(i);
}

// ---------------------------------------------------------------------------
// Deterministic fixed-order reduction of per-chunk partial amplitudes.
__global__ void k_reduce_partials(const double2* __restrict__ partial, int n_chunks, uint64_t n,
                                  double2* amp, double* prob, int prob_mode, int accumulate,
                                  const uint32_t* __restrict__ perm) {
    const uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint64_t i = perm ? perm[k] : k;
    if (i == 0xFFFFFFFFu) return;  // padding slot of the sorted kernel
    double2 s = make_double2(0.0, 0.0);
    for (int c = 0; c < n_chunks; ++c) {
        const double2 v = partial[uint64_t(c) * n + k];
        s.x += v.x;
        s.y += v.y;
    }
    if (accumulate) {
        s.x += amp[i].x;
        s.y += amp[i].y;
    }
    if (amp) amp[i] = s;
    if (prob) prob[i] = prob_mode == 2 ? s.x : s.x * s.x + s.y * s.y;
}

// Few assignments, many term chunks (C1: 256 x 592, C4: 1024 x 4736): one
// warp per assignment, lane l sums chunks l, l + 32, ... in order, then a
// fixed shuffle tree -- deterministic, and the chunk reads of an assignment
// are spread over 32 lanes instead of one thread's serial chain.
__global__ void k_reduce_partials_warp(const double2* __restrict__ partial, int n_chunks, uint64_t n,
                                       double2* amp, double* prob, int prob_mode, int accumulate,
                                       const uint32_t* __restrict__ perm) {
    const uint64_t k = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31u;
    if (k >= n) return;
    double2 s = make_double2(0.0, 0.0);
    for (int c = int(lane); c < n_chunks; c += 32) {
        const double2 v = partial[uint64_t(c) * n + k];
        s.x += v.x;
        s.y += v.y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s.x += __shfl_down_sync(0xFFFFFFFFu, s.x, o);
        s.y += __shfl_down_sync(0xFFFFFFFFu, s.y, o);
    }
    if (lane != 0) return;
    const uint64_t i = perm ? perm[k] : k;
    if (i == 0xFFFFFFFFu) return;
    if (accumulate) {
        s.x += amp[i].x;
        s.y += amp[i].y;
    }
    if (amp) amp[i] = s;
    if (prob) prob[i] = prob_mode == 2 ? s.x : s.x * s.x + s.y * s.y;
}

__global__ void k_amp_to_prob(const double2* __restrict__ amp, uint64_t n, double* prob, int mode) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double2 v = amp[i];
    prob[i] = mode == 2 ? v.x : v.x * v.x + v.y * v.y;
}

template <bool P64>
__device__ __forceinline__ Row<P64> load_row_global(const DevTable& t, uint64_t row) {
    Row<P64> v;
    v.load(t.rows + row * Row<P64>::kWords);
    return v;
}

// E3: phase indices of every (device row, assignment).
__global__ void k_debug_phase(const DevTable t, const uint64_t* __restrict__ asg, uint64_t n, uint8_t* out) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= t.n_rows * n) return;
    const uint64_t row = i / n, k = i % n;
    const uint64_t a = asg[k];
    uint32_t p, q, code;
    if (t.p64) {
        const Row<true> v = load_row_global<true>(t, row);
        p = v.p(a); q = v.q(a); code = v.code;
    } else {
        const Row<false> v = load_row_global<false>(t, row);
        p = v.p(a); q = v.q(a); code = v.code;
    }
    const uint32_t cls = (code & kCodeMask) >> 4, ka = cls >> 3, kb = cls & 7;
    out[i] = uint8_t((((ka + 4 * p) & 7) << 3) | ((kb + 4 * q) & 7));
}

// Per (term, assignment) exact product codes, one thread each, wide counters
// (an independent re-derivation of what the SWAR kernels accumulate).
__global__ void k_debug_codes(const DevTable t, const uint64_t* __restrict__ asg, uint64_t n, uint32_t* out5) {
    extern __shared__ __align__(128) unsigned char smem[];
    const SmemLut L = stage_lut(t, smem);
    __syncthreads();
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= t.n_terms * n) return;
    const uint64_t term = i / n, k = i % n;
    const uint64_t a = asg[k];
    Wide w{0, 0, 0, 0, 0};
    for (uint64_t row = t.term_row[term]; row < t.term_row[term + 1]; ++row) {
        uint32_t p, q, code;
        if (t.p64) {
            const Row<true> v = load_row_global<true>(t, row);
            p = v.p(a); q = v.q(a); code = v.code;
        } else {
            const Row<false> v = load_row_global<false>(t, row);
            p = v.p(a); q = v.q(a); code = v.code;
        }
        widen(w, L.codes[((code & kCodeMask) >> 2) + (p | (q << 1))]);
    }
    uint32_t* o = out5 + 5 * i;
    o[0] = w.j & 7u; o[1] = w.z; o[2] = w.s1; o[3] = w.a; o[4] = w.b;
}

template <class KernelT>
cudaError_t launch_one(KernelT kern, dim3 grid, size_t smem, cudaStream_t s, const DevTable& t,
                       const LaunchReq& r) {
    if (smem > 48 * 1024) {
        cudaError_t e = set_max_smem(kern, smem);
        if (e != cudaSuccess) return e;
    }
    kern<<<grid, kThreads, smem, s>>>(t, r);
    return cudaGetLastError();
}

template <bool P64, bool LONG>
cudaError_t launch_typed(const DevTable& t, const LaunchReq& r, KernelChoice kc, dim3 grid) {
    const bool tm = tmem_accumulators();
    if (kc == KC_SORTED) {
        // wide tables (48 KB per 128 threads) with TMEM: 256-thread CTAs, 2 per SM = 16 warps
        const bool wide = r.sorted_groups > kSortedGroups;
        const size_t sm = wide ? (tm ? sorted_smem_bytes<true, kSortedGroupsWide, 256>(t)
                                     : sorted_smem_bytes<false, kSortedGroupsWide>(t))
                               : (tm ? sorted_smem_bytes<true>(t) : sorted_smem_bytes<false>(t));
        auto kern = wide ? (tm ? k_eval_sorted<true, kSortedGroupsWide, 256> : k_eval_sorted<false, kSortedGroupsWide>)
                         : (tm ? k_eval_sorted<true> : k_eval_sorted<false>);
        if (r.d_dbg5) {  // plane-dump variant (pzx_debug_slice_codes): TMEM builds only
            if (!tm) return cudaErrorNotSupported;
            kern = wide ? k_eval_sorted<true, kSortedGroupsWide, 256, true> : k_eval_sorted<true, kSortedGroups, 128, true>;
        }
        cudaError_t e = set_max_smem(kern, sm);
        if (e != cudaSuccess) return e;
        kern<<<grid, sorted_threads(r.sorted_groups), sm, r.stream>>>(t, r);
        return cudaGetLastError();
    }
    if (kc == KC_SLICEWC) {
        const size_t sm = slicewc_smem_bytes<P64>(t);
        auto kern = r.d_dbg5 ? k_eval_slice_wc<P64, true> : k_eval_slice_wc<P64>;
        cudaError_t e = set_max_smem(kern, sm);
        if (e != cudaSuccess) return e;
        kern<<<dim3(grid.x, grid.y / kWarpChunks), kSliceThreads, sm, r.stream>>>(t, r);
        return cudaGetLastError();
    }
    if (kc == KC_PAGE) {
        const size_t sm = page_smem_bytes(t);
        auto kern = r.d_dbg5 ? k_eval_page<true> : k_eval_page<false>;
        cudaError_t e = set_max_smem(kern, sm);
        if (e != cudaSuccess) return e;
        kern<<<grid, kSliceThreads, sm, r.stream>>>(t, r);
        return cudaGetLastError();
    }
    if (kc == KC_SLICE2) {
        const size_t sm = slice2_smem_bytes<P64>(t);
        cudaError_t e = set_max_smem(k_eval_slice2<P64>, sm);
        if (e != cudaSuccess) return e;
        k_eval_slice2<P64><<<grid, kSliceThreads, sm, r.stream>>>(t, r);
        return cudaGetLastError();
    }
    if (kc == KC_SLICE || kc == KC_SLICER) {
        const bool rnd = kc == KC_SLICER;
        const bool small = slice_threads(r) == 32;
        const size_t sm = rnd ? (small ? slice_smem_bytes<P64, true, 32>(t) : slice_smem_bytes<P64, true, 128>(t))
                        : small ? slice_smem_bytes<P64, false, 32>(t)
                        : tm    ? slice_smem_bytes<P64, false, 128, true>(t)
                                : slice_smem_bytes<P64, false, 128>(t);
        auto kern = rnd ? (small ? k_eval_slice<P64, true, 32> : k_eval_slice<P64, true, 128>)
                  : small ? k_eval_slice<P64, false, 32>
                  : tm    ? k_eval_slice<P64, false, 128, true>
                          : k_eval_slice<P64, false, 128>;
        if (r.d_dbg5) {  // plane-dump variant (pzx_debug_slice_codes): the 128-thread TMEM kernel only
            if (rnd || small || !tm) return cudaErrorNotSupported;
            kern = k_eval_slice<P64, false, 128, true, true>;
        }
        cudaError_t e = set_max_smem(kern, sm);
        if (e != cudaSuccess) return e;
        kern<<<grid, small ? 32 : 128, sm, r.stream>>>(t, r);
        return cudaGetLastError();
    }
    const size_t sm = smem_lut_offset<P64>() + t.lut_layout.bytes;
    if (kc == KC_GRAY) return launch_one(k_eval_gray<P64, kGrayBits, LONG>, grid, sm, r.stream, t, r);
    return launch_one(k_eval_general<P64, kGeneralK, LONG>, grid, sm, r.stream, t, r);
}

}  // namespace

// ------------------------------------------------------------------ host ----

// the page kernel: 128-thread TMEM CTAs, warps of 1024 consecutive assignments
// (lane bits = assignment bits 5..9), tables with the page layout (P <= 32)
bool page_kernel_ok(const DevTable& t, const LaunchReq& r) {
    static const bool off = std::getenv("PZX_NO_PAGES") != nullptr;  // A/B knob
    return !off && t.page_ok && tmem_accumulators() && slice_threads(r) == kSliceThreads && (r.first % 1024) == 0;
}

KernelChoice choose_kernel(const DevTable& t, const LaunchReq& r) {
    if (r.kernel != KC_AUTO) return r.kernel;
    const bool enumerated = r.d_asg == nullptr || r.words_contiguous;
    if (enumerated && t.slice_ok && (r.first % (2 * kSliceG)) == 0 && slice_threads(r) == kSliceThreads &&
        tmem_accumulators() && slice2_enabled())
        return KC_SLICE2;
    if (enumerated && page_kernel_ok(t, r)) return KC_PAGE;
    if (enumerated && t.slice_ok && (r.first % kSliceG) == 0)
        return (slice_threads(r) == 32 && tmem_accumulators()) ? KC_SLICEWC : KC_SLICE;
    if (enumerated && (r.first % kGray) == 0) return KC_GRAY;
    // arbitrary word lists: sort, then the bit-sliced kernel with per-thread
    // Four-Russians tables (needs n_params <= 32 and terms <= 127 rows)
    if (t.sorted_ok && r.d_asg && !r.words_contiguous && r.n >= uint64_t(kSliceG)) return KC_SORTED;
    return KC_GENERAL;
}

bool kernel_supported(const DevTable& t, const LaunchReq& r, KernelChoice kc) {
    const bool enumerated = r.d_asg == nullptr || r.words_contiguous;
    if (kc == KC_SLICE) return enumerated && t.slice_ok && (r.first % kSliceG) == 0;
    if (kc == KC_PAGE) return enumerated && t.page_ok && tmem_accumulators() && (r.first % 1024) == 0;
    if (kc == KC_SLICE2) return enumerated && t.slice_ok && (r.first % (2 * kSliceG)) == 0;
    if (kc == KC_SLICER) return t.slice_ok != 0;
    if (kc == KC_SORTED) return t.sorted_ok != 0 && r.d_asg != nullptr;
    if (kc == KC_GRAY) return enumerated && (r.first % kGray) == 0;
    return true;
}

// bit-sliced kernels: 32-thread CTAs when the batch cannot give every SM a
// 128-thread block (small enumerated batches with huge tables, e.g. C4)
// 32-thread CTAs only when a 128-thread CTA would leave warps idle (batches
// of a few thousand assignments, C4); otherwise 128 threads with TMEM
// accumulators -- term chunking supplies the CTAs a small batch lacks
int sorted_threads(int sorted_groups) {
    return (sorted_groups > kSortedGroups && tmem_accumulators()) ? 256 : kSliceThreads;
}

int slice_threads(const LaunchReq& r) {
    return r.n < uint64_t(4) * kSliceThreads * kSliceG ? 32 : kSliceThreads;
}

int grid_assign_blocks(const DevTable&, const LaunchReq& r, KernelChoice kc) {
    const uint64_t per = kc == KC_SLICEWC                  ? uint64_t(32) * kSliceG
                       : kc == KC_SLICE2                   ? uint64_t(kSliceThreads) * 2 * kSliceG
                       : kc == KC_SORTED                   ? uint64_t(sorted_threads(r.sorted_groups)) * kSliceG
                       : (kc == KC_SLICE || kc == KC_SLICER) ? uint64_t(slice_threads(r)) * kSliceG
                       : kc == KC_PAGE                     ? uint64_t(kSliceThreads) * kSliceG
                       : kc == KC_GRAY  ? uint64_t(kThreads) * kGray
                                        : uint64_t(kThreads) * kGeneralK;
    return int((r.n + per - 1) / per);
}


int resident_ctas_per_sm(const DevTable& t, KernelChoice kc, int nt, int sorted_groups) {
    const bool lng = t.max_rows > uint32_t(kSegRows);
    int nb = 0;
    size_t sm = (t.p64 ? smem_lut_offset<true>() : smem_lut_offset<false>()) + t.lut_layout.bytes;
    cudaError_t e;
#define PZX_OCC(K) e = cached_occupancy(&nb, K, kThreads, sm)
    const bool tm = tmem_accumulators();
    if (kc == KC_SLICEWC) {
        sm = t.p64 ? slicewc_smem_bytes<true>(t) : slicewc_smem_bytes<false>(t);
        auto kern = t.p64 ? k_eval_slice_wc<true> : k_eval_slice_wc<false>;
        e = cached_occupancy(&nb, kern, kSliceThreads, sm);
    } else if (kc == KC_PAGE) {
        sm = page_smem_bytes(t);
        e = cached_occupancy(&nb, k_eval_page<false>, kSliceThreads, sm);
    } else if (kc == KC_SLICE2) {
        sm = t.p64 ? slice2_smem_bytes<true>(t) : slice2_smem_bytes<false>(t);
        auto kern = t.p64 ? k_eval_slice2<true> : k_eval_slice2<false>;
        e = cached_occupancy(&nb, kern, kSliceThreads, sm);
    } else if (kc == KC_SORTED) {
        const bool wide = sorted_groups > kSortedGroups;
        sm = wide ? (tm ? sorted_smem_bytes<true, kSortedGroupsWide, 256>(t) : sorted_smem_bytes<false, kSortedGroupsWide>(t))
                  : (tm ? sorted_smem_bytes<true>(t) : sorted_smem_bytes<false>(t));
        auto kern = wide ? (tm ? k_eval_sorted<true, kSortedGroupsWide, 256> : k_eval_sorted<false, kSortedGroupsWide>)
                         : (tm ? k_eval_sorted<true> : k_eval_sorted<false>);
        e = cached_occupancy(&nb, kern, sorted_threads(sorted_groups), sm);
    } else if (kc == KC_SLICE || kc == KC_SLICER) {
        const bool rnd = kc == KC_SLICER;
        if (nt == 32) {
            auto kern = t.p64 ? (rnd ? k_eval_slice<true, true, 32> : k_eval_slice<true, false, 32>)
                              : (rnd ? k_eval_slice<false, true, 32> : k_eval_slice<false, false, 32>);
            sm = t.p64 ? (rnd ? slice_smem_bytes<true, true, 32>(t) : slice_smem_bytes<true, false, 32>(t))
                       : (rnd ? slice_smem_bytes<false, true, 32>(t) : slice_smem_bytes<false, false, 32>(t));
            e = cached_occupancy(&nb, kern, 32, sm);
        } else {
            auto kern = t.p64 ? (rnd ? k_eval_slice<true, true, 128>
                                 : tm ? k_eval_slice<true, false, 128, true> : k_eval_slice<true, false, 128>)
                              : (rnd ? k_eval_slice<false, true, 128>
                                 : tm ? k_eval_slice<false, false, 128, true> : k_eval_slice<false, false, 128>);
            sm = t.p64 ? (rnd ? slice_smem_bytes<true, true, 128>(t)
                          : tm ? slice_smem_bytes<true, false, 128, true>(t) : slice_smem_bytes<true, false, 128>(t))
                       : (rnd ? slice_smem_bytes<false, true, 128>(t)
                          : tm ? slice_smem_bytes<false, false, 128, true>(t) : slice_smem_bytes<false, false, 128>(t));
            e = cached_occupancy(&nb, kern, 128, sm);
        }
    } else if (kc == KC_GRAY) {
        if (t.p64) { if (lng) PZX_OCC((k_eval_gray<true, kGrayBits, true>)); else PZX_OCC((k_eval_gray<true, kGrayBits, false>)); }
        else { if (lng) PZX_OCC((k_eval_gray<false, kGrayBits, true>)); else PZX_OCC((k_eval_gray<false, kGrayBits, false>)); }
    } else {
        if (t.p64) { if (lng) PZX_OCC((k_eval_general<true, kGeneralK, true>)); else PZX_OCC((k_eval_general<true, kGeneralK, false>)); }
        else { if (lng) PZX_OCC((k_eval_general<false, kGeneralK, true>)); else PZX_OCC((k_eval_general<false, kGeneralK, false>)); }
    }
#undef PZX_OCC
    return (e == cudaSuccess && nb > 0) ? nb : 1;
}

cudaError_t launch_evaluate(const DevTable& t, const LaunchReq& r, KernelChoice kc, uint64_t* launches) {
    if (r.n == 0) return cudaSuccess;
    const dim3 grid(grid_assign_blocks(t, r, kc), r.n_chunks);
    const bool lng = t.max_rows > uint32_t(kSegRows);
    cudaError_t e;
    if (t.p64) e = lng ? launch_typed<true, true>(t, r, kc, grid) : launch_typed<true, false>(t, r, kc, grid);
    else e = lng ? launch_typed<false, true>(t, r, kc, grid) : launch_typed<false, false>(t, r, kc, grid);
    ++*launches;
    if (e != cudaSuccess || r.n_chunks <= 1) return e;
    const int tpb = 256;
    if (r.n_chunks >= 64 && r.n * 32 <= uint64_t(1) << 22) {  // few assignments, many chunks
        k_reduce_partials_warp<<<int((r.n * 32 + tpb - 1) / tpb), tpb, 0, r.stream>>>(
            r.d_partial, r.n_chunks, r.n, r.d_amp, r.d_prob, r.prob_mode, r.accumulate, r.d_perm);
    } else {
        k_reduce_partials<<<int((r.n + tpb - 1) / tpb), tpb, 0, r.stream>>>(r.d_partial, r.n_chunks, r.n, r.d_amp,
                                                                            r.d_prob, r.prob_mode, r.accumulate,
                                                                            r.d_perm);
    }
    ++*launches;
    return cudaGetLastError();
}

namespace {
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
size_t cub_sort_temp(uint64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, int64_t(n));
    return bytes;
}
}  // namespace


// ---- padded high-part groups for the sorted kernel ------------------------
// The sorted words are regrouped so that the 32 words of every thread share
// their high part (bits >= low): each run of equal high part is padded to a
// multiple of 32 slots (padding repeats the run's last word, perm = ~0 so
// nothing is stored for it). A thread then needs one high-part parity per
// row instead of two.
__global__ void k_run_flags(const uint64_t* __restrict__ k, uint64_t n, uint32_t low, uint32_t* flag) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    flag[i] = (i == 0 || (k[i] >> low) != (k[i - 1] >> low)) ? 1u : 0u;
}
__global__ void k_run_starts(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ rid, uint64_t n,
                             uint32_t* start) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && flag[i]) start[rid[i] - 1] = uint32_t(i);
}
__global__ void k_run_pads(const uint32_t* __restrict__ start, const uint32_t* __restrict__ n_runs_p, uint64_t n,
                           uint32_t* pad) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t R = *n_runs_p;
    if (r >= R) return;
    const uint64_t len = (r + 1 < R ? start[r + 1] : n) - start[r];
    pad[r] = uint32_t((32 - len % 32) % 32);
}
__global__ void k_group_scatter(const uint64_t* __restrict__ k, const uint32_t* __restrict__ perm,
                                const uint32_t* __restrict__ rid, const uint32_t* __restrict__ pad_before,
                                const uint32_t* __restrict__ start, const uint32_t* __restrict__ pad,
                                const uint32_t* __restrict__ n_runs_p, uint64_t n, uint64_t* pw, uint32_t* pp) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t r = rid[i] - 1;
    const uint64_t s = i + pad_before[r];
    pw[s] = k[i];
    pp[s] = perm[i];
    const uint32_t R = *n_runs_p;
    const uint64_t last = (r + 1 < R ? start[r + 1] : n) - 1;
    if (i == last)  // the run's padding slots follow its last word
        for (uint32_t q = 1; q <= pad[r]; ++q) {
            pw[s + q] = k[i];
            pp[s + q] = 0xFFFFFFFFu;
        }
}

size_t cub_scan_temp(uint64_t n) {
    size_t t = 0;
    cub::DeviceScan::InclusiveSum(nullptr, t, static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                  int64_t(n));
    size_t t2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t2, static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                  int64_t(n));
    return t > t2 ? t : t2;
}

size_t group_scratch_bytes(uint64_t n) {
    return 5 * align256(n * 4) + align256(2 * n * 8 + 64 * 8) + align256(2 * n * 4 + 64 * 4) + align256(cub_scan_temp(n)) + 256;
}

size_t sort_base_bytes(uint64_t n) {
    return 2 * align256(n * 8) + 2 * align256(n * 4) + align256(cub_sort_temp(n));
}

size_t sort_scratch_bytes(uint64_t n) { return sort_base_bytes(n) + group_scratch_bytes(n); }

cudaError_t group_sorted(const uint64_t* d_sorted, const uint32_t* d_perm, uint64_t n, uint32_t low, void* scratch,
                         const uint64_t** d_pw, const uint32_t** d_pp, uint64_t* n_slots, cudaStream_t s,
                         uint64_t* launches) {
    unsigned char* p = static_cast<unsigned char*>(scratch);
    auto take = [&](size_t b) { unsigned char* q = p; p += align256(b); return q; };
    uint32_t* flag = reinterpret_cast<uint32_t*>(take(n * 4));
    uint32_t* rid = reinterpret_cast<uint32_t*>(take(n * 4));
    uint32_t* start = reinterpret_cast<uint32_t*>(take(n * 4));
    uint32_t* pad = reinterpret_cast<uint32_t*>(take(n * 4));
    uint32_t* padb = reinterpret_cast<uint32_t*>(take(n * 4));
    uint64_t* pw = reinterpret_cast<uint64_t*>(take(2 * n * 8 + 64 * 8));
    uint32_t* pp = reinterpret_cast<uint32_t*>(take(2 * n * 4 + 64 * 4));
    size_t temp = cub_scan_temp(n);
    void* tmp = take(temp);
    uint32_t* nr = reinterpret_cast<uint32_t*>(take(16));
    const int b = 256, g = int((n + b - 1) / b);
    cudaError_t e;
    k_run_flags<<<g, b, 0, s>>>(d_sorted, n, low, flag);
    if ((e = cub::DeviceScan::InclusiveSum(tmp, temp, flag, rid, int64_t(n), s)) != cudaSuccess) return e;
    k_run_starts<<<g, b, 0, s>>>(flag, rid, n, start);
    if ((e = cudaMemcpyAsync(nr, rid + (n - 1), 4, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
    k_run_pads<<<g, b, 0, s>>>(start, nr, n, pad);
    uint32_t R = 0;
    if ((e = cudaMemcpyAsync(&R, nr, 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    if ((e = cub::DeviceScan::ExclusiveSum(tmp, temp, pad, padb, int64_t(R), s)) != cudaSuccess) return e;
    uint32_t tail[2] = {0, 0};
    if ((e = cudaMemcpyAsync(&tail[0], padb + (R - 1), 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(&tail[1], pad + (R - 1), 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    *n_slots = n + uint64_t(tail[0]) + tail[1];
    if (*n_slots > 2 * n + 64) return cudaErrorInvalidValue;  // caller checks the ratio first
    k_group_scatter<<<g, b, 0, s>>>(d_sorted, d_perm, rid, padb, start, pad, nr, n, pw, pp);
    *launches += 6;
    *d_pw = pw;
    *d_pp = pp;
    return cudaGetLastError();
}

// number of padded slots for a given low-bit count, without building them
cudaError_t group_slots(const uint64_t* d_sorted, uint64_t n, uint32_t low, void* scratch, uint64_t* n_slots,
                        cudaStream_t s, uint64_t* launches) {
    unsigned char* p = static_cast<unsigned char*>(scratch);
    auto take = [&](size_t b) { unsigned char* q = p; p += align256(b); return q; };
    uint32_t* flag = reinterpret_cast<uint32_t*>(take(n * 4));
    uint32_t* rid = reinterpret_cast<uint32_t*>(take(n * 4));
    uint32_t* start = reinterpret_cast<uint32_t*>(take(n * 4));
    uint32_t* pad = reinterpret_cast<uint32_t*>(take(n * 4));
    uint32_t* padb = reinterpret_cast<uint32_t*>(take(n * 4));
    take(2 * n * 8 + 64 * 8);
    take(2 * n * 4 + 64 * 4);
    size_t temp = cub_scan_temp(n);
    void* tmp = take(temp);
    uint32_t* nr = reinterpret_cast<uint32_t*>(take(16));
    const int b = 256, g = int((n + b - 1) / b);
    cudaError_t e;
    k_run_flags<<<g, b, 0, s>>>(d_sorted, n, low, flag);
    if ((e = cub::DeviceScan::InclusiveSum(tmp, temp, flag, rid, int64_t(n), s)) != cudaSuccess) return e;
    k_run_starts<<<g, b, 0, s>>>(flag, rid, n, start);
    if ((e = cudaMemcpyAsync(nr, rid + (n - 1), 4, cudaMemcpyDeviceToDevice, s)) != cudaSuccess) return e;
    k_run_pads<<<g, b, 0, s>>>(start, nr, n, pad);
    uint32_t R = 0;
    if ((e = cudaMemcpyAsync(&R, nr, 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    if ((e = cub::DeviceScan::ExclusiveSum(tmp, temp, pad, padb, int64_t(R), s)) != cudaSuccess) return e;
    uint32_t tail[2] = {0, 0};
    if ((e = cudaMemcpyAsync(&tail[0], padb + (R - 1), 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(&tail[1], pad + (R - 1), 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    *n_slots = n + uint64_t(tail[0]) + tail[1];
    *launches += 4;
    return cudaSuccess;
}

cudaError_t sort_words(const uint64_t* d_words, uint64_t n, uint32_t n_params, void* scratch,
                       const uint64_t** d_sorted, const uint32_t** d_perm, cudaStream_t s, uint64_t* launches) {
    unsigned char* p = static_cast<unsigned char*>(scratch);
    uint64_t* keys_in = reinterpret_cast<uint64_t*>(p);
    p += align256(n * 8);
    uint64_t* keys_out = reinterpret_cast<uint64_t*>(p);
    p += align256(n * 8);
    uint32_t* vals_in = reinterpret_cast<uint32_t*>(p);
    p += align256(n * 4);
    uint32_t* vals_out = reinterpret_cast<uint32_t*>(p);
    p += align256(n * 4);
    size_t temp = cub_sort_temp(n);
    const uint64_t mask = n_params >= 64 ? ~uint64_t(0) : ((uint64_t(1) << n_params) - 1);
    k_mask_iota<<<int((n + 255) / 256), 256, 0, s>>>(d_words, n, mask, keys_in, vals_in);
    ++*launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int end_bit = n_params >= 64 ? 64 : int(n_params > 0 ? n_params : 1);
    e = cub::DeviceRadixSort::SortPairs(p, temp, keys_in, keys_out, vals_in, vals_out, int64_t(n), 0, end_bit, s);
    ++*launches;
    *d_sorted = keys_out;
    *d_perm = vals_out;
    return e;
}

cudaError_t launch_amp_to_prob(const double2* amp, uint64_t n, double* prob, int mode, cudaStream_t s,
                               uint64_t* launches) {
    if (n == 0) return cudaSuccess;
    k_amp_to_prob<<<int((n + 255) / 256), 256, 0, s>>>(amp, n, prob, mode);
    ++*launches;
    return cudaGetLastError();
}

// ---- marginal summing (sim-driver epilogue) ----------------
// words[p * G + b] = fixed[p] | b, b < G = 2^m
__global__ void k_expand_words(const uint64_t* __restrict__ fixed, uint64_t n_fixed, uint32_t m, uint64_t* words) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= (n_fixed << m)) return;
    words[i] = fixed[i >> m] | (i & ((uint64_t(1) << m) - 1));
}

// out[s] (+)= sum of in[s * len .. s * len + len - 1]: one CTA per segment,
// strided per-thread sums then a fixed-order tree -- deterministic
__global__ void k_segment_sum(const double* __restrict__ in, uint64_t len, uint64_t n_seg, double* out,
                              int accumulate) {
    __shared__ double red[256];
    const uint64_t s = blockIdx.x;
    if (s >= n_seg) return;
    const double* p = in + s * len;
    double acc = 0.0;
    for (uint64_t i = threadIdx.x; i < len; i += blockDim.x) acc += p[i];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (int(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[s] = accumulate ? out[s] + red[0] : red[0];
}

// ---- repeated weak simulation (PAPER App. F Alg. 2) --------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// one chain-rule step for every sample i: p0 = P(B_i || 0), pp = P(B_i);
// bit k of word i := 0 with probability p0 / pp, else 1 (counter-based RNG:
// the draw depends only on (seed, k, i), so runs are reproducible)
__global__ void k_sample_step(uint64_t* words, double* pprev, const double* __restrict__ p0, uint64_t n, uint32_t k,
                              uint64_t seed, unsigned int* err) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double pp = pprev[i], q = p0[i];
    if (!(pp > 0.0)) {
        atomicOr(err, 1u);
        return;
    }
    double ratio = q / pp;
    ratio = ratio < 0.0 ? 0.0 : (ratio > 1.0 ? 1.0 : ratio);
    const uint64_t h = splitmix64(seed ^ splitmix64((uint64_t(k) << 48) ^ i));
    const double u = double(h >> 11) * 0x1.0p-53;
    if (u < ratio) {
        pprev[i] = q;
    } else {
        words[i] |= uint64_t(1) << k;
        pprev[i] = pp - q;
    }
}

cudaError_t launch_sample_step(uint64_t* d_words, double* d_pprev, const double* d_p0, uint64_t n, uint32_t k,
                               uint64_t seed, unsigned int* d_err, cudaStream_t s, uint64_t* launches) {
    if (n == 0) return cudaSuccess;
    k_sample_step<<<int((n + 255) / 256), 256, 0, s>>>(d_words, d_pprev, d_p0, n, k, seed, d_err);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_sum_partials(const double2* parts, int n_parts, uint64_t n, double2* amp, double* prob,
                                int prob_mode, cudaStream_t s, uint64_t* launches) {
    if (n == 0) return cudaSuccess;
    k_reduce_partials<<<int((n + 255) / 256), 256, 0, s>>>(parts, n_parts, n, amp, prob, prob_mode, 0, nullptr);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_expand_words(const uint64_t* d_fixed, uint64_t n_fixed, uint32_t m, uint64_t* d_words,
                                cudaStream_t s, uint64_t* launches) {
    const uint64_t n = n_fixed << m;
    if (n == 0) return cudaSuccess;
    k_expand_words<<<int((n + 255) / 256), 256, 0, s>>>(d_fixed, n_fixed, m, d_words);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_segment_sum(const double* d_in, uint64_t len, uint64_t n_seg, double* d_out, int accumulate,
                               cudaStream_t s, uint64_t* launches) {
    if (n_seg == 0) return cudaSuccess;
    k_segment_sum<<<int(n_seg), 256, 0, s>>>(d_in, len, n_seg, d_out, accumulate);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_debug_phase(const DevTable& t, const uint64_t* d_asg, uint64_t n, uint8_t* d_out,
                               cudaStream_t s, uint64_t* launches) {
    const uint64_t total = t.n_rows * n;
    if (total == 0) return cudaSuccess;
    k_debug_phase<<<int((total + 255) / 256), 256, 0, s>>>(t, d_asg, n, d_out);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_debug_codes(const DevTable& t, const uint64_t* d_asg, uint64_t n, uint32_t* d_out5,
                               cudaStream_t s, uint64_t* launches) {
    const uint64_t total = t.n_terms * n;
    if (total == 0) return cudaSuccess;
    if (t.lut_layout.bytes > 48 * 1024)
        cudaFuncSetAttribute(k_debug_codes, cudaFuncAttributeMaxDynamicSharedMemorySize, int(t.lut_layout.bytes));
    k_debug_codes<<<int((total + 255) / 256), 256, t.lut_layout.bytes, s>>>(t, d_asg, n, d_out5);
    ++*launches;
    return cudaGetLastError();
}


// --------------------------------------------------------- exact kernel ----
// pzx_evaluate_exact: the SPEC's integer-ring backend contract (S:444, 486,
// 493: identical RingQuad outputs, no floats in the kernel path). Each thread
// owns one assignment and walks the rows of its term chunk (uniform loads,
// broadcast through L1), accumulating the wide counters of DESIGN.md §2. With
// k = nLM_t - s1, mn = min(s1, k), r = |s1 - k| a term's value is
//   lambda^s1 mu^k = 2^(mn/2 + r/4) w^(6 (mn/2)) (1 - w^2)^(mn % 2) {lambda|mu}^r / 2^(r/4)
//   value = F_t 2^fx_t * w^j * lambda^s1 mu^k * 3^min(a,b) * pi^(a-b)
// (lambda mu = 1 - w^2, (1 - w^2)^2 = -2 w^2): an odd-ish Z[w] numerator
// (power basis 1, w, w^2, w^3; w^4 = -1) times a binary exponent. Numerators
// are int64 (int128 products, narrowed like the reference's narrow(),
// ring.cpp:13-18); the sum over terms is an int128 numerator with a running
// exponent, rescaled like ring_add (ring.cpp:57-70: a spread beyond what the
// numerator can absorb is an overflow), and converted to the canonical
// RingQuad (ring.cpp:20-48) once per assignment.
using i128d = __int128;

__device__ __forceinline__ bool fits_i62(long long v) { return v < (1ll << 62) && v > -(1ll << 62); }
__device__ __forceinline__ bool fits_i64(i128d v) { return v == i128d((long long)v); }
__device__ __forceinline__ bool fits_i126(i128d v) { return v < (i128d(1) << 126) && v > -(i128d(1) << 126); }
__device__ __forceinline__ bool shl_ok(i128d v, int s) {
    if (v == 0) return true;
    if (s > 124) return false;
    const i128d lim = i128d(1) << (126 - s);
    return v < lim && v > -lim;
}

// out = x * y in Z[w]; false when x exceeds 62 bits or a coefficient of the
// product exceeds int64. With |x| < 2^62 and |y| < 2^63 every int128 partial
// sum stays below 2^127.
__device__ __forceinline__ bool zw_mul_dev(const long long* x, const long long* y, long long* out) {
    i128d t[4] = {0, 0, 0, 0};
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 4; ++i) ok &= fits_i62(x[i]);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const i128d p = i128d(x[i]) * y[j];
            if (i + j < 4) t[i + j] += p; else t[i + j - 4] -= p;
        }
#pragma unroll
    for (int k = 0; k < 4; ++k) { ok &= fits_i64(t[k]); out[k] = (long long)t[k]; }
    return ok;
}

// bit length of the largest |coefficient| (|INT64_MIN| counts as 64)
__device__ __forceinline__ int zw_bits(const long long* x) {
    unsigned long long o = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) o |= (unsigned long long)(x[i] < 0 ? -x[i] : x[i]);
    return 64 - __clzll((long long)o);
}

// x * y in Z[w] with int64 arithmetic (caller guarantees no overflow)
__device__ __forceinline__ void zw_mul64(const long long* x, const long long* y, long long* out) {
    long long t[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const long long p = x[i] * y[j];
            if (i + j < 4) t[i + j] += p; else t[i + j - 4] -= p;
        }
#pragma unroll
    for (int k = 0; k < 4; ++k) out[k] = t[k];
}

// value = (c0 + c1 w + c2 w^2 + c3 w^3) * 2^e, exact; any == false: zero
struct XAcc {
    i128d c[4];
    int e;
    bool any;
    bool ok;  // (exact kernel's shared-memory slots) no overflow so far
};

__device__ __forceinline__ void xacc_norm(XAcc& A) {
    for (;;) {
        const i128d o = A.c[0] | A.c[1] | A.c[2] | A.c[3];
        if (o == 0) { A.any = false; return; }
        const unsigned long long lo = (unsigned long long)o;
        const int tz = lo ? __ffsll((long long)lo) - 1 : 64;
        if (tz == 0) return;
#pragma unroll
        for (int k = 0; k < 4; ++k) A.c[k] >>= tz;
        A.e += tz;
    }
}

// A += v * 2^ev. The numerator is left unnormalised (normalising costs more
// than the rare rescue): the exponent only moves down to the smallest one seen,
// and a shift that would overflow first strips A's factors of 2.
__device__ __forceinline__ bool xacc_shift_in(XAcc& A, const i128d* v, int ev) {
    if (ev >= A.e) {
        const int sh = ev - A.e;
        bool fit = true;
#pragma unroll
        for (int k = 0; k < 4; ++k) fit &= shl_ok(v[k], sh);
        if (!fit) return false;
#pragma unroll
        for (int k = 0; k < 4; ++k) A.c[k] += v[k] << sh;
    } else {
        const int sh = A.e - ev;
        bool fit = true;
#pragma unroll
        for (int k = 0; k < 4; ++k) fit &= shl_ok(A.c[k], sh);
        if (!fit) return false;
#pragma unroll
        for (int k = 0; k < 4; ++k) A.c[k] = (A.c[k] << sh) + v[k];
        A.e = ev;
    }
    return true;
}

__device__ __forceinline__ void xacc_add(XAcc& A, const i128d* v, int ev, bool& ok) {
    if (!A.any) {
#pragma unroll
        for (int k = 0; k < 4; ++k) A.c[k] = v[k];
        A.e = ev;
        A.any = true;
        return;
    }
    if (!xacc_shift_in(A, v, ev)) {
        xacc_norm(A);
        if (!A.any) {
#pragma unroll
            for (int k = 0; k < 4; ++k) A.c[k] = v[k];
            A.e = ev;
            A.any = true;
            return;
        }
        ok &= xacc_shift_in(A, v, ev);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) ok &= fits_i126(A.c[k]);
}

// canonical RingQuad {a,b,c,d,exp} of A (w = (sqrt2 + i sqrt2)/2: numerator
// a = 2c0, b = c1 - c3, c = 2c2, d = c1 + c3 over 2^(1 - e)); exp = -1 marks an
// assignment whose value does not fit (PZX_E_OVERFLOW)
__device__ __forceinline__ void exact_store(const XAcc& A, bool ok, long long* out) {
    i128d a = 0, b = 0, cc = 0, d = 0;
    long long ex = 0;
    XAcc N = A;
    if (ok && N.any) xacc_norm(N);
    if (ok && N.any) {
        a = 2 * N.c[0]; b = N.c[1] - N.c[3]; cc = 2 * N.c[2]; d = N.c[1] + N.c[3];
        ex = 1 - (long long)N.e;
        if (ex < 0) {
            ok = shl_ok(a, int(-ex)) && shl_ok(b, int(-ex)) && shl_ok(cc, int(-ex)) && shl_ok(d, int(-ex));
            if (ok) { a <<= -ex; b <<= -ex; cc <<= -ex; d <<= -ex; }
            ex = 0;
        }
        while (ok && ex > 0 && ((((long long)a) | ((long long)b) | ((long long)cc) | ((long long)d)) & 1) == 0) {
            a >>= 1; b >>= 1; cc >>= 1; d >>= 1; --ex;  // exact: all even
        }
        ok = ok && fits_i64(a) && fits_i64(b) && fits_i64(cc) && fits_i64(d) && ex <= 0x7FFFFFFF;
    }
    out[0] = ok ? (long long)a : 0;
    out[1] = ok ? (long long)b : 0;
    out[2] = ok ? (long long)cc : 0;
    out[3] = ok ? (long long)d : 0;
    out[4] = ok ? ex : -1;
}

// one term's value at one assignment: numerator n[4] (int64 in int128) and exponent
__device__ __forceinline__ bool exact_term(const ExactDev& x, uint64_t term, const Wide& w, i128d* n, int& ev) {
    const uint32_t nlm = x.nlm[term];
    const int fx = x.fx[term];
    if (w.s1 > nlm || fx == INT_MIN) return false;
    const uint32_t k = nlm - w.s1, mn = min(w.s1, k);
    const uint32_t r = w.s1 >= k ? w.s1 - k : k - w.s1;
    const uint32_t m = min(w.a, w.b);
    const int dd = int(w.a) - int(w.b);
    const uint32_t ad = uint32_t(dd < 0 ? -dd : dd);
    const bool use_lam = w.s1 >= k;
    if ((use_lam ? r >= x.lam_n : r >= x.mu_n) || ad >= x.pd_n || m >= x.p3_n) return false;
    const int64_t* base = use_lam ? x.lam + 4 * r : x.mu + 4 * r;
    long long q[4], p[4], t[4], f[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        q[i] = base[i];
        p[i] = x.pd[4 * (int(x.pd_n) - 1 + dd) + i];
        f[i] = x.ft[4 * term + i];
    }
    if (mn & 1u) {  // * (1 - w^2): c - w^2 c = (c0 + c2, c1 + c3, c2 - c0, c3 - c1)
        const long long c0 = q[0], c1 = q[1], c2 = q[2], c3 = q[3];
        q[0] = c0 + c2; q[1] = c1 + c3; q[2] = c2 - c0; q[3] = c3 - c1;  // |c| < 2^62: no wrap
    }
    const long long t3 = x.p3[m];
    bool ok = true;
    // coefficient bound of a Z[w] product: |x y| < 4 |x| |y|, so when the bit
    // lengths of the four factors sum to <= 58 the whole chain fits int64
    if (zw_bits(q) + zw_bits(p) + (64 - __clzll(t3)) + zw_bits(f) + 4 <= 62) {
        zw_mul64(q, p, t);
#pragma unroll
        for (int i = 0; i < 4; ++i) t[i] *= t3;
        zw_mul64(t, f, p);
    } else {
        ok = zw_mul_dev(q, p, t);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const i128d v3 = i128d(t[i]) * t3;
            ok &= fits_i64(v3);
            t[i] = (long long)v3;
        }
        ok &= zw_mul_dev(t, f, p);
    }
    // w^j: j & 4 negates, j & 3 rotates (w^4 = -1)
    const uint32_t j = (w.j + 6u * (mn >> 1)) & 7u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int src = (i - int(j & 3u)) & 3;
        long long v0 = p[src];
        if (i < int(j & 3u)) v0 = -v0;
        if (j & 4u) v0 = -v0;
        n[i] = i128d(v0);
    }
    ev = fx + int(mn >> 1) + int(r >> 2);
    return ok;
}

// row consumer of stream_rows: KX assignments per thread, SWAR code words
// (flushed into wide counters at segment / term ends), the Z[w] epilogue per term
template <bool P64, int KX>
struct ExactCons {
    const SmemLut& L;
    const ExactDev& x;
    XAcc* acc_s;  // this thread's KX accumulators in shared memory: kept out of the
                  // row loop's registers (in registers the compiler copies all
                  // 32 of them on every row)
    uint64_t a[KX];
    uint32_t acc[KX];
    Wide w[KX];
    uint64_t term;
    __device__ __forceinline__ ExactCons(const SmemLut& l, const ExactDev& xx) : L(l), x(xx) {}
    __device__ __forceinline__ void row(const Row<P64>& v) {
        const uint32_t cb = L.codes_s + (v.code & kCodeMask);
#pragma unroll
        for (int k = 0; k < KX; ++k) acc[k] += lds_u32(cb | (v.p(a[k]) << 2) | (v.q(a[k]) << 3));
    }
    __device__ __forceinline__ void flush() {
#pragma unroll
        for (int k = 0; k < KX; ++k) { widen(w[k], acc[k]); acc[k] = 0; }
    }
    __device__ __forceinline__ void close_term() {
#pragma unroll
        for (int k = 0; k < KX; ++k) {
            if (w[k].z == 0 && acc_s[k].ok) {
                i128d nv[4];
                int ev = 0;
                bool ok = exact_term(x, term, w[k], nv, ev);
                if (ok) {
                    XAcc A = acc_s[k];
                    xacc_add(A, nv, ev, ok);
                    acc_s[k] = A;
                }
                acc_s[k].ok = ok;
            }
            w[k] = Wide{0, 0, 0, 0, 0};
        }
    }
    __device__ __forceinline__ void end_term(const double2) {
#pragma unroll
        for (int k = 0; k < KX; ++k) { widen(w[k], acc[k]); acc[k] = 0; }
        close_term();
        ++term;
    }
};

template <bool P64>
__host__ __device__ constexpr uint32_t exact_acc_offset(uint32_t lut_bytes) {
    return (smem_lut_offset<P64>() + lut_bytes + 15u) & ~15u;
}

template <bool P64, int KX>
__global__ void __launch_bounds__(kExactThreads) k_eval_exact(const DevTable t, const ExactDev x, const uint64_t* __restrict__ asg,
                                                      uint64_t first, uint64_t n, const uint64_t* __restrict__ chunk_terms,
                                                      int n_chunks, i128d* __restrict__ partial, uint32_t* __restrict__ pflag,
                                                      long long* __restrict__ out) {
    extern __shared__ __align__(128) unsigned char smem[];
    const SmemLut L = kernel_prologue(t, smem, smem_lut_offset<P64>());
    const uint64_t tb = n_chunks > 1 ? chunk_terms[blockIdx.y] : 0;
    const uint64_t te = n_chunks > 1 ? chunk_terms[blockIdx.y + 1] : t.n_terms;
    ExactCons<P64, KX> c(L, x);
    c.acc_s = reinterpret_cast<XAcc*>(smem + exact_acc_offset<P64>(t.lut_layout.bytes)) + threadIdx.x * KX;
    const uint64_t idx0 = uint64_t(blockIdx.x) * (kExactThreads * KX) + threadIdx.x;
#pragma unroll
    for (int k = 0; k < KX; ++k) {
        const uint64_t idx = idx0 + uint64_t(k) * kExactThreads;
        c.a[k] = idx < n ? (asg ? asg[idx] : first + idx) : 0;
        c.acc[k] = 0;
        c.w[k] = Wide{0, 0, 0, 0, 0};
        c.acc_s[k].any = false;
        c.acc_s[k].ok = true;
        c.acc_s[k].e = 0;
    }
    c.term = tb;
    if (tb < te) stream_rows<Row<P64>, true>(t, t.rows, t.term_c, tb, te, smem, c);
#pragma unroll
    for (int k = 0; k < KX; ++k) {
        const uint64_t idx = idx0 + uint64_t(k) * kExactThreads;
        if (idx >= n) continue;
        const XAcc A = c.acc_s[k];
        if (n_chunks > 1) {
            i128d* pp = partial + 5 * (uint64_t(blockIdx.y) * n + idx);
#pragma unroll
            for (int i = 0; i < 4; ++i) pp[i] = A.any ? A.c[i] : 0;
            pp[4] = A.any ? i128d(A.e) : i128d(INT_MIN);
            if (!A.ok) pflag[idx] = 1u;
        } else {
            exact_store(A, A.ok, out + 5 * idx);
        }
    }
}

// merge of the chunk partials of each assignment (exact, order-free) + canonical store
__global__ void k_exact_reduce(const i128d* __restrict__ partial, const uint32_t* __restrict__ pflag, int n_chunks,
                               uint64_t n, long long* __restrict__ out) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    XAcc A;
    A.any = false;
    A.e = 0;
    bool ok = pflag[i] == 0u;
    for (int c = 0; c < n_chunks && ok; ++c) {
        const i128d* pp = partial + 5 * (uint64_t(c) * n + i);
        if (pp[4] == i128d(INT_MIN)) continue;
        const i128d v[4] = {pp[0], pp[1], pp[2], pp[3]};
        xacc_add(A, v, int(pp[4]), ok);
    }
    exact_store(A, ok, out + 5 * i);
}

// exact sum of G canonical RingQuads per assignment (the term split's combine,
// partials of disjoint term ranges, all-gathered rank-major
// [G][n][5]). (a + b sqrt2 + i(c + d sqrt2)) 2^-exp in the w power basis is
// (a, b + d, c, d - b) 2^-exp (sqrt2 = w - w^3, i sqrt2 = w + w^3); the sum is
// exact, so every order gives the one canonical result (ring.hpp:15-16).
// exp = -1 in any part (an overflowed partial) marks the output overflowed.
__global__ void k_ringquad_sum(const long long* __restrict__ parts, uint32_t g, uint64_t n, long long* __restrict__ out) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    XAcc A;
    A.any = false;
    A.e = 0;
    bool ok = true;
    for (uint32_t r = 0; r < g && ok; ++r) {
        const long long* q = parts + 5 * (uint64_t(r) * n + i);
        const long long a = q[0], b = q[1], c = q[2], d = q[3], ex = q[4];
        if (ex < 0 || ex > 0x7FFFFFFF) { ok = false; break; }
        if ((a | b | c | d) == 0) continue;
        const i128d v[4] = {i128d(a), i128d(b) + d, i128d(c), i128d(d) - b};
        xacc_add(A, v, -int(ex), ok);
    }
    exact_store(A, ok, out + 5 * i);
}

cudaError_t launch_ringquad_sum(const int64_t* d_parts, uint32_t g, uint64_t n, int64_t* d_out, cudaStream_t s,
                                uint64_t* launches) {
    if (n == 0) return cudaSuccess;
    k_ringquad_sum<<<unsigned((n + 255) / 256), 256, 0, s>>>(reinterpret_cast<const long long*>(d_parts), g, n,
                                                             reinterpret_cast<long long*>(d_out));
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_exact(const DevTable& t, const ExactDev& x, const uint64_t* d_asg, uint64_t first, uint64_t n,
                         const uint64_t* d_chunk_terms, int n_chunks, void* d_partial, uint32_t* d_pflag,
                         int64_t* d_out, cudaStream_t s, uint64_t* launches, int kx) {
    if (n == 0) return cudaSuccess;
    const size_t sm = (t.p64 ? exact_acc_offset<true>(t.lut_layout.bytes) : exact_acc_offset<false>(t.lut_layout.bytes)) +
                      size_t(kExactThreads) * kx * sizeof(XAcc);
    auto kern = kx == 4 ? (t.p64 ? k_eval_exact<true, 4> : k_eval_exact<false, 4>)
              : kx == 1 ? (t.p64 ? k_eval_exact<true, 1> : k_eval_exact<false, 1>)
                        : (t.p64 ? k_eval_exact<true, 2> : k_eval_exact<false, 2>);
    if (sm > 48 * 1024) {
        cudaError_t e = set_max_smem(kern, sm);
        if (e != cudaSuccess) return e;
    }
    const dim3 grid(unsigned((n + kExactThreads * kx - 1) / (kExactThreads * kx)), unsigned(n_chunks));
    i128d* part = static_cast<i128d*>(d_partial);
    long long* o = reinterpret_cast<long long*>(d_out);
    kern<<<grid, kExactThreads, sm, s>>>(t, x, d_asg, first, n, d_chunk_terms, n_chunks, part, d_pflag, o);
    ++*launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || n_chunks <= 1) return e;
    k_exact_reduce<<<unsigned((n + 255) / 256), 256, 0, s>>>(part, d_pflag, n_chunks, n, o);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace pzxb
