// pzx_kernels.cu -- sm_100a evaluation kernels for the parametric scalar
//   S(a) = sum_t C_t prod_r V(k_alpha_r + 4 p_r(a), k_beta_r + 4 q_r(a)),
//   p_r(a) = parity(psi_r & a), q_r(a) = parity(phi_r & a)
// (PAPER §3.3 steps 1-7; SPEC eval_row / evaluate S:448-474).
//
// Design: a thread owns assignments, every thread of a CTA
// walks the SAME rows (broadcast loads, no divergence, no dummy padding), the
// term product is accumulated exactly in exponent form with one 32-bit SWAR
// add per row-eval (pzx_internal.h code layout), and each term is converted
// once per assignment to fp64 through small shared-memory tables.
//
//   k_eval_general<P64> : any batch; AND + POPC parity per (row, assignment).
//   k_eval_gray<P64>    : enumerated batches; a thread owns 16 assignments
//                         that differ only in the low 4 bits, so per row it
//                         needs 2 POPCs for all 16 (the low-bit parities come
//                         from the row's precomputed Walsh pattern).
#include <cuda_runtime.h>

#include "pzx_internal.h"

namespace pzxb {

namespace {

struct SmemLut {
    const uint32_t* codes;
    const double2* om;
    const double* u;
    const double* p3;
    const double2* pd;  // centred: pd[d], d in [-max_rows, max_rows]
};

__device__ __forceinline__ SmemLut stage_lut(const DevTable& t, unsigned char* smem) {
    const uint4* src = reinterpret_cast<const uint4*>(t.lut);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    const uint32_t n16 = t.lut_layout.bytes / 16;
    for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = __ldg(src + i);
    __syncthreads();
    SmemLut L;
    L.codes = reinterpret_cast<const uint32_t*>(smem + t.lut_layout.codes_off);
    L.om = reinterpret_cast<const double2*>(smem + t.lut_layout.om_off);
    L.u = reinterpret_cast<const double*>(smem + t.lut_layout.u_off);
    L.p3 = reinterpret_cast<const double*>(smem + t.lut_layout.p3_off);
    L.pd = reinterpret_cast<const double2*>(smem + t.lut_layout.pd_off) + t.lut_layout.max_rows;
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
    double r = L.u[s1];
    if (a | b) {
        const uint32_t mn = a < b ? a : b;
        r *= L.p3[mn];
        const double2 pd = L.pd[int(a) - int(b)];
        const double wr = w.x * pd.x - w.y * pd.y;
        const double wi = w.x * pd.y + w.y * pd.x;
        w.x = wr; w.y = wi;
    }
    w.x *= r; w.y *= r;
    amp.x += C.x * w.x - C.y * w.y;
    amp.y += C.x * w.y + C.y * w.x;
}

__device__ __forceinline__ void epilogue_packed(uint32_t acc, const double2 C, const SmemLut& L,
                                                double2& amp) {
    term_epilogue(acc >> kJShift, acc & kField, (acc >> kS1Shift) & kField,
                  (acc >> kAShift) & kField, (acc >> kBShift) & kField, C, L, amp);
}

struct Wide { uint32_t j, z, s1, a, b; };

__device__ __forceinline__ void widen(Wide& w, uint32_t acc) {
    w.j += acc >> kJShift;
    w.z += acc & kField;
    w.s1 += (acc >> kS1Shift) & kField;
    w.a += (acc >> kAShift) & kField;
    w.b += (acc >> kBShift) & kField;
}

__device__ __forceinline__ void term_range(const DevTable& t, const LaunchReq& r, uint64_t& tb,
                                           uint64_t& te) {
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
    if (r.accumulate) {
        const double2 o = r.d_amp[idx];
        amp.x += o.x; amp.y += o.y;
    }
    if (r.d_amp) r.d_amp[idx] = amp;
    if (r.d_prob) r.d_prob[idx] = r.prob_mode == 2 ? amp.x : amp.x * amp.x + amp.y * amp.y;
}

// Row access for both mask widths. parity bits are returned as 0/1.
template <bool P64>
struct RowView;

template <>
struct RowView<false> {
    uint32_t psi, phi, code, pat;
    __device__ __forceinline__ void load(const DevTable& t, uint64_t row) {
        const uint4 w = __ldg(t.rows + row);
        psi = w.x; phi = w.y; code = w.z; pat = w.w;
    }
    __device__ __forceinline__ uint32_t p(uint64_t a) const { return __popc(psi & uint32_t(a)) & 1u; }
    __device__ __forceinline__ uint32_t q(uint64_t a) const { return __popc(phi & uint32_t(a)) & 1u; }
};

template <>
struct RowView<true> {
    uint32_t psi_lo, psi_hi, phi_lo, phi_hi, code, pat;
    __device__ __forceinline__ void load(const DevTable& t, uint64_t row) {
        const uint4 w = __ldg(t.rows + row);
        const uint2 x = __ldg(t.aux + row);
        psi_lo = w.x; psi_hi = w.y; phi_lo = w.z; phi_hi = w.w; code = x.x; pat = x.y;
    }
    __device__ __forceinline__ uint32_t p(uint64_t a) const {
        return __popc((psi_lo & uint32_t(a)) ^ (psi_hi & uint32_t(a >> 32))) & 1u;
    }
    __device__ __forceinline__ uint32_t q(uint64_t a) const {
        return __popc((phi_lo & uint32_t(a)) ^ (phi_hi & uint32_t(a >> 32))) & 1u;
    }
};

// ---------------------------------------------------------------------------
// General kernel: K assignments per thread, any assignment words.
template <bool P64, int K>
__global__ void __launch_bounds__(kThreads) k_eval_general(const DevTable t, const LaunchReq r) {
    extern __shared__ __align__(16) unsigned char smem[];
    const SmemLut L = stage_lut(t, smem);
    uint64_t tb, te;
    term_range(t, r, tb, te);

    const uint64_t idx0 = uint64_t(blockIdx.x) * (kThreads * K) + threadIdx.x;
    uint64_t a[K];
    double2 amp[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const uint64_t idx = idx0 + uint64_t(k) * kThreads;
        a[k] = idx < r.n ? (r.d_asg ? r.d_asg[idx] : r.first + idx) : 0;
        amp[k] = make_double2(0.0, 0.0);
    }

    for (uint64_t term = tb; term < te; ++term) {
        const uint64_t r0 = t.term_row[term], r1 = t.term_row[term + 1];
        const double2 C = __ldg(t.term_c + term);
        if (r1 - r0 <= uint64_t(kSegRows)) {
            uint32_t acc[K];
#pragma unroll
            for (int k = 0; k < K; ++k) acc[k] = 0;
#pragma unroll 2
            for (uint64_t row = r0; row < r1; ++row) {
                RowView<P64> v;
                v.load(t, row);
                const uint32_t* cl = L.codes + (v.code >> 2);
#pragma unroll
                for (int k = 0; k < K; ++k) acc[k] += cl[v.p(a[k]) | (v.q(a[k]) << 1)];
            }
#pragma unroll
            for (int k = 0; k < K; ++k) epilogue_packed(acc[k], C, L, amp[k]);
        } else {
            Wide w[K];
#pragma unroll
            for (int k = 0; k < K; ++k) w[k] = Wide{0, 0, 0, 0, 0};
            for (uint64_t s0 = r0; s0 < r1; s0 += kSegRows) {
                const uint64_t s1 = s0 + kSegRows < r1 ? s0 + kSegRows : r1;
                uint32_t acc[K];
#pragma unroll
                for (int k = 0; k < K; ++k) acc[k] = 0;
                for (uint64_t row = s0; row < s1; ++row) {
                    RowView<P64> v;
                    v.load(t, row);
                    const uint32_t* cl = L.codes + (v.code >> 2);
#pragma unroll
                    for (int k = 0; k < K; ++k) acc[k] += cl[v.p(a[k]) | (v.q(a[k]) << 1)];
                }
#pragma unroll
                for (int k = 0; k < K; ++k) widen(w[k], acc[k]);
            }
#pragma unroll
            for (int k = 0; k < K; ++k)
                term_epilogue(w[k].j, w[k].z, w[k].s1, w[k].a, w[k].b, C, L, amp[k]);
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) store_result(r, idx0 + uint64_t(k) * kThreads, amp[k]);
}

// ---------------------------------------------------------------------------
// Enumerated kernel: thread owns kGray assignments base + g (base % kGray == 0).
// parity(m & (base | g)) = parity(m & base) ^ parity(m_low & g); the second
// term, for all g at once, is the row's Walsh pattern (host-precomputed).
template <bool P64>
__device__ __forceinline__ uint32_t flips(const RowView<P64>& v, uint64_t base) {
    const uint32_t p = v.p(base), q = v.q(base);
    return (0x55555555u * p) ^ (0xAAAAAAAAu * q);
}

template <bool P64>
__global__ void __launch_bounds__(kThreads) k_eval_gray(const DevTable t, const LaunchReq r) {
    extern __shared__ __align__(16) unsigned char smem[];
    const SmemLut L = stage_lut(t, smem);
    uint64_t tb, te;
    term_range(t, r, tb, te);

    const uint64_t off = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) * kGray;
    // explicit word lists reach this kernel only when the host verified that
    // they are contiguous and 16-aligned: the thread's first word is its base
    const uint64_t base = r.d_asg ? (off < r.n ? r.d_asg[off] : 0) : r.first + off;
    double2 amp[kGray];
#pragma unroll
    for (int g = 0; g < kGray; ++g) amp[g] = make_double2(0.0, 0.0);

    for (uint64_t term = tb; term < te; ++term) {
        const uint64_t r0 = t.term_row[term], r1 = t.term_row[term + 1];
        const double2 C = __ldg(t.term_c + term);
        if (r1 - r0 <= uint64_t(kSegRows)) {
            uint32_t acc[kGray];
#pragma unroll
            for (int g = 0; g < kGray; ++g) acc[g] = 0;
            for (uint64_t row = r0; row < r1; ++row) {
                RowView<P64> v;
                v.load(t, row);
                const uint32_t xi = v.pat ^ flips(v, base);
                const uint32_t* cl = L.codes + (v.code >> 2);
#pragma unroll
                for (int g = 0; g < kGray; ++g) acc[g] += cl[(xi >> (2 * g)) & 3u];
            }
#pragma unroll
            for (int g = 0; g < kGray; ++g) epilogue_packed(acc[g], C, L, amp[g]);
        } else {
            Wide w[kGray];
#pragma unroll
            for (int g = 0; g < kGray; ++g) w[g] = Wide{0, 0, 0, 0, 0};
            for (uint64_t s0 = r0; s0 < r1; s0 += kSegRows) {
                const uint64_t s1 = s0 + kSegRows < r1 ? s0 + kSegRows : r1;
                uint32_t acc[kGray];
#pragma unroll
                for (int g = 0; g < kGray; ++g) acc[g] = 0;
                for (uint64_t row = s0; row < s1; ++row) {
                    RowView<P64> v;
                    v.load(t, row);
                    const uint32_t xi = v.pat ^ flips(v, base);
                    const uint32_t* cl = L.codes + (v.code >> 2);
#pragma unroll
                    for (int g = 0; g < kGray; ++g) acc[g] += cl[(xi >> (2 * g)) & 3u];
                }
#pragma unroll
                for (int g = 0; g < kGray; ++g) widen(w[g], acc[g]);
            }
#pragma unroll
            for (int g = 0; g < kGray; ++g)
                term_epilogue(w[g].j, w[g].z, w[g].s1, w[g].a, w[g].b, C, L, amp[g]);
        }
    }
#pragma unroll
    for (int g = 0; g < kGray; ++g) store_result(r, off + g, amp[g]);
}

// ---------------------------------------------------------------------------
// Deterministic fixed-order reduction of per-chunk partial amplitudes.
__global__ void k_reduce_partials(const double2* __restrict__ partial, int n_chunks, uint64_t n,
                                  double2* amp, double* prob, int prob_mode, int accumulate) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double2 s = make_double2(0.0, 0.0);
    for (int c = 0; c < n_chunks; ++c) {
        const double2 v = partial[uint64_t(c) * n + i];
        s.x += v.x; s.y += v.y;
    }
    if (accumulate) { s.x += amp[i].x; s.y += amp[i].y; }
    if (amp) amp[i] = s;
    if (prob) prob[i] = prob_mode == 2 ? s.x : s.x * s.x + s.y * s.y;
}

__global__ void k_amp_to_prob(const double2* __restrict__ amp, uint64_t n, double* prob, int mode) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double2 v = amp[i];
    prob[i] = mode == 2 ? v.x : v.x * v.x + v.y * v.y;
}

// E3: phase indices of every (row, assignment), device row order.
__global__ void k_debug_phase(const DevTable t, const uint64_t* __restrict__ asg, uint64_t n,
                              uint8_t* out) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= t.n_rows * n) return;
    const uint64_t row = i / n, k = i % n;
    const uint64_t a = asg[k];
    uint32_t p, q, code;
    if (t.p64) {
        RowView<true> v; v.load(t, row);
        p = v.p(a); q = v.q(a); code = v.code;
    } else {
        RowView<false> v; v.load(t, row);
        p = v.p(a); q = v.q(a); code = v.code;
    }
    const uint32_t cls = code >> 4, ka = cls >> 3, kb = cls & 7;
    out[i] = uint8_t((((ka + 4 * p) & 7) << 3) | ((kb + 4 * q) & 7));
}

// Per (term, assignment) exact product codes, one thread each, wide counters
// (an independent re-derivation of what the SWAR kernels accumulate).
__global__ void k_debug_codes(const DevTable t, const uint64_t* __restrict__ asg, uint64_t n,
                              uint32_t* out5) {
    extern __shared__ __align__(16) unsigned char smem[];
    const SmemLut L = stage_lut(t, smem);
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= t.n_terms * n) return;
    const uint64_t term = i / n, k = i % n;
    const uint64_t a = asg[k];
    Wide w{0, 0, 0, 0, 0};
    for (uint64_t row = t.term_row[term]; row < t.term_row[term + 1]; ++row) {
        uint32_t p, q, code;
        if (t.p64) {
            RowView<true> v; v.load(t, row);
            p = v.p(a); q = v.q(a); code = v.code;
        } else {
            RowView<false> v; v.load(t, row);
            p = v.p(a); q = v.q(a); code = v.code;
        }
        widen(w, L.codes[(code >> 2) + (p | (q << 1))]);
    }
    uint32_t* o = out5 + 5 * i;
    o[0] = w.j & 7u; o[1] = w.z; o[2] = w.s1; o[3] = w.a; o[4] = w.b;
}

}  // namespace

// ------------------------------------------------------------------ host ----

KernelChoice choose_kernel(const DevTable& t, const LaunchReq& r) {
    if (r.kernel != KC_AUTO) return r.kernel;
    if ((r.d_asg == nullptr || r.words_contiguous) && (r.first % kGray) == 0) return KC_GRAY;
    return KC_GENERAL;
}

int grid_assign_blocks(const DevTable&, const LaunchReq& r, KernelChoice kc) {
    const uint64_t per = kc == KC_GRAY ? uint64_t(kThreads) * kGray : uint64_t(kThreads) * kGeneralK;
    return int((r.n + per - 1) / per);
}

cudaError_t launch_evaluate(const DevTable& t, const LaunchReq& r, KernelChoice kc,
                            uint64_t* launches) {
    if (r.n == 0) return cudaSuccess;
    const dim3 grid(grid_assign_blocks(t, r, kc), r.n_chunks);
    const size_t sm = t.lut_layout.bytes;
    if (sm > 48 * 1024) {
        cudaFuncSetAttribute(k_eval_gray<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        cudaFuncSetAttribute(k_eval_gray<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        cudaFuncSetAttribute(k_eval_general<true, kGeneralK>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        cudaFuncSetAttribute(k_eval_general<false, kGeneralK>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        cudaFuncSetAttribute(k_debug_codes, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    }
    if (kc == KC_GRAY) {
        if (t.p64) k_eval_gray<true><<<grid, kThreads, sm, r.stream>>>(t, r);
        else k_eval_gray<false><<<grid, kThreads, sm, r.stream>>>(t, r);
    } else {
        if (t.p64) k_eval_general<true, kGeneralK><<<grid, kThreads, sm, r.stream>>>(t, r);
        else k_eval_general<false, kGeneralK><<<grid, kThreads, sm, r.stream>>>(t, r);
    }
    ++*launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || r.n_chunks <= 1) return e;
    const int tpb = 256;
    k_reduce_partials<<<int((r.n + tpb - 1) / tpb), tpb, 0, r.stream>>>(
        r.d_partial, r.n_chunks, r.n, r.d_amp, r.d_prob, r.prob_mode, r.accumulate);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_amp_to_prob(const double2* amp, uint64_t n, double* prob, int mode,
                               cudaStream_t s, uint64_t* launches) {
    if (n == 0) return cudaSuccess;
    k_amp_to_prob<<<int((n + 255) / 256), 256, 0, s>>>(amp, n, prob, mode);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_debug_phase(const DevTable& t, const uint64_t* d_asg, uint64_t n,
                               uint8_t* d_out, cudaStream_t s, uint64_t* launches) {
    const uint64_t total = t.n_rows * n;
    if (total == 0) return cudaSuccess;
    k_debug_phase<<<int((total + 255) / 256), 256, 0, s>>>(t, d_asg, n, d_out);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_debug_codes(const DevTable& t, const uint64_t* d_asg, uint64_t n,
                               uint32_t* d_out5, cudaStream_t s, uint64_t* launches) {
    const uint64_t total = t.n_terms * n;
    if (total == 0) return cudaSuccess;
    k_debug_codes<<<int((total + 255) / 256), 256, t.lut_layout.bytes, s>>>(t, d_asg, n, d_out5);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace pzxb
