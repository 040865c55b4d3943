// pzx_group.cpp -- one host thread driving several GPUs through the C ABI
// (SURVEY §8b's `pzx_create(devices, n)` / REPLICATE | SPLIT_TERMS upload).
//
// REPLICATE: the table is uploaded to every device and a batch is cut into
// contiguous per-device slices evaluated concurrently (one std::thread per
// device) straight into the caller's output -- no inter-GPU traffic.
// SPLIT_TERMS: device d holds a row-balanced term range; every device
// evaluates the whole batch into partial amplitudes, which are copied peer to
// peer (NVLink) to the first device and summed there in device order by the
// fixed-order chunk reduction (deterministic), then |.|^2 / Re.
// The python/torch.distributed path (dist.py, bench.py) is the
// one-process-per-GPU alternative; this one serves C/C++ callers.
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "pzx_gpu.h"
#include "pzx_internal.h"

struct pzx_group {
    std::vector<int> devices;
    std::vector<pzx_ctx*> ctx;
    std::string err;
};

struct pzx_group_table {
    uint32_t mode = PZX_REPLICATE;
    std::vector<pzx_table*> t;  // one per device
};

namespace {

pzx_status fail(pzx_group* g, pzx_status st, const std::string& what) {
    g->err = what;
    return st;
}

// row-balanced contiguous term ranges
std::vector<uint64_t> term_cuts(const pzx_expr_view* e, int parts) {
    std::vector<uint64_t> cut(parts + 1, e->n_terms);
    cut[0] = 0;
    const uint64_t base = e->term_offset[0], rows = e->term_offset[e->n_terms] - base;
    uint64_t t = 0;
    for (int p = 1; p < parts; ++p) {
        const uint64_t want = base + rows * uint64_t(p) / uint64_t(parts);
        while (t < e->n_terms && e->term_offset[t] < want) ++t;
        cut[p] = std::max(t, cut[p - 1]);
    }
    return cut;
}

template <typename F>
pzx_status for_each_device(pzx_group* g, F&& f) {
    std::vector<pzx_status> st(g->ctx.size(), PZX_OK);
    std::vector<std::thread> th;
    for (size_t d = 0; d < g->ctx.size(); ++d) th.emplace_back([&, d] { st[d] = f(int(d)); });
    for (auto& x : th) x.join();
    for (size_t d = 0; d < st.size(); ++d)
        if (st[d]) return fail(g, st[d], std::string("device ") + std::to_string(g->devices[d]) + ": " +
                                           pzx_last_error(g->ctx[d]));
    return PZX_OK;
}

}  // namespace

extern "C" {

pzx_status pzx_group_create(const int* devices, int n_devices, pzx_group** out) {
    if (!devices || n_devices <= 0 || !out) return PZX_E_INVALID;
    *out = nullptr;
    std::unique_ptr<pzx_group> g(new (std::nothrow) pzx_group);
    if (!g) return PZX_E_OOM;
    for (int d = 0; d < n_devices; ++d) {
        pzx_ctx* c = nullptr;
        const pzx_status st = pzx_create(devices[d], &c);
        if (st) {
            for (pzx_ctx* x : g->ctx) pzx_destroy(x);
            return st;
        }
        g->devices.push_back(devices[d]);
        g->ctx.push_back(c);
    }
    // peer access to the first device (NVLink) where the hardware allows it
    for (int d = 1; d < n_devices; ++d) {
        if (devices[d] == devices[0]) continue;
        int ok = 0;
        if (cudaDeviceCanAccessPeer(&ok, devices[0], devices[d]) == cudaSuccess && ok) {
            cudaSetDevice(devices[0]);
            cudaDeviceEnablePeerAccess(devices[d], 0);
            cudaGetLastError();  // already enabled is fine
        }
    }
    *out = g.release();
    return PZX_OK;
}

void pzx_group_destroy(pzx_group* g) {
    if (!g) return;
    for (pzx_ctx* c : g->ctx) pzx_destroy(c);
    delete g;
}

const char* pzx_group_last_error(const pzx_group* g) { return g ? g->err.c_str() : "no group"; }

pzx_status pzx_group_upload_expr(pzx_group* g, const pzx_expr_view* e, uint32_t mode, pzx_group_table** out) {
    if (!g || !e || !out || (mode != PZX_REPLICATE && mode != PZX_SPLIT_TERMS)) return PZX_E_INVALID;
    *out = nullptr;
    std::unique_ptr<pzx_group_table> gt(new (std::nothrow) pzx_group_table);
    if (!gt) return PZX_E_OOM;
    gt->mode = mode;
    gt->t.assign(g->ctx.size(), nullptr);
    const int n = int(g->ctx.size());
    const std::vector<uint64_t> cut = mode == PZX_SPLIT_TERMS ? term_cuts(e, n) : std::vector<uint64_t>();
    const pzx_status st = for_each_device(g, [&](int d) {
        pzx_expr_view v = *e;
        if (mode == PZX_SPLIT_TERMS) {  // term_offset holds absolute indices: a sub-range is a valid view
            v.term_offset = e->term_offset + cut[d];
            v.term_scalar = e->term_scalar + 5 * cut[d];
            v.n_terms = cut[d + 1] - cut[d];
        }
        return pzx_table_upload_expr(g->ctx[d], &v, &gt->t[d]);
    });
    if (st) {
        pzx_group_table_free(gt.release());
        return st;
    }
    *out = gt.release();
    return PZX_OK;
}

void pzx_group_table_free(pzx_group_table* gt) {
    if (!gt) return;
    for (pzx_table* t : gt->t) pzx_table_free(t);
    delete gt;
}

pzx_status pzx_group_evaluate(pzx_group* g, const pzx_group_table* gt, const uint64_t* assignments, uint64_t first,
                              uint64_t n, double* amp, double* prob, uint32_t flags) {
    if (!g || !gt || gt->t.size() != g->ctx.size()) return PZX_E_INVALID;
    if (n == 0 || (!amp && !prob)) return PZX_OK;
    const int nd = int(g->ctx.size());
    if (gt->mode == PZX_REPLICATE) {  // contiguous slices, no collective
        return for_each_device(g, [&](int d) -> pzx_status {
            const uint64_t lo = n * uint64_t(d) / uint64_t(nd), hi = n * uint64_t(d + 1) / uint64_t(nd);
            if (hi == lo) return PZX_OK;
            double* a = amp ? amp + 2 * lo : nullptr;
            double* p = prob ? prob + lo : nullptr;
            return assignments ? pzx_evaluate(g->ctx[d], gt->t[d], assignments + lo, hi - lo, a, p, flags)
                               : pzx_evaluate_range(g->ctx[d], gt->t[d], first + lo, hi - lo, a, p, flags);
        });
    }
    // SPLIT_TERMS: partial amplitudes per device -> device 0 -> ordered sum
    std::vector<double*> part(nd, nullptr);
    std::vector<uint64_t*> words(nd, nullptr);
    double* stage = nullptr;
    double* d_amp = nullptr;
    double* d_prob = nullptr;
    auto cleanup = [&] {
        for (int d = 0; d < nd; ++d) {
            cudaSetDevice(g->devices[d]);
            if (part[d]) cudaFree(part[d]);
            if (words[d]) cudaFree(words[d]);
        }
        cudaSetDevice(g->devices[0]);
        for (void* p : {static_cast<void*>(stage), static_cast<void*>(d_amp), static_cast<void*>(d_prob)})
            if (p) cudaFree(p);
    };
    pzx_status st = for_each_device(g, [&](int d) -> pzx_status {
        if (cudaSetDevice(g->devices[d]) != cudaSuccess) return PZX_E_CUDA;
        if (cudaMalloc(reinterpret_cast<void**>(&part[d]), n * 16) != cudaSuccess) return PZX_E_OOM;
        if (assignments) {
            if (cudaMalloc(reinterpret_cast<void**>(&words[d]), n * 8) != cudaSuccess) return PZX_E_OOM;
            if (cudaMemcpy(words[d], assignments, n * 8, cudaMemcpyHostToDevice) != cudaSuccess) return PZX_E_CUDA;
        }
        const uint32_t f = flags & ~uint32_t(PZX_ACCUMULATE);
        pzx_status s = pzx_evaluate_device(g->ctx[d], gt->t[d], words[d], first, n, 0, UINT64_MAX, part[d],
                                           nullptr, f, nullptr);
        if (s) return s;
        return cudaDeviceSynchronize() == cudaSuccess ? PZX_OK : PZX_E_CUDA;
    });
    if (st) {
        cleanup();
        return st;
    }
    const int d0 = g->devices[0];
    cudaSetDevice(d0);
    uint64_t launches = 0;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&stage), size_t(nd) * n * 16);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&d_amp), n * 16);
    if (e == cudaSuccess && prob) e = cudaMalloc(reinterpret_cast<void**>(&d_prob), n * 8);
    for (int d = 0; d < nd && e == cudaSuccess; ++d)
        e = cudaMemcpyPeer(stage + 2 * n * uint64_t(d), d0, part[d], g->devices[d], n * 16);
    if (e == cudaSuccess)
        e = pzxb::launch_sum_partials(reinterpret_cast<const double2*>(stage), nd, n,
                                      reinterpret_cast<double2*>(d_amp), d_prob,
                                      (flags & PZX_PROB_REAL) ? 2 : 1, nullptr, &launches);
    if (e == cudaSuccess && amp) e = cudaMemcpy(amp, d_amp, n * 16, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && prob) e = cudaMemcpy(prob, d_prob, n * 8, cudaMemcpyDeviceToHost);
    cleanup();
    if (e != cudaSuccess) return fail(g, PZX_E_CUDA, std::string("term-split reduction: ") + cudaGetErrorString(e));
    return PZX_OK;
}

}  // extern "C"
