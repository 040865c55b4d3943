// pzx_reduce.cpp -- host-side parametric reducer: Clifford+T circuit -> closed
// polar-parameterised ZX diagram -> Clifford simplification + stabiliser
// decomposition -> the leaf-term list (scalar x subterms) the evaluator
// consumes (SPEC zx-core S:67-84, rewrite-engine S:131-244,
// decomposer S:246-317). The reference ships none of these: its core stops at
// the diagram data model (proj/core/include/pzx/diagram.hpp:40-102); this is
// a from-scratch C++ producer whose output is exactly the reference's leaf
// form -- a RingQuad scalar_ times pending_ subterms of the four kinds of
// subterm.hpp:19-36 -- so that every downstream step (normalize_subterm,
// the table compiler, the kernels, the oracle) is unchanged.
//
// Conventions (all scalars exact in Z[w][1/sqrt2], w = e^{i pi/4}):
//   Z spider, phase a: |0..0><0..0| + e^{ia} |1..1><1..1|
//   Hadamard edge:     H[x, y] = (-1)^{xy} / sqrt2
//   phase (k, mask):   k pi/4 + pi * parity(mask & a)     (ParamPhase, phase.hpp:34-52)
// The diagram is kept graph-like at all times: Z spiders only, Hadamard edges
// only, no self-loops or parallel edges (closed: no boundaries). Every rule's
// scalar is derived in DESIGN.md §11 by summing out the removed spiders; the
// tests check each rule and whole circuits against dense statevectors.
//
// Rules (SPEC names):
//   local_complement (LC)  k in {2,6}: neighbours -= phase, neighbourhood
//       complemented, scalar sqrt2^(1-n) * HalfPi(phase)   (App. B)
//   pivot                  k_u, k_v in {0,4} on an edge: PiPair(u, v),
//       sqrt2^(3 - d_u - d_v), U'/V'/W phase + complement rule
//   copy_state             degree-1 Pauli u on any v: PiPair(v, u), v removed
//   remove_identity        (0, {}) of degree 2: its neighbours fuse
//   scalar leftovers       isolated spider: Node; isolated edge: PhasePair/sqrt2
// Decomposition (T-like = odd k, any mask): two T-like spiders u, v split as
//   sum_{x,y} e^{i(a_u x + a_v y)} = [x = y] (fuse: phase a_u + a_v) +
//                                    [y = 1-x] (flip-fuse: phase a_u - a_v, e^{i a_v})
// (both phases even: two Clifford terms per pair of T-spiders); a single
// leftover T-spider splits on its value (2 terms).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "pzx_gpu.h"
#include "pzx_math.hpp"
#include <nvtx3/nvToolsExt.h>

using namespace pzxb;

namespace {

struct Ph {
    uint8_t k = 0;
    uint64_t m = 0;
};
inline Ph ph_add(Ph a, Ph b) { return {uint8_t((a.k + b.k) & 7), a.m ^ b.m}; }
inline Ph ph_sub(Ph a, Ph b) { return {uint8_t((a.k - b.k) & 7), a.m ^ b.m}; }
inline Ph ph_pi() { return {4, 0}; }
inline bool is_pauli(Ph p) { return (p.k & 3) == 0; }   // image {0, pi}
inline bool is_proper(Ph p) { return (p.k & 3) == 2; }  // image {pi/2, 3pi/2}
inline bool is_tlike(Ph p) { return (p.k & 1) != 0; }

struct Sub {
    uint8_t kind, psi_k, phi_k;
    uint64_t psi_m, phi_m;
};

// exact scalar num * sqrt2^s2 (num in Z[w]); zero() when a factor vanished
struct Scalar {
    Zw num = zw(1, 0, 0, 0);
    int s2 = 0;
    bool ok = true;  // false: an intermediate left int64 (reported as PZX_E_OVERFLOW)
    bool zero() const { return num.zero(); }
    void mul(const Zw& v) {
        i128 t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) t[i + j] += i128(num.c[i]) * v.c[j];
        for (int i = 0; i < 4; ++i) {
            const i128 r = t[i] - t[i + 4];
            if (r > INT64_MAX || r < INT64_MIN) ok = false;
            num.c[i] = int64_t(r);
        }
        norm();
    }
    void w(int k) { mul(zw_pow_w(k)); }
    void sqrt2(int p) { s2 += p; }
    // divide out sqrt2 while exact (sqrt2 = w - w^3; x / sqrt2 = x * sqrt2 / 2)
    void norm() {
        if (num.zero()) { s2 = 0; return; }
        for (;;) {
            const Zw t = zw_mul(num, zw(0, 1, 0, -1));
            if ((t.c[0] | t.c[1] | t.c[2] | t.c[3]) & 1) return;
            for (int i = 0; i < 4; ++i) num.c[i] = t.c[i] / 2;
            s2 += 1;
        }
    }
    bool to_quad(Quad& q) const {
        if (num.zero()) { q = Quad{}; return true; }
        Zw n = num;
        int e = s2;
        if (e & 1) { n = zw_mul(n, zw(0, 1, 0, -1)); e -= 1; }  // sqrt2^odd = sqrt2 * 2^((odd-1)/2)
        Quad base;
        if (!zw_to_quad(n, base)) return false;
        return quad_canon(base.a, base.b, base.c, base.d, int64_t(base.e) - e / 2, q);
    }
};

struct Dg {
    std::vector<Ph> ph;
    std::vector<std::vector<int>> adj;  // Hadamard edges, no self-loops, no parallels
    std::vector<char> alive;
    int n_alive = 0;
    Scalar sc;
    std::vector<Sub> subs;

    int add_vertex(Ph p) {
        ph.push_back(p);
        adj.emplace_back();
        alive.push_back(1);
        ++n_alive;
        return int(ph.size()) - 1;
    }
    bool has_edge(int u, int v) const {
        const auto& a = adj[u].size() < adj[v].size() ? adj[u] : adj[v];
        const int o = adj[u].size() < adj[v].size() ? v : u;
        return std::find(a.begin(), a.end(), o) != a.end();
    }
    void erase_edge(int u, int v) {
        auto& a = adj[u];
        a.erase(std::find(a.begin(), a.end(), v));
        auto& b = adj[v];
        b.erase(std::find(b.begin(), b.end(), u));
    }
    // one more Hadamard edge u-v: two parallel ones cancel (H[x,y]^2 = 1/2),
    // a self-loop is H[x,x] = (-1)^x / sqrt2 (phase pi)
    void add_h(int u, int v) {
        if (u == v) {
            ph[u] = ph_add(ph[u], ph_pi());
            sc.sqrt2(-1);
        } else if (has_edge(u, v)) {
            erase_edge(u, v);
            sc.sqrt2(-2);
        } else {
            adj[u].push_back(v);
            adj[v].push_back(u);
        }
    }
    // multiply by (-1)^{x_u x_v} = sqrt2 * (one more Hadamard edge)
    void toggle(int u, int v) {
        add_h(u, v);
        sc.sqrt2(1);
    }
    void remove_vertex(int u) {
        for (int w : adj[u]) {
            auto& b = adj[w];
            b.erase(std::find(b.begin(), b.end(), u));
        }
        adj[u].clear();
        alive[u] = 0;
        --n_alive;
    }
    // identify the values of v and u (v merged into u)
    void fuse(int u, int v) {
        ph[u] = ph_add(ph[u], ph[v]);
        std::vector<int> nb = adj[v];
        remove_vertex(v);
        for (int w : nb) add_h(u, w);
    }
    // x_v = 1 - x_u: e^{i a_v (1 - x)} = e^{i a_v} e^{-i a_v x}; v's neighbours see
    // (-1)^{(1-x) z} = (-1)^z (-1)^{xz}: phase pi and an edge to u
    void flip_fuse(int u, int v) {
        const Ph pv = ph[v];
        emit_exp(pv);
        ph[u] = ph_sub(ph[u], pv);
        std::vector<int> nb = adj[v];
        remove_vertex(v);
        for (int w : nb) {
            ph[w] = ph_add(ph[w], ph_pi());
            add_h(u, w);
        }
    }
    // ---- subterms (parameter-free ones fold into the scalar, as push_subterm,
    // diagram.cpp:114-120) ----
    void emit(uint8_t kind, Ph psi, Ph phi) {
        if (psi.m == 0 && phi.m == 0) {
            switch (kind) {
            case PZX_NODE: sc.mul(zw_add(zw(1, 0, 0, 0), zw_pow_w(psi.k))); break;
            case PZX_PHASE_PAIR: sc.mul(zw_pair_value(psi.k, phi.k)); break;
            case PZX_HALF_PI: sc.w(psi.k == 2 ? 1 : 7); break;
            case PZX_PI_PAIR: if (phi.k == 4) sc.w(psi.k); break;
            }
            return;
        }
        if (kind == PZX_NODE || kind == PZX_HALF_PI) phi = Ph{};
        subs.push_back(Sub{kind, psi.k, phi.k, psi.m, phi.m});
    }
    // e^{i phase}: w^k times (-1)^parity(mask) = PiPair((4, {}), (0, mask))
    void emit_exp(Ph p) {
        sc.w(p.k);
        if (p.m) subs.push_back(Sub{PZX_PI_PAIR, 4, 0, 0, p.m});
    }

    // ---- rules ----
    void lc(int u) {
        const Ph pu = ph[u];
        const std::vector<int> nb = adj[u];
        const int n = int(nb.size());
        remove_vertex(u);
        emit(PZX_HALF_PI, pu, Ph{});
        sc.sqrt2(1 - n);
        for (int i = 0; i < n; ++i) {
            ph[nb[i]] = ph_sub(ph[nb[i]], pu);
            for (int j = i + 1; j < n; ++j) toggle(nb[i], nb[j]);
        }
    }
    void pivot(int u, int v) {
        const Ph pu = ph[u], pv = ph[v];
        const int du = int(adj[u].size()), dv = int(adj[v].size());
        std::vector<int> U, V, W;
        for (int w : adj[u])
            if (w != v) U.push_back(w);
        for (int w : adj[v])
            if (w != u) V.push_back(w);
        std::sort(U.begin(), U.end());
        std::sort(V.begin(), V.end());
        std::vector<int> Up, Vp;
        std::set_intersection(U.begin(), U.end(), V.begin(), V.end(), std::back_inserter(W));
        std::set_difference(U.begin(), U.end(), W.begin(), W.end(), std::back_inserter(Up));
        std::set_difference(V.begin(), V.end(), W.begin(), W.end(), std::back_inserter(Vp));
        remove_vertex(u);
        remove_vertex(v);
        emit(PZX_PI_PAIR, pu, pv);
        sc.sqrt2(3 - du - dv);
        for (int w : Up) ph[w] = ph_add(ph[w], pv);
        for (int w : Vp) ph[w] = ph_add(ph[w], pu);
        for (int w : W) ph[w] = ph_add(ph_add(ph[w], ph_add(pu, pv)), ph_pi());
        for (int a : Up)
            for (int b : Vp) toggle(a, b);
        for (int a : Up)
            for (int b : W) toggle(a, b);
        for (int a : Vp)
            for (int b : W) toggle(a, b);
    }
    void copy(int u) {  // u: degree 1, Pauli
        const int v = adj[u][0];
        const Ph pu = ph[u], pv = ph[v];
        const int dv = int(adj[v].size());
        remove_vertex(u);
        std::vector<int> nb = adj[v];
        remove_vertex(v);
        emit(PZX_PI_PAIR, pv, pu);
        sc.sqrt2(1 - (dv - 1));
        for (int w : nb) ph[w] = ph_add(ph[w], pu);
    }

    // clifford_simp on the graph-like closed diagram; returns
    // false if the term vanished (a zero scalar)
    bool simp() {
        bool changed = true;
        while (changed && !sc.zero()) {
            changed = false;
            const int nv = int(ph.size());
            for (int u = 0; u < nv; ++u) {
                if (!alive[u]) continue;
                const size_t d = adj[u].size();
                if (d == 0) {  // isolated: 1 + e^{i psi}
                    remove_vertex(u);
                    emit(PZX_NODE, ph[u], Ph{});
                    changed = true;
                } else if (d == 1 && adj[adj[u][0]].size() == 1) {  // isolated edge
                    const int v = adj[u][0];
                    const Ph pu = ph[u], pv = ph[v];
                    remove_vertex(u);
                    remove_vertex(v);
                    emit(PZX_PHASE_PAIR, pu, pv);
                    sc.sqrt2(-1);
                    changed = true;
                } else if (d == 1 && is_pauli(ph[u])) {
                    copy(u);
                    changed = true;
                } else if (d == 2 && ph[u].k == 0 && ph[u].m == 0) {  // identity: neighbours fuse
                    const int a = adj[u][0], b = adj[u][1];
                    remove_vertex(u);
                    fuse(a, b);
                    changed = true;
                }
                if (sc.zero()) return false;
            }
            if (changed) continue;
            for (int u = 0; u < nv && !changed; ++u)
                if (alive[u] && is_proper(ph[u])) {
                    lc(u);
                    changed = true;
                }
            if (changed) continue;
            for (int u = 0; u < nv && !changed; ++u) {
                if (!alive[u] || !is_pauli(ph[u])) continue;
                for (int v : adj[u])
                    if (is_pauli(ph[v])) {
                        pivot(u, v);
                        changed = true;
                        break;
                    }
            }
        }
        return !sc.zero();
    }
    int tcount() const {
        int t = 0;
        for (size_t u = 0; u < ph.size(); ++u) t += alive[u] && is_tlike(ph[u]);
        return t;
    }
};

// ------------------------------------------------------------ circuits ----
struct Builder {
    Dg d;
    std::vector<int> f;        // frontier vertex per qubit
    std::vector<char> hpend;   // pending Hadamard between the frontier and the next spider
    // a Z spider on qubit q connected to the frontier by a plain wire
    int zvert(int q) {
        if (!hpend[q]) return f[q];
        const int v = d.add_vertex(Ph{});
        d.add_h(f[q], v);
        f[q] = v;
        hpend[q] = 0;
        return v;
    }
    // |b> = X-spider(pi b) / sqrt2 = Z(pi b) + Hadamard, / sqrt2
    void state(int q, Ph p) {
        f[q] = d.add_vertex(p);
        hpend[q] = 1;
        d.sc.sqrt2(-1);
    }
    void effect(int q, Ph p) {
        if (hpend[q]) {
            d.ph[f[q]] = ph_add(d.ph[f[q]], p);  // H . H = id: fuse into the frontier
        } else {
            const int v = d.add_vertex(p);
            d.add_h(f[q], v);
        }
        d.sc.sqrt2(-1);
    }
    void phase(int q, int k) {
        const int v = zvert(q);
        d.ph[v] = ph_add(d.ph[v], Ph{uint8_t(k & 7), 0});
    }
    void gate(const pzx_gate& g) {
        const int a = g.q0, b = g.q1;
        switch (g.op) {
        case PZX_G_H: hpend[a] ^= 1; break;
        case PZX_G_Z: phase(a, 4); break;
        case PZX_G_S: phase(a, 2); break;
        case PZX_G_SDG: phase(a, 6); break;
        case PZX_G_T: phase(a, 1); break;
        case PZX_G_TDG: phase(a, 7); break;
        case PZX_G_RZ: phase(a, g.k); break;
        case PZX_G_X: hpend[a] ^= 1; phase(a, 4); hpend[a] ^= 1; break;
        case PZX_G_CZ: {  // CZ = sqrt2 * (Z -H- Z)
            const int u = zvert(a), v = zvert(b);
            d.add_h(u, v);
            d.sc.sqrt2(1);
            break;
        }
        case PZX_G_CNOT: {  // CNOT = sqrt2 * (Z on the control -- X on the target)
            const int u = zvert(a);
            hpend[b] ^= 1;  // the X spider is a Z spider with Hadamards on its legs
            const int v = zvert(b);
            hpend[b] ^= 1;
            d.add_h(u, v);
            d.sc.sqrt2(1);
            break;
        }
        }
    }
};

bool valid_gate(const pzx_gate& g, uint32_t n) {
    if (g.op > PZX_G_RZ || g.q0 >= n) return false;
    if ((g.op == PZX_G_CNOT || g.op == PZX_G_CZ) && (g.q1 >= n || g.q1 == g.q0)) return false;
    return true;
}

pzx_gate adjoint(pzx_gate g) {
    switch (g.op) {
    case PZX_G_S: g.op = PZX_G_SDG; break;
    case PZX_G_SDG: g.op = PZX_G_S; break;
    case PZX_G_T: g.op = PZX_G_TDG; break;
    case PZX_G_TDG: g.op = PZX_G_T; break;
    case PZX_G_RZ: g.k = uint8_t((8 - g.k) & 7); break;
    default: break;
    }
    return g;
}

Ph spec_phase(int32_t s) {  // 0 / 1 fixed bit, 2 + p parameter p
    if (s == 0) return Ph{0, 0};
    if (s == 1) return Ph{4, 0};
    return Ph{0, uint64_t(1) << (s - 2)};
}

// ---------------------------------------------------------- expressions ----
// exact sum of leaf scalars (parameter-free reductions: the non-parametric
// path needs only the value), value = sum_i c_i w^i * 2^e
struct ExactSum {
    i128 c[4] = {0, 0, 0, 0};
    int e = 0;
    bool any = false, ok = true;
    static bool shl(i128& v, int s) {
        for (; s > 0; --s) {
            if (v > (i128(1) << 120) || v < -(i128(1) << 120)) return false;
            v *= 2;
        }
        return true;
    }
    void add(const Scalar& x) {
        if (x.num.zero()) return;
        Zw n = x.num;
        int s2 = x.s2;
        if (s2 & 1) { n = zw_mul(n, zw(0, 1, 0, -1)); s2 -= 1; }
        const int h = s2 / 2;
        i128 v[4] = {n.c[0], n.c[1], n.c[2], n.c[3]};
        if (!any) { for (int i = 0; i < 4; ++i) c[i] = v[i]; e = h; any = true; return; }
        if (h < e) {
            for (int i = 0; i < 4; ++i) ok = ok && shl(c[i], e - h);
            e = h;
        }
        for (int i = 0; i < 4; ++i) {
            ok = ok && shl(v[i], h - e);
            c[i] += v[i];
        }
    }
    void merge(const ExactSum& o) {
        if (!o.any) return;
        ok = ok && o.ok;
        Scalar tmp;  // add o term by term at its own exponent
        if (!any) { *this = o; return; }
        const int h = o.e;
        i128 v[4] = {o.c[0], o.c[1], o.c[2], o.c[3]};
        if (h < e) {
            for (int i = 0; i < 4; ++i) ok = ok && shl(c[i], e - h);
            e = h;
        }
        for (int i = 0; i < 4; ++i) {
            ok = ok && shl(v[i], h - e);
            c[i] += v[i];
        }
        (void)tmp;
    }
    // (c0 + c1 w + c2 w^2 + c3 w^3) 2^e = (2c0 + (c1 - c3) sqrt2 + i(2c2 + (c1 + c3) sqrt2)) / 2^(1 - e)
    bool to_quad(Quad& q) const {
        if (!any) { q = Quad{}; return true; }
        return ok && quad_canon(2 * c[0], c[1] - c[3], 2 * c[2], c[1] + c[3], int64_t(1) - e, q);
    }
};

}  // namespace

struct pzx_expr {
    uint32_t n_params = 0;
    std::vector<uint64_t> off{0};
    std::vector<int64_t> scal;
    std::vector<uint8_t> kind, psi_k, phi_k;
    std::vector<uint64_t> psi_m, phi_m;
    uint32_t t_count = 0, t_after_simp = 0;
    double seconds = 0;
    std::string err;
    bool sum_only = false;  // no parameters: leaves are summed into one exact scalar
    ExactSum total;
};

namespace {

struct Leafs {
    std::vector<Dg> out;
};

// depth-first decomposition of one diagram into leaves (closed, spider-free)
int decompose(Dg d, pzx_expr& ex, uint64_t cap, std::string& err) {
    std::vector<Dg> stack;
    stack.push_back(std::move(d));
    while (!stack.empty()) {
        Dg g = std::move(stack.back());
        stack.pop_back();
        if (!g.simp()) continue;
        if (!g.sc.ok) { err = "scalar out of int64"; return PZX_E_OVERFLOW; }
        if (g.n_alive == 0) {
            if (ex.sum_only) {
                ex.total.add(g.sc);
                if (!ex.total.ok) { err = "leaf sum out of range"; return PZX_E_OVERFLOW; }
                continue;
            }
            Quad q;
            if (!g.sc.to_quad(q)) { err = "leaf scalar out of RingQuad range"; return PZX_E_OVERFLOW; }
            if (q.a == 0 && q.b == 0 && q.c == 0 && q.d == 0) continue;
            const int64_t s[5] = {q.a, q.b, q.c, q.d, q.e};
            ex.scal.insert(ex.scal.end(), s, s + 5);
            for (const Sub& s2 : g.subs) {
                ex.kind.push_back(s2.kind);
                ex.psi_k.push_back(s2.psi_k);
                ex.phi_k.push_back(s2.phi_k);
                ex.psi_m.push_back(s2.psi_m);
                ex.phi_m.push_back(s2.phi_m);
            }
            ex.off.push_back(ex.kind.size());
            if (ex.off.size() - 1 > cap) { err = "term cap exceeded"; return PZX_E_CAPACITY; }
            continue;
        }
        int u = -1, v = -1;
        for (size_t i = 0; i < g.ph.size() && v < 0; ++i)
            if (g.alive[i] && is_tlike(g.ph[i])) (u < 0 ? u : v) = int(i);
        if (u < 0) { err = "simplification left a Clifford diagram unreduced"; return PZX_E_DOMAIN; }
        if (v >= 0) {  // T-pair: [x = y] + [y = 1 - x]
            Dg b = g;
            b.flip_fuse(u, v);
            g.fuse(u, v);
            stack.push_back(std::move(b));
            stack.push_back(std::move(g));
        } else {       // single T: x = 0 | x = 1
            Dg b = g;
            const Ph pu = g.ph[u];
            std::vector<int> nb = g.adj[u];
            g.remove_vertex(u);
            g.sc.sqrt2(-int(nb.size()));
            b.remove_vertex(u);
            b.sc.sqrt2(-int(nb.size()));
            b.emit_exp(pu);
            for (int w : nb) b.ph[w] = ph_add(b.ph[w], ph_pi());
            stack.push_back(std::move(b));
            stack.push_back(std::move(g));
        }
    }
    return PZX_OK;
}

// Split the decomposition tree at a fixed depth into independent subtrees and
// reduce them on host threads (SPEC decomposer concurrency: sibling branches
// are independent); the leaves are concatenated in DFS order, so the output is
// identical to the serial one.
int decompose_parallel(Dg root, pzx_expr& ex, uint64_t cap, std::string& err) {
    std::vector<Dg> frontier{std::move(root)}, leaves_done;
    // expand breadth-first to ~4x the host threads
    const unsigned nth = std::max(1u, std::thread::hardware_concurrency());
    std::vector<Dg> work;
    for (int depth = 0; depth < 12 && frontier.size() < 4 * nth; ++depth) {
        std::vector<Dg> next;
        bool any = false;
        for (Dg& g : frontier) {
            if (!g.simp()) continue;
            int u = -1, v = -1;
            for (size_t i = 0; i < g.ph.size() && v < 0; ++i)
                if (g.alive[i] && is_tlike(g.ph[i])) (u < 0 ? u : v) = int(i);
            if (u < 0) { next.push_back(std::move(g)); continue; }
            any = true;
            Dg b = g;
            if (v >= 0) {
                g.fuse(u, v);
                b.flip_fuse(u, v);
            } else {
                const Ph pu = g.ph[u];
                std::vector<int> nb = g.adj[u];
                g.remove_vertex(u);
                g.sc.sqrt2(-int(nb.size()));
                b.remove_vertex(u);
                b.sc.sqrt2(-int(nb.size()));
                b.emit_exp(pu);
                for (int w : nb) b.ph[w] = ph_add(b.ph[w], ph_pi());
            }
            next.push_back(std::move(g));
            next.push_back(std::move(b));
        }
        frontier.swap(next);
        if (!any) break;
    }
    const size_t nw = frontier.size();
    std::vector<pzx_expr> parts(nw);
    for (auto& p : parts) p.sum_only = ex.sum_only;
    std::vector<int> st(nw, PZX_OK);
    std::vector<std::string> errs(nw);
    std::atomic<size_t> next_job{0};
    auto run = [&] {
        for (;;) {
            const size_t j = next_job.fetch_add(1);
            if (j >= nw) return;
            st[j] = decompose(std::move(frontier[j]), parts[j], cap, errs[j]);
        }
    };
    std::vector<std::thread> th;
    for (unsigned i = 1; i < std::min<size_t>(nth, nw); ++i) th.emplace_back(run);
    run();
    for (auto& t : th) t.join();
    for (size_t j = 0; j < nw; ++j) {
        if (st[j]) { err = errs[j]; return st[j]; }
        if (ex.sum_only) {
            ex.total.merge(parts[j].total);
            if (!ex.total.ok) { err = "leaf sum out of range"; return PZX_E_OVERFLOW; }
            continue;
        }
        const uint64_t base = ex.kind.size();
        for (size_t i = 1; i < parts[j].off.size(); ++i) ex.off.push_back(base + parts[j].off[i]);
        auto app = [](auto& dst, const auto& src) { dst.insert(dst.end(), src.begin(), src.end()); };
        app(ex.scal, parts[j].scal);
        app(ex.kind, parts[j].kind);
        app(ex.psi_k, parts[j].psi_k);
        app(ex.phi_k, parts[j].phi_k);
        app(ex.psi_m, parts[j].psi_m);
        app(ex.phi_m, parts[j].phi_m);
        if (ex.off.size() - 1 > cap) { err = "term cap exceeded"; return PZX_E_CAPACITY; }
    }
    return PZX_OK;
}

}  // namespace

extern "C" {

pzx_status pzx_circuit_reduce(uint32_t n_qubits, const pzx_gate* gates, uint64_t n_gates, const int32_t* in_spec,
                              const int32_t* out_spec, uint32_t mode, uint64_t max_terms, pzx_expr** out) {
    if (!out || (n_gates && !gates) || !out_spec || n_qubits == 0 || n_qubits > 4096) return PZX_E_INVALID;
    nvtxRangePushA("pzx.circuit_reduce");
    struct Pop { ~Pop() { nvtxRangePop(); } } pop_at_exit;
    *out = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    std::unique_ptr<pzx_expr> ex(new (std::nothrow) pzx_expr);
    if (!ex) return PZX_E_OOM;
    uint32_t np = 0;
    for (uint32_t q = 0; q < n_qubits; ++q) {
        const int32_t s = out_spec[q];
        const int32_t si = in_spec ? in_spec[q] : 0;
        if (s < -1 || (s == -1 && mode != PZX_REDUCE_DOUBLED) || s > 2 + 63 || si < 0 || si > 2 + 63)
            return PZX_E_INVALID;
        if (s >= 2) np = std::max<uint32_t>(np, uint32_t(s - 1));
        if (si >= 2) np = std::max<uint32_t>(np, uint32_t(si - 1));
    }
    for (uint64_t i = 0; i < n_gates; ++i)
        if (!valid_gate(gates[i], n_qubits)) return PZX_E_PARSE;
    ex->n_params = np;
    Builder B;
    B.f.assign(n_qubits, -1);
    B.hpend.assign(n_qubits, 0);
    for (uint32_t q = 0; q < n_qubits; ++q) B.state(int(q), spec_phase(in_spec ? in_spec[q] : 0));
    uint32_t t = 0;
    auto count_t = [&](const pzx_gate& g) {
        t += g.op == PZX_G_T || g.op == PZX_G_TDG || (g.op == PZX_G_RZ && (g.k & 1));
    };
    for (uint64_t i = 0; i < n_gates; ++i) {
        B.gate(gates[i]);
        count_t(gates[i]);
    }
    if (mode == PZX_REDUCE_DOUBLED) {
        // U^dag (|a><a| (x) I) U with |0...0> inputs on both copies (SPEC double_diagram,
        // S:76-84; PAPER Fig. 3): measured wires get <a| then |a>, traced wires
        // run straight into the adjoint copy; parameters shared by both copies
        for (uint32_t q = 0; q < n_qubits; ++q)
            if (out_spec[q] >= 0) {
                B.effect(int(q), spec_phase(out_spec[q]));
                B.state(int(q), spec_phase(out_spec[q]));
            }
        for (uint64_t i = n_gates; i-- > 0;) {
            B.gate(adjoint(gates[i]));
            count_t(gates[i]);
        }
        for (uint32_t q = 0; q < n_qubits; ++q) B.effect(int(q), spec_phase(in_spec ? in_spec[q] : 0));
    } else {
        for (uint32_t q = 0; q < n_qubits; ++q) B.effect(int(q), spec_phase(out_spec[q]));
    }
    ex->t_count = t;
    Dg d = std::move(B.d);
    int st;
    if (!d.simp()) {
        st = PZX_OK;  // the whole value is 0: the empty expression
    } else {
        ex->t_after_simp = uint32_t(d.tcount());
        ex->sum_only = np == 0;
        st = decompose_parallel(std::move(d), *ex, max_terms ? max_terms : (uint64_t(1) << 26), ex->err);
    }
    if (st) return pzx_status(st);
    if (ex->sum_only && ex->total.any) {  // one constant term: the exact value
        Quad q;
        if (!ex->total.to_quad(q)) return PZX_E_OVERFLOW;
        if (q.a || q.b || q.c || q.d) {
            const int64_t v[5] = {q.a, q.b, q.c, q.d, q.e};
            ex->scal.assign(v, v + 5);
            ex->off.assign({0, 0});
        }
    }
    ex->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = ex.release();
    return PZX_OK;
}

pzx_status pzx_expr_get_view(const pzx_expr* e, pzx_expr_view* v) {
    if (!e || !v) return PZX_E_INVALID;
    v->n_params = e->n_params;
    v->n_terms = e->off.size() - 1;
    v->term_offset = e->off.data();
    v->term_scalar = e->scal.data();
    v->kind = e->kind.data();
    v->psi_k = e->psi_k.data();
    v->psi_mask = e->psi_m.data();
    v->phi_k = e->phi_k.data();
    v->phi_mask = e->phi_m.data();
    return PZX_OK;
}

pzx_status pzx_expr_info(const pzx_expr* e, uint32_t* t_count, uint32_t* t_after_simp, double* seconds) {
    if (!e) return PZX_E_INVALID;
    if (t_count) *t_count = e->t_count;
    if (t_after_simp) *t_after_simp = e->t_after_simp;
    if (seconds) *seconds = e->seconds;
    return PZX_OK;
}

void pzx_expr_free(pzx_expr* e) { delete e; }

}  // extern "C"
