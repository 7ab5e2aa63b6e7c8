// fg_oracle.cpp — TEST INFRASTRUCTURE ONLY: a CPU restatement of the
// reference's hot path (/root/reference/proj/src), used as a checker by
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.  It is
// never linked into, loaded by, or called from the product library.
//
// Every function cites the reference lines it restates.  Pinned: tests/
// compare it bit-for-bit with the unmodified reference (oracle/_ref) and with
// the golden fixtures in tests/golden/.
//
// Arithmetic: fp32 storage, fp64 accumulation in the reference's order, no FP
// contraction (built with -ffp-contract=off, like the reference's baseline
// x86-64 build), so sums round identically.

#include <algorithm>
#include <array>
#include <tuple>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "fg_b200.h"

namespace {

thread_local std::string g_err;

struct Fail : std::runtime_error {
    explicit Fail(const std::string& code, const std::string& msg)
        : std::runtime_error(code + ": " + msg) {}
};

template <typename F>
int run(F&& f) {
    try {
        f();
        g_err.clear();
        return FG_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FG_ERR;
    }
}

struct Sparse {  // one row view
    const uint32_t* idx = nullptr;
    const float* val = nullptr;
    uint64_t n = 0;
};

// ---------------------------------------------------------------- corpus
struct Store {
    uint64_t n = 0;
    uint32_t dim = 0;
    std::vector<float> dense;
    std::vector<uint64_t> lp, sp, kp, ep;
    std::vector<uint32_t> li, si, ki, ei;
    std::vector<float> lv, sv;
    std::vector<uint64_t> doc_id;
    std::vector<uint8_t> deleted;
    std::vector<double> sqnorm;
    std::vector<uint32_t> ts, tr, tt;  // KG triplets (sorted unique)
    std::vector<std::vector<std::pair<uint32_t, uint32_t>>> adj;

    Sparse learned(uint64_t i) const { return {li.data() + lp[i], lv.data() + lp[i], lp[i + 1] - lp[i]}; }
    Sparse stat(uint64_t i) const { return {si.data() + sp[i], sv.data() + sp[i], sp[i + 1] - sp[i]}; }
    const float* row(uint64_t i) const { return dense.data() + i * dim; }
    const uint32_t* kw_b(uint64_t i) const { return ki.data() + kp[i]; }
    const uint32_t* kw_e(uint64_t i) const { return ki.data() + kp[i + 1]; }
    const uint32_t* en_b(uint64_t i) const { return ei.data() + ep[i]; }
    const uint32_t* en_e(uint64_t i) const { return ei.data() + ep[i + 1]; }
    const std::vector<std::pair<uint32_t, uint32_t>>& nbrs(uint32_t e) const {
        static const std::vector<std::pair<uint32_t, uint32_t>> none;
        return e < adj.size() ? adj[e] : none;
    }
    bool has_relation(uint32_t a, uint32_t b) const {  // types.cpp:52-57
        const auto& l = nbrs(a);
        auto it = std::lower_bound(l.begin(), l.end(), std::make_pair(b, 0u));
        return it != l.end() && it->first == b;
    }
};

// scoring.cpp:10-18 — dense dot, index order, fp64 accumulate
double dot_dense(const float* a, const float* b, uint32_t d) {
    double s = 0.0;
    for (uint32_t i = 0; i < d; ++i) s += static_cast<double>(a[i]) * static_cast<double>(b[i]);
    return s;
}

// scoring.cpp:24-74 — shared indices in ascending order (merge == probe order)
double dot_sparse(const Sparse& a, const Sparse& b) {
    if (a.n == 0 || b.n == 0) return 0.0;
    double s = 0.0;
    uint64_t i = 0, j = 0;
    while (i < a.n && j < b.n) {
        if (a.idx[i] < b.idx[j]) {
            ++i;
        } else if (b.idx[j] < a.idx[i]) {
            ++j;
        } else {
            s += static_cast<double>(a.val[i]) * static_cast<double>(b.val[j]);
            ++i;
            ++j;
        }
    }
    return s;
}

// A weighted query vector (corpus.cpp:86-103).
struct QVec {
    std::vector<float> dense;
    std::vector<uint32_t> li, si;
    std::vector<float> lv, sv;
    double sqnorm = 0.0;
    Sparse learned() const { return {li.data(), lv.data(), li.size()}; }
    Sparse stat() const { return {si.data(), sv.data(), si.size()}; }
};

// scoring.cpp:88-99 — dense, then learned, then statistical
double score(const Store& s, const float* qd, uint32_t qdim, const Sparse& ql, const Sparse& qs,
             uint64_t doc) {
    if (qdim != s.dim)
        throw Fail("dim-mismatch", "dense dimensions differ: " + std::to_string(qdim) + " vs " +
                                       std::to_string(s.dim));
    double acc = dot_dense(qd, s.row(doc), s.dim);
    acc += dot_sparse(ql, s.learned(doc));
    acc += dot_sparse(qs, s.stat(doc));
    return acc;
}
double pair(const Store& s, uint64_t a, uint64_t b) {
    return score(s, s.row(a), s.dim, s.learned(a), s.stat(a), b);
}

void check_weights(const fg_weights& w) {  // types.cpp:10-18
    const float p[4] = {w.dense, w.learned, w.statistical, w.entity};
    for (float x : p)
        if (!std::isfinite(x) || x < 0.0f) throw Fail("invalid-weights", "weights must be finite and non-negative");
    if (w.dense <= 0.0f && w.learned <= 0.0f && w.statistical <= 0.0f)
        throw Fail("invalid-weights", "at least one vector-path weight must be positive");
}

fg_weights weights_of(const fg_query_view& q, uint64_t i) {
    return q.weights ? q.weights[i] : fg_weights{1.f, 1.f, 1.f, 0.f};
}

QVec weighted(const fg_query_view& q, uint64_t i) {  // corpus.cpp:86-103
    const fg_weights w = weights_of(q, i);
    QVec v;
    const float* x = q.dense + i * q.dense_dim;
    for (uint32_t j = 0; j < q.dense_dim; ++j) v.dense.push_back(w.dense * x[j]);
    auto scale = [&](const fg_sparse_view& sv, float wt, std::vector<uint32_t>& oi, std::vector<float>& ov) {
        if (!sv.ptr || wt == 0.0f) return;
        for (uint64_t j = sv.ptr[i]; j < sv.ptr[i + 1]; ++j) {
            oi.push_back(sv.idx[j]);
            ov.push_back(wt * sv.val[j]);
        }
    };
    scale(q.learned, w.learned, v.li, v.lv);
    scale(q.statistical, w.statistical, v.si, v.sv);
    double acc = dot_dense(v.dense.data(), v.dense.data(), static_cast<uint32_t>(v.dense.size()));
    acc += dot_sparse(v.learned(), v.learned());
    acc += dot_sparse(v.stat(), v.stat());
    v.sqnorm = acc;
    return v;
}

// ---------------------------------------------------------------- rng.hpp:17-41
struct Mix {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
};
uint64_t seed_for(uint64_t seed, uint64_t stream) {
    Mix m{seed ^ (0xA0761D6478BD642FULL * (stream + 1))};
    return m.next();
}
uint64_t draw(Mix& m, uint64_t bound) {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(m.next()) * bound) >> 64);
}

// ---------------------------------------------------------------- k-NN graph
struct Entry {
    uint32_t id;
    double sc;
    bool fresh;
};
bool better(const Entry& a, const Entry& b) {  // knn_graph.cpp:15-18
    return a.sc != b.sc ? a.sc > b.sc : a.id < b.id;
}
using Lists = std::vector<std::vector<Entry>>;

Lists knn_init(const Store& s, uint32_t k, uint64_t seed) {  // knn_graph.cpp:26-73
    const uint64_t n = s.n;
    if (k == 0) throw Fail("invalid-k", "neighbour count must be positive");
    if (n < static_cast<uint64_t>(k) + 1)
        throw Fail("corpus-too-small", "need at least " + std::to_string(k + 1) + " documents for k=" + std::to_string(k));
    Lists L(n);
    for (uint64_t u = 0; u < n; ++u) {
        Mix rng{seed_for(seed, u)};
        std::vector<uint32_t> pick;
        if (static_cast<uint64_t>(k) * 4 < n) {
            while (pick.size() < k) {
                const auto c = static_cast<uint32_t>(draw(rng, n));
                if (c == u || std::count(pick.begin(), pick.end(), c)) continue;
                pick.push_back(c);
            }
        } else {
            std::vector<uint32_t> all;
            for (uint32_t i = 0; i < n; ++i)
                if (i != u) all.push_back(i);
            for (uint32_t i = 0; i < k; ++i) {
                std::swap(all[i], all[i + draw(rng, all.size() - i)]);
                pick.push_back(all[i]);
            }
        }
        for (uint32_t v : pick) L[u].push_back({v, pair(s, u, v), true});
        std::sort(L[u].begin(), L[u].end(), better);
    }
    return L;
}

// knn_graph.cpp:75-148 restricted to nodes [lo, hi): rows outside the range
// of `L` are left as they are (the test harness of the vertex-range sharded
// build gathers the ranges; the pass is double-buffered, so the union of the
// ranges equals the full pass).
uint64_t knn_pass_range(const Store& s, Lists& L, uint32_t k, uint64_t lo, uint64_t hi);

uint64_t knn_pass(const Store& s, Lists& L, uint32_t k) { return knn_pass_range(s, L, k, 0, L.size()); }

uint64_t knn_pass_range(const Store& s, Lists& L, uint32_t k, uint64_t lo, uint64_t hi) {
    const uint64_t n = L.size();
    Lists R(n);
    for (uint64_t u = 0; u < n; ++u)
        for (const Entry& e : L[u]) R[e.id].push_back({static_cast<uint32_t>(u), e.sc, e.fresh});
    for (auto& r : R) {
        std::sort(r.begin(), r.end(), better);
        if (r.size() > k) r.resize(k);
    }
    Lists next = L;
    uint64_t replaced = 0;
    for (uint64_t u = lo; u < hi; ++u) {
        std::map<uint32_t, bool> pool;  // candidate -> some path fresh
        auto via = [&](const Entry& h1) {
            for (const auto* side : {&L[h1.id], &R[h1.id]})
                for (const Entry& h2 : *side) {
                    if (h2.id == u) continue;
                    pool[h2.id] = pool[h2.id] || h1.fresh || h2.fresh;
                }
        };
        for (const Entry& e : L[u]) via(e);
        for (const Entry& e : R[u]) via(e);
        std::vector<uint32_t> have;
        for (const Entry& e : L[u]) have.push_back(e.id);
        std::sort(have.begin(), have.end());
        std::vector<Entry> m = L[u];
        for (Entry& e : m) e.fresh = false;
        for (const auto& [c, fresh] : pool)
            if (fresh && !std::binary_search(have.begin(), have.end(), c)) m.push_back({c, pair(s, u, c), true});
        std::sort(m.begin(), m.end(), better);
        if (m.size() > k) m.resize(k);
        for (const Entry& e : m) replaced += !std::binary_search(have.begin(), have.end(), e.id);
        next[u] = std::move(m);
    }
    L = std::move(next);
    return replaced;
}

Lists knn_build(const Store& s, uint32_t k, uint32_t iters, double conv, uint64_t seed) {  // :150-166
    if (s.n >= 2 && k >= s.n) k = static_cast<uint32_t>(s.n - 1);
    Lists L = knn_init(s, k, seed);
    for (uint32_t it = 0; it < iters; ++it) {
        const uint64_t ch = knn_pass(s, L, k);
        if (static_cast<double>(ch) / (static_cast<double>(s.n) * k) < conv) break;
    }
    return L;
}

// ---------------------------------------------------------------- refinery
struct Refined {
    std::vector<std::vector<uint32_t>> semantic, keyword, kept, ordered;
    std::vector<std::vector<double>> ordered_sc;
    std::vector<std::vector<uint32_t>> detours;
};

bool sorted_has(const uint32_t* b, const uint32_t* e, uint32_t x) { return std::binary_search(b, e, x); }

Refined refine(const Store& s, const Lists& L, uint32_t degree, bool per_nb) {  // refine.cpp:167-217
    const uint64_t n = L.size();
    Refined R;
    R.semantic.resize(n);
    R.keyword.resize(n);
    R.kept.resize(n);
    R.ordered.resize(n);
    R.ordered_sc.resize(n);
    R.detours.resize(n);
    for (uint64_t u = 0; u < n; ++u) {
        const auto& c = L[u];
        const size_t k = c.size();
        std::vector<double> P(k * k, 0.0);  // refine.cpp:11-23
        for (size_t i = 0; i < k; ++i)
            for (size_t j = i + 1; j < k; ++j) P[i * k + j] = P[j * k + i] = pair(s, c[i].id, c[j].id);
        std::vector<uint32_t> det(k, 0);  // refine.cpp:25-39 (strict <)
        for (size_t v = 0; v < k; ++v)
            for (size_t x = 0; x < k; ++x)
                if (x != v && std::max(-c[x].sc, -P[x * k + v]) < -c[v].sc) ++det[v];
        std::vector<size_t> ord(k);  // refine.cpp:41-65
        std::iota(ord.begin(), ord.end(), 0);
        std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) {
            if (det[a] != det[b]) return det[a] < det[b];
            if (c[a].sc != c[b].sc) return c[a].sc > c[b].sc;
            return c[a].id < c[b].id;
        });
        for (size_t r = 0; r < k; ++r) {
            R.ordered[u].push_back(c[ord[r]].id);
            R.ordered_sc[u].push_back(c[ord[r]].sc);
            R.detours[u].push_back(det[ord[r]]);
        }
        if (k == 0) continue;
        // refine.cpp:67-118 — prune walk + keyword recycling
        std::vector<size_t> keptp{0};
        for (size_t r = 1; r < k; ++r) {
            const uint32_t vid = c[ord[r]].id;
            const double self = s.sqnorm[vid];
            size_t pruner = k;
            for (size_t w : keptp)
                if (P[ord[w] * k + ord[r]] >= self) {
                    pruner = w;
                    break;
                }
            if (pruner == k && keptp.size() < degree) {
                keptp.push_back(r);
                continue;
            }
            std::vector<uint32_t> shared;
            std::set_intersection(s.kw_b(u), s.kw_e(u), s.kw_b(vid), s.kw_e(vid), std::back_inserter(shared));
            if (shared.empty()) continue;
            bool covered = true;
            for (uint32_t t : shared) {
                bool hit = false;
                if (per_nb && pruner != k) {
                    const uint32_t pid = c[ord[pruner]].id;
                    hit = sorted_has(s.kw_b(pid), s.kw_e(pid), t);
                } else {
                    for (size_t w : keptp) {
                        const uint32_t wid = c[ord[w]].id;
                        if (sorted_has(s.kw_b(wid), s.kw_e(wid), t)) {
                            hit = true;
                            break;
                        }
                    }
                }
                if (!hit) {
                    covered = false;
                    break;
                }
            }
            if (!covered) R.keyword[u].push_back(vid);
        }
        for (size_t w : keptp) R.kept[u].push_back(c[ord[w]].id);
    }
    // refine.cpp:123-163 — merge with reverse keepers
    std::vector<std::vector<std::pair<uint32_t, uint32_t>>> keepers(n);
    for (uint64_t w = 0; w < n; ++w)
        for (size_t p = 0; p < R.kept[w].size(); ++p)
            keepers[R.kept[w][p]].push_back({static_cast<uint32_t>(p), static_cast<uint32_t>(w)});
    const uint32_t half = degree / 2;
    for (uint64_t u = 0; u < n; ++u) {
        auto& out = R.semantic[u];
        auto has = [&](uint32_t x) { return std::find(out.begin(), out.end(), x) != out.end(); };
        const size_t fwd = std::min<size_t>(half, R.kept[u].size());
        out.assign(R.kept[u].begin(), R.kept[u].begin() + fwd);
        std::sort(keepers[u].begin(), keepers[u].end());
        for (const auto& [p, w] : keepers[u]) {
            if (out.size() >= fwd + half) break;
            if (!has(w)) out.push_back(w);
        }
        for (size_t i = fwd; i < R.kept[u].size() && out.size() < degree; ++i)
            if (!has(R.kept[u][i])) out.push_back(R.kept[u][i]);
        for (uint32_t x : R.ordered[u]) {
            if (out.size() >= degree) break;
            if (!has(x)) out.push_back(x);
        }
        auto& kw = R.keyword[u];  // refine.cpp:207-215
        kw.erase(std::remove_if(kw.begin(), kw.end(), has), kw.end());
    }
    return R;
}

// ---------------------------------------------------------------- index
struct Index {
    Store* s = nullptr;
    std::unique_ptr<Store> own;
    uint32_t degree = 0;
    std::vector<std::vector<uint32_t>> semantic, keyword;
    std::vector<std::vector<std::array<uint32_t, 4>>> logical;  // (source, relation, target, via)
    std::map<uint32_t, std::vector<uint32_t>> emap;
    std::vector<uint32_t> norm_order;
};

void finish_index(Index& x, bool derive_logical, uint32_t cap) {
    const Store& s = *x.s;
    x.emap.clear();  // logical.cpp:9-15
    for (uint64_t u = 0; u < s.n; ++u)
        for (const uint32_t* e = s.en_b(u); e != s.en_e(u); ++e) x.emap[*e].push_back(static_cast<uint32_t>(u));
    if (derive_logical) {  // logical.cpp:17-55
        x.logical.assign(s.n, {});
        for (uint64_t u = 0; u < s.n; ++u) {
            for (const uint32_t* sp = s.en_b(u); sp != s.en_e(u); ++sp) {
                std::vector<std::array<uint32_t, 4>> g;
                long prev = -1;
                for (const auto& [t, r] : s.nbrs(*sp)) {
                    if (static_cast<long>(t) == prev) continue;
                    prev = t;
                    if (sorted_has(s.en_b(u), s.en_e(u), t)) continue;
                    auto it = x.emap.find(t);
                    if (it == x.emap.end()) continue;
                    for (uint32_t v : it->second)
                        if (v != u) g.push_back({*sp, r, t, v});
                }
                std::stable_sort(g.begin(), g.end(), [&](const auto& a, const auto& b) {
                    const size_t da = s.nbrs(a[2]).size(), db = s.nbrs(b[2]).size();
                    if (da != db) return da > db;
                    if (a[2] != b[2]) return a[2] < b[2];
                    return a[3] < b[3];
                });
                if (g.size() > cap) g.resize(cap);
                x.logical[u].insert(x.logical[u].end(), g.begin(), g.end());
            }
        }
    }
    if (x.norm_order.size() != s.n) {  // index.cpp:12-23
        x.norm_order.resize(s.n);
        std::iota(x.norm_order.begin(), x.norm_order.end(), 0u);
        std::sort(x.norm_order.begin(), x.norm_order.end(), [&](uint32_t a, uint32_t b) {
            return s.sqnorm[a] != s.sqnorm[b] ? s.sqnorm[a] > s.sqnorm[b] : a < b;
        });
    }
}

// ---------------------------------------------------------------- search
struct PE {
    double d;
    uint32_t node;
};
bool pe_less(const PE& a, const PE& b) { return a.d != b.d ? a.d < b.d : a.node < b.node; }

struct SortedPool {  // search.cpp:19-54
    size_t cap;
    std::vector<PE> v;
    long offer(PE e) {
        auto it = std::find_if(v.begin(), v.end(), [&](const PE& x) { return x.node == e.node; });
        if (it != v.end()) {
            if (!pe_less(e, *it)) return -1;
            v.erase(it);
        } else if (v.size() == cap && !pe_less(e, v.back())) {
            return -1;
        }
        v.insert(std::upper_bound(v.begin(), v.end(), e, pe_less), e);
        if (v.size() > cap) {
            const long ev = v.back().node;
            v.pop_back();
            return ev;
        }
        return -1;
    }
};

struct NodeSt {
    double raw = 0;
    uint32_t ent = 0, hop = 0;
    bool ctx = false, scored = false, expanded = false;
};

void search_one(const Index& x, const fg_query_view& q, uint64_t qi, const fg_search_opts& o,
                std::vector<PE>& hits, uint32_t& warn, uint64_t& expanded) {
    const Store& s = *x.s;
    const fg_weights w = weights_of(q, qi);
    const uint32_t K = q.k ? q.k[qi] : 10, B = q.beam_width ? q.beam_width[qi] : 64;
    const uint32_t H = q.max_entity_hops ? q.max_entity_hops[qi] : 2;
    std::vector<uint32_t> req, ents;
    if (q.required_keywords.ptr)
        req.assign(q.required_keywords.idx + q.required_keywords.ptr[qi], q.required_keywords.idx + q.required_keywords.ptr[qi + 1]);
    if (q.entities.ptr) ents.assign(q.entities.idx + q.entities.ptr[qi], q.entities.idx + q.entities.ptr[qi + 1]);
    check_weights(w);  // types.cpp:20-27
    if (K == 0) throw Fail("invalid-k", "k must be positive");
    if (B < K) throw Fail("beam-too-small", "beam_width must be at least k");
    if (w.entity > 0.0f && ents.empty()) throw Fail("entities-required", "entity weight is positive but the query names no entities");
    const QVec qv = weighted(q, qi);
    const double we = w.entity;
    std::vector<NodeSt> st(s.n);
    SortedPool cand{B, {}}, top{K, {}};
    std::vector<uint32_t> twin;
    std::vector<bool> in_twin(s.n, false);
    auto adj = [&](uint32_t v) { return (st[v].ctx && st[v].hop >= 1) ? st[v].raw - we / static_cast<double>(st[v].hop) : st[v].raw; };
    auto shares = [&](uint32_t v) {
        for (uint32_t t : req)
            if (sorted_has(s.kw_b(v), s.kw_e(v), t)) return true;
        return false;
    };
    auto offer = [&](uint32_t v) {  // search.cpp:171-181
        const PE e{adj(v), v};
        cand.offer(e);
        if (s.deleted[v]) return;
        const long ev = top.offer(e);
        if (ev >= 0 && !req.empty() && !in_twin[ev] && shares(static_cast<uint32_t>(ev))) {
            in_twin[ev] = true;
            twin.push_back(static_cast<uint32_t>(ev));
        }
    };
    auto ensure = [&](uint32_t v) {
        if (st[v].scored) return;
        st[v].scored = true;
        st[v].raw = -score(s, qv.dense.data(), static_cast<uint32_t>(qv.dense.size()), qv.learned(), qv.stat(), v);
    };
    auto assign = [&](uint32_t v, uint32_t e, uint32_t h) {  // search.cpp:191-198
        NodeSt& z = st[v];
        if (z.ctx && (z.hop < h || (z.hop == h && z.ent <= e))) return;
        z.ctx = true;
        z.ent = e;
        z.hop = h;
    };
    // seeds (search.cpp:67-98)
    std::vector<std::tuple<uint32_t, uint32_t, bool>> seeds;
    if (!ents.empty() && w.entity > 0.0f) {
        for (uint32_t e : ents) {
            auto it = x.emap.find(e);
            if (it == x.emap.end()) continue;
            for (uint32_t v : it->second) seeds.emplace_back(v, e, true);
        }
        std::sort(seeds.begin(), seeds.end());
        seeds.erase(std::unique(seeds.begin(), seeds.end(), [](const auto& a, const auto& b) { return std::get<0>(a) == std::get<0>(b); }), seeds.end());
        if (seeds.empty()) warn |= FG_WARN_ENTITY_FALLBACK;
    }
    if (seeds.empty())
        for (size_t i = 0; i < std::min<size_t>(o.entry_count, x.norm_order.size()); ++i) seeds.emplace_back(x.norm_order[i], 0, false);
    for (const auto& [v, e, has] : seeds) ensure(v);
    for (const auto& [v, e, has] : seeds) {
        if (has) assign(v, e, 0);
        offer(v);
    }
    // best-first loop (search.cpp:218-264)
    expanded = 0;
    while (true) {
        auto it = std::find_if(cand.v.begin(), cand.v.end(), [&](const PE& e) { return !st[e.node].expanded; });
        if (it == cand.v.end()) break;
        const uint32_t u = it->node;
        st[u].expanded = true;
        ++expanded;
        std::vector<uint32_t> nb;
        std::vector<std::pair<uint32_t, uint32_t>> lctx;
        auto add = [&](uint32_t v) {
            if (std::find(nb.begin(), nb.end(), v) == nb.end()) nb.push_back(v);
        };
        for (uint32_t v : x.semantic[u]) add(v);
        if (!req.empty() && shares(u))
            for (uint32_t v : x.keyword[u]) add(v);
        const bool prop = st[u].ctx && st[u].hop < H;
        if (prop)
            for (const auto& le : x.logical[u])
                if (le[0] == st[u].ent) {
                    add(le[3]);
                    lctx.emplace_back(le[3], le[2]);
                }
        for (uint32_t v : nb) {
            ensure(v);
            if (prop) {
                for (const uint32_t* e = s.en_b(v); e != s.en_e(v); ++e)
                    if (s.has_relation(st[u].ent, *e)) {
                        assign(v, *e, st[u].hop + 1);
                        break;
                    }
                for (const auto& [via, tgt] : lctx)
                    if (via == v) assign(v, tgt, st[u].hop + 1);
            }
            offer(v);
        }
    }
    // keyword_postfilter (search.cpp:100-139)
    std::vector<PE> m = top.v;
    if (!req.empty())
        for (uint32_t v : twin) m.push_back({adj(v), v});
    std::sort(m.begin(), m.end(), [](const PE& a, const PE& b) { return a.node != b.node ? a.node < b.node : a.d < b.d; });
    m.erase(std::unique(m.begin(), m.end(), [](const PE& a, const PE& b) { return a.node == b.node; }), m.end());
    std::sort(m.begin(), m.end(), pe_less);
    for (const PE& e : m) {
        if (hits.size() == K) break;
        if (s.deleted[e.node]) continue;
        if (!req.empty()) {
            size_t c = 0;
            for (uint32_t t : req) c += sorted_has(s.kw_b(e.node), s.kw_e(e.node), t);
            if (o.conjunctive_filter ? c != req.size() : c == 0) continue;
        }
        hits.push_back(e);
    }
    if (!req.empty() && hits.size() < K) warn |= FG_WARN_KEYWORD_SHORTFALL;
}

void put_row(fg_search_results* out, uint64_t i, const Store& s, const std::vector<PE>& hits, bool neg) {
    out->hit_count[i] = static_cast<uint32_t>(hits.size());
    for (size_t j = 0; j < hits.size(); ++j) {
        out->node[i * out->hit_stride + j] = hits[j].node;
        out->doc_id[i * out->hit_stride + j] = s.doc_id[hits[j].node];
        out->score[i * out->hit_stride + j] = neg ? -hits[j].d : hits[j].d;
    }
}
void put_err(fg_search_results* out, uint64_t i, const std::string& e) {
    if (!out->errors || !out->error_stride) return;
    char* d = out->errors + i * out->error_stride;
    std::strncpy(d, e.c_str(), out->error_stride - 1);
    d[out->error_stride - 1] = 0;
}

void knn_out(const Lists& L, fg_knn_lists* o) {
    o->k = L.empty() ? o->k : static_cast<uint32_t>(L[0].size());
    for (size_t u = 0; u < L.size(); ++u)
        for (size_t j = 0; j < L[u].size(); ++j) {
            o->ids[u * o->k + j] = L[u][j].id;
            o->scores[u * o->k + j] = L[u][j].sc;
            o->fresh[u * o->k + j] = L[u][j].fresh;
        }
}
Lists knn_in(const fg_knn_lists* l) {
    Lists L(l->n);
    for (uint64_t u = 0; u < l->n; ++u)
        for (uint32_t j = 0; j < l->k; ++j)
            L[u].push_back({l->ids[u * l->k + j], l->scores[u * l->k + j], l->fresh[u * l->k + j] != 0});
    return L;
}

}  // namespace

extern "C" {

const char* fgo_last_error(void) { return g_err.c_str(); }

int fgo_store_create(const fg_corpus_view* v, const fg_kg_view* kg, void** out) {
    return run([&] {
        auto s = std::make_unique<Store>();
        s->n = v->n;
        s->dim = v->dense_dim;
        s->dense.assign(v->dense, v->dense + v->n * v->dense_dim);
        auto csr = [&](const uint64_t* p, const uint32_t* i, const float* x, std::vector<uint64_t>& op,
                       std::vector<uint32_t>& oi, std::vector<float>* ov) {
            op.assign(v->n + 1, 0);
            if (!p) return;
            for (uint64_t r = 0; r < v->n; ++r) op[r + 1] = p[r + 1] - p[0];
            oi.assign(i + p[0], i + p[v->n]);
            if (ov) ov->assign(x + p[0], x + p[v->n]);
        };
        csr(v->learned.ptr, v->learned.idx, v->learned.val, s->lp, s->li, &s->lv);
        csr(v->statistical.ptr, v->statistical.idx, v->statistical.val, s->sp, s->si, &s->sv);
        if (v->keywords.ptr)
            csr(v->keywords.ptr, v->keywords.idx, nullptr, s->kp, s->ki, nullptr);
        else {
            s->kp = s->sp;
            s->ki = s->si;
        }
        csr(v->entities.ptr, v->entities.idx, nullptr, s->ep, s->ei, nullptr);
        s->doc_id.resize(v->n);
        s->deleted.assign(v->n, 0);
        for (uint64_t i = 0; i < v->n; ++i) {
            s->doc_id[i] = v->doc_id ? v->doc_id[i] : i;
            if (v->deleted) s->deleted[i] = v->deleted[i] != 0;
        }
        s->sqnorm.resize(v->n);  // finalize_fused (types.cpp:74-79)
        for (uint64_t i = 0; i < v->n; ++i) s->sqnorm[i] = pair(*s, i, i);
        if (kg && kg->count) {  // types.cpp:29-45
            std::vector<std::array<uint32_t, 3>> t;
            for (uint64_t i = 0; i < kg->count; ++i) t.push_back({kg->source[i], kg->relation[i], kg->target[i]});
            std::sort(t.begin(), t.end());
            t.erase(std::unique(t.begin(), t.end()), t.end());
            uint32_t mx = 0;
            for (const auto& x : t) mx = std::max({mx, x[0], x[2]});
            s->adj.resize(mx + 1);
            for (const auto& x : t) {
                s->ts.push_back(x[0]);
                s->tr.push_back(x[1]);
                s->tt.push_back(x[2]);
                s->adj[x[0]].emplace_back(x[2], x[1]);
                s->adj[x[2]].emplace_back(x[0], x[1]);
            }
            for (auto& l : s->adj) {
                std::sort(l.begin(), l.end());
                l.erase(std::unique(l.begin(), l.end()), l.end());
            }
        }
        *out = s.release();
    });
}
void fgo_store_free(void* h) { delete static_cast<Store*>(h); }
int fgo_store_sqnorm(void* h, double* out) {
    const Store& s = *static_cast<Store*>(h);
    std::copy(s.sqnorm.begin(), s.sqnorm.end(), out);
    return FG_OK;
}

int fgo_build_query_vector(const fg_query_view* q, uint64_t i, float* dense, uint32_t* ln, float* lv,
                           uint32_t* sn, float* sv, double* sq) {
    return run([&] {
        const QVec v = weighted(*q, i);
        std::copy(v.dense.begin(), v.dense.end(), dense);
        *ln = static_cast<uint32_t>(v.lv.size());
        std::copy(v.lv.begin(), v.lv.end(), lv);
        *sn = static_cast<uint32_t>(v.sv.size());
        std::copy(v.sv.begin(), v.sv.end(), sv);
        *sq = v.sqnorm;
    });
}

int fgo_batch_scores(void* h, const fg_query_view* q, uint64_t qi, const uint32_t* ids, uint64_t m,
                     unsigned, double* out) {
    return run([&] {
        const Store& s = *static_cast<Store*>(h);
        const QVec v = weighted(*q, qi);
        for (uint64_t i = 0; i < m; ++i) {
            if (ids[i] >= s.n) throw Fail("unknown-id", "node " + std::to_string(ids[i]) + " out of range");
            out[i] = score(s, v.dense.data(), static_cast<uint32_t>(v.dense.size()), v.learned(), v.stat(), ids[i]);
        }
    });
}

int fgo_pair_scores(void* h, const uint32_t* a, const uint32_t* b, uint64_t m, double* out) {
    return run([&] {
        const Store& s = *static_cast<Store*>(h);
        for (uint64_t i = 0; i < m; ++i) out[i] = pair(s, a[i], b[i]);
    });
}

int fgo_knn_init(void* h, uint32_t k, uint64_t seed, unsigned, fg_knn_lists* out) {
    return run([&] { knn_out(knn_init(*static_cast<Store*>(h), k, seed), out); });
}
int fgo_knn_iterate(void* h, fg_knn_lists* l, unsigned, uint64_t* changed) {
    return run([&] {
        Lists L = knn_in(l);
        *changed = knn_pass(*static_cast<Store*>(h), L, l->k);
        knn_out(L, l);
    });
}
int fgo_knn_iterate_range(void* h, fg_knn_lists* l, uint64_t lo, uint64_t hi, uint64_t* changed) {
    return run([&] {
        Lists L = knn_in(l);
        *changed = knn_pass_range(*static_cast<Store*>(h), L, l->k, lo, hi);
        knn_out(L, l);
    });
}
int fgo_knn_build(void* h, const fg_knn_params* p, unsigned, fg_knn_lists* out) {
    return run([&] { knn_out(knn_build(*static_cast<Store*>(h), p->k, p->max_iterations, p->convergence, p->seed), out); });
}

int fgo_refine(void* h, const fg_knn_lists* knn, const fg_refine_params* p, unsigned, fg_refined* out,
               fg_refine_trace* tr) {
    return run([&] {
        const Store& s = *static_cast<Store*>(h);
        const Refined R = refine(s, knn_in(knn), p->degree, p->per_neighbour_keyword_check != 0);
        for (uint64_t u = 0; u < knn->n; ++u) {
            std::copy(R.semantic[u].begin(), R.semantic[u].end(), out->semantic + u * p->degree);
            out->keyword_count[u] = static_cast<uint32_t>(R.keyword[u].size());
            std::copy(R.keyword[u].begin(), R.keyword[u].end(), out->keyword + u * out->keyword_cap);
            if (!tr) continue;
            for (size_t j = 0; j < R.ordered[u].size(); ++j) {
                if (tr->ordered_ids) tr->ordered_ids[u * knn->k + j] = R.ordered[u][j];
                if (tr->ordered_scores) tr->ordered_scores[u * knn->k + j] = R.ordered_sc[u][j];
                if (tr->detours) tr->detours[u * knn->k + j] = R.detours[u][j];
            }
            if (tr->kept_count) tr->kept_count[u] = static_cast<uint32_t>(R.kept[u].size());
            if (tr->kept) std::copy(R.kept[u].begin(), R.kept[u].end(), tr->kept + u * p->degree);
        }
    });
}

int fgo_index_build(void* h, const fg_build_params* p, unsigned, void** out) {  // index.cpp:25-71
    return run([&] {
        Store* s = static_cast<Store*>(h);
        if (p->degree % 2) throw Fail("degree-not-even", "semantic degree must be even, got " + std::to_string(p->degree));
        if (p->knn_k < p->degree) throw Fail("invalid-k", "knn_k must be at least the degree");
        if (s->n < static_cast<uint64_t>(p->degree) + 1)
            throw Fail("corpus-too-small", "need more than degree=" + std::to_string(p->degree) + " documents");
        auto x = std::make_unique<Index>();
        x->own = std::make_unique<Store>(std::move(*s));
        x->s = x->own.get();
        x->degree = p->degree;
        const Lists L = knn_build(*x->s, p->knn_k, p->knn_iterations, 0.01, p->seed);
        Refined R = refine(*x->s, L, p->degree, p->per_neighbour_keyword_check != 0);
        x->semantic = std::move(R.semantic);
        x->keyword = std::move(R.keyword);
        finish_index(*x, true, p->logical_cap);
        *out = x.release();
    });
}

int fgo_index_create(void* h, const fg_graph_view* g, uint32_t, void** out) {
    return run([&] {
        Store* s = static_cast<Store*>(h);
        auto x = std::make_unique<Index>();
        x->own = std::make_unique<Store>(std::move(*s));
        x->s = x->own.get();
        const uint64_t n = x->s->n;
        x->degree = g->degree;
        x->semantic.resize(n);
        x->keyword.resize(n);
        x->logical.resize(n);
        for (uint64_t u = 0; u < n; ++u) {
            x->semantic[u].assign(g->semantic + u * g->degree, g->semantic + (u + 1) * g->degree);
            if (g->keyword.ptr) x->keyword[u].assign(g->keyword.idx + g->keyword.ptr[u], g->keyword.idx + g->keyword.ptr[u + 1]);
            if (g->logical_ptr)
                for (uint64_t e = g->logical_ptr[u]; e < g->logical_ptr[u + 1]; ++e)
                    x->logical[u].push_back({g->logical[4 * e], g->logical[4 * e + 1], g->logical[4 * e + 2], g->logical[4 * e + 3]});
        }
        if (g->norm_order) x->norm_order.assign(g->norm_order, g->norm_order + n);
        finish_index(*x, false, 0);
        *out = x.release();
    });
}
void fgo_index_free(void* h) { delete static_cast<Index*>(h); }

int fgo_index_sizes(void* h, uint32_t* degree, uint64_t* kt, uint64_t* lt) {
    const Index& x = *static_cast<Index*>(h);
    *degree = x.degree;
    *kt = 0;
    *lt = 0;
    for (const auto& k : x.keyword) *kt += k.size();
    for (const auto& l : x.logical) *lt += l.size();
    return FG_OK;
}
int fgo_index_export(void* h, uint32_t* sem, uint64_t* kp, uint32_t* ki, uint64_t* lp, uint32_t* lg, uint32_t* no) {
    const Index& x = *static_cast<Index*>(h);
    uint64_t a = 0, b = 0;
    kp[0] = lp[0] = 0;
    for (uint64_t u = 0; u < x.s->n; ++u) {
        std::copy(x.semantic[u].begin(), x.semantic[u].end(), sem + u * x.degree);
        for (uint32_t v : x.keyword[u]) ki[a++] = v;
        kp[u + 1] = a;
        for (const auto& e : x.logical[u]) {
            std::copy(e.begin(), e.end(), lg + 4 * b);
            ++b;
        }
        lp[u + 1] = b;
    }
    std::copy(x.norm_order.begin(), x.norm_order.end(), no);
    return FG_OK;
}
int fgo_index_set_deleted(void* h, const uint8_t* f) {
    Index& x = *static_cast<Index*>(h);
    for (uint64_t i = 0; i < x.s->n; ++i) x.s->deleted[i] = f[i] != 0;
    return FG_OK;
}

int fgo_batch_query(void* h, const fg_query_view* q, const fg_search_opts* o, unsigned, fg_search_results* out) {
    return run([&] {
        const Index& x = *static_cast<Index*>(h);
        const fg_search_opts opts = o ? *o : fg_search_opts{32, 1};
        for (uint64_t i = 0; i < q->count; ++i) {  // search.cpp:282-293 (per-query errors)
            std::vector<PE> hits;
            uint32_t warn = 0;
            uint64_t exp = 0;
            std::string err;
            try {
                search_one(x, *q, i, opts, hits, warn, exp);
            } catch (const std::exception& e) {
                err = e.what();
                hits.clear();
                warn = 0;
                exp = 0;
            }
            put_row(out, i, *x.s, hits, true);
            if (out->expanded) out->expanded[i] = exp;
            if (out->warnings) out->warnings[i] = warn;
            put_err(out, i, err);
        }
    });
}

int fgo_brute_force(void* h, const fg_query_view* q, unsigned, fg_search_results* out) {  // eval.cpp:14-51
    return run([&] {
        const Store& s = *static_cast<Store*>(h);
        for (uint64_t i = 0; i < q->count; ++i) {
            std::vector<PE> hits;
            std::string err;
            try {
                check_weights(weights_of(*q, i));
                const uint32_t K = q->k ? q->k[i] : 10;
                if (K == 0) throw Fail("invalid-k", "k must be positive");
                const QVec v = weighted(*q, i);
                std::vector<uint32_t> req;
                if (q->required_keywords.ptr)
                    req.assign(q->required_keywords.idx + q->required_keywords.ptr[i], q->required_keywords.idx + q->required_keywords.ptr[i + 1]);
                std::vector<std::pair<double, uint32_t>> all;
                for (uint64_t d = 0; d < s.n; ++d) {
                    if (s.deleted[d]) continue;
                    bool ok = true;
                    for (uint32_t t : req) ok = ok && sorted_has(s.kw_b(d), s.kw_e(d), t);
                    if (!ok) continue;
                    all.emplace_back(score(s, v.dense.data(), static_cast<uint32_t>(v.dense.size()), v.learned(), v.stat(), d),
                                     static_cast<uint32_t>(d));
                }
                const size_t take = std::min<size_t>(K, all.size());
                std::partial_sort(all.begin(), all.begin() + take, all.end(), [&](const auto& a, const auto& b) {
                    return a.first != b.first ? a.first > b.first : s.doc_id[a.second] < s.doc_id[b.second];
                });
                for (size_t j = 0; j < take; ++j) hits.push_back({all[j].first, all[j].second});
            } catch (const std::exception& e) {
                err = e.what();
                hits.clear();
            }
            put_row(out, i, s, hits, false);
            put_err(out, i, err);
        }
    });
}

}  // extern "C"
