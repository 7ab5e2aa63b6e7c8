// index.cu — build_hybrid_index orchestration (index.cpp:25-71) over the
// device kernels, plus the host-side integer stages the survey keeps on the
// host: entity map and logical edges (logical.cpp:9-68), KG adjacency
// (types.cpp:29-45) and the norm order (index.cpp:12-23).
#include <algorithm>
#include <array>
#include <chrono>
#include <numeric>
#include <thread>

#include "index.hpp"
#include "knn.cuh"

namespace fgb {
namespace {

using Clock = std::chrono::steady_clock;
double secs(Clock::time_point a) { return std::chrono::duration<double>(Clock::now() - a).count(); }

template <typename Fn>
void parallel_rows(uint64_t n, Fn&& fn) {
    const unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    if (n < 4096 || nt == 1) {
        for (uint64_t i = 0; i < n; ++i) fn(i);
        return;
    }
    std::vector<std::thread> pool;
    const uint64_t chunk = (n + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
        const uint64_t b = t * chunk, e = std::min(n, b + chunk);
        if (b >= e) break;
        pool.emplace_back([&, b, e] {
            for (uint64_t i = b; i < e; ++i) fn(i);
        });
    }
    for (auto& t : pool) t.join();
}

// KnowledgeGraph(triplets) (types.cpp:29-45): sorted unique triplets and the
// undirected adjacency entity -> sorted unique (neighbor, relation).
struct HostKg {
    std::vector<std::vector<std::pair<uint32_t, uint32_t>>> adj;  // dense by entity id
    const std::vector<std::pair<uint32_t, uint32_t>>& nb(uint32_t e) const {
        static const std::vector<std::pair<uint32_t, uint32_t>> none;
        return e < adj.size() ? adj[e] : none;
    }
};

HostKg make_kg(const fg_kg_view* kg) {
    HostKg h;
    if (!kg || kg->count == 0) return h;
    uint32_t mx = 0;
    for (uint64_t i = 0; i < kg->count; ++i) mx = std::max({mx, kg->source[i], kg->target[i]});
    h.adj.resize(static_cast<size_t>(mx) + 1);
    for (uint64_t i = 0; i < kg->count; ++i) {
        h.adj[kg->source[i]].emplace_back(kg->target[i], kg->relation[i]);
        h.adj[kg->target[i]].emplace_back(kg->source[i], kg->relation[i]);
    }
    for (auto& l : h.adj) {
        std::sort(l.begin(), l.end());
        l.erase(std::unique(l.begin(), l.end()), l.end());
    }
    return h;
}

// derive_logical_edges_for (logical.cpp:17-55).
void logical_for(const fg_corpus& c, uint32_t node, const HostKg& kg,
                 const std::map<uint32_t, std::vector<uint32_t>>& emap, uint32_t cap,
                 std::vector<uint32_t>& out) {
    const uint32_t* ob = c.entities.begin(node);
    const uint32_t* oe = c.entities.end(node);
    struct E {
        uint32_t s, r, t, v;
    };
    std::vector<E> group;
    for (const uint32_t* sp = ob; sp != oe; ++sp) {
        const uint32_t source = *sp;
        group.clear();
        bool have_prev = false;
        uint32_t prev = 0;
        for (const auto& [target, relation] : kg.nb(source)) {
            if (have_prev && target == prev) continue;
            have_prev = true;
            prev = target;
            if (std::binary_search(ob, oe, target)) continue;
            auto it = emap.find(target);
            if (it == emap.end()) continue;
            for (uint32_t via : it->second) {
                if (via == node) continue;
                group.push_back({source, relation, target, via});
            }
        }
        std::stable_sort(group.begin(), group.end(), [&](const E& a, const E& b) {
            const size_t da = kg.nb(a.t).size(), db = kg.nb(b.t).size();
            if (da != db) return da > db;
            if (a.t != b.t) return a.t < b.t;
            return a.v < b.v;
        });
        if (group.size() > cap) group.resize(cap);
        for (const E& e : group) out.insert(out.end(), {e.s, e.r, e.t, e.v});
    }
}

}  // namespace

__global__ void gather_meta_kernel(const uint4* meta, const uint32_t* ids, uint64_t m, uint4* out) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i < m) out[i] = meta[ids[i]];
}

void index_finish(fg_index& ix, const fg_kg_view* kgv) {
    fg_corpus& c = *ix.corpus;
    cudaStream_t s = c.stream;
    const uint64_t n = c.n;
    auto t0 = Clock::now();

    // entity map (logical.cpp:9-15)
    ix.entity_map.clear();
    for (uint64_t u = 0; u < n; ++u)
        for (const uint32_t* e = c.entities.begin(u); e != c.entities.end(u); ++e)
            ix.entity_map[*e].push_back(static_cast<uint32_t>(u));

    // KnowledgeGraph triplets as the reference keeps them (types.cpp:29-40:
    // sorted by (source, relation, target), duplicates removed)
    {
        std::vector<std::array<uint32_t, 3>> t;
        if (kgv)
            for (uint64_t i = 0; i < kgv->count; ++i) t.push_back({kgv->source[i], kgv->relation[i], kgv->target[i]});
        std::sort(t.begin(), t.end());
        t.erase(std::unique(t.begin(), t.end()), t.end());
        ix.triplets.clear();
        for (const auto& x : t) ix.triplets.insert(ix.triplets.end(), x.begin(), x.end());
    }
    // logical edges, unless given
    const HostKg kg = make_kg(kgv);
    if (ix.lg_ptr_h.empty()) {
        std::vector<std::vector<uint32_t>> per(n);
        parallel_rows(n, [&](uint64_t u) {
            logical_for(c, static_cast<uint32_t>(u), kg, ix.entity_map, ix.logical_cap, per[u]);
        });
        ix.lg_ptr_h.assign(n + 1, 0);
        for (uint64_t u = 0; u < n; ++u) ix.lg_ptr_h[u + 1] = ix.lg_ptr_h[u] + per[u].size() / 4;
        ix.lg_h.clear();
        ix.lg_h.reserve(ix.lg_ptr_h[n] * 4);
        for (auto& v : per) ix.lg_h.insert(ix.lg_h.end(), v.begin(), v.end());
    }
    ix.max_logical_group = 0;
    for (uint64_t u = 0; u < n; ++u) {  // largest (node, source) group
        uint32_t run = 0;
        for (uint64_t e = ix.lg_ptr_h[u]; e < ix.lg_ptr_h[u + 1]; ++e) {
            run = (e > ix.lg_ptr_h[u] && ix.lg_h[4 * e] == ix.lg_h[4 * (e - 1)]) ? run + 1 : 1;
            ix.max_logical_group = std::max(ix.max_logical_group, run);
        }
    }
    ix.lg_ptr.upload(ix.lg_ptr_h, s);
    {
        std::vector<uint4> lg(std::max<uint64_t>(ix.lg_ptr_h[n], 1));
        for (uint64_t e = 0; e < ix.lg_ptr_h[n]; ++e)
            lg[e] = make_uint4(ix.lg_h[4 * e], ix.lg_h[4 * e + 1], ix.lg_h[4 * e + 2], ix.lg_h[4 * e + 3]);
        ix.lg.upload(lg, s);
        FGB_CUDA(cudaStreamSynchronize(s));
    }
    // KG adjacency for has_relation (types.cpp:52-57): neighbours only
    {
        std::vector<uint64_t> ptr(kg.adj.size() + 1, 0);
        std::vector<uint32_t> nbr;
        for (size_t e = 0; e < kg.adj.size(); ++e) {
            uint32_t prev = 0xFFFFFFFFu;
            for (const auto& [t, r] : kg.adj[e]) {
                if (t != prev) nbr.push_back(t);
                prev = t;
            }
            ptr[e + 1] = nbr.size();
        }
        ix.kg_rows = static_cast<uint32_t>(kg.adj.size());
        ix.kg_ptr.upload(ptr, s);
        if (nbr.empty()) nbr.push_back(0);
        ix.kg_nbr.upload(nbr, s);
        FGB_CUDA(cudaStreamSynchronize(s));
    }
    ix.build_seconds[2] = secs(t0);

    // norm order (index.cpp:12-23): squared norm desc, id asc
    t0 = Clock::now();
    if (ix.norm_order_h.size() != n) {
        ix.norm_order_h.resize(n);
        std::iota(ix.norm_order_h.begin(), ix.norm_order_h.end(), 0u);
        const auto& sq = c.sqnorm_h;
        std::sort(ix.norm_order_h.begin(), ix.norm_order_h.end(), [&](uint32_t a, uint32_t b) {
            if (sq[a] != sq[b]) return sq[a] > sq[b];
            return a < b;
        });
    }
    ix.norm_order.upload(ix.norm_order_h, s);
    if (c.dc.meta && n) {
        const uint64_t me = n * ix.degree;
        ix.edge_meta.alloc(me);
        gather_meta_kernel<<<(unsigned)((me + 255) / 256), 256, 0, s>>>(c.dc.meta, ix.semantic.get(), me,
                                                                         ix.edge_meta.get());
        FGB_LAUNCH("gather_meta_kernel");
        ix.norm_meta.alloc(n);
        gather_meta_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c.dc.meta, ix.norm_order.get(), n,
                                                                        ix.norm_meta.get());
        FGB_LAUNCH("gather_meta_kernel");
    }
    ix.max_kw_edges = 0;
    for (size_t u = 0; u < ix.keyword_h.rows(); ++u)
        ix.max_kw_edges = std::max<uint32_t>(ix.max_kw_edges, static_cast<uint32_t>(ix.keyword_h.len(u)));
    ix.kw_ptr.upload(ix.keyword_h.ptr, s);
    ix.kw_idx.upload(ix.keyword_h.idx.empty() ? std::vector<uint32_t>(1, 0) : ix.keyword_h.idx, s);
    FGB_CUDA(cudaStreamSynchronize(s));
    ix.build_seconds[3] = secs(t0);
    if (!ix.ev0) {
        FGB_CUDA(cudaEventCreate(&ix.ev0));
        FGB_CUDA(cudaEventCreate(&ix.ev1));
    }
}

}  // namespace fgb

using namespace fgb;

extern "C" {

int fg_index_build(fg_corpus* c, const fg_kg_view* kg, const fg_build_params* p, fg_index** out) {
    return guarded([&] {
        if (!c || !p || !out) throw Error("invalid-argument", "null pointer");
        if (p->degree % 2 != 0)
            throw Error("degree-not-even", "semantic degree must be even, got " + std::to_string(p->degree));
        if (p->knn_k < p->degree) throw Error("invalid-k", "knn_k must be at least the degree");
        if (c->n < static_cast<uint64_t>(p->degree) + 1)
            throw Error("corpus-too-small",
                        "need more than degree=" + std::to_string(p->degree) + " documents");
        FGB_CUDA(cudaSetDevice(c->device));
        cudaStream_t s = c->stream;
        auto ix = std::make_unique<fg_index>();
        ix->corpus = c;
        ix->degree = p->degree;
        ix->knn_k = p->knn_k;
        ix->logical_cap = p->logical_cap;
        ix->default_hops = p->default_entity_hops;
        ix->seed = p->seed;
        const auto t_all = Clock::now();

        auto t0 = Clock::now();
        DevKnn g;
        knn_build_device(*c, p->knn_k, p->knn_iterations, 0.01, p->seed, g, s);
        FGB_CUDA(cudaStreamSynchronize(s));
        ix->build_seconds[0] = secs(t0);

        t0 = Clock::now();
        RefineOut r;
        refine_device(*c, g, p->degree, p->per_neighbour_keyword_check != 0, r, s);
        const uint64_t n = c->n;
        ix->semantic = std::move(r.semantic);
        ix->semantic_h.resize(n * p->degree);
        ix->semantic.download(ix->semantic_h.data(), n * p->degree, s);
        std::vector<uint32_t> kw(n * g.k), kwc(n);
        r.keyword.download(kw.data(), n * g.k, s);
        r.kw_count.download(kwc.data(), n, s);
        FGB_CUDA(cudaStreamSynchronize(s));
        ix->keyword_h.ptr.assign(n + 1, 0);
        for (uint64_t u = 0; u < n; ++u) ix->keyword_h.ptr[u + 1] = ix->keyword_h.ptr[u] + kwc[u];
        ix->keyword_h.idx.resize(ix->keyword_h.ptr[n]);
        for (uint64_t u = 0; u < n; ++u)
            std::copy(kw.begin() + u * g.k, kw.begin() + u * g.k + kwc[u],
                      ix->keyword_h.idx.begin() + ix->keyword_h.ptr[u]);
        ix->build_seconds[1] = secs(t0);

        index_finish(*ix, kg);
        ix->build_seconds[4] = secs(t_all);
        *out = ix.release();
    });
}

int fg_index_create(fg_corpus* c, const fg_kg_view* kg, const fg_graph_view* gv, fg_index** out) {
    return guarded([&] {
        if (!c || !gv || !out || !gv->semantic) throw Error("invalid-argument", "null pointer");
        FGB_CUDA(cudaSetDevice(c->device));
        auto ix = std::make_unique<fg_index>();
        ix->corpus = c;
        ix->degree = gv->degree;
        const uint64_t n = c->n;
        for (uint64_t i = 0; i < n * gv->degree; ++i)
            if (gv->semantic[i] >= n) throw Error("invariant-violation", "semantic edge out of range");
        ix->semantic_h.assign(gv->semantic, gv->semantic + n * gv->degree);
        ix->semantic.upload(ix->semantic_h, c->stream);
        ix->keyword_h.ptr.assign(n + 1, 0);
        if (gv->keyword.ptr) {
            for (uint64_t u = 0; u < n; ++u) ix->keyword_h.ptr[u + 1] = gv->keyword.ptr[u + 1] - gv->keyword.ptr[0];
            ix->keyword_h.idx.assign(gv->keyword.idx + gv->keyword.ptr[0], gv->keyword.idx + gv->keyword.ptr[n]);
        }
        if (gv->logical_ptr) {
            ix->lg_ptr_h.assign(n + 1, 0);
            for (uint64_t u = 0; u < n; ++u) ix->lg_ptr_h[u + 1] = gv->logical_ptr[u + 1] - gv->logical_ptr[0];
            ix->lg_h.assign(gv->logical + 4 * gv->logical_ptr[0], gv->logical + 4 * gv->logical_ptr[n]);
        }
        if (gv->norm_order) ix->norm_order_h.assign(gv->norm_order, gv->norm_order + n);
        index_finish(*ix, kg);
        *out = ix.release();
    });
}

int fg_index_sizes(const fg_index* ix, uint32_t* degree, uint64_t* kw_total, uint64_t* lg_total) {
    return guarded([&] {
        if (degree) *degree = ix->degree;
        if (kw_total) *kw_total = ix->keyword_h.idx.size();
        if (lg_total) *lg_total = ix->lg_h.size() / 4;
    });
}

int fg_index_export(const fg_index* ix, uint32_t* semantic, uint64_t* kptr, uint32_t* kidx,
                    uint64_t* lptr, uint32_t* logical, uint32_t* norm_order) {
    return guarded([&] {
        if (semantic) std::copy(ix->semantic_h.begin(), ix->semantic_h.end(), semantic);
        if (kptr) std::copy(ix->keyword_h.ptr.begin(), ix->keyword_h.ptr.end(), kptr);
        if (kidx) std::copy(ix->keyword_h.idx.begin(), ix->keyword_h.idx.end(), kidx);
        if (lptr) std::copy(ix->lg_ptr_h.begin(), ix->lg_ptr_h.end(), lptr);
        if (logical) std::copy(ix->lg_h.begin(), ix->lg_h.end(), logical);
        if (norm_order) std::copy(ix->norm_order_h.begin(), ix->norm_order_h.end(), norm_order);
    });
}

int fg_index_build_times(const fg_index* ix, double* s5) {
    return guarded([&] { std::copy(ix->build_seconds, ix->build_seconds + 5, s5); });
}

int fg_index_free(fg_index* ix) {
    if (ix) {
        if (ix->corpus) cudaSetDevice(ix->corpus->device);
        if (ix->ev0) cudaEventDestroy(ix->ev0);
        if (ix->ev1) cudaEventDestroy(ix->ev1);
        delete ix;
    }
    return FG_OK;
}

}  // extern "C"
