// fusegraph_b200_shim.cpp — the reference-side binding: re-implements the
// reference's hot-path entry points (namespace fusegraph, headers unchanged)
// on top of the C-ABI of libfgb200.so (include/fg_b200.h).  A maintainer
// links this translation unit ahead of the reference's own objects; every
// caller (CLI, eval, insert_batch, the test suites) then runs on the B200.
//
//   scoring.hpp:32   batch_scores        -> fg_batch_scores
//   knn_graph.hpp:52 init_random_graph   -> fg_knn_init
//   knn_graph.hpp:56 nn_descent_iterate  -> fg_knn_iterate
//   knn_graph.hpp:59 build_knn_graph     -> fg_knn_build
//   refine.hpp:87    refine_graph        -> fg_refine
//   index.hpp:60     build_hybrid_index  -> fg_index_build (fg_knn_build + fg_refine with a trace)
//   search.hpp:84    search              -> fg_batch_query (one row)
//   search.hpp:86    batch_query         -> fg_batch_query
//   eval.hpp:20      brute_force_topk    -> fg_brute_force_topk
//
// Errors come back as fusegraph::Error with the reference's codes.

#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "fg_b200.h"
#include "fusegraph/eval.hpp"
#include "fusegraph/index.hpp"
#include "fusegraph/knn_graph.hpp"
#include "fusegraph/logical.hpp"
#include "fusegraph/refine.hpp"
#include "fusegraph/scoring.hpp"
#include "fusegraph/search.hpp"

namespace fusegraph {
namespace {

[[noreturn]] void rethrow() {
    const std::string code = fg_last_error_code();
    std::string what = fg_last_error_message();
    const std::string prefix = code + ": ";
    if (what.rfind(prefix, 0) == 0) what = what.substr(prefix.size());
    throw Error(code, what);
}
void ok(int st) {
    if (st != FG_OK) rethrow();
}

// SoA copy of a DocumentStore + the view over it.
struct Flat {
    std::vector<float> dense;
    std::vector<uint64_t> lp{0}, sp{0}, kp{0}, ep{0}, ids;
    std::vector<uint32_t> li, si, ki, ei;
    std::vector<float> lv, sv;
    std::vector<uint8_t> del;
    fg_corpus_view v{};

    explicit Flat(const DocumentStore& st) {
        const uint32_t dim = st.size() ? static_cast<uint32_t>(st.docs[0].vector.dense.dim()) : 0;
        for (const auto& d : st.docs) {
            if (d.vector.dense.dim() != dim)
                throw Error("dim-mismatch", "dense dimensions differ within the corpus");
            dense.insert(dense.end(), d.vector.dense.values.begin(), d.vector.dense.values.end());
            li.insert(li.end(), d.vector.learned.indices.begin(), d.vector.learned.indices.end());
            lv.insert(lv.end(), d.vector.learned.values.begin(), d.vector.learned.values.end());
            lp.push_back(li.size());
            si.insert(si.end(), d.vector.statistical.indices.begin(), d.vector.statistical.indices.end());
            sv.insert(sv.end(), d.vector.statistical.values.begin(), d.vector.statistical.values.end());
            sp.push_back(si.size());
            ki.insert(ki.end(), d.keywords.begin(), d.keywords.end());
            kp.push_back(ki.size());
            ei.insert(ei.end(), d.entities.begin(), d.entities.end());
            ep.push_back(ei.size());
            ids.push_back(d.doc_id);
            del.push_back(d.deleted ? 1 : 0);
        }
        v.n = st.size();
        v.dense_dim = dim;
        v.dense = dense.data();
        v.learned = {lp.data(), li.data(), lv.data()};
        v.statistical = {sp.data(), si.data(), sv.data()};
        v.keywords = {kp.data(), ki.data()};
        v.entities = {ep.data(), ei.data()};
        v.doc_id = ids.data();
        v.deleted = del.data();
    }
};

struct Corpus {  // RAII device corpus
    fg_corpus* h = nullptr;
    explicit Corpus(const DocumentStore& st) {
        Flat f(st);
        ok(fg_corpus_upload(&f.v, 0, &h));
    }
    ~Corpus() { fg_corpus_free(h); }
};

struct KgFlat {
    std::vector<uint32_t> s, r, t;
    fg_kg_view v{};
    explicit KgFlat(const KnowledgeGraph& kg) {
        for (const auto& x : kg.triplets()) {
            s.push_back(x.source);
            r.push_back(x.relation);
            t.push_back(x.target);
        }
        v = {s.size(), s.data(), r.data(), t.data()};
    }
};

struct QueryFlat {
    std::vector<float> dense;
    std::vector<uint64_t> lp{0}, sp{0}, rp{0}, ep{0};
    std::vector<uint32_t> li, si, ri, ei, k, beam, hops;
    std::vector<float> lv, sv;
    std::vector<fg_weights> w;
    fg_query_view v{};
    explicit QueryFlat(std::span<const QuerySpec> qs) {
        const uint32_t dim = qs.empty() ? 0 : static_cast<uint32_t>(qs[0].vector.dense.dim());
        for (const auto& q : qs) {
            // ragged dense dims cannot share one view: pad (the device check
            // then rejects them with dim-mismatch like the reference does)
            std::vector<float> d = q.vector.dense.values;
            d.resize(dim, 0.0f);
            dense.insert(dense.end(), d.begin(), d.end());
            li.insert(li.end(), q.vector.learned.indices.begin(), q.vector.learned.indices.end());
            lv.insert(lv.end(), q.vector.learned.values.begin(), q.vector.learned.values.end());
            lp.push_back(li.size());
            si.insert(si.end(), q.vector.statistical.indices.begin(), q.vector.statistical.indices.end());
            sv.insert(sv.end(), q.vector.statistical.values.begin(), q.vector.statistical.values.end());
            sp.push_back(si.size());
            ri.insert(ri.end(), q.required_keywords.begin(), q.required_keywords.end());
            rp.push_back(ri.size());
            ei.insert(ei.end(), q.entities.begin(), q.entities.end());
            ep.push_back(ei.size());
            w.push_back({q.weights.dense, q.weights.learned, q.weights.statistical, q.weights.entity});
            k.push_back(q.k);
            beam.push_back(q.beam_width);
            hops.push_back(q.max_entity_hops);
        }
        v.count = qs.size();
        v.dense_dim = dim;
        v.dense = dense.data();
        v.learned = {lp.data(), li.data(), lv.data()};
        v.statistical = {sp.data(), si.data(), sv.data()};
        v.weights = w.data();
        v.required_keywords = {rp.data(), ri.data()};
        v.entities = {ep.data(), ei.data()};
        v.k = k.data();
        v.beam_width = beam.data();
        v.max_entity_hops = hops.data();
    }
};

KnnGraph to_graph(uint64_t n, uint32_t k, const std::vector<uint32_t>& ids,
                  const std::vector<double>& sc, const std::vector<uint8_t>& fr) {
    KnnGraph g;
    g.k = k;
    g.lists.resize(n);
    for (uint64_t u = 0; u < n; ++u)
        for (uint32_t j = 0; j < k; ++j)
            g.lists[u].push_back({ids[u * k + j], sc[u * k + j], fr[u * k + j] != 0});
    return g;
}

// Device mirror of a HybridIndex, cached by identity + a content fingerprint
// (mark_delete / insert_batch mutate the struct in place).
struct IndexCache {
    std::mutex mu;
    const HybridIndex* key = nullptr;
    uint64_t fp = 0;
    std::unique_ptr<Corpus> corpus;
    fg_index* ix = nullptr;

    static uint64_t fingerprint(const HybridIndex& x) {
        uint64_t h = 1469598103934665603ull ^ x.size();
        auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
        for (std::size_t u = 0; u < x.size(); ++u) {
            mix(x.store.docs[u].deleted);
            mix(x.semantic[u].empty() ? ~0u : x.semantic[u][0]);
            mix(x.keyword[u].size());
            mix(x.logical[u].size());
        }
        return h;
    }

    fg_index* get(const HybridIndex& x) {
        const uint64_t f = fingerprint(x);
        if (ix && key == &x && fp == f) return ix;
        if (ix) fg_index_free(ix);
        ix = nullptr;
        corpus = std::make_unique<Corpus>(x.store);
        const uint64_t n = x.size();
        std::vector<uint32_t> sem(n * x.degree), ki, lg, norm(x.norm_order);
        std::vector<uint64_t> kp{0}, lp{0};
        for (uint64_t u = 0; u < n; ++u) {
            std::copy(x.semantic[u].begin(), x.semantic[u].end(), sem.begin() + u * x.degree);
            ki.insert(ki.end(), x.keyword[u].begin(), x.keyword[u].end());
            kp.push_back(ki.size());
            for (const auto& e : x.logical[u]) lg.insert(lg.end(), {e.source, e.relation, e.target, e.via});
            lp.push_back(lg.size() / 4);
        }
        KgFlat kg(x.kg);
        fg_graph_view gv{x.degree, sem.data(), {kp.data(), ki.data()}, lp.data(), lg.data(), norm.data()};
        ok(fg_index_create(corpus->h, &kg.v, &gv, &ix));
        key = &x;
        fp = f;
        return ix;
    }
};
IndexCache g_cache;

std::vector<SearchResult> run_gpu(const HybridIndex& index, std::span<const QuerySpec> queries,
                                  const SearchOptions& opts);

// Host validation first (validate_query, then the dense-dim check that the
// reference's dense_dot raises), so error precedence matches search().
std::vector<SearchResult> run_batch(const HybridIndex& index, std::span<const QuerySpec> queries,
                                    const SearchOptions& opts) {
    std::vector<SearchResult> out(queries.size());
    std::vector<QuerySpec> ok_q;
    std::vector<std::size_t> pos;
    const std::size_t dim = index.size() ? index.store.docs[0].vector.dense.dim() : 0;
    for (std::size_t i = 0; i < queries.size(); ++i) {
        try {
            validate_query(queries[i]);
            if (queries[i].vector.dense.dim() != dim)
                throw Error("dim-mismatch", "dense dimensions differ: " +
                                                std::to_string(queries[i].vector.dense.dim()) + " vs " +
                                                std::to_string(dim));
            ok_q.push_back(queries[i]);
            pos.push_back(i);
        } catch (const Error& e) {
            out[i].error = e.what();
        }
    }
    auto r = run_gpu(index, ok_q, opts);
    for (std::size_t j = 0; j < pos.size(); ++j) out[pos[j]] = std::move(r[j]);
    return out;
}

std::vector<SearchResult> run_gpu(const HybridIndex& index, std::span<const QuerySpec> queries,
                                  const SearchOptions& opts) {
    std::vector<SearchResult> out(queries.size());
    if (queries.empty()) return out;
    std::lock_guard<std::mutex> lock(g_cache.mu);
    fg_index* ix = g_cache.get(index);
    QueryFlat qf(queries);
    uint32_t kmax = 1;
    for (const auto& q : queries) kmax = std::max(kmax, q.k);
    const uint64_t nq = queries.size();
    std::vector<uint64_t> doc(nq * kmax), expanded(nq);
    std::vector<uint32_t> node(nq * kmax), cnt(nq), warn(nq);
    std::vector<double> score(nq * kmax);
    std::vector<char> err(nq * 256, 0);
    fg_search_results r{kmax, doc.data(), node.data(), score.data(), cnt.data(), expanded.data(),
                        nullptr, warn.data(), err.data(), 256};
    fg_search_opts o{opts.entry_count, opts.conjunctive_filter ? 1 : 0};
    ok(fg_batch_query(ix, &qf.v, &o, &r));
    for (uint64_t i = 0; i < nq; ++i) {
        SearchResult& s = out[i];
        s.error = std::string(err.data() + i * 256);
        s.expanded = expanded[i];
        if (warn[i] & FG_WARN_ENTITY_FALLBACK) s.warnings.emplace_back("entity-fallback");
        if (warn[i] & FG_WARN_KEYWORD_SHORTFALL) s.warnings.emplace_back("keyword-shortfall");
        for (uint32_t j = 0; j < cnt[i]; ++j)
            s.hits.push_back({doc[i * kmax + j], node[i * kmax + j], score[i * kmax + j]});
    }
    return out;
}

}  // namespace

std::vector<Score> batch_scores(const FusedVector& weighted_query, std::span<const uint32_t> ids,
                                const DocumentStore& store, unsigned) {
    for (uint32_t id : ids) (void)store.doc(id);  // unknown-id, like store.doc()
    std::vector<Score> out(ids.size());
    if (ids.empty()) return out;
    Corpus c(store);
    QuerySpec q;
    q.vector = weighted_query;  // already weighted: unit weights keep it as is
    QueryFlat qf(std::span<const QuerySpec>(&q, 1));
    if (qf.v.dense_dim != store.dense_dim && store.size())
        throw Error("dim-mismatch", "dense dimensions differ: " + std::to_string(qf.v.dense_dim) +
                                        " vs " + std::to_string(store.docs[0].vector.dense.dim()));
    ok(fg_batch_scores(c.h, &qf.v, 0, ids.data(), ids.size(), out.data()));
    return out;
}

KnnGraph init_random_graph(const DocumentStore& store, uint32_t k, uint64_t seed, unsigned) {
    Corpus c(store);
    const uint64_t n = store.size();
    std::vector<uint32_t> ids(n * k);
    std::vector<double> sc(n * k);
    std::vector<uint8_t> fr(n * k);
    fg_knn_lists l{n, k, ids.data(), sc.data(), fr.data()};
    ok(fg_knn_init(c.h, k, seed, &l));
    return to_graph(n, k, ids, sc, fr);
}

std::size_t nn_descent_iterate(const DocumentStore& store, KnnGraph& graph, unsigned) {
    Corpus c(store);
    const uint64_t n = graph.size();
    const uint32_t k = graph.k;
    std::vector<uint32_t> ids(n * k);
    std::vector<double> sc(n * k);
    std::vector<uint8_t> fr(n * k);
    for (uint64_t u = 0; u < n; ++u)
        for (uint32_t j = 0; j < k; ++j) {
            ids[u * k + j] = graph.lists[u][j].id;
            sc[u * k + j] = graph.lists[u][j].score;
            fr[u * k + j] = graph.lists[u][j].fresh;
        }
    fg_knn_lists l{n, k, ids.data(), sc.data(), fr.data()};
    uint64_t changed = 0;
    ok(fg_knn_iterate(c.h, &l, &changed));
    graph = to_graph(n, k, ids, sc, fr);
    return changed;
}

KnnGraph build_knn_graph(const DocumentStore& store, const KnnBuildParams& p) {
    Corpus c(store);
    const uint64_t n = store.size();
    const uint32_t kk = (n >= 2 && p.k >= n) ? static_cast<uint32_t>(n - 1) : p.k;
    std::vector<uint32_t> ids(n * kk);
    std::vector<double> sc(n * kk);
    std::vector<uint8_t> fr(n * kk);
    fg_knn_lists l{n, kk, ids.data(), sc.data(), fr.data()};
    fg_knn_params kp{p.k, p.max_iterations, p.convergence, p.seed};
    ok(fg_knn_build(c.h, &kp, &l, nullptr));
    return to_graph(n, l.k, ids, sc, fr);
}

RefinedEdges refine_graph(const DocumentStore& store, const KnnGraph& knn, const RefineParams& p,
                          RefineTrace* trace) {
    Corpus c(store);
    const uint64_t n = knn.size();
    const uint32_t k = knn.k;
    std::vector<uint32_t> ids(n * k);
    std::vector<double> sc(n * k);
    std::vector<uint8_t> fr(n * k);
    for (uint64_t u = 0; u < n; ++u)
        for (uint32_t j = 0; j < k; ++j) {
            ids[u * k + j] = knn.lists[u][j].id;
            sc[u * k + j] = knn.lists[u][j].score;
            fr[u * k + j] = knn.lists[u][j].fresh;
        }
    fg_knn_lists l{n, k, ids.data(), sc.data(), fr.data()};
    std::vector<uint32_t> sem(n * p.degree), kw(n * k), kwc(n), oid(n * k), det(n * k),
        kept(n * p.degree), keptc(n);
    std::vector<double> osc(n * k);
    fg_refined out{sem.data(), k, kw.data(), kwc.data()};
    fg_refine_trace tr{oid.data(), osc.data(), det.data(), kept.data(), keptc.data()};
    fg_refine_params rp{p.degree, p.per_neighbour_keyword_check ? 1 : 0};
    ok(fg_refine(c.h, &l, &rp, &out, trace ? &tr : nullptr));
    RefinedEdges e;
    e.semantic.resize(n);
    e.keyword.resize(n);
    if (trace) {
        trace->ordered.assign(n, {});
        trace->detours.assign(n, {});
        trace->kept.assign(n, {});
    }
    for (uint64_t u = 0; u < n; ++u) {
        e.semantic[u].assign(sem.begin() + u * p.degree, sem.begin() + (u + 1) * p.degree);
        e.keyword[u].assign(kw.begin() + u * k, kw.begin() + u * k + kwc[u]);
        if (!trace) continue;
        for (uint32_t j = 0; j < k; ++j) {
            trace->ordered[u].push_back({oid[u * k + j], osc[u * k + j]});
            trace->detours[u].push_back(det[u * k + j]);
        }
        trace->kept[u].assign(kept.begin() + u * p.degree, kept.begin() + u * p.degree + keptc[u]);
    }
    return e;
}

HybridIndex build_hybrid_index(DocumentStore store, KnowledgeGraph kg, const BuildParams& params,
                               RefineTrace* trace) {
    if (params.degree % 2 != 0)
        throw Error("degree-not-even", "semantic degree must be even, got " + std::to_string(params.degree));
    if (params.knn_k < params.degree) throw Error("invalid-k", "knn_k must be at least the degree");
    if (store.size() < params.degree + 1)
        throw Error("corpus-too-small", "need more than degree=" + std::to_string(params.degree) + " documents");
    HybridIndex index;
    index.degree = params.degree;
    index.knn_k = params.knn_k;
    index.logical_cap = params.logical_cap;
    index.default_entity_hops = params.default_entity_hops;
    index.build_seed = params.seed;
    const uint64_t n = store.size();
    if (trace) {  // stage by stage so the refinery trace can be returned
        KnnBuildParams kp;
        kp.k = params.knn_k;
        kp.max_iterations = params.knn_iterations;
        kp.seed = params.seed;
        KnnGraph g = build_knn_graph(store, kp);
        RefineParams rp;
        rp.degree = params.degree;
        rp.per_neighbour_keyword_check = params.per_neighbour_keyword_check;
        RefinedEdges e = refine_graph(store, g, rp, trace);
        index.semantic = std::move(e.semantic);
        index.keyword = std::move(e.keyword);
        index.store = std::move(store);
        index.kg = std::move(kg);
        index.entity_map = build_entity_map(index.store);
        LogicalParams lp;
        lp.per_entity_cap = params.logical_cap;
        index.logical = derive_logical_edges(index.store, index.kg, index.entity_map, lp);
        rebuild_norm_order(index);
        return index;
    }
    Corpus c(store);
    KgFlat kf(kg);
    fg_build_params bp{params.degree, params.knn_k, params.knn_iterations, params.seed,
                       params.logical_cap, params.default_entity_hops,
                       params.per_neighbour_keyword_check ? 1 : 0};
    fg_index* ix = nullptr;
    ok(fg_index_build(c.h, &kf.v, &bp, &ix));
    uint32_t deg = 0;
    uint64_t kt = 0, lt = 0;
    ok(fg_index_sizes(ix, &deg, &kt, &lt));
    std::vector<uint32_t> sem(n * deg), ki(kt), lg(lt * 4), norm(n);
    std::vector<uint64_t> kp(n + 1), lp(n + 1);
    ok(fg_index_export(ix, sem.data(), kp.data(), ki.data(), lp.data(), lg.data(), norm.data()));
    fg_index_free(ix);
    index.semantic.resize(n);
    index.keyword.resize(n);
    index.logical.resize(n);
    for (uint64_t u = 0; u < n; ++u) {
        index.semantic[u].assign(sem.begin() + u * deg, sem.begin() + (u + 1) * deg);
        index.keyword[u].assign(ki.begin() + kp[u], ki.begin() + kp[u + 1]);
        for (uint64_t e = lp[u]; e < lp[u + 1]; ++e)
            index.logical[u].push_back({lg[4 * e], lg[4 * e + 1], lg[4 * e + 2], lg[4 * e + 3]});
    }
    index.norm_order = std::move(norm);
    index.store = std::move(store);
    index.kg = std::move(kg);
    index.entity_map = build_entity_map(index.store);
    return index;
}

SearchResult search(const HybridIndex& index, const QuerySpec& q, const SearchOptions& opts) {
    auto r = run_batch(index, std::span<const QuerySpec>(&q, 1), opts);
    if (!r[0].error.empty()) {
        const std::string& w = r[0].error;
        const auto colon = w.find(": ");
        throw Error(w.substr(0, colon), colon == std::string::npos ? w : w.substr(colon + 2));
    }
    return std::move(r[0]);
}

std::vector<SearchResult> batch_query(const HybridIndex& index, std::span<const QuerySpec> queries,
                                      unsigned, const SearchOptions& opts) {
    return run_batch(index, queries, opts);
}

std::vector<SearchHit> brute_force_topk(const DocumentStore& store, const QuerySpec& q, unsigned) {
    validate_weights(q.weights);
    if (q.k == 0) throw Error("invalid-k", "k must be positive");
    Corpus c(store);
    QueryFlat qf(std::span<const QuerySpec>(&q, 1));
    std::vector<uint64_t> doc(q.k);
    std::vector<uint32_t> node(q.k), cnt(1);
    std::vector<double> score(q.k);
    std::vector<char> err(256, 0);
    fg_search_results r{q.k, doc.data(), node.data(), score.data(), cnt.data(), nullptr, nullptr,
                        nullptr, err.data(), 256};
    ok(fg_brute_force_topk(c.h, &qf.v, &r));
    if (err[0]) {
        const std::string w(err.data());
        const auto colon = w.find(": ");
        throw Error(w.substr(0, colon), w.substr(colon + 2));
    }
    std::vector<SearchHit> hits;
    for (uint32_t j = 0; j < cnt[0]; ++j) hits.push_back({doc[j], node[j], score[j]});
    return hits;
}

}  // namespace fusegraph
