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
//   update.hpp:33    insert_batch        -> fg_index_insert (device mirror updated in place)
//   update.hpp:38    mark_delete         -> fg_corpus_set_deleted (device mirror updated in place)
//
// Device mirrors (corpus + index) are cached by an O(1) key (see Mirrors)
// and reused across calls: batch_scores / knn / refine / brute force reuse
// the uploaded corpus, searches on an index returned by build_hybrid_index
// reuse the build's own device index.
//
// Errors come back as fusegraph::Error with the reference's codes.

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_set>
#include <vector>

#include "fg_b200.h"
#include "fusegraph/corpus.hpp"
#include "fusegraph/eval.hpp"
#include "fusegraph/index.hpp"
#include "fusegraph/knn_graph.hpp"
#include "fusegraph/logical.hpp"
#include "fusegraph/refine.hpp"
#include "fusegraph/scoring.hpp"
#include "fusegraph/search.hpp"
#include "fusegraph/update.hpp"
#include "fusegraph_b200_shim.hpp"

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

// O(1) identity of a DocumentStore / HybridIndex: the heap buffers of its
// tables (they survive moves, so an index returned by value keeps its key)
// plus a checksum of a fixed sample of 64 nodes.  The reference declares a
// built index immutable except through the maintenance API (index.hpp:33),
// and insert_batch / mark_delete below update the device mirror in place,
// so no per-call O(n) walk is needed; the sample catches a destroyed index
// whose buffers were reused by a new one.  Code that edits the structs
// directly calls fusegraph::b200::invalidate_device_mirrors().
uint64_t mix(uint64_t h, uint64_t v) { return (h ^ v) * 1099511628211ull; }
uint64_t bits_of(double d) {
    uint64_t b;
    std::memcpy(&b, &d, 8);
    return b;
}
uint64_t store_sample(const DocumentStore& st) {
    uint64_t h = mix(1469598103934665603ull, st.size());
    h = mix(h, st.dense_dim);
    const std::size_t n = st.size();
    for (std::size_t i = 0; i < 64 && n; ++i) {
        const auto& d = st.docs[(i * 0x9E3779B97F4A7C15ull) % n];
        h = mix(h, d.doc_id);
        h = mix(h, d.deleted);
        h = mix(h, bits_of(d.vector.squared_norm));
        h = mix(h, d.vector.learned.indices.size() + (d.vector.statistical.indices.size() << 20));
    }
    return h;
}
struct StoreKey {
    const void* docs = nullptr;
    std::size_t n = 0;
    uint64_t sample = 0;
    bool operator==(const StoreKey&) const = default;
};
StoreKey store_key(const DocumentStore& st) { return {st.docs.data(), st.size(), store_sample(st)}; }

struct IndexKey {
    StoreKey store;
    const void* semantic = nullptr;
    const void* norm = nullptr;
    uint64_t sample = 0;
    bool operator==(const IndexKey&) const = default;
};
IndexKey index_key(const HybridIndex& x) {
    uint64_t h = mix(1469598103934665603ull, x.degree);
    h = mix(h, x.kg.triplets().size());
    const std::size_t n = x.size();
    for (std::size_t i = 0; i < 64 && n && x.semantic.size() == n; ++i) {
        const std::size_t u = (i * 0x9E3779B97F4A7C15ull) % n;
        for (uint32_t v : x.semantic[u]) h = mix(h, v);
        h = mix(h, x.keyword[u].size());
        h = mix(h, x.logical[u].size());
        h = mix(h, x.norm_order.size() == n ? x.norm_order[u] : ~0ull);
    }
    return {store_key(x.store), x.semantic.data(), x.norm_order.data(), h};
}

// Device mirrors, most recent first (two of each: a 1M-doc mirror is ~5 GB).
struct Mirrors {
    std::mutex mu;
    struct C {
        StoreKey key;
        std::shared_ptr<Corpus> corpus;
    };
    struct I {
        IndexKey key;
        std::shared_ptr<Corpus> corpus;
        fg_index* ix = nullptr;
    };
    std::vector<C> corpora;
    std::vector<I> indexes;
    static constexpr std::size_t kKeep = 2;

    ~Mirrors() { clear(); }
    void clear() {
        for (auto& e : indexes) fg_index_free(e.ix);
        indexes.clear();
        corpora.clear();
    }
    std::shared_ptr<Corpus> corpus(const DocumentStore& st) {
        const StoreKey k = store_key(st);
        for (std::size_t i = 0; i < corpora.size(); ++i)
            if (corpora[i].key == k) {
                std::rotate(corpora.begin(), corpora.begin() + i, corpora.begin() + i + 1);
                return corpora[0].corpus;
            }
        for (auto& e : indexes)  // an index mirror's corpus serves its store
            if (e.key.store == k) return remember(k, e.corpus);
        return remember(k, std::make_shared<Corpus>(st));
    }
    std::shared_ptr<Corpus> remember(const StoreKey& k, std::shared_ptr<Corpus> c) {
        corpora.insert(corpora.begin(), {k, c});
        if (corpora.size() > kKeep) corpora.pop_back();
        return c;
    }
    void adopt(const IndexKey& k, std::shared_ptr<Corpus> c, fg_index* ix) {
        indexes.insert(indexes.begin(), {k, std::move(c), ix});
        if (indexes.size() > kKeep) {
            fg_index_free(indexes.back().ix);
            indexes.pop_back();
        }
    }
    I* find(const IndexKey& k) {
        for (std::size_t i = 0; i < indexes.size(); ++i)
            if (indexes[i].key == k) {
                std::rotate(indexes.begin(), indexes.begin() + i, indexes.begin() + i + 1);
                return &indexes[0];
            }
        return nullptr;
    }
    fg_index* index(const HybridIndex& x);
    // the struct changed through the maintenance API and the mirror `ix`
    // was updated to match: re-key it (and its corpus) to the new content
    void rekey(fg_index* ix, const IndexKey& k) {
        for (auto& e : indexes)
            if (e.ix == ix) {
                for (auto& c : corpora)
                    if (c.corpus == e.corpus) c.key = k.store;
                e.key = k;
            }
    }
    // mark_delete: push the deleted flags to the mirror of the index (if any)
    void set_deleted(const IndexKey& before, const HybridIndex& x) {
        I* e = find(before);
        if (!e) return;
        std::vector<uint8_t> flags(x.size());
        for (std::size_t u = 0; u < x.size(); ++u) flags[u] = x.store.docs[u].deleted ? 1 : 0;
        ok(fg_corpus_set_deleted(e->corpus->h, flags.data()));
        rekey(e->ix, index_key(x));
    }
};
Mirrors g_mirrors;

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

// Device mirror of a HybridIndex: found by key, else uploaded from the host
// struct (its corpus mirror reused when the store is already on the device).
fg_index* Mirrors::index(const HybridIndex& x) {
    const IndexKey k = index_key(x);
    if (I* e = find(k)) return e->ix;
    auto c = corpus(x.store);
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
    fg_index* ix = nullptr;
    ok(fg_index_create(c->h, &kg.v, &gv, &ix));
    adopt(k, c, ix);
    return ix;
}

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
    std::lock_guard<std::mutex> lock(g_mirrors.mu);
    fg_index* ix = g_mirrors.index(index);
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
    std::lock_guard<std::mutex> lock(g_mirrors.mu);
    const auto c = g_mirrors.corpus(store);
    QuerySpec q;
    q.vector = weighted_query;  // already weighted: unit weights keep it as is
    QueryFlat qf(std::span<const QuerySpec>(&q, 1));
    if (qf.v.dense_dim != store.dense_dim && store.size())
        throw Error("dim-mismatch", "dense dimensions differ: " + std::to_string(qf.v.dense_dim) +
                                        " vs " + std::to_string(store.docs[0].vector.dense.dim()));
    ok(fg_batch_scores(c->h, &qf.v, 0, ids.data(), ids.size(), out.data()));
    return out;
}

KnnGraph init_random_graph(const DocumentStore& store, uint32_t k, uint64_t seed, unsigned) {
    std::lock_guard<std::mutex> lock(g_mirrors.mu);
    const auto c = g_mirrors.corpus(store);
    const uint64_t n = store.size();
    std::vector<uint32_t> ids(n * k);
    std::vector<double> sc(n * k);
    std::vector<uint8_t> fr(n * k);
    fg_knn_lists l{n, k, ids.data(), sc.data(), fr.data()};
    ok(fg_knn_init(c->h, k, seed, &l));
    return to_graph(n, k, ids, sc, fr);
}

std::size_t nn_descent_iterate(const DocumentStore& store, KnnGraph& graph, unsigned) {
    std::lock_guard<std::mutex> lock(g_mirrors.mu);
    const auto c = g_mirrors.corpus(store);
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
    ok(fg_knn_iterate(c->h, &l, &changed));
    graph = to_graph(n, k, ids, sc, fr);
    return changed;
}

KnnGraph build_knn_graph(const DocumentStore& store, const KnnBuildParams& p) {
    std::lock_guard<std::mutex> lock(g_mirrors.mu);
    const auto c = g_mirrors.corpus(store);
    const uint64_t n = store.size();
    const uint32_t kk = (n >= 2 && p.k >= n) ? static_cast<uint32_t>(n - 1) : p.k;
    std::vector<uint32_t> ids(n * kk);
    std::vector<double> sc(n * kk);
    std::vector<uint8_t> fr(n * kk);
    fg_knn_lists l{n, kk, ids.data(), sc.data(), fr.data()};
    fg_knn_params kp{p.k, p.max_iterations, p.convergence, p.seed};
    ok(fg_knn_build(c->h, &kp, &l, nullptr));
    return to_graph(n, l.k, ids, sc, fr);
}

RefinedEdges refine_graph(const DocumentStore& store, const KnnGraph& knn, const RefineParams& p,
                          RefineTrace* trace) {
    std::lock_guard<std::mutex> lock(g_mirrors.mu);
    const auto c = g_mirrors.corpus(store);
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
    ok(fg_refine(c->h, &l, &rp, &out, trace ? &tr : nullptr));
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

namespace {
// Host copies of the device index's edge tables into the reference struct.
void pull_edges(fg_index* ix, HybridIndex& index, uint64_t nn) {
    uint32_t deg = 0;
    uint64_t kt = 0, lt = 0;
    ok(fg_index_sizes(ix, &deg, &kt, &lt));
    std::vector<uint32_t> sem(nn * deg), ki(kt), lg(lt * 4), norm(nn);
    std::vector<uint64_t> kp(nn + 1), lp(nn + 1);
    ok(fg_index_export(ix, sem.data(), kp.data(), ki.data(), lp.data(), lg.data(), norm.data()));
    index.semantic.resize(nn);
    index.keyword.resize(nn);
    index.logical.resize(nn);
    for (uint64_t u = 0; u < nn; ++u) {
        index.semantic[u].assign(sem.begin() + u * deg, sem.begin() + (u + 1) * deg);
        index.keyword[u].assign(ki.begin() + kp[u], ki.begin() + kp[u + 1]);
        index.logical[u].clear();
        for (uint64_t e = lp[u]; e < lp[u + 1]; ++e)
            index.logical[u].push_back({lg[4 * e], lg[4 * e + 1], lg[4 * e + 2], lg[4 * e + 3]});
    }
    index.norm_order = std::move(norm);
}
}  // namespace

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
    std::lock_guard<std::mutex> lock(g_mirrors.mu);
    const bool timing = [] {
        const char* te = std::getenv("FGB_HOST_TIMING");
        return te && te[0] != '0';
    }();
    auto t0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!timing) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[shim build] %-20s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    };
    const auto c = g_mirrors.corpus(store);
    mark("corpus mirror");
    KgFlat kf(kg);
    fg_build_params bp{params.degree, params.knn_k, params.knn_iterations, params.seed,
                       params.logical_cap, params.default_entity_hops,
                       params.per_neighbour_keyword_check ? 1 : 0};
    fg_index* ix = nullptr;
    ok(fg_index_build(c->h, &kf.v, &bp, &ix));
    mark("fg_index_build");
    try {
        pull_edges(ix, index, n);
        mark("pull_edges");
    } catch (...) {
        fg_index_free(ix);
        throw;
    }
    index.store = std::move(store);  // the docs buffer (and so the corpus key) moves along
    index.kg = std::move(kg);
    index.entity_map = build_entity_map(index.store);
    mark("host index");
    g_mirrors.adopt(index_key(index), c, ix);  // searches on the result reuse the build's mirror
    mark("adopt");
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
    std::lock_guard<std::mutex> lock(g_mirrors.mu);
    const auto c = g_mirrors.corpus(store);
    QueryFlat qf(std::span<const QuerySpec>(&q, 1));
    std::vector<uint64_t> doc(q.k);
    std::vector<uint32_t> node(q.k), cnt(1);
    std::vector<double> score(q.k);
    std::vector<char> err(256, 0);
    fg_search_results r{q.k, doc.data(), node.data(), score.data(), cnt.data(), nullptr, nullptr,
                        nullptr, err.data(), 256};
    ok(fg_brute_force_topk(c->h, &qf.v, &r));
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

// ---------------------------------------------------------------- maintenance
// update.hpp:33-38.  Both keep the device mirror current in place, so the
// next search runs on the B200 without a re-upload.
namespace fusegraph {

void insert_batch(HybridIndex& index, std::vector<DocumentRecord> new_docs, const InsertParams& params) {
    if (new_docs.empty()) return;
    const uint32_t kk = params.knn_k ? params.knn_k : index.knn_k;
    if (kk < index.degree) throw Error("invalid-k", "insert candidate width must be at least the degree");
    // host validation first, with the reference's checks and messages
    // (update.cpp:44-63), so a bad batch leaves host and device untouched
    for (DocumentRecord& doc : new_docs) {
        const std::string where = "doc " + std::to_string(doc.doc_id);
        if (index.store.id_to_node.count(doc.doc_id))
            throw Error("duplicate-id", where + ": id already in the index");
        if (doc.vector.dense.dim() != index.store.dense_dim)
            throw Error("dim-mismatch", where + ": dense dimension " + std::to_string(doc.vector.dense.dim()) +
                                            " differs from corpus " + std::to_string(index.store.dense_dim));
        validate_fused(doc.vector, where);
        doc.keywords = sorted_unique(std::move(doc.keywords));
        doc.entities = sorted_unique(std::move(doc.entities));
        doc.deleted = false;
        finalize_fused(doc.vector);
    }
    {  // update.cpp:58-62 reports the first doc whose id occurs earlier in the batch
        std::unordered_set<uint64_t> seen;
        seen.reserve(new_docs.size() * 2);
        for (const DocumentRecord& doc : new_docs)
            if (!seen.insert(doc.doc_id).second)
                throw Error("duplicate-id", "doc " + std::to_string(doc.doc_id) + ": id repeated within the batch");
    }
    std::lock_guard<std::mutex> lock(g_mirrors.mu);
    const bool timing = [] {
        const char* te = std::getenv("FGB_HOST_TIMING");
        return te && te[0] != '0';
    }();
    auto t0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!timing) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[shim insert] %-20s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    };
    mark("validate");
    fg_index* ix = g_mirrors.index(index);
    mark("mirror lookup");
    DocumentStore batch;
    batch.dense_dim = index.store.dense_dim;
    batch.docs = new_docs;
    Flat f(batch);
    fg_insert_params p{kk, params.nn_descent_iterations, params.threads};
    mark("flatten");
    ok(fg_index_insert(ix, &f.v, &p));  // device corpus appended, edges linked in HBM
    mark("fg_index_insert");
    // mirror the device result into the reference struct
    const uint64_t n_old = index.size(), nb = new_docs.size();
    index.store.docs.reserve(n_old + nb);
    for (uint64_t i = 0; i < nb; ++i) {
        index.store.id_to_node[new_docs[i].doc_id] = static_cast<uint32_t>(n_old + i);
        for (uint32_t e : new_docs[i].entities) index.entity_map[e].push_back(static_cast<uint32_t>(n_old + i));
        index.store.docs.push_back(std::move(new_docs[i]));
    }
    mark("host docs");
    pull_edges(ix, index, n_old + nb);
    mark("pull_edges");
    g_mirrors.rekey(ix, index_key(index));
    mark("rekey");
}

void mark_delete(HybridIndex& index, std::span<const uint64_t> doc_ids) {
    std::vector<uint32_t> nodes;  // resolve every id first (update.cpp:199-205)
    nodes.reserve(doc_ids.size());
    for (uint64_t id : doc_ids) nodes.push_back(index.store.node_of(id));
    std::lock_guard<std::mutex> lock(g_mirrors.mu);
    const IndexKey before = index_key(index);
    for (uint32_t node : nodes) index.store.docs[node].deleted = true;
    g_mirrors.set_deleted(before, index);
}

namespace b200 {
void invalidate_device_mirrors() {
    std::lock_guard<std::mutex> lock(g_mirrors.mu);
    g_mirrors.clear();
}
}  // namespace b200

}  // namespace fusegraph
