// ref_glue.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A C-ABI over the UNMODIFIED reference library (/root/reference/proj/src,
// compiled with -Dfusegraph=fusegraph_ref by oracle/Makefile into
// oracle/_ref/libfgref.so).  It converts the flat fg_*_view structs of
// include/fg_b200.h into the reference's AoS types and calls the reference's
// public API, so tests and bench.py's reference arm can run the real
// reference on exactly the bytes the GPU path sees.  Only tests/,
// __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) load
// this library.
//
// All calls are wrapped: a fusegraph::Error is returned as FG_ERR with its
// what() string available from fgref_last_error().

#include <algorithm>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "fg_b200.h"
#include "fusegraph/corpus.hpp"
#include "fusegraph/eval.hpp"
#include "fusegraph/index.hpp"
#include "fusegraph/io.hpp"
#include "fusegraph/knn_graph.hpp"
#include "fusegraph/logical.hpp"
#include "fusegraph/refine.hpp"
#include "fusegraph/rng.hpp"
#include "fusegraph/scoring.hpp"
#include "fusegraph/search.hpp"
#include "fusegraph/update.hpp"
#include "fusegraph/synth.hpp"
#include "fusegraph/types.hpp"

namespace R = fusegraph;  // renamed to fusegraph_ref by the build

namespace {

thread_local std::string g_error;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        g_error.clear();
        return FG_OK;
    } catch (const std::exception& e) {
        g_error = e.what();
        return FG_ERR;
    }
}

R::SparseVector sparse_row(const fg_sparse_view& s, uint64_t row) {
    R::SparseVector v;
    if (!s.ptr) return v;
    const uint64_t b = s.ptr[row], e = s.ptr[row + 1];
    v.indices.assign(s.idx + b, s.idx + e);
    v.values.assign(s.val + b, s.val + e);
    return v;
}

std::vector<uint32_t> list_row(const fg_list_view& l, uint64_t row) {
    if (!l.ptr) return {};
    return std::vector<uint32_t>(l.idx + l.ptr[row], l.idx + l.ptr[row + 1]);
}

R::FusedVector query_vector(const fg_query_view& q, uint64_t i) {
    R::FusedVector v;
    v.dense.values.assign(q.dense + i * q.dense_dim, q.dense + (i + 1) * q.dense_dim);
    v.learned = sparse_row(q.learned, i);
    v.statistical = sparse_row(q.statistical, i);
    R::finalize_fused(v);
    return v;
}

R::QuerySpec query_spec(const fg_query_view& q, uint64_t i) {
    R::QuerySpec s;
    s.vector = query_vector(q, i);
    if (q.weights) {
        s.weights.dense = q.weights[i].dense;
        s.weights.learned = q.weights[i].learned;
        s.weights.statistical = q.weights[i].statistical;
        s.weights.entity = q.weights[i].entity;
    }
    s.required_keywords = list_row(q.required_keywords, i);
    s.entities = list_row(q.entities, i);
    if (q.k) s.k = q.k[i];
    if (q.beam_width) s.beam_width = q.beam_width[i];
    if (q.max_entity_hops) s.max_entity_hops = q.max_entity_hops[i];
    return s;
}

R::KnowledgeGraph make_kg(const fg_kg_view* kg) {
    std::vector<R::Triplet> t;
    if (kg)
        for (uint64_t i = 0; i < kg->count; ++i)
            t.push_back({kg->source[i], kg->relation[i], kg->target[i]});
    return R::KnowledgeGraph(std::move(t));
}

// CSR mirror of a DocumentStore, used to hand generated data back to Python.
struct CsrCorpus {
    uint32_t dim = 0, ldim = 0, sdim = 0;
    std::vector<float> dense;
    std::vector<uint64_t> lptr{0}, sptr{0}, kptr{0}, eptr{0}, doc_id;
    std::vector<uint32_t> lidx, sidx, kidx, eidx;
    std::vector<float> lval, sval;
    std::vector<uint8_t> deleted;
    std::vector<uint32_t> ts, tr, tt;

    void fill(const R::DocumentStore& st, const R::KnowledgeGraph* kg) {
        dim = st.dense_dim;
        ldim = st.learned_dim;
        sdim = st.statistical_dim;
        dense.reserve(st.size() * dim);
        for (const auto& d : st.docs) {
            dense.insert(dense.end(), d.vector.dense.values.begin(), d.vector.dense.values.end());
            lidx.insert(lidx.end(), d.vector.learned.indices.begin(), d.vector.learned.indices.end());
            lval.insert(lval.end(), d.vector.learned.values.begin(), d.vector.learned.values.end());
            lptr.push_back(lidx.size());
            sidx.insert(sidx.end(), d.vector.statistical.indices.begin(),
                        d.vector.statistical.indices.end());
            sval.insert(sval.end(), d.vector.statistical.values.begin(),
                        d.vector.statistical.values.end());
            sptr.push_back(sidx.size());
            kidx.insert(kidx.end(), d.keywords.begin(), d.keywords.end());
            kptr.push_back(kidx.size());
            eidx.insert(eidx.end(), d.entities.begin(), d.entities.end());
            eptr.push_back(eidx.size());
            doc_id.push_back(d.doc_id);
            deleted.push_back(d.deleted ? 1 : 0);
        }
        if (kg)
            for (const auto& t : kg->triplets()) {
                ts.push_back(t.source);
                tr.push_back(t.relation);
                tt.push_back(t.target);
            }
    }
    void view(fg_corpus_view* v, fg_kg_view* k) const {
        if (v) {
            std::memset(v, 0, sizeof *v);
            v->n = doc_id.size();
            v->dense_dim = dim;
            v->learned_dim = ldim;
            v->statistical_dim = sdim;
            v->dense = dense.data();
            v->learned = {lptr.data(), lidx.data(), lval.data()};
            v->statistical = {sptr.data(), sidx.data(), sval.data()};
            v->keywords = {kptr.data(), kidx.data()};
            v->entities = {eptr.data(), eidx.data()};
            v->doc_id = doc_id.data();
            v->deleted = deleted.data();
        }
        if (k) *k = {ts.size(), ts.data(), tr.data(), tt.data()};
    }
};

R::SynthParams synth_params(const fg_synth_params* p) {
    R::SynthParams s;
    s.docs = p->docs;
    s.dense_dim = p->dense_dim;
    s.clusters = p->clusters;
    s.cluster_spread = p->cluster_spread;
    s.learned_vocab = p->learned_vocab;
    s.learned_nnz = p->learned_nnz;
    s.statistical_vocab = p->statistical_vocab;
    s.statistical_nnz = p->statistical_nnz;
    s.zipf_exponent = p->zipf_exponent;
    s.entity_vocab = p->entity_vocab;
    s.entity_rate = p->entity_rate;
    s.max_entities_per_doc = p->max_entities_per_doc;
    s.kg_triplets = p->kg_triplets;
    s.relation_vocab = p->relation_vocab;
    s.chains = p->chains;
    s.answers_per_chain = p->answers_per_chain;
    s.seed = p->seed;
    return s;
}

void put_results(const std::vector<R::SearchResult>& rs, fg_search_results* out) {
    for (std::size_t i = 0; i < rs.size(); ++i) {
        const auto& r = rs[i];
        const uint32_t h = static_cast<uint32_t>(std::min<std::size_t>(r.hits.size(), out->hit_stride));
        out->hit_count[i] = h;
        for (uint32_t j = 0; j < h; ++j) {
            out->doc_id[i * out->hit_stride + j] = r.hits[j].doc_id;
            out->node[i * out->hit_stride + j] = r.hits[j].node;
            out->score[i * out->hit_stride + j] = r.hits[j].score;
        }
        if (out->expanded) out->expanded[i] = r.expanded;
        if (out->scored) out->scored[i] = 0;
        if (out->warnings) {
            uint32_t w = 0;
            for (const auto& s : r.warnings) {
                if (s == "entity-fallback") w |= FG_WARN_ENTITY_FALLBACK;
                if (s == "keyword-shortfall") w |= FG_WARN_KEYWORD_SHORTFALL;
            }
            out->warnings[i] = w;
        }
        if (out->errors && out->error_stride) {
            char* dst = out->errors + i * out->error_stride;
            std::strncpy(dst, r.error.c_str(), out->error_stride - 1);
            dst[out->error_stride - 1] = 0;
        }
    }
}

R::KnnGraph knn_from(const fg_knn_lists* l) {
    R::KnnGraph g;
    g.k = l->k;
    g.lists.resize(l->n);
    for (uint64_t u = 0; u < l->n; ++u) {
        g.lists[u].resize(l->k);
        for (uint32_t j = 0; j < l->k; ++j) {
            const uint64_t s = u * l->k + j;
            g.lists[u][j] = {l->ids[s], l->scores[s], l->fresh[s] != 0};
        }
    }
    return g;
}

void knn_to(const R::KnnGraph& g, fg_knn_lists* l) {
    l->k = g.k;
    for (uint64_t u = 0; u < g.lists.size(); ++u)
        for (uint32_t j = 0; j < g.k; ++j) {
            const uint64_t s = u * g.k + j;
            const auto& e = g.lists[u][j];
            l->ids[s] = e.id;
            l->scores[s] = e.score;
            l->fresh[s] = e.fresh ? 1 : 0;
        }
}

}  // namespace

struct fgref_synth {
    CsrCorpus csr;
    std::vector<R::ChainInfo> chains;
};
struct fgref_store {
    R::DocumentStore store;
    R::KnowledgeGraph kg;
};
struct fgref_index {
    R::HybridIndex index;
};

extern "C" {

const char* fgref_last_error(void) { return g_error.c_str(); }

// ---- synthetic data through the reference generator (synth.cpp:140-222)
int fgref_synth_generate(const fg_synth_params* p, fgref_synth** out) {
    return guarded([&] {
        auto h = std::make_unique<fgref_synth>();
        R::SynthData data = R::generate_corpus(synth_params(p));
        h->csr.fill(data.store, &data.kg);
        h->chains = std::move(data.chains);
        *out = h.release();
    });
}
int fgref_synth_view(const fgref_synth* h, fg_corpus_view* v, fg_kg_view* kg, uint64_t* chains) {
    h->csr.view(v, kg);
    if (chains) *chains = h->chains.size();
    return FG_OK;
}
int fgref_synth_chain(const fgref_synth* h, uint64_t c, uint32_t ent[3], uint64_t docs[2],
                      uint64_t* answers, float* dense, uint32_t* lnnz, uint32_t* lidx, float* lval,
                      uint32_t* snnz, uint32_t* sidx, float* sval) {
    const auto& ch = h->chains.at(c);
    ent[0] = ch.e0;
    ent[1] = ch.e1;
    ent[2] = ch.e2;
    docs[0] = ch.seed_doc;
    docs[1] = ch.bridge_doc;
    std::copy(ch.answer_docs.begin(), ch.answer_docs.end(), answers);
    std::copy(ch.query_vector.dense.values.begin(), ch.query_vector.dense.values.end(), dense);
    *lnnz = static_cast<uint32_t>(ch.query_vector.learned.nnz());
    std::copy(ch.query_vector.learned.indices.begin(), ch.query_vector.learned.indices.end(), lidx);
    std::copy(ch.query_vector.learned.values.begin(), ch.query_vector.learned.values.end(), lval);
    *snnz = static_cast<uint32_t>(ch.query_vector.statistical.nnz());
    std::copy(ch.query_vector.statistical.indices.begin(), ch.query_vector.statistical.indices.end(),
              sidx);
    std::copy(ch.query_vector.statistical.values.begin(), ch.query_vector.statistical.values.end(),
              sval);
    return FG_OK;
}
void fgref_synth_free(fgref_synth* h) { delete h; }

// random_query_vector + random_simplex_weights from SplitMix64(mix_seed(seed, stream)),
// fixed nnz per query (the generator draws exactly min(nnz, vocab) terms).
int fgref_synth_queries(const fg_synth_params* p, uint64_t stream, uint64_t count, int with_weights,
                        float* dense, uint32_t* lidx, float* lval, uint32_t* sidx, float* sval,
                        fg_weights* weights) {
    return guarded([&] {
        const R::SynthParams sp = synth_params(p);
        R::SplitMix64 rng(R::mix_seed(p->seed, stream));
        const uint32_t ln = std::min(p->learned_nnz, p->learned_vocab);
        const uint32_t sn = std::min(p->statistical_nnz, p->statistical_vocab);
        for (uint64_t i = 0; i < count; ++i) {
            R::FusedVector v = R::random_query_vector(sp, rng);
            std::copy(v.dense.values.begin(), v.dense.values.end(), dense + i * p->dense_dim);
            std::copy(v.learned.indices.begin(), v.learned.indices.end(), lidx + i * ln);
            std::copy(v.learned.values.begin(), v.learned.values.end(), lval + i * ln);
            std::copy(v.statistical.indices.begin(), v.statistical.indices.end(), sidx + i * sn);
            std::copy(v.statistical.values.begin(), v.statistical.values.end(), sval + i * sn);
            if (with_weights) {
                R::Weights w = R::random_simplex_weights(rng);
                weights[i] = {w.dense, w.learned, w.statistical, w.entity};
            }
        }
    });
}

// ---- DocumentStore from flat arrays (make_document + validate_corpus)
int fgref_store_create(const fg_corpus_view* v, const fg_kg_view* kg, fgref_store** out) {
    return guarded([&] {
        auto h = std::make_unique<fgref_store>();
        h->store.docs.reserve(v->n);
        for (uint64_t i = 0; i < v->n; ++i) {
            R::DenseVector d;
            d.values.assign(v->dense + i * v->dense_dim, v->dense + (i + 1) * v->dense_dim);
            std::optional<std::vector<uint32_t>> kw;
            if (v->keywords.ptr) kw = list_row(v->keywords, i);
            h->store.docs.push_back(R::make_document(v->doc_id ? v->doc_id[i] : i, std::move(d),
                                                     sparse_row(v->learned, i),
                                                     sparse_row(v->statistical, i), kw,
                                                     list_row(v->entities, i)));
            if (v->deleted) h->store.docs.back().deleted = v->deleted[i] != 0;
        }
        R::validate_corpus(h->store);
        h->kg = make_kg(kg);
        *out = h.release();
    });
}
void fgref_store_free(fgref_store* h) { delete h; }

int fgref_store_sqnorm(const fgref_store* h, double* out) {
    for (std::size_t i = 0; i < h->store.size(); ++i) out[i] = h->store.docs[i].vector.squared_norm;
    return FG_OK;
}

// ---- scoring.hpp / corpus.hpp
int fgref_build_query_vector(const fg_query_view* q, uint64_t i, float* dense_out, uint32_t* lnnz,
                             float* lval, uint32_t* snnz, float* sval, double* sqnorm) {
    return guarded([&] {
        R::Weights w;
        w.dense = q->weights[i].dense;
        w.learned = q->weights[i].learned;
        w.statistical = q->weights[i].statistical;
        w.entity = q->weights[i].entity;
        R::FusedVector v = R::build_query_vector(query_vector(*q, i), w);
        std::copy(v.dense.values.begin(), v.dense.values.end(), dense_out);
        *lnnz = static_cast<uint32_t>(v.learned.nnz());
        std::copy(v.learned.values.begin(), v.learned.values.end(), lval);
        *snnz = static_cast<uint32_t>(v.statistical.nnz());
        std::copy(v.statistical.values.begin(), v.statistical.values.end(), sval);
        *sqnorm = v.squared_norm;
    });
}

int fgref_batch_scores(const fgref_store* h, const fg_query_view* q, uint64_t qi,
                       const uint32_t* ids, uint64_t m, unsigned threads, double* out) {
    return guarded([&] {
        R::Weights w;
        w.dense = q->weights[qi].dense;
        w.learned = q->weights[qi].learned;
        w.statistical = q->weights[qi].statistical;
        w.entity = q->weights[qi].entity;
        const R::FusedVector wq = R::build_query_vector(query_vector(*q, qi), w);
        auto s = R::batch_scores(wq, std::span<const uint32_t>(ids, m), h->store, threads);
        std::copy(s.begin(), s.end(), out);
    });
}

int fgref_pair_scores(const fgref_store* h, const uint32_t* a, const uint32_t* b, uint64_t m,
                      double* out) {
    return guarded([&] {
        for (uint64_t i = 0; i < m; ++i)
            out[i] = R::hybrid_score(h->store.doc(a[i]).vector, h->store.doc(b[i]).vector);
    });
}

// ---- knn_graph.hpp
int fgref_knn_init(const fgref_store* h, uint32_t k, uint64_t seed, unsigned threads,
                   fg_knn_lists* out) {
    return guarded([&] { knn_to(R::init_random_graph(h->store, k, seed, threads), out); });
}
int fgref_knn_iterate(const fgref_store* h, fg_knn_lists* lists, unsigned threads,
                      uint64_t* changed) {
    return guarded([&] {
        R::KnnGraph g = knn_from(lists);
        *changed = R::nn_descent_iterate(h->store, g, threads);
        knn_to(g, lists);
    });
}
int fgref_knn_build(const fgref_store* h, const fg_knn_params* p, unsigned threads,
                    fg_knn_lists* out) {
    return guarded([&] {
        R::KnnBuildParams kp;
        kp.k = p->k;
        kp.max_iterations = p->max_iterations;
        kp.convergence = p->convergence;
        kp.seed = p->seed;
        kp.threads = threads;
        knn_to(R::build_knn_graph(h->store, kp), out);
    });
}

// ---- refine.hpp
int fgref_refine(const fgref_store* h, const fg_knn_lists* knn, const fg_refine_params* p,
                 unsigned threads, fg_refined* out, fg_refine_trace* trace) {
    return guarded([&] {
        R::RefineParams rp;
        rp.degree = p->degree;
        rp.per_neighbour_keyword_check = p->per_neighbour_keyword_check != 0;
        rp.threads = threads;
        R::RefineTrace tr;
        R::RefinedEdges e = R::refine_graph(h->store, knn_from(knn), rp, trace ? &tr : nullptr);
        const uint32_t k = knn->k;
        for (uint64_t u = 0; u < knn->n; ++u) {
            std::copy(e.semantic[u].begin(), e.semantic[u].end(), out->semantic + u * p->degree);
            out->keyword_count[u] = static_cast<uint32_t>(e.keyword[u].size());
            std::copy(e.keyword[u].begin(), e.keyword[u].end(), out->keyword + u * out->keyword_cap);
            if (!trace) continue;
            for (uint32_t j = 0; j < tr.ordered[u].size(); ++j) {
                if (trace->ordered_ids) trace->ordered_ids[u * k + j] = tr.ordered[u][j].id;
                if (trace->ordered_scores) trace->ordered_scores[u * k + j] = tr.ordered[u][j].score;
                if (trace->detours) trace->detours[u * k + j] = tr.detours[u][j];
            }
            if (trace->kept_count) trace->kept_count[u] = static_cast<uint32_t>(tr.kept[u].size());
            if (trace->kept)
                std::copy(tr.kept[u].begin(), tr.kept[u].end(), trace->kept + u * p->degree);
        }
    });
}

// ---- index.hpp (takes ownership of the store's contents)
int fgref_index_build(fgref_store* h, const fg_build_params* p, unsigned threads,
                      fgref_index** out) {
    return guarded([&] {
        R::BuildParams bp;
        bp.degree = p->degree;
        bp.knn_k = p->knn_k;
        bp.knn_iterations = p->knn_iterations;
        bp.seed = p->seed;
        bp.logical_cap = p->logical_cap;
        bp.default_entity_hops = p->default_entity_hops;
        bp.per_neighbour_keyword_check = p->per_neighbour_keyword_check != 0;
        bp.threads = threads;
        auto ix = std::make_unique<fgref_index>();
        ix->index = R::build_hybrid_index(std::move(h->store), std::move(h->kg), bp);
        *out = ix.release();
    });
}

// HybridIndex assembled from given edge tables (no build): the reference
// search then runs on exactly the graph the GPU produced.
int fgref_index_create(fgref_store* h, const fg_graph_view* g, uint32_t knn_k, fgref_index** out) {
    return guarded([&] {
        auto ix = std::make_unique<fgref_index>();
        R::HybridIndex& x = ix->index;
        const std::size_t n = h->store.size();
        x.degree = g->degree;
        x.knn_k = knn_k;
        x.semantic.resize(n);
        x.keyword.resize(n);
        x.logical.resize(n);
        for (std::size_t u = 0; u < n; ++u) {
            x.semantic[u].assign(g->semantic + u * g->degree, g->semantic + (u + 1) * g->degree);
            x.keyword[u] = list_row(g->keyword, u);
            if (g->logical_ptr)
                for (uint64_t e = g->logical_ptr[u]; e < g->logical_ptr[u + 1]; ++e)
                    x.logical[u].push_back({g->logical[4 * e], g->logical[4 * e + 1],
                                            g->logical[4 * e + 2], g->logical[4 * e + 3]});
        }
        x.store = std::move(h->store);
        x.kg = std::move(h->kg);
        x.entity_map = R::build_entity_map(x.store);
        if (g->norm_order)
            x.norm_order.assign(g->norm_order, g->norm_order + n);
        else
            R::rebuild_norm_order(x);
        *out = ix.release();
    });
}
void fgref_index_free(fgref_index* h) { delete h; }

int fgref_index_sizes(const fgref_index* h, uint32_t* degree, uint64_t* kw_total,
                      uint64_t* logical_total) {
    const auto& x = h->index;
    *degree = x.degree;
    uint64_t a = 0, b = 0;
    for (std::size_t u = 0; u < x.size(); ++u) {
        a += x.keyword[u].size();
        b += x.logical[u].size();
    }
    *kw_total = a;
    *logical_total = b;
    return FG_OK;
}

int fgref_index_export(const fgref_index* h, uint32_t* semantic, uint64_t* kptr, uint32_t* kidx,
                       uint64_t* lptr, uint32_t* logical, uint32_t* norm_order) {
    const auto& x = h->index;
    uint64_t a = 0, b = 0;
    if (kptr) kptr[0] = 0;
    if (lptr) lptr[0] = 0;
    for (std::size_t u = 0; u < x.size(); ++u) {
        if (semantic) std::copy(x.semantic[u].begin(), x.semantic[u].end(), semantic + u * x.degree);
        for (uint32_t v : x.keyword[u]) {
            if (kidx) kidx[a] = v;
            ++a;
        }
        if (kptr) kptr[u + 1] = a;
        for (const auto& e : x.logical[u]) {
            if (logical) {
                logical[4 * b] = e.source;
                logical[4 * b + 1] = e.relation;
                logical[4 * b + 2] = e.target;
                logical[4 * b + 3] = e.via;
            }
            ++b;
        }
        if (lptr) lptr[u + 1] = b;
    }
    if (norm_order) std::copy(x.norm_order.begin(), x.norm_order.end(), norm_order);
    return FG_OK;
}

int fgref_index_set_deleted(fgref_index* h, const uint8_t* flags) {
    for (std::size_t i = 0; i < h->index.size(); ++i) h->index.store.docs[i].deleted = flags[i] != 0;
    return FG_OK;
}

int fgref_index_serialize(const fgref_index* h, const char* path, uint64_t* bytes) {
    return guarded([&] { *bytes = R::serialize_index(h->index, path); });
}
int fgref_index_deserialize(const char* path, fgref_index** out) {
    return guarded([&] {
        auto ix = std::make_unique<fgref_index>();
        ix->index = R::deserialize_index(path, false);
        *out = ix.release();
    });
}
// insert_batch (update.hpp:33): documents built exactly as fgref_store_create
// builds them (make_document), then the reference's own insertion.
int fgref_index_insert(fgref_index* h, const fg_corpus_view* v, uint32_t knn_k, uint32_t iters) {
    return guarded([&] {
        std::vector<R::DocumentRecord> docs;
        for (uint64_t i = 0; i < v->n; ++i) {
            R::DenseVector d;
            d.values.assign(v->dense + i * v->dense_dim, v->dense + (i + 1) * v->dense_dim);
            std::optional<std::vector<uint32_t>> kw;
            if (v->keywords.ptr) kw = list_row(v->keywords, i);
            docs.push_back(R::make_document(v->doc_id ? v->doc_id[i] : i, std::move(d), sparse_row(v->learned, i),
                                            sparse_row(v->statistical, i), kw, list_row(v->entities, i)));
        }
        R::InsertParams p;
        p.knn_k = knn_k;
        p.nn_descent_iterations = iters;
        R::insert_batch(h->index, std::move(docs), p);
    });
}

int fgref_index_validate(const fgref_index* h) {
    return guarded([&] { R::validate_index(h->index); });
}

// ---- search.hpp / eval.hpp
int fgref_batch_query(const fgref_index* h, const fg_query_view* q, const fg_search_opts* o,
                      unsigned threads, fg_search_results* out) {
    return guarded([&] {
        std::vector<R::QuerySpec> qs;
        qs.reserve(q->count);
        for (uint64_t i = 0; i < q->count; ++i) qs.push_back(query_spec(*q, i));
        R::SearchOptions opts;
        if (o) {
            opts.entry_count = o->entry_count;
            opts.conjunctive_filter = o->conjunctive_filter != 0;
        }
        put_results(R::batch_query(h->index, qs, threads, opts), out);
    });
}

// Same, with query conversion outside the timed region: prepare once, run many.
struct fgref_queries {
    std::vector<R::QuerySpec> qs;
};
int fgref_queries_create(const fg_query_view* q, fgref_queries** out) {
    return guarded([&] {
        auto h = std::make_unique<fgref_queries>();
        for (uint64_t i = 0; i < q->count; ++i) h->qs.push_back(query_spec(*q, i));
        *out = h.release();
    });
}
void fgref_queries_free(fgref_queries* h) { delete h; }
int fgref_batch_query_prepared(const fgref_index* h, const fgref_queries* q, uint64_t begin,
                               uint64_t end, const fg_search_opts* o, unsigned threads,
                               fg_search_results* out) {
    return guarded([&] {
        R::SearchOptions opts;
        if (o) {
            opts.entry_count = o->entry_count;
            opts.conjunctive_filter = o->conjunctive_filter != 0;
        }
        std::span<const R::QuerySpec> sub(q->qs.data() + begin, end - begin);
        put_results(R::batch_query(h->index, sub, threads, opts), out);
    });
}

int fgref_brute_force(const fgref_store* h, const fg_query_view* q, unsigned threads,
                      fg_search_results* out) {
    return guarded([&] {
        std::vector<R::SearchResult> rs(q->count);
        for (uint64_t i = 0; i < q->count; ++i) rs[i].hits = R::brute_force_topk(h->store, query_spec(*q, i), threads);
        put_results(rs, out);
    });
}
int fgref_index_brute_force(const fgref_index* h, const fg_query_view* q, unsigned threads,
                            fg_search_results* out) {
    return guarded([&] {
        std::vector<R::SearchResult> rs(q->count);
        for (uint64_t i = 0; i < q->count; ++i)
            rs[i].hits = R::brute_force_topk(h->index.store, query_spec(*q, i), threads);
        put_results(rs, out);
    });
}

}  // extern "C"
