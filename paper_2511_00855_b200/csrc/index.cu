// index.cu — build_hybrid_index orchestration (index.cpp:25-71) over the
// device kernels, plus the host-side integer stages the survey keeps on the
// host: entity map and logical edges (logical.cpp:9-68), KG adjacency
// (types.cpp:29-45) and the norm order (index.cpp:12-23).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <cmath>
#include <unordered_set>
#include <unordered_map>
#include <array>
#include <chrono>
#include <numeric>
#include <exception>
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

std::shared_ptr<SearchWorkspace> search_workspace(int device) {
    static std::mutex mu;
    static std::map<int, std::weak_ptr<SearchWorkspace>> live;
    std::lock_guard<std::mutex> lock(mu);
    std::shared_ptr<SearchWorkspace> w = live[device].lock();
    if (!w) {
        w = std::make_shared<SearchWorkspace>();
        live[device] = w;
    }
    return w;
}

void index_finish(fg_index& ix, const fg_kg_view* kgv) {
    fg_corpus& c = *ix.corpus;
    ix.device = c.device;
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


// ---------------------------------------------------------------- insert_batch
// insert_batch (update.cpp:33-197) on the device index.  Candidate sources:
// (a) the batched beam search of each new doc over the current index (unit
// weights, k = kk, beam 2kk; search.cpp), (b) NN-Descent among the batch
// (knn.cu) seeded mix_seed(build_seed, n_old); then the per-node refinery
// (refine_node_kernel) over the merged candidates, the batch-local reverse
// half, keyword recycling and logical edges for the new nodes, and the
// deterministic weakest-reverse-slot replacement on existing nodes (host loop
// over exact GPU pair scores), the norm order rebuilt.
namespace {

struct Cand {
    uint32_t id;
    double score;
};

void check_sparse(const fg_sparse_view& sv, uint64_t i, const std::string& where, const char* path) {
    if (!sv.ptr) return;
    for (uint64_t j = sv.ptr[i]; j < sv.ptr[i + 1]; ++j) {
        if (j > sv.ptr[i] && sv.idx[j] <= sv.idx[j - 1])
            throw Error("unsorted-sparse", where + ": " + path + " indices must be strictly ascending");
        if (!std::isfinite(sv.val[j]))
            throw Error("nonfinite-value", where + ": " + path + " holds a non-finite value");
        if (sv.val[j] == 0.0f)
            throw Error("zero-sparse-value", where + ": " + path + " stores an explicit zero at index " +
                                                 std::to_string(sv.idx[j]));
    }
}

// check_sparse's conditions without building messages (the common, valid case)
bool sparse_ok(const fg_sparse_view& sv, uint64_t i) {
    if (!sv.ptr) return true;
    for (uint64_t j = sv.ptr[i]; j < sv.ptr[i + 1]; ++j)
        if ((j > sv.ptr[i] && sv.idx[j] <= sv.idx[j - 1]) || !std::isfinite(sv.val[j]) || sv.val[j] == 0.0f)
            return false;
    return true;
}

void insert_batch_device(fg_index& ix, const fg_corpus_view& in, const fg_insert_params& p) {
    fg_corpus& c = *ix.corpus;
    cudaStream_t s = c.stream;
    const uint64_t n_old = c.n, batch = in.n;
    const uint32_t d = ix.degree;
    const uint32_t kk = p.knn_k ? p.knn_k : ix.knn_k;
    if (batch == 0) return;
    if (kk < d) throw Error("invalid-k", "insert candidate width must be at least the degree");
    HostTimer mark_t("insert");
    auto mark = [&](const char* what) { mark_t.mark(what); };

    // ---- validate before touching anything (update.cpp:43-63)
    std::unordered_set<uint64_t> ids(c.doc_id.begin(), c.doc_id.end());
    std::vector<uint64_t> doc_id(batch);
    // value checks of every row on host threads; the errors are raised below
    // in the reference's order (first offending doc, its first failed check)
    std::vector<uint8_t> bad(batch, 0);
    parallel_rows(batch, [&](uint64_t i) {
        bool ok = true;
        for (uint32_t j = 0; j < in.dense_dim && ok; ++j) ok = std::isfinite(in.dense[i * in.dense_dim + j]);
        bad[i] = !(ok && sparse_ok(in.learned, i) && sparse_ok(in.statistical, i));
    });
    for (uint64_t i = 0; i < batch; ++i) {
        doc_id[i] = in.doc_id ? in.doc_id[i] : n_old + i;
        auto where = [&] { return "doc " + std::to_string(doc_id[i]); };  // (built only for an error)
        if (ids.count(doc_id[i])) throw Error("duplicate-id", where() + ": id already in the index");
        if (in.dense_dim != c.dim)
            throw Error("dim-mismatch", where() + ": dense dimension " + std::to_string(in.dense_dim) +
                                            " differs from corpus " + std::to_string(c.dim));
        if (!bad[i]) continue;
        for (uint32_t j = 0; j < in.dense_dim; ++j)
            if (!std::isfinite(in.dense[i * in.dense_dim + j]))
                throw Error("nonfinite-value", where() + ": dense holds a non-finite value");
        check_sparse(in.learned, i, where(), "learned");
        check_sparse(in.statistical, i, where(), "statistical");
    }
    {  // update.cpp:58-62 reports the first doc whose id occurs earlier in the batch
        std::unordered_set<uint64_t> seen;
        seen.reserve(batch * 2);
        for (uint64_t i = 0; i < batch; ++i)
            if (!seen.insert(doc_id[i]).second)
                throw Error("duplicate-id", "doc " + std::to_string(doc_id[i]) + ": id repeated within the batch");
    }
    // keywords / entities sorted unique (update.cpp:58-59), keywords default to
    // the statistical support (make_document, corpus.cpp:113-117)
    auto sorted_unique = [&](const fg_list_view& lv, bool kw) {
        HostList out;
        for (uint64_t i = 0; i < batch; ++i) {
            std::vector<uint32_t> row;
            if (lv.ptr)
                row.assign(lv.idx + lv.ptr[i], lv.idx + lv.ptr[i + 1]);
            else if (kw && in.statistical.ptr)
                row.assign(in.statistical.idx + in.statistical.ptr[i], in.statistical.idx + in.statistical.ptr[i + 1]);
            std::sort(row.begin(), row.end());
            row.erase(std::unique(row.begin(), row.end()), row.end());
            out.idx.insert(out.idx.end(), row.begin(), row.end());
            out.ptr.push_back(out.idx.size());
        }
        return out;
    };
    const HostList kws = sorted_unique(in.keywords, true), ents = sorted_unique(in.entities, false);

    fg_corpus_view v = in;
    v.doc_id = doc_id.data();
    v.deleted = nullptr;
    v.keywords = fg_list_view{kws.ptr.data(), kws.idx.data()};
    v.entities = fg_list_view{ents.ptr.data(), ents.idx.data()};
    mark("validate");
    // ---- append the documents first (update.cpp:94-103): the new rows have no
    // edges yet, so (a) cannot reach them, and (b) reads them in place
    const CorpusMark before = corpus_mark(c);
    corpus_append(c, v);
    struct Rollback {
        fg_corpus& c;
        CorpusMark m;
        bool armed = true;
        ~Rollback() {
            if (armed) corpus_rollback(c, m);
        }
    } rollback{c, before};
    mark("corpus append");

    // ---- (b) neighbour-descent among the batch itself (update.cpp:71-88), on
    // a zero-copy view of rows [n_old, n_old + batch) (local ids 0..batch-1, as
    // the reference's batch store), on its own stream from a helper thread
    // while (a) searches the current graph
    std::vector<std::vector<Cand>> from_index(batch), from_batch(batch);
    std::exception_ptr b_err;
    std::thread tb([&] {
        try {
            FGB_CUDA(cudaSetDevice(c.device));
            if (batch > 1) {
                fg_corpus view;  // non-owning: its DevBufs stay empty
                view.device = c.device;
                view.n = batch;
                view.dim = c.dim;
                view.dstride = c.dstride;
                view.max_lnnz = c.max_lnnz;
                view.max_snnz = c.max_snnz;
                view.l_vocab = c.l_vocab;
                view.s_vocab = c.s_vocab;
                view.learned_dim = c.learned_dim;
                view.statistical_dim = c.statistical_dim;
                view.max_sqnorm = c.max_sqnorm;
                view.max_dnorm = c.max_dnorm;
                view.dc = corpus_rows(c.dc, n_old, batch);
                FGB_CUDA(cudaStreamCreateWithFlags(&view.stream, cudaStreamNonBlocking));
                struct StreamGuard {
                    cudaStream_t s;
                    ~StreamGuard() { cudaStreamDestroy(s); }
                } sg{view.stream};
                DevKnn g;
                const uint32_t kb = std::min<uint32_t>(kk, static_cast<uint32_t>(batch - 1));
                knn_build_device(view, kb, p.nn_descent_iterations, 0.01, mix_seed(ix.seed, n_old), g, view.stream);
                std::vector<uint32_t> gid(batch * g.k);
                std::vector<double> gsc(batch * g.k);
                g.ids.download(gid.data(), gid.size(), view.stream);
                g.scores.download(gsc.data(), gsc.size(), view.stream);
                FGB_CUDA(cudaStreamSynchronize(view.stream));
                for (uint64_t i = 0; i < batch; ++i)
                    for (uint32_t j = 0; j < g.k; ++j)
                        from_batch[i].push_back({static_cast<uint32_t>(n_old + gid[i * g.k + j]), gsc[i * g.k + j]});
            }
        } catch (...) {
            b_err = std::current_exception();
        }
    });
    struct Joiner {
        std::thread& t;
        ~Joiner() {
            if (t.joinable()) t.join();
        }
    } joiner{tb};
    // ---- (a) nearest existing nodes through the current graph (update.cpp:18-29)
    {
        std::vector<fg_weights> w(batch, fg_weights{1.f, 1.f, 1.f, 0.f});
        std::vector<uint32_t> kq(batch, kk), bq(batch, 2 * kk);
        fg_query_view q{};
        q.count = batch;
        q.dense_dim = in.dense_dim;
        q.dense = in.dense;
        q.learned = in.learned;
        q.statistical = in.statistical;
        q.weights = w.data();
        q.k = kq.data();
        q.beam_width = bq.data();
        std::vector<uint64_t> rd(batch * kk);
        std::vector<uint32_t> rn(batch * kk), rc(batch);
        std::vector<double> rs(batch * kk);
        std::vector<char> errs(batch * 256);
        fg_search_results r{};
        r.hit_stride = kk;
        r.doc_id = rd.data();
        r.node = rn.data();
        r.score = rs.data();
        r.hit_count = rc.data();
        r.errors = errs.data();
        r.error_stride = 256;
        fg_search_opts o{32, 1};  // SearchOptions{} (kDefaultEntryCount, index.hpp:55)
        if (fg_batch_query(&ix, &q, &o, &r) != FG_OK) throw Error(fg_last_error_code(), fg_last_error_message());
        for (uint64_t i = 0; i < batch; ++i) {
            if (errs[i * 256]) {
                const std::string e(&errs[i * 256]);
                throw Error(e.substr(0, e.find(':')), e);
            }
            for (uint32_t j = 0; j < rc[i]; ++j) from_index[i].push_back({rn[i * kk + j], rs[i * kk + j]});
        }
    }
    mark("search candidates");
    tb.join();
    if (b_err) std::rethrow_exception(b_err);
    for (uint64_t i = 0; i < batch; ++i)
        if (from_index[i].size() + from_batch[i].size() < d)
            throw Error("corpus-too-small", "doc " + std::to_string(doc_id[i]) + ": only " +
                                                std::to_string(from_index[i].size() + from_batch[i].size()) +
                                                " insert candidates for degree " + std::to_string(d));
    mark("batch nn-descent");
    rollback.armed = false;  // past the last check: the insert commits
    // ---- merged candidates, the per-node refinery (update.cpp:105-125)
    std::vector<std::vector<Cand>> cands(batch);
    for (uint64_t i = 0; i < batch; ++i) {
        auto& cl = cands[i];
        cl = from_index[i];
        cl.insert(cl.end(), from_batch[i].begin(), from_batch[i].end());
        std::sort(cl.begin(), cl.end(), [](const Cand& a, const Cand& b) {
            if (a.score != b.score) return a.score > b.score;
            return a.id < b.id;
        });
        if (cl.size() > kk) cl.resize(kk);
    }
    std::vector<std::vector<uint32_t>> kept(batch), recycled(batch), ordered(batch);
    for (uint64_t i0 = 0; i0 < batch;) {  // runs of equal candidate counts share a launch
        uint64_t i1 = i0 + 1;
        while (i1 < batch && cands[i1].size() == cands[i0].size()) ++i1;
        const uint32_t L = static_cast<uint32_t>(cands[i0].size());
        const uint64_t rows = i1 - i0;
        DevKnn g;
        g.alloc(rows, L);
        std::vector<uint32_t> gid(rows * L);
        std::vector<double> gsc(rows * L);
        for (uint64_t r = 0; r < rows; ++r)
            for (uint32_t j = 0; j < L; ++j) {
                gid[r * L + j] = cands[i0 + r][j].id;
                gsc[r * L + j] = cands[i0 + r][j].score;
            }
        g.ids.upload(gid, s);
        g.scores.upload(gsc, s);
        RefineOut out;
        refine_alloc(g, d, out, s);
        refine_nodes(c, g, false, n_old + i0, n_old + i1, out, s, n_old + i0);
        std::vector<uint32_t> ko(rows * d), kc(rows), ro(rows * L), rcn(rows), oo(rows * L);
        out.kept.download(ko.data(), ko.size(), s);
        out.kept_count.download(kc.data(), rows, s);
        out.keyword.download(ro.data(), ro.size(), s);
        out.kw_count.download(rcn.data(), rows, s);
        out.ordered.download(oo.data(), oo.size(), s);
        FGB_CUDA(cudaStreamSynchronize(s));
        for (uint64_t r = 0; r < rows; ++r) {
            kept[i0 + r].assign(ko.begin() + r * d, ko.begin() + r * d + kc[r]);
            recycled[i0 + r].assign(ro.begin() + r * L, ro.begin() + r * L + rcn[r]);
            ordered[i0 + r].assign(oo.begin() + r * L, oo.begin() + r * L + L);
        }
        i0 = i1;
    }

    mark("refinery");
    // ---- reverse half among the batch, new semantic / keyword lists (update.cpp:127-165)
    const uint32_t half = d / 2;
    std::vector<std::vector<std::pair<uint32_t, uint32_t>>> keepers(batch);  // (pos, keeper)
    for (uint64_t w = 0; w < batch; ++w)
        for (size_t q = 0; q < kept[w].size(); ++q)
            if (kept[w][q] >= n_old)
                keepers[kept[w][q] - n_old].emplace_back(static_cast<uint32_t>(q), static_cast<uint32_t>(n_old + w));
    const uint64_t n = n_old + batch;
    ix.semantic_h.resize(n * d);
    std::vector<std::vector<uint32_t>> new_kw(batch);
    std::vector<uint8_t> short_list(batch, 0);
    parallel_rows(batch, [&](uint64_t i) {  // (rows independent: node i writes only its own lists)
        std::vector<uint32_t> list;
        list.reserve(d);
        auto has = [&](uint32_t id) { return std::find(list.begin(), list.end(), id) != list.end(); };
        const size_t forward = std::min<size_t>(half, kept[i].size());
        for (size_t q = 0; q < forward; ++q) list.push_back(kept[i][q]);
        std::sort(keepers[i].begin(), keepers[i].end());
        for (const auto& [pos, w] : keepers[i]) {
            if (list.size() >= forward + half) break;
            if (!has(w)) list.push_back(w);
        }
        for (size_t q = forward; q < kept[i].size() && list.size() < d; ++q)
            if (!has(kept[i][q])) list.push_back(kept[i][q]);
        for (uint32_t id : ordered[i]) {
            if (list.size() >= d) break;
            if (!has(id)) list.push_back(id);
        }
        if (list.size() != d) {
            short_list[i] = 1;
            return;
        }
        std::copy(list.begin(), list.end(), ix.semantic_h.begin() + (n_old + i) * d);
        for (uint32_t id : recycled[i])
            if (!has(id)) new_kw[i].push_back(id);
    });
    for (uint8_t sh : short_list)
        if (sh) throw Error("invariant-violation", "insert produced a short semantic list");

    mark("new lists");
    // ---- existing nodes: weakest reverse slot replacement (update.cpp:167-193),
    // in the reference's order over exact pair scores computed on the GPU
    // pair list: per touched w its (d - half) reverse-slot pairs once, then one
    // (w, u) pair per kept edge; indices into `ps` replace hash lookups
    std::vector<uint32_t> pa, pb;
    std::vector<uint64_t> slot_base(n_old, ~0ull);
    std::vector<std::vector<uint64_t>> edge_pair(batch);
    for (uint64_t i = 0; i < batch; ++i) {
        edge_pair[i].assign(kept[i].size(), ~0ull);
        for (size_t q = 0; q < kept[i].size(); ++q) {
            const uint32_t w = kept[i][q];
            if (w >= n_old) continue;
            if (slot_base[w] == ~0ull) {
                slot_base[w] = pa.size();
                for (uint32_t sl = half; sl < d; ++sl) {
                    pa.push_back(w);
                    pb.push_back(ix.semantic_h[static_cast<uint64_t>(w) * d + sl]);
                }
            }
            edge_pair[i][q] = pa.size();
            pa.push_back(w);
            pb.push_back(static_cast<uint32_t>(n_old + i));
        }
    }
    std::vector<double> ps(pa.size());
    if (!pa.empty() &&
        fg_pair_scores(&c, pa.data(), pb.data(), pa.size(), ps.data()) != FG_OK)
        throw Error(fg_last_error_code(), fg_last_error_message());
    // current score of each reverse slot of w (slot_base[w] + sl - half),
    // updated in place as slots are replaced (update.cpp:167-193).  An edge
    // (u -> w) reads and writes only w's list and slot scores, so the edges
    // are grouped by w — each group keeping the reference's (u, q) order —
    // and the groups run on host threads.
    std::vector<uint32_t> touched;  // existing nodes with kept edges, first-touch order
    std::vector<uint32_t> gcount;
    std::vector<uint32_t> gidx(n_old, ~0u);
    for (uint64_t i = 0; i < batch; ++i)
        for (uint32_t w : kept[i])
            if (w < n_old) {
                if (gidx[w] == ~0u) {
                    gidx[w] = static_cast<uint32_t>(touched.size());
                    touched.push_back(w);
                    gcount.push_back(0);
                }
                ++gcount[gidx[w]];
            }
    std::vector<uint64_t> gstart(touched.size() + 1, 0);
    for (size_t g = 0; g < touched.size(); ++g) gstart[g + 1] = gstart[g] + gcount[g];
    std::vector<std::pair<uint32_t, uint32_t>> gedge(gstart.back());  // (i, q) per group, in order
    for (uint64_t i = 0; i < batch; ++i)
        for (size_t q = 0; q < kept[i].size(); ++q) {
            const uint32_t w = kept[i][q];
            if (w < n_old) gedge[gstart[gidx[w]]++] = {static_cast<uint32_t>(i), static_cast<uint32_t>(q)};
        }
    for (size_t g = touched.size(); g > 0; --g) gstart[g] = gstart[g - 1];  // (restore the starts)
    gstart[0] = 0;
    parallel_rows(touched.size(), [&](uint64_t g) {
        const uint32_t w = touched[g];
        uint32_t* sem = ix.semantic_h.data() + static_cast<uint64_t>(w) * d;
        double* sc = ps.data() + slot_base[w];
        for (uint64_t e = gstart[g]; e < gstart[g + 1]; ++e) {
            const auto [i, q] = gedge[e];
            const uint32_t u = static_cast<uint32_t>(n_old + i);
            if (std::find(sem, sem + d, u) != sem + d) continue;
            const size_t weakest = static_cast<size_t>(std::min_element(sc, sc + (d - half)) - sc);
            const double incoming = ps[edge_pair[i][q]];
            if (incoming > sc[weakest]) {
                sem[half + weakest] = u;
                sc[weakest] = incoming;
            }
        }
    });

    mark("reverse slots");
    // ---- keyword and logical edges, entity map, norm order; device refresh
    HostList kw;
    kw.ptr.assign(1, 0);
    for (uint64_t u = 0; u < n_old; ++u) {
        kw.idx.insert(kw.idx.end(), ix.keyword_h.begin(u), ix.keyword_h.end(u));
        kw.ptr.push_back(kw.idx.size());
    }
    for (uint64_t i = 0; i < batch; ++i) {
        kw.idx.insert(kw.idx.end(), new_kw[i].begin(), new_kw[i].end());
        kw.ptr.push_back(kw.idx.size());
    }
    ix.keyword_h = std::move(kw);
    std::vector<uint32_t> ks, kr, kt;
    for (size_t t = 0; t + 2 < ix.triplets.size(); t += 3) {
        ks.push_back(ix.triplets[t]);
        kr.push_back(ix.triplets[t + 1]);
        kt.push_back(ix.triplets[t + 2]);
    }
    const fg_kg_view kgv{ks.size(), ks.data(), kr.data(), kt.data()};
    ix.entity_map.clear();  // build_entity_map order == appending the new nodes
    for (uint64_t u = 0; u < n; ++u)
        for (const uint32_t* e = c.entities.begin(u); e != c.entities.end(u); ++e)
            ix.entity_map[*e].push_back(static_cast<uint32_t>(u));
    {
        const HostKg hk = make_kg(&kgv);
        for (uint64_t i = 0; i < batch; ++i) {
            std::vector<uint32_t> e;
            logical_for(c, static_cast<uint32_t>(n_old + i), hk, ix.entity_map, ix.logical_cap, e);
            ix.lg_h.insert(ix.lg_h.end(), e.begin(), e.end());
            ix.lg_ptr_h.push_back(ix.lg_ptr_h.back() + e.size() / 4);
        }
    }
    mark("keyword/logical/entity map");
    ix.semantic.upload(ix.semantic_h, s);
    ix.norm_order_h.clear();  // rebuild_norm_order (index.cpp:12-23)
    index_finish(ix, &kgv);
    mark("upload + index_finish");
}

}  // namespace
}  // namespace fgb

using namespace fgb;

extern "C" {

int fg_index_insert(fg_index* ix, const fg_corpus_view* docs, const fg_insert_params* params) {
    return guarded([&] {
        if (!ix || !docs) throw Error("invalid-argument", "null pointer");
        FGB_CUDA(cudaSetDevice(ix->corpus->device));
        const fg_insert_params p = params ? *params : fg_insert_params{0, 10, 1};
        insert_batch_device(*ix, *docs, p);
    });
}


int fg_index_build_stats(const fg_index* ix, uint64_t* stats4) {
    return guarded([&] {
        if (!ix || !stats4) throw Error("invalid-argument", "null pointer");
        for (int i = 0; i < 4; ++i) stats4[i] = ix->knn_stats[i];
    });
}

int fg_index_build_stats_ex(const fg_index* ix, uint64_t* stats, uint32_t count) {
    return guarded([&] {
        if (!ix || !stats) throw Error("invalid-argument", "null pointer");
        for (uint32_t i = 0; i < count && i < 6; ++i) stats[i] = ix->knn_stats[i];
        for (uint32_t i = 6; i < count; ++i) stats[i] = 0;
    });
}

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
        HostTimer ht("index_build");
        KnnStats ks;
        knn_build_device(*c, p->knn_k, p->knn_iterations, 0.01, p->seed, g, s, &ks);
        ix->knn_stats[0] = ks.passes;
        ix->knn_stats[1] = ks.candidates;
        ix->knn_stats[2] = ks.dense_rows;
        ix->knn_stats[3] = static_cast<uint64_t>(ks.pass_seconds * 1e6);
        ix->knn_stats[4] = ks.sketched;
        ix->knn_stats[5] = ks.sketch_rejected;
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
        ht.mark("refine");

        index_finish(*ix, kg);
        ht.mark("finish");
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
        // the corpus may already be gone (garbage-collected first): use the
        // index's own device record only
        cudaSetDevice(ix->device);
        if (ix->ev0) cudaEventDestroy(ix->ev0);
        if (ix->ev1) cudaEventDestroy(ix->ev1);
        delete ix;
    }
    return FG_OK;
}

}  // extern "C"
