// synth.cpp — synthetic corpora straight into CSR, bit-identical to the
// reference generator (synth.cpp:140-222, rng.hpp:17-54) but without its AoS
// DocumentStore and on all host threads.
//
// The reference draws every random number from ONE sequential SplitMix64
// stream, whose state is a counter (state += gamma per draw).  Generation is
// split accordingly:
//   phase 1 (sequential, cheap): walk the stream doc by doc, drawing the
//     entity lists, clusters and sparse supports (whose draw count depends on
//     Zipf rejections), and only *skip* the 2*dim draws of each dense vector
//     and the nnz draws of each sparse value list by advancing the counter;
//   phase 2 (parallel): recompute the skipped dense Gaussians (Box-Muller,
//     the expensive part) and sparse values from their saved counter states.
// A dense Box-Muller draw consumes more than two numbers only if u1 == 0
// (probability 2^-53); phase 2 checks every end state and, should that ever
// happen, the whole corpus is regenerated sequentially.  The float/double
// expression shapes below are the reference's, compiled without FP
// contraction, so the bytes match generate_corpus exactly (checked against
// the reference in tests/test_synth.py).

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "fg_internal.hpp"

struct fg_host_corpus {
    uint32_t dim = 0, ldim = 0, sdim = 0;
    std::vector<float> dense;
    std::vector<uint64_t> lptr, sptr, kptr, eptr, doc_id;
    std::vector<uint32_t> lidx, sidx, kidx, eidx;
    std::vector<float> lval, sval;
    std::vector<uint8_t> deleted;
    std::vector<uint32_t> ts, tr, tt;
    struct Chain {
        uint32_t e[3];
        uint64_t seed_doc, bridge_doc;
        std::vector<uint64_t> answers;
        std::vector<float> dense;
        std::vector<uint32_t> lidx, sidx;
        std::vector<float> lval, sval;
    };
    std::vector<Chain> chains;
};

namespace fgb {
namespace {

// rng.hpp:50-55 (same expression).
double gaussian(SplitMix64& rng) {
    double u1 = uniform01(rng);
    while (u1 <= 0.0) u1 = uniform01(rng);
    const double u2 = uniform01(rng);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586477 * u2);
}

// Zipf CDF over ranks 1..vocab (synth.cpp:13-23) with an exact guide table:
// draw() returns lower_bound(cum, u) like zipf_draw (synth.cpp:25-28).
struct Zipf {
    static constexpr int kBits = 16;
    std::vector<double> cum;
    std::vector<uint32_t> guide;  // guide[b] = lower_bound(cum, b / 2^kBits)

    void init(uint32_t vocab, double exponent) {
        cum.resize(vocab);
        double total = 0.0;
        for (uint32_t r = 0; r < vocab; ++r) {
            total += 1.0 / std::pow(static_cast<double>(r + 1), exponent);
            cum[r] = total;
        }
        for (double& c : cum) c /= total;
        const std::size_t g = std::size_t{1} << kBits;
        guide.resize(g + 1);
        for (std::size_t b = 0; b <= g; ++b) {
            const double x = static_cast<double>(b) / static_cast<double>(g);  // exact
            guide[b] = static_cast<uint32_t>(std::lower_bound(cum.begin(), cum.end(), x) - cum.begin());
        }
    }
    uint32_t draw(double u) const {
        const std::size_t b = static_cast<std::size_t>(u * static_cast<double>(1u << kBits));  // exact
        const auto lo = cum.begin() + guide[b];
        const auto hi = cum.begin() + std::min<std::size_t>(guide[b + 1] + 1, cum.size());
        return static_cast<uint32_t>(std::lower_bound(lo, hi, u) - cum.begin());
    }
};

// One sparse vocabulary (synth.cpp:33-78): global Zipf head + per-cluster
// topic block of width vocab/clusters.
struct SparseModel {
    uint32_t vocab = 0, block = 0, n_blocks = 0;
    Zipf global, blockz;
    std::vector<uint8_t> seen;  // dedupe bitmap (phase 1 is single-threaded)

    void init(uint32_t v, uint32_t clusters, double exponent) {
        vocab = v;
        if (vocab == 0) return;
        block = std::max(1u, vocab / std::max(clusters, 1u));
        n_blocks = std::max(1u, vocab / block);
        global.init(vocab, exponent);
        blockz.init(block, exponent);
        seen.assign(vocab, 0);
    }

    // Support draw of sample(): returns the sorted indices; the nnz value
    // draws that follow are skipped (rng advanced) when skip_values.
    void support(uint32_t cluster, uint32_t nnz, SplitMix64& rng, std::vector<uint32_t>& picked) {
        picked.clear();
        if (vocab == 0 || nnz == 0) return;
        const uint32_t start = (cluster % n_blocks) * block;
        const uint32_t take = std::min(nnz, vocab);
        if (take == vocab) {
            picked.resize(take);
            for (uint32_t i = 0; i < take; ++i) picked[i] = i;
        }
        while (picked.size() < take) {
            const uint32_t idx = uniform01(rng) < 0.6 ? start + blockz.draw(uniform01(rng))
                                                      : global.draw(uniform01(rng));
            if (seen[idx]) continue;
            seen[idx] = 1;
            picked.push_back(idx);
        }
        for (uint32_t i : picked) seen[i] = 0;
        std::sort(picked.begin(), picked.end());
    }
    static float value(SplitMix64& rng) { return static_cast<float>(0.1 + 0.9 * uniform01(rng)); }
};

// synth.cpp:80-87.
void normalize(float* v, uint32_t n) {
    double ss = 0.0;
    for (uint32_t i = 0; i < n; ++i) ss += static_cast<double>(v[i]) * v[i];
    if (ss <= 0.0) return;
    const auto inv = static_cast<float>(1.0 / std::sqrt(ss));
    for (uint32_t i = 0; i < n; ++i) v[i] *= inv;
}

// synth.cpp:91-113.
void sample_dense(const std::vector<float>& centers, uint32_t dim, uint32_t nc, uint32_t cluster,
                  float spread, SplitMix64& rng, float* out) {
    const float* c = centers.data() + static_cast<std::size_t>(cluster % nc) * dim;
    for (uint32_t i = 0; i < dim; ++i) out[i] = c[i] + spread * static_cast<float>(gaussian(rng));
    normalize(out, dim);
}

struct Model {
    fg_synth_params p;
    uint32_t clusters = 1, nc = 1;
    std::vector<float> centers;
    SparseModel learned, stat;

    explicit Model(const fg_synth_params& params) : p(params) {
        clusters = std::max(p.clusters, 1u);
        nc = clusters;  // make_centers sizes max(clusters, 1)
        SplitMix64 crng(mix_seed(p.seed, 0));
        centers.resize(static_cast<std::size_t>(nc) * p.dense_dim);
        for (uint32_t c = 0; c < nc; ++c) {
            float* x = centers.data() + static_cast<std::size_t>(c) * p.dense_dim;
            for (uint32_t i = 0; i < p.dense_dim; ++i) x[i] = static_cast<float>(gaussian(crng));
            normalize(x, p.dense_dim);
        }
        learned.init(p.learned_vocab, p.clusters, p.zipf_exponent);
        stat.init(p.statistical_vocab, p.clusters, p.zipf_exponent);
    }
};

void append_row(std::vector<uint64_t>& ptr, std::vector<uint32_t>& idx, const std::vector<uint32_t>& v) {
    idx.insert(idx.end(), v.begin(), v.end());
    ptr.push_back(idx.size());
}

std::vector<uint32_t> sorted_unique(std::vector<uint32_t> v) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    return v;
}

// Generates the corpus. `parallel` selects the two-phase path; the
// sequential path is the literal walk (used as the fallback).
bool generate(const fg_synth_params& p, unsigned threads, bool parallel, fg_host_corpus& h) {
    Model m(p);
    const uint32_t dim = p.dense_dim;
    SplitMix64 rng(mix_seed(p.seed, 1));
    const uint64_t ndocs_total =
        static_cast<uint64_t>(p.docs) + static_cast<uint64_t>(p.chains) * (2 + p.answers_per_chain);
    h = fg_host_corpus{};
    h.dim = dim;
    h.dense.resize(ndocs_total * dim);
    h.lptr.assign(1, 0);
    h.sptr.assign(1, 0);
    h.kptr.assign(1, 0);
    h.eptr.assign(1, 0);
    h.doc_id.resize(ndocs_total);
    for (uint64_t i = 0; i < ndocs_total; ++i) h.doc_id[i] = i;
    h.deleted.assign(ndocs_total, 0);

    const uint32_t ltake = std::min(p.learned_nnz, p.learned_vocab);
    const uint32_t stake = std::min(p.statistical_nnz, p.statistical_vocab);
    std::vector<uint64_t> dense_state, lval_state, sval_state;  // phase-2 work list
    std::vector<uint32_t> cluster_of;
    if (parallel) {
        dense_state.resize(p.docs);
        lval_state.resize(p.docs);
        sval_state.resize(p.docs);
        cluster_of.resize(p.docs);
    }
    std::vector<uint32_t> sup;
    uint64_t next_id = 0;

    // sample_doc (synth.cpp:151-160) for docs generated in full here.
    // The reference builds each doc as make_document(id, sample_dense(..),
    // learned.sample(..), statistical.sample(..), ..) (synth.cpp:153-158); the
    // three draws are function ARGUMENTS, which GCC evaluates right to left on
    // x86-64, so the stream order is statistical, learned, dense.
    auto full_doc = [&](uint32_t cluster, std::vector<uint32_t> ents) {
        m.stat.support(cluster, p.statistical_nnz, rng, sup);
        append_row(h.sptr, h.sidx, sup);
        for (std::size_t i = 0; i < sup.size(); ++i) h.sval.push_back(SparseModel::value(rng));
        append_row(h.kptr, h.kidx, sup);  // keywords = statistical support (corpus.cpp:116)
        m.learned.support(cluster, p.learned_nnz, rng, sup);
        append_row(h.lptr, h.lidx, sup);
        for (std::size_t i = 0; i < sup.size(); ++i) h.lval.push_back(SparseModel::value(rng));
        float* d = h.dense.data() + next_id * dim;
        sample_dense(m.centers, dim, m.nc, cluster, p.cluster_spread, rng, d);
        append_row(h.eptr, h.eidx, sorted_unique(std::move(ents)));
        return next_id++;
    };

    for (uint32_t i = 0; i < p.docs; ++i) {
        std::vector<uint32_t> ents;
        if (p.entity_vocab > 0 && uniform01(rng) < p.entity_rate) {
            const auto count = 1 + bounded(rng, p.max_entities_per_doc);
            for (uint64_t e = 0; e < count; ++e)
                ents.push_back(static_cast<uint32_t>(bounded(rng, p.entity_vocab)));
        }
        const auto cluster = static_cast<uint32_t>(bounded(rng, m.clusters));
        if (!parallel) {
            full_doc(cluster, std::move(ents));
            continue;
        }
        m.stat.support(cluster, p.statistical_nnz, rng, sup);
        append_row(h.sptr, h.sidx, sup);
        append_row(h.kptr, h.kidx, sup);
        sval_state[i] = rng.state;
        rng.state += SplitMix64::kGamma * sup.size();  // skip the value draws
        m.learned.support(cluster, p.learned_nnz, rng, sup);
        append_row(h.lptr, h.lidx, sup);
        lval_state[i] = rng.state;
        rng.state += SplitMix64::kGamma * sup.size();
        dense_state[i] = rng.state;
        rng.state += SplitMix64::kGamma * (2ull * dim);  // skip the Box-Muller draws
        cluster_of[i] = cluster;
        append_row(h.eptr, h.eidx, sorted_unique(std::move(ents)));
        ++next_id;
    }
    (void)ltake;
    (void)stake;

    std::vector<std::array<uint32_t, 3>> trip;
    if (p.entity_vocab > 1) {
        for (uint32_t t = 0; t < p.kg_triplets; ++t) {
            const auto s = static_cast<uint32_t>(bounded(rng, p.entity_vocab));
            auto o = static_cast<uint32_t>(bounded(rng, p.entity_vocab));
            if (o == s) o = (o + 1) % p.entity_vocab;
            const auto r = static_cast<uint32_t>(bounded(rng, std::max(p.relation_vocab, 1u)));
            trip.push_back({s, r, o});
        }
    }

    // Planted chains (synth.cpp:181-218): fully sequential (small).
    for (uint32_t c = 0; c < p.chains; ++c) {
        fg_host_corpus::Chain ch;
        ch.e[0] = p.entity_vocab + 3 * c;
        ch.e[1] = ch.e[0] + 1;
        ch.e[2] = ch.e[0] + 2;
        trip.push_back({ch.e[0], 0, ch.e[1]});
        trip.push_back({ch.e[1], 0, ch.e[2]});
        const auto qc = static_cast<uint32_t>(bounded(rng, m.clusters));
        ch.dense.resize(dim);
        sample_dense(m.centers, dim, m.nc, qc, p.cluster_spread, rng, ch.dense.data());
        m.learned.support(qc, p.learned_nnz, rng, ch.lidx);
        for (std::size_t i = 0; i < ch.lidx.size(); ++i) ch.lval.push_back(SparseModel::value(rng));
        m.stat.support(qc, p.statistical_nnz, rng, ch.sidx);
        for (std::size_t i = 0; i < ch.sidx.size(); ++i) ch.sval.push_back(SparseModel::value(rng));
        ch.seed_doc = full_doc(static_cast<uint32_t>(bounded(rng, m.clusters)), {ch.e[0]});
        ch.bridge_doc = full_doc(static_cast<uint32_t>(bounded(rng, m.clusters)), {ch.e[1]});
        for (uint32_t a = 0; a < p.answers_per_chain; ++a) {
            float* d = h.dense.data() + next_id * dim;
            for (uint32_t i = 0; i < dim; ++i)
                d[i] = -ch.dense[i] + 0.05f * static_cast<float>(gaussian(rng));
            normalize(d, dim);
            append_row(h.lptr, h.lidx, {});
            append_row(h.sptr, h.sidx, {});
            append_row(h.kptr, h.kidx, {});
            append_row(h.eptr, h.eidx, {ch.e[2]});
            ch.answers.push_back(next_id++);
        }
        h.chains.push_back(std::move(ch));
    }
    // In the parallel walk only the chain docs (appended after the regular
    // docs) have pushed their values so far; park them, size the arrays, and
    // put them back behind the regular docs' slots after phase 2.
    std::vector<float> lval_chain, sval_chain;
    if (parallel) {
        lval_chain.swap(h.lval);
        sval_chain.swap(h.sval);
    }
    h.lval.resize(h.lidx.size());
    h.sval.resize(h.sidx.size());

    if (parallel && p.docs > 0) {
        // Phase 2: dense Box-Muller + sparse values from saved counter states.
        std::atomic<bool> shifted{false};
        std::atomic<uint32_t> cursor{0};
        const unsigned nt = std::max(1u, threads);
        auto work = [&] {
            constexpr uint32_t kChunk = 256;
            for (;;) {
                const uint32_t b = cursor.fetch_add(kChunk);
                if (b >= p.docs) return;
                const uint32_t e = std::min(p.docs, b + kChunk);
                for (uint32_t i = b; i < e; ++i) {
                    SplitMix64 r(dense_state[i]);
                    const uint32_t cluster = cluster_of[i];
                    sample_dense(m.centers, dim, m.nc, cluster, p.cluster_spread, r,
                                 h.dense.data() + static_cast<std::size_t>(i) * dim);
                    if (r.state != dense_state[i] + SplitMix64::kGamma * (2ull * dim)) shifted = true;
                    SplitMix64 lr(lval_state[i]);
                    for (uint64_t j = h.lptr[i]; j < h.lptr[i + 1]; ++j) h.lval[j] = SparseModel::value(lr);
                    SplitMix64 sr(sval_state[i]);
                    for (uint64_t j = h.sptr[i]; j < h.sptr[i + 1]; ++j) h.sval[j] = SparseModel::value(sr);
                }
            }
        };
        std::vector<std::thread> pool;
        for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work);
        work();
        for (auto& t : pool) t.join();
        if (shifted) return false;
    }
    if (parallel) {
        std::copy(lval_chain.begin(), lval_chain.end(), h.lval.begin() + static_cast<std::ptrdiff_t>(h.lptr[p.docs]));
        std::copy(sval_chain.begin(), sval_chain.end(), h.sval.begin() + static_cast<std::ptrdiff_t>(h.sptr[p.docs]));
    }

    // validate_corpus dimension fields (corpus.cpp:64-69) and KnowledgeGraph
    // normalisation (types.cpp:29-45: sort by (s, r, t), unique).
    for (uint64_t i = 0; i < ndocs_total; ++i) {
        if (h.lptr[i + 1] > h.lptr[i]) h.ldim = std::max(h.ldim, h.lidx[h.lptr[i + 1] - 1] + 1);
        if (h.sptr[i + 1] > h.sptr[i]) h.sdim = std::max(h.sdim, h.sidx[h.sptr[i + 1] - 1] + 1);
    }
    std::sort(trip.begin(), trip.end(), [](const auto& a, const auto& b) {
        if (a[0] != b[0]) return a[0] < b[0];
        if (a[1] != b[1]) return a[1] < b[1];
        return a[2] < b[2];
    });
    trip.erase(std::unique(trip.begin(), trip.end()), trip.end());
    for (const auto& t : trip) {
        h.ts.push_back(t[0]);
        h.tr.push_back(t[1]);
        h.tt.push_back(t[2]);
    }
    return true;
}

}  // namespace
}  // namespace fgb

extern "C" {

int fg_synth_generate(const fg_synth_params* p, unsigned threads, fg_host_corpus** out) {
    return fgb::guarded([&] {
        if (!p || !out) throw fgb::Error("invalid-argument", "null pointer");
        if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
        auto h = std::make_unique<fg_host_corpus>();
        if (!fgb::generate(*p, threads, true, *h)) fgb::generate(*p, 1, false, *h);
        if (h->doc_id.empty()) throw fgb::Error("empty-corpus", "corpus holds no documents");
        *out = h.release();
    });
}

int fg_host_corpus_view(const fg_host_corpus* h, fg_corpus_view* v, fg_kg_view* kg,
                        uint64_t* chain_count) {
    return fgb::guarded([&] {
        if (!h) throw fgb::Error("invalid-argument", "null corpus");
        if (v) {
            std::memset(v, 0, sizeof *v);
            v->n = h->doc_id.size();
            v->dense_dim = h->dim;
            v->learned_dim = h->ldim;
            v->statistical_dim = h->sdim;
            v->dense = h->dense.data();
            v->learned = {h->lptr.data(), h->lidx.data(), h->lval.data()};
            v->statistical = {h->sptr.data(), h->sidx.data(), h->sval.data()};
            v->keywords = {h->kptr.data(), h->kidx.data()};
            v->entities = {h->eptr.data(), h->eidx.data()};
            v->doc_id = h->doc_id.data();
            v->deleted = h->deleted.data();
        }
        if (kg) *kg = {h->ts.size(), h->ts.data(), h->tr.data(), h->tt.data()};
        if (chain_count) *chain_count = h->chains.size();
    });
}

int fg_host_corpus_chain(const fg_host_corpus* h, uint64_t c, uint32_t ent[3], uint64_t docs[2],
                         uint64_t* answers, float* dense, uint32_t* lnnz, uint32_t* lidx,
                         float* lval, uint32_t* snnz, uint32_t* sidx, float* sval) {
    return fgb::guarded([&] {
        if (!h || c >= h->chains.size()) throw fgb::Error("unknown-id", "no such chain");
        const auto& ch = h->chains[c];
        std::copy(ch.e, ch.e + 3, ent);
        docs[0] = ch.seed_doc;
        docs[1] = ch.bridge_doc;
        std::copy(ch.answers.begin(), ch.answers.end(), answers);
        std::copy(ch.dense.begin(), ch.dense.end(), dense);
        *lnnz = static_cast<uint32_t>(ch.lidx.size());
        std::copy(ch.lidx.begin(), ch.lidx.end(), lidx);
        std::copy(ch.lval.begin(), ch.lval.end(), lval);
        *snnz = static_cast<uint32_t>(ch.sidx.size());
        std::copy(ch.sidx.begin(), ch.sidx.end(), sidx);
        std::copy(ch.sval.begin(), ch.sval.end(), sval);
    });
}

int fg_host_corpus_free(fg_host_corpus* h) {
    delete h;
    return FG_OK;
}

// random_query_vector + random_simplex_weights (synth.cpp:117-138) per query.
int fg_synth_queries(const fg_synth_params* p, uint64_t stream, uint64_t count, int with_weights,
                     float* dense, uint32_t* lidx, float* lval, uint32_t* sidx, float* sval,
                     fg_weights* weights) {
    return fgb::guarded([&] {
        using namespace fgb;
        Model m(*p);
        SplitMix64 rng(mix_seed(p->seed, stream));
        const uint32_t ln = std::min(p->learned_nnz, p->learned_vocab);
        const uint32_t sn = std::min(p->statistical_nnz, p->statistical_vocab);
        std::vector<uint32_t> sup;
        for (uint64_t i = 0; i < count; ++i) {
            const auto cluster = static_cast<uint32_t>(bounded(rng, m.clusters));
            sample_dense(m.centers, p->dense_dim, m.nc, cluster, p->cluster_spread, rng,
                         dense + i * p->dense_dim);
            m.learned.support(cluster, p->learned_nnz, rng, sup);
            std::copy(sup.begin(), sup.end(), lidx + i * ln);
            for (uint32_t j = 0; j < sup.size(); ++j) lval[i * ln + j] = SparseModel::value(rng);
            m.stat.support(cluster, p->statistical_nnz, rng, sup);
            std::copy(sup.begin(), sup.end(), sidx + i * sn);
            for (uint32_t j = 0; j < sup.size(); ++j) sval[i * sn + j] = SparseModel::value(rng);
            if (with_weights) {
                double parts[3];
                double total = 0.0;
                for (double& x : parts) {
                    x = -std::log(std::max(uniform01(rng), 1e-300));
                    total += x;
                }
                weights[i].dense = static_cast<float>(parts[0] / total);
                weights[i].learned = static_cast<float>(parts[1] / total);
                weights[i].statistical = static_cast<float>(parts[2] / total);
                weights[i].entity = 0.0f;
            }
        }
    });
}

}  // extern "C"
