// mirror_check.cpp — checks the drop-in's device-mirror lifetime contract
// (SURVEY §8(b) "Ownership"): a search on a cached mirror returns exactly
// what a fresh upload of the same host struct returns, after mark_delete,
// after insert_batch, and for new indexes built at the same address (the
// loop below destroys and rebuilds an index in one stack slot).  Linked
// like acceptance_b200: the shim in front of the reference objects.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "fusegraph/corpus.hpp"
#include "fusegraph/eval.hpp"
#include "fusegraph/index.hpp"
#include "fusegraph/rng.hpp"
#include "fusegraph/search.hpp"
#include "fusegraph/synth.hpp"
#include "fusegraph/update.hpp"
#include "fusegraph_b200_shim.hpp"

using namespace fusegraph;

namespace {
int failures = 0;

void expect(bool ok, const std::string& what) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++failures;
}

std::vector<SearchResult> run(const HybridIndex& ix, const std::vector<QuerySpec>& qs) {
    return batch_query(ix, qs, 1, SearchOptions{});
}

bool same(const std::vector<SearchResult>& a, const std::vector<SearchResult>& b) {
    if (a.size() != b.size()) return false;
    for (std::size_t i = 0; i < a.size(); ++i) {
        if (a[i].hits.size() != b[i].hits.size() || a[i].expanded != b[i].expanded) return false;
        for (std::size_t j = 0; j < a[i].hits.size(); ++j)
            if (a[i].hits[j].doc_id != b[i].hits[j].doc_id || a[i].hits[j].score != b[i].hits[j].score)
                return false;
    }
    return true;
}

// the cached mirror answers like a fresh upload of the current host struct
bool mirror_is_current(const HybridIndex& ix, const std::vector<QuerySpec>& qs) {
    const auto cached = run(ix, qs);
    b200::invalidate_device_mirrors();
    const auto fresh = run(ix, qs);
    return same(cached, fresh);
}

std::vector<QuerySpec> queries(const SynthParams& sp, uint64_t seed, int count) {
    SplitMix64 rng(seed);
    std::vector<QuerySpec> qs;
    for (int i = 0; i < count; ++i) {
        QuerySpec q;
        q.vector = random_query_vector(sp, rng);
        q.k = 10;
        q.beam_width = 64;
        qs.push_back(q);
    }
    return qs;
}
}  // namespace

int main() {
    BuildParams bp;
    bp.degree = 16;
    bp.knn_k = 32;
    SynthParams sp;
    sp.docs = 1500;
    sp.seed = 71;
    SynthData data = generate_corpus(sp);
    DocumentStore base;
    base.docs.assign(data.store.docs.begin(), data.store.docs.begin() + 1300);
    std::vector<DocumentRecord> extra(data.store.docs.begin() + 1300, data.store.docs.end());
    validate_corpus(base);
    const auto qs = queries(sp, 7100, 40);

    HybridIndex ix = build_hybrid_index(std::move(base), {}, bp);
    expect(mirror_is_current(ix, qs), "search after build reuses the build's device index");

    // mark_delete: flags pushed to the mirror in place
    const auto before = run(ix, qs);
    std::vector<uint64_t> del;
    for (int i = 0; i < 10; ++i) del.push_back(before[i].hits[0].doc_id);
    mark_delete(ix, del);
    const auto after = run(ix, qs);
    bool gone = true;
    for (const auto& r : after)
        for (const auto& h : r.hits)
            for (uint64_t d : del) gone &= h.doc_id != d;
    expect(gone, "mark_delete: deleted docs never returned");
    expect(mirror_is_current(ix, qs), "mark_delete: mirror equals a fresh upload");

    // insert_batch: device index appended and linked in place
    insert_batch(ix, extra);
    expect(ix.size() == 1500 && ix.semantic.size() == 1500 && ix.norm_order.size() == 1500,
           "insert_batch: host struct extended");
    expect(mirror_is_current(ix, qs), "insert_batch: mirror equals a fresh upload");

    // indexes destroyed and rebuilt in the same stack slot
    for (int round = 0; round < 3; ++round) {
        SynthParams sp2 = sp;
        sp2.seed = 100 + round;
        sp2.docs = 1200;
        SynthData d2 = generate_corpus(sp2);
        const auto q2 = queries(sp2, 7200 + round, 20);
        HybridIndex slot = build_hybrid_index(std::move(d2.store), {}, bp);
        const auto r1 = run(slot, q2);
        b200::invalidate_device_mirrors();
        expect(same(r1, run(slot, q2)), "rebuilt index in a reused slot, round " + std::to_string(round));
    }
    std::printf("%d failure(s)\n", failures);
    return failures ? 1 : 0;
}
