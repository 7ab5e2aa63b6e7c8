// index.hpp — the device-resident HybridIndex (index.hpp:33-52 of the reference).
#pragma once

#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "fg_cuda.hpp"

struct fg_index {
    fg_corpus* corpus = nullptr;  // not owned
    int device = 0;               // the corpus's device (freeing must not touch the corpus)
    uint32_t degree = 0, knn_k = 0, logical_cap = 64, default_hops = 2;
    uint64_t seed = 0;

    // device edge tables
    fgb::DevBuf<uint32_t> semantic;  // n x degree
    fgb::DevBuf<uint64_t> kw_ptr;    // keyword edges CSR
    fgb::DevBuf<uint32_t> kw_idx;
    fgb::DevBuf<uint64_t> lg_ptr;    // logical edges CSR, uint4 = (source, relation, target, via)
    fgb::DevBuf<uint4> lg;
    fgb::DevBuf<uint32_t> norm_order;
    // gather records (DevCorpus::meta) of every semantic edge's target and of
    // the nodes in norm order: the plain search reads them coalesced with the
    // adjacency list instead of one dependent scattered load per candidate
    fgb::DevBuf<uint4> edge_meta;   // n x degree
    fgb::DevBuf<uint4> norm_meta;   // n
    fgb::DevBuf<uint64_t> kg_ptr;    // entity -> sorted unique related entities
    fgb::DevBuf<uint32_t> kg_nbr;
    uint32_t kg_rows = 0;

    // host mirrors (export, seeds, logical derivation)
    std::vector<uint32_t> semantic_h;
    fgb::HostList keyword_h;
    std::vector<uint64_t> lg_ptr_h;
    std::vector<uint32_t> lg_h;  // 4 per edge
    std::vector<uint32_t> norm_order_h;
    std::map<uint32_t, std::vector<uint32_t>> entity_map;  // EntityMap (logical.hpp:21)
    std::vector<uint32_t> triplets;  // KnowledgeGraph::triplets(): (s, r, t) sorted, unique
    uint32_t max_kw_edges = 0, max_logical_group = 0;
    double build_seconds[5] = {0, 0, 0, 0, 0};
    // passes, candidates scored, dense rows, pass-kernel microseconds,
    // candidates bounded by sparse sketches, candidates the sketches rejected
    uint64_t knn_stats[6] = {0, 0, 0, 0, 0, 0};

    // search scratch + batch buffers: shared by every index on the device
    // (fgb::search_workspace), grown on demand, reused across calls
    std::shared_ptr<fgb::SearchWorkspace> ws;
    std::mutex search_mu;
    double last_kernel_ms = 0.0;
    const char* last_kernel = "";
    uint64_t last_launches = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

namespace fgb {
// The device's shared search workspace (created on first use, freed with the
// last index that holds it).  Callers lock ws->mu around its use.
std::shared_ptr<SearchWorkspace> search_workspace(int device);
// Uploads host edge tables into ix (device + host mirrors) and derives the
// KG adjacency; entity map from the corpus.
void index_finish(fg_index& ix, const fg_kg_view* kg);
}  // namespace fgb
