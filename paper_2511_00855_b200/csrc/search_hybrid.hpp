// search_hybrid.hpp — launcher of the certified-approximate beam search for
// batches with entity context and/or required keywords (search.cpp:141-280).
#pragma once

#include "search_plain.hpp"

namespace fgb {

struct HybridLaunch {
    PlainLaunch p;                 // corpus, graph, queries, pools, results (as the plain kernel)
    // entity seeds (select_entry_points, search.cpp:67-98): node-deduped, smallest entity
    const uint64_t* seed_ptr;
    const uint32_t* seed_node;
    const uint32_t* seed_ent;
    const double* rewards;         // per entity query: w_k / hop for hop = 1..rstride (host-divided)
    uint32_t rstride;
    // index edges beyond the semantic lists
    const uint64_t* kw_ptr;        // keyword edges (index.hpp:33-52)
    const uint32_t* kw_idx;
    const uint64_t* lg_ptr;        // logical edges: uint4 (source, relation, target, via)
    const uint4* lg;
    const uint64_t* kg_ptr;        // entity -> sorted related entities
    const uint32_t* kg_nbr;
    uint32_t kg_rows;
    int conjunctive;               // SearchOptions::conjunctive_filter
    uint32_t reqcap;               // max required keywords per query
    uint32_t lccap;                // max logical edges of one node
    uint32_t seencap;              // per-expansion dedupe hash (power of two >= 2 x list length)
    // per query-warp scratch in HBM
    uint32_t* expbits;             // expanded flags (entity-context batches)
    uint32_t* twinbits;            // in-twin-pool flags (keyword batches)
    uint32_t* twin_node;           // twin pool, twcap per warp
    double* twin_d;
    uint32_t twcap;
    uint4* ctx;                    // entity context: (node, entity, hop, has), ctxcap per warp
    uint32_t ctxcap;
    const uint32_t* qlist;         // optional subset of query ids (overflow re-runs)
    uint32_t qlist_n;
    unsigned long long* timing;    // optional phase cycles (FGB_SEARCH_TIMING=1), kHyb* slots
    uint32_t variant;              // kHybBoth / kHybCtx / kHybReq: the instantiation to run
};

// Kernel instantiations by the batch's features: entity context only,
// required keywords only, or both (also forced plain batches).
enum : uint32_t { kHybBoth = 0, kHybCtx = 1, kHybReq = 2 };

enum : int {
    kHybSelect = 0, kHybList, kHybVisit, kHybSparse, kHybDense, kHybCand, kHybTopk, kHybFinal,
    kHybPhases, kHybBatches = kHybPhases, kHybExpanded, kHybQueries, kHybCount
};

enum : uint32_t { HERR_TWIN = 1, HERR_CTX = 2, HERR_CUCKOO = 4 };

// Per-warp shared memory of the hybrid kernel; 0 when the batch does not fit.
size_t hybrid_warp_smem(const HybridLaunch& a);
uint64_t hybrid_slots(const HybridLaunch& a, uint64_t nq, int device);
void launch_search_hybrid(const HybridLaunch& a, uint64_t blocks, cudaStream_t s);

}  // namespace fgb
