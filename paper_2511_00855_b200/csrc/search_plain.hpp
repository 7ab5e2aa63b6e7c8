// search_plain.hpp — launcher of the certified-approximate beam search for
// "plain" query batches (no entity context, no required keywords).
#pragma once

#include "fg_cuda.hpp"

namespace fgb {

struct PlainLaunch {
    DevCorpus c;
    const uint32_t* semantic;
    uint32_t degree;
    DevQueries q;
    const uint32_t* norm_order;
    const uint4* edge_meta;     // gather record of semantic[u][j] (n x degree)
    const uint4* norm_meta;     // gather record of norm_order[i]
    uint32_t entry_count;
    const uint8_t* qflags;      // QF_VALID | QF_FALLBACK
    uint32_t vocab[2];          // per sparse path (learned, statistical): bitmap width, 0 = hash
    int mode;                   // lookup mode of the batch's active paths (approx::kMode*)
    uint32_t cap[2];            // per sparse path: hash capacity / staged value slots
    uint32_t beamcap, kcap;     // max beam / k in the batch
    double* gpool_d;            // non-null: the cand pools live in HBM (beamcap per query-warp), not smem
    uint32_t* gpool_n;
    double max_norm;            // >= sqrt(max sqnorm) of the corpus
    double max_dnorm;           // >= max dense-row norm of the corpus
    double eps_coef;            // fp64 error-bound coefficient (see search_plain.cu)
    double eps32_coef;          // fp32 dense-partial error coefficient
    uint32_t* visited;          // per-warp exact bitsets, nwords each
    uint64_t nwords;
    uint32_t* touched;          // per-warp touched lists, tcap each
    uint32_t tcap;
    uint32_t hit_stride;
    uint32_t* r_node;
    double* r_score;
    uint32_t* r_count;
    unsigned long long* r_expanded;
    unsigned long long* r_scored;
    uint32_t* r_warn;
    uint32_t* r_err;
    unsigned int* work;
    unsigned long long* timing;  // optional phase timing (kPlainPh* slots)
    unsigned long long* stats;   // [0] exact resolutions, [1] exact final entries
    int prefetch;
    double eps_scale;           // test hook: inflate the error bound (forces resolutions)
};

enum : int {
    kPlainPhSeeds = 0, kPlainPhSelect, kPlainPhAdj, kPlainPhSparse, kPlainPhDense,
    kPlainPhMerge, kPlainPhFinal, kPlainPhQueries, kPlainPhExpanded, kPlainPhStart, kPlainPhEndMin,
    kPlainPhEndMax, kPlainPhCount
};

// Per-warp shared memory of the plain kernel; 0 when the batch does not fit.
size_t plain_warp_smem(const PlainLaunch& a);
// Grid slots (query-warps) the launcher will use for `nq` queries.
uint64_t plain_slots(const PlainLaunch& a, uint64_t nq, int device);
void launch_search_plain(const PlainLaunch& a, uint64_t nq, int device, cudaStream_t s);

}  // namespace fgb
