// knn.cuh — device-resident NN-Descent state shared by knn.cu / index.
#pragma once

#include "fg_cuda.hpp"

namespace fgb {

// KnnGraph on the device: row u = k entries sorted by (score desc, id asc).
struct DevKnn {
    uint64_t n = 0;
    uint32_t k = 0;
    DevBuf<uint32_t> ids;
    DevBuf<double> scores;
    DevBuf<uint8_t> fresh;
    void alloc(uint64_t n_, uint32_t k_) {
        n = n_;
        k = k_;
        ids.alloc(n * k);
        scores.alloc(n * k);
        fresh.alloc(n * k);
    }
};

// Reverse lists of a snapshot (knn_graph.cpp:78-89).
struct ReverseLists {
    DevBuf<uint32_t> ids;    // n x k
    DevBuf<uint32_t> cnt;    // n
    DevBuf<uint8_t> fresh;   // n x k
    // sort workspace, grow-only: a ReverseLists kept across passes allocates
    // nothing after the first (each pass otherwise mapped and freed ~2 GB at 1M)
    DevBuf<uint64_t> keys_a, keys_b;
    DevBuf<uint32_t> vals_a, vals_b, tkeys_a, tkeys_b, tcnt, tstart;
    DevBuf<unsigned char> temp;
    // node visiting order of the pass kernel (graph locality, set after
    // pass 1 by knn_build_device; empty: identity)
    DevBuf<uint32_t> order;
    // pass statistics (knn_build_device with a KnnStats): candidate / dense
    // row counters, device time of the pass kernels
    DevBuf<unsigned long long> counts;
    // sparse sketches (512 B per document) and their scale for the pass
    // kernel's sketch screening (knn_sketch_prepare; empty: off)
    DevBuf<uint4> sketch;
    DevBuf<unsigned int> sk_gmax;
    uint32_t sk_paths = 0;
    bool sk_on = false;  // screening enabled for the next passes
    // pass flags (overflow, failed cuckoo tables) and the replaced count
    // before a pass (its re-run restores it)
    mutable DevBuf<unsigned int> flags;
    mutable DevBuf<unsigned long long> changed0;
    double pass_ms = 0.0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    ReverseLists() = default;
    ReverseLists(const ReverseLists&) = delete;
    ReverseLists& operator=(const ReverseLists&) = delete;
    ~ReverseLists() {
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
    }
};

// NN-Descent totals over a build: passes, candidates scored (sum over passes
// and nodes of S_u, the fresh new two-hop candidates), dense rows read after
// screening, device seconds of the pass kernels.
struct KnnStats {
    uint64_t passes = 0, candidates = 0, dense_rows = 0;
    uint64_t sketched = 0, sketch_rejected = 0;  // candidates bounded by sketches / rejected by them
    double pass_seconds = 0.0;
};

// init_random_graph (knn_graph.cpp:52-73) into g (allocated n x k).
void knn_init_device(const fg_corpus& c, uint32_t k, uint64_t seed, DevKnn& g, cudaStream_t s);
void knn_reverse_lists(const DevKnn& g, ReverseLists& R, cudaStream_t s);
// Sketch screening policy (FGB_KNN_SKETCH: 0 off, 1 = a build's first pass
// (default), 2 = every pass incl. single fg_knn_iterate calls) and the
// sketches themselves (built into R).
int knn_sketch_policy();
uint32_t knn_sketch_passes();  // passes screened under policy 1 (1)
void knn_sketch_prepare(const fg_corpus& c, ReverseLists& R, cudaStream_t s);
// Stops the screening for the next passes; the sketches stay allocated until R
// dies (a device free synchronises the whole device, which would stall the
// insert path's concurrent search behind this pass).
void knn_sketch_disable(ReverseLists& R);
// The two-hop join for nodes [lo, hi) of g into the same rows of next.
void knn_pass_range(const fg_corpus& c, const DevKnn& g, const ReverseLists& R, uint64_t lo, uint64_t hi,
                    DevKnn& next, unsigned long long* d_changed, cudaStream_t s);
// nn_descent_iterate (knn_graph.cpp:75-148), in place; returns #replaced.
uint64_t knn_iterate_device(const fg_corpus& c, DevKnn& g, cudaStream_t s);
// Same, reusing R / next / changed across passes (knn_build_device).
uint64_t knn_iterate_device(const fg_corpus& c, DevKnn& g, cudaStream_t s, ReverseLists& R, DevKnn& next,
                            DevBuf<unsigned long long>& changed);
// build_knn_graph (knn_graph.cpp:150-166); returns the number of passes run.
uint32_t knn_build_device(const fg_corpus& c, uint32_t k_req, uint32_t max_iterations,
                          double convergence, uint64_t seed, DevKnn& g, cudaStream_t s, KnnStats* stats = nullptr);

struct RefineOut {
    uint32_t degree = 0, k = 0;
    DevBuf<uint32_t> semantic;   // n x degree
    DevBuf<uint32_t> keyword;    // n x k (recycled, reach order)
    DevBuf<uint32_t> kw_count;   // n
    DevBuf<uint32_t> ordered;    // n x k ranked candidate ids
    DevBuf<double> ordered_sc;   // n x k
    DevBuf<uint32_t> detours;    // n x k
    DevBuf<uint32_t> kept;       // n x degree
    DevBuf<uint32_t> kept_count; // n
};

// refine_graph (refine.cpp:167-217).
void refine_device(const fg_corpus& c, const DevKnn& g, uint32_t degree, bool per_neighbour,
                   RefineOut& out, cudaStream_t s);
// Its two halves: the per-node refinery (ranked candidates, detours, IP prune +
// keyword recycling) for nodes [lo, hi) — `out` allocated for all n — and
// merge_reverse_edges + keyword disjointness over every node (needs all kept lists).
void refine_alloc(const DevKnn& g, uint32_t degree, RefineOut& out, cudaStream_t s);
void refine_nodes(const fg_corpus& c, const DevKnn& g, bool per_neighbour, uint64_t lo, uint64_t hi,
                  RefineOut& out, cudaStream_t s, uint64_t row0 = 0);
void refine_merge(uint64_t n, RefineOut& out, cudaStream_t s);

}  // namespace fgb
