// build_shard.cu — build_hybrid_index (index.cpp:25-71) sharded by vertex
// range over G ranks (one GPU each), SURVEY §8(e).
//
// Rank r owns nodes [r*cn, min(n, (r+1)*cn)), cn = ceil(n / G).  The corpus
// is replicated.  Per NN-Descent pass every rank derives the reverse lists
// from the full snapshot (identical everywhere), runs the two-hop join for
// its own range into the next buffer, then one all-gather of the new
// {ids, scores, fresh} rows over NVLink (NCCL, in place) plus an all-reduce of
// the replaced count makes every rank's next snapshot complete.  The pass is
// double-buffered in the reference (knn_graph.cpp:91,141-144), so the result
// is identical for any G.  The refinery runs per node on its range, one
// all-gather of the ranked candidates / kept / recycled lists, and
// merge_reverse_edges + keyword disjointness run replicated over all nodes.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2" — inside a PyTorch
// process this resolves to the NCCL torch already loaded), so the library has
// no hard NCCL dependency.  `sim_ranks` > 1 without a communicator runs every
// rank's range computation in this one process (no collective needed: all
// ranks write their slice of the same buffers) — the partition logic then
// runs and is parity-tested on a single GPU.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <vector>

#include "fg_cuda.hpp"
#include "index.hpp"
#include "knn.cuh"

namespace fgb {
namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            a.h = dlopen(name, RTLD_NOW | RTLD_LOCAL);  // (GLOBAL would shadow the NCCL torch loads later)
            if (a.h) break;
        }
        if (!a.h) return a;
        a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(a.h, "ncclGetUniqueId"));
        a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(a.h, "ncclCommInitRank"));
        a.allGather = reinterpret_cast<decltype(a.allGather)>(dlsym(a.h, "ncclAllGather"));
        a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(a.h, "ncclAllReduce"));
        a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(a.h, "ncclCommDestroy"));
        a.errorString = reinterpret_cast<decltype(a.errorString)>(dlsym(a.h, "ncclGetErrorString"));
        return a;
    }();
    if (!api.h || !api.allGather || !api.commInitRank)
        throw Error("nccl-unavailable", "libnccl.so.2 could not be loaded for the sharded build");
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error("nccl-error", std::string(what) + ": " + (nccl().errorString ? nccl().errorString(r) : "?"));
}

using Clock = std::chrono::steady_clock;
double secs(Clock::time_point a) { return std::chrono::duration<double>(Clock::now() - a).count(); }

}  // namespace
}  // namespace fgb

struct fg_comm {
    int rank = 0, size = 1, device = 0;
    ncclComm_t comm = nullptr;
    // host transport (fg_comm_init_host): collectives through callbacks
    fg_host_all_gather_fn host_gather = nullptr;
    fg_host_sum_u64_fn host_sum = nullptr;
    void* host_ctx = nullptr;
};

namespace fgb {
namespace {

// The collective side of the sharded build: all-gather of equal per-rank
// slices (in place) and an all-reduce of the replaced count.  `comm` null:
// single-process simulation (every slice is already written locally).
struct Shards {
    fg_comm* comm;
    uint32_t G;
    uint64_t n, cn, n_pad;
    std::vector<int> mine;  // ranks computed by this process
    uint64_t lo(int r) const { return std::min<uint64_t>(n, r * cn); }
    uint64_t hi(int r) const { return std::min<uint64_t>(n, (r + 1) * cn); }

    template <typename T>
    void gather(DevBuf<T>& buf, uint64_t row_elems, cudaStream_t s) const {
        if (!comm || G == 1) return;
        const size_t count = cn * row_elems * sizeof(T);
        unsigned char* base = reinterpret_cast<unsigned char*>(buf.get());
        if (comm->host_gather) {  // device -> host -> callback -> device
            std::vector<unsigned char> mine(count), all(count * G);
            FGB_CUDA(cudaMemcpyAsync(mine.data(), base + comm->rank * count, count, cudaMemcpyDeviceToHost, s));
            FGB_CUDA(cudaStreamSynchronize(s));
            if (comm->host_gather(comm->host_ctx, mine.data(), all.data(), count) != 0)
                throw Error("comm-error", "host all-gather callback failed");
            FGB_CUDA(cudaMemcpyAsync(base, all.data(), all.size(), cudaMemcpyHostToDevice, s));
            FGB_CUDA(cudaStreamSynchronize(s));
            return;
        }
        nccl_check(nccl().allGather(base + comm->rank * count, base, count, ncclUint8, comm->comm, s),
                   "ncclAllGather");
    }
    void sum(DevBuf<unsigned long long>& x, cudaStream_t s) const {
        if (!comm || G == 1) return;
        if (comm->host_sum) {
            uint64_t v = 0;
            FGB_CUDA(cudaMemcpyAsync(&v, x.get(), 8, cudaMemcpyDeviceToHost, s));
            FGB_CUDA(cudaStreamSynchronize(s));
            if (comm->host_sum(comm->host_ctx, &v, 1) != 0) throw Error("comm-error", "host sum callback failed");
            FGB_CUDA(cudaMemcpyAsync(x.get(), &v, 8, cudaMemcpyHostToDevice, s));
            FGB_CUDA(cudaStreamSynchronize(s));
            return;
        }
        nccl_check(nccl().allReduce(x.get(), x.get(), 1, ncclUint64, ncclSum, comm->comm, s), "ncclAllReduce");
    }
};

// Padded DevKnn: n_pad rows allocated (all-gather slices), n logical.
void alloc_padded(DevKnn& g, uint64_t n, uint64_t n_pad, uint32_t k) {
    g.alloc(n_pad, k);
    g.n = n;
}

void build_sharded(fg_index& ix, const fg_build_params& p, const Shards& sh, cudaStream_t s) {
    fg_corpus& c = *ix.corpus;
    const uint64_t n = c.n;
    uint32_t k = p.knn_k;
    if (n >= 2 && k >= n) k = static_cast<uint32_t>(n - 1);  // knn_graph.cpp:153-156

    // ---- NN-Descent (knn_graph.cpp:150-166), vertex-range passes
    auto t0 = Clock::now();
    DevKnn g;
    {
        DevKnn g0;
        knn_init_device(c, k, p.seed, g0, s);  // replicated: n*k seeded picks, scored
        alloc_padded(g, n, sh.n_pad, k);
        FGB_CUDA(cudaMemcpyAsync(g.ids.get(), g0.ids.get(), n * k * 4, cudaMemcpyDeviceToDevice, s));
        FGB_CUDA(cudaMemcpyAsync(g.scores.get(), g0.scores.get(), n * k * 8, cudaMemcpyDeviceToDevice, s));
        FGB_CUDA(cudaMemcpyAsync(g.fresh.get(), g0.fresh.get(), n * k, cudaMemcpyDeviceToDevice, s));
    }
    const double denom = static_cast<double>(n) * k;
    DevBuf<unsigned long long> changed(1);
    ReverseLists R;  // sort workspace and lists reused across passes
    DevKnn next;
    const int sk_policy = knn_sketch_policy();
    if (sk_policy >= 1) knn_sketch_prepare(c, R, s);  // (sketches of the whole replicated corpus)
    for (uint32_t it = 0; it < p.knn_iterations; ++it) {
        if (it == knn_sketch_passes() && sk_policy == 1) knn_sketch_disable(R);
        knn_reverse_lists(g, R, s);
        if (it == 0) alloc_padded(next, n, sh.n_pad, k);
        changed.zero(s);
        for (int r : sh.mine) knn_pass_range(c, g, R, sh.lo(r), sh.hi(r), next, changed.get(), s);
        sh.gather(next.ids, k, s);
        sh.gather(next.scores, k, s);
        sh.gather(next.fresh, k, s);
        sh.sum(changed, s);
        unsigned long long h = 0;
        changed.download(&h, 1, s);
        FGB_CUDA(cudaStreamSynchronize(s));
        std::swap(g.ids, next.ids);  // the old snapshot's buffers serve the next pass
        std::swap(g.scores, next.scores);
        std::swap(g.fresh, next.fresh);
        if (static_cast<double>(h) / denom < 0.01) break;
    }
    ix.build_seconds[0] = secs(t0);

    // ---- refinery: per-node on the range, then the global reverse merge
    t0 = Clock::now();
    RefineOut r;
    {
        DevKnn shape;  // allocation shape only: n_pad rows
        shape.n = sh.n_pad;
        shape.k = k;
        refine_alloc(shape, p.degree, r, s);
    }
    for (int rk : sh.mine) refine_nodes(c, g, p.per_neighbour_keyword_check != 0, sh.lo(rk), sh.hi(rk), r, s);
    sh.gather(r.ordered, k, s);
    sh.gather(r.ordered_sc, k, s);
    sh.gather(r.detours, k, s);
    sh.gather(r.kept, p.degree, s);
    sh.gather(r.kept_count, 1, s);
    sh.gather(r.keyword, k, s);
    sh.gather(r.kw_count, 1, s);
    refine_merge(n, r, s);
    ix.semantic = std::move(r.semantic);
    ix.semantic_h.resize(n * p.degree);
    ix.semantic.download(ix.semantic_h.data(), n * p.degree, s);
    std::vector<uint32_t> kw(n * k), kwc(n);
    r.keyword.download(kw.data(), n * k, s);
    r.kw_count.download(kwc.data(), n, s);
    FGB_CUDA(cudaStreamSynchronize(s));
    ix.keyword_h.ptr.assign(n + 1, 0);
    for (uint64_t u = 0; u < n; ++u) ix.keyword_h.ptr[u + 1] = ix.keyword_h.ptr[u] + kwc[u];
    ix.keyword_h.idx.resize(ix.keyword_h.ptr[n]);
    for (uint64_t u = 0; u < n; ++u)
        std::copy(kw.begin() + u * k, kw.begin() + u * k + kwc[u], ix.keyword_h.idx.begin() + ix.keyword_h.ptr[u]);
    ix.build_seconds[1] = secs(t0);
}

}  // namespace
}  // namespace fgb

using namespace fgb;

extern "C" {

int fg_comm_unique_id(uint8_t* out) {
    return guarded([&] {
        if (!out) throw Error("invalid-argument", "null pointer");
        ncclUniqueId id;
        nccl_check(nccl().getUniqueId(&id), "ncclGetUniqueId");
        static_assert(sizeof(id.internal) == FG_COMM_ID_BYTES, "ncclUniqueId size");
        std::memcpy(out, id.internal, sizeof(id.internal));
    });
}

int fg_comm_init(int nranks, int rank, const uint8_t* id, int device, fg_comm** out) {
    return guarded([&] {
        if (!id || !out) throw Error("invalid-argument", "null pointer");
        if (nranks < 1 || rank < 0 || rank >= nranks) throw Error("invalid-argument", "bad rank / size");
        require_device(device);
        auto c = std::make_unique<fg_comm>();
        c->rank = rank;
        c->size = nranks;
        c->device = device;
        ncclUniqueId uid;
        std::memcpy(uid.internal, id, sizeof(uid.internal));
        nccl_check(nccl().commInitRank(&c->comm, nranks, uid, rank), "ncclCommInitRank");
        *out = c.release();
    });
}

int fg_comm_init_host(int nranks, int rank, int device, fg_host_all_gather_fn all_gather, fg_host_sum_u64_fn sum_u64,
                      void* ctx, fg_comm** out) {
    return guarded([&] {
        if (!all_gather || !sum_u64 || !out) throw Error("invalid-argument", "null pointer");
        if (nranks < 1 || rank < 0 || rank >= nranks) throw Error("invalid-argument", "bad rank / size");
        require_device(device);
        auto c = std::make_unique<fg_comm>();
        c->rank = rank;
        c->size = nranks;
        c->device = device;
        c->host_gather = all_gather;
        c->host_sum = sum_u64;
        c->host_ctx = ctx;
        *out = c.release();
    });
}

int fg_comm_free(fg_comm* comm) {
    if (comm) {
        if (comm->comm && nccl().commDestroy) nccl().commDestroy(comm->comm);
        delete comm;
    }
    return FG_OK;
}

int fg_index_build_sharded(fg_corpus* c, const fg_kg_view* kg, const fg_build_params* p, fg_comm* comm,
                           uint32_t sim_ranks, fg_index** out) {
    return guarded([&] {
        if (!c || !p || !out) throw Error("invalid-argument", "null pointer");
        if (p->degree % 2 != 0)
            throw Error("degree-not-even", "semantic degree must be even, got " + std::to_string(p->degree));
        if (p->knn_k < p->degree) throw Error("invalid-k", "knn_k must be at least the degree");
        if (c->n < static_cast<uint64_t>(p->degree) + 1)
            throw Error("corpus-too-small",
                        "need more than degree=" + std::to_string(p->degree) + " documents");
        if (comm && comm->device != c->device)
            throw Error("invalid-argument", "communicator and corpus live on different devices");
        FGB_CUDA(cudaSetDevice(c->device));
        Shards sh;
        sh.comm = comm;
        sh.G = comm ? static_cast<uint32_t>(comm->size) : std::max(1u, sim_ranks);
        sh.n = c->n;
        sh.cn = (c->n + sh.G - 1) / sh.G;
        sh.n_pad = sh.cn * sh.G;
        if (comm)
            sh.mine = {comm->rank};
        else
            for (uint32_t r = 0; r < sh.G; ++r) sh.mine.push_back(static_cast<int>(r));
        auto ix = std::make_unique<fg_index>();
        ix->corpus = c;
        ix->degree = p->degree;
        ix->knn_k = p->knn_k;
        ix->logical_cap = p->logical_cap;
        ix->default_hops = p->default_entity_hops;
        ix->seed = p->seed;
        const auto t_all = Clock::now();
        build_sharded(*ix, *p, sh, c->stream);
        index_finish(*ix, kg);
        ix->build_seconds[4] = secs(t_all);
        *out = ix.release();
    });
}

}  // extern "C"
