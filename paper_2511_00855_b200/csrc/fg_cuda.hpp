// fg_cuda.hpp — host-side CUDA plumbing: checked calls, owning device
// buffers, the fg_corpus handle, and the device query batch.
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "device_common.cuh"
#include "fg_internal.hpp"

namespace fgb {

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (e == cudaErrorMemoryAllocation)
            throw Error("out-of-memory", std::string(what) + ": " + cudaGetErrorString(e));
        throw Error("cuda-error", std::string(what) + ": " + cudaGetErrorString(e));
    }
}
#define FGB_CUDA(x) ::fgb::cuda_check((x), #x)
#define FGB_LAUNCH(what) ::fgb::cuda_check(cudaGetLastError(), what)

inline void require_device(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        throw Error("no-cuda-device", "no CUDA device is visible (the B200 path has no CPU fallback)");
    }
    if (device < 0 || device >= n)
        throw Error("no-cuda-device", "device " + std::to_string(device) + " out of range");
    FGB_CUDA(cudaSetDevice(device));
}

// Device memory comes from the device's stream-ordered pool (cudaMallocAsync
// on a private stream, release threshold unlimited): freed blocks stay cached,
// so repeated API calls (batch_query, insert_batch, small builds) run without
// driver allocations.  A free first synchronises the device — the same
// guarantee cudaFree gives — so no queued kernel can still use the block when
// the pool hands it out again.  (abi_common.cpp)
void* pool_alloc(size_t bytes, int* device);
void pool_free(void* p, int device) noexcept;

// Owning device allocation.
template <typename T>
class DevBuf {
public:
    DevBuf() = default;
    explicit DevBuf(size_t n) { alloc(n); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_), dev_(o.dev_) {
        o.p_ = nullptr;
        o.n_ = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            dev_ = o.dev_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }

    void alloc(size_t n) {
        release();
        if (n) p_ = static_cast<T*>(pool_alloc(n * sizeof(T), &dev_));
        n_ = n;
    }
    void ensure(size_t n) {
        if (n > n_) alloc(n);
    }
    void release() {
        if (p_) pool_free(p_, dev_);
        p_ = nullptr;
        n_ = 0;
    }
    void upload(const T* src, size_t n, cudaStream_t s = 0) {
        ensure(n);
        if (n) FGB_CUDA(cudaMemcpyAsync(p_, src, n * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void upload(const std::vector<T>& v, cudaStream_t s = 0) { upload(v.data(), v.size(), s); }
    void download(T* dst, size_t n, cudaStream_t s = 0) const {
        if (n) FGB_CUDA(cudaMemcpyAsync(dst, p_, n * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
    void zero(cudaStream_t s = 0) {
        if (n_) FGB_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s));
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
    int dev_ = 0;
};

// Grow-only page-locked host buffer (device->host staging at DMA speed).
template <typename T>
class PinnedBuf {
public:
    PinnedBuf() = default;
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    ~PinnedBuf() {
        if (p_) cudaFreeHost(p_);
    }
    void ensure(size_t n) {
        if (n <= n_) return;
        if (p_) cudaFreeHost(p_);
        p_ = nullptr;
        n_ = 0;
        FGB_CUDA(cudaMallocHost(&p_, n * sizeof(T)));
        n_ = n;
    }
    T* get() const { return p_; }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
};

// Host-side CSR copy of a sorted-id list per row.
struct HostList {
    std::vector<uint64_t> ptr{0};
    std::vector<uint32_t> idx;
    size_t rows() const { return ptr.size() - 1; }
    const uint32_t* begin(size_t r) const { return idx.data() + ptr[r]; }
    const uint32_t* end(size_t r) const { return idx.data() + ptr[r + 1]; }
    size_t len(size_t r) const { return ptr[r + 1] - ptr[r]; }
};

}  // namespace fgb

// The device mirror of a DocumentStore.
struct fg_corpus {
    int device = 0;
    uint64_t n = 0;
    uint32_t dim = 0, dstride = 0;
    uint32_t max_lnnz = 0, max_snnz = 0;
    uint64_t l_nnz_total4 = 0, s_nnz_total4 = 0;  // padded posting counts / 4
    uint32_t l_vocab = 0, s_vocab = 0;             // 1 + the largest term id per path
    uint32_t learned_dim = 0, statistical_dim = 0; // DocumentStore vocabulary bounds (types.hpp:121-122)
    fgb::DevCorpus dc{};
    fgb::DevBuf<float> dense, l_val, s_val;
    fgb::DevBuf<uint64_t> l_off, s_off, kw_ptr, ent_ptr;
    fgb::DevBuf<uint32_t> l_nnz, s_nnz, l_idx, s_idx, kw_idx, ent_idx;
    fgb::DevBuf<double> sqnorm, dnorm;
    fgb::DevBuf<uint4> meta;
    fgb::DevBuf<uint8_t> deleted;
    // host copies used by host-side stages (entity map, logical edges, seeds)
    std::vector<uint64_t> doc_id;
    std::vector<uint8_t> deleted_h;
    fgb::HostList keywords, entities;
    std::vector<double> sqnorm_h;
    double max_sqnorm = 0.0;  // max over docs of the unit-weight self score (error bounds)
    double max_dnorm = 0.0;   // max over docs of the dense-row norm (error bounds)
    cudaStream_t stream = nullptr;
};

namespace fgb {

// A query batch on the device (raw vectors; weights applied in-kernel with
// the reference's fp32 product, corpus.cpp:89,96).
struct DevQueries {
    uint64_t count;
    uint32_t dim;
    const float* dense;     // count * dim
    const float4* weights;  // (dense, learned, statistical, entity)
    const uint64_t* l_ptr;
    const uint32_t* l_idx;
    const float* l_val;
    const uint64_t* s_ptr;
    const uint32_t* s_idx;
    const float* s_val;
    const uint64_t* req_ptr;
    const uint32_t* req_idx;
    const uint32_t* k;
    const uint32_t* beam;
    const uint32_t* hops;
};

// Owning device copy of an fg_query_view (missing CSRs become empty rows).
struct QueryUpload {
    DevBuf<float> dense, l_val, s_val;
    DevBuf<float4> weights;
    DevBuf<uint64_t> l_ptr, s_ptr, req_ptr;
    DevBuf<uint32_t> l_idx, s_idx, req_idx, k, beam, hops;
    uint32_t max_lnnz = 0, max_snnz = 0, max_req = 0, max_k = 0, max_beam = 0;
    uint64_t h2d_bytes = 0;
    DevQueries dq{};

    void upload(const fg_query_view& q, cudaStream_t s);
};

// Per-index search I/O: device copies of a batch, its seeds and results, and
// the pinned staging the results come back through. Grow-only and reused, so a
// steady stream of batch_query calls does no cudaMalloc/cudaFree (each of those
// synchronises the device and contends with driver clients such as nvidia-smi).
struct SearchIo {
    QueryUpload up;
    DevBuf<uint64_t> sptr;
    DevBuf<uint32_t> snode, sent;
    DevBuf<uint8_t> shas, qflags;
    DevBuf<double> rew;  // per entity query: w_k / hop (hybrid kernel)
    DevBuf<uint32_t> r_node, r_count, r_warn, r_err;
    DevBuf<double> r_score;
    DevBuf<unsigned long long> r_exp, r_sc;
    DevBuf<unsigned int> work;
    PinnedBuf<unsigned char> host;
};

// Search scratch of one device, shared by all its indexes: per-warp visited /
// expanded / twin bitsets (all-zero between calls: every kernel clears what
// it set), touched lists, twin pools and entity-context tables, plus the
// batch I/O above.  One batch_query at a time per device holds `mu`; every
// call synchronises its stream before releasing it.
struct SearchWorkspace {
    std::mutex mu;
    SearchIo io;
    DevBuf<uint32_t> bits;
    DevBuf<uint32_t> lists;
    DevBuf<unsigned char> misc;
    DevBuf<unsigned char> gpool;  // cand pools in HBM for very large beams
};

inline uint32_t round4(uint32_t x) { return (x + 3u) & ~3u; }

// Derived device state of an uploaded corpus (norms, gather records, maxima).
void corpus_finalize(fg_corpus& c);
// Appends the rows of `v` (insert_batch); validation is the caller's.
void corpus_append(fg_corpus& c, const fg_corpus_view& v);
// Undo of corpus_append (insert_batch failing after the append).
struct CorpusMark {
    uint64_t n, l4, s4;
};
CorpusMark corpus_mark(const fg_corpus& c);
void corpus_rollback(fg_corpus& c, const CorpusMark& m);
// Zero-copy view of rows [first, first + count) as a corpus of `count` rows.
DevCorpus corpus_rows(const DevCorpus& d, uint64_t first, uint64_t count);

}  // namespace fgb
