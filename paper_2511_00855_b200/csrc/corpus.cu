// corpus.cu — the device DocumentStore, squared norms, query staging and the
// K1 entry points (batch_scores, pair scores, build_query_vector).
#include <algorithm>
#include <cmath>
#include <mutex>
#include <thread>

#include "fg_cuda.hpp"
#include "query_stage.cuh"

namespace fgb {
namespace {

// finalize_fused (types.cpp:74-79): dense self-dot, then learned, then
// statistical self sparse dot (every term shared, ascending order).
__global__ void sqnorm_kernel(DevCorpus c, double* out, double* dnorm) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= c.n) return;
    const float* row = c.dense + i * c.dstride;
    double acc = 0.0;
    for (uint32_t j = 0; j < c.dim; ++j) acc = __fma_rn((double)row[j], (double)row[j], acc);
    dnorm[i] = sqrt(acc);
    double l = 0.0;
    for (uint32_t j = 0; j < c.l_nnz[i]; ++j) {
        const double v = c.l_val[c.l_off[i] + j];
        l = __fma_rn(v, v, l);
    }
    acc = __dadd_rn(acc, l);
    double s = 0.0;
    for (uint32_t j = 0; j < c.s_nnz[i]; ++j) {
        const double v = c.s_val[c.s_off[i] + j];
        s = __fma_rn(v, v, s);
    }
    out[i] = __dadd_rn(acc, s);
}

// hybrid_score(doc a, doc b) with both rows in global memory: dense chain +
// merge-join in ascending index order (scoring.cpp:24-42).
__device__ double sparse_merge(const uint32_t* idx, const float* val, uint64_t oa, uint32_t na,
                               uint64_t ob, uint32_t nb) {
    double acc = 0.0;
    uint32_t i = 0, j = 0;
    while (i < na && j < nb) {
        const uint32_t a = idx[oa + i], b = idx[ob + j];
        if (a < b) {
            ++i;
        } else if (b < a) {
            ++j;
        } else {
            acc = __fma_rn((double)val[oa + i], (double)val[ob + j], acc);
            ++i;
            ++j;
        }
    }
    return acc;
}

// Packed per-node gather record (DevCorpus::meta).
__global__ void meta_kernel(DevCorpus c, const double* dnorm, uint4* meta) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= c.n) return;
    meta[i] = make_uint4(static_cast<uint32_t>(c.l_off[i] >> 2), static_cast<uint32_t>(c.s_off[i] >> 2),
                         c.l_nnz[i] | (c.s_nnz[i] << 16), __float_as_uint(__double2float_ru(dnorm[i])));
}

__global__ void pair_kernel(DevCorpus c, const uint32_t* a, const uint32_t* b, uint64_t m,
                            double* out) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= m) return;
    const uint64_t u = a[t], v = b[t];
    const float* ru = c.dense + u * c.dstride;
    const float* rv = c.dense + v * c.dstride;
    double acc = 0.0;
    for (uint32_t j = 0; j < c.dim; ++j) acc = __fma_rn((double)ru[j], (double)rv[j], acc);
    acc = __dadd_rn(acc, sparse_merge(c.l_idx, c.l_val, c.l_off[u], c.l_nnz[u], c.l_off[v], c.l_nnz[v]));
    acc = __dadd_rn(acc, sparse_merge(c.s_idx, c.s_val, c.s_off[u], c.s_nnz[u], c.s_off[v], c.s_nnz[v]));
    out[t] = acc;
}

// batch_scores (scoring.cpp:101-109): every block stages the weighted query
// in shared memory; one thread per id.
__global__ void batch_scores_kernel(DevCorpus c, DevQueries q, uint64_t qi, const uint32_t* ids,
                                    uint64_t m, double* out, uint32_t lcap, uint32_t scap) {
    extern __shared__ __align__(16) unsigned char smem[];
    SmemQuery sq;
    stage_query(q, qi, c.dstride, smem, lcap, scap, threadIdx.x, blockDim.x, sq,
                [] { __syncthreads(); });
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t < m) out[t] = hybrid_score(c, sq, ids[t]);
}

// Runs fn(lo, hi) over [0, n) on up to 32 host threads (contiguous ranges).
template <typename Fn>
void host_parallel(uint64_t n, Fn fn) {
    const uint64_t hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    const uint64_t parts = std::min<uint64_t>(hw, std::max<uint64_t>(1, n / 65536));
    if (parts <= 1) {
        fn(uint64_t(0), n);
        return;
    }
    std::vector<std::thread> th;
    for (uint64_t p = 0; p < parts; ++p) th.emplace_back(fn, n * p / parts, n * (p + 1) / parts);
    for (auto& t : th) t.join();
}

// Double-buffered pinned staging for streaming large host data to the
// device: the host packs chunk i + 1 while the copy engine moves chunk i.
struct PinnedStage {
    static constexpr size_t kBytes = size_t(32) << 20;  // per buffer
    unsigned char* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int cur = 0;
    PinnedStage() {
        for (int i = 0; i < 2; ++i) {
            FGB_CUDA(cudaMallocHost(&buf[i], kBytes));
            FGB_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        }
    }
    ~PinnedStage() {
        for (int i = 0; i < 2; ++i) {
            if (ev[i]) cudaEventSynchronize(ev[i]), cudaEventDestroy(ev[i]);
            if (buf[i]) cudaFreeHost(buf[i]);
        }
    }
    unsigned char* next() {  // a buffer whose previous copy has finished
        cur ^= 1;
        FGB_CUDA(cudaEventSynchronize(ev[cur]));
        return buf[cur];
    }
    void sent(cudaStream_t s) { FGB_CUDA(cudaEventRecord(ev[cur], s)); }
};

// Host -> device copy of a large unpadded host array: its pages are locked
// in place for the copy (DMA at link speed; 3 GB of dense rows in ~0.2 s vs
// ~0.3 s through the pinned stage and 0.3-0.6 s pageable, B200 box).
template <typename T>
void upload_locked(DevBuf<T>& dst, const T* src, size_t n, cudaStream_t s) {
    dst.ensure(n);
    void* p = const_cast<T*>(src);
    const bool pinned = cudaHostRegister(p, n * sizeof(T), cudaHostRegisterDefault) == cudaSuccess;
    if (!pinned) cudaGetLastError();
    FGB_CUDA(cudaMemcpyAsync(dst.get(), src, n * sizeof(T), cudaMemcpyHostToDevice, s));
    FGB_CUDA(cudaStreamSynchronize(s));
    if (pinned) cudaHostUnregister(p);
}

// Dense rows (dim floats each) into the device's dstride-padded layout.
void stream_dense(const float* src, uint64_t n, uint32_t dim, uint32_t dstride, float* dst, PinnedStage& st,
                  cudaStream_t s) {
    const uint64_t rows = std::max<uint64_t>(1, PinnedStage::kBytes / (dstride * 4ull));
    for (uint64_t r0 = 0; r0 < n; r0 += rows) {
        const uint64_t r1 = std::min(n, r0 + rows);
        float* p = reinterpret_cast<float*>(st.next());
        host_parallel(r1 - r0, [&](uint64_t lo, uint64_t hi) {
            if (dim == dstride) {
                std::memcpy(p + lo * dstride, src + (r0 + lo) * dim, (hi - lo) * dim * 4ull);
                return;
            }
            for (uint64_t i = lo; i < hi; ++i) {
                std::memcpy(p + i * dstride, src + (r0 + i) * dim, dim * 4ull);
                std::memset(p + i * dstride + dim, 0, (dstride - dim) * 4ull);
            }
        });
        FGB_CUDA(cudaMemcpyAsync(dst + r0 * dstride, p, (r1 - r0) * dstride * 4ull, cudaMemcpyHostToDevice, s));
        st.sent(s);
    }
}

// One sparse path packed straight into pinned chunks and streamed into the
// padded device layout (rows padded to 4 entries with (kPad, 0), validated
// strictly ascending — the first offending row is reported).  Returns the
// padded entry count; *vocab = 1 + the largest term id.
uint64_t stream_sparse(const fg_sparse_view& sv, uint64_t n, std::vector<uint64_t>& off, std::vector<uint32_t>& nnz,
                       uint32_t& max_nnz, uint32_t& vocab, DevBuf<uint32_t>& didx, DevBuf<float>& dval,
                       PinnedStage& st, cudaStream_t s, const char* path) {
    off.resize(n);
    nnz.resize(n);
    uint64_t total = 0;
    max_nnz = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t len = sv.ptr ? sv.ptr[i + 1] - sv.ptr[i] : 0;
        if (len > 0xFFFFFFFFull) throw Error("invalid-argument", "sparse row too long");
        off[i] = total;
        nnz[i] = static_cast<uint32_t>(len);
        max_nnz = std::max<uint32_t>(max_nnz, nnz[i]);
        total += round4(nnz[i]);
    }
    vocab = 0;
    const uint64_t cap = PinnedStage::kBytes / 8;  // entries per chunk (idx half, val half)
    if (round4(max_nnz) > cap) throw Error("invalid-argument", "sparse row too long");
    didx.ensure(std::max<uint64_t>(total, 4));
    dval.ensure(std::max<uint64_t>(total, 4));
    if (total == 0) {
        const uint32_t pi[4] = {kPad, kPad, kPad, kPad};
        const float pv[4] = {0.f, 0.f, 0.f, 0.f};
        didx.upload(pi, 4, s);
        dval.upload(pv, 4, s);
        FGB_CUDA(cudaStreamSynchronize(s));
        return 0;
    }
    std::mutex mu;
    for (uint64_t r0 = 0; r0 < n;) {
        uint64_t r1 = r0;
        while (r1 < n && off[r1] + round4(nnz[r1]) - off[r0] <= cap) ++r1;
        const uint64_t base = off[r0], cnt = (r1 < n ? off[r1] : total) - base;
        unsigned char* p = st.next();
        uint32_t* pi = reinterpret_cast<uint32_t*>(p);
        float* pv = reinterpret_cast<float*>(p + cap * 4);
        uint64_t bad = n;
        host_parallel(r1 - r0, [&](uint64_t lo, uint64_t hi) {
            uint32_t v_max = 0;
            uint64_t my_bad = n;
            for (uint64_t i = r0 + lo; i < r0 + hi; ++i) {
                const uint64_t b = sv.ptr[i], o = off[i] - base;
                const uint32_t m = nnz[i];
                for (uint32_t j = 0; j < m; ++j) {
                    const uint32_t x = sv.idx[b + j];
                    if (j > 0 && x <= sv.idx[b + j - 1] && my_bad == n) my_bad = i;
                    pi[o + j] = x;
                    pv[o + j] = sv.val[b + j];
                    v_max = std::max(v_max, x + 1);
                }
                for (uint32_t j = m; j < round4(m); ++j) {
                    pi[o + j] = kPad;
                    pv[o + j] = 0.0f;
                }
            }
            std::lock_guard<std::mutex> lock(mu);
            vocab = std::max(vocab, v_max);
            bad = std::min(bad, my_bad);
        });
        if (bad < n)
            throw Error("unsorted-sparse", "doc " + std::to_string(bad) + ": " + path +
                                               " indices must be strictly ascending");
        FGB_CUDA(cudaMemcpyAsync(didx.get() + base, pi, cnt * 4, cudaMemcpyHostToDevice, s));
        FGB_CUDA(cudaMemcpyAsync(dval.get() + base, pv, cnt * 4, cudaMemcpyHostToDevice, s));
        st.sent(s);
        r0 = r1;
    }
    return total;
}

// Padded device layout of one sparse path (rows padded to 4 entries with
// (kPad, 0)); rows are validated strictly ascending, the first offending row
// is reported.  *vocab = 1 + the largest term id (0 when empty).
void build_sparse(const fg_sparse_view& sv, uint64_t n, std::vector<uint64_t>& off,
                  std::vector<uint32_t>& nnz, std::vector<uint32_t>& idx, std::vector<float>& val,
                  uint32_t& max_nnz, const char* path, uint32_t* vocab = nullptr) {
    off.resize(n);
    nnz.resize(n);
    uint64_t total = 0;
    max_nnz = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t len = sv.ptr ? sv.ptr[i + 1] - sv.ptr[i] : 0;
        if (len > 0xFFFFFFFFull) throw Error("invalid-argument", "sparse row too long");
        off[i] = total;
        nnz[i] = static_cast<uint32_t>(len);
        max_nnz = std::max<uint32_t>(max_nnz, nnz[i]);
        total += round4(nnz[i]);
    }
    idx.resize(total);
    val.resize(total);
    std::mutex mu;
    uint64_t bad = n;
    uint32_t voc = 0;
    host_parallel(n, [&](uint64_t lo, uint64_t hi) {
        uint32_t v_max = 0;
        uint64_t my_bad = n;
        for (uint64_t i = lo; i < hi; ++i) {
            const uint64_t b = sv.ptr ? sv.ptr[i] : 0, o = off[i];
            const uint32_t m = nnz[i];
            for (uint32_t j = 0; j < m; ++j) {
                const uint32_t x = sv.idx[b + j];
                if (j > 0 && x <= sv.idx[b + j - 1] && my_bad == n) my_bad = i;
                idx[o + j] = x;
                val[o + j] = sv.val[b + j];
                v_max = std::max(v_max, x + 1);
            }
            for (uint32_t j = m; j < round4(m); ++j) {
                idx[o + j] = kPad;
                val[o + j] = 0.0f;
            }
        }
        std::lock_guard<std::mutex> lock(mu);
        voc = std::max(voc, v_max);
        bad = std::min(bad, my_bad);
    });
    if (bad < n)
        throw Error("unsorted-sparse", "doc " + std::to_string(bad) + ": " + path + " indices must be strictly ascending");
    if (vocab) *vocab = voc;
}

void copy_list(const fg_list_view& lv, uint64_t n, HostList& out) {
    out.ptr.assign(n + 1, 0);
    out.idx.clear();
    if (!lv.ptr) return;
    for (uint64_t i = 0; i < n; ++i) out.ptr[i + 1] = lv.ptr[i + 1] - lv.ptr[0];
    out.idx.assign(lv.idx + lv.ptr[0], lv.idx + lv.ptr[n]);
}

}  // namespace

void QueryUpload::upload(const fg_query_view& q, cudaStream_t s) {
    const uint64_t nq = q.count;
    auto csr = [&](const uint64_t* ptr, const uint32_t* idx, const float* val, DevBuf<uint64_t>& dp,
                   DevBuf<uint32_t>& di, DevBuf<float>* dv, uint32_t& mx) {
        std::vector<uint64_t> p(nq + 1, 0);
        mx = 0;
        if (ptr)
            for (uint64_t i = 0; i < nq; ++i) {
                p[i + 1] = ptr[i + 1] - ptr[0];
                mx = std::max<uint32_t>(mx, static_cast<uint32_t>(ptr[i + 1] - ptr[i]));
            }
        dp.upload(p, s);
        const uint64_t total = p[nq];
        di.ensure(std::max<uint64_t>(total, 1));
        if (total) di.upload(idx + ptr[0], total, s);
        if (dv) {
            dv->ensure(std::max<uint64_t>(total, 1));
            if (total) dv->upload(val + ptr[0], total, s);
        }
        h2d_bytes += p.size() * 8 + total * (dv ? 8 : 4);
    };
    h2d_bytes = 0;
    dense.ensure(std::max<uint64_t>(nq * q.dense_dim, 1));
    dense.upload(q.dense, nq * q.dense_dim, s);
    std::vector<float4> w(nq);
    for (uint64_t i = 0; i < nq; ++i)
        w[i] = q.weights ? make_float4(q.weights[i].dense, q.weights[i].learned,
                                       q.weights[i].statistical, q.weights[i].entity)
                         : make_float4(1.f, 1.f, 1.f, 0.f);
    weights.upload(w, s);
    csr(q.learned.ptr, q.learned.idx, q.learned.val, l_ptr, l_idx, &l_val, max_lnnz);
    csr(q.statistical.ptr, q.statistical.idx, q.statistical.val, s_ptr, s_idx, &s_val, max_snnz);
    csr(q.required_keywords.ptr, q.required_keywords.idx, nullptr, req_ptr, req_idx, nullptr, max_req);
    auto per = [&](const uint32_t* src, uint32_t dflt, DevBuf<uint32_t>& dst, uint32_t& mx) {
        std::vector<uint32_t> v(nq);
        mx = 0;
        for (uint64_t i = 0; i < nq; ++i) {
            v[i] = src ? src[i] : dflt;
            mx = std::max(mx, v[i]);
        }
        dst.upload(v, s);
        h2d_bytes += nq * 4;
    };
    uint32_t mh = 0;
    per(q.k, 10, k, max_k);
    per(q.beam_width, 64, beam, max_beam);
    per(q.max_entity_hops, 2, hops, mh);
    h2d_bytes += nq * q.dense_dim * 4 + nq * 16;
    dq = DevQueries{nq,         q.dense_dim, dense.get(),   weights.get(), l_ptr.get(),
                    l_idx.get(), l_val.get(), s_ptr.get(),   s_idx.get(),   s_val.get(),
                    req_ptr.get(), req_idx.get(), k.get(),    beam.get(),    hops.get()};
}


// Device-derived state of a corpus whose rows are uploaded: the DevCorpus
// view, squared norms (finalize_fused, types.cpp:74-79), the packed gather
// records, and the host copies / maxima the error bounds use.
void corpus_finalize(fg_corpus& c) {
    const uint64_t n = c.n;
    cudaStream_t s = c.stream;
    c.sqnorm.alloc(n);
    c.dnorm.alloc(n);

    c.dc = DevCorpus{n,
              c.dim,
              c.dstride,
              c.dense.get(),
              c.l_off.get(),
              c.l_nnz.get(),
              c.l_idx.get(),
              c.l_val.get(),
              c.s_off.get(),
              c.s_nnz.get(),
              c.s_idx.get(),
              c.s_val.get(),
              c.kw_ptr.get(),
              c.kw_idx.get(),
              c.ent_ptr.get(),
              c.ent_idx.get(),
              c.sqnorm.get(),
              c.dnorm.get(),
              c.deleted.get(),
              nullptr};
    sqnorm_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c.dc, c.sqnorm.get(), c.dnorm.get());
    FGB_LAUNCH("sqnorm_kernel");
    // offsets / 4 must fit 32 bits and nnz 16 bits for the packed record
    const uint64_t l_end = c.l_nnz_total4, s_end = c.s_nnz_total4;
    if (c.max_lnnz < 65536 && c.max_snnz < 65536 && l_end < (1ull << 32) && s_end < (1ull << 32)) {
        c.meta.alloc(n);
        meta_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(c.dc, c.dnorm.get(), c.meta.get());
        FGB_LAUNCH("meta_kernel");
        c.dc.meta = c.meta.get();
    }
    c.sqnorm_h.resize(n);
    c.sqnorm.download(c.sqnorm_h.data(), n, s);
    FGB_CUDA(cudaStreamSynchronize(s));
    c.max_sqnorm = 0.0;
    for (double x : c.sqnorm_h) c.max_sqnorm = std::max(c.max_sqnorm, x);
    {
        std::vector<double> dn(n);
        c.dnorm.download(dn.data(), n, s);
        FGB_CUDA(cudaStreamSynchronize(s));
        c.max_dnorm = 0.0;
        for (double x : dn) c.max_dnorm = std::max(c.max_dnorm, x);
    }
}

// Appends the rows of `v` to the device corpus (insert_batch, update.cpp:94-103):
// device arrays are reallocated with the old rows copied device-to-device and
// the new ones uploaded; keywords default to the statistical support as
// make_document does (corpus.cpp:113-117).  Validation happens in the caller.
void corpus_append(fg_corpus& c, const fg_corpus_view& v) {
    const uint64_t n0 = c.n, b = v.n, n = n0 + b;
    cudaStream_t s = c.stream;
    {
        DevBuf<float> dense(n * c.dstride);
        FGB_CUDA(cudaMemcpyAsync(dense.get(), c.dense.get(), n0 * c.dstride * 4, cudaMemcpyDeviceToDevice, s));
        if (c.dim == c.dstride) {  // (rows need no padding: straight from the caller's array)
            FGB_CUDA(cudaMemcpyAsync(dense.get() + n0 * c.dstride, v.dense, b * c.dim * 4, cudaMemcpyHostToDevice, s));
        } else {
            std::vector<float> pad(b * c.dstride, 0.0f);
            for (uint64_t i = 0; i < b; ++i) std::memcpy(pad.data() + i * c.dstride, v.dense + i * c.dim, c.dim * 4);
            FGB_CUDA(cudaMemcpyAsync(dense.get() + n0 * c.dstride, pad.data(), pad.size() * 4, cudaMemcpyHostToDevice, s));
            FGB_CUDA(cudaStreamSynchronize(s));  // (pad dies here)
        }
        FGB_CUDA(cudaStreamSynchronize(s));
        c.dense = std::move(dense);
    }
    for (int p = 0; p < 2; ++p) {
        const bool learned = p == 0;
        std::vector<uint64_t> off;
        std::vector<uint32_t> nnz, idx;
        std::vector<float> val;
        uint32_t mx = 0;
        build_sparse(learned ? v.learned : v.statistical, b, off, nnz, idx, val, mx,
                     learned ? "learned" : "statistical");
        uint64_t& total4 = learned ? c.l_nnz_total4 : c.s_nnz_total4;
        const uint64_t base = total4 * 4, add = idx.size();
        for (auto& o : off) o += base;
        DevBuf<uint64_t>& doff = learned ? c.l_off : c.s_off;
        DevBuf<uint32_t>& dnnz = learned ? c.l_nnz : c.s_nnz;
        DevBuf<uint32_t>& didx = learned ? c.l_idx : c.s_idx;
        DevBuf<float>& dval = learned ? c.l_val : c.s_val;
        DevBuf<uint64_t> noff(n);
        DevBuf<uint32_t> nnnz(n), nidx(std::max<uint64_t>(base + add, 4));
        DevBuf<float> nval(std::max<uint64_t>(base + add, 4));
        FGB_CUDA(cudaMemcpyAsync(noff.get(), doff.get(), n0 * 8, cudaMemcpyDeviceToDevice, s));
        FGB_CUDA(cudaMemcpyAsync(nnnz.get(), dnnz.get(), n0 * 4, cudaMemcpyDeviceToDevice, s));
        FGB_CUDA(cudaMemcpyAsync(noff.get() + n0, off.data(), b * 8, cudaMemcpyHostToDevice, s));
        FGB_CUDA(cudaMemcpyAsync(nnnz.get() + n0, nnz.data(), b * 4, cudaMemcpyHostToDevice, s));
        if (base) {
            FGB_CUDA(cudaMemcpyAsync(nidx.get(), didx.get(), base * 4, cudaMemcpyDeviceToDevice, s));
            FGB_CUDA(cudaMemcpyAsync(nval.get(), dval.get(), base * 4, cudaMemcpyDeviceToDevice, s));
        }
        if (add) {
            FGB_CUDA(cudaMemcpyAsync(nidx.get() + base, idx.data(), add * 4, cudaMemcpyHostToDevice, s));
            FGB_CUDA(cudaMemcpyAsync(nval.get() + base, val.data(), add * 4, cudaMemcpyHostToDevice, s));
        }
        FGB_CUDA(cudaStreamSynchronize(s));
        doff = std::move(noff);
        dnnz = std::move(nnnz);
        didx = std::move(nidx);
        dval = std::move(nval);
        total4 += add / 4;
        (learned ? c.max_lnnz : c.max_snnz) = std::max(learned ? c.max_lnnz : c.max_snnz, mx);
        uint32_t& voc = learned ? c.l_vocab : c.s_vocab;
        for (uint32_t t : idx)
            if (t != kPad) voc = std::max(voc, t + 1);
    }
    HostList kw, ents;
    if (v.keywords.ptr) {
        copy_list(v.keywords, b, kw);
    } else {
        kw.ptr.assign(b + 1, 0);
        for (uint64_t i = 0; i < b; ++i) {
            const uint64_t lo = v.statistical.ptr ? v.statistical.ptr[i] : 0;
            const uint64_t hi = v.statistical.ptr ? v.statistical.ptr[i + 1] : 0;
            kw.idx.insert(kw.idx.end(), v.statistical.idx + lo, v.statistical.idx + hi);
            kw.ptr[i + 1] = kw.idx.size();
        }
    }
    copy_list(v.entities, b, ents);
    auto extend = [&](HostList& dst, const HostList& src) {
        const uint64_t base = dst.ptr.back();
        for (uint64_t i = 0; i < b; ++i) dst.ptr.push_back(base + src.ptr[i + 1]);
        dst.idx.insert(dst.idx.end(), src.idx.begin(), src.idx.end());
    };
    extend(c.keywords, kw);
    extend(c.entities, ents);
    c.kw_ptr.upload(c.keywords.ptr, s);
    c.kw_idx.upload(c.keywords.idx.empty() ? std::vector<uint32_t>(1, 0) : c.keywords.idx, s);
    c.ent_ptr.upload(c.entities.ptr, s);
    c.ent_idx.upload(c.entities.idx.empty() ? std::vector<uint32_t>(1, 0) : c.entities.idx, s);
    for (uint64_t i = 0; i < b; ++i) c.doc_id.push_back(v.doc_id ? v.doc_id[i] : n0 + i);
    c.deleted_h.resize(n, 0);
    c.deleted.upload(c.deleted_h, s);
    FGB_CUDA(cudaStreamSynchronize(s));
    c.n = n;
    corpus_finalize(c);
}

CorpusMark corpus_mark(const fg_corpus& c) { return {c.n, c.l_nnz_total4, c.s_nnz_total4}; }

void corpus_rollback(fg_corpus& c, const CorpusMark& m) {
    // the device arrays keep their (unused) tail; maxima and vocabulary
    // bounds stay as upper bounds (they only widen error bounds / smem sizing)
    c.n = m.n;
    c.dc.n = m.n;
    c.l_nnz_total4 = m.l4;
    c.s_nnz_total4 = m.s4;
    c.doc_id.resize(m.n);
    c.deleted_h.resize(m.n);
    c.sqnorm_h.resize(m.n);
    for (HostList* h : {&c.keywords, &c.entities}) {
        h->ptr.resize(m.n + 1);
        h->idx.resize(h->ptr.back());
    }
}

DevCorpus corpus_rows(const DevCorpus& d, uint64_t first, uint64_t count) {
    DevCorpus v = d;
    v.n = count;
    v.dense = d.dense + first * d.dstride;
    v.l_off = d.l_off + first;
    v.l_nnz = d.l_nnz + first;
    v.s_off = d.s_off + first;
    v.s_nnz = d.s_nnz + first;
    v.kw_ptr = d.kw_ptr + first;
    v.ent_ptr = d.ent_ptr + first;
    v.sqnorm = d.sqnorm + first;
    v.dnorm = d.dnorm + first;
    v.deleted = d.deleted + first;
    v.meta = d.meta ? d.meta + first : nullptr;
    return v;  // idx/val arrays stay shared: offsets are absolute
}

}  // namespace fgb

using namespace fgb;

extern "C" {

int fg_corpus_upload(const fg_corpus_view* v, int device, fg_corpus** out) {
    return guarded([&] {
        if (!v || !out) throw Error("invalid-argument", "null pointer");
        if (v->n == 0) throw Error("empty-corpus", "corpus holds no documents");
        if (v->n >= 0x7FFFFFFFull) throw Error("invalid-argument", "corpus exceeds 2^31-1 nodes");
        require_device(device);
        HostTimer ht("corpus_upload");
        auto c = std::make_unique<fg_corpus>();
        c->device = device;
        c->n = v->n;
        c->dim = v->dense_dim;
        c->dstride = round4(std::max<uint32_t>(v->dense_dim, 1));
        c->learned_dim = v->learned_dim;
        c->statistical_dim = v->statistical_dim;
        FGB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        cudaStream_t s = c->stream;
        const uint64_t n = v->n;

        // dense rows zero padded to 16 B, then both sparse paths: packed
        // on host threads straight into pinned chunks while the previous
        // chunk is copied
        if (n * c->dstride * 4ull < (size_t(64) << 20)) {  // small corpora: pageable copies
            std::vector<float> pad(n * c->dstride, 0.0f);
            for (uint64_t i = 0; i < n; ++i)
                std::memcpy(pad.data() + i * c->dstride, v->dense + i * c->dim, c->dim * 4ull);
            c->dense.upload(pad, s);
            for (int path = 0; path < 2; ++path) {
                std::vector<uint64_t> off;
                std::vector<uint32_t> nnz, idx;
                std::vector<float> val;
                const bool learned = path == 0;
                build_sparse(learned ? v->learned : v->statistical, n, off, nnz, idx, val,
                             learned ? c->max_lnnz : c->max_snnz, learned ? "learned" : "statistical",
                             learned ? &c->l_vocab : &c->s_vocab);
                (learned ? c->l_nnz_total4 : c->s_nnz_total4) = idx.size() / 4;
                if (idx.empty()) {
                    idx.assign(4, kPad);
                    val.assign(4, 0.f);
                }
                (learned ? c->l_off : c->s_off).upload(off, s);
                (learned ? c->l_nnz : c->s_nnz).upload(nnz, s);
                (learned ? c->l_idx : c->s_idx).upload(idx, s);
                (learned ? c->l_val : c->s_val).upload(val, s);
                FGB_CUDA(cudaStreamSynchronize(s));
            }
        } else {
            PinnedStage st;
            // unpadded rows up to 4 GB: page-locked in place (1M docs: 0.38-0.40 s
            // vs 0.45 s through the stage); larger corpora through the pinned
            // stage (10M docs: 4.2-4.7 s vs 6.5 s — locking 30 GB of pages costs
            // more than the staged copies; tools/upload_probe.py)
            const char* le = std::getenv("FGB_UPLOAD_LOCK");  // dev A/B: 0 = stage, 1 = lock
            const bool lock = le ? le[0] != '0' : n * c->dstride * 4ull <= (4ull << 30);
            if (c->dim == c->dstride && lock) {
                upload_locked(c->dense, v->dense, n * c->dstride, s);
            } else {
                c->dense.ensure(n * c->dstride);
                stream_dense(v->dense, n, c->dim, c->dstride, c->dense.get(), st, s);
            }
            ht.mark("dense");
            std::vector<uint64_t> off;
            std::vector<uint32_t> nnz;
            const uint64_t lt = stream_sparse(v->learned, n, off, nnz, c->max_lnnz, c->l_vocab, c->l_idx, c->l_val,
                                              st, s, "learned");
            c->l_nnz_total4 = lt / 4;
            c->l_off.upload(off, s);
            c->l_nnz.upload(nnz, s);
            FGB_CUDA(cudaStreamSynchronize(s));
            ht.mark("learned");
            const uint64_t stt = stream_sparse(v->statistical, n, off, nnz, c->max_snnz, c->s_vocab, c->s_idx,
                                               c->s_val, st, s, "statistical");
            c->s_nnz_total4 = stt / 4;
            c->s_off.upload(off, s);
            c->s_nnz.upload(nnz, s);
            FGB_CUDA(cudaStreamSynchronize(s));
            ht.mark("statistical");
        }
        // keywords default to the statistical support (corpus.cpp:116)
        if (v->keywords.ptr) {
            copy_list(v->keywords, n, c->keywords);
        } else {
            fg_list_view kv{v->statistical.ptr, v->statistical.idx};
            copy_list(kv, n, c->keywords);
        }
        copy_list(v->entities, n, c->entities);
        for (uint64_t i = 0; i < n; ++i) {
            if (!std::is_sorted(c->entities.begin(i), c->entities.end(i)) ||
                !std::is_sorted(c->keywords.begin(i), c->keywords.end(i)))
                throw Error("unsorted-sparse", "doc " + std::to_string(i) +
                                                   ": keyword/entity lists must be sorted");
        }
        c->kw_ptr.upload(c->keywords.ptr, s);
        c->kw_idx.upload(c->keywords.idx.empty() ? std::vector<uint32_t>(1, 0) : c->keywords.idx, s);
        c->ent_ptr.upload(c->entities.ptr, s);
        c->ent_idx.upload(c->entities.idx.empty() ? std::vector<uint32_t>(1, 0) : c->entities.idx, s);
        c->doc_id.resize(n);
        for (uint64_t i = 0; i < n; ++i) c->doc_id[i] = v->doc_id ? v->doc_id[i] : i;
        c->deleted_h.assign(n, 0);
        if (v->deleted)
            for (uint64_t i = 0; i < n; ++i) c->deleted_h[i] = v->deleted[i] ? 1 : 0;
        c->deleted.upload(c->deleted_h, s);
        ht.mark("lists");
        corpus_finalize(*c);
        ht.mark("done");
        *out = c.release();
    });
}

int fg_corpus_free(fg_corpus* c) {
    if (c) {
        cudaSetDevice(c->device);
        if (c->stream) cudaStreamDestroy(c->stream);
        delete c;
    }
    return FG_OK;
}

int fg_corpus_size(const fg_corpus* c, uint64_t* n, uint32_t* dim) {
    return guarded([&] {
        if (!c) throw Error("invalid-argument", "null corpus");
        if (n) *n = c->n;
        if (dim) *dim = c->dim;
    });
}

int fg_corpus_sqnorm(const fg_corpus* c, double* out) {
    return guarded([&] { std::copy(c->sqnorm_h.begin(), c->sqnorm_h.end(), out); });
}

int fg_corpus_set_deleted(fg_corpus* c, const uint8_t* flags) {
    return guarded([&] {
        FGB_CUDA(cudaSetDevice(c->device));
        for (uint64_t i = 0; i < c->n; ++i) c->deleted_h[i] = flags[i] ? 1 : 0;
        c->deleted.upload(c->deleted_h, c->stream);
        FGB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

// build_query_vector (corpus.cpp:86-103) on the host: the fp32 products the
// kernels apply in-register, exposed for the fusion-weight API and tests.
int fg_build_query_vector(const fg_query_view* q, uint64_t i, float* dense_out, uint32_t* lnnz,
                          float* lval, uint32_t* snnz, float* sval, double* sqnorm) {
    return guarded([&] {
        if (!q || i >= q->count) throw Error("invalid-argument", "query index out of range");
        const fg_weights w = q->weights ? q->weights[i] : fg_weights{1.f, 1.f, 1.f, 0.f};
        const float* x = q->dense + i * q->dense_dim;
        double acc = 0.0;
        for (uint32_t j = 0; j < q->dense_dim; ++j) {
            dense_out[j] = w.dense * x[j];
            acc += static_cast<double>(dense_out[j]) * static_cast<double>(dense_out[j]);
        }
        auto scale = [&](const fg_sparse_view& sv, float wt, uint32_t* nnz, float* out) {
            double a = 0.0;
            *nnz = 0;
            if (!sv.ptr || wt == 0.0f) return a;
            const uint64_t b = sv.ptr[i], e = sv.ptr[i + 1];
            for (uint64_t j = b; j < e; ++j) {
                out[j - b] = wt * sv.val[j];
                a += static_cast<double>(out[j - b]) * static_cast<double>(out[j - b]);
            }
            *nnz = static_cast<uint32_t>(e - b);
            return a;
        };
        const double l = scale(q->learned, w.learned, lnnz, lval);
        const double s = scale(q->statistical, w.statistical, snnz, sval);
        acc += l;
        acc += s;
        if (sqnorm) *sqnorm = acc;
    });
}

int fg_batch_scores(const fg_corpus* c, const fg_query_view* q, uint64_t qi, const uint32_t* ids,
                    uint64_t m, double* out) {
    return guarded([&] {
        if (!c || !q || qi >= q->count) throw Error("invalid-argument", "bad query");
        FGB_CUDA(cudaSetDevice(c->device));
        if (q->dense_dim != c->dim)
            throw Error("dim-mismatch", "dense dimensions differ: " + std::to_string(q->dense_dim) +
                                            " vs " + std::to_string(c->dim));
        for (uint64_t i = 0; i < m; ++i)
            if (ids[i] >= c->n)
                throw Error("unknown-id", "node " + std::to_string(ids[i]) + " out of range");
        if (m == 0) return;
        cudaStream_t s = c->stream;
        // single-query sub-view
        fg_query_view one = *q;
        one.count = 1;
        one.dense = q->dense + qi * q->dense_dim;
        uint64_t lp[2], sp[2];
        if (q->learned.ptr) {
            lp[0] = q->learned.ptr[qi];
            lp[1] = q->learned.ptr[qi + 1];
            one.learned.ptr = lp;
        }
        if (q->statistical.ptr) {
            sp[0] = q->statistical.ptr[qi];
            sp[1] = q->statistical.ptr[qi + 1];
            one.statistical.ptr = sp;
        }
        if (q->weights) one.weights = q->weights + qi;
        one.required_keywords = {nullptr, nullptr};
        one.entities = {nullptr, nullptr};
        one.k = nullptr;
        one.beam_width = nullptr;
        one.max_entity_hops = nullptr;
        QueryUpload up;
        up.upload(one, s);
        DevBuf<uint32_t> d_ids;
        d_ids.upload(ids, m, s);
        DevBuf<double> d_out(m);
        const uint32_t lcap = hash_capacity(up.max_lnnz), scap = hash_capacity(up.max_snnz);
        const size_t sm = stage_bytes(c->dstride, lcap, scap);
        if (sm > 48 * 1024)
            FGB_CUDA(cudaFuncSetAttribute(batch_scores_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        batch_scores_kernel<<<(unsigned)((m + 127) / 128), 128, sm, s>>>(c->dc, up.dq, 0, d_ids.get(), m,
                                                                     d_out.get(), lcap, scap);
        FGB_LAUNCH("batch_scores_kernel");
        d_out.download(out, m, s);
        FGB_CUDA(cudaStreamSynchronize(s));
    });
}

int fg_pair_scores(const fg_corpus* c, const uint32_t* a, const uint32_t* b, uint64_t m,
                   double* out) {
    return guarded([&] {
        if (!c) throw Error("invalid-argument", "null corpus");
        FGB_CUDA(cudaSetDevice(c->device));
        for (uint64_t i = 0; i < m; ++i)
            if (a[i] >= c->n || b[i] >= c->n)
                throw Error("unknown-id", "node out of range");
        if (m == 0) return;
        cudaStream_t s = c->stream;
        DevBuf<uint32_t> da, db;
        da.upload(a, m, s);
        db.upload(b, m, s);
        DevBuf<double> d_out(m);
        pair_kernel<<<(unsigned)((m + 127) / 128), 128, 0, s>>>(c->dc, da.get(), db.get(), m, d_out.get());
        FGB_LAUNCH("pair_kernel");
        d_out.download(out, m, s);
        FGB_CUDA(cudaStreamSynchronize(s));
    });
}

}  // extern "C"
