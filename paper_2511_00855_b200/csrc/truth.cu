// truth.cu — K6: exhaustive weighted top-k (brute_force_topk, eval.cpp:14-51).
//
// Stage 1: grid (P, queries): each CTA stages one weighted query in shared
// memory and scores a strided slice of the corpus bit-exactly (one thread per
// document), skipping deleted documents and — when keywords are required —
// documents lacking any of them (conjunctive, eval.cpp:29-37).  Every thread
// keeps a private sorted top-k (score desc, doc_id asc, eval.cpp:40-44) in
// global scratch; the CTA then merges its threads' lists head by head into k
// partial winners.  Stage 2: one CTA per query merges the P partial lists.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "fg_cuda.hpp"
#include "query_stage.cuh"

namespace fgb {
namespace {

constexpr int kTruthThreads = 128;

__device__ __forceinline__ bool before(double s1, uint64_t d1, double s2, uint64_t d2) {
    return s1 != s2 ? s1 > s2 : d1 < d2;
}

struct Lists {
    double* s;
    uint64_t* d;
    uint32_t* n;
};

// Merge kTruthThreads sorted lists (list t at [t*stride, t*stride+len[t]))
// into out[0..k).
__device__ uint32_t block_merge(Lists in, const uint32_t* len, uint32_t stride, uint32_t k, Lists out) {
    __shared__ double hs[kTruthThreads];
    __shared__ uint64_t hd[kTruthThreads];
    __shared__ uint32_t win;
    const uint32_t tid = threadIdx.x;
    uint32_t head = 0, taken = 0;
    for (; taken < k; ++taken) {
        const bool has = head < len[tid];
        hs[tid] = has ? in.s[(uint64_t)tid * stride + head] : 0.0;
        hd[tid] = has ? in.d[(uint64_t)tid * stride + head] : ~0ull;
        __syncthreads();
        if (tid == 0) {
            uint32_t b = 0xFFFFFFFFu;
            for (uint32_t t = 0; t < kTruthThreads; ++t) {
                if (hd[t] == ~0ull) continue;
                if (b == 0xFFFFFFFFu || before(hs[t], hd[t], hs[b], hd[b])) b = t;
            }
            win = b;
        }
        __syncthreads();
        const uint32_t w = win;
        if (w == 0xFFFFFFFFu) break;
        if (tid == w) {
            out.s[taken] = in.s[(uint64_t)tid * stride + head];
            out.d[taken] = in.d[(uint64_t)tid * stride + head];
            out.n[taken] = in.n[(uint64_t)tid * stride + head];
            ++head;
        }
        __syncthreads();
    }
    return taken;
}

struct TruthArgs {
    DevCorpus c;
    DevQueries q;
    const uint64_t* doc_id;
    const uint8_t* valid;
    uint32_t lcap, scap, kmax, P;
    uint64_t q0;  // first query of this chunk
    Lists scratch;         // [chunk][P][threads][kmax]
    uint32_t* scratch_len; // [chunk][P][threads]
    Lists partial;         // [chunk][P][kmax]
    uint32_t* partial_len; // [chunk][P]
};

__global__ void __launch_bounds__(kTruthThreads) truth_score_kernel(TruthArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint64_t ql = blockIdx.y, qi = a.q0 + ql;
    if (!a.valid[qi]) return;
    const uint32_t k = a.q.k[qi];
    SmemQuery sq;
    stage_query(a.q, qi, a.c.dstride, smem, a.lcap, a.scap, threadIdx.x, blockDim.x, sq,
                [] { __syncthreads(); });
    const uint64_t rb = a.q.req_ptr[qi], re = a.q.req_ptr[qi + 1];
    const uint64_t slot = (ql * a.P + blockIdx.x) * kTruthThreads + threadIdx.x;
    Lists my{a.scratch.s + slot * a.kmax, a.scratch.d + slot * a.kmax, a.scratch.n + slot * a.kmax};
    uint32_t len = 0;
    const uint64_t step = (uint64_t)a.P * kTruthThreads;
    for (uint64_t node = (uint64_t)blockIdx.x * kTruthThreads + threadIdx.x; node < a.c.n; node += step) {
        if (a.c.deleted[node]) continue;
        if (re > rb) {
            bool ok = true;
            const uint64_t kb = a.c.kw_ptr[node], ke = a.c.kw_ptr[node + 1];
            for (uint64_t r = rb; r < re && ok; ++r) ok = sorted_contains(a.c.kw_idx, kb, ke, a.q.req_idx[r]);
            if (!ok) continue;
        }
        const double s = hybrid_score(a.c, sq, node);
        const uint64_t d = a.doc_id[node];
        if (len == k && !before(s, d, my.s[k - 1], my.d[k - 1])) continue;
        uint32_t i = len < k ? len : k - 1;
        while (i > 0 && before(s, d, my.s[i - 1], my.d[i - 1])) {
            my.s[i] = my.s[i - 1];
            my.d[i] = my.d[i - 1];
            my.n[i] = my.n[i - 1];
            --i;
        }
        my.s[i] = s;
        my.d[i] = d;
        my.n[i] = static_cast<uint32_t>(node);
        if (len < k) ++len;
    }
    __shared__ uint32_t lens[kTruthThreads];
    lens[threadIdx.x] = len;
    __syncthreads();
    const uint64_t base = (ql * a.P + blockIdx.x) * kTruthThreads * (uint64_t)a.kmax;
    Lists in{a.scratch.s + base, a.scratch.d + base, a.scratch.n + base};
    const uint64_t pslot = ql * a.P + blockIdx.x;
    Lists out{a.partial.s + pslot * a.kmax, a.partial.d + pslot * a.kmax, a.partial.n + pslot * a.kmax};
    const uint32_t got = block_merge(in, lens, a.kmax, k, out);
    if (threadIdx.x == 0) a.partial_len[pslot] = got;
}

// One CTA per query: merge the P partial lists (P <= kTruthThreads).
__global__ void __launch_bounds__(kTruthThreads) truth_merge_kernel(TruthArgs a, Lists res,
                                                                    uint32_t* r_count,
                                                                    uint32_t hit_stride) {
    const uint64_t ql = blockIdx.x, qi = a.q0 + ql;
    if (!a.valid[qi]) {
        if (threadIdx.x == 0) r_count[qi] = 0;
        return;
    }
    const uint32_t k = a.q.k[qi];
    __shared__ uint32_t lens[kTruthThreads];
    lens[threadIdx.x] = threadIdx.x < a.P ? a.partial_len[ql * a.P + threadIdx.x] : 0;
    __syncthreads();
    const uint64_t base = ql * a.P * (uint64_t)a.kmax;
    Lists in{a.partial.s + base, a.partial.d + base, a.partial.n + base};
    Lists out{res.s + qi * hit_stride, res.d + qi * hit_stride, res.n + qi * hit_stride};
    const uint32_t got = block_merge(in, lens, a.kmax, k, out);
    if (threadIdx.x == 0) r_count[qi] = got;
}

}  // namespace
}  // namespace fgb

using namespace fgb;

extern "C" {

int fg_brute_force_topk(const fg_corpus* c, const fg_query_view* q, fg_search_results* out) {
    return guarded([&] {
        if (!c || !q || !out) throw Error("invalid-argument", "null pointer");
        FGB_CUDA(cudaSetDevice(c->device));
        cudaStream_t s = c->stream;
        const uint64_t nq = q->count;
        std::vector<uint8_t> valid(std::max<uint64_t>(nq, 1), 0);
        std::vector<std::string> errs(nq);
        uint32_t kmax = 1;
        for (uint64_t i = 0; i < nq; ++i) {
            const fg_weights w = q->weights ? q->weights[i] : fg_weights{1.f, 1.f, 1.f, 0.f};
            const uint32_t k = q->k ? q->k[i] : 10;
            try {  // validate_weights + k (eval.cpp:16-17)
                const float parts[4] = {w.dense, w.learned, w.statistical, w.entity};
                for (float p : parts)
                    if (!std::isfinite(p) || p < 0.0f)
                        throw Error("invalid-weights", "weights must be finite and non-negative");
                if (w.dense <= 0.0f && w.learned <= 0.0f && w.statistical <= 0.0f)
                    throw Error("invalid-weights", "at least one vector-path weight must be positive");
                if (k == 0) throw Error("invalid-k", "k must be positive");
                if (q->dense_dim != c->dim)
                    throw Error("dim-mismatch", "dense dimensions differ: " + std::to_string(q->dense_dim) +
                                                    " vs " + std::to_string(c->dim));
            } catch (const Error& e) {
                errs[i] = e.what();
                continue;
            }
            valid[i] = 1;
            kmax = std::max(kmax, k);
        }
        if (out->hit_stride < kmax && nq) throw Error("invalid-argument", "hit_stride < max k");
        if (kmax > 4096) throw Error("invalid-k", "brute force supports k <= 4096");
        QueryUpload up;
        up.upload(*q, s);
        DevBuf<uint8_t> d_valid;
        d_valid.upload(valid, s);
        DevBuf<uint64_t> d_doc;
        d_doc.upload(c->doc_id, s);
        int sms = 0;
        FGB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
        const uint32_t P = static_cast<uint32_t>(std::min<uint64_t>(
            kTruthThreads, std::max<uint64_t>(1, (c->n + kTruthThreads * 64 - 1) / (kTruthThreads * 64))));
        // chunk so that scratch stays bounded (~2 GB)
        const uint64_t per_q = (uint64_t)P * kTruthThreads * kmax * 20 + (uint64_t)P * kmax * 20 + 64;
        const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(std::max<uint64_t>(nq, 1), (2ull << 30) / per_q));
        DevBuf<double> ss(chunk * P * kTruthThreads * kmax), ps(chunk * P * kmax);
        DevBuf<uint64_t> sd(chunk * P * kTruthThreads * kmax), pd(chunk * P * kmax);
        DevBuf<uint32_t> sn(chunk * P * kTruthThreads * kmax), pn(chunk * P * kmax),
            slen(chunk * P * kTruthThreads), plen(chunk * P);
        const uint32_t stride = std::max(out->hit_stride, 1u);
        DevBuf<uint32_t> r_node(std::max<uint64_t>(nq * stride, 1)), r_count(std::max<uint64_t>(nq, 1));
        DevBuf<double> r_score(std::max<uint64_t>(nq * stride, 1));
        DevBuf<uint64_t> r_doc(std::max<uint64_t>(nq * stride, 1));
        const uint32_t lcap = hash_capacity(up.max_lnnz), scap = hash_capacity(up.max_snnz);
        const size_t sm = stage_bytes(c->dstride, lcap, scap);
        FGB_CUDA(cudaFuncSetAttribute(truth_score_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        for (uint64_t q0 = 0; q0 < nq; q0 += chunk) {
            const uint64_t qc = std::min(chunk, nq - q0);
            TruthArgs a{c->dc, up.dq, d_doc.get(), d_valid.get(), lcap, scap, kmax, P, q0,
                        Lists{ss.get(), sd.get(), sn.get()}, slen.get(),
                        Lists{ps.get(), pd.get(), pn.get()}, plen.get()};
            truth_score_kernel<<<dim3(P, (unsigned)qc), kTruthThreads, sm, s>>>(a);
            FGB_LAUNCH("truth_score_kernel");
            truth_merge_kernel<<<(unsigned)qc, kTruthThreads, 0, s>>>(
                a, Lists{r_score.get(), r_doc.get(), r_node.get()}, r_count.get(), stride);
            FGB_LAUNCH("truth_merge_kernel");
        }
        std::vector<uint32_t> h_node(nq * stride), h_count(nq);
        std::vector<double> h_score(nq * stride);
        r_node.download(h_node.data(), nq * stride, s);
        r_score.download(h_score.data(), nq * stride, s);
        r_count.download(h_count.data(), nq, s);
        FGB_CUDA(cudaStreamSynchronize(s));
        for (uint64_t i = 0; i < nq; ++i) {
            const uint32_t cnt = valid[i] ? h_count[i] : 0;
            out->hit_count[i] = cnt;
            for (uint32_t j = 0; j < cnt; ++j) {
                const uint32_t node = h_node[i * stride + j];
                out->node[i * out->hit_stride + j] = node;
                out->doc_id[i * out->hit_stride + j] = c->doc_id[node];
                out->score[i * out->hit_stride + j] = h_score[i * stride + j];
            }
            if (out->expanded) out->expanded[i] = 0;
            if (out->scored) out->scored[i] = valid[i] ? c->n : 0;
            if (out->warnings) out->warnings[i] = 0;
            if (out->errors && out->error_stride) {
                char* dst = out->errors + i * out->error_stride;
                std::strncpy(dst, errs[i].c_str(), out->error_stride - 1);
                dst[out->error_stride - 1] = 0;
            }
        }
    });
}

}  // extern "C"
