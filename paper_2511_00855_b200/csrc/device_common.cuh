// device_common.cuh — device-side layout of the corpus and the bit-exact
// hybrid distance (K1), shared by every kernel.
//
// Parity contract (scoring.cpp:10-99): a hybrid score is
//     acc  = sum_i (double)q_i * (double)d_i        (index order)
//     acc += sum_{shared t, ascending} (double)ql_t * (double)dl_t
//     acc += sum_{shared t, ascending} (double)qs_t * (double)ds_t
// with every product exact in fp64 (fp32 x fp32 fits in 48 bits) and every
// sum rounded once.  We evaluate each sum as a sequential chain of
// __fma_rn(a, b, acc) — exact product + one rounding, identical to the
// reference's `acc += a * b` — in the same order, so every score is
// BIT-IDENTICAL to fusegraph::hybrid_score.  One thread owns one
// (query, candidate) chain; parallelism comes from many candidates.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace fgb {

constexpr uint32_t kPad = 0xFFFFFFFFu;    // padding index in sparse rows
constexpr uint32_t kEmpty = 0xFFFFFFFFu;  // empty hash slot

// DocumentStore on HBM (types.hpp:119-133), structure-of-arrays:
//  dense   n x dstride fp32, dstride = dim rounded up to 4 (16-B rows, zero pad)
//  sparse  per path: row offset (multiple of 4 entries) + nnz, idx/val arrays
//          padded per row to a multiple of 4 with (kPad, 0) so rows load as
//          uint4/float4 (and bulk-copy at 16-B granularity)
//  keywords, entities: plain CSR (sorted ids per doc)
struct DevCorpus {
    uint64_t n;
    uint32_t dim, dstride;
    const float* dense;
    const uint64_t* l_off;
    const uint32_t* l_nnz;
    const uint32_t* l_idx;
    const float* l_val;
    const uint64_t* s_off;
    const uint32_t* s_nnz;
    const uint32_t* s_idx;
    const float* s_val;
    const uint64_t* kw_ptr;
    const uint32_t* kw_idx;
    const uint64_t* ent_ptr;
    const uint32_t* ent_idx;
    const double* sqnorm;
    const double* dnorm;  // sqrt of the dense self-dot (screening bounds only)
    const uint8_t* deleted;
    // packed per-node record for one-load gathers (nullptr when a row has
    // >= 65,536 postings): x = l_off / 4, y = s_off / 4,
    // z = l_nnz | s_nnz << 16, w = bits of float(dnorm) rounded up
    const uint4* meta;
};

// ---------------------------------------------------------------- hashing
__device__ __forceinline__ uint32_t hslot(uint32_t key, uint32_t mask) {
    return (key * 2654435761u) & mask;  // mask = capacity - 1 (power of two)
}

// Insert key->val into an open-addressing table (keys pre-set to kEmpty).
// Keys are unique per table (strictly ascending sparse indices).
__device__ __forceinline__ void hash_insert(uint32_t* keys, float* vals, uint32_t mask,
                                            uint32_t key, float val) {
    uint32_t s = hslot(key, mask);
    while (true) {
        const uint32_t prev = atomicCAS(&keys[s], kEmpty, key);
        if (prev == kEmpty || prev == key) {
            vals[s] = val;
            return;
        }
        s = (s + 1) & mask;
    }
}

__device__ __forceinline__ bool hash_find(const uint32_t* keys, const float* vals, uint32_t mask,
                                          uint32_t key, float& out) {
    uint32_t s = hslot(key, mask);
    while (true) {
        const uint32_t k = keys[s];
        if (k == key) {
            out = vals[s];
            return true;
        }
        if (k == kEmpty) return false;
        s = (s + 1) & mask;
    }
}

__host__ __device__ inline uint32_t hash_capacity(uint32_t nnz) {
    uint32_t c = 16;
    while (c < 2 * nnz) c <<= 1;
    return c;
}

// Bit filter in front of each hash: 2 * capacity words = 64 filter bits per
// hash slot (>= 128 per query term), so a document term that is not a query
// term is rejected by one shared-memory load and a bit test; only filter hits
// (the ~nnz-overlap true matches plus <1% false positives) probe the hash.
__host__ __device__ inline uint32_t filter_words(uint32_t cap) { return 2 * cap; }

__device__ __forceinline__ bool filter_hit(const uint32_t* f, uint32_t fmask, uint32_t key) {
    return (f[(key >> 5) & fmask] >> (key & 31)) & 1u;
}

// A weighted query (or a document acting as one) staged in shared memory:
// dense part as fp64 (dstride doubles, zero padded — the exact widening of
// the fp32 weighted values, so the chain needs one conversion per product),
// and per sparse path a bit filter + hash.
struct SmemQuery {
    const double* dense;  // nullptr: dense path disabled (weight 0) -> contributes +0.0
    const uint32_t* lkeys;
    const float* lvals;
    const uint32_t* lfilt;
    uint32_t lmask;       // 0: learned path empty/disabled
    const uint32_t* skeys;
    const float* svals;
    const uint32_t* sfilt;
    uint32_t smask;
};

// Bytes a staged query/document occupies in shared memory.
__host__ __device__ inline size_t stage_bytes(uint32_t dstride, uint32_t lcap, uint32_t scap) {
    return static_cast<size_t>(dstride) * 8 +
           static_cast<size_t>(lcap + scap) * 8 +
           static_cast<size_t>(filter_words(lcap) + filter_words(scap)) * 4;
}

struct StagePtrs {
    double* dense;
    uint32_t* lkeys;
    float* lvals;
    uint32_t* lfilt;
    uint32_t* skeys;
    float* svals;
    uint32_t* sfilt;
};

__device__ __forceinline__ StagePtrs stage_layout(unsigned char* smem, uint32_t dstride,
                                                  uint32_t lcap, uint32_t scap) {
    StagePtrs p;
    p.dense = reinterpret_cast<double*>(smem);
    p.lkeys = reinterpret_cast<uint32_t*>(p.dense + dstride);
    p.lvals = reinterpret_cast<float*>(p.lkeys + lcap);
    p.skeys = reinterpret_cast<uint32_t*>(p.lvals + lcap);
    p.svals = reinterpret_cast<float*>(p.skeys + scap);
    p.lfilt = reinterpret_cast<uint32_t*>(p.svals + scap);
    p.sfilt = p.lfilt + filter_words(lcap);
    return p;
}

// Dense dot of the staged query against row `node`, sequential over i.
//
// Each step is acc = RN(acc + p_i) with p_i = q_i * d_i computed by DMUL: the
// product of two fp32 values widened to fp64 is EXACT, so RN(acc + p_i) is
// the same rounding as the reference's `acc += a * b` (one rounding of the
// exact a*b + acc).  On B200 a DADD chain has a shorter dependent latency and
// twice the issue rate of a DFMA chain (tools/ubench_chain.cu: 10.2 vs 11.5
// cycles/element, 21.6 vs 16 elements/clk/SM), and the DMULs sit off the chain.
template <uint32_t kStage = 8>
__device__ __forceinline__ double dense_chain(const DevCorpus& c, const double* q, uint64_t node) {
    // Software-pipelined: the next kStage float4 of the row are in flight
    // while the current ones feed the (inherently sequential) fp64 chain.
    const float4* row = reinterpret_cast<const float4*>(c.dense + node * c.dstride);
    const double2* q2 = reinterpret_cast<const double2*>(q);
    const uint32_t n4 = c.dstride >> 2;
    double acc = 0.0;
    float4 cur[kStage], nxt[kStage];
    if (n4 % kStage == 0) {  // d = 128, 768, ...: no per-element guards
#pragma unroll
        for (uint32_t j = 0; j < kStage; ++j) cur[j] = __ldg(row + j);
        for (uint32_t i = 0; i < n4; i += kStage) {
            const bool more = i + kStage < n4;
#pragma unroll
            for (uint32_t j = 0; j < kStage; ++j) nxt[j] = more ? __ldg(row + i + kStage + j) : cur[j];
#pragma unroll
            for (uint32_t j = 0; j < kStage; ++j) {
                const double2 a = q2[2 * (i + j)], b = q2[2 * (i + j) + 1];
                acc = __dadd_rn(acc, __dmul_rn(a.x, (double)cur[j].x));
                acc = __dadd_rn(acc, __dmul_rn(a.y, (double)cur[j].y));
                acc = __dadd_rn(acc, __dmul_rn(b.x, (double)cur[j].z));
                acc = __dadd_rn(acc, __dmul_rn(b.y, (double)cur[j].w));
            }
#pragma unroll
            for (uint32_t j = 0; j < kStage; ++j) cur[j] = nxt[j];
        }
        return acc;
    }
#pragma unroll
    for (uint32_t j = 0; j < kStage; ++j) cur[j] = j < n4 ? __ldg(row + j) : make_float4(0, 0, 0, 0);
    for (uint32_t i = 0; i < n4; i += kStage) {
#pragma unroll
        for (uint32_t j = 0; j < kStage; ++j)
            nxt[j] = i + kStage + j < n4 ? __ldg(row + i + kStage + j) : make_float4(0, 0, 0, 0);
#pragma unroll
        for (uint32_t j = 0; j < kStage; ++j) {
            if (i + j < n4) {
                const double2 a = q2[2 * (i + j)], b = q2[2 * (i + j) + 1];
                acc = __dadd_rn(acc, __dmul_rn(a.x, (double)cur[j].x));
                acc = __dadd_rn(acc, __dmul_rn(a.y, (double)cur[j].y));
                acc = __dadd_rn(acc, __dmul_rn(b.x, (double)cur[j].z));
                acc = __dadd_rn(acc, __dmul_rn(b.y, (double)cur[j].w));
            }
        }
#pragma unroll
        for (uint32_t j = 0; j < kStage; ++j) cur[j] = nxt[j];
    }
    return acc;
}

// One probe of a (filtered) query path: adds q_t * v in the chain when t is a
// query term.  Terms arrive in ascending order (sorted rows).
__device__ __forceinline__ void probe_term(uint32_t t, float v, const uint32_t* keys,
                                           const float* vals, uint32_t mask,
                                           const uint32_t* filt, double& acc) {
    if (t == kPad || !filter_hit(filt, 2 * mask + 1, t)) return;
    float q;
    if (hash_find(keys, vals, mask, t, q)) acc = __fma_rn((double)q, (double)v, acc);
}

// Sparse dot: walk the document row in ascending index order and probe the
// query's filter+hash; matches accumulate in ascending shared-index order,
// exactly the merge/probe order of sparse_dot_impl (scoring.cpp:24-74).
template <uint32_t kStage = 4>  // kStage x 4 entries per stage, the next stage in flight
__device__ __forceinline__ double sparse_chain(const uint32_t* idx, const float* val, uint64_t off,
                                               uint32_t nnz, const uint32_t* keys,
                                               const float* vals, uint32_t mask,
                                               const uint32_t* filt) {
    double acc = 0.0;
    const uint4* i4 = reinterpret_cast<const uint4*>(idx + off);
    const float4* v4 = reinterpret_cast<const float4*>(val + off);
    const uint32_t n4 = (nnz + 3) >> 2;
    const uint4 padi = make_uint4(kPad, kPad, kPad, kPad);
    uint4 ci[kStage], ni[kStage];
    float4 cv[kStage], nv[kStage];
#pragma unroll
    for (uint32_t j = 0; j < kStage; ++j) {
        ci[j] = j < n4 ? __ldg(i4 + j) : padi;
        cv[j] = j < n4 ? __ldg(v4 + j) : make_float4(0, 0, 0, 0);
    }
    for (uint32_t i = 0; i < n4; i += kStage) {
#pragma unroll
        for (uint32_t j = 0; j < kStage; ++j) {
            const bool in = i + kStage + j < n4;
            ni[j] = in ? __ldg(i4 + i + kStage + j) : padi;
            nv[j] = in ? __ldg(v4 + i + kStage + j) : make_float4(0, 0, 0, 0);
        }
#pragma unroll
        for (uint32_t j = 0; j < kStage; ++j) {
            probe_term(ci[j].x, cv[j].x, keys, vals, mask, filt, acc);
            probe_term(ci[j].y, cv[j].y, keys, vals, mask, filt, acc);
            probe_term(ci[j].z, cv[j].z, keys, vals, mask, filt, acc);
            probe_term(ci[j].w, cv[j].w, keys, vals, mask, filt, acc);
        }
#pragma unroll
        for (uint32_t j = 0; j < kStage; ++j) {
            ci[j] = ni[j];
            cv[j] = nv[j];
        }
    }
    return acc;
}

// TMA bulk prefetch of a contiguous span into L2 (one instruction per span,
// no registers or shared memory; 16-B aligned, multiple of 16 bytes).
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Pull a whole document row (dense + the sparse postings a query will walk)
// toward L2 up front, so the chain's stage-by-stage loads hit L2 instead of
// paying a DRAM round trip per stage.
__device__ __forceinline__ void prefetch_row(const DevCorpus& c, const SmemQuery& q, uint64_t node) {
    if (q.dense) l2_prefetch(c.dense + node * c.dstride, c.dstride * 4);
    if (q.lmask) {
        const uint32_t b = ((c.l_nnz[node] + 3) & ~3u) * 4;
        if (b) {
            l2_prefetch(c.l_idx + c.l_off[node], b);
            l2_prefetch(c.l_val + c.l_off[node], b);
        }
    }
    if (q.smask) {
        const uint32_t b = ((c.s_nnz[node] + 3) & ~3u) * 4;
        if (b) {
            l2_prefetch(c.s_idx + c.s_off[node], b);
            l2_prefetch(c.s_val + c.s_off[node], b);
        }
    }
}

// Sparse spans only (the dense row is fetched after screening decides).
__device__ __forceinline__ void prefetch_sparse(const DevCorpus& c, const SmemQuery& q, uint64_t node) {
    if (q.lmask) {
        const uint32_t b = ((c.l_nnz[node] + 3) & ~3u) * 4;
        if (b) {
            l2_prefetch(c.l_idx + c.l_off[node], b);
            l2_prefetch(c.l_val + c.l_off[node], b);
        }
    }
    if (q.smask) {
        const uint32_t b = ((c.s_nnz[node] + 3) & ~3u) * 4;
        if (b) {
            l2_prefetch(c.s_idx + c.s_off[node], b);
            l2_prefetch(c.s_val + c.s_off[node], b);
        }
    }
}

// hybrid_score(weighted query, doc) (scoring.cpp:88-99): dense, then learned,
// then statistical, in that fixed order.
template <uint32_t kStage = 8>
__device__ __forceinline__ double hybrid_score(const DevCorpus& c, const SmemQuery& q,
                                               uint64_t node) {
    prefetch_row(c, q, node);
    double acc = q.dense ? dense_chain<kStage>(c, q.dense, node) : 0.0;
    acc = __dadd_rn(acc, q.lmask ? sparse_chain(c.l_idx, c.l_val, c.l_off[node], c.l_nnz[node],
                                                q.lkeys, q.lvals, q.lmask, q.lfilt)
                                 : 0.0);
    acc = __dadd_rn(acc, q.smask ? sparse_chain(c.s_idx, c.s_val, c.s_off[node], c.s_nnz[node],
                                                q.skeys, q.svals, q.smask, q.sfilt)
                                 : 0.0);
    return acc;
}

// Exact-score screening.  For a candidate whose sparse parts L, S are known,
// the final computed score RN(RN(D + L) + S) (D = the dense chain) is at most
//   L + S + |q||d| + 1e-11 (|q||d| + |L| + |S|)
// (the chain's rounding error is <= d * 2^-53 * sum|q_i d_i| <= 1e-13 |q||d|
// for d <= 9000, two more roundings add 2^-52 relative; the margin covers the
// norms' own rounding).  A candidate whose bound is below a threshold score
// can never beat it, so its 4*d-byte dense row is never read.
__device__ __forceinline__ double score_upper_bound(double qn, double dn, double l, double s) {
    const double qd = qn * dn;
    return l + s + qd + 1e-11 * (qd + fabs(l) + fabs(s)) + 1e-300;
}

__device__ __forceinline__ double sparse_part(const DevCorpus& c, const SmemQuery& q, uint64_t node,
                                              bool learned) {
    if (learned)
        return q.lmask ? sparse_chain(c.l_idx, c.l_val, c.l_off[node], c.l_nnz[node], q.lkeys, q.lvals,
                                      q.lmask, q.lfilt)
                       : 0.0;
    return q.smask ? sparse_chain(c.s_idx, c.s_val, c.s_off[node], c.s_nnz[node], q.skeys, q.svals,
                                  q.smask, q.sfilt)
                   : 0.0;
}

// hybrid_score with screening: returns false (and no score) when the upper
// bound is < `floor`; otherwise the exact, bit-identical score in `out`.
// Partial sums are combined in the reference's order (dense + learned, then
// + statistical), so the result equals hybrid_score exactly.
template <uint32_t kStage = 8>
__device__ __forceinline__ bool hybrid_score_screened(const DevCorpus& c, const SmemQuery& q,
                                                      uint64_t node, double qnorm, double floor,
                                                      double& out) {
    const double l = sparse_part(c, q, node, true);
    const double s = sparse_part(c, q, node, false);
    if (q.dense && score_upper_bound(qnorm, c.dnorm[node], l, s) < floor) return false;
    if (!q.dense && score_upper_bound(0.0, 0.0, l, s) < floor) return false;
    // the whole row toward L2 in one bulk request: only the first stage of
    // the chain below waits for DRAM
    if (q.dense) l2_prefetch(c.dense + node * c.dstride, c.dstride * 4);
    double acc = q.dense ? dense_chain<kStage>(c, q.dense, node) : 0.0;
    acc = __dadd_rn(acc, l);
    out = __dadd_rn(acc, s);
    return true;
}

// Sorted-list membership (sorted_contains, types.cpp:86-88).
__device__ __forceinline__ bool sorted_contains(const uint32_t* a, uint64_t b, uint64_t e,
                                               uint32_t x) {
    while (b < e) {
        const uint64_t m = (b + e) >> 1;
        const uint32_t v = a[m];
        if (v < x)
            b = m + 1;
        else if (v > x)
            e = m;
        else
            return true;
    }
    return false;
}

// SplitMix64 / mix_seed / bounded (rng.hpp:17-41) on the device.
struct DevRng {
    uint64_t state;
    __device__ explicit DevRng(uint64_t seed) : state(seed) {}
    __device__ uint64_t next() {
        uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
};
__device__ __forceinline__ uint64_t dev_mix_seed(uint64_t seed, uint64_t stream) {
    DevRng m(seed ^ (0xA0761D6478BD642FULL * (stream + 1)));
    return m.next();
}
__device__ __forceinline__ uint64_t dev_bounded(DevRng& r, uint64_t bound) {
    return __umul64hi(r.next(), bound);
}

// KnnEntry ordering `better` (knn_graph.cpp:15-18): score desc, id asc.
__device__ __forceinline__ bool better(double sa, uint32_t ia, double sb, uint32_t ib) {
    return sa != sb ? sa > sb : ia < ib;
}

// Orderable key of a double: ascending u64 order == ascending double order
// (no NaNs on this path).
__device__ __forceinline__ uint64_t order_key(double d) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(d));
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

}  // namespace fgb
