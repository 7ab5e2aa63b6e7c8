// stage_doc.cuh — stage a corpus row as the "query" side of pair scores
// (unit weights: pair_score, knn_graph.cpp:20-22).
#pragma once

#include "device_common.cuh"

namespace fgb {

__host__ __device__ inline size_t doc_stage_bytes(uint32_t dstride, uint32_t lcap, uint32_t scap) {
    return stage_bytes(dstride, lcap, scap);
}

template <typename Sync>
__device__ __forceinline__ void stage_doc(const DevCorpus& c, uint64_t u, unsigned char* smem,
                                          uint32_t lcap, uint32_t scap, uint32_t tid,
                                          uint32_t nthreads, SmemQuery& sq, Sync sync) {
    const StagePtrs p = stage_layout(smem, c.dstride, lcap, scap);
    const float* row = c.dense + u * c.dstride;
    for (uint32_t j = tid; j < c.dstride; j += nthreads) p.dense[j] = static_cast<double>(row[j]);
    for (uint32_t j = tid; j < lcap; j += nthreads) p.lkeys[j] = kEmpty;
    for (uint32_t j = tid; j < scap; j += nthreads) p.skeys[j] = kEmpty;
    for (uint32_t j = tid; j < filter_words(lcap); j += nthreads) p.lfilt[j] = 0;
    for (uint32_t j = tid; j < filter_words(scap); j += nthreads) p.sfilt[j] = 0;
    sync();
    const uint32_t ln = c.l_nnz[u], sn = c.s_nnz[u];
    const uint64_t lo = c.l_off[u], so = c.s_off[u];
    for (uint32_t j = tid; j < ln; j += nthreads) {
        const uint32_t t = c.l_idx[lo + j];
        hash_insert(p.lkeys, p.lvals, lcap - 1, t, c.l_val[lo + j]);
        atomicOr(&p.lfilt[(t >> 5) & (filter_words(lcap) - 1)], 1u << (t & 31));
    }
    for (uint32_t j = tid; j < sn; j += nthreads) {
        const uint32_t t = c.s_idx[so + j];
        hash_insert(p.skeys, p.svals, scap - 1, t, c.s_val[so + j]);
        atomicOr(&p.sfilt[(t >> 5) & (filter_words(scap) - 1)], 1u << (t & 31));
    }
    sync();
    sq.dense = p.dense;
    sq.lkeys = p.lkeys;
    sq.lvals = p.lvals;
    sq.lfilt = p.lfilt;
    sq.lmask = ln ? lcap - 1 : 0;
    sq.skeys = p.skeys;
    sq.svals = p.svals;
    sq.sfilt = p.sfilt;
    sq.smask = sn ? scap - 1 : 0;
}

}  // namespace fgb
