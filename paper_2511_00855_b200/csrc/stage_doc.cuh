// stage_doc.cuh — stage a corpus row as the "query" side of pair scores
// (unit weights: pair_score, knn_graph.cpp:20-22).
#pragma once

#include "device_common.cuh"

namespace fgb {

__host__ __device__ inline size_t doc_stage_bytes(uint32_t dstride, uint32_t lcap, uint32_t scap) {
    return static_cast<size_t>(dstride) * 4 + static_cast<size_t>(lcap + scap) * 8;
}

template <typename Sync>
__device__ __forceinline__ void stage_doc(const DevCorpus& c, uint64_t u, unsigned char* smem,
                                          uint32_t lcap, uint32_t scap, uint32_t tid,
                                          uint32_t nthreads, SmemQuery& sq, Sync sync) {
    float* dense = reinterpret_cast<float*>(smem);
    uint32_t* lkeys = reinterpret_cast<uint32_t*>(dense + c.dstride);
    float* lvals = reinterpret_cast<float*>(lkeys + lcap);
    uint32_t* skeys = reinterpret_cast<uint32_t*>(lvals + lcap);
    float* svals = reinterpret_cast<float*>(skeys + scap);
    const float* row = c.dense + u * c.dstride;
    for (uint32_t j = tid; j < c.dstride; j += nthreads) dense[j] = row[j];
    for (uint32_t j = tid; j < lcap; j += nthreads) lkeys[j] = kEmpty;
    for (uint32_t j = tid; j < scap; j += nthreads) skeys[j] = kEmpty;
    sync();
    const uint32_t ln = c.l_nnz[u], sn = c.s_nnz[u];
    const uint64_t lo = c.l_off[u], so = c.s_off[u];
    for (uint32_t j = tid; j < ln; j += nthreads) hash_insert(lkeys, lvals, lcap - 1, c.l_idx[lo + j], c.l_val[lo + j]);
    for (uint32_t j = tid; j < sn; j += nthreads) hash_insert(skeys, svals, scap - 1, c.s_idx[so + j], c.s_val[so + j]);
    sync();
    sq.dense = dense;
    sq.lkeys = lkeys;
    sq.lvals = lvals;
    sq.lmask = ln ? lcap - 1 : 0;
    sq.skeys = skeys;
    sq.svals = svals;
    sq.smask = sn ? scap - 1 : 0;
}

}  // namespace fgb
