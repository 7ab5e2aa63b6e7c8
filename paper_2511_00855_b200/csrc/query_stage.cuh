// query_stage.cuh — stage one weighted query into shared memory.
//
// build_query_vector (corpus.cpp:86-103) is applied on the fly: dense
// entries become w_dense * x in fp32 (__fmul_rn, the reference's rounding),
// a zero-weight path is dropped, and each sparse path becomes an
// open-addressing hash (term -> w * value) that document rows probe.
#pragma once

#include "fg_cuda.hpp"

namespace fgb {

size_t stage_bytes(uint32_t dstride, uint32_t lcap, uint32_t scap);

// Executed cooperatively by `nthreads` threads (tid in [0, nthreads));
// `sync` must synchronise exactly those threads.  smem must be 16-B aligned
// and hold stage_bytes(dstride, lcap, scap) bytes.
template <typename Sync>
__device__ __forceinline__ void stage_query(const DevQueries& q, uint64_t qi, uint32_t dstride,
                                            unsigned char* smem, uint32_t lcap, uint32_t scap,
                                            uint32_t tid, uint32_t nthreads, SmemQuery& sq,
                                            Sync sync) {
    float* dense = reinterpret_cast<float*>(smem);
    uint32_t* lkeys = reinterpret_cast<uint32_t*>(dense + dstride);
    float* lvals = reinterpret_cast<float*>(lkeys + lcap);
    uint32_t* skeys = reinterpret_cast<uint32_t*>(lvals + lcap);
    float* svals = reinterpret_cast<float*>(skeys + scap);
    const float4 w = q.weights[qi];
    const float* x = q.dense + qi * q.dim;
    for (uint32_t j = tid; j < dstride; j += nthreads)
        dense[j] = j < q.dim ? __fmul_rn(w.x, x[j]) : 0.0f;
    for (uint32_t j = tid; j < lcap; j += nthreads) lkeys[j] = kEmpty;
    for (uint32_t j = tid; j < scap; j += nthreads) skeys[j] = kEmpty;
    sync();
    const uint64_t lb = q.l_ptr[qi], le = q.l_ptr[qi + 1];
    const uint64_t sb = q.s_ptr[qi], se = q.s_ptr[qi + 1];
    const bool use_l = w.y != 0.0f && le > lb;
    const bool use_s = w.z != 0.0f && se > sb;
    if (use_l)
        for (uint64_t j = lb + tid; j < le; j += nthreads)
            hash_insert(lkeys, lvals, lcap - 1, q.l_idx[j], __fmul_rn(w.y, q.l_val[j]));
    if (use_s)
        for (uint64_t j = sb + tid; j < se; j += nthreads)
            hash_insert(skeys, svals, scap - 1, q.s_idx[j], __fmul_rn(w.z, q.s_val[j]));
    sync();
    sq.dense = w.x != 0.0f ? dense : nullptr;
    sq.lkeys = lkeys;
    sq.lvals = lvals;
    sq.lmask = use_l ? lcap - 1 : 0;
    sq.skeys = skeys;
    sq.svals = svals;
    sq.smask = use_s ? scap - 1 : 0;
}

}  // namespace fgb
