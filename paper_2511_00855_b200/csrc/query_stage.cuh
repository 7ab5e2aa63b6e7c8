// query_stage.cuh — stage one weighted query into shared memory.
//
// build_query_vector (corpus.cpp:86-103) is applied on the fly: dense
// entries become w_dense * x in fp32 (__fmul_rn, the reference's rounding,
// then widened exactly to fp64), a zero-weight path is dropped, and each
// sparse path becomes a bit filter + open-addressing hash (term -> w * value)
// that document rows probe.
#pragma once

#include "fg_cuda.hpp"

namespace fgb {

// Executed cooperatively by `nthreads` threads (tid in [0, nthreads));
// `sync` must synchronise exactly those threads.  smem must be 16-B aligned
// and hold stage_bytes(dstride, lcap, scap) bytes.
template <typename Sync>
__device__ __forceinline__ void stage_query(const DevQueries& q, uint64_t qi, uint32_t dstride,
                                            unsigned char* smem, uint32_t lcap, uint32_t scap,
                                            uint32_t tid, uint32_t nthreads, SmemQuery& sq,
                                            Sync sync) {
    const StagePtrs p = stage_layout(smem, dstride, lcap, scap);
    const float4 w = q.weights[qi];
    const float* x = q.dense + qi * q.dim;
    for (uint32_t j = tid; j < dstride; j += nthreads)
        p.dense[j] = j < q.dim ? static_cast<double>(__fmul_rn(w.x, x[j])) : 0.0;
    for (uint32_t j = tid; j < lcap; j += nthreads) p.lkeys[j] = kEmpty;
    for (uint32_t j = tid; j < scap; j += nthreads) p.skeys[j] = kEmpty;
    for (uint32_t j = tid; j < filter_words(lcap); j += nthreads) p.lfilt[j] = 0;
    for (uint32_t j = tid; j < filter_words(scap); j += nthreads) p.sfilt[j] = 0;
    sync();
    const uint64_t lb = q.l_ptr[qi], le = q.l_ptr[qi + 1];
    const uint64_t sb = q.s_ptr[qi], se = q.s_ptr[qi + 1];
    const bool use_l = w.y != 0.0f && le > lb;
    const bool use_s = w.z != 0.0f && se > sb;
    if (use_l)
        for (uint64_t j = lb + tid; j < le; j += nthreads) {
            const uint32_t t = q.l_idx[j];
            hash_insert(p.lkeys, p.lvals, lcap - 1, t, __fmul_rn(w.y, q.l_val[j]));
            atomicOr(&p.lfilt[(t >> 5) & (filter_words(lcap) - 1)], 1u << (t & 31));
        }
    if (use_s)
        for (uint64_t j = sb + tid; j < se; j += nthreads) {
            const uint32_t t = q.s_idx[j];
            hash_insert(p.skeys, p.svals, scap - 1, t, __fmul_rn(w.z, q.s_val[j]));
            atomicOr(&p.sfilt[(t >> 5) & (filter_words(scap) - 1)], 1u << (t & 31));
        }
    sync();
    sq.dense = w.x != 0.0f ? p.dense : nullptr;
    sq.lkeys = p.lkeys;
    sq.lvals = p.lvals;
    sq.lfilt = p.lfilt;
    sq.lmask = use_l ? lcap - 1 : 0;
    sq.skeys = p.skeys;
    sq.svals = p.svals;
    sq.sfilt = p.sfilt;
    sq.smask = use_s ? scap - 1 : 0;
}

}  // namespace fgb
