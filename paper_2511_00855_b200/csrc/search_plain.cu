// search_plain.cu — K5 for plain query batches (no entity context, no
// required keywords): best-first beam search (search.cpp:141-280) with
// CERTIFIED APPROXIMATE scoring and bit-identical results.
//
// Why.  The reference's hybrid score is a sequential fp64 sum (dense products
// in index order, then each sparse path's shared-term products in ascending
// order, scoring.cpp:10-99).  Reproducing those roundings needs one thread to
// walk the whole 4 KB row serially: an uncoalesced, latency-bound stream
// (tools/ubench_chain.cu: <= 2 elements/clk/SM from DRAM).  But a search only
// needs the ORDER of distances, plus the exact values of the k results.
//
// How.  Each first-time neighbour is scored by the whole warp with coalesced
// 16-byte loads: the same exact fp64 products (fp32 x fp32 is exact in fp64),
// summed in a different order (per-lane partial sums + a butterfly).  Both
// sums are within gamma_m * sum|p_i| of the exact real sum, and
// sum|p_i| <= |q_w| * |d| <= |q_w| * sqrt(max sqnorm) (Cauchy-Schwarz over the
// concatenated paths; sqnorm = the doc's unit-weight self score), so
//     |approx - reference| <= eps = (N + M + 8) u |q_w| max|d|
// (N, M = the two summation depths, u = 2^-53).  Every comparison the search
// makes (batch sort, pool rank, eviction) is CERTIFIED when the two distances
// differ by more than 2.5 eps; otherwise both entries are re-scored with the
// reference's exact chain (hybrid_score, device_common.cuh) and compared
// exactly (node id breaks ties, search.cpp:13-16).  So every decision equals
// the reference's, the pools hold the same nodes in the same order, the
// expansion sequence is identical, and the final top-k entries are re-scored
// exactly: ids, order, scores, `expanded` and `scored` are bit-identical.
//
// Plain-query semantics used (search.cpp:22-42, 171-181): distances never
// change after scoring, so a re-offer of a scored node is a no-op and the
// pools' contents do not depend on offer order — each expansion's first-time
// neighbours merge as one sorted batch; deleted nodes enter cand, never topk.
#include <cstdio>
#include <cstdlib>
#include <algorithm>

#include "approx_score.cuh"
#include "plain_common.cuh"
#include "query_stage.cuh"
#include "search_plain.hpp"

namespace fgb {
namespace {

using namespace pc;
using approx::q_lookup_t;
using approx::kSG;
using approx::dense_group;
using approx::sparse_group;
#ifndef FGB_PLAIN_MIN_WARPS
#define FGB_PLAIN_MIN_WARPS 12
#endif
constexpr int kMinWarps = FGB_PLAIN_MIN_WARPS;  // launch bound: query-warps per SM (register budget)
enum : uint32_t { QF_VALID = 1, QF_ENTITY = 2, QF_FALLBACK = 4 };

struct PlainMem {
    float* qd;
    unsigned char* path[2];  // per sparse path: bitmap (bm, pre, qv) or hash (keys, vals, filt)
    double* cand_d;
    uint32_t* cand_n;
    double* topk_d;
    uint32_t* topk_n;
    uint32_t* br;
};

__device__ __forceinline__ PlainMem carve(unsigned char* base, const PlainLaunch& a, uint64_t slot) {
    PlainMem m;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        unsigned char* p = base + off;
        off += al16(bytes);
        return p;
    };
    m.qd = reinterpret_cast<float*>(take(a.c.dstride * 4));
    const bool ck = a.mode == approx::kModeCuckoo;
    m.path[0] = take(path_bytes(a.vocab[0], a.cap[0], ck));
    m.path[1] = take(path_bytes(a.vocab[1], a.cap[1], ck));
    m.cand_d = a.gpool_d ? a.gpool_d + slot * a.beamcap : reinterpret_cast<double*>(take(a.beamcap * 8));
    m.topk_d = reinterpret_cast<double*>(take(a.kcap * 8));
    m.cand_n = a.gpool_n ? a.gpool_n + slot * a.beamcap : reinterpret_cast<uint32_t*>(take(a.beamcap * 4));
    m.topk_n = reinterpret_cast<uint32_t*>(take(a.kcap * 4));
    m.br = reinterpret_cast<uint32_t*>(take(32 * 4));
    return m;
}

template <int NQ4, bool kTime, int kMode>
#ifdef FGB_PLAIN_MAXNREG
__global__ void __maxnreg__(FGB_PLAIN_MAXNREG) search_plain_kernel(PlainLaunch a) {
#else
__global__ void __launch_bounds__(32, kMinWarps) search_plain_kernel(PlainLaunch a) {
#endif
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t slot = blockIdx.x;
    PlainMem w = carve(smem_raw, a, slot);
    uint32_t* visited = a.visited + slot * a.nwords;
    uint32_t* touched = a.touched + slot * a.tcap;
    const DevCorpus& c = a.c;
    unsigned long long ph[kTime ? kPlainPhQueries : 1] = {};
    long long tmark = kTime ? clock64() : 0;
    auto phase_end = [&](int k) {
        if constexpr (kTime) {
            const long long t = clock64();
            ph[k] += t - tmark;
            tmark = t;
        }
    };
    unsigned long long resolved = 0, final_exact = 0;
    if (kTime && lane == 0) atomicMin(&a.timing[kPlainPhStart], globaltimer());

#pragma unroll 1
    while (true) {
        uint32_t qi = 0;
        if (lane == 0) qi = atomicAdd(a.work, 1u);
        qi = __shfl_sync(kFull, qi, 0);
        if (qi >= a.q.count) break;
        const uint32_t flags = a.qflags[qi];
        if (!(flags & QF_VALID)) {
            if (lane == 0) {
                a.r_count[qi] = 0;
                a.r_expanded[qi] = 0;
                a.r_scored[qi] = 0;
                a.r_warn[qi] = 0;
                a.r_err[qi] = 0;
            }
            continue;
        }
        const uint32_t K = a.q.k[qi], B = a.q.beam[qi];
        // ---- stage the weighted query (build_query_vector, corpus.cpp:86-103)
        QueryQ Q;
        double qd2 = 0.0, qs2 = 0.0;
        {
            const float wd = a.q.weights[qi].x;
            const float* x = a.q.dense + qi * a.q.dim;
            for (uint32_t j = lane; j < c.dstride; j += 32) {
                const float v = j < a.q.dim ? __fmul_rn(wd, x[j]) : 0.0f;
                w.qd[j] = v;
                qd2 += (double)v * (double)v;
            }
            Q.qd = wd != 0.0f ? w.qd : nullptr;
            if (!Q.qd) qd2 = 0.0;
        }
        constexpr bool kCk = kMode == approx::kModeCuckoo;
        qs2 += stage_path(a.q, a.vocab, a.cap, qi, 0, w.path[0], Q.p[0], lane, kCk);
        qs2 += stage_path(a.q, a.vocab, a.cap, qi, 1, w.path[1], Q.p[1], lane, kCk);
        __syncwarp();
        if (kCk && (a.prefetch & 0x100) && (qi & 1) == 0) Q.p[0].hm1 = Q.p[1].hm1 = 0;  // test hook: forced failure
        if (kCk && ((Q.p[0].on && !Q.p[0].hm1) || (Q.p[1].on && !Q.p[1].hm1))) {
            if (lane == 0) {  // no cuckoo table: the host re-runs the batch with hash lookups
                a.r_count[qi] = 0;
                a.r_err[qi] = 4;
            }
            continue;
        }
        // |weighted dense query| (screening) and |weighted query| over all paths (error bound)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            qd2 += __shfl_xor_sync(kFull, qd2, o);
            qs2 += __shfl_xor_sync(kFull, qs2, o);
        }
        const double qnorm = sqrt_ub(qd2);
        // |approx - reference| <= eps: fp32 dense partials (gamma_4 in fp32 of
        // sum |q_i d_i| <= |q_d| max|d_dense|) + fp64 sums (depths N, M) of all
        // products (sum |p| <= |q_w| max|d|, Cauchy-Schwarz)
        const double eps = (a.eps32_coef * qnorm * a.max_dnorm + a.eps_coef * sqrt_ub(qd2 + qs2) * a.max_norm) *
                               a.eps_scale + 1e-300;
        const double tol = 2.5 * eps;

        const Pool topk{w.topk_d, w.topk_n, K};
        const Pool cand{w.cand_d, w.cand_n, B};
        uint32_t tsize = 0, csize = 0, ntouched = 0, cursor = 0;
        uint32_t seed_next = 0, adj_u = 0, adj_b = a.degree;
        unsigned long long expanded = 0, scored = 0;

#pragma unroll 1
        while (true) {
            // ---- the next lane-held batch: the entry_count largest-norm seeds
            // (search.cpp:205-216), then the neighbours of the first
            // unexpanded cand entry, 32 at a time (search.cpp:218-264)
            uint32_t node = 0;
            uint4 nm = make_uint4(0, 0, 0, 0);  // the node's gather record, loaded with its id
            bool v = false;
            if (seed_next < a.entry_count) {
                const uint32_t i = seed_next + lane;
                v = i < a.entry_count;
                if (v) {
                    node = a.norm_order[i];
                    nm = __ldg(a.norm_meta + i);
                }
                seed_next += 32;
            } else {
                if (adj_b >= a.degree) {
                    phase_end(kPlainPhSeeds);
                    int upos = -1;
                    for (uint32_t b = cursor; b < csize && upos < 0; b += 32) {
                        const uint32_t i = b + lane;
                        const uint32_t m = __ballot_sync(kFull, i < csize && !(w.cand_n[i] & kExp));
                        if (m) upos = static_cast<int>(b + __ffs(m) - 1);
                    }
                    phase_end(kPlainPhSelect);
                    if (upos < 0) break;
                    cursor = upos;
                    __syncwarp();
                    adj_u = w.cand_n[upos] & kId;
                    __syncwarp();
                    if (lane == 0) w.cand_n[upos] |= kExp;
                    __syncwarp();
                    ++expanded;
                    adj_b = 0;
                }
                const uint32_t j = adj_b + lane;
                v = j < a.degree;
                if (v) {
                    const uint64_t e = static_cast<uint64_t>(adj_u) * a.degree + j;
                    node = a.semantic[e];
                    nm = __ldg(a.edge_meta + e);
                }
                adj_b += 32;
            }
            // first-time test (a repeated neighbour loses the test-and-set to
            // its first copy, so no explicit dedupe is needed)
            bool fresh = false;
            if (v) {
                const uint32_t bit = 1u << (node & 31);
                fresh = (atomicOr(&visited[node >> 5], bit) & bit) == 0;
            }
            const uint32_t fm = __ballot_sync(kFull, fresh);
            phase_end(kPlainPhAdj);
            if (!fm) continue;

            // ---- score the F fresh nodes, compacted into lanes 0..F-1
            const uint32_t F = __popc(fm);
            const uint32_t src = __fns(fm, 0, lane + 1);
            const uint32_t sl = src < 32 ? src : 0;
            const uint32_t cn = __shfl_sync(kFull, node, sl);
            uint4 mt;  // one 16-B record: sparse offsets/lengths, dense norm
            mt.x = __shfl_sync(kFull, nm.x, sl);
            mt.y = __shfl_sync(kFull, nm.y, sl);
            mt.z = __shfl_sync(kFull, nm.z, sl);
            mt.w = __shfl_sync(kFull, nm.w, sl);
            const bool mine = lane < F;
            if (mine && ntouched + lane < a.tcap) touched[ntouched + lane] = cn;
            ntouched += F;
            scored += F;
            if (mine && Q.qd && (a.prefetch & 2))
                l2_prefetch(c.dense + static_cast<uint64_t>(cn) * c.dstride, c.dstride * 4);
            if (mine && (a.prefetch & 4)) {  // postings of the groups after the first
#pragma unroll
                for (int path = 0; path < 2; ++path) {
                    const uint32_t nz = path ? (mt.z >> 16) : (mt.z & 0xFFFFu);
                    if (Q.p[path].on && nz && lane >= kSG) {
                        const uint64_t o = 4ull * (path ? mt.y : mt.x);
                        l2_prefetch((path ? c.s_idx : c.l_idx) + o, ((nz + 3) & ~3u) * 4);
                        l2_prefetch((path ? c.s_val : c.l_val) + o, ((nz + 3) & ~3u) * 4);
                    }
                }
            }
            double L = 0.0, S = 0.0;
#pragma unroll 1
            for (int path = 0; path < 2; ++path) {
                const bool learned = path == 0;
                const PathQ P = learned ? Q.p[0] : Q.p[1];  // (a select, not a dynamic index)
                if (!P.on) continue;
                const uint32_t* pidx = learned ? c.l_idx : c.s_idx;
                const float* pval = learned ? c.l_val : c.s_val;
                const uint32_t off4 = learned ? mt.x : mt.y, pnnz = learned ? (mt.z & 0xFFFFu) : (mt.z >> 16);
                double r;
                if constexpr (kMode == approx::kModeCuckoo)
                    r = sparse_group<approx::kLookCuckoo>(pidx, pval, P, off4, pnnz, lane, F);
                else if constexpr (kMode == approx::kModeBitmap)
                    r = sparse_group<true>(pidx, pval, P, off4, pnnz, lane, F);
                else if constexpr (kMode == approx::kModeHash)
                    r = sparse_group<false>(pidx, pval, P, off4, pnnz, lane, F);
                else
                    r = P.vocab ? sparse_group<true>(pidx, pval, P, off4, pnnz, lane, F)
                                : sparse_group<false>(pidx, pval, P, off4, pnnz, lane, F);
                if (learned)
                    L = r;
                else
                    S = r;
            }
            phase_end(kPlainPhSparse);
            // screening against both full pools' worst entries (an offer
            // below both is a no-op); bounds widened by the error terms
            bool keep = mine;
            if (mine && csize == B && tsize == K) {
                const double floor = fmin(-w.cand_d[csize - 1], -w.topk_d[tsize - 1]) - 4.0 * eps;
                const double dn = Q.qd ? (double)__uint_as_float(mt.w) : 0.0;
                const double ub = score_upper_bound(Q.qd ? qnorm : 0.0, dn, L, S) + 2.0 * eps;
                keep = !(ub < floor);
            }
            const uint32_t km = __ballot_sync(kFull, keep);
            if (keep && Q.qd && (a.prefetch & 1))
                l2_prefetch(c.dense + static_cast<uint64_t>(cn) * c.dstride, c.dstride * 4);
            const double D = Q.qd ? dense_group<NQ4>(c, Q.qd, cn, lane, km) : 0.0;
            phase_end(kPlainPhDense);
            const uint32_t m = __popc(km);
            if (m == 0) continue;
            double d = keep ? -__dadd_rn(__dadd_rn(D, L), S) : dinf();
            uint32_t n = keep ? cn : kEmpty;

            // ---- certify: sort the batch, then every adjacent pair and every
            // new entry's neighbours at its rank in both pools must be
            // decided by the stored distances; otherwise re-score exactly
            uint32_t rank_t = 0, rank_c = 0, tm = 0;
            double td = dinf();
            uint32_t tn = kEmpty;
#pragma unroll 1
            while (true) {
                warp_sort(d, n, lane);
                const double dn2 = __shfl_down_sync(kFull, d, 1);
                const uint32_t nn2 = __shfl_down_sync(kFull, n, 1);
                const bool bad = lane < 31 && n != kEmpty && nn2 != kEmpty && !certain(d, n, dn2, nn2, tol);
                // (every shuffle runs on all 32 lanes: never inside a short-circuit)
                const bool prev_bad = __shfl_up_sync(kFull, bad, 1);
                bool fix = (bad || (prev_bad && lane > 0)) && n != kEmpty && !(n & kExact);
#ifdef FGB_DEBUG_PLAIN
                if (lane < m && n == kEmpty)
                    printf("BAD lane %u m %u F %u km %08x d %g L %g S %g D %g keep %d cn %u\n", lane, m, F, km, d, L, S, D,
                           (int)keep, cn);
                if (lane < m && (n & kId) >= c.n)
                    printf("BADID lane %u m %u F %u km %08x d %g n %08x keep %d cn %u\n", lane, m, F, km, d, n,
                           (int)keep, cn);
#endif
                // topk view: the non-deleted entries, in order (search.cpp:174)
                const bool ok = lane < m && !c.deleted[n & kId];
                const uint32_t om = __ballot_sync(kFull, ok);
                const uint32_t ts = __fns(om, 0, lane + 1);
                tm = __popc(om);
                td = __shfl_sync(kFull, d, ts < 32 ? ts : 0);
                tn = __shfl_sync(kFull, n, ts < 32 ? ts : 0);
                if (lane >= tm) {
                    td = dinf();
                    tn = kEmpty;
                }
                bool need_t = false, need_c = false;
                if (!__any_sync(kFull, fix)) {
                    if (lane < tm) {
                        rank_t = pool_rank(topk, tsize, td, tn & kId);
                        need_t = (rank_t > 0 && !certain(w.topk_d[rank_t - 1], w.topk_n[rank_t - 1], td, tn, tol)) ||
                                 (rank_t < tsize && !certain(td, tn, w.topk_d[rank_t], w.topk_n[rank_t], tol));
                    }
                    if (lane < m) {
                        rank_c = pool_rank(cand, csize, d, n & kId);
                        need_c = (rank_c > 0 && !certain(w.cand_d[rank_c - 1], w.cand_n[rank_c - 1], d, n, tol)) ||
                                 (rank_c < csize && !certain(d, n, w.cand_d[rank_c], w.cand_n[rank_c], tol));
                    }
                    // a topk view entry in doubt marks its batch lane
                    const uint32_t myview = __popc(om & ((1u << lane) - 1));
                    const bool view_doubt = __shfl_sync(kFull, need_t, myview & 31);
                    fix = need_c || (ok && view_doubt);
                    fix = fix && !(n & kExact);
                }
                const uint32_t ntm = __ballot_sync(kFull, need_t), ncm = __ballot_sync(kFull, need_c);
                const uint32_t fxm = __ballot_sync(kFull, fix);
                if (!fxm && !ntm && !ncm) break;
                if (fix) {
                    d = exact_dist<kMode>(c, Q, n & kId);
                    n |= kExact;
                }
                resolved += __popc(fxm);
                // pool entries around the doubtful ranks get exact distances too
#pragma unroll 1
                for (int pi = 0; pi < 2; ++pi) {
                    const Pool& P = pi ? cand : topk;
                    const uint32_t sz = pi ? csize : tsize;
                    uint32_t nm = pi ? ncm : ntm;
                    const uint32_t rk = pi ? rank_c : rank_t;
                    while (nm) {
                        const uint32_t j = __ffs(nm) - 1;
                        nm &= nm - 1;
                        const int i = static_cast<int>(__shfl_sync(kFull, rk, j)) - 4 + static_cast<int>(lane);
                        const bool pf = lane < 8 && i >= 0 && i < static_cast<int>(sz) && !(P.n[i] & kExact);
                        if (pf) {
                            P.d[i] = exact_dist<kMode>(c, Q, P.n[i] & kId);
                            P.n[i] |= kExact;
                        }
                        resolved += __popc(__ballot_sync(kFull, pf));
                        __syncwarp();
                    }
                }
            }
            pool_insert(topk, tsize, td, tn, tm, rank_t, lane, w.br);
            const uint32_t p0 = pool_insert(cand, csize, d, n, m, rank_c, lane, w.br);
            cursor = min(cursor, p0);
            phase_end(kPlainPhMerge);
        }

        // ---- results: the top-k with the reference's exact scores
        // (keyword_postfilter with no required keywords: topk as is, search.cpp:100-139)
        for (uint32_t i = lane; i < tsize; i += 32) {
            if (!(w.topk_n[i] & kExact)) {
                w.topk_d[i] = exact_dist<kMode>(c, Q, w.topk_n[i] & kId);
                ++final_exact;
            }
            a.r_node[static_cast<uint64_t>(qi) * a.hit_stride + i] = w.topk_n[i] & kId;
            a.r_score[static_cast<uint64_t>(qi) * a.hit_stride + i] = -w.topk_d[i];
        }
        if (lane == 0) {
            a.r_count[qi] = tsize;
            a.r_expanded[qi] = expanded;
            a.r_scored[qi] = scored;
            a.r_warn[qi] = (flags & QF_FALLBACK) ? 1u : 0u;
            a.r_err[qi] = 0;
        }
        // ---- reset the visited bits
        if (ntouched <= a.tcap) {
            for (uint32_t i = lane; i < ntouched; i += 32) visited[touched[i] >> 5] = 0;
        } else {
            for (uint64_t i = lane; i < a.nwords; i += 32) visited[i] = 0;
        }
        __syncwarp();
        phase_end(kPlainPhFinal);
        if (kTime && lane == 0) {
            for (int k = 0; k < kPlainPhQueries; ++k) {
                atomicAdd(&a.timing[k], ph[k]);
                ph[k] = 0;
            }
            atomicAdd(&a.timing[kPlainPhQueries], 1ull);
            atomicAdd(&a.timing[kPlainPhExpanded], expanded);
        }
    }
    if (kTime && lane == 0) {  // the tail: spread of the query-warps' finish times
        const unsigned long long t = globaltimer();
        atomicMin(&a.timing[kPlainPhEndMin], t);
        atomicMax(&a.timing[kPlainPhEndMax], t);
    }
    if (a.stats) {
        const unsigned long long fe = __reduce_add_sync(kFull, static_cast<unsigned>(final_exact));
        if (lane == 0) {
            atomicAdd(&a.stats[0], resolved);
            atomicAdd(&a.stats[1], fe);
        }
    }
}

// (the phase-timing variant exists in the mixed mode only)
template <int NQ4, int kMode>
void launch_m(const PlainLaunch& a, uint64_t blocks, size_t smem, cudaStream_t s) {
    if (a.timing) {
        FGB_CUDA(cudaFuncSetAttribute(search_plain_kernel<NQ4, true, approx::kModeMixed>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        search_plain_kernel<NQ4, true, approx::kModeMixed><<<(unsigned)blocks, 32, smem, s>>>(a);
    } else {
        FGB_CUDA(cudaFuncSetAttribute(search_plain_kernel<NQ4, false, kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        search_plain_kernel<NQ4, false, kMode><<<(unsigned)blocks, 32, smem, s>>>(a);
    }
    FGB_LAUNCH("search_plain_kernel");
}

template <int NQ4>
void launch_t(const PlainLaunch& a, uint64_t blocks, size_t smem, cudaStream_t s) {
    switch (a.mode) {
        case approx::kModeHash: launch_m<NQ4, approx::kModeHash>(a, blocks, smem, s); break;
        case approx::kModeCuckoo: launch_m<NQ4, approx::kModeCuckoo>(a, blocks, smem, s); break;
        default: launch_m<NQ4, approx::kModeMixed>(a, blocks, smem, s); break;
    }
}

int nq4_of(const PlainLaunch& a) {
    const uint32_t need = ((a.c.dstride >> 2) + 31) / 32;
    for (int v : {1, 2, 3, 4, 6, 8})
        if (static_cast<uint32_t>(v) >= need) return v;
    return 0;
}

template <int NQ4>
const void* kernel_ptr(int mode) {
    switch (mode) {
        case approx::kModeHash: return reinterpret_cast<const void*>(search_plain_kernel<NQ4, false, approx::kModeHash>);
        case approx::kModeCuckoo: return reinterpret_cast<const void*>(search_plain_kernel<NQ4, false, approx::kModeCuckoo>);
        default: return reinterpret_cast<const void*>(search_plain_kernel<NQ4, false, approx::kModeMixed>);
    }
}

const void* kernel_for(int v, int mode) {
    switch (v) {
        case 1: return kernel_ptr<1>(mode);
        case 2: return kernel_ptr<2>(mode);
        case 3: return kernel_ptr<3>(mode);
        case 4: return kernel_ptr<4>(mode);
        case 6: return kernel_ptr<6>(mode);
        case 8: return kernel_ptr<8>(mode);
        default: return nullptr;
    }
}

}  // namespace

size_t plain_warp_smem(const PlainLaunch& a) {
    if (nq4_of(a) == 0) return 0;  // dense rows wider than 1,024 floats: general kernel
    const bool ck = a.mode == approx::kModeCuckoo;
    const size_t b = al16(a.c.dstride * 4) + al16(path_bytes(a.vocab[0], a.cap[0], ck)) +
                     al16(path_bytes(a.vocab[1], a.cap[1], ck)) + (a.gpool_d ? 0 : al16(a.beamcap * 8)) + al16(a.kcap * 8) +
                     (a.gpool_n ? 0 : al16(a.beamcap * 4)) + al16(a.kcap * 4) + al16(32 * 4);
    return b <= 227 * 1024 ? b : 0;
}

uint64_t plain_slots(const PlainLaunch& a, uint64_t nq, int device) {
    const size_t smem = plain_warp_smem(a);
    const void* k = kernel_for(nq4_of(a), a.mode);
    FGB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0, sms = 0;
    FGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32, smem));
    FGB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    per_sm = std::max(per_sm, 1);
    if (const char* e = std::getenv("FGB_SEARCH_WARPS_PER_SM"))  // dev: occupancy sweeps
        per_sm = std::max(1, std::min(per_sm, std::atoi(e)));
    // (a balanced grid — the fewest warps finishing in the same number of
    // waves — measured 3% SLOWER at 10K queries: throughput tracks the
    // resident warps even while the last wave drains)
    return std::max<uint64_t>(1, std::min<uint64_t>(nq, static_cast<uint64_t>(sms) * per_sm));
}

void launch_search_plain(const PlainLaunch& a, uint64_t nq, int device, cudaStream_t s) {
    const size_t smem = plain_warp_smem(a);
    const uint64_t blocks = plain_slots(a, nq, device);
    switch (nq4_of(a)) {
        case 1: launch_t<1>(a, blocks, smem, s); break;
        case 2: launch_t<2>(a, blocks, smem, s); break;
        case 3: launch_t<3>(a, blocks, smem, s); break;
        case 4: launch_t<4>(a, blocks, smem, s); break;
        case 6: launch_t<6>(a, blocks, smem, s); break;
        case 8: launch_t<8>(a, blocks, smem, s); break;
        default: throw Error("internal", "plain search: unsupported dense width");
    }
}

}  // namespace fgb
