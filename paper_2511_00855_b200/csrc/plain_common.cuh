// plain_common.cuh — pieces shared by the certified-approximate search
// kernels (search_plain.cu: plain batches; search_hybrid.cu: entity-context
// and required-keyword batches): pool entries and their certified ordering,
// the exact distance chain, and the staged sparse query paths.
#pragma once

#include <cstdint>

#include "approx_score.cuh"
#include "fg_cuda.hpp"

namespace fgb {
namespace pc {

using approx::PathQ;
using approx::q_lookup;
constexpr uint32_t kExp = 0x80000000u;    // cand entry expanded
constexpr uint32_t kExact = 0x40000000u;  // stored distance is the reference's exact value
constexpr uint32_t kId = 0x3FFFFFFFu;
constexpr uint32_t kFull = 0xFFFFFFFFu;

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7FF0000000000000ll); }

// An upper bound of sqrt(x) (x >= 0) without the fp64 sqrt's out-of-line
// slow path: fp32 rounded up, MUFU sqrt, widened by 2^-18 (> its error).
__device__ __forceinline__ double sqrt_ub(double x) {
    const float f = __double2float_ru(x);
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(f));
    return static_cast<double>(r) * (1.0 + 0x1p-18) + 1e-300;
}
// (The search kernels avoid every out-of-line call — fp64 sqrt and division
// have one — because ptxas 12.9 for sm_100a clobbered live registers around
// such calls in these large kernels.)

__device__ __forceinline__ bool eless(double d1, uint32_t n1, double d2, uint32_t n2) {
    return d1 < d2 || (d1 == d2 && n1 < n2);  // entry_less (search.cpp:13-16)
}

// The two stored distances decide their order exactly.
__device__ __forceinline__ bool certain(double da, uint32_t na, double db, uint32_t nb, double tol) {
    return ((na & nb & kExact) != 0) || fabs(da - db) > tol;
}

struct QueryQ {
    const float* qd;  // weighted dense query (fp32, zero padded to dstride); nullptr: path off
    PathQ p[2];       // learned, statistical
};

// The reference's exact distance — the sequential chains of
// scoring.cpp:10-99 (dense in index order, then each sparse path's shared
// terms in ascending order; products of fp32 values exact in fp64, so one
// FMA per term rounds exactly like the reference's `acc += a * b`).  The rare
// path (uncertain comparisons, top-k entries).  Rows stream as 16-byte loads
// kept 8 (dense) / 2 groups (sparse) ahead of the chain; the zero padding of
// dense rows and the (kPad, 0) padding of posting groups add nothing.
// (Kept inline: an out-of-line call here corrupted live batch registers
// under sm_100a ptxas 12.9 — tools/smoke_plain.py reproduced it.)
template <int kMode = approx::kModeMixed>
__device__ __forceinline__ double exact_dist(const DevCorpus& c, const QueryQ& Q, uint32_t node) {
    double acc = 0.0;
    if (Q.qd) {
        constexpr uint32_t S = 8;
        const float4* row = reinterpret_cast<const float4*>(c.dense + static_cast<uint64_t>(node) * c.dstride);
        const float4* q4 = reinterpret_cast<const float4*>(Q.qd);
        const uint32_t n4 = c.dstride >> 2;
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        float4 cur[S];
#pragma unroll
        for (uint32_t j = 0; j < S; ++j) cur[j] = j < n4 ? __ldg(row + j) : z;
#pragma unroll 1
        for (uint32_t i = 0; i < n4; i += S) {
            float4 nxt[S];
#pragma unroll
            for (uint32_t j = 0; j < S; ++j) nxt[j] = i + S + j < n4 ? __ldg(row + i + S + j) : z;
#pragma unroll
            for (uint32_t j = 0; j < S; ++j) {
                if (i + j < n4) {
                    const float4 q = q4[i + j];
                    acc = __fma_rn((double)q.x, (double)cur[j].x, acc);
                    acc = __fma_rn((double)q.y, (double)cur[j].y, acc);
                    acc = __fma_rn((double)q.z, (double)cur[j].z, acc);
                    acc = __fma_rn((double)q.w, (double)cur[j].w, acc);
                }
            }
#pragma unroll
            for (uint32_t j = 0; j < S; ++j) cur[j] = nxt[j];
        }
    }
#pragma unroll 1
    for (int path = 0; path < 2; ++path) {
        double s = 0.0;
        const bool learned = path == 0;
        const PathQ P = learned ? Q.p[0] : Q.p[1];
        if (P.on) {
            const uint64_t off = learned ? c.l_off[node] : c.s_off[node];
            const uint32_t n4 = ((learned ? c.l_nnz[node] : c.s_nnz[node]) + 3) >> 2;
            const uint4* i4 = reinterpret_cast<const uint4*>((learned ? c.l_idx : c.s_idx) + off);
            const float4* v4 = reinterpret_cast<const float4*>((learned ? c.l_val : c.s_val) + off);
            const uint4 pi = make_uint4(kPad, kPad, kPad, kPad);
            const float4 pv = make_float4(0.f, 0.f, 0.f, 0.f);
            uint4 ci[2];
            float4 cv[2];
#pragma unroll
            for (uint32_t j = 0; j < 2; ++j) {
                ci[j] = j < n4 ? __ldg(i4 + j) : pi;
                cv[j] = j < n4 ? __ldg(v4 + j) : pv;
            }
#pragma unroll 1
            for (uint32_t g = 0; g < n4; g += 2) {
                uint4 ni[2];
                float4 nv[2];
#pragma unroll
                for (uint32_t j = 0; j < 2; ++j) {
                    ni[j] = g + 2 + j < n4 ? __ldg(i4 + g + 2 + j) : pi;
                    nv[j] = g + 2 + j < n4 ? __ldg(v4 + g + 2 + j) : pv;
                }
#pragma unroll
                for (uint32_t j = 0; j < 2; ++j) {
                    const uint32_t t[4] = {ci[j].x, ci[j].y, ci[j].z, ci[j].w};
                    const float v[4] = {cv[j].x, cv[j].y, cv[j].z, cv[j].w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        bool f;
                        const float q = approx::q_lookup_m<kMode>(P, t[e], f);
                        if (f) s = __fma_rn((double)q, (double)v[e], s);
                    }
                }
#pragma unroll
                for (uint32_t j = 0; j < 2; ++j) {
                    ci[j] = ni[j];
                    cv[j] = nv[j];
                }
            }
        }
        acc = __dadd_rn(acc, s);
    }
    return -acc;
}

// ------------------------------------------------------------ pools
struct Pool {
    double* d;
    uint32_t* n;  // node | kExact (| kExp for cand)
    uint32_t cap;
};

// # entries strictly before (d, node) by the stored keys.
__device__ __forceinline__ uint32_t pool_rank(const Pool& p, uint32_t size, double d, uint32_t node) {
    uint32_t lo = 0, hi = size;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (eless(p.d[mid], p.n[mid] & kId, d, node))
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// Bitonic sort of one (d, n) per lane by (d, node); invalid lanes carry
// (+inf, kEmpty) and sort last.
__device__ __forceinline__ void warp_sort(double& d, uint32_t& n, uint32_t lane) {
#pragma unroll
    for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            const double od = __shfl_xor_sync(kFull, d, j);
            const uint32_t on = __shfl_xor_sync(kFull, n, j);
            const bool up = (lane & k) == 0;
            const bool lower = (lane & j) == 0;
            const bool other_less = eless(od, on & kId, d, n & kId);
            const bool take = (lower == up) ? other_less : (!other_less && (od != d || on != n));
            if (take) {
                d = od;
                n = on;
            }
        }
    }
}

// Inserts m <= 32 new entries (sorted, lanes < m, ranks certified exact and
// non-decreasing) into the pool: the set result of offering them one by one
// (Pool::offer, search.cpp:26-42).  Returns the smallest insertion position.
__device__ __forceinline__ uint32_t pool_insert(const Pool& p, uint32_t& size, double d, uint32_t n, uint32_t m,
                                                uint32_t rank, uint32_t lane, uint32_t* br) {
    const uint32_t mypos = lane < m ? lane + rank : p.cap;
    uint32_t p0 = mypos;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) p0 = min(p0, __shfl_xor_sync(kFull, p0, o));
    if (p0 >= p.cap) return p.cap;
    __syncwarp();
    if (lane < m) br[lane] = rank;
    __syncwarp();
    // pool entry i >= p0 moves right by #{j : rank_j <= i}; right to left,
    // each lane's count only shrinks (i decreases by 32 per step)
    int b = static_cast<int>(((size - 1) / 32) * 32);
    uint32_t sh = m;
    {
        const uint32_t i = b + lane;
        while (sh > 0 && br[sh - 1] > i) --sh;
    }
#pragma unroll 1
    for (; size > p0 && b >= static_cast<int>(p0 & ~31u); b -= 32) {
        const uint32_t i = b + lane;
        while (sh > 0 && br[sh - 1] > i) --sh;
        const bool v = i < size && i >= p0;
        double dd = 0;
        uint32_t nn = 0;
        if (v) {
            dd = p.d[i];
            nn = p.n[i];
        }
        __syncwarp();
        if (v && i + sh < p.cap) {
            p.d[i + sh] = dd;
            p.n[i + sh] = nn;
        }
        __syncwarp();
    }
    if (lane < m && mypos < p.cap) {
        p.d[mypos] = d;
        p.n[mypos] = n;  // new entries are unexpanded
    }
    __syncwarp();
    size = min(size + m, p.cap);
    return p0;
}

__host__ __device__ __forceinline__ size_t al16(size_t b) { return (b + 15) & ~size_t(15); }

// Bytes of one staged sparse path (PlainLaunch::vocab/cap; cuckoo: a
// two-choice table of cap slots, cap >= 4 x the query's terms, plus the
// term list it is built from).
__host__ __device__ __forceinline__ size_t path_bytes(uint32_t vocab, uint32_t cap, bool cuckoo = false) {
    if (cuckoo) return 2 * al16(cap * 4) + al16(cap * 2);
    if (vocab) {
        const size_t W = approx::bitmap_words(vocab);
        return al16(W * 4) + al16(W * 2) + al16(cap * 4);
    }
    return al16(cap * 4) + al16(cap * 4) + al16(filter_words(cap) * 4);
}

// Stages sparse path `path` of query qi (build_query_vector: fp32 w * v,
// a zero weight drops the path, corpus.cpp:86-103); returns sum of (w v)^2.
__device__ inline double stage_path(const DevQueries& q, const uint32_t* vocabs, const uint32_t* caps, uint64_t qi, int path,
                             unsigned char* mem, PathQ& P, uint32_t lane, bool cuckoo = false) {
    const uint64_t lb = path ? q.s_ptr[qi] : q.l_ptr[qi], le = path ? q.s_ptr[qi + 1] : q.l_ptr[qi + 1];
    const uint32_t* qidx = path ? q.s_idx : q.l_idx;
    const float* qval = path ? q.s_val : q.l_val;
    const float wt = path ? q.weights[qi].z : q.weights[qi].y;
    const uint32_t vocab = vocabs[path], cap = caps[path];
    P.on = wt != 0.0f && le > lb;
    P.vocab = vocab;
    double ss = 0.0;
    if (vocab) {
        const uint32_t W = approx::bitmap_words(vocab);
        P.wm1 = W - 1;
        uint32_t* bm = reinterpret_cast<uint32_t*>(mem);
        uint16_t* pre = reinterpret_cast<uint16_t*>(mem + al16(W * 4));
        float* qv = reinterpret_cast<float*>(mem + al16(W * 4) + al16(W * 2));
        P.bm = bm;
        P.pre = pre;
        P.qv = qv;
        if (!P.on) return 0.0;
        for (uint32_t i = lane; i < W; i += 32) bm[i] = 0;
        __syncwarp();
        for (uint64_t j = lb + lane; j < le; j += 32) {
            const uint32_t t = qidx[j];
            if (t < vocab) atomicOr(&bm[t >> 5], 1u << (t & 31));
        }
        __syncwarp();
        // exclusive prefix of the word popcounts over 32 contiguous chunks
        const uint32_t per = (W + 31) / 32, b0 = min(W, lane * per), b1 = min(W, b0 + per);
        uint32_t cnt = 0;
        for (uint32_t i = b0; i < b1; ++i) cnt += __popc(bm[i]);
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
        }
        uint32_t run = incl - cnt;
        for (uint32_t i = b0; i < b1; ++i) {
            pre[i] = static_cast<uint16_t>(run);
            run += __popc(bm[i]);
        }
        __syncwarp();
        for (uint64_t j = lb + lane; j < le; j += 32) {
            const uint32_t t = qidx[j];
            const float v = __fmul_rn(wt, qval[j]);
            ss += (double)v * (double)v;
            if (t < vocab) qv[pre[t >> 5] + __popc(bm[t >> 5] & ((1u << (t & 31)) - 1u))] = v;
        }
        __syncwarp();
        return ss;
    }
    if (cuckoo) {
        // two-choice cuckoo table: every lookup probes exactly two slots (no
        // data-dependent probe loop, so lanes of a warp never diverge on it)
        uint32_t* keys = reinterpret_cast<uint32_t*>(mem);
        float* vals = reinterpret_cast<float*>(mem + al16(cap * 4));
        uint32_t* tk = reinterpret_cast<uint32_t*>(mem + 2 * al16(cap * 4));
        float* tv = reinterpret_cast<float*>(tk + cap / 4);
        P.keys = keys;
        P.vals = vals;
        P.mask = cap - 1;
        P.hshift = 32u - static_cast<uint32_t>(__ffs(cap) - 1);
        P.hm1 = P.hm2 = 1u;
        if (!P.on) return 0.0;
        const uint32_t nt = static_cast<uint32_t>(le - lb);  // <= cap / 4 (host)
        for (uint64_t j = lb + lane; j < le; j += 32) {
            const float v = __fmul_rn(wt, qval[j]);
            ss += (double)v * (double)v;
            tk[j - lb] = qidx[j];
            tv[j - lb] = v;
        }
        approx::cuckoo_fill(P, keys, vals, tk, tv, nt, cap, lane);
        return ss;
    }
    uint32_t* keys = reinterpret_cast<uint32_t*>(mem);
    float* vals = reinterpret_cast<float*>(mem + al16(cap * 4));
    uint32_t* filt = reinterpret_cast<uint32_t*>(mem + 2 * al16(cap * 4));
    P.keys = keys;
    P.vals = vals;
    P.filt = filt;
    P.mask = cap - 1;
    if (!P.on) return 0.0;
    for (uint32_t j = lane; j < cap; j += 32) keys[j] = kEmpty;
    for (uint32_t j = lane; j < filter_words(cap); j += 32) filt[j] = 0;
    __syncwarp();
    for (uint64_t j = lb + lane; j < le; j += 32) {
        const uint32_t t = qidx[j];
        const float v = __fmul_rn(wt, qval[j]);
        ss += (double)v * (double)v;
        hash_insert(keys, vals, cap - 1, t, v);
        atomicOr(&filt[(t >> 5) & (filter_words(cap) - 1)], 1u << (t & 31));
    }
    __syncwarp();
    return ss;
}


}  // namespace pc
}  // namespace fgb
