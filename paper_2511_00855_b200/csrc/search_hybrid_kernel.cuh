#pragma once
// search_hybrid.cu — K5 for batches with entity context and/or required
// keywords: best-first beam search (search.cpp:141-280) with CERTIFIED
// APPROXIMATE scoring and bit-identical results, the plain kernel's design
// (search_plain.cu) extended by the reference's three order-sensitive
// features:
//
//  * Entity context (search.cpp:191-198, 239-261).  Each expansion of a node
//    u with context (ent, hop < max_hops) assigns every neighbour o the
//    smallest entity related to ent(u) (a KG relation to one of o's entities,
//    or a logical edge (via = o, target)) at hop(u) + 1 when that beats o's
//    current (hop, entity).  A node's adjusted distance raw - w_k / hop only
//    ever decreases (hop 0 is assigned to seeds only), so Pool::offer keeps
//    set semantics: each pool holds the best `capacity` nodes by their best
//    offered distance.  A neighbour is therefore offered when it is new or its
//    hop dropped (an unchanged re-offer is a no-op): new ones merge as one
//    certified batch exactly as in the plain kernel; an improved one is first
//    erased from the pools, then merges with the batch (its expanded flag
//    lives in a per-warp bitset).  Context updates of one batch are
//    independent per node (a neighbour list is node-unique after the
//    reach-order dedupe), so lanes apply them in parallel.
//  * Required keywords (search.cpp:163-181).  Keyword edges join the
//    neighbour list of nodes that share a required keyword, and top-k
//    evictions that share one enter the twin pool — which depends on the
//    offer ORDER.  The top-k pool is therefore kept EXACT: every offer that
//    can enter it (non-deleted, better than its current back + the error
//    margin) is re-scored with the reference's chain first; then, for keyword
//    queries, those offers replay Pool::offer one by one in reach order
//    (evictions feeding the twin pool), and otherwise merge as a batch.
//  * keyword_postfilter (search.cpp:100-139) over the exact top-k and the
//    twin pool (twin nodes re-scored exactly at the end with their final
//    context, as the reference's `adjusted(node)`).
//
// The cand pool stays approximate + certified (search_plain.cu header): every
// comparison decided by stored distances more than 2.5 eps apart, otherwise
// both sides re-scored exactly.  With rewards the error bound gains the
// rounding of the one subtraction: |RN(a - r) - RN(b - r)| <= |a - b| +
// u (|a - r| + |b - r|) <= |a - b| + 2u (|q_w| max|d| + w_k).
#include <algorithm>
#include <cstdlib>

#include "approx_score.cuh"
#include "plain_common.cuh"
#include "search_hybrid.hpp"

namespace fgb {
namespace {

using namespace pc;
using approx::dense_group;
using approx::kSG;
using approx::sparse_group;
constexpr int kMinWarps = 10;  // launch bound: query-warps per SM (register budget)
constexpr uint32_t kXq = 64;   // exact re-score requests per certification round
constexpr uint32_t kStage = 64;  // staged offers (< 32 carried + one window of 32)
enum : uint32_t { QF_VALID = 1, QF_ENTITY = 2, QF_FALLBACK = 4 };

struct HybridMem {
    float* qd;
    unsigned char* path[2];
    double* cand_d;
    uint32_t* cand_n;
    double* topk_d;
    uint32_t* topk_n;
    uint32_t* br;
    uint32_t* req;
    uint32_t* lc;    // (via, target) pairs of the expanded node's logical group
    uint32_t* seen;  // reach-order dedupe of one expansion's neighbour list
    uint32_t* xn;    // exact re-score requests: node
    uint32_t* xi;    //   cand position (pool entries)
    double* xd;      //   result
    unsigned long long* ph;  // phase timing slots
    // offers staged across the windows of one neighbour list (reach order):
    // windows with few new nodes (keyword / logical tails) share a batch
    uint4* st_meta;
    uint32_t* st_node;
    uint32_t* st_fl;  // assigned hop | improved << 31
};

__device__ __forceinline__ HybridMem carve(unsigned char* base, const HybridLaunch& h) {
    const PlainLaunch& a = h.p;
    HybridMem m;
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
    m.cand_d = reinterpret_cast<double*>(take(a.beamcap * 8));
    m.topk_d = reinterpret_cast<double*>(take(a.kcap * 8));
    m.cand_n = reinterpret_cast<uint32_t*>(take(a.beamcap * 4));
    m.topk_n = reinterpret_cast<uint32_t*>(take(a.kcap * 4));
    m.br = reinterpret_cast<uint32_t*>(take(32 * 4));
    m.req = reinterpret_cast<uint32_t*>(take(h.reqcap * 4 + 4));
    m.lc = reinterpret_cast<uint32_t*>(take(h.lccap * 8 + 8));
    m.seen = reinterpret_cast<uint32_t*>(take(h.seencap * 4));
    m.xd = reinterpret_cast<double*>(take(kXq * 8));
    m.xn = reinterpret_cast<uint32_t*>(take(kXq * 4));
    m.xi = reinterpret_cast<uint32_t*>(take(kXq * 4));
    m.ph = reinterpret_cast<unsigned long long*>(take(kHybCount * 8));
    m.st_meta = reinterpret_cast<uint4*>(take(kStage * 16));
    m.st_node = reinterpret_cast<uint32_t*>(take(kStage * 4));
    m.st_fl = reinterpret_cast<uint32_t*>(take(kStage * 4));
    return m;
}

size_t carve_bytes(const HybridLaunch& h) {
    const PlainLaunch& a = h.p;
    const bool ck = a.mode == approx::kModeCuckoo;
    return al16(a.c.dstride * 4) + al16(path_bytes(a.vocab[0], a.cap[0], ck)) + al16(path_bytes(a.vocab[1], a.cap[1], ck)) +
           al16(a.beamcap * 8) + al16(a.kcap * 8) + al16(a.beamcap * 4) + al16(a.kcap * 4) + al16(32 * 4) +
           al16(h.reqcap * 4 + 4) + al16(h.lccap * 8 + 8) + al16(h.seencap * 4) + al16(kXq * 8) + 2 * al16(kXq * 4) +
           al16(kHybCount * 8) + al16(kStage * 16) + 2 * al16(kStage * 4);
}

// ---------------------------------------------------------------- helpers
// shares_required (search.cpp:163-167): the node's keywords hold ANY required term.
__device__ __forceinline__ bool shares_required(const DevCorpus& c, uint32_t node, const uint32_t* req, uint32_t R,
                                                uint32_t lane) {
    bool hit = false;
    const uint64_t b = c.kw_ptr[node], e = c.kw_ptr[node + 1];
    for (uint32_t i = lane; i < R; i += 32) hit |= sorted_contains(c.kw_idx, b, e, req[i]);
    return __any_sync(kFull, hit);
}

// KnowledgeGraph::has_relation (types.cpp:52-57) on the device adjacency.
__device__ __forceinline__ bool has_rel(const HybridLaunch& h, uint32_t x, uint32_t y) {
    if (x >= h.kg_rows) return false;
    return sorted_contains(h.kg_nbr, h.kg_ptr[x], h.kg_ptr[x + 1], y);
}

// Entity-context table (per warp, HBM): open addressing on the node id,
// entries (node, entity, hop, has).  Probes are bounded by the capacity; the
// kernel raises HERR_CTX once half the slots are used and the host re-runs
// the query with a 4x table.
__device__ __forceinline__ uint4 ctx_get(const uint4* t, uint32_t cap, uint32_t node) {
    uint32_t s = hslot(node, cap - 1);
    for (uint32_t probe = 0; probe < cap; ++probe) {
        const uint4 e = t[s];
        if (e.x == node) return e;
        if (e.x == kEmpty) break;
        s = (s + 1) & (cap - 1);
    }
    return make_uint4(kEmpty, 0, 0, 0);
}
__device__ __forceinline__ int ctx_claim(uint4* t, uint32_t cap, uint32_t node, bool& claimed) {
    uint32_t s = hslot(node, cap - 1);
    claimed = false;
    for (uint32_t probe = 0; probe < cap; ++probe) {
        const uint32_t prev = atomicCAS(reinterpret_cast<uint32_t*>(t + s), kEmpty, node);
        if (prev == kEmpty) {
            claimed = true;
            return static_cast<int>(s);
        }
        if (prev == node) return static_cast<int>(s);
        s = (s + 1) & (cap - 1);
    }
    return -1;
}

// The reference's exact adjusted distance (search.cpp:156-161, 183-187):
// RN(raw - w_k / hop) for a node with context at hop >= 1, raw otherwise.
// `rew` = the query's row of host-computed rewards w_k / hop (hop 1.. in
// order): the kernel has no fp64 division — its slow path is an out-of-line
// CALL, and with calls in this kernel ptxas 12.9 (sm_100a) clobbered live
// registers (pool sizes and batch nodes, caught by the acceptance suite's
// criterion 5).
template <int kMode>
__device__ __forceinline__ double exact_adj(const DevCorpus& c, const QueryQ& Q, uint32_t node, const uint4* ctx,
                                            uint32_t ctxcap, const double* rew) {
    double d = exact_dist<kMode>(c, Q, node);
    if (ctx) {
        const uint4 e = ctx_get(ctx, ctxcap, node);
        if (e.x == node && e.w && e.z >= 1) d = __dsub_rn(d, rew[e.z - 1]);
    }
    return d;
}

// Per-expansion dedupe set in smem (keys pre-set to kEmpty).
__device__ __forceinline__ bool seen_has(const uint32_t* t, uint32_t cap, uint32_t x) {
    uint32_t s = hslot(x, cap - 1);
    for (uint32_t probe = 0; probe < cap; ++probe) {
        const uint32_t k = t[s];
        if (k == x) return true;
        if (k == kEmpty) return false;
        s = (s + 1) & (cap - 1);
    }
    return false;
}
__device__ __forceinline__ void seen_add(uint32_t* t, uint32_t cap, uint32_t x) {
    uint32_t s = hslot(x, cap - 1);
    for (uint32_t probe = 0; probe < cap; ++probe) {
        const uint32_t prev = atomicCAS(&t[s], kEmpty, x);
        if (prev == kEmpty || prev == x) return;
        s = (s + 1) & (cap - 1);
    }
}

// Removes the batch's improved nodes (lanes in `im`, node ids in bn) from a
// sorted pool, keeping the order; returns the new size.
__device__ __forceinline__ uint32_t pool_erase(double* pd, uint32_t* pn, uint32_t size, uint32_t im, uint32_t bn,
                                               uint32_t lane) {
    uint32_t wpos = 0;
#pragma unroll 1
    for (uint32_t b = 0; b < size; b += 32) {
        const uint32_t i = b + lane;
        const bool valid = i < size;
        double dd = 0.0;
        uint32_t nn = kEmpty;
        if (valid) {
            dd = pd[i];
            nn = pn[i];
        }
        bool drop = false;
        uint32_t mm = im;
        while (mm) {
            const uint32_t j = __ffs(mm) - 1;
            mm &= mm - 1;
            const uint32_t x = __shfl_sync(kFull, bn, j) & kId;  // (every lane shuffles: never inside &&)
            drop |= valid && (nn & kId) == x;
        }
        const bool keep = valid && !drop;
        const uint32_t km = __ballot_sync(kFull, keep);
        __syncwarp();
        if (keep) {
            const uint32_t p = wpos + __popc(km & ((1u << lane) - 1u));
            pd[p] = dd;
            pn[p] = nn;
        }
        wpos += __popc(km);
        __syncwarp();
    }
    return wpos;
}

template <int NQ4, int kMode, bool kCtx, bool kReq>
__global__ void __launch_bounds__(32, kMinWarps) search_hybrid_kernel(HybridLaunch h) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const PlainLaunch& a = h.p;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const uint64_t slot = blockIdx.x;
    HybridMem w = carve(smem_raw, h);
    uint32_t* visited = a.visited + slot * a.nwords;
    uint32_t* touched = a.touched + slot * a.tcap;
    uint32_t* expbits = h.expbits ? h.expbits + slot * a.nwords : nullptr;
    uint32_t* twinbits = h.twinbits ? h.twinbits + slot * a.nwords : nullptr;
    uint32_t* twin_node = h.twin_node ? h.twin_node + slot * h.twcap : nullptr;
    double* twin_d = h.twin_d ? h.twin_d + slot * h.twcap : nullptr;
    uint4* ctx = h.ctx ? h.ctx + slot * h.ctxcap : nullptr;
    const DevCorpus& c = a.c;
    unsigned long long resolved = 0, final_exact = 0;
    // optional phase timing: lane 0 accumulates into the warp's smem slots
    const bool T = h.timing != nullptr;
    unsigned long long* ph = w.ph;
    if (T && lane == 0)
        for (int k = 0; k < kHybCount; ++k) ph[k] = 0;
    long long tmark = T ? clock64() : 0;
    auto mark = [&](int k) {
        if (T) {
            const long long t = clock64();
            if (lane == 0) ph[k] += t - tmark;
            tmark = t;
        }
    };

#pragma unroll 1
    while (true) {
        uint32_t qi = 0;
        if (lane == 0) qi = atomicAdd(a.work, 1u);
        qi = __shfl_sync(kFull, qi, 0);
        if (h.qlist) {
            if (qi >= h.qlist_n) break;
            qi = h.qlist[qi];
        } else if (qi >= a.q.count) {
            break;
        }
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
        const uint32_t K = a.q.k[qi], B = a.q.beam[qi], H = a.q.hops[qi];
        const bool ctx_mode = kCtx && (flags & QF_ENTITY) != 0 && ctx != nullptr;
        const uint4* ctxq = ctx_mode ? ctx : nullptr;
        const double went = static_cast<double>(a.q.weights[qi].w);
        const double* rtab = ctx_mode ? h.rewards + static_cast<uint64_t>(qi) * h.rstride : nullptr;

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
        const uint64_t rb = kReq ? a.q.req_ptr[qi] : 0;
        const uint32_t R = kReq ? static_cast<uint32_t>(a.q.req_ptr[qi + 1] - rb) : 0u;
        for (uint32_t i = lane; i < R; i += 32) w.req[i] = a.q.req_idx[rb + i];
        __syncwarp();
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            qd2 += __shfl_xor_sync(kFull, qd2, o);
            qs2 += __shfl_xor_sync(kFull, qs2, o);
        }
        const double qnorm = sqrt_ub(qd2);
        const double qall = sqrt_ub(qd2 + qs2);
        double eps = (a.eps32_coef * qnorm * a.max_dnorm + a.eps_coef * qall * a.max_norm) *
                         a.eps_scale + 1e-300;
        if (ctx_mode) eps += (qall * a.max_norm + went) * 0x1p-51 * a.eps_scale;  // the reward subtraction
        const double tol = 2.5 * eps;

        const Pool topk{w.topk_d, w.topk_n, K};
        const Pool cand{w.cand_d, w.cand_n, B};
        uint32_t tsize = 0, csize = 0, ntouched = 0, cursor = 0, ntwin = 0, err = 0, ctx_used = 0;
        if (kCk && (a.prefetch & 0x100) && (qi & 1) == 0) Q.p[0].hm1 = Q.p[1].hm1 = 0;  // test hook: forced failure
        // no cuckoo table for a path (practically never at <= 1/4 load): the
        // host re-runs the query with the fallback lookups
        if (kCk && ((Q.p[0].on && !Q.p[0].hm1) || (Q.p[1].on && !Q.p[1].hm1))) err = HERR_CUCKOO;
        unsigned long long expanded = 0, scored = 0;
        // batch generator state: seeds (search.cpp:205-216), then expansions
        const uint64_t sb = ctx_mode ? h.seed_ptr[qi] : 0;
        const uint32_t nseeds = ctx_mode ? static_cast<uint32_t>(h.seed_ptr[qi + 1] - sb) : a.entry_count;
        uint32_t seed_next = 0, adj_u = 0, adj_b = 0, L = 0, nkw = 0, nlc = 0, uent = 0, uhop = 0;
        uint64_t kwb = 0;
        bool propagate = false, multi = false;

        uint32_t nst = 0;  // offers staged (w.st_*), in reach order
#pragma unroll 1
        while (err == 0) {
            mark(kHybTopk);  // (the previous batch's top-k step)
            // leftovers of a finished list are scored before the next selection
            const bool drain = nst > 0 && seed_next >= nseeds && adj_b >= L;
            if (!drain) {
            uint32_t node = 0, sent = 0;
            uint4 nm = make_uint4(0, 0, 0, 0);
            bool v = false, is_seed = false;
            if (seed_next < nseeds) {
                is_seed = true;
                const uint32_t i = seed_next + lane;
                v = i < nseeds;
                if (v) {
                    if (ctx_mode) {
                        node = h.seed_node[sb + i];
                        sent = h.seed_ent[sb + i];
                        nm = __ldg(c.meta + node);
                    } else {
                        node = a.norm_order[i];
                        nm = __ldg(a.norm_meta + i);
                    }
                }
                seed_next += 32;
            } else {
                if (adj_b >= L) {
                    // first unexpanded cand entry (search.cpp:219-226)
                    int upos = -1;
                    for (uint32_t b = cursor; b < csize && upos < 0; b += 32) {
                        const uint32_t i = b + lane;
                        const uint32_t m = __ballot_sync(kFull, i < csize && !(w.cand_n[i] & kExp));
                        if (m) upos = static_cast<int>(b + __ffs(m) - 1);
                    }
                    if (upos < 0) break;
                    if (T && lane == 0) ++ph[kHybExpanded];
                    cursor = upos;
                    __syncwarp();
                    adj_u = w.cand_n[upos] & kId;
                    __syncwarp();
                    if (lane == 0) {
                        w.cand_n[upos] |= kExp;
                        if (expbits) atomicOr(&expbits[adj_u >> 5], 1u << (adj_u & 31));
                    }
                    __syncwarp();
                    ++expanded;
                    // neighbour list in reach order (search.cpp:228-245): semantic,
                    // keyword edges if u shares a required keyword, logical vias
                    // of group ent(u) while hop(u) < max hops
                    propagate = false;
                    if (ctx_mode) {
                        const uint4 e = ctx_get(ctx, h.ctxcap, adj_u);
                        if (e.x == adj_u && e.w && e.z < H) {
                            propagate = true;
                            uent = e.y;
                            uhop = e.z;
                        }
                    }
                    nkw = 0;
                    if (R > 0 && shares_required(c, adj_u, w.req, R, lane)) {
                        kwb = h.kw_ptr[adj_u];
                        nkw = static_cast<uint32_t>(h.kw_ptr[adj_u + 1] - kwb);
                    }
                    nlc = 0;
                    if (propagate) {
                        const uint64_t lb = h.lg_ptr[adj_u], le = h.lg_ptr[adj_u + 1];
                        for (uint64_t j = lb; j < le; j += 32) {
                            const uint64_t e = j + lane;
                            uint4 ed = make_uint4(0, 0, 0, 0);
                            bool hit = false;
                            if (e < le) {
                                ed = h.lg[e];
                                hit = ed.x == uent;
                            }
                            const uint32_t m = __ballot_sync(kFull, hit);
                            const uint32_t pos = nlc + __popc(m & lt);
                            if (hit && pos < h.lccap) {
                                w.lc[2 * pos] = ed.w;
                                w.lc[2 * pos + 1] = ed.z;
                            }
                            nlc += __popc(m);
                        }
                        nlc = min(nlc, h.lccap);
                        __syncwarp();
                    }
                    L = a.degree + nkw + nlc;
                    multi = L > 32;
                    if (multi) {
                        for (uint32_t i = lane; i < h.seencap; i += 32) w.seen[i] = kEmpty;
                        __syncwarp();
                    }
                    adj_b = 0;
                    mark(kHybSelect);
                }
                const uint32_t j = adj_b + lane;
                v = j < L;
                if (v) {
                    if (j < a.degree) {
                        const uint64_t e = static_cast<uint64_t>(adj_u) * a.degree + j;
                        node = a.semantic[e];
                        nm = __ldg(a.edge_meta + e);
                    } else if (j < a.degree + nkw) {
                        node = h.kw_idx[kwb + (j - a.degree)];
                        nm = __ldg(c.meta + node);
                    } else {
                        node = w.lc[2 * (j - a.degree - nkw)];
                        nm = __ldg(c.meta + node);
                    }
                }
                // reach-order dedupe (search.cpp:229-232): the first copy wins
                const uint32_t vm = __ballot_sync(kFull, v);
                const uint32_t peers = __match_any_sync(kFull, v ? node : kEmpty);
                bool keep = v && (peers & vm & lt) == 0;
                if (multi) {
                    const bool dup = keep && adj_b > 0 && seen_has(w.seen, h.seencap, node);
                    __syncwarp();
                    keep = keep && !dup;
                    if (keep) seen_add(w.seen, h.seencap, node);
                    __syncwarp();
                }
                v = keep;
                adj_b += 32;
            }
            if (T && lane == 0) ++ph[kHybBatches];
            mark(kHybList);
            bool fresh = false;
            if (v) {
                const uint32_t bit = 1u << (node & 31);
                fresh = (atomicOr(&visited[node >> 5], bit) & bit) == 0;
            }
            // ---- entity context (assign_ctx, search.cpp:191-198, 248-260)
            uint32_t ahop = 0;  // hop assigned by this batch (0: none, no reward)
            bool improved = false;
            if (ctx_mode) {
                bool claimed = false;
                if (is_seed) {
                    if (v) {
                        const int s = ctx_claim(ctx, h.ctxcap, node, claimed);
                        if (s >= 0) ctx[s] = make_uint4(node, sent, 0, 1);
                    }
                } else if (propagate && v) {
                    const uint32_t hop = uhop + 1;
                    uint32_t ce = kEmpty;
                    const uint64_t eb = c.ent_ptr[node], ee = c.ent_ptr[node + 1];
                    for (uint64_t e = eb; e < ee; ++e) {  // smallest related entity of o
                        const uint32_t ent = c.ent_idx[e];
                        if (has_rel(h, uent, ent)) {
                            ce = ent;
                            break;
                        }
                    }
                    for (uint32_t j = 0; j < nlc; ++j)
                        if (w.lc[2 * j] == node) ce = min(ce, w.lc[2 * j + 1]);
                    if (ce != kEmpty) {
                        const int s = ctx_claim(ctx, h.ctxcap, node, claimed);
                        if (s >= 0) {
                            const uint4 cur = claimed ? make_uint4(node, 0, 0, 0) : ctx[s];
                            if (!cur.w || hop < cur.z || (hop == cur.z && ce < cur.y)) {
                                improved = !fresh && (!cur.w || hop < cur.z);
                                ctx[s] = make_uint4(node, ce, hop, 1u);
                                ahop = hop;
                            }
                        }
                    }
                }
                ctx_used += __popc(__ballot_sync(kFull, claimed));
                if (ctx_used * 2 > h.ctxcap) err |= HERR_CTX;
            }
            const uint32_t frm = __ballot_sync(kFull, fresh);
            {
                const uint32_t pos = ntouched + __popc(frm & lt);
                if (fresh && pos < a.tcap) touched[pos] = node;
                ntouched += __popc(frm);
                scored += __popc(frm);
            }
            const uint32_t fm = __ballot_sync(kFull, fresh || improved);
            if (fresh || improved) {  // stage the offers in reach order
                const uint32_t pos = nst + __popc(fm & lt);
                w.st_node[pos] = node;
                w.st_meta[pos] = nm;
                w.st_fl[pos] = ahop | (improved ? 0x80000000u : 0u);
            }
            nst += __popc(fm);
            __syncwarp();
            mark(kHybVisit);
            // score once a batch is full or the list (seeds / expansion) ends
            if (nst == 0 || (nst < 32 && !(seed_next >= nseeds && adj_b >= L))) continue;
            }  // (!drain)

            // ---- score the F staged offers (new or improved nodes) in lanes 0..F-1
            const uint32_t F = min(nst, 32u);
            const bool mine = lane < F;
            uint32_t cn = 0, chop = 0;
            uint4 mt = make_uint4(0, 0, 0, 0);
            bool cimp = false;
            if (mine) {
                cn = w.st_node[lane];
                mt = w.st_meta[lane];
                const uint32_t fl = w.st_fl[lane];
                chop = fl & 0x7FFFFFFFu;
                cimp = (fl >> 31) != 0;
            }
            __syncwarp();
            if (nst > F && lane < nst - F) {  // carry the rest (< 32) to the front
                w.st_node[lane] = w.st_node[F + lane];
                w.st_meta[lane] = w.st_meta[F + lane];
                w.st_fl[lane] = w.st_fl[F + lane];
            }
            __syncwarp();
            nst -= F;
            const double rew = (mine && chop) ? rtab[chop - 1] : 0.0;
            if (mine && (a.prefetch & 4)) {
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
            double Ls = 0.0, Ss = 0.0;
#pragma unroll 1
            for (int path = 0; path < 2; ++path) {
                const bool learned = path == 0;
                const PathQ P = learned ? Q.p[0] : Q.p[1];
                if (!P.on) continue;
                const uint32_t* pidx = learned ? c.l_idx : c.s_idx;
                const float* pval = learned ? c.l_val : c.s_val;
                const uint32_t off4 = learned ? mt.x : mt.y, pnnz = learned ? (mt.z & 0xFFFFu) : (mt.z >> 16);
                double r;
                if constexpr (kMode == approx::kModeCuckoo)
                    r = sparse_group<approx::kLookCuckoo>(pidx, pval, P, off4, pnnz, lane, F);
                else if constexpr (kMode == approx::kModeHash)
                    r = sparse_group<false>(pidx, pval, P, off4, pnnz, lane, F);
                else
                    r = P.vocab ? sparse_group<true>(pidx, pval, P, off4, pnnz, lane, F)
                                : sparse_group<false>(pidx, pval, P, off4, pnnz, lane, F);
                if (learned)
                    Ls = r;
                else
                    Ss = r;
            }
            // screening against both full pools' worst entries (a node below
            // both cannot be in either pool, so its offer is a no-op)
            bool keep = mine;
            if (mine && csize == B && tsize == K) {
                const double floor = fmin(-w.cand_d[csize - 1], -w.topk_d[tsize - 1]) - 4.0 * eps;
                const double dn = Q.qd ? (double)__uint_as_float(mt.w) : 0.0;
                const double ub = score_upper_bound(Q.qd ? qnorm : 0.0, dn, Ls, Ss) + 2.0 * eps + rew;
                keep = !(ub < floor);
            }
            const uint32_t km = __ballot_sync(kFull, keep);
            mark(kHybSparse);
            if (keep && Q.qd && (a.prefetch & 1))
                l2_prefetch(c.dense + static_cast<uint64_t>(cn) * c.dstride, c.dstride * 4);
            // (2 dense rows per round trip: 4 cost this larger kernel two query-warps per SM)
            const double D = Q.qd ? dense_group<NQ4, 2>(c, Q.qd, cn, lane, km) : 0.0;
            const uint32_t m = __popc(km);
            mark(kHybDense);
            if (m == 0) continue;
            double d = keep ? __dsub_rn(-__dadd_rn(__dadd_rn(D, Ls), Ss), rew) : dinf();
            uint32_t n = keep ? cn : kEmpty;
            if (keep && cimp && expbits && ((expbits[cn >> 5] >> (cn & 31)) & 1u)) n |= kExp;

            // improved nodes leave the pools before the batch merges (their new
            // distance is strictly better: erase + insert == Pool::offer)
            const uint32_t im = __ballot_sync(kFull, keep && cimp);
            if (im) {
                csize = pool_erase(w.cand_d, w.cand_n, csize, im, n, lane);
                cursor = 0;
                if (R == 0) tsize = pool_erase(w.topk_d, w.topk_n, tsize, im, n, lane);
            }
#ifdef FGB_DEBUG_HYB
            {
                const uint32_t vm2 = __ballot_sync(kFull, n != kEmpty);
                if (lane == 0 && vm2 != ((m == 32) ? kFull : ((1u << m) - 1u)) && __popc(vm2) != m)
                    printf("PRE m %u F %u km %08x vm %08x im %08x seed %d csize %u tsize %u\n", m, F, km, vm2, im,
                           (int)is_seed, csize, tsize);
            }
#endif
            // ---- certify the batch order and its ranks in cand (search_plain.cu);
            // top-k candidates (non-deleted, able to enter at the current back)
            // are made exact here too.  Every exact re-score of the batch goes
            // through ONE call site (the request list below): each inlined copy
            // of the chain is ~1.5K instructions, and the kernel's speed
            // depends on its hot loop staying in the instruction cache.
            uint32_t rank_c = 0;
            bool qt = false;
#pragma unroll 1
            while (true) {
                warp_sort(d, n, lane);
#ifdef FGB_DEBUG_HYB
                if (lane < m && n == kEmpty) printf("SORT lane %u m %u d %g\n", lane, m, d);
                if (lane < m && n != kEmpty && (n & kId) >= c.n) printf("BADID lane %u m %u n %08x d %g\n", lane, m, n, d);
#endif
                const double dn2 = __shfl_down_sync(kFull, d, 1);
                const uint32_t nn2 = __shfl_down_sync(kFull, n, 1);
                const bool bad = lane < 31 && n != kEmpty && nn2 != kEmpty && !certain(d, n, dn2, nn2, tol);
                const bool prev_bad = __shfl_up_sync(kFull, bad, 1);
                bool fix = (bad || (prev_bad && lane > 0)) && n != kEmpty && !(n & kExact);
                bool need_c = false;
                qt = false;
                if (!__any_sync(kFull, fix)) {
                    if (lane < m) {
                        rank_c = pool_rank(cand, csize, d, n & kId);
                        need_c = (rank_c > 0 && !certain(w.cand_d[rank_c - 1], w.cand_n[rank_c - 1], d, n, tol)) ||
                                 (rank_c < csize && !certain(d, n, w.cand_d[rank_c], w.cand_n[rank_c], tol));
                        qt = !c.deleted[n & kId] && (tsize < K || d < w.topk_d[tsize - 1] + tol);
                    }
                    fix = (need_c || qt) && !(n & kExact);
                }
                const uint32_t ncm = __ballot_sync(kFull, need_c);
                const uint32_t fxm = __ballot_sync(kFull, fix);
                if (!fxm && !ncm) break;
                // requests: the batch lanes to fix, then the cand entries around
                // the doubtful ranks (leftovers past kXq wait for the next round)
                const uint32_t nfix = __popc(fxm);
                if (fix) w.xn[__popc(fxm & lt)] = n & kId;
                uint32_t nreq = nfix;
                uint32_t nm2 = ncm;
                while (nm2) {
                    const uint32_t j = __ffs(nm2) - 1;
                    nm2 &= nm2 - 1;
                    const int i = static_cast<int>(__shfl_sync(kFull, rank_c, j)) - 4 + static_cast<int>(lane);
                    const bool pf = lane < 8 && i >= 0 && i < static_cast<int>(csize) && !(w.cand_n[i] & kExact);
                    const uint32_t pm = __ballot_sync(kFull, pf);
                    if (nreq + __popc(pm) > kXq) break;
                    if (pf) {
                        const uint32_t r = nreq + __popc(pm & lt);
                        w.xn[r] = w.cand_n[i] & kId;
                        w.xi[r] = static_cast<uint32_t>(i);
                    }
                    nreq += __popc(pm);
                }
                __syncwarp();
                for (uint32_t r = lane; r < nreq; r += 32) w.xd[r] = exact_adj<kMode>(c, Q, w.xn[r], ctxq, h.ctxcap, rtab);
                __syncwarp();
                if (fix) {
                    d = w.xd[__popc(fxm & lt)];
                    n |= kExact;
                }
                for (uint32_t r = nfix + lane; r < nreq; r += 32) {
                    const uint32_t i = w.xi[r];
                    if (!(w.cand_n[i] & kExact)) {  // (two windows may name one entry)
                        w.cand_d[i] = w.xd[r];
                        w.cand_n[i] |= kExact;
                    }
                }
                resolved += nreq;
                __syncwarp();
            }
            qt = qt && (tsize < K || d <= w.topk_d[tsize - 1]);  // (ties: the node id decides below)
            const uint32_t p0 = pool_insert(cand, csize, d, n, m, rank_c, lane, w.br);
            cursor = min(cursor, p0);
            mark(kHybCand);

            const uint32_t qm = __ballot_sync(kFull, qt);
            if (qm && R == 0) {
                // set semantics: merge as one exact sorted batch
                const uint32_t ts = __fns(qm, 0, lane + 1);
                const uint32_t tm = __popc(qm);
                double td = __shfl_sync(kFull, d, ts < 32 ? ts : 0);
                uint32_t tn = __shfl_sync(kFull, n, ts < 32 ? ts : 0);
                uint32_t rank_t = 0;
                if (lane < tm)
                    rank_t = pool_rank(topk, tsize, td, tn & kId);
                else {
                    td = dinf();
                    tn = kEmpty;
                }
                pool_insert(topk, tsize, td, tn, tm, rank_t, lane, w.br);
            } else if (qm) {
                // keyword query: Pool::offer in reach order (the compacted
                // pre-sort order), evictions sharing a required keyword feed
                // the twin pool (search.cpp:171-181)
                for (uint32_t j = 0; j < F; ++j) {
                    const uint32_t x = __shfl_sync(kFull, cn, j);
                    const uint32_t at = __ballot_sync(kFull, lane < m && (n & kId) == x) & qm;
                    if (!at) continue;
                    const double dx = __shfl_sync(kFull, d, __ffs(at) - 1);
                    // pool find (search.cpp:28-33)
                    int pos = -1;
                    for (uint32_t b = 0; b < tsize && pos < 0; b += 32) {
                        const uint32_t fmk = __ballot_sync(kFull, b + lane < tsize && (w.topk_n[b + lane] & kId) == x);
                        if (fmk) pos = static_cast<int>(b + __ffs(fmk) - 1);
                    }
                    uint32_t ev = kEmpty;
                    if (lane == 0) {
                        bool go = true;
                        uint32_t sz = tsize;
                        if (pos >= 0) {
                            if (!(dx < w.topk_d[pos])) {
                                go = false;
                            } else {
                                for (uint32_t i = pos + 1; i < sz; ++i) {
                                    w.topk_d[i - 1] = w.topk_d[i];
                                    w.topk_n[i - 1] = w.topk_n[i];
                                }
                                --sz;
                            }
                        } else if (sz == K && !eless(dx, x, w.topk_d[sz - 1], w.topk_n[sz - 1] & kId)) {
                            go = false;
                        }
                        if (go) {
                            uint32_t ins = 0;  // upper_bound
                            while (ins < sz && !eless(dx, x, w.topk_d[ins], w.topk_n[ins] & kId)) ++ins;
                            if (sz == K) ev = w.topk_n[sz - 1] & kId;
                            const uint32_t last = min(sz, K - 1);
                            for (int i = static_cast<int>(last) - 1; i >= static_cast<int>(ins); --i) {
                                w.topk_d[i + 1] = w.topk_d[i];
                                w.topk_n[i + 1] = w.topk_n[i];
                            }
                            w.topk_d[ins] = dx;
                            w.topk_n[ins] = x | kExact;
                            if (sz < K) ++sz;
                        }
                        tsize = sz;
                    }
                    tsize = __shfl_sync(kFull, tsize, 0);
                    ev = __shfl_sync(kFull, ev, 0);
                    __syncwarp();
                    if (ev != kEmpty && !((twinbits[ev >> 5] >> (ev & 31)) & 1u) &&
                        shares_required(c, ev, w.req, R, lane)) {
                        if (ntwin < h.twcap) {
                            if (lane == 0) {
                                twinbits[ev >> 5] |= 1u << (ev & 31);
                                twin_node[ntwin] = ev;
                            }
                            ++ntwin;
                        } else {
                            err |= HERR_TWIN;
                        }
                        __syncwarp();
                    }
                }
            }
        }

        mark(kHybSelect);
        // ---- results: keyword_postfilter (search.cpp:100-139)
        uint32_t out = 0;
        if (err == 0 && R == 0) {
            for (uint32_t i = lane; i < tsize; i += 32) {  // (every top-k entry entered exact)
                a.r_node[static_cast<uint64_t>(qi) * a.hit_stride + i] = w.topk_n[i] & kId;
                a.r_score[static_cast<uint64_t>(qi) * a.hit_stride + i] = -w.topk_d[i];
            }
            out = tsize;
        } else if (err == 0) {
            // twin entries at their final adjusted distance, exactly
            for (uint32_t i = lane; i < ntwin; i += 32) twin_d[i] = exact_adj<kMode>(c, Q, twin_node[i], ctxq, h.ctxcap, rtab);
            __syncwarp();
            const uint32_t total = tsize + ntwin;
            while (out < K) {
                double bd = dinf();
                uint32_t bn = kEmpty;
                for (uint32_t i = lane; i < total; i += 32) {
                    const double dd = i < tsize ? w.topk_d[i] : twin_d[i - tsize];
                    const uint32_t nn = i < tsize ? (w.topk_n[i] == kEmpty ? kEmpty : (w.topk_n[i] & kId))
                                                  : twin_node[i - tsize];
                    if (nn != kEmpty && eless(dd, nn, bd, bn)) {
                        bd = dd;
                        bn = nn;
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const double od = __shfl_xor_sync(kFull, bd, o);
                    const uint32_t on = __shfl_xor_sync(kFull, bn, o);
                    if (eless(od, on, bd, bn)) {
                        bd = od;
                        bn = on;
                    }
                }
                if (bn == kEmpty) break;
                __syncwarp();
                for (uint32_t i = lane; i < total; i += 32) {  // consume every copy of the node
                    if (i < tsize) {
                        if (w.topk_n[i] != kEmpty && (w.topk_n[i] & kId) == bn) w.topk_n[i] = kEmpty;
                    } else if (twin_node[i - tsize] == bn) {
                        twin_node[i - tsize] = kEmpty;
                    }
                }
                __syncwarp();
                if (c.deleted[bn]) continue;
                bool all = true, any = false;
                const uint64_t kb = c.kw_ptr[bn], ke = c.kw_ptr[bn + 1];
                for (uint32_t i = lane; i < R; i += 32) {
                    const bool hh = sorted_contains(c.kw_idx, kb, ke, w.req[i]);
                    all &= hh;
                    any |= hh;
                }
                all = __all_sync(kFull, all);
                any = __any_sync(kFull, any);
                if (h.conjunctive ? !all : !any) continue;
                if (lane == 0) {
                    a.r_node[static_cast<uint64_t>(qi) * a.hit_stride + out] = bn;
                    a.r_score[static_cast<uint64_t>(qi) * a.hit_stride + out] = -bd;
                }
                ++out;
            }
            // twin flags and nodes back to empty (the list may have been consumed)
            for (uint32_t i = lane; i < ntwin; i += 32) twin_node[i] = kEmpty;
        }
        if (lane == 0) {
            a.r_count[qi] = out;
            a.r_expanded[qi] = expanded;
            a.r_scored[qi] = scored;
            uint32_t warn = (flags & QF_FALLBACK) ? 1u : 0u;
            if (R > 0 && out < K) warn |= 2u;
            a.r_warn[qi] = warn;
            a.r_err[qi] = err;
        }
        // ---- reset the per-warp scratch
        if (ntouched <= a.tcap) {
            for (uint32_t i = lane; i < ntouched; i += 32) {
                const uint32_t x = touched[i];
                visited[x >> 5] = 0;
                if (expbits) expbits[x >> 5] = 0;
                if (twinbits) twinbits[x >> 5] = 0;
            }
        } else {
            for (uint64_t i = lane; i < a.nwords; i += 32) {
                visited[i] = 0;
                if (expbits) expbits[i] = 0;
                if (twinbits) twinbits[i] = 0;
            }
        }
        if (ctx_mode)
            for (uint32_t i = lane; i < h.ctxcap; i += 32) ctx[i] = make_uint4(kEmpty, 0, 0, 0);
        __syncwarp();
        mark(kHybFinal);
        if (T && lane == 0) ++ph[kHybQueries];
    }
    if (T && lane == 0)
        for (int k = 0; k < kHybCount; ++k) atomicAdd(&h.timing[k], ph[k]);
    if (a.stats) {
        const unsigned long long fe = __reduce_add_sync(kFull, static_cast<unsigned>(final_exact));
        if (lane == 0) {
            atomicAdd(&a.stats[0], resolved);
            atomicAdd(&a.stats[1], fe);
        }
    }
}

// Per-variant launchers (search_hybrid_{c,r,cr}.cu instantiate the kernel for
// entity-context-only, keyword-only and mixed batches: each instantiation
// carries only its features' code — instruction-cache footprint).
template <bool kCtx, bool kReq>
const void* hybrid_kernel_ptr(int nq4, int mode) {
    switch (nq4) {
#define FGB_HYBP(V)                                                                                         \
    case V:                                                                                                 \
        return mode == approx::kModeCuckoo                                                                  \
                   ? reinterpret_cast<const void*>(search_hybrid_kernel<V, approx::kModeCuckoo, kCtx, kReq>)\
               : mode == approx::kModeHash                                                                  \
                   ? reinterpret_cast<const void*>(search_hybrid_kernel<V, approx::kModeHash, kCtx, kReq>)  \
                   : reinterpret_cast<const void*>(search_hybrid_kernel<V, approx::kModeMixed, kCtx, kReq>);
        FGB_HYBP(1)
        FGB_HYBP(2)
        FGB_HYBP(3)
        FGB_HYBP(4)
        FGB_HYBP(6)
        FGB_HYBP(8)
#undef FGB_HYBP
        default: return nullptr;
    }
}

template <bool kCtx, bool kReq>
void hybrid_launch_variant(const HybridLaunch& h, int nq4, uint64_t blocks, size_t smem, cudaStream_t s) {
    switch (nq4) {
#define FGB_HYB(V)                                                                                               \
    case V:                                                                                                      \
        if (h.p.mode == approx::kModeCuckoo) {                                                                   \
            FGB_CUDA(cudaFuncSetAttribute(search_hybrid_kernel<V, approx::kModeCuckoo, kCtx, kReq>,              \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));              \
            search_hybrid_kernel<V, approx::kModeCuckoo, kCtx, kReq><<<(unsigned)blocks, 32, smem, s>>>(h);      \
        } else if (h.p.mode == approx::kModeHash) {                                                              \
            FGB_CUDA(cudaFuncSetAttribute(search_hybrid_kernel<V, approx::kModeHash, kCtx, kReq>,                \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));              \
            search_hybrid_kernel<V, approx::kModeHash, kCtx, kReq><<<(unsigned)blocks, 32, smem, s>>>(h);        \
        } else {                                                                                                 \
            FGB_CUDA(cudaFuncSetAttribute(search_hybrid_kernel<V, approx::kModeMixed, kCtx, kReq>,               \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));              \
            search_hybrid_kernel<V, approx::kModeMixed, kCtx, kReq><<<(unsigned)blocks, 32, smem, s>>>(h);       \
        }                                                                                                        \
        break;
        FGB_HYB(1)
        FGB_HYB(2)
        FGB_HYB(3)
        FGB_HYB(4)
        FGB_HYB(6)
        FGB_HYB(8)
#undef FGB_HYB
        default: throw Error("internal", "hybrid search: unsupported dense width");
    }
}

}  // namespace

}  // namespace fgb
