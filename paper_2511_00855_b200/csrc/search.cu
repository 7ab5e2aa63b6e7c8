// search.cu — K5: batched beam search (search.cpp:141-293) on the GPU.
//
// One WARP owns one query at a time (persistent warps pull query ids from a
// global counter).  Per-query state lives in that warp's slice of shared
// memory: the staged weighted query (dense + sparse hashes), the sorted
// `cand` beam and `topk` pools, and the current expansion's neighbour list.
// Visited ("scored") flags are an exact per-warp bitset in HBM (n bits,
// cleared through a touched list), so no per-query O(n) state is allocated.
//
// Exactness.  Scores are bit-identical to the reference (device_common.cuh).
// The best-first order is the reference's: expand the first unexpanded
// cand entry; neighbours in reach order (semantic, keyword if u shares a
// required keyword, logical vias of group ent(u) while hop < max hops).
//  * Plain queries (no entity context possible): a re-offer of an already
//    scored node is a no-op in Pool::offer (its distance never changes and
//    the pool's worst entry only improves), so only first-time neighbours are
//    offered; the cand pool content is offer-order independent
//    (search.cpp:22-24), so they merge as one sorted batch.  topk merges as a
//    batch too unless required keywords make the twin pool order-dependent,
//    in which case lane 0 replays the offers in reach order (search.cpp:171-181).
//  * Entity-context queries: context propagation runs first for the whole
//    neighbour list in reach order (it depends only on u's context and each
//    neighbour's own state), then every neighbour whose adjusted distance is
//    new or changed is offered in reach order with warp-cooperative
//    single-entry offers (exactly Pool::offer, search.cpp:26-42).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "approx_score.cuh"
#include "fg_cuda.hpp"
#include "index.hpp"
#include "query_stage.cuh"
#include "search_hybrid.hpp"
#include "search_plain.hpp"
#include "tma.cuh"

namespace fgb {
namespace {

constexpr uint32_t kFlagExp = 0x80000000u;  // cand entry expanded
constexpr uint32_t kNodeMask = 0x7FFFFFFFu;
constexpr int kWarpsPerBlock = 1;  // one query-warp per CTA: CTAs pack SMs by smem
constexpr uint32_t kFull = 0xFFFFFFFFu;

enum : uint32_t { QF_VALID = 1, QF_ENTITY = 2, QF_FALLBACK = 4 };
enum : uint32_t { ERR_TWIN = 1, ERR_CTX = 2 };

struct SearchArgs {
    DevCorpus c;
    const uint32_t* semantic;
    uint32_t degree;
    const uint64_t* kw_ptr;
    const uint32_t* kw_idx;
    const uint64_t* lg_ptr;
    const uint4* lg;
    const uint64_t* kg_ptr;
    const uint32_t* kg_nbr;
    uint32_t kg_rows;
    DevQueries q;
    const uint64_t* seed_ptr;
    const uint32_t* seed_node;
    const uint32_t* seed_ent;
    const uint8_t* seed_has;
    const uint32_t* norm_order;
    uint32_t entry_count;
    const uint8_t* qflags;
    int conjunctive;
    uint32_t lcap, scap, beamcap, kcap, nbcap, lccap, reqcap;
    uint32_t warp_smem;
    // TMA row staging: rb slots of slot_words 4-byte words each; inside a
    // slot: dense [0, dstride), learned idx/val, statistical idx/val
    uint32_t rb, slot_words, o_lidx, o_lval, o_sidx, o_sval;
    uint32_t* visited;
    uint32_t* expbits;
    uint32_t* twinbits;
    uint64_t nwords;
    uint32_t* touched;
    uint32_t tcap;
    uint32_t* twin_node;
    double* twin_raw;
    uint32_t twcap;
    uint4* ctx;
    uint32_t ctxcap;
    uint32_t hit_stride;
    uint32_t* r_node;
    double* r_score;
    uint32_t* r_count;
    unsigned long long* r_expanded;
    unsigned long long* r_scored;
    uint32_t* r_warn;
    uint32_t* r_err;
    unsigned int* work;
    const uint32_t* qlist;  // optional subset of query ids to run (overflow re-runs)
    uint32_t qlist_n;
    // optional phase timing (FGB_SEARCH_TIMING=1): clock64 cycles summed over
    // warps per phase, see kPhase* below
    unsigned long long* timing;
    int prefetch;  // L2 row prefetch of first-time neighbours (FGB_SEARCH_PREFETCH, default on)
};

// Phase-timing slots (warp-level cycles unless noted)
enum : int {
    kPhSeeds = 0, kPhSelect, kPhAdj, kPhDedupe, kPhScore, kPhMerge, kPhFinal,
    kPhLaneSparse, kPhLaneDense, kPhLaneScored, kPhLaneDenseRows, kPhQueries, kPhExpanded,
    kPhCount
};

__device__ __forceinline__ bool eless(double d1, uint32_t n1, double d2, uint32_t n2) {
    return d1 < d2 || (d1 == d2 && n1 < n2);  // entry_less (search.cpp:13-16)
}

// Per-warp shared-memory views.
struct WarpMem {
    unsigned char* stage;
    double* cand_d;
    uint32_t* cand_n;
    double* topk_d;
    double* topk_raw;
    uint32_t* topk_n;
    double* nd;       // dist per new node
    uint32_t* nb;     // neighbour ids, reach order
    uint32_t* nnew;   // positions (in nb) of first-time neighbours
    uint8_t* nflag;   // per nb position: 1 new, 2 ctx changed
    uint32_t* lc;     // (via, target) pairs of the logical group
    uint32_t* req;    // required keywords (sorted)
    double* bd;       // batch sort buffer
    uint32_t* bn;
    float* rows;      // rb staged document rows (TMA destination)
    uint64_t* bar;    // mbarrier of the staging rounds
};

__device__ WarpMem carve(unsigned char* base, const SearchArgs& a) {
    WarpMem m;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        unsigned char* p = base + off;
        off += (bytes + 15) & ~size_t(15);
        return p;
    };
    m.stage = take(stage_bytes(a.c.dstride, a.lcap, a.scap));
    m.cand_d = reinterpret_cast<double*>(take(a.beamcap * 8));
    m.topk_d = reinterpret_cast<double*>(take(a.kcap * 8));
    m.topk_raw = reinterpret_cast<double*>(take(a.kcap * 8));
    m.nd = reinterpret_cast<double*>(take(a.nbcap * 8));
    m.bd = reinterpret_cast<double*>(take(32 * 8));
    m.cand_n = reinterpret_cast<uint32_t*>(take(a.beamcap * 4));
    m.topk_n = reinterpret_cast<uint32_t*>(take(a.kcap * 4));
    m.nb = reinterpret_cast<uint32_t*>(take(a.nbcap * 4));
    m.nnew = reinterpret_cast<uint32_t*>(take(a.nbcap * 4));
    m.nflag = reinterpret_cast<uint8_t*>(take(a.nbcap));
    m.lc = reinterpret_cast<uint32_t*>(take(a.lccap * 8 + 8));
    m.req = reinterpret_cast<uint32_t*>(take(a.reqcap * 4 + 4));
    m.bn = reinterpret_cast<uint32_t*>(take(32 * 4));
    m.bar = reinterpret_cast<uint64_t*>(take(16));
    m.rows = reinterpret_cast<float*>(take(static_cast<size_t>(a.rb) * a.slot_words * 4));
    return m;
}

// ---------------------------------------------------------------- staged K1
// Scores `count` nodes (node_of(i), i < count) against the staged query,
// rb rows per round: every lane owning a row issues TMA bulk copies of its
// dense row and sparse postings into its smem slot, one mbarrier completes
// the round, then each lane runs its bit-exact chain from shared memory
// (slot stride = 4 mod 32 words, so the lanes' 16-byte reads never conflict).
template <typename NodeOf, typename Sink>
__device__ void score_staged(const SearchArgs& a, const SmemQuery& sq, const WarpMem& w,
                             uint32_t lane, uint32_t& phase, uint32_t count, NodeOf node_of,
                             Sink sink, double qnorm = 0.0,
                             double floor = -__builtin_huge_val()) {
    const DevCorpus& c = a.c;
    if (a.rb == 0) {  // register path: each lane streams its own row
        for (uint32_t b = 0; b < count; b += 32) {
            if (b + lane < count) {
                // screened: a node whose exact-score bound cannot reach either
                // full pool's worst entry gets +inf (never offered, never read)
                double s;
                bool scored;
                if (a.timing) {
                    const uint32_t node = node_of(b + lane);
                    const long long t0 = clock64();
                    const double l = sparse_part(c, sq, node, true);
                    const double sp = sparse_part(c, sq, node, false);
                    const long long t1 = clock64();
                    scored = !(score_upper_bound(sq.dense ? qnorm : 0.0, sq.dense ? c.dnorm[node] : 0.0, l, sp) < floor);
                    if (scored) {
                        if (sq.dense) l2_prefetch(c.dense + (uint64_t)node * c.dstride, c.dstride * 4);
                        double acc = sq.dense ? dense_chain<8>(c, sq.dense, node) : 0.0;
                        acc = __dadd_rn(acc, l);
                        s = __dadd_rn(acc, sp);
                    }
                    const long long t2 = clock64();
                    atomicAdd(&a.timing[kPhLaneSparse], (unsigned long long)(t1 - t0));
                    atomicAdd(&a.timing[kPhLaneDense], (unsigned long long)(t2 - t1));
                    atomicAdd(&a.timing[kPhLaneScored], 1ull);
                    if (scored) atomicAdd(&a.timing[kPhLaneDenseRows], 1ull);
                } else {
                    scored = hybrid_score_screened<8>(c, sq, node_of(b + lane), qnorm, floor, s);
                }
                sink(b + lane, scored ? -s : __longlong_as_double(0x7FF0000000000000ll));
            }
        }
        __syncwarp();
        return;
    }
    for (uint32_t b = 0; b < count; b += a.rb) {
        const uint32_t cnt = min(a.rb, count - b);
        const bool mine = lane < cnt;
        uint32_t node = 0, ln = 0, sn = 0, bytes = 0;
        uint64_t lo = 0, so = 0;
        if (mine) {
            node = node_of(b + lane);
            if (sq.lmask) {
                ln = c.l_nnz[node];
                lo = c.l_off[node];
            }
            if (sq.smask) {
                sn = c.s_nnz[node];
                so = c.s_off[node];
            }
            bytes = (sq.dense ? c.dstride * 4 : 0) + ((ln + 3) & ~3u) * 8 + ((sn + 3) & ~3u) * 8;
        }
        uint32_t total = bytes;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(kFull, total, o);
        if (lane == 0) {
            fence_proxy_async();
            mbar_arrive_expect_tx(w.bar, total);
        }
        __syncwarp();
        float* slot = w.rows + static_cast<size_t>(lane) * a.slot_words;
        if (mine) {
            if (sq.dense) bulk_g2s(slot, c.dense + static_cast<uint64_t>(node) * c.dstride, c.dstride * 4, w.bar);
            if (ln) {
                const uint32_t nb = ((ln + 3) & ~3u) * 4;
                bulk_g2s(slot + a.o_lidx, c.l_idx + lo, nb, w.bar);
                bulk_g2s(slot + a.o_lval, c.l_val + lo, nb, w.bar);
            }
            if (sn) {
                const uint32_t nb = ((sn + 3) & ~3u) * 4;
                bulk_g2s(slot + a.o_sidx, c.s_idx + so, nb, w.bar);
                bulk_g2s(slot + a.o_sval, c.s_val + so, nb, w.bar);
            }
        }
        mbar_wait(w.bar, phase);
        phase ^= 1u;
        if (mine) {
            double acc = 0.0;
            if (sq.dense) {
                const float4* r4 = reinterpret_cast<const float4*>(slot);
                const double2* q2 = reinterpret_cast<const double2*>(sq.dense);
                const uint32_t n4 = c.dstride >> 2;
#pragma unroll 4
                for (uint32_t i = 0; i < n4; ++i) {
                    const float4 d = r4[i];
                    const double2 qa = q2[2 * i], qb = q2[2 * i + 1];
                    acc = __fma_rn(qa.x, (double)d.x, acc);
                    acc = __fma_rn(qa.y, (double)d.y, acc);
                    acc = __fma_rn(qb.x, (double)d.z, acc);
                    acc = __fma_rn(qb.y, (double)d.w, acc);
                }
            }
            auto sparse = [&](const uint32_t* idx, const float* val, uint32_t nnz, const uint32_t* keys,
                              const float* vals, uint32_t mask, const uint32_t* filt) {
                double s = 0.0;  // ascending index order, 16-byte smem reads
                const uint4* i4 = reinterpret_cast<const uint4*>(idx);
                const float4* v4 = reinterpret_cast<const float4*>(val);
                for (uint32_t j = 0; j < (nnz + 3) / 4; ++j) {
                    const uint4 ii = i4[j];
                    const float4 vv = v4[j];
                    probe_term(ii.x, vv.x, keys, vals, mask, filt, s);
                    probe_term(ii.y, vv.y, keys, vals, mask, filt, s);
                    probe_term(ii.z, vv.z, keys, vals, mask, filt, s);
                    probe_term(ii.w, vv.w, keys, vals, mask, filt, s);
                }
                return s;
            };
            const uint32_t* si = reinterpret_cast<const uint32_t*>(slot);
            acc = __dadd_rn(acc, ln ? sparse(si + a.o_lidx, slot + a.o_lval, ln, sq.lkeys, sq.lvals, sq.lmask, sq.lfilt) : 0.0);
            acc = __dadd_rn(acc, sn ? sparse(si + a.o_sidx, slot + a.o_sval, sn, sq.skeys, sq.svals, sq.smask, sq.sfilt) : 0.0);
            sink(b + lane, -acc);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- pools
// Sorted pool (dist asc, node asc) in smem: warp-cooperative primitives.
struct PoolRef {
    double* d;
    uint32_t* n;   // node | kFlagExp (cand) ; node (topk)
    uint32_t cap;
};

__device__ __forceinline__ int pool_find(const PoolRef& p, uint32_t size, uint32_t node,
                                         uint32_t lane) {
    for (uint32_t b = 0; b < size; b += 32) {
        const uint32_t i = b + lane;
        const bool hit = i < size && (p.n[i] & kNodeMask) == node;
        const uint32_t m = __ballot_sync(kFull, hit);
        if (m) return static_cast<int>(b + __ffs(m) - 1);
    }
    return -1;
}

// # entries strictly less than (d, node) (== upper_bound with unique nodes).
__device__ __forceinline__ uint32_t pool_rank(const PoolRef& p, uint32_t size, double d,
                                              uint32_t node) {
    uint32_t lo = 0, hi = size;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (eless(p.d[mid], p.n[mid] & kNodeMask, d, node))
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// Pool::offer (search.cpp:26-42), all lanes with uniform arguments.
// Returns the evicted node or -1; `flag` is stored with the node.
__device__ int64_t pool_offer(const PoolRef& p, uint32_t& size, double d, uint32_t node,
                              uint32_t flag, uint32_t lane) {
    const int pos = pool_find(p, size, node, lane);
    if (pos >= 0) {
        if (!eless(d, node, p.d[pos], node)) return -1;  // no improvement
        flag = p.n[pos] & kFlagExp;
        for (uint32_t b = pos + 1; b < size; b += 32) {  // erase: shift left
            const uint32_t i = b + lane;
            double dd = 0;
            uint32_t nn = 0;
            if (i < size) {
                dd = p.d[i];
                nn = p.n[i];
            }
            __syncwarp();
            if (i < size) {
                p.d[i - 1] = dd;
                p.n[i - 1] = nn;
            }
            __syncwarp();
        }
        --size;
    } else if (size == p.cap) {
        if (!eless(d, node, p.d[size - 1], p.n[size - 1] & kNodeMask)) return -1;
    }
    const uint32_t ins = pool_rank(p, size, d, node);
    int64_t evicted = -1;
    if (size == p.cap) evicted = p.n[size - 1] & kNodeMask;
    __syncwarp();
    const uint32_t last = min(size, p.cap - 1);  // entries [ins, last) move right by one
    if (last > ins) {
        for (int b = static_cast<int>(((last - 1 - ins) / 32) * 32 + ins); b >= static_cast<int>(ins); b -= 32) {
            const uint32_t i = b + lane;
            double dd = 0;
            uint32_t nn = 0;
            const bool v = i < last;
            if (v) {
                dd = p.d[i];
                nn = p.n[i];
            }
            __syncwarp();
            if (v) {
                p.d[i + 1] = dd;
                p.n[i + 1] = nn;
            }
            __syncwarp();
        }
    }
    if (lane == 0) {
        p.d[ins] = d;
        p.n[ins] = node | flag;
    }
    __syncwarp();
    if (size < p.cap) ++size;
    return evicted;
}

// Batch merge of m <= 32 new entries (sorted, in bd/bn, all absent from the
// pool) — the set result of offering them one by one.  Returns the smallest
// insertion position (or cap when nothing entered).
__device__ uint32_t pool_merge(const PoolRef& p, uint32_t& size, const double* bd,
                               const uint32_t* bn, uint32_t m, uint32_t lane) {
    if (m == 0) return p.cap;
    uint32_t mypos = p.cap, rank = 0xFFFFFFFFu;
    double md = 0;
    uint32_t mn = 0;
    if (lane < m) {
        md = bd[lane];
        mn = bn[lane];
        rank = pool_rank(p, size, md, mn);  // # pool entries < new entry `lane`
        mypos = lane + rank;
    }
    uint32_t p0 = mypos;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) p0 = min(p0, __shfl_xor_sync(kFull, p0, o));
    if (p0 >= p.cap) return p.cap;  // every new entry is worse than a full pool
    __syncwarp();
    // Entries before p0 stay; entry i >= p0 moves right by #{j : rank_j <= i}
    // (ranks are non-decreasing in j), processed right to left.
    if (size > p0) {
        // ranks to shared memory (the sorted bn slots are no longer needed)
        uint32_t* br = const_cast<uint32_t*>(bn);
        __syncwarp();
        if (lane < m) br[lane] = rank;
        __syncwarp();
        for (int b = static_cast<int>(((size - 1) / 32) * 32); b >= static_cast<int>(p0 & ~31u); b -= 32) {
            const uint32_t i = b + lane;
            const bool v = i < size && i >= p0;
            uint32_t lo = 0, hi = m;  // shift = #{j : rank_j <= i} (upper bound)
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (br[mid] <= i)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            const uint32_t shift = lo;
            double dd = 0;
            uint32_t nn = 0;
            const uint32_t np = i + shift;
            if (v) {
                dd = p.d[i];
                nn = p.n[i];
            }
            __syncwarp();
            if (v && np < p.cap) {
                p.d[np] = dd;
                p.n[np] = nn;
            }
            __syncwarp();
        }
    }
    if (lane < m && mypos < p.cap) {
        p.d[mypos] = md;
        p.n[mypos] = mn;  // new entries are unexpanded
    }
    __syncwarp();
    size = min(size + m, p.cap);
    uint32_t mn_pos = mypos;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mn_pos = min(mn_pos, __shfl_xor_sync(kFull, mn_pos, o));
    return mn_pos;
}

// Warp bitonic sort of one (dist, node) pair per lane (invalid lanes carry +inf).
__device__ __forceinline__ void warp_sort(double& d, uint32_t& n, uint32_t lane) {
#pragma unroll
    for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            const double od = __shfl_xor_sync(kFull, d, j);
            const uint32_t on = __shfl_xor_sync(kFull, n, j);
            const bool up = (lane & k) == 0;
            const bool lower = (lane & j) == 0;
            const bool other_less = eless(od, on, d, n);
            const bool take = (lower == up) ? other_less : (!other_less && (od != d || on != n));
            if (take) {
                d = od;
                n = on;
            }
        }
    }
}

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ bool bit_test_set(uint32_t* bits, uint32_t node) {
    const uint32_t m = 1u << (node & 31);
    return (atomicOr(&bits[node >> 5], m) & m) != 0;
}
__device__ __forceinline__ bool bit_test(const uint32_t* bits, uint32_t node) {
    return (bits[node >> 5] >> (node & 31)) & 1u;
}

// shares_required (search.cpp:163-167): u holds ANY required keyword.
__device__ bool shares_required(const DevCorpus& c, uint32_t node, const uint32_t* req, uint32_t R,
                                uint32_t lane) {
    bool hit = false;
    const uint64_t b = c.kw_ptr[node], e = c.kw_ptr[node + 1];
    for (uint32_t i = lane; i < R; i += 32) hit |= sorted_contains(c.kw_idx, b, e, req[i]);
    return __any_sync(kFull, hit);
}

// has_relation (types.cpp:52-57) on the device adjacency.
__device__ bool has_relation(const SearchArgs& a, uint32_t x, uint32_t y) {
    if (x >= a.kg_rows) return false;
    return sorted_contains(a.kg_nbr, a.kg_ptr[x], a.kg_ptr[x + 1], y);
}

// Entity-context table (per warp, global memory): (node, ent, hop, has).
// Probes are bounded by the capacity: a full table never spins.  The kernel
// flags ERR_CTX once the load factor passes 1/2 and the host re-runs that
// query with a larger table (fg_batch_query), so a -1 from ctx_slot only
// occurs on a query whose result is discarded anyway.
__device__ int ctx_find(const uint4* t, uint32_t cap, uint32_t node) {
    uint32_t s = hslot(node, cap - 1);
    for (uint32_t probe = 0; probe < cap; ++probe) {
        const uint4 e = t[s];
        if (e.x == node) return static_cast<int>(s);
        if (e.x == kEmpty) return -1;
        s = (s + 1) & (cap - 1);
    }
    return -1;
}
__device__ int ctx_slot(uint4* t, uint32_t cap, uint32_t node, uint32_t& used) {
    uint32_t s = hslot(node, cap - 1);
    for (uint32_t probe = 0; probe < cap; ++probe) {
        const uint4 e = t[s];
        if (e.x == node) return static_cast<int>(s);
        if (e.x == kEmpty) {
            t[s] = make_uint4(node, 0, 0, 0);
            ++used;
            return static_cast<int>(s);
        }
        s = (s + 1) & (cap - 1);
    }
    used = cap;  // full: the caller's load-factor test raises ERR_CTX
    return -1;
}

__global__ void __launch_bounds__(kWarpsPerBlock * 32) search_kernel(SearchArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t slot = blockIdx.x * (uint64_t)kWarpsPerBlock + warp;
    WarpMem w = carve(smem_raw + static_cast<size_t>(warp) * a.warp_smem, a);
    uint32_t* visited = a.visited + slot * a.nwords;
    uint32_t* expbits = a.expbits ? a.expbits + slot * a.nwords : nullptr;
    uint32_t* twinbits = a.twinbits ? a.twinbits + slot * a.nwords : nullptr;
    uint32_t* touched = a.touched + slot * a.tcap;
    uint32_t* twin_node = a.twin_node ? a.twin_node + slot * a.twcap : nullptr;
    double* twin_raw = a.twin_raw ? a.twin_raw + slot * a.twcap : nullptr;
    uint4* ctx = a.ctx ? a.ctx + slot * a.ctxcap : nullptr;
    const DevCorpus& c = a.c;
    uint32_t phase = 0;  // staging mbarrier phase (persists across queries)
    if (lane == 0) {
        mbar_init(w.bar, 1);
        fence_proxy_async();
    }
    __syncwarp();

    unsigned long long ph[kPhLaneSparse] = {};
    long long tmark = clock64();
    auto phase_end = [&](int k) {  // attribute cycles since the last mark to phase k
        if (a.timing) {
            const long long t = clock64();
            ph[k] += t - tmark;
            tmark = t;
        }
    };
    while (true) {
        uint32_t qi = 0;
        if (lane == 0) qi = atomicAdd(a.work, 1u);
        qi = __shfl_sync(kFull, qi, 0);
        if (a.qlist) {  // re-run of the queries that overflowed their scratch
            if (qi >= a.qlist_n) break;
            qi = a.qlist[qi];
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
        const double went = static_cast<double>(a.q.weights[qi].w);
        const bool ctx_mode = (flags & QF_ENTITY) != 0;
        SmemQuery sq;
        stage_query(a.q, qi, c.dstride, w.stage, a.lcap, a.scap, lane, 32, sq, [] { __syncwarp(); });
        double qnorm = 0.0;  // |weighted query dense| for the screening bound
        if (sq.dense) {
            for (uint32_t j = lane; j < c.dstride; j += 32) qnorm += sq.dense[j] * sq.dense[j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) qnorm += __shfl_xor_sync(kFull, qnorm, o);
            qnorm = sqrt(qnorm) * (1.0 + 1e-12);
        }
        const uint64_t rb = a.q.req_ptr[qi];
        const uint32_t R = static_cast<uint32_t>(a.q.req_ptr[qi + 1] - rb);
        for (uint32_t i = lane; i < R; i += 32) w.req[i] = a.q.req_idx[rb + i];
        __syncwarp();

        PoolRef cand{w.cand_d, w.cand_n, B};
        PoolRef topk{w.topk_d, w.topk_n, K};
        uint32_t csize = 0, tsize = 0, ntouched = 0, ntwin = 0, ctx_used = 0, err = 0;
        unsigned long long expanded = 0, scored = 0;
        bool tover = false;

        // ---- helpers bound to this query -------------------------------
        auto touch = [&](uint32_t node, bool mine) {  // record a visited node
            const uint32_t m = __ballot_sync(kFull, mine);
            const uint32_t pos = ntouched + __popc(m & ((1u << lane) - 1));
            if (mine && pos < a.tcap) touched[pos] = node;
            ntouched += __popc(m);
        };
        // topk offer by lane 0 in reach order, twin pool on eviction
        auto topk_offer_seq = [&](uint32_t node, double dist, double raw) {
            // (all lanes call; lane 0 does the work; state kept uniform via shfl)
            int64_t ev = -1;
            double ev_raw = 0;
            if (lane == 0) {
                int pos = -1;
                for (uint32_t i = 0; i < tsize; ++i)
                    if (w.topk_n[i] == node) pos = static_cast<int>(i);
                bool go = true;
                if (pos >= 0) {
                    if (!eless(dist, node, w.topk_d[pos], node)) {
                        go = false;
                    } else {
                        for (uint32_t i = pos + 1; i < tsize; ++i) {
                            w.topk_d[i - 1] = w.topk_d[i];
                            w.topk_n[i - 1] = w.topk_n[i];
                            w.topk_raw[i - 1] = w.topk_raw[i];
                        }
                        --tsize;
                    }
                } else if (tsize == K && !eless(dist, node, w.topk_d[tsize - 1], w.topk_n[tsize - 1])) {
                    go = false;
                }
                if (go) {
                    uint32_t ins = 0;
                    while (ins < tsize && !eless(dist, node, w.topk_d[ins], w.topk_n[ins])) ++ins;
                    if (tsize == K) {
                        ev = w.topk_n[tsize - 1];
                        ev_raw = w.topk_raw[tsize - 1];
                    }
                    const uint32_t last = min(tsize, K - 1);
                    for (int i = static_cast<int>(last) - 1; i >= static_cast<int>(ins); --i) {
                        w.topk_d[i + 1] = w.topk_d[i];
                        w.topk_n[i + 1] = w.topk_n[i];
                        w.topk_raw[i + 1] = w.topk_raw[i];
                    }
                    w.topk_d[ins] = dist;
                    w.topk_n[ins] = node;
                    w.topk_raw[ins] = raw;
                    if (tsize < K) ++tsize;
                }
            }
            tsize = __shfl_sync(kFull, tsize, 0);
            ev = __shfl_sync(kFull, ev, 0);
            ev_raw = __shfl_sync(kFull, ev_raw, 0);
            __syncwarp();
            if (ev >= 0 && R > 0) {
                const uint32_t e = static_cast<uint32_t>(ev);
                if (!bit_test(twinbits, e) && shares_required(c, e, w.req, R, lane)) {
                    if (lane == 0) {
                        twinbits[e >> 5] |= 1u << (e & 31);
                        if (ntwin < a.twcap) {
                            twin_node[ntwin] = e;
                            twin_raw[ntwin] = ev_raw;
                        }
                    }
                    if (ntwin >= a.twcap) err |= ERR_TWIN;
                    ++ntwin;
                }
            }
        };
        // adjusted distance (search.cpp:156-161)
        auto adjusted = [&](double raw, uint32_t node) {
            if (!ctx_mode) return raw;
            const int s = ctx_find(ctx, a.ctxcap, node);
            if (s >= 0) {
                const uint4 e = ctx[s];
                if (e.w && e.z >= 1) return raw - went / static_cast<double>(e.z);
            }
            return raw;
        };
        // assign_ctx (search.cpp:191-198), lane 0; returns true on change
        auto assign_ctx = [&](uint32_t node, uint32_t ent, uint32_t hop) {
            const int s = ctx_slot(ctx, a.ctxcap, node, ctx_used);
            if (s < 0) return false;
            const uint4 e = ctx[s];
            if (e.w && (e.z < hop || (e.z == hop && e.y <= ent))) return false;
            ctx[s] = make_uint4(node, ent, hop, 1u);
            return true;
        };
        // deleted nodes never reach topk (search.cpp:174)
        auto is_deleted = [&](uint32_t node) { return c.deleted[node] != 0; };

        // ---- seeds (search.cpp:205-216) --------------------------------
        const bool norm_seeds = !(flags & QF_ENTITY);
        const uint64_t sb = norm_seeds ? 0 : a.seed_ptr[qi];
        const uint32_t nseeds = norm_seeds ? a.entry_count
                                           : static_cast<uint32_t>(a.seed_ptr[qi + 1] - sb);
        for (uint32_t base = 0; base < nseeds; base += 32) {
            const uint32_t i = base + lane;
            const bool v = i < nseeds;
            uint32_t node = 0, ent = 0;
            bool has = false;
            double raw = 0;
            if (v) {
                node = norm_seeds ? a.norm_order[i] : a.seed_node[sb + i];
                if (!norm_seeds) {
                    ent = a.seed_ent[sb + i];
                    has = a.seed_has[sb + i] != 0;
                }
                bit_test_set(visited, node);
            }
            const uint32_t cnt_s = min(32u, nseeds - base);
            score_staged(a, sq, w, lane, phase, cnt_s,
                         [&](uint32_t j) {
                             return norm_seeds ? a.norm_order[base + j] : a.seed_node[sb + base + j];
                         },
                         [&](uint32_t j, double d) { w.nd[j] = d; });
            if (v) raw = w.nd[lane];
            __syncwarp();
            touch(node, v);
            scored += __popc(__ballot_sync(kFull, v));
            const uint32_t cnt = min(32u, nseeds - base);
            for (uint32_t j = 0; j < cnt; ++j) {  // offers in seed order
                const uint32_t nj = __shfl_sync(kFull, node, j);
                const uint32_t ej = __shfl_sync(kFull, ent, j);
                const bool hj = __shfl_sync(kFull, has, j);
                const double rj = __shfl_sync(kFull, raw, j);
                if (hj && lane == 0) assign_ctx(nj, ej, 0);
                ctx_used = __shfl_sync(kFull, ctx_used, 0);
                __syncwarp();
                const double dj = adjusted(rj, nj);
                pool_offer(cand, csize, dj, nj, 0, lane);
                if (!is_deleted(nj)) topk_offer_seq(nj, dj, rj);
            }
        }
        if (ctx_used * 2 > a.ctxcap) err |= ERR_CTX;
        phase_end(kPhSeeds);

        // ---- best-first expansion (search.cpp:218-264) ------------------
        uint32_t cursor = 0;
        while (err == 0) {
            int upos = -1;
            for (uint32_t b = cursor; b < csize && upos < 0; b += 32) {
                const uint32_t i = b + lane;
                const bool un = i < csize && !(w.cand_n[i] & kFlagExp);
                const uint32_t m = __ballot_sync(kFull, un);
                if (m) upos = static_cast<int>(b + __ffs(m) - 1);
            }
            phase_end(kPhSelect);
            if (upos < 0) break;
            cursor = upos;
            const uint32_t u = w.cand_n[upos] & kNodeMask;
            if (lane == 0) {
                w.cand_n[upos] |= kFlagExp;
                if (expbits) expbits[u >> 5] |= 1u << (u & 31);
            }
            __syncwarp();
            ++expanded;

            // neighbours in reach order
            uint32_t nbc = a.degree;
            for (uint32_t j = lane; j < a.degree; j += 32) w.nb[j] = a.semantic[(uint64_t)u * a.degree + j];
            if (R > 0 && shares_required(c, u, w.req, R, lane)) {
                const uint64_t kb = a.kw_ptr[u], ke = a.kw_ptr[u + 1];
                for (uint64_t j = kb + lane; j < ke; j += 32) w.nb[nbc + (j - kb)] = a.kw_idx[j];
                nbc += static_cast<uint32_t>(ke - kb);
            }
            bool propagate = false;
            uint32_t uent = 0, uhop = 0, nlc = 0;
            if (ctx_mode) {
                const int s = ctx_find(ctx, a.ctxcap, u);
                if (s >= 0 && ctx[s].w) {
                    uent = ctx[s].y;
                    uhop = ctx[s].z;
                    propagate = uhop < H;
                }
                if (propagate) {
                    const uint64_t lb = a.lg_ptr[u], le = a.lg_ptr[u + 1];
                    for (uint64_t j = lb; j < le; j += 32) {  // group source == ent(u)
                        const uint64_t e = j + lane;
                        uint4 ed = make_uint4(0, 0, 0, 0);
                        const bool hit = e < le && (ed = a.lg[e]).x == uent;
                        const uint32_t m = __ballot_sync(kFull, hit);
                        const uint32_t pos = nlc + __popc(m & ((1u << lane) - 1));
                        if (hit) {
                            w.nb[nbc + pos] = ed.w;
                            w.lc[2 * pos] = ed.w;
                            w.lc[2 * pos + 1] = ed.z;
                        }
                        nlc += __popc(m);
                    }
                    nbc += nlc;
                }
            }
            __syncwarp();
            phase_end(kPhAdj);

            // dedupe (reach order) + first-time detection
            uint32_t nnew = 0, nkeep = 0;
            for (uint32_t b = 0; b < nbc; b += 32) {
                const uint32_t i = b + lane;
                const bool v = i < nbc;
                const uint32_t x = v ? w.nb[i] : kEmpty;
                bool keep = v;
                if (v) {  // drop repeats of an earlier position
                    for (uint32_t j = 0; j < i && keep; ++j) keep = w.nb[j] != x;
                }
                bool fresh = false;
                if (keep) fresh = !bit_test_set(visited, x);
                // first-time neighbours: pull their whole rows toward L2 now,
                // one bulk prefetch per span, so the scoring chains below
                // stream from L2 instead of paying a DRAM trip per stage
                if (fresh && a.prefetch) prefetch_sparse(c, sq, x);
                __syncwarp();
                const uint32_t km = __ballot_sync(kFull, keep);
                const uint32_t kpos = nkeep + __popc(km & ((1u << lane) - 1));
                if (keep) {
                    w.nb[kpos] = x;  // compact in place (kpos <= i)
                    w.nflag[kpos] = fresh ? 1 : 0;
                }
                const uint32_t fm = __ballot_sync(kFull, fresh);
                if (fresh) w.nnew[nnew + __popc(fm & ((1u << lane) - 1))] = kpos;
                touch(x, fresh);
                nkeep += __popc(km);
                nnew += __popc(fm);
                __syncwarp();
            }
            nbc = nkeep;
            scored += nnew;
            phase_end(kPhDedupe);

            // score first-time neighbours, lane per node.  Plain queries screen
            // against the worst entries of BOTH pools when both are full (an
            // offer below both is a no-op); entity-context queries may re-offer
            // a node later with a better distance, so they always score.
            double floor = -__longlong_as_double(0x7FF0000000000000ll);
            if (!ctx_mode && csize == B && tsize == K)
                floor = fmin(-w.cand_d[csize - 1], -w.topk_d[tsize - 1]);
            score_staged(a, sq, w, lane, phase, nnew, [&](uint32_t i) { return w.nb[w.nnew[i]]; },
                         [&](uint32_t i, double d) { w.nd[w.nnew[i]] = d; }, qnorm, floor);
            __syncwarp();
            phase_end(kPhScore);

            if (!ctx_mode) {
                // cand: one sorted batch per 32 new nodes (order independent)
                for (uint32_t b = 0; b < nnew; b += 32) {
                    const uint32_t i = b + lane;
                    double d = __longlong_as_double(0x7FF0000000000000ll);
                    uint32_t nn = kEmpty;
                    if (i < nnew) {
                        nn = w.nb[w.nnew[i]];
                        d = w.nd[w.nnew[i]];
                    }
                    warp_sort(d, nn, lane);
                    w.bd[lane] = d;
                    w.bn[lane] = nn;
                    __syncwarp();
                    const uint32_t m = min(32u, nnew - b);
                    const uint32_t p0 = pool_merge(cand, csize, w.bd, w.bn, m, lane);
                    cursor = min(cursor, p0);
                    if (R == 0) {  // topk batch, deleted nodes skipped
                        const bool ok = lane < m && !is_deleted(nn);
                        const uint32_t om = __ballot_sync(kFull, ok);
                        // keep sorted order among the survivors
                        const uint32_t pos = __popc(om & ((1u << lane) - 1));
                        __syncwarp();
                        if (ok) {
                            w.bd[pos] = d;
                            w.bn[pos] = nn;
                        }
                        __syncwarp();
                        pool_merge(topk, tsize, w.bd, w.bn, __popc(om), lane);
                    }
                    __syncwarp();
                }
                if (R > 0) {  // twin pool depends on the offer order
                    for (uint32_t i = 0; i < nnew; ++i) {
                        const uint32_t pos = w.nnew[i];
                        const uint32_t node = w.nb[pos];
                        if (!is_deleted(node)) topk_offer_seq(node, w.nd[pos], w.nd[pos]);
                    }
                }
            } else {
                // context propagation over the whole list (lane 0, reach order)
                if (propagate && lane == 0) {
                    const uint32_t hop = uhop + 1;
                    for (uint32_t i = 0; i < nbc; ++i) {
                        const uint32_t o = w.nb[i];
                        bool changed = false;
                        const uint64_t eb = c.ent_ptr[o], ee = c.ent_ptr[o + 1];
                        for (uint64_t e = eb; e < ee; ++e) {
                            const uint32_t ent = c.ent_idx[e];
                            if (has_relation(a, uent, ent)) {
                                changed |= assign_ctx(o, ent, hop);
                                break;
                            }
                        }
                        for (uint32_t j = 0; j < nlc; ++j)
                            if (w.lc[2 * j] == o) changed |= assign_ctx(o, w.lc[2 * j + 1], hop);
                        if (changed) w.nflag[i] |= 2;
                    }
                }
                ctx_used = __shfl_sync(kFull, ctx_used, 0);
                __syncwarp();
                if (ctx_used * 2 > a.ctxcap) err |= ERR_CTX;
                // raw distance of re-offered (context-changed) old nodes
                for (uint32_t b = 0; b < nbc; b += 32) {
                    const uint32_t i = b + lane;
                    if (i < nbc && w.nflag[i] == 2) w.nd[i] = -hybrid_score<12>(c, sq, w.nb[i]);
                }
                __syncwarp();
                for (uint32_t i = 0; i < nbc; ++i) {
                    if (!w.nflag[i]) continue;  // unchanged old node: a no-op offer
                    const uint32_t o = w.nb[i];
                    const double raw = w.nd[i];
                    const double d = adjusted(raw, o);
                    const uint32_t fl = (expbits && bit_test(expbits, o)) ? kFlagExp : 0u;
                    pool_offer(cand, csize, d, o, fl, lane);
                    if (!is_deleted(o)) topk_offer_seq(o, d, raw);
                }
                cursor = 0;
            }
            phase_end(kPhMerge);
        }

        // ---- keyword_postfilter (search.cpp:100-139) ---------------------
        // candidates: topk (+ twin pool when keywords are required)
        const uint32_t ntw = R > 0 ? min(ntwin, a.twcap) : 0;
        if (lane == 0)
            for (uint32_t i = 0; i < ntw; ++i) twin_raw[i] = adjusted(twin_raw[i], twin_node[i]);
        __syncwarp();
        uint32_t out = 0;
        const uint32_t total = tsize + ntw;
        while (out < K) {
            // best remaining (dist, node) over topk ∪ twin
            double bd = __longlong_as_double(0x7FF0000000000000ll);
            uint32_t bnode = kEmpty;
            for (uint32_t i = lane; i < total; i += 32) {
                const double d = i < tsize ? w.topk_d[i] : twin_raw[i - tsize];
                const uint32_t nn = i < tsize ? w.topk_n[i] : twin_node[i - tsize];
                if (nn != kEmpty && eless(d, nn, bd, bnode)) {
                    bd = d;
                    bnode = nn;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double od = __shfl_xor_sync(kFull, bd, o);
                const uint32_t on = __shfl_xor_sync(kFull, bnode, o);
                if (eless(od, on, bd, bnode)) {
                    bd = od;
                    bnode = on;
                }
            }
            if (bnode == kEmpty) break;
            for (uint32_t i = lane; i < total; i += 32) {  // consume every copy of the node
                if (i < tsize) {
                    if (w.topk_n[i] == bnode) w.topk_n[i] = kEmpty;
                } else if (twin_node[i - tsize] == bnode) {
                    twin_node[i - tsize] = kEmpty;
                }
            }
            __syncwarp();
            if (is_deleted(bnode)) continue;
            if (R > 0) {
                bool all = true, any = false;
                const uint64_t kb = c.kw_ptr[bnode], ke = c.kw_ptr[bnode + 1];
                for (uint32_t i = lane; i < R; i += 32) {
                    const bool h = sorted_contains(c.kw_idx, kb, ke, w.req[i]);
                    all &= h;
                    any |= h;
                }
                all = __all_sync(kFull, all);
                any = __any_sync(kFull, any);
                if (a.conjunctive ? !all : !any) continue;
            }
            if (lane == 0) {
                a.r_node[(uint64_t)qi * a.hit_stride + out] = bnode;
                a.r_score[(uint64_t)qi * a.hit_stride + out] = -bd;
            }
            ++out;
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

        // ---- reset per-warp scratch ---------------------------------------
        if (ntouched > a.tcap) tover = true;
        if (!tover) {
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
        if (ctx) {
            for (uint32_t i = lane; i < a.ctxcap; i += 32) ctx[i] = make_uint4(kEmpty, 0, 0, 0);
        }
        __syncwarp();
        phase_end(kPhFinal);
        if (a.timing && lane == 0) {
            for (int k = 0; k < kPhLaneSparse; ++k) atomicAdd(&a.timing[k], ph[k]);
            atomicAdd(&a.timing[kPhQueries], 1ull);
            atomicAdd(&a.timing[kPhExpanded], expanded);
            for (int k = 0; k < kPhLaneSparse; ++k) ph[k] = 0;
        }
    }
}

}  // namespace
}  // namespace fgb


namespace fgb {
namespace {
constexpr uint64_t kId30 = 0x3FFFFFFFull;  // node ids must fit 30 bits in the plain kernel's pools
constexpr uint32_t kGpoolBeam = 1536;       // beams above this keep the plain kernel's cand pool in HBM (B200, 1M docs: beam 1024 smem 45.9K vs HBM 43.0K QPS; 2048: 19.9K vs 20.5K; 3008: 10.3K vs 13.1K)

// Device results -> the caller's fg_search_results (ids -> doc ids, per-query
// validation errors, counters); records the kernel time of ev0..ev1.
void finish_results(fg_index* ix, const fg_corpus& c, const fg_query_view* q, fg_search_results* out,
                    std::vector<std::string>& errs, uint64_t nq, uint32_t stride, cudaStream_t s,
                    double extra_ms = 0.0) {
    (void)q;
    SearchIo& io = ix->ws->io;
    // pinned staging: 8-byte fields first, then the 4-byte ones
    const uint64_t hits = nq * stride;
    const uint64_t bytes = hits * 12 + nq * 32 + 16;
    // large batches come back through grow-only pinned staging (DMA speed);
    // small ones through pageable memory — a first cudaMallocHost costs
    // milliseconds, more than a small batch's whole search (insert_batch)
    std::vector<unsigned char> small;
    unsigned char* h = nullptr;
    if (bytes <= (512u << 10) && io.host.get() == nullptr) {
        small.resize(bytes);
        h = small.data();
    } else {
        io.host.ensure(bytes);
        h = io.host.get();
    }
    double* h_score = reinterpret_cast<double*>(h);
    unsigned long long* h_exp = reinterpret_cast<unsigned long long*>(h_score + hits);
    unsigned long long* h_sc = h_exp + nq;
    uint32_t* h_node = reinterpret_cast<uint32_t*>(h_sc + nq);
    uint32_t* h_count = h_node + hits;
    uint32_t* h_warn = h_count + nq;
    uint32_t* h_err = h_warn + nq;
    io.r_node.download(h_node, hits, s);
    io.r_score.download(h_score, hits, s);
    io.r_count.download(h_count, nq, s);
    io.r_warn.download(h_warn, nq, s);
    io.r_err.download(h_err, nq, s);
    io.r_exp.download(h_exp, nq, s);
    io.r_sc.download(h_sc, nq, s);
    FGB_CUDA(cudaStreamSynchronize(s));
    float ms = 0;
    FGB_CUDA(cudaEventElapsedTime(&ms, ix->ev0, ix->ev1));
    ix->last_kernel_ms = ms + extra_ms;
    for (uint64_t i = 0; i < nq; ++i) {
        // still overflowing after the re-runs at the largest scratch size:
        // this query alone fails (batch_query's per-query capture, search.cpp:286-290)
        if (h_err[i] && errs[i].empty())
            errs[i] = "internal: search scratch overflow (twin pool / entity-context table)";
        const uint32_t cnt = errs[i].empty() ? h_count[i] : 0;
        out->hit_count[i] = cnt;
        for (uint32_t j = 0; j < cnt; ++j) {
            const uint32_t node = h_node[i * stride + j];
            out->node[i * out->hit_stride + j] = node;
            out->doc_id[i * out->hit_stride + j] = c.doc_id[node];
            out->score[i * out->hit_stride + j] = h_score[i * stride + j];
        }
        if (out->expanded) out->expanded[i] = errs[i].empty() ? h_exp[i] : 0;
        if (out->scored) out->scored[i] = errs[i].empty() ? h_sc[i] : 0;
        if (out->warnings) out->warnings[i] = errs[i].empty() ? h_warn[i] : 0;
        if (out->errors && out->error_stride) {
            char* dst = out->errors + i * out->error_stride;
            std::strncpy(dst, errs[i].c_str(), out->error_stride - 1);
            dst[out->error_stride - 1] = 0;
        }
    }
}
// Entity-context / required-keyword batches on the certified kernel
// (search_hybrid.cu).  Queries that overflow their twin pool or context table
// are re-run alone with 4x larger tables; false when the batch does not fit
// the kernel's shared memory (the caller falls back to search_kernel).
bool run_hybrid(fg_index* ix, fg_corpus& c, SearchWorkspace& W, const PlainLaunch& pl,
                const std::array<uint32_t, 5>& ck_fallback, const fg_query_view* q,
                const std::vector<uint8_t>& qflags, uint32_t max_seeds, uint32_t max_req, bool any_ctx,
                bool any_req, bool conj,
                uint64_t nq, uint32_t stride, std::vector<std::string>& errs, fg_search_results* out,
                cudaStream_t s) {
    SearchIo& io = W.io;
    const uint64_t n = c.n;
    HybridLaunch h{};
    h.p = pl;
    h.seed_ptr = io.sptr.get();
    h.seed_node = io.snode.get();
    h.seed_ent = io.sent.get();
    // rewards w_k / hop (search.cpp:156-161) divided here, in the
    // reference's double arithmetic: the kernel does no fp64 division
    if (any_ctx) {
        uint32_t hmax = 1;
        for (uint64_t i = 0; i < nq; ++i)
            if (qflags[i] & QF_ENTITY)
                hmax = std::max(hmax, q->max_entity_hops ? q->max_entity_hops[i] : 2u);
        if (hmax > 4096) return false;  // (the exact-chain kernel divides on the device)
        h.rstride = hmax;
        std::vector<double> tab(nq * hmax, 0.0);
        for (uint64_t i = 0; i < nq; ++i)
            if (qflags[i] & QF_ENTITY) {
                const double went = static_cast<double>(q->weights[i].entity);
                for (uint32_t hop = 1; hop <= hmax; ++hop) tab[i * hmax + hop - 1] = went / static_cast<double>(hop);
            }
        io.rew.upload(tab, s);
        h.rewards = io.rew.get();
    }
    h.kw_ptr = ix->kw_ptr.get();
    h.kw_idx = ix->kw_idx.get();
    h.lg_ptr = ix->lg_ptr.get();
    h.lg = ix->lg.get();
    h.kg_ptr = ix->kg_ptr.get();
    h.kg_nbr = ix->kg_nbr.get();
    h.kg_rows = ix->kg_rows;
    h.conjunctive = conj ? 1 : 0;
    h.variant = any_ctx && !any_req ? kHybCtx : (any_req && !any_ctx ? kHybReq : kHybBoth);
    h.reqcap = std::max(max_req, 1u);
    h.lccap = std::max(ix->max_logical_group, 1u);
    const uint32_t list_max = ix->degree + (any_req ? ix->max_kw_edges : 0) + (any_ctx ? h.lccap : 0);
    h.seencap = 64;
    while (2 * h.seencap < 3 * list_max) h.seencap <<= 1;  // load <= 2/3
    if (hybrid_warp_smem(h) == 0) return false;
    uint64_t all_slots = hybrid_slots(h, nq, c.device);
    h.p.hit_stride = stride;
    h.p.r_node = io.r_node.get();
    h.p.r_score = io.r_score.get();
    h.p.r_count = io.r_count.get();
    h.p.r_expanded = io.r_exp.get();
    h.p.r_scored = io.r_sc.get();
    h.p.r_warn = io.r_warn.get();
    h.p.r_err = io.r_err.get();
    h.p.work = io.work.get();
    h.p.timing = nullptr;
    h.p.nwords = (n + 31) / 32;
    h.p.tcap = 1024;
    while (h.p.tcap < 65536 && h.p.tcap < n) h.p.tcap <<= 1;
    uint32_t twcap0 = any_req ? 4096 : 0, ctxcap0 = 0;
    if (any_ctx) {
        ctxcap0 = 8192;
        while (ctxcap0 < 4ull * max_seeds && ctxcap0 < (1u << 26)) ctxcap0 <<= 1;
    }
    if (const char* e = std::getenv("FGB_SEARCH_SCRATCH0")) {  // test hook: force re-runs
        const uint32_t v = static_cast<uint32_t>(std::atoi(e));
        if (v >= 2 && (v & (v - 1)) == 0) {
            if (any_req) twcap0 = v;
            if (any_ctx) ctxcap0 = v;
        }
    }
    DevBuf<unsigned long long> stats;
    const char* se = std::getenv("FGB_SEARCH_STATS");
    if ((se && se[0] == '1') || h.p.eps_scale != 1.0) {
        stats.alloc(2);
        stats.zero(s);
        h.p.stats = stats.get();
    }
    DevBuf<unsigned long long> timing;
    if (const char* te = std::getenv("FGB_SEARCH_TIMING"); te && te[0] == '1') {
        timing.alloc(kHybCount);
        timing.zero(s);
        h.timing = timing.get();
    }
    std::vector<uint32_t> rerun;
    DevBuf<uint32_t> d_rerun;
    float ms_prev = 0.f;
    int grow = 0;  // scratch growth steps (twin / context tables)
    for (int attempt = 0;; ++attempt) {
        h.twcap = twcap0 << (2 * grow);
        h.ctxcap = ctxcap0 << (2 * grow);
        const uint64_t slots = attempt ? std::min<uint64_t>(all_slots, rerun.size()) : all_slots;
        const uint64_t nbits = 1 + (any_ctx ? 1 : 0) + (any_req ? 1 : 0);
        const uint64_t bits_words = slots * h.p.nwords * nbits;
        if (W.bits.size() < bits_words) {
            W.bits.alloc(bits_words);
            W.bits.zero(s);
        }
        uint32_t* bits = W.bits.get();
        h.p.visited = bits;
        h.expbits = any_ctx ? bits + slots * h.p.nwords : nullptr;
        h.twinbits = any_req ? bits + slots * h.p.nwords * (any_ctx ? 2 : 1) : nullptr;
        W.lists.ensure(std::max<uint64_t>(slots * (static_cast<uint64_t>(h.p.tcap) + h.twcap), 1));
        h.p.touched = W.lists.get();
        h.twin_node = any_req ? h.p.touched + slots * h.p.tcap : nullptr;
        const uint64_t misc = slots * (static_cast<uint64_t>(h.twcap) * 8 + static_cast<uint64_t>(h.ctxcap) * 16);
        W.misc.ensure(std::max<uint64_t>(misc, 16));
        h.twin_d = any_req ? reinterpret_cast<double*>(W.misc.get()) : nullptr;
        h.ctx = any_ctx ? reinterpret_cast<uint4*>(W.misc.get() + slots * h.twcap * 8) : nullptr;
        if (any_ctx) FGB_CUDA(cudaMemsetAsync(h.ctx, 0xFF, slots * h.ctxcap * 16, s));
        h.qlist = attempt ? d_rerun.get() : nullptr;
        h.qlist_n = static_cast<uint32_t>(rerun.size());
        FGB_CUDA(cudaMemsetAsync(h.p.work, 0, sizeof(unsigned int), s));
        FGB_CUDA(cudaEventRecord(ix->ev0, s));
        launch_search_hybrid(h, slots, s);
        FGB_CUDA(cudaEventRecord(ix->ev1, s));
        ix->last_launches = attempt + 1;
        ix->last_kernel = "search_hybrid_kernel";
        std::vector<uint32_t> h_err(nq);
        io.r_err.download(h_err.data(), nq, s);
        FGB_CUDA(cudaStreamSynchronize(s));
        rerun.clear();
        uint32_t err_any = 0;
        for (uint64_t i = 0; i < nq; ++i)
            if (h_err[i]) {
                rerun.push_back(static_cast<uint32_t>(i));
                err_any |= h_err[i];
            }
        if (err_any & (HERR_TWIN | HERR_CTX)) ++grow;
        if ((err_any & HERR_CUCKOO) && h.p.mode == approx::kModeCuckoo) {
            // a query without a cuckoo table: the re-run takes the fallback lookups
            h.p.mode = static_cast<int>(ck_fallback[0]);
            h.p.vocab[0] = ck_fallback[1];
            h.p.vocab[1] = ck_fallback[2];
            h.p.cap[0] = ck_fallback[3];
            h.p.cap[1] = ck_fallback[4];
            if (hybrid_warp_smem(h) == 0) return false;  // (the general kernel re-runs the batch)
            all_slots = hybrid_slots(h, nq, c.device);
        }
        constexpr uint64_t kMaxScratch = 1ull << 30;  // bytes of twin + context tables per launch
        const uint64_t next_slots = std::min<uint64_t>(all_slots, rerun.size());
        const uint64_t next_bytes = next_slots * ((uint64_t(h.twcap) * 12 + uint64_t(h.ctxcap) * 16) << 2);
        if (rerun.empty() || next_bytes > kMaxScratch) break;
        float ms = 0;
        FGB_CUDA(cudaEventElapsedTime(&ms, ix->ev0, ix->ev1));
        ms_prev += ms;
        d_rerun.upload(rerun, s);
    }
    if (h.p.stats) {
        unsigned long long st[2] = {};
        stats.download(st, 2, s);
        FGB_CUDA(cudaStreamSynchronize(s));
        std::fprintf(stderr, "[hybrid stats] exact resolutions %llu, exact final entries %llu\n", st[0], st[1]);
    }
    if (h.timing) {
        unsigned long long t[kHybCount] = {};
        timing.download(t, kHybCount, s);
        FGB_CUDA(cudaStreamSynchronize(s));
        const double X = t[kHybExpanded] ? (double)t[kHybExpanded] : 1.0;
        static const char* names[] = {"select+lists", "gather+dedupe", "visited+ctx", "sparse", "dense",
                                      "cand certify", "top-k", "final"};
        std::fprintf(stderr, "[hybrid timing] %llu queries, %.1f expansions/query, %.2f batches/expansion\n",
                     t[kHybQueries], X / std::max(1ull, t[kHybQueries]), t[kHybBatches] / X);
        for (int k = 0; k < kHybPhases; ++k)
            std::fprintf(stderr, "  %-16s %10.0f cycles/expansion\n", names[k], t[k] / X);
    }
    finish_results(ix, c, q, out, errs, nq, stride, s, ms_prev);
    return true;
}

}  // namespace
}  // namespace fgb

using namespace fgb;

extern "C" {

int fg_batch_query(const fg_index* cix, const fg_query_view* q, const fg_search_opts* opts,
                   fg_search_results* out) {
    return guarded([&] {
        if (!cix || !q || !out) throw Error("invalid-argument", "null pointer");
        fg_index* ix = const_cast<fg_index*>(cix);
        std::lock_guard<std::mutex> lock(ix->search_mu);
        HostTimer ht("batch_query");
        fg_corpus& c = *ix->corpus;
        if (!ix->ws) ix->ws = search_workspace(c.device);
        SearchWorkspace& W = *ix->ws;
        std::lock_guard<std::mutex> wlock(W.mu);
        FGB_CUDA(cudaSetDevice(c.device));
        cudaStream_t s = c.stream;
        const uint64_t nq = q->count;
        const uint32_t entry_count = opts ? opts->entry_count : 32;
        const bool conj = opts ? opts->conjunctive_filter != 0 : true;
        const uint64_t n = c.n;

        // ---- host: validation (types.cpp:20-27) and seeds (search.cpp:67-98)
        std::vector<uint8_t> qflags(nq, 0);
        std::vector<std::string> errs(nq);
        std::vector<uint64_t> seed_ptr(nq + 1, 0);
        std::vector<uint32_t> seed_node, seed_ent;
        std::vector<uint8_t> seed_has;
        uint32_t max_k = 1, max_beam = 1, max_seeds = 0;
        const uint32_t norm_seeds = static_cast<uint32_t>(std::min<uint64_t>(entry_count, n));
        for (uint64_t i = 0; i < nq; ++i) {
            const fg_weights wt = q->weights ? q->weights[i] : fg_weights{1.f, 1.f, 1.f, 0.f};
            const uint32_t k = q->k ? q->k[i] : 10;
            const uint32_t beam = q->beam_width ? q->beam_width[i] : 64;
            const uint64_t ne = q->entities.ptr ? q->entities.ptr[i + 1] - q->entities.ptr[i] : 0;
            try {
                const float parts[4] = {wt.dense, wt.learned, wt.statistical, wt.entity};
                for (float p : parts)
                    if (!std::isfinite(p) || p < 0.0f)
                        throw Error("invalid-weights", "weights must be finite and non-negative");
                if (wt.dense <= 0.0f && wt.learned <= 0.0f && wt.statistical <= 0.0f)
                    throw Error("invalid-weights", "at least one vector-path weight must be positive");
                if (k == 0) throw Error("invalid-k", "k must be positive");
                if (beam < k) throw Error("beam-too-small", "beam_width must be at least k");
                if (wt.entity > 0.0f && ne == 0)
                    throw Error("entities-required",
                                "entity weight is positive but the query names no entities");
                if (q->dense_dim != c.dim)
                    throw Error("dim-mismatch", "dense dimensions differ: " +
                                                    std::to_string(q->dense_dim) + " vs " +
                                                    std::to_string(c.dim));
            } catch (const Error& e) {
                errs[i] = e.what();
                seed_ptr[i + 1] = seed_node.size();
                continue;
            }
            uint8_t f = QF_VALID;
            if (ne > 0 && wt.entity > 0.0f) {
                std::vector<std::pair<uint32_t, uint32_t>> seeds;  // (node, entity)
                for (uint64_t j = q->entities.ptr[i]; j < q->entities.ptr[i + 1]; ++j) {
                    const uint32_t e = q->entities.idx[j];
                    auto it = ix->entity_map.find(e);
                    if (it == ix->entity_map.end()) continue;
                    for (uint32_t node : it->second) seeds.emplace_back(node, e);
                }
                if (!seeds.empty()) {
                    std::sort(seeds.begin(), seeds.end());
                    uint32_t cnt = 0;
                    for (size_t j = 0; j < seeds.size(); ++j) {
                        if (j > 0 && seeds[j].first == seeds[j - 1].first) continue;
                        seed_node.push_back(seeds[j].first);
                        seed_ent.push_back(seeds[j].second);
                        seed_has.push_back(1);
                        ++cnt;
                    }
                    max_seeds = std::max(max_seeds, cnt);
                    f |= QF_ENTITY;
                } else {
                    f |= QF_FALLBACK;
                }
            }
            seed_ptr[i + 1] = seed_node.size();
            qflags[i] = f;
            max_k = std::max(max_k, k);
            max_beam = std::max(max_beam, beam);
        }
        if (out->hit_stride < max_k && nq) throw Error("invalid-argument", "hit_stride < max k");
        bool any_ctx = false, any_req = false;
        uint32_t max_req = 0;
        for (uint64_t i = 0; i < nq; ++i) {
            any_ctx |= (qflags[i] & QF_ENTITY) != 0;
            const uint64_t r = q->required_keywords.ptr
                                   ? q->required_keywords.ptr[i + 1] - q->required_keywords.ptr[i]
                                   : 0;
            if ((qflags[i] & QF_VALID) && r) {
                any_req = true;
                max_req = std::max<uint32_t>(max_req, static_cast<uint32_t>(r));
            }
        }

        ht.mark("validate+seeds");
        // ---- device copies of the batch (buffers reused across calls)
        SearchIo& io = W.io;
        QueryUpload& up = io.up;
        up.upload(*q, s);
        DevBuf<uint64_t>& d_sptr = io.sptr;
        DevBuf<uint32_t>&d_snode = io.snode, &d_sent = io.sent;
        DevBuf<uint8_t>&d_shas = io.shas, &d_qflags = io.qflags;
        d_sptr.upload(seed_ptr, s);
        if (seed_node.empty()) {
            seed_node.push_back(0);
            seed_ent.push_back(0);
            seed_has.push_back(0);
        }
        d_snode.upload(seed_node, s);
        d_sent.upload(seed_ent, s);
        d_shas.upload(seed_has, s);
        d_qflags.upload(qflags.empty() ? std::vector<uint8_t>(1, 0) : qflags, s);
        const uint32_t stride = std::max(out->hit_stride, 1u);
        const uint64_t nq1 = std::max<uint64_t>(nq, 1);
        io.r_node.ensure(nq1 * stride);
        io.r_score.ensure(nq1 * stride);
        io.r_count.ensure(nq1);
        io.r_warn.ensure(nq1);
        io.r_err.ensure(nq1);
        io.r_exp.ensure(nq1);
        io.r_sc.ensure(nq1);
        DevBuf<uint32_t>&r_node = io.r_node, &r_count = io.r_count, &r_warn = io.r_warn, &r_err = io.r_err;
        DevBuf<double>& r_score = io.r_score;
        DevBuf<unsigned long long>&r_exp = io.r_exp, &r_sc = io.r_sc;
        io.work.ensure(1);
        FGB_CUDA(cudaMemsetAsync(io.work.get(), 0, sizeof(unsigned int), s));
        ht.mark("upload");
        DevBuf<unsigned int>& work = io.work;

        // ---- plain batches (no entity context, no required keywords): the
        // certified-approximate kernel (search_plain.cu), bit-identical results
        // Entity-context / required-keyword batches: the certified kernel of
        // search_hybrid.cu (FGB_SEARCH_HYBRID=0: the exact-chain search_kernel)
        const char* pe = std::getenv("FGB_SEARCH_PLAIN");
        const char* he = std::getenv("FGB_SEARCH_HYBRID");
        const char* fe = std::getenv("FGB_SEARCH_FORCE_HYBRID");  // dev A/B: plain batches on the hybrid kernel
        const bool special = any_ctx || any_req || (fe && fe[0] == '1');
        const bool cert_ok = (!pe || pe[0] != '0') && (!special || !he || he[0] != '0') && n < kId30 && c.dc.meta &&
                             ix->edge_meta.get();
        if (cert_ok && nq) {
            PlainLaunch pl{};
            pl.c = c.dc;
            pl.semantic = ix->semantic.get();
            pl.degree = ix->degree;
            pl.q = up.dq;
            pl.norm_order = ix->norm_order.get();
            pl.edge_meta = ix->edge_meta.get();
            pl.norm_meta = ix->norm_meta.get();
            pl.entry_count = norm_seeds;
            pl.qflags = d_qflags.get();
            std::array<uint32_t, 5> ck_fallback{};  // the lookup selection a failed cuckoo build falls back to
            // sparse paths: bitmap + rank lookups for vocabularies up to 64K
            // terms, filter + hash otherwise (FGB_SEARCH_BITMAP=0: hash only)
            const char* be = std::getenv("FGB_SEARCH_BITMAP");
            const bool bitmaps = !(be && be[0] == '0');
            pl.cap[0] = hash_capacity(up.max_lnnz);
            pl.cap[1] = hash_capacity(up.max_snnz);
            pl.vocab[0] = bitmaps && c.l_vocab <= 65536 ? c.l_vocab : 0;
            pl.vocab[1] = bitmaps && c.s_vocab <= 65536 ? c.s_vocab : 0;
            // one lookup mode per batch: when the batch walks both sparse
            // paths and one needs the hash, both take it — running both
            // modes' sparse groups overflows the instruction cache (C3/C4
            // simplex batches at 1M docs: 41.6K -> 44.1K QPS).  Queries whose
            // learned terms mostly hit (C4's chain queries without the hop
            // reward) lose on the hash's probe loops: 79.3K -> 70.2K QPS
            // (tools/mode_probe.py); FGB_SEARCH_MIXED=1 keeps both modes.
            const char* me = std::getenv("FGB_SEARCH_MIXED");  // dev: keep both modes (A/B)
            if (!(me && me[0] == '1') && up.max_lnnz && up.max_snnz && (pl.vocab[0] == 0) != (pl.vocab[1] == 0))
                pl.vocab[0] = pl.vocab[1] = 0;
            {  // hash-only batches run the hash-only instantiation (C4 plain batches
                // +3.5%); bitmap batches keep the per-path dispatch, which measured
                // 5% faster than a bitmap-only instantiation at configs[1] (B200)
                const bool l_on = up.max_lnnz > 0, s_on = up.max_snnz > 0;
                const bool all_hash = (!l_on || !pl.vocab[0]) && (!s_on || !pl.vocab[1]);
                pl.mode = all_hash ? approx::kModeHash : approx::kModeMixed;
                if (const char* e = std::getenv("FGB_SEARCH_MODE"); e && e[0] == '2') pl.mode = approx::kModeMixed;
                // every batch: two-choice cuckoo tables for both sparse paths
                // (FGB_SEARCH_CUCKOO=0: the bitmap / filter + hash selection
                // above).  B200, 200K docs, identical results: C2 shape bitmap
                // 139.6K -> 153.2K QPS, C3/C4 hash 59.3K -> 93.8K QPS.
                const char* ce = std::getenv("FGB_SEARCH_CUCKOO");
                const char* te0 = std::getenv("FGB_SEARCH_TIMING");  // (the timing variant is per-path dispatch)
                ck_fallback = {static_cast<uint32_t>(pl.mode), pl.vocab[0], pl.vocab[1], pl.cap[0], pl.cap[1]};
                if (!(ce && ce[0] == '0') && !(te0 && te0[0] == '1')) {
                    pl.mode = approx::kModeCuckoo;
                    auto ck_cap = [](uint32_t nnz) {
                        uint32_t c = 16;
                        while (c < 4 * nnz) c <<= 1;
                        return c;
                    };
                    pl.vocab[0] = pl.vocab[1] = 0;
                    pl.cap[0] = ck_cap(up.max_lnnz);
                    pl.cap[1] = ck_cap(up.max_snnz);
                }
            }
            pl.beamcap = std::max(max_beam, 32u);
            pl.kcap = std::max(max_k, 1u);
            pl.max_norm = std::sqrt(std::max(c.max_sqnorm, 0.0)) * (1.0 + 1e-9);
            // |approx - reference| <= eps_coef * |q_w| * max|d| (search_plain.cu):
            // fp32 partials of <= 4 products (gamma_4 in fp32), fp64 sums of the
            // partials (depth M) and the reference's own sequential sums (depth N)
            const double N = double(c.dstride) + c.max_lnnz + c.max_snnz + 2;
            const double M = (c.dstride >> 2) + 2.0 * ((std::max(c.max_lnnz, c.max_snnz) + 127) / 128) + 16;
            const double u32 = std::ldexp(1.0, -24), u64 = std::ldexp(1.0, -53);
            pl.eps32_coef = 4.0 * u32 / (1.0 - 4.0 * u32) * 1.01 + 1e-30;
            pl.eps_coef = (N + M + 8) * u64 * 1.01;
            pl.max_dnorm = c.max_dnorm * (1.0 + 1e-6);
            pl.eps_scale = 1.0;
            if (const char* e = std::getenv("FGB_EPS_SCALE")) pl.eps_scale = std::atof(e);
            // bulk L2 prefetches (bit mask): the screened survivors' dense rows (1),
            // every first-time neighbour's dense row (2: slowed demand loads,
            // tools/ubench_latency.cu), the postings of the sparse groups after
            // the first (4: +2% at 1M docs)
            pl.prefetch = 5;
            if (const char* e = std::getenv("FGB_SEARCH_PREFETCH")) pl.prefetch = std::atoi(e);
            if (special) {
                if (run_hybrid(ix, c, W, pl, ck_fallback, q, qflags, max_seeds, max_req, any_ctx, any_req, conj, nq, stride, errs, out, s))
                    return;
            } else {
              // very large beams keep their cand pools in HBM (L1/L2 cached):
              // in shared memory they would cut the query-warps per SM
              // (FGB_SEARCH_GPOOL=0/1 forces the choice)
              bool gpool = pl.beamcap > kGpoolBeam;
              if (const char* e = std::getenv("FGB_SEARCH_GPOOL")) gpool = e[0] == '1';
              if (gpool) {
                  pl.gpool_d = reinterpret_cast<double*>(1);  // (placeholders: smem sizing only)
                  pl.gpool_n = reinterpret_cast<uint32_t*>(1);
              }
              for (int ck_pass = 0; ck_pass < 2 && plain_warp_smem(pl) > 0; ++ck_pass) {
                const uint64_t slots = plain_slots(pl, nq, c.device);
                if (gpool) {
                    W.gpool.ensure(slots * pl.beamcap * 12);
                    pl.gpool_d = reinterpret_cast<double*>(W.gpool.get());
                    pl.gpool_n = reinterpret_cast<uint32_t*>(W.gpool.get() + slots * pl.beamcap * 8);
                }
                pl.nwords = (n + 31) / 32;
                // touched-list capacity: a query visits at most n nodes
                pl.tcap = 1024;
                while (pl.tcap < 65536 && pl.tcap < n) pl.tcap <<= 1;
                if (W.bits.size() < slots * pl.nwords) {
                    W.bits.alloc(slots * pl.nwords);
                    W.bits.zero(s);
                }
                pl.visited = W.bits.get();
                W.lists.ensure(slots * pl.tcap);
                pl.touched = W.lists.get();
                pl.hit_stride = stride;
                pl.r_node = r_node.get();
                pl.r_score = r_score.get();
                pl.r_count = r_count.get();
                pl.r_expanded = r_exp.get();
                pl.r_scored = r_sc.get();
                pl.r_warn = r_warn.get();
                pl.r_err = r_err.get();
                pl.work = work.get();
                DevBuf<unsigned long long> timing, stats;
                const char* te = std::getenv("FGB_SEARCH_TIMING");
                if (te && te[0] == '1') {
                    timing.alloc(kPlainPhCount);
                    timing.zero(s);
                    FGB_CUDA(cudaMemsetAsync(timing.get() + kPlainPhStart, 0xFF, 16, s));  // Start, EndMin = max
                    pl.timing = timing.get();
                }
                const char* se = std::getenv("FGB_SEARCH_STATS");
                if ((se && se[0] == '1') || pl.eps_scale != 1.0) {
                    stats.alloc(2);
                    stats.zero(s);
                    pl.stats = stats.get();
                }
                ht.mark("plain scratch");
                FGB_CUDA(cudaEventRecord(ix->ev0, s));
                launch_search_plain(pl, nq, c.device, s);
                FGB_CUDA(cudaEventRecord(ix->ev1, s));
                ht.mark("plain kernel");
                if (pl.mode == approx::kModeCuckoo) {
                    // a query without a cuckoo table (r_err 4; practically
                    // never at <= 1/4 load): the batch runs again with hash lookups
                    std::vector<uint32_t> h_err(nq);
                    r_err.download(h_err.data(), nq, s);
                    FGB_CUDA(cudaStreamSynchronize(s));
                    if (std::any_of(h_err.begin(), h_err.end(), [](uint32_t e) { return e == 4; })) {
                        pl.mode = static_cast<int>(ck_fallback[0]);
                        pl.vocab[0] = ck_fallback[1];
                        pl.vocab[1] = ck_fallback[2];
                        pl.cap[0] = ck_fallback[3];
                        pl.cap[1] = ck_fallback[4];
                        pl.gpool_d = gpool ? reinterpret_cast<double*>(1) : nullptr;
                        pl.gpool_n = gpool ? reinterpret_cast<uint32_t*>(1) : nullptr;
                        FGB_CUDA(cudaMemsetAsync(io.work.get(), 0, sizeof(unsigned int), s));
                        continue;
                    }
                }
                if (pl.timing || pl.stats) {
                    unsigned long long t[kPlainPhCount] = {}, st[2] = {};
                    if (pl.timing) timing.download(t, kPlainPhCount, s);
                    if (pl.stats) stats.download(st, 2, s);
                    FGB_CUDA(cudaStreamSynchronize(s));
                    float ms = 0;
                    FGB_CUDA(cudaEventElapsedTime(&ms, ix->ev0, ix->ev1));
                    if (pl.timing) {
                        const double X = t[kPlainPhExpanded] ? (double)t[kPlainPhExpanded] : 1.0;
                        static const char* names[] = {"seeds", "select", "adjacency+visited", "sparse", "dense",
                                                      "merge", "final"};
                        std::fprintf(stderr, "[plain timing] %llu queries, %.1f expansions/query, %llu warps, %.3f ms\n",
                                     t[kPlainPhQueries], X / std::max(1ull, t[kPlainPhQueries]),
                                     (unsigned long long)slots, ms);
                        for (int k = 0; k < kPlainPhQueries; ++k)
                            std::fprintf(stderr, "  %-18s %10.0f cycles/expansion\n", names[k], t[k] / X);
                        std::fprintf(stderr, "  warps finish between %.3f and %.3f ms after the first start\n",
                                     (t[kPlainPhEndMin] - t[kPlainPhStart]) * 1e-6,
                                     (t[kPlainPhEndMax] - t[kPlainPhStart]) * 1e-6);
                    }
                    if (pl.stats)
                        std::fprintf(stderr, "[plain stats] exact resolutions %llu, exact final entries %llu\n",
                                     st[0], st[1]);
                }
                finish_results(ix, c, q, out, errs, nq, stride, s);
                ht.mark("results");
                ix->last_launches = 1;
                ix->last_kernel = "search_plain_kernel";
                return;
              }
            }
        }

        // ---- geometry
        SearchArgs a{};
        a.c = c.dc;
        a.semantic = ix->semantic.get();
        a.degree = ix->degree;
        a.kw_ptr = ix->kw_ptr.get();
        a.kw_idx = ix->kw_idx.get();
        a.lg_ptr = ix->lg_ptr.get();
        a.lg = ix->lg.get();
        a.kg_ptr = ix->kg_ptr.get();
        a.kg_nbr = ix->kg_nbr.get();
        a.kg_rows = ix->kg_rows;
        a.q = up.dq;
        a.seed_ptr = d_sptr.get();
        a.seed_node = d_snode.get();
        a.seed_ent = d_sent.get();
        a.seed_has = d_shas.get();
        a.norm_order = ix->norm_order.get();
        a.entry_count = norm_seeds;
        a.qflags = d_qflags.get();
        a.conjunctive = conj ? 1 : 0;
        a.lcap = hash_capacity(up.max_lnnz);
        a.scap = hash_capacity(up.max_snnz);
        a.beamcap = std::max(max_beam, 32u);
        a.kcap = std::max(max_k, 1u);
        a.lccap = std::max(ix->max_logical_group, 1u);
        a.nbcap = ix->degree + (any_req ? ix->max_kw_edges : 0) + (any_ctx ? a.lccap : 0) + 32;
        a.reqcap = std::max(max_req, 1u);
        auto al = [](size_t b) { return (b + 15) & ~size_t(15); };
        size_t ws = al(stage_bytes(c.dstride, a.lcap, a.scap));
        ws += al(a.beamcap * 8) + 2 * al(a.kcap * 8) + al(a.nbcap * 8) + al(32 * 8);
        ws += al(a.beamcap * 4) + al(a.kcap * 4) + 2 * al(a.nbcap * 4) + al(a.nbcap);
        ws += al(a.lccap * 8 + 8) + al(a.reqcap * 4 + 4) + al(32 * 4) + 16;
        // staging slot: dense | learned idx | learned val | stat idx | stat val,
        // stride = 4 (mod 32) words so 8 lanes' 16-byte reads hit 32 banks
        a.o_lidx = c.dstride;
        a.o_lval = a.o_lidx + round4(c.max_lnnz);
        a.o_sidx = a.o_lval + round4(c.max_lnnz);
        a.o_sval = a.o_sidx + round4(c.max_snnz);
        a.slot_words = a.o_sval + round4(c.max_snnz);
        while (a.slot_words % 32 != 4) a.slot_words += 4;
        // rows per staging round: the larger of {16, 8, 4} that still lets
        // >= 2 query-warps share an SM (the chain latency is hidden by
        // concurrent queries, the copy latency by wide rounds)
        // Measured on B200 (tools/prof_search.py, 100K docs): the register path
        // (rb = 0: every lane streams its own row with an 8-float4 prefetch) beats
        // TMA staging of 4/8/16 rows per round by 2.8x at beam 256 and 1.7x at
        // beam 2048 — staging slots cost query-warps per SM, and the sequential
        // fp64 chains need those warps to hide their latency.
        a.rb = 0;
        if (const char* e = std::getenv("FGB_SEARCH_RB")) a.rb = static_cast<uint32_t>(std::atoi(e));
        if (a.rb > 32) a.rb = 32;
        ws += al(static_cast<size_t>(a.rb) * a.slot_words * 4);
        a.warp_smem = static_cast<uint32_t>(ws);
        const size_t block_smem = ws * kWarpsPerBlock;
        if (block_smem > 227 * 1024)
            throw Error("beam-too-small", "beam/query too large for the search kernel's shared memory");
        FGB_CUDA(cudaFuncSetAttribute(search_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)block_smem));
        int per_sm = 0, sms = 0;
        FGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, search_kernel,
                                                               kWarpsPerBlock * 32, block_smem));
        FGB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
        per_sm = std::max(per_sm, 1);
        const uint64_t want_blocks = (nq + kWarpsPerBlock - 1) / kWarpsPerBlock;
        const uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>(want_blocks, (uint64_t)sms * per_sm));
        const uint64_t slots = blocks * kWarpsPerBlock;

        // ---- per-warp scratch (reused across calls).  The twin pool and the
        // entity-context table start at 8,192 slots (the context table at
        // least 4x the largest seed set); a query that overflows them is
        // re-run alone with 4x larger tables (up to kMaxScratch), so only a
        // query that still overflows there fails, through its own error.
        a.nwords = (n + 31) / 32;
        a.tcap = 16384;
        uint32_t twcap0 = any_req ? 8192 : 0, ctxcap0 = 0;
        if (any_ctx) {
            ctxcap0 = 8192;
            while (ctxcap0 < 4ull * max_seeds && ctxcap0 < (1u << 26)) ctxcap0 <<= 1;
        }
        if (const char* e = std::getenv("FGB_SEARCH_SCRATCH0")) {  // test hook: force re-runs
            const uint32_t v = static_cast<uint32_t>(std::atoi(e));
            if (v >= 2 && (v & (v - 1)) == 0) {
                if (any_req) twcap0 = v;
                if (any_ctx) ctxcap0 = v;
            }
        }
        float ms_prev = 0.f;
        std::vector<uint32_t> rerun;
        DevBuf<uint32_t> d_rerun;
        DevBuf<unsigned long long> timing;
        const char* te = std::getenv("FGB_SEARCH_TIMING");
        if (te && te[0] == '1') {
            timing.alloc(kPhCount);
            timing.zero(s);
            a.timing = timing.get();
        }
        a.prefetch = 1;
        if (const char* e = std::getenv("FGB_SEARCH_PREFETCH")) a.prefetch = std::atoi(e);
        const uint64_t all_blocks = blocks;
        for (int attempt = 0;; ++attempt) {
        a.twcap = twcap0 << (2 * attempt);
        a.ctxcap = ctxcap0 << (2 * attempt);
        // a re-run needs one query-warp per overflowed query at most
        const uint64_t blocks = attempt ? std::min<uint64_t>(all_blocks, rerun.size()) : all_blocks;
        const uint64_t slots = blocks * kWarpsPerBlock;
        const uint64_t nbitsets = 1 + (any_ctx ? 1 : 0) + (any_req ? 1 : 0);
        const uint64_t bits_words = slots * a.nwords * nbitsets;
        if (W.bits.size() < bits_words) {
            W.bits.alloc(bits_words);
            W.bits.zero(s);
        }
        uint32_t* bits = W.bits.get();
        a.visited = bits;
        a.expbits = any_ctx ? bits + slots * a.nwords : nullptr;
        a.twinbits = any_req ? bits + slots * a.nwords * (any_ctx ? 2 : 1) : nullptr;
        const uint64_t list_words = slots * (a.tcap + a.twcap);
        W.lists.ensure(std::max<uint64_t>(list_words, 1));
        a.touched = W.lists.get();
        a.twin_node = any_req ? a.touched + slots * a.tcap : nullptr;
        const uint64_t misc = slots * (static_cast<uint64_t>(a.twcap) * 8 + static_cast<uint64_t>(a.ctxcap) * 16);
        W.misc.ensure(std::max<uint64_t>(misc, 16));
        a.twin_raw = any_req ? reinterpret_cast<double*>(W.misc.get()) : nullptr;
        a.ctx = any_ctx ? reinterpret_cast<uint4*>(W.misc.get() + slots * a.twcap * 8) : nullptr;
        if (any_ctx) FGB_CUDA(cudaMemsetAsync(a.ctx, 0xFF, slots * a.ctxcap * 16, s));
        a.hit_stride = stride;
        a.r_node = r_node.get();
        a.r_score = r_score.get();
        a.r_count = r_count.get();
        a.r_expanded = r_exp.get();
        a.r_scored = r_sc.get();
        a.r_warn = r_warn.get();
        a.r_err = r_err.get();
        a.work = work.get();
        a.qlist = attempt ? d_rerun.get() : nullptr;
        a.qlist_n = static_cast<uint32_t>(rerun.size());
        if (attempt) FGB_CUDA(cudaMemsetAsync(work.get(), 0, sizeof(unsigned int), s));
        FGB_CUDA(cudaEventRecord(ix->ev0, s));
        if (nq) search_kernel<<<(unsigned)blocks, kWarpsPerBlock * 32, block_smem, s>>>(a);
        FGB_LAUNCH("search_kernel");
        FGB_CUDA(cudaEventRecord(ix->ev1, s));
        ix->last_launches = nq ? attempt + 1 : 0;
        ix->last_kernel = "search_kernel";
        // overflowed queries: re-run them alone with larger scratch
        constexpr uint64_t kMaxScratch = 1ull << 30;  // bytes of twin + context tables per launch
        std::vector<uint32_t> h_err(nq);
        if (nq) r_err.download(h_err.data(), nq, s);
        FGB_CUDA(cudaStreamSynchronize(s));
        rerun.clear();
        for (uint64_t i = 0; i < nq; ++i)
            if (h_err[i]) rerun.push_back(static_cast<uint32_t>(i));
        const uint64_t next_slots = std::min<uint64_t>(all_blocks, rerun.size()) * kWarpsPerBlock;
        const uint64_t next_bytes = next_slots * ((uint64_t(a.twcap) * 12 + uint64_t(a.ctxcap) * 16) << 2);
        if (rerun.empty() || next_bytes > kMaxScratch) break;
        float ms = 0;
        FGB_CUDA(cudaEventElapsedTime(&ms, ix->ev0, ix->ev1));
        ms_prev += ms;
        d_rerun.upload(rerun, s);
        }  // attempts

        finish_results(ix, c, q, out, errs, nq, stride, s, ms_prev);
        if (a.timing) {
            unsigned long long t[kPhCount];
            timing.download(t, kPhCount, s);
            FGB_CUDA(cudaStreamSynchronize(s));
            const double X = t[kPhExpanded] ? (double)t[kPhExpanded] : 1.0;
            static const char* names[] = {"seeds", "select", "adjacency", "dedupe+visited", "score",
                                          "merge", "final"};
            std::fprintf(stderr, "[search timing] %llu queries, %.1f expansions/query, %d warps, %.3f ms\n",
                         t[kPhQueries], X / std::max(1ull, t[kPhQueries]), (int)all_blocks, ix->last_kernel_ms);
            for (int k = 0; k < kPhLaneSparse; ++k)
                std::fprintf(stderr, "  %-15s %10.0f cycles/expansion\n", names[k], t[k] / X);
            std::fprintf(stderr, "  lane: sparse %.0f cycles/node, dense %.0f cycles/node, scored %llu, dense rows %llu\n",
                         t[kPhLaneSparse] / std::max(1.0, (double)t[kPhLaneScored]),
                         t[kPhLaneDense] / std::max(1.0, (double)t[kPhLaneDenseRows]),
                         t[kPhLaneScored], t[kPhLaneDenseRows]);
        }
    });
}

int fg_last_search_kernel(const fg_index* ix, const char** name) {
    return guarded([&] {
        if (!ix || !name) throw Error("invalid-argument", "null pointer");
        *name = ix->last_kernel;
    });
}

int fg_last_search_stats(const fg_index* ix, double* kernel_ms, uint64_t* launches) {
    return guarded([&] {
        if (kernel_ms) *kernel_ms = ix->last_kernel_ms;
        if (launches) *launches = ix->last_launches;
    });
}

}  // extern "C"
