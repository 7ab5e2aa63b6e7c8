// knn.cu — K3: NN-Descent on the GPU (knn_graph.cpp:52-166).
//
// One pass is three device stages, double-buffered like the reference:
//   1. reverse lists: every forward entry (u -> v, score, fresh) is sorted by
//      (target v, score desc, source u asc) with two stable CUB radix sorts,
//      and each target keeps its first k (knn_graph.cpp:78-89);
//   2. one CTA per node u gathers the two-hop pool through forward+reverse
//      lists into a shared-memory hash set (OR-ing path freshness,
//      knn_graph.cpp:94-120), drops u's own list members, and scores every
//      surviving candidate bit-exactly, one thread per candidate, against u
//      staged in shared memory (pair_score, knn_graph.cpp:20-22);
//   3. candidates that beat the running k-th entry merge into a sorted top-k
//      kept in shared memory (better: score desc, id asc); the result and the
//      replaced count are written to the next buffer (knn_graph.cpp:122-141).
#include <cub/cub.cuh>
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "approx_score.cuh"
#include "fg_cuda.hpp"
#include "knn.cuh"
#include "stage_doc.cuh"

namespace fgb {
namespace {

constexpr int kPassThreads = 256;  // two CTAs per SM (launch bound below)
// Candidates scored between two merges grow 1, 2, then kSRounds batches of
// kPassThreads (the first merges raise the screening threshold of a random
// initial list quickly; later rounds amortise the merge's barriers).
constexpr int kSRounds = 4;
constexpr int kSCap = kSRounds * kPassThreads;  // entering candidates buffered per round
constexpr uint32_t kSortMin = 32;  // entering batches above this size certify sorted (default)

// Rejection sampling (knn_graph.cpp:28-36) when 4k < n.
__global__ void knn_sample_kernel(uint64_t n, uint32_t k, uint64_t seed, uint32_t* ids) {
    const uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (u >= n) return;
    DevRng rng(dev_mix_seed(seed, u));
    uint32_t* picks = ids + u * k;
    uint32_t cnt = 0;
    while (cnt < k) {
        const uint32_t cand = static_cast<uint32_t>(dev_bounded(rng, n));
        if (cand == u) continue;
        bool dup = false;
        for (uint32_t j = 0; j < cnt; ++j) dup |= picks[j] == cand;
        if (dup) continue;
        picks[cnt++] = cand;
    }
}

// Scores the k picks of u and sorts them by `better` (knn_graph.cpp:63-72).
__global__ void knn_init_score_kernel(DevCorpus c, uint32_t k, uint32_t* ids, double* scores,
                                      uint8_t* fresh, uint32_t lcap, uint32_t scap) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint64_t u = blockIdx.x;
    SmemQuery sq;
    stage_doc(c, u, smem, lcap, scap, threadIdx.x, blockDim.x, sq, [] { __syncthreads(); });
    double* sc = reinterpret_cast<double*>(smem + doc_stage_bytes(c.dstride, lcap, scap));
    uint32_t* id = reinterpret_cast<uint32_t*>(sc + k);
    for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) {
        id[j] = ids[u * k + j];
        sc[j] = hybrid_score(c, sq, id[j]);
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < k; j += blockDim.x) {
        uint32_t pos = 0;
        for (uint32_t i = 0; i < k; ++i) pos += better(sc[i], id[i], sc[j], id[j]);
        ids[u * k + pos] = id[j];
        scores[u * k + pos] = sc[j];
        fresh[u * k + pos] = 1;
    }
}

__global__ void score_keys_kernel(const double* scores, uint64_t m, uint64_t* keys,
                                  uint32_t* vals) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    keys[i] = order_key(scores[i]);
    vals[i] = static_cast<uint32_t>(i);
}

__global__ void target_keys_kernel(const uint32_t* ids, const uint32_t* order, uint64_t m,
                                   uint32_t* keys, uint32_t* cnt) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint32_t t = ids[order[i]];
    keys[i] = t;
    atomicAdd(&cnt[t], 1u);
}

// R[v] = first min(k, cnt) entries of v's segment (sorted score desc, u asc).
__global__ void reverse_fill_kernel(uint64_t n, uint32_t k, const uint32_t* order,
                                    const uint32_t* cnt, const uint32_t* start,
                                    const uint8_t* fresh, uint32_t* rids, uint8_t* rfresh,
                                    uint32_t* rcnt) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= n * k) return;
    const uint64_t v = t / k;
    const uint32_t j = static_cast<uint32_t>(t % k);
    const uint32_t c = min(cnt[v], k);
    if (j == 0) rcnt[v] = c;
    if (j >= c) return;
    const uint32_t e = order[start[v] + j];
    rids[t] = e / k;
    rfresh[t] = fresh[e];
}

struct PassArgs {
    DevCorpus c;
    uint32_t k;
    const uint32_t* L_ids;
    const double* L_sc;
    const uint8_t* L_fr;
    const uint32_t* R_ids;
    const uint8_t* R_fr;
    const uint32_t* R_cnt;
    uint32_t* N_ids;
    double* N_sc;
    uint8_t* N_fr;
    unsigned long long* changed;
    uint32_t pool_cap;  // power of two
    uint32_t lcap, scap;
    uint64_t lo;        // first node of this launch (vertex-range sharding)
    // certified screening (NQ4 > 0): |approx - exact| <= eps32 * (|u_d| * max_dnorm + |u| * max_norm)
    // + eps64 * |u| * max_norm (search_plain.cu's bound with unit weights)
    double eps32, eps64, max_dnorm, max_norm;
    uint32_t l_vocab;   // learned-path bitmap width (0: hash lookups)
    // dev (FGB_KNN_TIMING=1): thread 0's cycles per phase + counters, summed
    unsigned long long* timing;
    int prefetch;       // L2 prefetch of the postings of the sparse groups after the first
    uint32_t sort_min;  // entering batches larger than this certify sorted
    uint32_t nparts;    // the two-hop pool is processed in nparts hash parts (power of two)
    uint32_t pshift;    // part of id = (id * 0x9E3779B1) >> pshift
    unsigned int* overflow;  // pool overflow counter (0 after a correct pass)
    const uint32_t* order;   // CTA b processes node order[lo + b] (graph locality); nullptr: lo + b
    unsigned long long* counts;  // [0] candidates scored (sum of S_u), [1] dense rows read
    uint32_t ck_cap[2];          // cuckoo variant: table slots per path (power of two >= 4 max nnz)
    unsigned int* ck_fail;       // cuckoo variant: nodes without a table (the host re-runs the pass)
    uint32_t ck_test_fail;       // test hook (FGB_KNN_CUCKOO=2): nodes u % 7 == 3 fail their tables
    // sparse sketch screening (approx_score.cuh sketch_group; nullptr: off)
    const uint4* sketch;
    const unsigned int* sk_gmax;  // bits of the corpus's max |sparse value| (the sketch scale)
    uint32_t sk_off;              // shared-memory byte offset of u's quantised bucket sums
    uint32_t sk_paths;            // bit 0: learned, bit 1: statistical
};

// The sketch scale g_v from the corpus's max |value| (identical in the
// sketch build and in the bound).
__device__ __forceinline__ double sketch_gv(unsigned int gmax_bits) {
    return static_cast<double>(__uint_as_float(gmax_bits)) * 1.001 / 3.0;
}

// Max |value| over the rows of c (both sparse paths; through the per-row
// offsets, so a row view of a larger corpus — the insert path's batch — sees
// exactly its own postings).  Non-negative floats order like their bits.
__global__ void sketch_max_kernel(DevCorpus c, uint32_t paths, unsigned int* out) {
    float mx = 0.f;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t doc = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); doc < c.n; doc += warps)
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            if (!((paths >> p) & 1u)) continue;
            const uint64_t off = p ? c.s_off[doc] : c.l_off[doc];
            const uint32_t nnz = p ? c.s_nnz[doc] : c.l_nnz[doc];
            for (uint32_t j = lane; j < nnz; j += 32) mx = fmaxf(mx, fabsf((p ? c.s_val : c.l_val)[off + j]));
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    if (lane == 0 && mx > 0.f) atomicMax(out, __float_as_uint(mx));
}

// One warp per document: bucket maxima of |value| quantised up to 2 bits,
// q = ceil(|v| / g_v) in 0..3 (so q g_v >= |v|), packed into the document's
// 512-byte row.
__global__ void sketch_build_kernel(DevCorpus c, uint32_t paths, const unsigned int* gmax, uint4* sk) {
    extern __shared__ uint32_t skb[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t doc = blockIdx.x * (uint64_t)(blockDim.x >> 5) + warp;
    if (doc >= c.n) return;  // (warp-uniform; warps never synchronise with each other)
    uint32_t* b = skb + warp * approx::kSketchBuckets;
    for (uint32_t i = lane; i < approx::kSketchBuckets; i += 32) b[i] = 0;
    __syncwarp();
    const double gv = sketch_gv(*gmax);
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        if (!((paths >> p) & 1u) || gv <= 0.0) continue;
        const uint64_t off = p ? c.s_off[doc] : c.l_off[doc];
        const uint32_t nnz = p ? c.s_nnz[doc] : c.l_nnz[doc];
        const uint32_t* idx = p ? c.s_idx : c.l_idx;
        const float* val = p ? c.s_val : c.l_val;
        for (uint32_t j = lane; j < nnz; j += 32) {
            const double x = static_cast<double>(fabsf(val[off + j])) / gv * (1.0 + 1e-12);
            const uint32_t q = static_cast<uint32_t>(fmin(3.0, ceil(x)));
            atomicMax(&b[approx::sketch_bucket(idx[off + j], p)], q);
        }
    }
    __syncwarp();
    uint32_t w[4];  // lane L: buckets 64 L + 16 w + 4 t + i -> word w, byte i, bits 2t
#pragma unroll
    for (int ww = 0; ww < 4; ++ww) {
        uint32_t word = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int i = 0; i < 4; ++i) word |= b[64 * lane + 16 * ww + 4 * t + i] << (8 * i + 2 * t);
        w[ww] = word;
    }
    sk[doc * (approx::kSketchBytes / 16) + lane] = make_uint4(w[0], w[1], w[2], w[3]);
}

// Shared-memory bytes of one path's cuckoo table: keys, values, staged row.
__host__ __device__ __forceinline__ size_t ck_bytes(uint32_t cap) {
    return (static_cast<size_t>(cap) * 8 + static_cast<size_t>(cap / 4) * 8 + 15) & ~size_t(15);
}

enum : int {
    kKnPhInit = 0, kKnPhPool, kKnPhScore, kKnPhMerge, kKnPhExact, kKnPhFinal,  // cycles (thread 0)
    kKnCand, kKnDense, kKnEnter, kKnRounds, kKnResolved, kKnSketch, kKnCount   // counters
};

// Probes are bounded: a full table (a part far above its expected size)
// raises *overflow and the host fails the build loudly instead of spinning.
__device__ __forceinline__ void pool_insert(uint32_t* keys, uint32_t* fbits, uint32_t mask,
                                            uint32_t id, bool fresh, uint32_t cap, unsigned int* overflow) {
    uint32_t s = hslot(id, mask);
    for (uint32_t probe = 0; probe < cap; ++probe) {
        const uint32_t prev = atomicCAS(&keys[s], kEmpty, id);
        if (prev == kEmpty || prev == id) {
            if (fresh) atomicOr(&fbits[s >> 5], 1u << (s & 31));
            return;
        }
        s = (s + 1) & mask;
    }
    atomicAdd(overflow, 1u);
}

// Exact scores (hybrid_score's arithmetic, element order unchanged) of the
// list entries fix[0..n) (bit 31 set: T[index], else S[index]).  The dense
// rows are staged into `rows` (room for `cap` rows of stride dstride + 1
// floats: one thread per row then reads conflict-free) by the whole CTA with
// coalesced 16-B loads; one thread per entry runs the chain from shared
// memory (a chain streamed from global memory waits on ~100 dependent
// stages).  Every thread of the CTA calls it.
template <int NQ4>
__device__ void exact_entries(const PassArgs& a, const SmemQuery& sq, const uint32_t* fix, uint32_t n,
                              unsigned char* area, size_t area_bytes, double* T_sc, uint8_t* T_ex,
                              const uint32_t* T_id, double* S_sc, uint8_t* S_ex, const uint32_t* S_id) {
    const uint32_t tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
    const uint32_t rs = a.c.dstride + 1, n4 = a.c.dstride >> 2;
    // rows + each entry's two sparse-chain results (the dense and the sparse
    // chains of an entry run on different threads)
    const uint32_t sub = nt / 3;  // entries per sub-batch (three chains each)
    const size_t xbytes = static_cast<size_t>(sub) * 16 + 16;
    const uint32_t cap = area_bytes < xbytes ? 0u : static_cast<uint32_t>((area_bytes - xbytes) / (rs * 4ull));
    float* rows = reinterpret_cast<float*>(area);
    double* xsp = reinterpret_cast<double*>(area + ((static_cast<size_t>(cap) * rs * 4 + 15) & ~size_t(15)));
    auto node_of = [&](uint32_t code) { return (code >> 31) ? T_id[code & 0x7FFFFFFFu] : S_id[code]; };
    if (cap == 0) {  // no room for a row (tiny pools): the chain from global memory
        for (uint32_t r = tid; r < n; r += nt) {
            const uint32_t code = fix[r];
            const double acc = hybrid_score<2>(a.c, sq, node_of(code));
            if (code >> 31) {
                T_sc[code & 0x7FFFFFFFu] = acc;
                T_ex[code & 0x7FFFFFFFu] = 1;
            } else {
                S_sc[code] = acc;
                S_ex[code] = 1;
            }
        }
        __syncthreads();
        return;
    }
    // a chunk covers max(cap, sub) entries: the dense rows of the first cap
    // are staged in shared memory, the others' chains stream their rows from
    // L2 (prefetched in bulk first), so all of a chunk's chains run at once
    const uint32_t span = max(cap, sub);
    for (uint32_t b0 = 0; b0 < n; b0 += span) {
        const uint32_t nb = min(span, n - b0);
        const uint32_t staged = min(nb, cap);
        for (uint32_t r = staged + tid; r < nb; r += nt)
            l2_prefetch(a.c.dense + static_cast<uint64_t>(node_of(fix[b0 + r])) * a.c.dstride, a.c.dstride * 4);
        for (uint32_t r = warp; r < staged; r += nwarps) {
            const float4* src =
                reinterpret_cast<const float4*>(a.c.dense + static_cast<uint64_t>(node_of(fix[b0 + r])) * a.c.dstride);
            float4 v[NQ4];
#pragma unroll
            for (int q = 0; q < NQ4; ++q) v[q] = __ldg(src + min(q * 32 + lane, n4 - 1));
#pragma unroll
            for (int q = 0; q < NQ4; ++q) {
                const uint32_t c4 = q * 32 + lane;
                if (c4 < n4) {
                    float* d = rows + r * rs + 4 * c4;
                    d[0] = v[q].x;
                    d[1] = v[q].y;
                    d[2] = v[q].z;
                    d[3] = v[q].w;
                }
            }
        }
        __syncthreads();
        // the three chains of an entry are independent (hybrid_score only
        // adds their results in order): per sub-batch of up to nt/3 entries,
        // thread r runs entry r's dense chain while threads nbs + r and
        // 2 nbs + r run its learned and statistical chains
        for (uint32_t s0 = 0; s0 < nb; s0 += sub) {
            const uint32_t nbs = min(sub, nb - s0);
            if (tid >= nbs && tid < 3 * nbs) {
                const bool lp = tid < 2 * nbs;
                const uint32_t r = s0 + (lp ? tid - nbs : tid - 2 * nbs);
                const uint32_t node = node_of(fix[b0 + r]);
                double x = 0.0;
                if (lp ? sq.lmask != 0 : sq.smask != 0)
                    x = sparse_chain(lp ? a.c.l_idx : a.c.s_idx, lp ? a.c.l_val : a.c.s_val,
                                     lp ? a.c.l_off[node] : a.c.s_off[node], lp ? a.c.l_nnz[node] : a.c.s_nnz[node],
                                     lp ? sq.lkeys : sq.skeys, lp ? sq.lvals : sq.svals, lp ? sq.lmask : sq.smask,
                                     lp ? sq.lfilt : sq.sfilt);
                xsp[2 * (r - s0) + (lp ? 0 : 1)] = x;
            }
            double acc = 0.0;
            if (tid < nbs && s0 + tid < staged) {
                const float* row = rows + (s0 + tid) * rs;
#pragma unroll 8
                for (uint32_t j = 0; j < a.c.dstride; ++j)
                    acc = __dadd_rn(acc, __dmul_rn(sq.dense[j], static_cast<double>(row[j])));
            } else if (tid < nbs) {  // streamed row, 8 x 16 B in flight
                const float4* src = reinterpret_cast<const float4*>(
                    a.c.dense + static_cast<uint64_t>(node_of(fix[b0 + s0 + tid])) * a.c.dstride);
                for (uint32_t j4 = 0; j4 < n4; j4 += 8) {
                    float4 v[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) v[q] = __ldg(src + min(j4 + q, n4 - 1));
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        if (j4 + q < n4) {
                            const uint32_t j = 4 * (j4 + q);
                            acc = __dadd_rn(acc, __dmul_rn(sq.dense[j], static_cast<double>(v[q].x)));
                            acc = __dadd_rn(acc, __dmul_rn(sq.dense[j + 1], static_cast<double>(v[q].y)));
                            acc = __dadd_rn(acc, __dmul_rn(sq.dense[j + 2], static_cast<double>(v[q].z)));
                            acc = __dadd_rn(acc, __dmul_rn(sq.dense[j + 3], static_cast<double>(v[q].w)));
                        }
                }
            }
            __syncthreads();
            if (tid < nbs) {
                const uint32_t code = fix[b0 + s0 + tid];
                acc = __dadd_rn(acc, xsp[2 * tid]);
                acc = __dadd_rn(acc, xsp[2 * tid + 1]);
                if (code >> 31) {
                    T_sc[code & 0x7FFFFFFFu] = acc;
                    T_ex[code & 0x7FFFFFFFu] = 1;
                } else {
                    S_sc[code] = acc;
                    S_ex[code] = 1;
                }
            }
            __syncthreads();
        }
    }
}

// Resolves every entry whose mark is set (mk[0..cnt), tflag = bit 31 for the
// T list) in chunks of at most capf gathered into fixl (the pool's flag
// words: pool_cap / 16 of them, fewer than a round's entries for small pools).
template <int NQ4>
__device__ void resolve_marked(const PassArgs& a, const SmemQuery& sq, uint8_t* mk, uint32_t cnt, uint32_t tflag,
                               uint32_t* fixl, uint32_t capf, uint32_t* counter, unsigned char* area,
                               size_t area_bytes, double* T_sc, uint8_t* T_ex, const uint32_t* T_id, double* S_sc,
                               uint8_t* S_ex, const uint32_t* S_id) {
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    while (true) {
        __syncthreads();  // every thread has read the previous count
        if (tid == 0) *counter = 0;
        __syncthreads();
        for (uint32_t i = tid; i < cnt; i += nt)
            if (mk[i]) {
                const uint32_t slot = atomicAdd(counter, 1u);
                if (slot < capf) {
                    fixl[slot] = tflag | i;
                    mk[i] = 0;
                }
            }
        __syncthreads();
        const uint32_t total = *counter;
        const uint32_t nf = min(total, capf);
        if (nf) exact_entries<NQ4>(a, sq, fixl, nf, area, area_bytes, T_sc, T_ex, T_id, S_sc, S_ex, S_id);
        if (total <= capf) break;
    }
    __syncthreads();
}

// #entries of the sorted list (sc, id)[0, n) that are better than (v, id)
__device__ __forceinline__ uint32_t count_better(const double* sc, const uint32_t* id, uint32_t n, double v,
                                                 uint32_t vid) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (better(sc[mid], id[mid], v, vid))
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// Sorted certification of a round's entering batch S (m > kSortMin) against
// the list T (see the call site).  mrg: >= k + 1 words of scratch holding the
// merged order's first k + 1 entries (bit 31: an S index, else a T index).
template <int NQ4>
__device__ void merge_certify_sorted(const PassArgs& a, const SmemQuery& sq, uint32_t m, uint32_t k, uint32_t n_res,
                                     double eps, uint32_t* keys, uint32_t* fbits, double* T_sc, const uint32_t* T_id,
                                     uint8_t* T_ex, uint8_t* T_mk, double* S_sc, uint32_t* S_id, uint8_t* S_ex,
                                     uint8_t* S_mk, uint32_t* mrg, uint32_t* n_mark) {
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    __shared__ uint32_t any_mark;
    const uint32_t p2 = 1u << (32 - __clz(m - 1));  // m <= kSCap, a power of two
    auto certain = [&](double va, uint8_t ea, double vb, uint8_t eb) {
        return (ea && eb) || fabs(va - vb) > 1.25 * ((ea ? 0.0 : eps) + (eb ? 0.0 : eps));
    };
    auto val = [&](uint32_t e) { return e >> 31 ? S_sc[e & 0x7FFFFFFFu] : T_sc[e]; };
    auto ex = [&](uint32_t e) { return e >> 31 ? S_ex[e & 0x7FFFFFFFu] : T_ex[e]; };
    auto mark = [&](uint32_t e) {
        if (e >> 31) {
            const uint32_t i = e & 0x7FFFFFFFu;
            if (!S_ex[i]) {
                S_mk[i] = 1;
                any_mark = 1;
            }
        } else if (!T_ex[e]) {
            T_mk[e] = 1;
            any_mark = 1;
        }
    };
    while (true) {
        // bitonic sort of S[0, p2) by `better` on the stored values (padding
        // entries are worse than every candidate and sort to the end)
        for (uint32_t i = m + tid; i < p2; i += nt) {
            S_sc[i] = -__longlong_as_double(0x7FF0000000000000LL);
            S_id[i] = 0xFFFFFFFFu;
            S_ex[i] = 1;
        }
        __syncthreads();
        for (uint32_t size = 2; size <= p2; size <<= 1) {
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t i = tid; i < p2; i += nt) {
                    const uint32_t j = i ^ stride;
                    if (j <= i) continue;
                    const bool first = (i & size) == 0;  // this half ends better-first
                    const bool sw = first ? better(S_sc[j], S_id[j], S_sc[i], S_id[i])
                                          : better(S_sc[i], S_id[i], S_sc[j], S_id[j]);
                    if (sw) {
                        const double ts = S_sc[i];
                        S_sc[i] = S_sc[j];
                        S_sc[j] = ts;
                        const uint32_t ti = S_id[i];
                        S_id[i] = S_id[j];
                        S_id[j] = ti;
                        const uint8_t te = S_ex[i];
                        S_ex[i] = S_ex[j];
                        S_ex[j] = te;
                    }
                }
                __syncthreads();
            }
        }
        // merged positions of the first k + 1 entries
        for (uint32_t i = tid; i < m; i += nt) {
            const uint32_t pos = i + count_better(T_sc, T_id, k, S_sc[i], S_id[i]);
            if (pos <= k) mrg[pos] = 0x80000000u | i;
            S_mk[i] = 0;
        }
        for (uint32_t j = tid; j < k; j += nt) {
            const uint32_t pos = j + count_better(S_sc, S_id, m, T_sc[j], T_id[j]);
            if (pos <= k) mrg[pos] = j;
            T_mk[j] = 0;
        }
        if (tid == 0) any_mark = 0;
        __syncthreads();
        // adjacent pairs inside the list: (p, p + 1), p + 1 < k
        for (uint32_t p = tid; p + 1 < k; p += nt) {
            const uint32_t x = mrg[p], y = mrg[p + 1];
            if (!certain(val(x), ex(x), val(y), ex(y))) {
                mark(x);
                mark(y);
            }
        }
        // the k-th entry against every entry merged below it
        const uint32_t b = mrg[k - 1];
        const double bv = val(b);
        const uint8_t be = ex(b);
        for (uint32_t i = tid; i < m; i += nt)
            if (i + count_better(T_sc, T_id, k, S_sc[i], S_id[i]) >= k && !certain(bv, be, S_sc[i], S_ex[i])) {
                mark(b);
                mark(0x80000000u | i);
            }
        for (uint32_t j = tid; j < k; j += nt)
            if (j + count_better(S_sc, S_id, m, T_sc[j], T_id[j]) >= k && !certain(bv, be, T_sc[j], T_ex[j])) {
                mark(b);
                mark(j);
            }
        __syncthreads();
        if (!any_mark) break;
        unsigned char* area = reinterpret_cast<unsigned char*>(keys + ((n_res + 3) & ~3u));
        const size_t area_bytes = static_cast<size_t>(a.pool_cap - ((n_res + 3) & ~3u)) * 4;
        resolve_marked<NQ4>(a, sq, S_mk, m, 0u, fbits, a.pool_cap / 16, n_mark, area, area_bytes, T_sc, T_ex, T_id,
                            S_sc, S_ex, S_id);
        resolve_marked<NQ4>(a, sq, T_mk, k, 0x80000000u, fbits, a.pool_cap / 16, n_mark, area, area_bytes, T_sc,
                            T_ex, T_id, S_sc, S_ex, S_id);
    }
    __syncthreads();
}

constexpr uint32_t kSkFirst = 512;  // candidates moved to the front by sketch_order

// Block-wide exclusive scan of two counters (blockDim.x <= 1024).
__device__ __forceinline__ void block_excl_scan2(uint32_t& x, uint32_t& y, uint32_t* wsum) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t ix = x, iy = y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t tx = __shfl_up_sync(0xFFFFFFFFu, ix, o), ty = __shfl_up_sync(0xFFFFFFFFu, iy, o);
        if (lane >= o) {
            ix += tx;
            iy += ty;
        }
    }
    if (lane == 31) {
        wsum[2 * warp] = ix;
        wsum[2 * warp + 1] = iy;
    }
    __syncthreads();
    uint32_t bx = 0, by = 0;
    for (uint32_t w = 0; w < warp; ++w) {
        bx += wsum[2 * w];
        by += wsum[2 * w + 1];
    }
    __syncthreads();
    x = bx + ix - x;
    y = by + iy - y;
}

// Computes every candidate's sketch bound into bnd[0, n_c) and moves the
// ~kSkFirst highest to the front of keys/bnd (in-place swap partition).
// hist: 256 free words, hpos: kSCap free words.
template <class Args>
__device__ void sketch_order(const Args& a, uint32_t* keys, uint16_t* bnd, uint32_t n_c, double unorm, double eps,
                             double sk_scale, const uint32_t* uq, uint32_t* hist, uint32_t* hpos, uint32_t lane) {
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    for (uint32_t b2 = 0; b2 < n_c; b2 += nt) {
        const uint32_t s = b2 + tid;
        const bool cand = s < n_c;  // (a prefix of each warp)
        const uint32_t cn = cand ? keys[s] : 0u;
        const uint32_t F = __popc(__ballot_sync(approx::kFull, cand));
        if (!F) continue;  // warp-uniform
        const uint4 mt = cand ? __ldg(a.c.meta + cn) : make_uint4(0, 0, 0, 0);
        const uint32_t sb = approx::sketch_group(a.sketch, uq, cn, lane, F);
        if (cand) {
            const double b = score_upper_bound(unorm, (double)__uint_as_float(mt.w), static_cast<double>(sb) * sk_scale,
                                               0.0) + 2.0 * eps;
            bnd[s] = __bfloat16_as_ushort(__float2bfloat16_ru(__double2float_ru(b)));
        }
    }
    if (n_c <= kSkFirst) {
        __syncthreads();
        return;
    }
    // radix select of the kSkFirst-th largest key (bf16 bits of non-negative
    // values order as integers): high byte, then low byte within its bin
    __shared__ uint32_t sel_hi, sel_above, sel_t, sel_m1, sel_ws[64];
    for (uint32_t i = tid; i < 256; i += nt) hist[i] = 0;
    __syncthreads();
    for (uint32_t s = tid; s < n_c; s += nt) atomicAdd(&hist[bnd[s] >> 8], 1u);
    __syncthreads();
    if (tid == 0) {
        uint32_t acc = 0, b = 255;
        while (b > 0 && acc + hist[b] < kSkFirst) acc += hist[b--];
        sel_hi = b;
        sel_above = acc;
    }
    __syncthreads();
    const uint32_t hi = sel_hi;
    for (uint32_t i = tid; i < 256; i += nt) hist[i] = 0;
    __syncthreads();
    for (uint32_t s = tid; s < n_c; s += nt)
        if ((bnd[s] >> 8) == hi) atomicAdd(&hist[bnd[s] & 0xFFu], 1u);
    __syncthreads();
    if (tid == 0) {
        uint32_t acc = sel_above, b = 255;
        while (b > 0 && acc + hist[b] < kSkFirst) acc += hist[b--];
        sel_t = (hi << 8) | b;
        sel_m1 = 0;
    }
    __syncthreads();
    const uint32_t T = sel_t;
    uint32_t m1c = 0;
    for (uint32_t s = tid; s < n_c; s += nt) m1c += bnd[s] >= T;
    m1c = __reduce_add_sync(0xFFFFFFFFu, m1c);
    if (lane == 0 && m1c) atomicAdd(&sel_m1, m1c);
    __syncthreads();
    const uint32_t m1 = sel_m1;
    if (m1 > kSCap) return;  // (ties at the threshold: stays unordered; CTA-uniform)
    // swap the r-th misplaced low (position < m1, key < T) with the r-th
    // misplaced high (position >= m1, key >= T); contiguous chunks per thread
    const uint32_t chunk = (n_c + nt - 1) / nt;
    const uint32_t c0 = min(n_c, tid * chunk), c1 = min(n_c, c0 + chunk);
    uint32_t nh = 0, nl = 0;
    for (uint32_t s = c0; s < c1; ++s) {
        const bool h = bnd[s] >= T;
        nh += h && s >= m1;
        nl += !h && s < m1;
    }
    block_excl_scan2(nh, nl, sel_ws);
    for (uint32_t s = c0; s < c1; ++s)
        if (s >= m1 && bnd[s] >= T) hpos[nh++] = s;
    __syncthreads();
    for (uint32_t s = c0; s < c1; ++s)
        if (s < m1 && bnd[s] < T) {
            const uint32_t hp = hpos[nl++];
            const uint32_t tk = keys[s];
            keys[s] = keys[hp];
            keys[hp] = tk;
            const uint16_t tb = bnd[s];
            bnd[s] = bnd[hp];
            bnd[hp] = tb;
        }
    __syncthreads();
}

// One NN-Descent pass for node u = lo + blockIdx.x.  NQ4 > 0: candidates
// are scored warp-cooperatively (coalesced rows, approx_score.cuh) and
// rejected when certified worse than the running k-th entry; only the rest
// get the exact chain.  NQ4 == 0 (dense rows > 1,024 floats): exact chains,
// thread per candidate.
template <int NQ4, bool kCk>
__global__ void __launch_bounds__(kPassThreads, 2) knn_pass_kernel(PassArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t k = a.k;
    const uint64_t u = a.order ? a.order[a.lo + blockIdx.x] : a.lo + blockIdx.x;
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    SmemQuery sq;
    unsigned char* p = smem + ((doc_stage_bytes(a.c.dstride, a.lcap, a.scap) + 15) & ~size_t(15));
    uint32_t* keys = reinterpret_cast<uint32_t*>(p);
    uint32_t* fbits = keys + a.pool_cap;
    uint32_t* hbits = fbits + a.pool_cap / 32;  // "already in L[u]"
    double* T_sc = reinterpret_cast<double*>(hbits + a.pool_cap / 32);
    double* T2_sc = T_sc + k;
    double* S_sc = T2_sc + k;
    uint32_t* T_id = reinterpret_cast<uint32_t*>(S_sc + kSCap);
    uint32_t* T2_id = T_id + k;
    uint32_t* S_id = T2_id + k;
    uint8_t* T_new = reinterpret_cast<uint8_t*>(S_id + kSCap);
    uint8_t* T2_new = T_new + k;
    // exactness of the stored scores (1: the reference's exact value, 0: the
    // certified approximation +- eps) and resolution marks
    uint8_t* T_ex = T2_new + k;
    uint8_t* T2_ex = T_ex + k;
    uint8_t* S_ex = T2_ex + k;
    uint8_t* T_mk = S_ex + kSCap;
    uint8_t* S_mk = T_mk + k;
    __shared__ uint32_t S_cnt, n_mark, t_marked;
    long long t_mark = (a.timing && threadIdx.x == 0) ? clock64() : 0;
    auto lap = [&](int ph) {
        if (a.timing && threadIdx.x == 0) {
            const long long t = clock64();
            atomicAdd(&a.timing[ph], static_cast<unsigned long long>(t - t_mark));
            t_mark = t;
        }
    };
    auto count = [&](int slot, uint32_t v) {
        if (a.timing && v) atomicAdd(&a.timing[slot], static_cast<unsigned long long>(v));
    };
    uint32_t cand_total = 0, dense_rows = 0;  // (thread 0 / lane 0 of each warp)
    uint32_t sk_total = 0, sk_rej = 0;        // candidates sketched (thread 0) / rejected by it (lane 0)

    for (uint32_t j = tid; j < k; j += nt) {
        T_id[j] = a.L_ids[u * k + j];
        T_sc[j] = a.L_sc[u * k + j];
        T_new[j] = 0;
        T_ex[j] = 1;
    }
    if (tid == 0) S_cnt = 0;
    stage_doc(a.c, u, smem, a.lcap, a.scap, tid, nt, sq, [] { __syncthreads(); });
    lap(kKnPhInit);

    // Score fresh, new candidates; merge survivors into the running top-k.
    const double unorm = a.c.dnorm[u];
    // u's dense row in fp32 (approximate path), after the flag arrays
    float* qd = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(S_mk + kSCap) + 15) & ~uintptr_t(15));
    approx::PathQ P[2];
    double eps = 0.0;
    double sk_scale = 0.0;  // g_u g_v (sketch screening)
    if constexpr (NQ4 > 0) {
        for (uint32_t j = tid; j < a.c.dstride; j += nt) qd[j] = a.c.dense[u * a.c.dstride + j];
        for (int p = 0; p < 2; ++p) {
            P[p].on = p == 0 ? sq.lmask != 0 : sq.smask != 0;
            P[p].vocab = 0;  // hash lookups on the staged row
            P[p].keys = p == 0 ? sq.lkeys : sq.skeys;
            P[p].vals = p == 0 ? sq.lvals : sq.svals;
            P[p].filt = p == 0 ? sq.lfilt : sq.sfilt;
            P[p].mask = p == 0 ? sq.lmask : sq.smask;
        }
        if constexpr (kCk) {
            // u's sparse rows as two-choice cuckoo tables (exactly two probes
            // per lookup): warp 0 builds, the others read the multipliers
            __shared__ uint32_t ck_hm[2][2];
            unsigned char* ckm = reinterpret_cast<unsigned char*>(qd + a.c.dstride);
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                const uint32_t cap = a.ck_cap[p];
                uint32_t* ck = reinterpret_cast<uint32_t*>(ckm + (p ? ck_bytes(a.ck_cap[0]) : 0));
                float* cv = reinterpret_cast<float*>(ck + cap);
                P[p].vocab = 0;
                P[p].keys = ck;
                P[p].vals = cv;
                P[p].mask = cap - 1;
                P[p].hshift = 32u - static_cast<uint32_t>(__ffs(cap) - 1);
                if (!cap) continue;  // (the learned path on its bitmap)
                if (tid < 32 && P[p].on) {
                    uint32_t* tk = reinterpret_cast<uint32_t*>(cv + cap);
                    float* tv = reinterpret_cast<float*>(tk + cap / 4);
                    const uint64_t ro = p ? a.c.s_off[u] : a.c.l_off[u];
                    const uint32_t rn = p ? a.c.s_nnz[u] : a.c.l_nnz[u];
                    for (uint32_t j = tid; j < rn; j += 32) {
                        tk[j] = (p ? a.c.s_idx : a.c.l_idx)[ro + j];
                        tv[j] = (p ? a.c.s_val : a.c.l_val)[ro + j];
                    }
                    approx::cuckoo_fill(P[p], ck, cv, tk, tv, rn, cap, tid);
                    if (tid == 0) {
                        ck_hm[p][0] = P[p].hm1;
                        ck_hm[p][1] = P[p].hm2;
                    }
                }
            }
            __syncthreads();
            bool bad = a.ck_test_fail && u % 7 == 3;
#pragma unroll
            for (int p = 0; p < 2; ++p)
                if (P[p].on && a.ck_cap[p]) {
                    P[p].hm1 = ck_hm[p][0];
                    P[p].hm2 = ck_hm[p][1];
                    bad |= P[p].hm1 == 0;
                }
            if (bad) {  // (uniform over the CTA) nothing of u is written; the host re-runs the pass
                if (tid == 0) atomicAdd(a.ck_fail, 1u);
                return;
            }
        }
        if (a.l_vocab && P[0].on) {
            // learned path of u as a bitmap + rank structure (branch-free lookups)
            const uint32_t W = approx::bitmap_words(a.l_vocab);
            uint32_t* bm = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(qd + a.c.dstride) +
                                                       (kCk ? ck_bytes(a.ck_cap[0]) + ck_bytes(a.ck_cap[1]) : 0));
            uint16_t* pre = reinterpret_cast<uint16_t*>(bm + ((W + 3) & ~3u));
            float* qv = reinterpret_cast<float*>(pre + ((W + 7) & ~7u));
            const uint64_t lo = a.c.l_off[u];
            const uint32_t ln = a.c.l_nnz[u];
            const uint32_t* ui = a.c.l_idx + lo;
            for (uint32_t w = tid; w < W; w += nt) bm[w] = 0;
            __syncthreads();
            for (uint32_t j = tid; j < ln; j += nt) {
                const uint32_t t = ui[j];
                atomicOr(&bm[t >> 5], 1u << (t & 31));
                qv[j] = a.c.l_val[lo + j];  // u's row is ascending: rank = position
            }
            for (uint32_t w = tid; w < W; w += nt) {  // #terms < 32 w (lower bound in the sorted row)
                uint32_t b = 0, e = ln;
                while (b < e) {
                    const uint32_t mid = (b + e) >> 1;
                    if (ui[mid] < 32 * w)
                        b = mid + 1;
                    else
                        e = mid;
                }
                pre[w] = static_cast<uint16_t>(b);
            }
            P[0].vocab = a.l_vocab;
            P[0].wm1 = W - 1;
            P[0].bm = bm;
            P[0].pre = pre;
            P[0].qv = qv;
        }
        if (a.sketch) {
            // u's bucket sums U_b = sum |u_t| (fp32, pool table as scratch:
            // it is initialised per part below), quantised up to bytes with
            // g_u = max U_b * 1.001 / 255: uq_b g_u >= 1.0001 U_b (1 +- 1e-7)
            // covers the fp32 sums' rounding (<= 240 terms: 1.5e-5)
            __shared__ unsigned int sk_max;
            float* ub = reinterpret_cast<float*>(keys);
            for (uint32_t j = tid; j < approx::kSketchBuckets; j += nt) ub[j] = 0.f;
            if (tid == 0) sk_max = 0;
            __syncthreads();
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                if (!((a.sk_paths >> p) & 1u)) continue;
                const uint64_t off = p ? a.c.s_off[u] : a.c.l_off[u];
                const uint32_t nnz = p ? a.c.s_nnz[u] : a.c.l_nnz[u];
                for (uint32_t j = tid; j < nnz; j += nt)
                    atomicAdd(&ub[approx::sketch_bucket((p ? a.c.s_idx : a.c.l_idx)[off + j], p)],
                              fabsf((p ? a.c.s_val : a.c.l_val)[off + j]));
            }
            __syncthreads();
            float mx = 0.f;
            for (uint32_t j = tid; j < approx::kSketchBuckets; j += nt) mx = fmaxf(mx, ub[j]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
            if ((tid & 31) == 0 && mx > 0.f) atomicMax(&sk_max, __float_as_uint(mx));
            __syncthreads();
            const float gu = __uint_as_float(sk_max) * 1.001f / 255.f;
            uint32_t* uqw = reinterpret_cast<uint32_t*>(smem + a.sk_off);
            for (uint32_t w = tid; w < approx::kSketchBuckets / 4; w += nt) {
                uint32_t word = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t q = gu > 0.f ? min(255u, static_cast<uint32_t>(ceilf(ub[4 * w + i] * 1.0001f / gu))) : 0u;
                    word |= q << (8 * i);
                }
                uqw[w] = word;
            }
            sk_scale = static_cast<double>(gu) * sketch_gv(*a.sk_gmax) * (1.0 + 1e-12);
        }
        eps = a.eps32 * unorm * (1.0 + 1e-10) * a.max_dnorm +
              a.eps32 * sqrt(a.c.sqnorm[u]) * (1.0 + 1e-10) * a.max_norm +  // fp32 sparse products
              a.eps64 * sqrt(a.c.sqnorm[u]) * (1.0 + 1e-10) * a.max_norm + 1e-300;
        __syncthreads();
    }
    const uint32_t lane = tid & 31;
    // two stored scores decide their order (both exact, or apart by more than
    // both error bounds; 1.25x margin for the subtraction's own rounding)
    auto certain = [&](double va, uint8_t ea, double vb, uint8_t eb) {
        return (ea && eb) || fabs(va - vb) > 1.25 * ((ea ? 0.0 : eps) + (eb ? 0.0 : eps));
    };
    // The two-hop pool is built and scored in `nparts` parts: candidate ids
    // are split by a multiplicative hash, so each part's set fits a pool of
    // pool_cap slots (<= 16K: two CTAs share an SM and overlap each other's
    // barrier waits).  The result is the top-k of the union either way.
    const uint32_t mask = a.pool_cap - 1;
    auto part_of = [&](uint32_t id) { return a.nparts == 1 ? 0u : (id * 0x9E3779B1u) >> a.pshift; };
    for (uint32_t part = 0; part < a.nparts; ++part) {
    for (uint32_t j = tid; j < a.pool_cap; j += nt) keys[j] = kEmpty;
    for (uint32_t j = tid; j < a.pool_cap / 32; j += nt) {
        fbits[j] = 0;
        hbits[j] = 0;
    }
    __syncthreads();
    // L[u] members of this part: mark as "have" (their scores are known;
    // knn_graph.cpp:122-131 — the snapshot list, not the evolving one)
    for (uint32_t j = tid; j < k; j += nt) {
        const uint32_t id = a.L_ids[u * k + j];
        if (part_of(id) != part) continue;
        uint32_t s = hslot(id, mask);
        for (uint32_t probe = 0; probe < a.pool_cap; ++probe) {
            const uint32_t prev = atomicCAS(&keys[s], kEmpty, id);
            if (prev == kEmpty || prev == id) break;
            s = (s + 1) & mask;
        }
        atomicOr(&hbits[s >> 5], 1u << (s & 31));
    }
    __syncthreads();
    // Two-hop pool through forward + reverse adjacency (knn_graph.cpp:97-110).
    // u's first hops (forward list, then reverse list) are staged in shared
    // memory (the candidate buffers are free until scoring); each thread then
    // has kHopU second-hop loads in flight before its inserts (the pool is a
    // set with OR-ed freshness, so insertion order does not matter).
    const uint32_t rc_u = a.R_cnt[u];
    const uint32_t nh1 = k + rc_u;
    uint32_t* hop_id = S_id;
    uint32_t* hop_rc = reinterpret_cast<uint32_t*>(S_sc);
    uint8_t* hop_fr = S_ex;
    for (uint32_t h = tid; h < nh1; h += nt) {
        const uint32_t h1 = h < k ? a.L_ids[u * k + h] : a.R_ids[u * k + (h - k)];
        hop_id[h] = h1;
        hop_fr[h] = h < k ? a.L_fr[u * k + h] : a.R_fr[u * k + (h - k)];
        hop_rc[h] = a.R_cnt[h1];
    }
    __syncthreads();
    const uint32_t items = nh1 * (2 * k);
    constexpr uint32_t kHopU = 4;
    for (uint32_t it0 = tid; it0 < items; it0 += nt * kHopU) {
        uint32_t h2[kHopU];
        uint8_t f2[kHopU];
        bool ok[kHopU], f1[kHopU];
#pragma unroll
        for (uint32_t q = 0; q < kHopU; ++q) {
            const uint32_t it = min(it0 + q * nt, items - 1);
            const uint32_t h = it / (2 * k), j = it % (2 * k);
            const uint64_t h1 = hop_id[h];
            const bool fwd = j < k;
            const uint32_t jj = fwd ? j : j - k;
            ok[q] = it0 + q * nt < items && (fwd || jj < hop_rc[h]);
            f1[q] = hop_fr[h];
            // (unconditional loads: jj < k stays inside h1's row)
            h2[q] = fwd ? a.L_ids[h1 * k + jj] : a.R_ids[h1 * k + jj];
            f2[q] = fwd ? a.L_fr[h1 * k + jj] : a.R_fr[h1 * k + jj];
        }
#pragma unroll
        for (uint32_t q = 0; q < kHopU; ++q)
            if (ok[q] && h2[q] != u && part_of(h2[q]) == part)
                pool_insert(keys, fbits, mask, h2[q], f1[q] || f2[q], a.pool_cap, a.overflow);
    }
    __syncthreads();
    lap(kKnPhPool);

    // compact the candidates (fresh, not already in L[u]) to the front of
    // keys[]: the scoring rounds then cover only real candidates (late passes
    // have ~100 in a 32K-slot table, and every round costs a memory round
    // trip).  In place: a chunk's reads finish before its writes, and writes
    // land below the slots read so far.  The result does not depend on the
    // order candidates are scored in (the top-k of a set).
    __shared__ uint32_t n_cand;
    if (tid == 0) n_cand = 0;
    __syncthreads();
    for (uint32_t base = 0; base < a.pool_cap; base += nt) {  // pool_cap: a power of two >= nt
        const uint32_t s = base + tid;
        const uint32_t id = keys[s];
        const bool cand = id != kEmpty && ((fbits[s >> 5] >> (s & 31)) & 1u) &&
                          !((hbits[s >> 5] >> (s & 31)) & 1u);
        const uint32_t cm = __ballot_sync(0xFFFFFFFFu, cand);
        uint32_t wb = 0;
        if (lane == 0 && cm) wb = atomicAdd(&n_cand, static_cast<uint32_t>(__popc(cm)));
        wb = __shfl_sync(0xFFFFFFFFu, wb, 0);
        __syncthreads();
        if (cand) keys[wb + __popc(cm & ((1u << lane) - 1u))] = id;
    }
    __syncthreads();
    const uint32_t n_c = n_cand;
    cand_total += n_c;
    if (a.sketch) sk_total += n_c;
    // Sketch ORDER (NQ4 > 0 with sketches, when the pool has room): every
    // candidate's sketch bound is computed first and stored (bf16 rounded
    // up, above the compacted list); the ~kSkFirst candidates with the
    // highest bounds are swapped to the front, so the first round's exact
    // scores lift the k-th entry close to its final value and the others
    // are screened against it by their stored bounds.  (The result is the
    // top-k of the set either way; only the work changes.)
    uint16_t* bnd = nullptr;
    uint32_t n_res = n_c;  // words of keys[] in use (resolutions stage rows above them)
    if constexpr (NQ4 > 0) {
        const uint32_t nc_al = (n_c + 1) & ~1u;
        if (a.sketch && n_c > 0 && ((nc_al + nc_al / 2 + 3) & ~3u) <= a.pool_cap) {
            bnd = reinterpret_cast<uint16_t*>(keys + nc_al);
            n_res = nc_al + nc_al / 2;
            sketch_order(a, keys, bnd, n_c, unorm, eps, sk_scale, reinterpret_cast<const uint32_t*>(smem + a.sk_off),
                         reinterpret_cast<uint32_t*>(S_sc), S_id, lane);
        }
    }
    uint32_t round = 0;
    for (uint32_t base = 0; base < n_c; ++round) {
      const uint32_t grow = part > 0 ? uint32_t(kSRounds) : round == 0 ? 1u : round == 1 ? 2u : uint32_t(kSRounds);
      const uint32_t end = min(n_c, base + grow * nt);
      for (uint32_t b2 = base; b2 < end; b2 += nt) {
        const uint32_t s = b2 + tid;
        const bool cand = s < end;
        const uint32_t id = cand ? keys[s] : kEmpty;
        const double tau = T_sc[k - 1];
        const uint32_t tau_id = T_id[k - 1];
        if constexpr (NQ4 > 0) {
            // the k-th entry's value is exact or within eps: a candidate whose
            // approximation is below it by more than both bounds never enters
            const double tau_lo = tau - (T_ex[k - 1] ? 0.0 : eps);
            // stored sketch bounds (+ |u||v| + 2 eps, rounded up) screen first
            const bool live = cand && !(bnd && static_cast<double>(__bfloat162float(
                                                   __ushort_as_bfloat16(bnd[s]))) < tau_lo);
            if ((a.timing || a.counts) && bnd) {
                const uint32_t rej = __popc(__ballot_sync(approx::kFull, cand && !live));
                if (lane == 0) {
                    count(kKnSketch, rej);
                    sk_rej += rej;
                }
            }
            const uint32_t fm = __ballot_sync(approx::kFull, live);
            uint32_t F = __popc(fm);
            const uint32_t src = __fns(fm, 0, lane + 1);
            uint32_t cn = __shfl_sync(approx::kFull, id, src < 32 ? src : 0);
            bool mine = lane < F;
            uint4 mt = mine ? __ldg(a.c.meta + cn) : make_uint4(0, 0, 0, 0);
            if (a.sketch && !bnd && F) {  // warp-uniform
                // sketch screening: candidates whose sparse bound + |u||v| is
                // certified below the k-th never load their postings
                const uint32_t sb = approx::sketch_group(a.sketch, reinterpret_cast<const uint32_t*>(smem + a.sk_off),
                                                         cn, lane, F);
                const bool pass = mine && !(score_upper_bound(unorm, (double)__uint_as_float(mt.w),
                                                              static_cast<double>(sb) * sk_scale, 0.0) +
                                                2.0 * eps < tau_lo);
                const uint32_t pm = __ballot_sync(approx::kFull, pass);
                if (lane == 0) {
                    count(kKnSketch, F - __popc(pm));
                    sk_rej += F - __popc(pm);
                }
                const uint32_t s2 = __fns(pm, 0, lane + 1);
                const uint32_t sl = s2 < 32 ? s2 : 0;
                cn = __shfl_sync(approx::kFull, cn, sl);
                mt.x = __shfl_sync(approx::kFull, mt.x, sl);
                mt.y = __shfl_sync(approx::kFull, mt.y, sl);
                mt.z = __shfl_sync(approx::kFull, mt.z, sl);
                mt.w = __shfl_sync(approx::kFull, mt.w, sl);
                F = __popc(pm);
                mine = lane < F;
            }
            if (F) {  // warp-uniform
                if (a.prefetch && mine && lane >= approx::kSG) {
#pragma unroll
                    for (int pth = 0; pth < 2; ++pth) {
                        const uint32_t nz = pth ? (mt.z >> 16) : (mt.z & 0xFFFFu);
                        if (P[pth].on && nz) {
                            const uint64_t o = 4ull * (pth ? mt.y : mt.x);
                            l2_prefetch((pth ? a.c.s_idx : a.c.l_idx) + o, ((nz + 3) & ~3u) * 4);
                            l2_prefetch((pth ? a.c.s_val : a.c.l_val) + o, ((nz + 3) & ~3u) * 4);
                        }
                    }
                }
                double L = 0.0, S = 0.0;
                if constexpr (kCk) {  // learned: bitmap or cuckoo; statistical: cuckoo
                    if (P[0].on)
                        L = P[0].vocab ? approx::sparse_group<true, true>(a.c.l_idx, a.c.l_val, P[0], mt.x,
                                                                          mt.z & 0xFFFFu, lane, F)
                                       : approx::sparse_group<approx::kLookCuckoo, true>(a.c.l_idx, a.c.l_val, P[0],
                                                                                         mt.x, mt.z & 0xFFFFu, lane, F);
                    if (P[1].on)
                        S = approx::sparse_group<approx::kLookCuckoo, true>(a.c.s_idx, a.c.s_val, P[1], mt.y,
                                                                            mt.z >> 16, lane, F);
                } else {
                    if (P[0].on)
                        L = P[0].vocab ? approx::sparse_group<true, true>(a.c.l_idx, a.c.l_val, P[0], mt.x, mt.z & 0xFFFFu, lane, F)
                                       : approx::sparse_group<false, true>(a.c.l_idx, a.c.l_val, P[0], mt.x, mt.z & 0xFFFFu, lane, F);
                    if (P[1].on) S = approx::sparse_group<false, true>(a.c.s_idx, a.c.s_val, P[1], mt.y, mt.z >> 16, lane, F);
                }
                // screening: the exact score is <= the bound (+ the approximation error)
                bool keep = mine && !(score_upper_bound(unorm, (double)__uint_as_float(mt.w), L, S) + 2.0 * eps < tau_lo);
                const uint32_t km = __ballot_sync(approx::kFull, keep);
                if (lane == 0) {
                    count(kKnCand, F);
                    count(kKnDense, __popc(km));
                    dense_rows += __popc(km);
                }
                const double D = approx::dense_group<NQ4, 2>(a.c, qd, cn, lane, km);
                const double v = __dadd_rn(__dadd_rn(D, L), S);
                if (keep && !(v + eps < tau_lo)) {  // may enter: kept with its approximation
                    const uint32_t slot = atomicAdd(&S_cnt, 1u);
                    S_sc[slot] = v;
                    S_id[slot] = cn;
                    S_ex[slot] = 0;
                }
            }
        } else {
            double sc;
            // screened: candidates whose exact-score upper bound (sparse parts +
            // |u||v|) is below the running k-th score never read their dense row
            if (cand && hybrid_score_screened(a.c, sq, id, unorm, tau, sc)) {
                if (better(sc, id, tau, tau_id)) {
                    const uint32_t slot = atomicAdd(&S_cnt, 1u);
                    S_sc[slot] = sc;
                    S_id[slot] = id;
                    S_ex[slot] = 1;
                }
            }
        }
      }
        base = end;
        __syncthreads();
        const uint32_t m = S_cnt;
        __syncthreads();  // everyone holds m before S_cnt can change again
        lap(kKnPhScore);
        if (tid == 0) {
            count(kKnEnter, m);
            count(kKnRounds, 1);
        }
        if (m == 0) continue;
        bool sorted = false;
        if constexpr (NQ4 > 0) {
            if (m > a.sort_min) {
                // Large batches: sort S by its stored values, then certify
                // only what the new top-k depends on — adjacent pairs of the
                // merged order inside positions [0, k) (certified adjacent
                // orders compose transitively into the true order) and the
                // k-th entry against every entry merged below it.  O(m log^2 m
                // + k) instead of O(m (k + m)), and pairs that both fall out
                // of the list are never resolved.  Loops until nothing is
                // uncertain (every round resolves at least one approximation).
                sorted = true;
                merge_certify_sorted<NQ4>(a, sq, m, k, n_res, eps, keys, fbits, T_sc, T_id, T_ex, T_mk, S_sc, S_id,
                                          S_ex, S_mk, reinterpret_cast<uint32_t*>(T2_sc), &n_mark);
            }
        }
        if constexpr (NQ4 > 0) if (!sorted) {
            // certify every comparison the rank-merge makes (S x T, S x S);
            // uncertain entries get the reference's exact score, until none is
            while (true) {
                for (uint32_t i = tid; i < m; i += nt) S_mk[i] = 0;
                for (uint32_t i = tid; i < k; i += nt) T_mk[i] = 0;
                if (tid == 0) {
                    n_mark = 0;
                    t_marked = 0;
                }
                __syncthreads();
                for (uint32_t i = tid; i < m; i += nt) {
                    bool mk = false;
                    for (uint32_t q = 0; q < k; ++q)
                        if (!certain(S_sc[i], S_ex[i], T_sc[q], T_ex[q])) {
                            mk = true;
                            if (!T_ex[q]) {
                                T_mk[q] = 1;
                                t_marked = 1;
                            }
                        }
                    for (uint32_t q = 0; q < m; ++q)
                        if (q != i && !certain(S_sc[i], S_ex[i], S_sc[q], S_ex[q])) mk = true;
                    if (mk && !S_ex[i]) {
                        S_mk[i] = 1;
                        atomicAdd(&n_mark, 1u);
                    }
                }
                __syncthreads();
                if (n_mark == 0 && t_marked == 0) break;
                if (tid == 0) count(kKnResolved, n_mark + t_marked);
                // resolve through rows staged above the compacted candidate
                // list (the pool's upper part and its flag words are free)
                unsigned char* area = reinterpret_cast<unsigned char*>(keys + ((n_res + 3) & ~3u));
                const size_t area_bytes = static_cast<size_t>(a.pool_cap - ((n_res + 3) & ~3u)) * 4;
                resolve_marked<NQ4>(a, sq, S_mk, m, 0u, fbits, a.pool_cap / 16, &n_mark, area, area_bytes, T_sc,
                                    T_ex, T_id, S_sc, S_ex, S_id);
                resolve_marked<NQ4>(a, sq, T_mk, k, 0x80000000u, fbits, a.pool_cap / 16, &n_mark, area, area_bytes,
                                    T_sc, T_ex, T_id, S_sc, S_ex, S_id);
            }
        }
        if (sorted) {
            // both sorted: positions by binary search (ids are pairwise distinct)
            for (uint32_t i = tid; i < k; i += nt) {
                const uint32_t pos = i + count_better(S_sc, S_id, m, T_sc[i], T_id[i]);
                if (pos < k) {
                    T2_sc[pos] = T_sc[i];
                    T2_id[pos] = T_id[i];
                    T2_new[pos] = T_new[i];
                    T2_ex[pos] = T_ex[i];
                }
            }
            for (uint32_t i = tid; i < min(m, k); i += nt) {
                const uint32_t pos = i + count_better(T_sc, T_id, k, S_sc[i], S_id[i]);
                if (pos < k) {
                    T2_sc[pos] = S_sc[i];
                    T2_id[pos] = S_id[i];
                    T2_new[pos] = 1;
                    T2_ex[pos] = S_ex[i];
                }
            }
        } else {
        // rank-merge T (sorted) with S (unsorted); ids are pairwise distinct
        for (uint32_t i = tid; i < k; i += nt) {
            uint32_t pos = i;
            for (uint32_t q = 0; q < m; ++q) pos += better(S_sc[q], S_id[q], T_sc[i], T_id[i]);
            if (pos < k) {
                T2_sc[pos] = T_sc[i];
                T2_id[pos] = T_id[i];
                T2_new[pos] = T_new[i];
                T2_ex[pos] = T_ex[i];
            }
        }
        for (uint32_t i = tid; i < m; i += nt) {
            uint32_t pos = 0;
            for (uint32_t q = 0; q < m; ++q) pos += better(S_sc[q], S_id[q], S_sc[i], S_id[i]);
            uint32_t lo = 0, hi = k;  // #T entries better than S[i]
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (better(T_sc[mid], T_id[mid], S_sc[i], S_id[i]))
                    lo = mid + 1;
                else
                    hi = mid;
            }
            pos += lo;
            if (pos < k) {
                T2_sc[pos] = S_sc[i];
                T2_id[pos] = S_id[i];
                T2_new[pos] = 1;
                T2_ex[pos] = S_ex[i];
            }
        }
        }
        __syncthreads();
        for (uint32_t i = tid; i < k; i += nt) {
            T_sc[i] = T2_sc[i];
            T_id[i] = T2_id[i];
            T_new[i] = T2_new[i];
            T_ex[i] = T2_ex[i];
        }
        if (tid == 0) S_cnt = 0;
        __syncthreads();
        lap(kKnPhMerge);
    }
    }  // parts

    // the list's entries that carry approximations get their exact scores
    // (the order among them was certified, so it is the exact order).  Their
    // dense rows are staged in shared memory by the whole CTA (coalesced; the
    // pool table is free now; row stride dstride + 1 floats so one thread per
    // row reads conflict-free), then one thread per entry runs the
    // reference's chain (hybrid_score's arithmetic, element order unchanged).
    if constexpr (NQ4 > 0) {
        for (uint32_t i = tid; i < k; i += nt) T_mk[i] = !T_ex[i];
        resolve_marked<NQ4>(a, sq, T_mk, k, 0x80000000u, fbits, a.pool_cap / 16, &n_mark,
                            reinterpret_cast<unsigned char*>(keys), size_t(a.pool_cap) * 4, T_sc, T_ex, T_id, S_sc,
                            S_ex, S_id);
    }
    lap(kKnPhExact);

    uint32_t mine = 0;
    for (uint32_t i = tid; i < k; i += nt) {
        a.N_ids[u * k + i] = T_id[i];
        a.N_sc[u * k + i] = T_sc[i];
        a.N_fr[u * k + i] = T_new[i];  // old entries participated (fresh=false)
        mine += T_new[i];
    }
    mine = __reduce_add_sync(0xFFFFFFFFu, mine);
    if ((tid & 31) == 0 && mine) atomicAdd(a.changed, (unsigned long long)mine);
    lap(kKnPhFinal);
    if (a.counts) {
        if (tid == 0) atomicAdd(&a.counts[0], static_cast<unsigned long long>(cand_total));
        if (lane == 0 && dense_rows) atomicAdd(&a.counts[1], static_cast<unsigned long long>(dense_rows));
        if (tid == 0 && sk_total) atomicAdd(&a.counts[2], static_cast<unsigned long long>(sk_total));
        if (lane == 0 && sk_rej) atomicAdd(&a.counts[3], static_cast<unsigned long long>(sk_rej));
    }
}

size_t pass_smem(uint32_t dstride, uint32_t lcap, uint32_t scap, uint32_t k, uint32_t pool_cap,
                 uint32_t l_vocab, const uint32_t* ck_cap, bool sketch = false) {
    size_t b = (doc_stage_bytes(dstride, lcap, scap) + 15) & ~size_t(15);
    b += static_cast<size_t>(pool_cap) * 4 + 2 * (pool_cap / 32) * 4;
    b += (2 * k + kSCap) * 8 + (2 * k + kSCap) * 4;
    b += 2 * k + 3 * k + 2 * kSCap + 16;                  // new / exact / mark flags, alignment
    b += static_cast<size_t>(dstride) * 4;                // fp32 dense row of u
    if (ck_cap) b += ck_bytes(ck_cap[0]) + ck_bytes(ck_cap[1]);  // u's cuckoo tables
    if (l_vocab) {                                        // u's learned bitmap, prefix, values
        const size_t W = approx::bitmap_words(l_vocab);
        b += ((W + 3) & ~size_t(3)) * 4 + ((W + 7) & ~size_t(7)) * 2 + static_cast<size_t>(lcap) * 4;
    }
    if (sketch) b = ((b + 15) & ~size_t(15)) + approx::kSketchBuckets;  // u's quantised bucket sums (last)
    return b;
}

// Pool slots for `items` expected distinct candidates (load factor <= 2/3).
uint32_t pool_slots(double items) {
    uint32_t cap = kPassThreads;
    while (cap < items * 1.5) cap <<= 1;
    return cap;
}

// The pool plan of a pass: the worst-case distinct two-hop candidates of a
// node, min(n, (2k)^2 + k), split into the fewest power-of-two hash parts
// whose pools let two CTAs share an SM (<= kSmemTwo bytes each, with a 4
// sigma + 64 margin per part for the hash split; a part that still
// overflows fails the pass loudly).
constexpr size_t kSmemTwo = 113 * 1024;
void pool_plan(uint64_t n, uint32_t k, uint32_t dstride, uint32_t lcap, uint32_t scap, uint32_t l_vocab,
               const uint32_t* ck_cap, bool sketch, uint32_t& cap, uint32_t& nparts) {
    const double worst = static_cast<double>(std::min<uint64_t>(n, 4ull * k * k + k));
    for (nparts = 1;; nparts <<= 1) {
        const double per = nparts == 1 ? worst : worst / nparts + 4.0 * std::sqrt(worst / nparts) + 64.0;
        cap = pool_slots(per);
        if (pass_smem(dstride, lcap, scap, k, cap, l_vocab, ck_cap, sketch) <= kSmemTwo || cap <= kPassThreads || nparts >= 64)
            return;
    }
}

int pass_nq4(uint32_t dstride) {
    const uint32_t need = ((dstride >> 2) + 31) / 32;
    for (int v : {1, 2, 3, 4, 6, 8})
        if (static_cast<uint32_t>(v) >= need) return v;
    return 0;
}

template <int NQ4>
void launch_pass(const PassArgs& a, uint64_t blocks, size_t sm, cudaStream_t s) {
    if constexpr (NQ4 > 0) {
        if (a.ck_cap[0] || a.ck_cap[1]) {
            FGB_CUDA(cudaFuncSetAttribute(knn_pass_kernel<NQ4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)sm));
            knn_pass_kernel<NQ4, true><<<(unsigned)blocks, kPassThreads, sm, s>>>(a);
            return;
        }
    }
    FGB_CUDA(cudaFuncSetAttribute(knn_pass_kernel<NQ4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    knn_pass_kernel<NQ4, false><<<(unsigned)blocks, kPassThreads, sm, s>>>(a);
    FGB_LAUNCH("knn_pass_kernel");
}

// Host-side partial Fisher-Yates (knn_graph.cpp:37-46) when 4k >= n.
void sample_fisher_yates(uint64_t n, uint32_t k, uint64_t seed, std::vector<uint32_t>& ids) {
    ids.resize(n * k);
    std::vector<uint32_t> all;
    for (uint64_t u = 0; u < n; ++u) {
        SplitMix64 rng(mix_seed(seed, u));
        all.clear();
        for (uint32_t i = 0; i < n; ++i)
            if (i != u) all.push_back(i);
        for (uint32_t i = 0; i < k; ++i) {
            const auto j = i + static_cast<uint32_t>(bounded(rng, all.size() - i));
            std::swap(all[i], all[j]);
            ids[u * k + i] = all[i];
        }
    }
}

}  // namespace

void knn_init_device(const fg_corpus& c, uint32_t k, uint64_t seed, DevKnn& g, cudaStream_t s) {
    if (k == 0) throw Error("invalid-k", "neighbour count must be positive");
    if (c.n < static_cast<uint64_t>(k) + 1)
        throw Error("corpus-too-small", "need at least " + std::to_string(k + 1) +
                                            " documents for k=" + std::to_string(k));
    g.alloc(c.n, k);
    if (static_cast<uint64_t>(k) * 4 < c.n) {
        knn_sample_kernel<<<(unsigned)((c.n + 255) / 256), 256, 0, s>>>(c.n, k, seed, g.ids.get());
        FGB_LAUNCH("knn_sample_kernel");
    } else {
        std::vector<uint32_t> ids;
        sample_fisher_yates(c.n, k, seed, ids);
        g.ids.upload(ids, s);
    }
    const uint32_t lcap = hash_capacity(c.max_lnnz), scap = hash_capacity(c.max_snnz);
    const size_t sm = doc_stage_bytes(c.dstride, lcap, scap) + static_cast<size_t>(k) * 12 + 16;
    FGB_CUDA(cudaFuncSetAttribute(knn_init_score_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sm));
    knn_init_score_kernel<<<(unsigned)c.n, std::min<uint32_t>(256, ((k + 31) / 32) * 32), sm, s>>>(
        c.dc, k, g.ids.get(), g.scores.get(), g.fresh.get(), lcap, scap);
    FGB_LAUNCH("knn_init_score_kernel");
}

// Reverse lists of the snapshot g (knn_graph.cpp:78-89): R[v] = the first
// min(k, |{u : v in L[u]}|) sources by (score desc, u asc), with freshness.
void knn_reverse_lists(const DevKnn& g, ReverseLists& R, cudaStream_t s) {
    const uint64_t n = g.n;
    const uint32_t k = g.k;
    const uint64_t m = n * k;
    // CUB's sorts/scans take int item counts
    if (m >= 0x7FFFFFFFull) throw Error("invalid-argument", "n*k exceeds 2^31-1 list entries");
    auto& keys_a = R.keys_a;
    auto& keys_b = R.keys_b;
    auto& vals_a = R.vals_a;
    auto& vals_b = R.vals_b;
    auto& tkeys_a = R.tkeys_a;
    auto& tkeys_b = R.tkeys_b;
    auto& cnt = R.tcnt;
    auto& start = R.tstart;
    keys_a.ensure(m);
    keys_b.ensure(m);
    vals_a.ensure(m);
    vals_b.ensure(m);
    tkeys_a.ensure(m);
    tkeys_b.ensure(m);
    if (cnt.size() != n) cnt.alloc(n);  // zeroed whole below
    start.ensure(n);
    R.ids.ensure(m);
    R.cnt.ensure(n);
    R.fresh.ensure(m);
    cnt.zero(s);
    const unsigned gb = (unsigned)((m + 255) / 256);
    score_keys_kernel<<<gb, 256, 0, s>>>(g.scores.get(), m, keys_a.get(), vals_a.get());
    FGB_LAUNCH("score_keys_kernel");
    size_t tb1 = 0, tb2 = 0, tb3 = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, tb1, keys_a.get(), keys_b.get(), vals_a.get(),
                                              vals_b.get(), (int)m, 0, 64, s);
    int bits = 1;
    while ((1ull << bits) < n) ++bits;
    cub::DeviceRadixSort::SortPairs(nullptr, tb2, tkeys_a.get(), tkeys_b.get(), vals_b.get(),
                                    vals_a.get(), (int)m, 0, bits, s);
    cub::DeviceScan::ExclusiveSum(nullptr, tb3, cnt.get(), start.get(), (int)n, s);
    DevBuf<unsigned char>& temp = R.temp;
    temp.ensure(std::max({tb1, tb2, tb3, size_t(16)}));
    size_t tb = temp.size();
    FGB_CUDA(cub::DeviceRadixSort::SortPairsDescending(temp.get(), tb, keys_a.get(), keys_b.get(),
                                                       vals_a.get(), vals_b.get(), (int)m, 0, 64, s));
    target_keys_kernel<<<gb, 256, 0, s>>>(g.ids.get(), vals_b.get(), m, tkeys_a.get(), cnt.get());
    FGB_LAUNCH("target_keys_kernel");
    tb = temp.size();
    FGB_CUDA(cub::DeviceRadixSort::SortPairs(temp.get(), tb, tkeys_a.get(), tkeys_b.get(),
                                             vals_b.get(), vals_a.get(), (int)m, 0, bits, s));
    tb = temp.size();
    FGB_CUDA(cub::DeviceScan::ExclusiveSum(temp.get(), tb, cnt.get(), start.get(), (int)n, s));
    reverse_fill_kernel<<<gb, 256, 0, s>>>(n, k, vals_a.get(), cnt.get(), start.get(),
                                           g.fresh.get(), R.ids.get(), R.fresh.get(), R.cnt.get());
    FGB_LAUNCH("reverse_fill_kernel");
}

constexpr uint64_t kSketchMinNodes = 8192;

int knn_sketch_policy() {
    const char* e = std::getenv("FGB_KNN_SKETCH");
    return e ? std::atoi(e) : 1;
}

uint32_t knn_sketch_passes() {
    const char* e = std::getenv("FGB_KNN_SKETCH_PASSES");  // dev A/B: passes screened under policy 1
    return e ? static_cast<uint32_t>(std::max(1, std::atoi(e))) : 1u;
}

void knn_sketch_prepare(const fg_corpus& c, ReverseLists& R, cudaStream_t s) {
    R.sk_paths = (c.max_lnnz ? 1u : 0u) | (c.max_snnz ? 2u : 0u);
    if (!R.sk_paths || !c.dc.meta || pass_nq4(c.dstride) == 0) return;  // (exact-chain passes: no screening)
    // small corpora: a pass is a few launch latencies, the sketches' build
    // and allocation would add to it (the reference's 2,400-doc insert
    // criterion runs in ~5 ms)
    if (c.n < kSketchMinNodes) return;
    R.sk_on = true;
    if (R.sketch.size() == c.n * (approx::kSketchBytes / 16)) return;
    R.sketch.alloc(c.n * (approx::kSketchBytes / 16));
    R.sk_gmax.alloc(1);
    R.sk_gmax.zero(s);
    sketch_max_kernel<<<1184, 256, 0, s>>>(c.dc, R.sk_paths, R.sk_gmax.get());
    FGB_LAUNCH("sketch_max_kernel");
    constexpr uint32_t kWarps = 4;  // 32 KB of bucket maxima per CTA
    sketch_build_kernel<<<(unsigned)((c.n + kWarps - 1) / kWarps), 32 * kWarps, kWarps * approx::kSketchBuckets * 4, s>>>(
        c.dc, R.sk_paths, R.sk_gmax.get(), R.sketch.get());
    FGB_LAUNCH("sketch_build_kernel");
}

void knn_sketch_disable(ReverseLists& R) { R.sk_on = false; }

// The per-node two-hop join (knn_graph.cpp:91-142) for nodes [lo, hi) of the
// snapshot g (with its reverse lists R) into rows [lo, hi) of next; adds the
// number of replaced entries to *d_changed (device).
void knn_pass_range(const fg_corpus& c, const DevKnn& g, const ReverseLists& R, uint64_t lo, uint64_t hi,
                    DevKnn& next, unsigned long long* d_changed, cudaStream_t s) {
    if (hi <= lo) return;
    const uint32_t k = g.k;
    const uint32_t lcap = hash_capacity(c.max_lnnz), scap = hash_capacity(c.max_snnz);
    PassArgs a{c.dc,           k,           g.ids.get(),   g.scores.get(), g.fresh.get(),
               R.ids.get(),    R.fresh.get(), R.cnt.get(),  next.ids.get(), next.scores.get(),
               next.fresh.get(), d_changed, 0, lcap, scap, lo,
               0.0, 0.0, 0.0, 0.0, 0, nullptr, 0, kSortMin, 1, 32, nullptr, nullptr, nullptr};
    if (R.counts.size() == 4) a.counts = R.counts.get();
    // (results do not depend on the order nodes are processed in)
    if (R.order.size() == g.n && lo == 0 && hi == g.n) a.order = R.order.get();
    if (const char* e = std::getenv("FGB_KNN_SORT_MIN")) a.sort_min = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("FGB_KNN_PREFETCH")) a.prefetch = std::atoi(e);
    DevBuf<unsigned long long> timing;
    const char* te = std::getenv("FGB_KNN_TIMING");
    if (te && te[0] == '1') {
        timing.alloc(kKnCount);
        timing.zero(s);
        a.timing = timing.get();
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (a.timing) {
        FGB_CUDA(cudaEventCreate(&e0));
        FGB_CUDA(cudaEventCreate(&e1));
        FGB_CUDA(cudaEventRecord(e0, s));
    }
    // error bound of the approximate pair scores (search_plain's, unit weights)
    const double N = double(c.dstride) + c.max_lnnz + c.max_snnz + 2;
    const double M = (c.dstride >> 2) + 2.0 * ((std::max(c.max_lnnz, c.max_snnz) + 127) / 128) + 16;
    const double u32 = std::ldexp(1.0, -24), u64 = std::ldexp(1.0, -53);
    a.eps32 = 4.0 * u32 / (1.0 - 4.0 * u32) * 1.01 + 1e-30;
    a.eps64 = (N + M + 8) * u64 * 1.01;
    if (const char* e = std::getenv("FGB_KNN_EPS_SCALE")) {  // tests: force the exact resolutions
        a.eps32 *= std::atof(e);
        a.eps64 *= std::atof(e);
    }
    a.max_dnorm = c.max_dnorm * (1.0 + 1e-6);
    a.max_norm = std::sqrt(std::max(c.max_sqnorm, 0.0)) * (1.0 + 1e-9);
    int nq4 = c.dc.meta ? pass_nq4(c.dstride) : 0;
    if (const char* e = std::getenv("FGB_KNN_EXACT"))  // dev: the exact-chain-only pass
        if (e[0] == '1') nq4 = 0;
    // u's sparse rows: two-choice cuckoo tables (FGB_KNN_CUCKOO=0: learned
    // bitmap + filter/hash); a node without a table (practically never at
    // <= 1/4 load) fails the cuckoo launch and the pass re-runs without
    bool ck = nq4 > 0;
    if (const char* e = std::getenv("FGB_KNN_CUCKOO"); e && e[0] == '0') ck = false;
    if (const char* e = std::getenv("FGB_KNN_CUCKOO"); e && e[0] == '2') a.ck_test_fail = 1;
    // (kept in R across passes: a device free synchronises the whole device)
    DevBuf<unsigned int>& flags = R.flags;  // [0] pool overflow, [1] nodes without a cuckoo table
    flags.ensure(2);
    DevBuf<unsigned long long>& changed0 = R.changed0;
    if (ck) {
        changed0.ensure(1);
        FGB_CUDA(cudaMemcpyAsync(changed0.get(), d_changed, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s));
    }
    const uint64_t blocks = hi - lo;
    size_t sm = 0;
    for (;;) {
        auto ck_cap = [](uint32_t nnz) {
            uint32_t v = 16;
            while (v < 4 * nnz) v <<= 1;
            return v;
        };
        // the learned path keeps its bitmap where the vocabulary allows (a
        // bitmap beat the cuckoo table in this kernel: 1M C2 NN-Descent
        // 12.25 s vs 12.84 s); hash-sized paths take cuckoo tables
        a.l_vocab = c.l_vocab <= 65536 ? c.l_vocab : 0;
        a.ck_cap[0] = ck && !a.l_vocab && c.max_lnnz ? ck_cap(c.max_lnnz) : 0;
        a.ck_cap[1] = ck && c.max_snnz ? ck_cap(c.max_snnz) : 0;
        const bool sk = nq4 > 0 && R.sk_on && R.sketch.size() == g.n * (approx::kSketchBytes / 16);
        pool_plan(g.n, k, c.dstride, lcap, scap, a.l_vocab, a.ck_cap, sk, a.pool_cap, a.nparts);
        if (pass_smem(c.dstride, lcap, scap, k, a.pool_cap, a.l_vocab, a.ck_cap, sk) > 227 * 1024) {
            a.l_vocab = 0;
            a.ck_cap[0] = ck && c.max_lnnz ? ck_cap(c.max_lnnz) : 0;
            pool_plan(g.n, k, c.dstride, lcap, scap, 0, a.ck_cap, sk, a.pool_cap, a.nparts);
        }
        if (const char* e = std::getenv("FGB_KNN_PARTS")) {  // dev/test: force a part count (power of two)
            const uint32_t v = static_cast<uint32_t>(std::atoi(e));
            if (v >= 1 && (v & (v - 1)) == 0) {
                a.nparts = v;
                const double worst = static_cast<double>(std::min<uint64_t>(g.n, 4ull * k * k + k));
                a.pool_cap = pool_slots(v == 1 ? worst : worst / v + 4.0 * std::sqrt(worst / v) + 64.0);
            }
        }
        a.pshift = 32 - static_cast<uint32_t>(__builtin_ctz(a.nparts));
        flags.zero(s);
        a.overflow = flags.get();
        a.ck_fail = flags.get() + 1;
        // (the sketch's u-side sums use the pool table as scratch: >= 2,048 slots)
        const bool use_sk = sk && a.pool_cap >= approx::kSketchBuckets;
        sm = pass_smem(c.dstride, lcap, scap, k, a.pool_cap, a.l_vocab, a.ck_cap, use_sk);
        a.sketch = use_sk ? R.sketch.get() : nullptr;
        a.sk_gmax = use_sk ? R.sk_gmax.get() : nullptr;
        a.sk_paths = R.sk_paths;
        a.sk_off = use_sk ? static_cast<uint32_t>(sm - approx::kSketchBuckets) : 0;
        if (sm > 227 * 1024)
            throw Error("invalid-argument", "knn_k too large for the shared-memory pool (" +
                                                std::to_string(sm) + " B)");
        switch (nq4) {
            case 1: launch_pass<1>(a, blocks, sm, s); break;
            case 2: launch_pass<2>(a, blocks, sm, s); break;
            case 3: launch_pass<3>(a, blocks, sm, s); break;
            case 4: launch_pass<4>(a, blocks, sm, s); break;
            case 6: launch_pass<6>(a, blocks, sm, s); break;
            case 8: launch_pass<8>(a, blocks, sm, s); break;
            default: launch_pass<0>(a, blocks, sm, s); break;
        }
        unsigned int fl[2] = {0, 0};
        flags.download(fl, 2, s);
        FGB_CUDA(cudaStreamSynchronize(s));
        if (fl[0]) throw Error("internal", "NN-Descent pool overflow (" + std::to_string(fl[0]) + " candidates)");
        if (!fl[1]) break;
        // (the dev counters of the failed launch stay summed)
        ck = false;
        a.ck_test_fail = 0;
        FGB_CUDA(cudaMemcpyAsync(d_changed, changed0.get(), sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s));
    }
    if (a.timing) {
        FGB_CUDA(cudaEventRecord(e1, s));
        unsigned long long t[kKnCount];
        timing.download(t, kKnCount, s);
        FGB_CUDA(cudaStreamSynchronize(s));
        float ms = 0;
        FGB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        const double nb = double(blocks);
        std::fprintf(stderr,
                     "[knn pass] %llu nodes, %.1f ms, smem %zu B, pool_cap %u x %u parts | cycles/node: init %.0f pool %.0f "
                     "score %.0f merge %.0f exact %.0f final %.0f | per node: cand %.1f dense %.1f enter %.1f rounds %.1f "
                     "resolved %.2f sketch-rejected %.1f\n",
                     (unsigned long long)blocks, ms, sm, a.pool_cap, a.nparts, t[kKnPhInit] / nb, t[kKnPhPool] / nb,
                     t[kKnPhScore] / nb, t[kKnPhMerge] / nb, t[kKnPhExact] / nb, t[kKnPhFinal] / nb, t[kKnCand] / nb, t[kKnDense] / nb,
                     t[kKnEnter] / nb, t[kKnRounds] / nb, t[kKnResolved] / nb, t[kKnSketch] / nb);
    }
}

uint64_t knn_iterate_device(const fg_corpus& c, DevKnn& g, cudaStream_t s, ReverseLists& R, DevKnn& next,
                            DevBuf<unsigned long long>& changed) {
    HostTimer ht("knn_iterate");
    knn_reverse_lists(g, R, s);
    ht.mark("reverse lists");
    if (next.n != g.n || next.k != g.k) next.alloc(g.n, g.k);
    if (changed.size() != 1) changed.alloc(1);
    changed.zero(s);
    if (!R.ev0) {
        FGB_CUDA(cudaEventCreate(&R.ev0));
        FGB_CUDA(cudaEventCreate(&R.ev1));
    }
    FGB_CUDA(cudaEventRecord(R.ev0, s));
    knn_pass_range(c, g, R, 0, g.n, next, changed.get(), s);
    FGB_CUDA(cudaEventRecord(R.ev1, s));
    ht.mark("pass kernel");
    unsigned long long h_changed = 0;
    changed.download(&h_changed, 1, s);
    FGB_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    FGB_CUDA(cudaEventElapsedTime(&ms, R.ev0, R.ev1));
    R.pass_ms += ms;
    std::swap(g.ids, next.ids);  // the old snapshot's buffers serve the next pass
    std::swap(g.scores, next.scores);
    std::swap(g.fresh, next.fresh);
    return h_changed;
}

uint64_t knn_iterate_device(const fg_corpus& c, DevKnn& g, cudaStream_t s) {
    ReverseLists R;
    if (knn_sketch_policy() >= 2) knn_sketch_prepare(c, R, s);
    DevKnn next;
    DevBuf<unsigned long long> changed;
    return knn_iterate_device(c, g, s, R, next, changed);
}

// BFS order over the first kOrderNbrs entries of every forward list (a
// permutation of [0, n)), uploaded to `order`.
constexpr uint64_t kOrderMinNodes = 65536;
constexpr uint32_t kOrderNbrs = 16;
void locality_order(const DevKnn& g, DevBuf<uint32_t>& order, cudaStream_t s) {
    const uint64_t n = g.n;
    const uint32_t k = g.k, w = std::min(k, kOrderNbrs);
    std::vector<uint32_t> ids(n * k);
    g.ids.download(ids.data(), ids.size(), s);
    FGB_CUDA(cudaStreamSynchronize(s));
    std::vector<uint32_t> ord;
    ord.reserve(n);
    std::vector<uint8_t> seen(n, 0);
    for (uint64_t root = 0; root < n; ++root) {
        if (seen[root]) continue;
        seen[root] = 1;
        uint64_t head = ord.size();
        ord.push_back(static_cast<uint32_t>(root));
        while (head < ord.size()) {
            const uint64_t u = ord[head++];
            const uint32_t* l = ids.data() + u * k;
            for (uint32_t j = 0; j < w; ++j)
                if (!seen[l[j]]) {
                    seen[l[j]] = 1;
                    ord.push_back(l[j]);
                }
        }
    }
    order.upload(ord, s);
}

uint32_t knn_build_device(const fg_corpus& c, uint32_t k_req, uint32_t max_iterations,
                          double convergence, uint64_t seed, DevKnn& g, cudaStream_t s, KnnStats* stats) {
    uint32_t k = k_req;
    if (c.n >= 2 && k >= c.n) k = static_cast<uint32_t>(c.n - 1);  // knn_graph.cpp:153-156
    HostTimer ht("knn_build");
    knn_init_device(c, k, seed, g, s);
    ht.mark("init");
    const double denom = static_cast<double>(c.n) * k;
    uint32_t passes = 0;
    ReverseLists R;
    if (stats) {
        R.counts.alloc(4);
        R.counts.zero(s);
    }
    DevKnn next;
    DevBuf<unsigned long long> d_changed;
    const int sk_policy = knn_sketch_policy();
    if (sk_policy >= 1) {
        knn_sketch_prepare(c, R, s);
        ht.mark("sketch");
    }
    for (uint32_t it = 0; it < max_iterations; ++it) {
        const uint64_t changed = knn_iterate_device(c, g, s, R, next, d_changed);
        ht.mark("pass");
        ++passes;
        // pass 1's candidates are random: the sketch bound rejects most of
        // them; later passes score neighbourhoods, where it rarely does
        if (it + 1 == knn_sketch_passes() && sk_policy == 1) knn_sketch_disable(R);
        if (static_cast<double>(changed) / denom < convergence) break;
        // After pass 1 the lists are neighbourhoods: later passes visit the
        // nodes in BFS order over them, so the CTAs resident at one time work
        // on overlapping two-hop pools and their candidate rows meet in L2.
        const char* oe = std::getenv("FGB_KNN_ORDER");
        if (it == 0 && c.n >= kOrderMinNodes && !(oe && oe[0] == '0')) {
            locality_order(g, R.order, s);
            ht.mark("order");
        }
    }
    if (stats) {
        unsigned long long h[4] = {0, 0, 0, 0};
        R.counts.download(h, 4, s);
        FGB_CUDA(cudaStreamSynchronize(s));
        stats->passes = passes;
        stats->candidates = h[0];
        stats->dense_rows = h[1];
        stats->sketched = h[2];
        stats->sketch_rejected = h[3];
        stats->pass_seconds = R.pass_ms / 1e3;
    }
    return passes;
}

}  // namespace fgb

using namespace fgb;

namespace {
void lists_to_host(const DevKnn& g, fg_knn_lists* out, cudaStream_t s) {
    out->k = g.k;
    g.ids.download(out->ids, g.n * g.k, s);
    g.scores.download(out->scores, g.n * g.k, s);
    g.fresh.download(out->fresh, g.n * g.k, s);
    FGB_CUDA(cudaStreamSynchronize(s));
}
void lists_to_device(const fg_knn_lists* in, DevKnn& g, cudaStream_t s) {
    g.alloc(in->n, in->k);
    g.ids.upload(in->ids, in->n * in->k, s);
    g.scores.upload(in->scores, in->n * in->k, s);
    g.fresh.upload(in->fresh, in->n * in->k, s);
}
}  // namespace

extern "C" {

int fg_knn_init(const fg_corpus* c, uint32_t k, uint64_t seed, fg_knn_lists* out) {
    return guarded([&] {
        if (!c || !out) throw Error("invalid-argument", "null pointer");
        FGB_CUDA(cudaSetDevice(c->device));
        DevKnn g;
        knn_init_device(*c, k, seed, g, c->stream);
        lists_to_host(g, out, c->stream);
    });
}

int fg_knn_iterate(const fg_corpus* c, fg_knn_lists* lists, uint64_t* changed) {
    return guarded([&] {
        if (!c || !lists) throw Error("invalid-argument", "null pointer");
        if (lists->n != c->n) throw Error("invalid-argument", "list count differs from corpus");
        FGB_CUDA(cudaSetDevice(c->device));
        DevKnn g;
        lists_to_device(lists, g, c->stream);
        const uint64_t ch = knn_iterate_device(*c, g, c->stream);
        lists_to_host(g, lists, c->stream);
        if (changed) *changed = ch;
    });
}

int fg_knn_build(const fg_corpus* c, const fg_knn_params* p, fg_knn_lists* out, uint32_t* passes) {
    return guarded([&] {
        if (!c || !p || !out) throw Error("invalid-argument", "null pointer");
        FGB_CUDA(cudaSetDevice(c->device));
        DevKnn g;
        const uint32_t ps = knn_build_device(*c, p->k, p->max_iterations, p->convergence, p->seed, g,
                                             c->stream);
        out->n = c->n;
        lists_to_host(g, out, c->stream);
        if (passes) *passes = ps;
    });
}

}  // extern "C"
