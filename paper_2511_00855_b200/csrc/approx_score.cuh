// approx_score.cuh — warp-cooperative approximate hybrid scores (coalesced
// row loads) used behind a certified error bound by the plain search
// (search_plain.cu) and the NN-Descent pass (knn.cu).  The exact chains stay
// in device_common.cuh.
#pragma once

#include "device_common.cuh"

namespace fgb {
namespace approx {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr int kSG = 8;  // sparse rows in flight per warp round trip

// One padding posting group (never matches a query term, value 0).
static __device__ const uint4 g_pad_idx4 = {kPad, kPad, kPad, kPad};
static __device__ const float4 g_pad_val4 = {0.f, 0.f, 0.f, 0.f};

// One sparse query path staged in shared memory.  Vocabularies up to 64K
// terms use a bitmap + rank structure (membership = one word test, value
// index = the word's prefix count + a popcount: branch-free); larger ones a
// bit filter in front of an open-addressing hash (device_common.cuh).
// Words of a query-term bitmap over [0, vocab): the smallest power of two W
// with 32 * W > vocab (bits >= vocab stay zero; see q_lookup_t).
__host__ __device__ inline uint32_t bitmap_words(uint32_t vocab) {
    uint32_t w = 1;
    while (32ull * w <= vocab) w <<= 1;
    return w;
}

struct PathQ {
    uint32_t on;     // path active for this query (weight != 0, query nnz > 0)
    uint32_t vocab;  // > 0: bitmap mode over [0, vocab)
    uint32_t wm1;    // bitmap words - 1 (a power of two minus one, 32 * words > vocab)
    const uint32_t* bm;
    const uint16_t* pre;
    const float* qv;  // weighted values (fp32, as build_query_vector) in ascending term order
    const uint32_t* keys;
    const float* vals;
    const uint32_t* filt;
    uint32_t mask;
    uint32_t hm1, hm2, hshift;  // cuckoo layout: slots (t * hm1) >> hshift and (t * hm2) >> hshift
};

// Lookup layouts: filter + open-addressing hash (0), bitmap + rank (1),
// two-choice cuckoo table (2: branch-free, exactly two probes).
enum : int { kLookHash = 0, kLookBitmap = 1, kLookCuckoo = 2 };

// The weighted query value of term t (found=false, 0 when absent).
template <int kLook>
__device__ __forceinline__ float q_lookup_t(const PathQ& P, uint32_t t, bool& found) {
    if constexpr (kLook == kLookCuckoo) {
        // both candidate slots always probed: no divergence between lanes
        const uint32_t s1 = (t * P.hm1) >> P.hshift, s2 = (t * P.hm2) >> P.hshift;
        const uint32_t k1 = P.keys[s1], k2 = P.keys[s2];
        const bool h1 = k1 == t, h2 = k2 == t;
        found = (h1 || h2) && t != kPad;
        float q = 0.0f;
        if (found) q = P.vals[h1 ? s1 : s2];
        return q;
    } else if constexpr (kLook == kLookBitmap) {
        // the bitmap spans a power of two of words past the vocabulary, so
        // masking maps the padding id (0xFFFFFFFF) to a bit that is never set
        const uint32_t tw = (t >> 5) & P.wm1;
        const uint32_t word = P.bm[tw];
        const uint32_t pre = P.pre[tw];
        found = (word >> (t & 31)) & 1u;
        const float q = P.qv[pre + __popc(word & ((1u << (t & 31)) - 1u))];
        return found ? q : 0.0f;
    } else {
        found = false;
        float q = 0.0f;
        if (t != kPad && filter_hit(P.filt, 2 * P.mask + 1, t)) found = hash_find(P.keys, P.vals, P.mask, t, q);
        return found ? q : 0.0f;
    }
}

__device__ __forceinline__ float q_lookup(const PathQ& P, uint32_t t, bool& found) {
    return P.vocab ? q_lookup_t<kLookBitmap>(P, t, found) : q_lookup_t<kLookHash>(P, t, found);
}

// Lookup modes of a search kernel instantiation: every active sparse path of
// the batch uses the hash (0) or the bitmap (1), or each path its own (2).
// One mode per instantiation keeps a single lookup variant in the hot loop
// (instruction-cache footprint).
enum : int { kModeHash = 0, kModeBitmap = 1, kModeMixed = 2, kModeCuckoo = 3 };
template <int kMode>
__device__ __forceinline__ float q_lookup_m(const PathQ& P, uint32_t t, bool& found) {
    if constexpr (kMode == kModeBitmap)
        return q_lookup_t<kLookBitmap>(P, t, found);
    else if constexpr (kMode == kModeHash)
        return q_lookup_t<kLookHash>(P, t, found);
    else if constexpr (kMode == kModeCuckoo)
        return q_lookup_t<kLookCuckoo>(P, t, found);
    else
        return q_lookup(P, t, found);
}

// Odd multipliers of the cuckoo tables, tried in order until every query
// term has a slot (a table at <= 1/4 load practically never needs the second).
__device__ __constant__ const uint32_t kCuckooMul[8][2] = {
    {0x9E3779B1u, 0x85EBCA77u}, {0xC2B2AE3Du, 0x27D4EB2Fu}, {0x165667B1u, 0xD3A2646Du}, {0xFD7046C5u, 0xB55A4F09u},
    {0x2545F491u, 0x4F1BBCDDu}, {0x68E31DA5u, 0x1B873593u}, {0xCC9E2D51u, 0x7FEB352Du}, {0x846CA68Bu, 0xE6546B65u}};

// Fills a two-choice cuckoo table of `cap` slots (a power of two, >= 4 nt)
// with the nt pairs tk/tv (staged in shared memory; warp-cooperative, lane 0
// inserts — a table at <= 1/4 load takes a few kicks at most).  Sets P.hm1/
// P.hm2 (P.hshift must be set); P.hm1 = 0 when no multiplier pair worked.
__device__ inline void cuckoo_fill(PathQ& P, uint32_t* keys, float* vals, const uint32_t* tk, const float* tv,
                                   uint32_t nt, uint32_t cap, uint32_t lane) {
    bool ok = false;
    for (int seed = 0; seed < 8 && !ok; ++seed) {
        const uint32_t m1 = kCuckooMul[seed][0], m2 = kCuckooMul[seed][1], sh = P.hshift;
        for (uint32_t j = lane; j < cap; j += 32) keys[j] = kEmpty;
        __syncwarp();
        uint32_t good = 1;
        if (lane == 0) {
            for (uint32_t j = 0; j < nt && good; ++j) {
                uint32_t key = tk[j];
                float val = tv[j];
                uint32_t pos = (key * m1) >> sh;
                good = 0;
                for (uint32_t kick = 0; kick < 4 * nt + 16; ++kick) {
                    const uint32_t old = keys[pos];
                    const float oldv = vals[pos];
                    keys[pos] = key;
                    vals[pos] = val;
                    if (old == kEmpty) {
                        good = 1;
                        break;
                    }
                    key = old;
                    val = oldv;
                    const uint32_t p1 = (key * m1) >> sh;
                    pos = pos == p1 ? (key * m2) >> sh : p1;
                }
            }
        }
        ok = __shfl_sync(kFull, good, 0) != 0;
        P.hm1 = m1;
        P.hm2 = m2;
        __syncwarp();
    }
    if (!ok) P.hm1 = 0;  // no table found: the caller fails the query (or node)
}

// ------------------------------------------------------------ scoring
// The query terms among 4 postings.  kF32 = false: exact fp64 products summed
// in fp64 (each product predicated on the lookup hit).  kF32 = true: fp32
// products accumulated by FMA (a missing term contributes q = 0), converted
// once — |error| <= gamma_4 (fp32) * sum|q_i v_i| <= gamma_4 |q_sparse| |d|,
// which the caller's bound must carry (knn.cu; the search keeps fp64: its
// tighter bound resolves 14x fewer comparisons exactly).
template <int kBitmap, bool kF32 = false>
__device__ __forceinline__ double probe4(const uint4& ii, const float4& vv, const PathQ& P) {
    bool f0, f1, f2, f3;
    const float q0 = q_lookup_t<kBitmap>(P, ii.x, f0), q1 = q_lookup_t<kBitmap>(P, ii.y, f1);
    const float q2 = q_lookup_t<kBitmap>(P, ii.z, f2), q3 = q_lookup_t<kBitmap>(P, ii.w, f3);
    if constexpr (kF32) {
        float s = q0 * vv.x;
        s = __fmaf_rn(q1, vv.y, s);
        s = __fmaf_rn(q2, vv.z, s);
        s = __fmaf_rn(q3, vv.w, s);
        return static_cast<double>(s);
    } else {
        double s = 0.0;
        if (f0) s = __fma_rn((double)q0, (double)vv.x, s);
        if (f1) s = __fma_rn((double)q1, (double)vv.y, s);
        if (f2) s = __fma_rn((double)q2, (double)vv.z, s);
        if (f3) s = __fma_rn((double)q3, (double)vv.w, s);
        return s;
    }
}

// Reduce-scatter of kSG per-lane partial sums: node k's total (over all 32
// lanes) ends in lanes [4k, 4k + 4) (bit-identical there).  9 shuffles
// instead of 8 full butterflies.
__device__ __forceinline__ double reduce_scatter8(double (&x)[8], uint32_t lane) {
    const bool b4 = (lane >> 4) & 1u, b3 = (lane >> 3) & 1u, b2 = (lane >> 2) & 1u;
    double y[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double send = b4 ? x[i] : x[i + 4];
        y[i] = (b4 ? x[i + 4] : x[i]) + __shfl_xor_sync(kFull, send, 16);
    }
    double z[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double send = b3 ? y[i] : y[i + 2];
        z[i] = (b3 ? y[i + 2] : y[i]) + __shfl_xor_sync(kFull, send, 8);
    }
    double r = (b2 ? z[1] : z[0]) + __shfl_xor_sync(kFull, b2 ? z[0] : z[1], 4);
    r += __shfl_xor_sync(kFull, r, 2);
    r += __shfl_xor_sync(kFull, r, 1);
    return r;
}

// Warp-cooperative approximate sparse dot of one path for the F nodes held
// by lanes 0..F-1 ((off4, nnz) each); lane j receives node j's sum.  kSG
// nodes' first 128 postings (idx + val, coalesced 512 B each) are in flight
// per round trip; postings 128.. of longer rows follow in a rolled loop.
template <int kBitmap, bool kF32 = false>
__device__ __forceinline__ double sparse_group(const uint32_t* idx, const float* val, const PathQ P, uint32_t off4,
                                            uint32_t nnz, uint32_t lane, uint32_t F) {
    double mine = 0.0;
    const uint4* i4 = reinterpret_cast<const uint4*>(idx);
    const float4* v4 = reinterpret_cast<const float4*>(val);
#pragma unroll 1
    for (uint32_t g = 0; g < F; g += kSG) {
        uint4 ii[kSG];
        float4 vv[kSG];
        // unpredicated loads (lanes past a row read the shared padding
        // record): a predicated load-or-default lets the compiler convert
        // each value right under its load, which serialises the round trips
#pragma unroll
        for (int k = 0; k < kSG; ++k) {
            const uint32_t j = g + k;
            const uint32_t oj = __shfl_sync(kFull, off4, j & 31);
            const uint32_t nj = __shfl_sync(kFull, nnz, j & 31);
            const bool in = j < F && 4 * lane < nj;
            ii[k] = __ldg(in ? i4 + oj + lane : &g_pad_idx4);
            vv[k] = __ldg(in ? v4 + oj + lane : &g_pad_val4);
        }
        // every probe depends on every load of the group (through a shuffle
        // ptxas cannot fold), so all kSG x 2 loads are issued before the
        // first probe instead of one pair per probe
        uint32_t tok = 0;
#pragma unroll
        for (int k = 0; k < kSG; ++k) tok += ii[k].x + __float_as_uint(vv[k].x);
        tok = __shfl_sync(kFull, tok, lane);
        PathQ Pg = P;
        Pg.wm1 = min(P.wm1, P.wm1 | tok);
        Pg.mask = min(P.mask, P.mask | tok);
        if constexpr (kBitmap == kLookCuckoo) Pg.hshift = min(P.hshift, P.hshift | tok);
        double part[8];
#pragma unroll
        for (int k = 0; k < kSG; ++k) part[k] = probe4<kBitmap, kF32>(ii[k], vv[k], Pg);
        const double r = reduce_scatter8(part, lane);
        const uint32_t k = lane - g;  // owner lane g + k takes node k's sum from lane 4k
        const double got = __shfl_sync(kFull, r, (4 * k) & 31);
        if (lane >= g && lane < g + kSG) mine = got;
    }
    // postings 128.. of long rows (none for nnz <= 128)
    uint32_t lm = __ballot_sync(kFull, lane < F && nnz > 128);
#pragma unroll 1
    while (lm) {
        const uint32_t j = __ffs(lm) - 1;
        lm &= lm - 1;
        const uint32_t oj = __shfl_sync(kFull, off4, j), nj = __shfl_sync(kFull, nnz, j);
        double e = 0.0;
        for (uint32_t base = 32; 4 * base < nj; base += 32)
            if (4 * (base + lane) < nj) e += probe4<kBitmap, kF32>(__ldg(i4 + oj + base + lane), __ldg(v4 + oj + base + lane), P);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(kFull, e, o);
        if (lane == j) mine += e;
    }
    return mine;
}

// ---- sparse sketch bound (NN-Descent pass 1)
// Every document carries a 512-byte SKETCH of its sparse paths: 2,048
// buckets of 2 bits, bucket b holding q_b = ceil(max |v_t| / g_v) over the
// terms t of the document in b (learned term t -> t & 2047, statistical term
// t -> (t + 1024) & 2047; g_v = the corpus's max |value| / 3 with margin).
// For a node u with bucket sums U_b = sum |u_t| quantised up to bytes
// (uq_b g_u >= U_b),
//     L(u, v) + S(u, v) <= sum_t |u_t| |v_t| <= sum_b U_b max_b |v|
//                       <= g_u g_v sum_b uq_b q_b,
// an exact integer dot (dp4a over the unpacked 2-bit lanes).  On pass 1's
// random two-hop candidates it rejects ~3/4 of them without touching their
// postings (C2 shape: the sparse part dominates the score), and one 16-byte
// load per lane covers a candidate (16 candidates per round trip).
// (1,024 buckets of 4 bits, half the unpack + dp4a work: 66% more survivors
// and pass 1 4.16 s vs 3.96 s at 1M, measured; screening every pass instead
// of the first: NN-Descent 11.66 s vs 10.60 s.)
constexpr uint32_t kSketchBuckets = 2048;
constexpr uint32_t kSketchBytes = kSketchBuckets / 4;  // per document
__device__ __forceinline__ uint32_t sketch_bucket(uint32_t t, int path) {
    return (t + (path ? kSketchBuckets / 2 : 0u)) & (kSketchBuckets - 1);
}
// Packing: bucket 16 w + 4 t + i of a lane's 64 lives in byte i, bits 2t..2t+1
// of the lane's word w; (word >> 2t) & 0x03030303 holds buckets 16 w + 4 t ..
// + 3 as bytes, matching u's byte word 4 w + t.

// Reduce-scatter of 16 per-lane u32 partial sums: row r's total ends in
// lanes [2r, 2r + 2).
__device__ __forceinline__ uint32_t reduce_scatter16_u32(uint32_t (&x)[16], uint32_t lane) {
    const bool b4 = (lane >> 4) & 1u, b3 = (lane >> 3) & 1u, b2 = (lane >> 2) & 1u, b1 = (lane >> 1) & 1u;
    uint32_t y[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t send = b4 ? x[i] : x[i + 8];
        y[i] = (b4 ? x[i + 8] : x[i]) + __shfl_xor_sync(kFull, send, 16);
    }
    uint32_t z[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t send = b3 ? y[i] : y[i + 4];
        z[i] = (b3 ? y[i + 4] : y[i]) + __shfl_xor_sync(kFull, send, 8);
    }
    uint32_t w[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const uint32_t send = b2 ? z[i] : z[i + 2];
        w[i] = (b2 ? z[i + 2] : z[i]) + __shfl_xor_sync(kFull, send, 4);
    }
    uint32_t r = (b1 ? w[1] : w[0]) + __shfl_xor_sync(kFull, b1 ? w[0] : w[1], 2);
    r += __shfl_xor_sync(kFull, r, 1);
    return r;
}

// Integer sketch dot sum_b uq_b q_b(node) for the F nodes held by lanes
// 0..F-1; lane j receives node j's.  uq = u's quantised bucket sums in shared
// memory (2,048 bytes); lane L covers buckets [64 L, 64 L + 64).
__device__ __forceinline__ uint32_t sketch_group(const uint4* sketch, const uint32_t* uq, uint32_t node,
                                                 uint32_t lane, uint32_t F) {
    uint32_t mine = 0;
#pragma unroll 1
    for (uint32_t g = 0; g < F; g += 16) {
        uint4 v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const uint32_t j = g + k;
            const uint32_t nj = __shfl_sync(kFull, node, j & 31);
            v[k] = __ldg(sketch + static_cast<uint64_t>(j < F ? nj : 0u) * (kSketchBytes / 16) + lane);
        }
        uint32_t part[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) part[k] = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const uint4 u4 = reinterpret_cast<const uint4*>(uq)[4 * lane + w];  // u's bytes 64 L + 16 w ..
            const uint32_t uw[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const uint32_t word = w == 0 ? v[k].x : w == 1 ? v[k].y : w == 2 ? v[k].z : v[k].w;
#pragma unroll
                for (int t = 0; t < 4; ++t) part[k] = __dp4a((word >> (2 * t)) & 0x03030303u, uw[t], part[k]);
            }
        }
        const uint32_t r = reduce_scatter16_u32(part, lane);
        const uint32_t k = lane - g;
        const uint32_t got = __shfl_sync(kFull, r, (2 * k) & 31);
        if (lane >= g && lane < g + 16) mine = got;
    }
    return mine;
}

template <int NQ4>
__device__ __forceinline__ void dense_load(const DevCorpus& c, uint32_t node, uint32_t lane, float4 (&b)[NQ4]) {
    const float4* row = reinterpret_cast<const float4*>(c.dense + static_cast<uint64_t>(node) * c.dstride);
    const uint32_t n4 = c.dstride >> 2;
    // (clamped, unpredicated: columns past the row are multiplied by nothing)
#pragma unroll
    for (int k = 0; k < NQ4; ++k) b[k] = __ldg(row + min(k * 32 + lane, n4 - 1));
}

// Rows in flight per round trip of dense_group: 4 up to d = 768 (search at
// configs[1]: 113K -> 120K QPS over 2 rows, B200), 8 for d <= 128, so a batch
// of F candidates costs F/rows dependent round trips.
template <int NQ4>
constexpr int dense_rows() { return NQ4 == 1 ? 8 : (NQ4 <= 6 ? 4 : 2); }

// Reduce-scatter of R per-lane partial sums (R a power of two <= 8): row r's
// total (over all 32 lanes) ends in lanes [r * 32/R, (r + 1) * 32/R).
template <int R>
__device__ __forceinline__ double reduce_scatter(double (&x)[R], uint32_t lane) {
#pragma unroll
    for (int cnt = R, stride = 16; cnt > 1; cnt >>= 1, stride >>= 1) {
        const bool b = (lane & stride) != 0;
#pragma unroll
        for (int i = 0; i < cnt / 2; ++i) {
            const double send = b ? x[i] : x[i + cnt / 2];
            x[i] = (b ? x[i + cnt / 2] : x[i]) + __shfl_xor_sync(kFull, send, stride);
        }
    }
    double r = x[0];
#pragma unroll
    for (int stride = 16 / R; stride > 0; stride >>= 1) r += __shfl_xor_sync(kFull, r, stride);
    return r;
}

// Warp-cooperative approximate dense dot (coalesced 512-B loads per warp
// instruction) for every lane-held node in `mask`, dense_rows<NQ4>() rows
// per round trip; fp32 partials of 4 elements, accumulated in fp64.
template <int NQ4, int R = dense_rows<NQ4>()>
__device__ __forceinline__ double dense_group(const DevCorpus& c, const float* qd, uint32_t node, uint32_t lane,
                                              uint32_t mask) {
    double mine = 0.0;
    const float4* q4 = reinterpret_cast<const float4*>(qd);
    const uint32_t n4 = c.dstride >> 2;
    uint32_t m = mask;
#pragma unroll 1
    while (m) {
        uint32_t j[R];
        const uint32_t j0 = __ffs(m) - 1;
#pragma unroll
        for (int r = 0; r < R; ++r) {  // (missing rows repeat j0: L1 hits, results unused)
            j[r] = m ? __ffs(m) - 1 : j0;
            m &= m - 1;
        }
        float4 rows[R][NQ4];
#pragma unroll
        for (int r = 0; r < R; ++r) dense_load<NQ4>(c, __shfl_sync(kFull, node, j[r]), lane, rows[r]);
        double s[R];
#pragma unroll
        for (int r = 0; r < R; ++r) s[r] = 0.0;
#pragma unroll
        for (int k = 0; k < NQ4; ++k) {
            const uint32_t col = k * 32 + lane;
            if (col < n4) {
                const float4 q = q4[col];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    float p = q.x * rows[r][k].x;
                    p = __fmaf_rn(q.y, rows[r][k].y, p);
                    p = __fmaf_rn(q.z, rows[r][k].z, p);
                    p = __fmaf_rn(q.w, rows[r][k].w, p);
                    s[r] += (double)p;
                }
            }
        }
        const double tot = reduce_scatter<R>(s, lane);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double g = __shfl_sync(kFull, tot, r * (32 / R));
            if (lane == j[r] && (r == 0 || j[r] != j0)) mine = g;
        }
    }
    return mine;
}

}  // namespace approx
}  // namespace fgb
