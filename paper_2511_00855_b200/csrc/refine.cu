// refine.cu — K4: the edge refinery on the GPU (refine.cpp:11-217).
//
// refine_node_kernel, one CTA per node u:
//   * candidate Gram: every pair (i<j) of u's k candidates is scored
//     bit-exactly (candidate_pair_scores, refine.cpp:11-23).  The dense part
//     is a tiled SIMT "GEMM" whose every output keeps its sequential k-order
//     (each thread owns whole dot products; the candidates' dense rows stream
//     through shared memory in 64-float chunks), the sparse parts a merge-join;
//   * detour counts, strict `<` (refine.cpp:25-39), and the rank sort by
//     (detours asc, score desc, id asc) (refine.cpp:41-65) — thread per
//     candidate, rank by counting;
//   * the IP prune walk with keyword recycling (refine.cpp:67-118) — one warp
//     walks the ranked list in order; the "first kept pruner" is a ballot, and
//     the union keyword coverage is a shared-memory hash of the kept set.
// merge_reverse_edges (refine.cpp:123-163) then runs as two stable radix sorts
// of the kept entries by (target, position, keeper) plus a warp per node, and
// the keyword lists drop ids that ended up semantic (refine.cpp:203-215).
#include <cub/cub.cuh>

#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "fg_cuda.hpp"
#include "knn.cuh"
#include "tcgen05.cuh"

namespace fgb {
namespace {

constexpr int kRefineThreads = 256;
constexpr uint32_t kTile = 64;        // dense floats per staged chunk
constexpr uint32_t kTileStride = kTile + 1;
constexpr int kMaxPairsPerThread = 8;
constexpr uint32_t kTileD = 32;       // dense doubles per staged chunk (even-k Gram)
// staged-tile region (floats): the odd-k row tile or the even-k transposed double tile
__host__ __device__ constexpr uint32_t tile_floats(uint32_t k) {
    return k * kTileStride > kTileD * (k + 2) * 2 ? k * kTileStride : kTileD * (k + 2) * 2;
}

// Sparse pair dot by a block merge-join (ascending term ids, matching
// products in order).  Rows start on 4-posting boundaries and are padded with
// (kPad, 0), so each side is a sequence of 16-B blocks.  One step compares a
// block of A with a block of B (16 compares), accumulates A's matches in lane
// order, and advances the side whose last term is smaller (both when equal):
// a match is found exactly once and the matched terms come out ascending, so
// the fma chain is the merge_dot of scoring.cpp:24-74.  The step is branch-
// free (selects and predicated loads), so the 32 lanes of a warp — each on its
// own pair — stay converged; the element-wise merge this replaces diverged on
// every step (70% of the kernel's stall samples at 200K docs).
__device__ __forceinline__ void match4(uint32_t t, float vt, const uint4& b, const float4& vb, double& acc) {
    const float sel = t == b.x ? vb.x : t == b.y ? vb.y : t == b.z ? vb.z : vb.w;
    const bool hit = t != kPad && (t == b.x || t == b.y || t == b.z || t == b.w);
    const double f = __fma_rn((double)vt, (double)sel, acc);
    acc = hit ? f : acc;
}

__device__ double merge_dot(const uint32_t* idx, const float* val, uint64_t oa, uint32_t na,
                            uint64_t ob, uint32_t nb) {
    double acc = 0.0;
    if (na == 0 || nb == 0) return acc;
    const uint4* A4 = reinterpret_cast<const uint4*>(idx + oa);
    const uint4* B4 = reinterpret_cast<const uint4*>(idx + ob);
    const float4* VA = reinterpret_cast<const float4*>(val + oa);
    const float4* VB = reinterpret_cast<const float4*>(val + ob);
    const uint32_t na4 = (na + 3) >> 2, nb4 = (nb + 3) >> 2;
    uint4 ca = __ldg(A4), cb = __ldg(B4);
    float4 cva = __ldg(VA), cvb = __ldg(VB);
    uint32_t i = 0, j = 0;
    uint4 xa = __ldg(A4 + min(1u, na4 - 1)), xb = __ldg(B4 + min(1u, nb4 - 1));
    float4 xva = __ldg(VA + min(1u, na4 - 1)), xvb = __ldg(VB + min(1u, nb4 - 1));
    while (i < na4 && j < nb4) {
        match4(ca.x, cva.x, cb, cvb, acc);
        match4(ca.y, cva.y, cb, cvb, acc);
        match4(ca.z, cva.z, cb, cvb, acc);
        match4(ca.w, cva.w, cb, cvb, acc);
        const bool adv_a = ca.w <= cb.w, adv_b = cb.w <= ca.w;
        if (adv_a) {
            ++i;
            ca = xa;
            cva = xva;
            const uint32_t nx = min(i + 1, na4 - 1);
            xa = __ldg(A4 + nx);
            xva = __ldg(VA + nx);
        }
        if (adv_b) {
            ++j;
            cb = xb;
            cvb = xvb;
            const uint32_t nx = min(j + 1, nb4 - 1);
            xb = __ldg(B4 + nx);
            xvb = __ldg(VB + nx);
        }
    }
    return acc;
}

__device__ __forceinline__ void pair_of(uint32_t p, uint32_t k, uint32_t& i, uint32_t& j) {
    // p enumerates (i, j), i < j, row by row
    i = 0;
    uint32_t rem = p;
    while (rem >= k - 1 - i) {
        rem -= k - 1 - i;
        ++i;
    }
    j = i + 1 + rem;
}

struct RefineArgs {
    DevCorpus c;
    uint32_t k, degree;
    int per_neighbour;
    const uint32_t* L_ids;
    const double* L_sc;
    uint32_t* ordered;     // n x k
    double* ordered_sc;    // n x k
    uint32_t* detours;     // n x k
    uint32_t* kept;        // n x degree
    uint32_t* kept_count;  // n
    uint32_t* recycled;    // n x k
    uint32_t* rec_count;   // n
    uint32_t kwcap;        // kept-keyword hash capacity (power of two)
    uint32_t ukw_cap;      // max keyword list length
    uint64_t lo;           // first node of this launch (vertex-range sharding)
    uint64_t row0;         // node of row 0 of the list/output arrays (inserts: n_old)
    // tensor-core Gram (gram_tc): on/off, bytes of the operand-stage / P
    // union, the certification bound and optional counters
    int tc;
    uint32_t tc_union;
    double tc_eps;
    int tc_check;
    unsigned long long* tc_stats;  // [0] pairs, [1] exact resolutions, [2] max |err|/(|a||b|) bits
};

// Generic (odd k) Gram: each thread owns up to kMaxPairsPerThread pairs.
__device__ __forceinline__ void gram_pairs(const RefineArgs& a, uint32_t k, const uint32_t* cid, double* P,
                                           float* tile) {
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    const uint32_t npairs = k * (k - 1) / 2;
    for (uint32_t pbase = 0; pbase < npairs; pbase += nt * kMaxPairsPerThread) {
        double acc[kMaxPairsPerThread];
        uint32_t pi[kMaxPairsPerThread], pj[kMaxPairsPerThread];
#pragma unroll
        for (int q = 0; q < kMaxPairsPerThread; ++q) {
            acc[q] = 0.0;
            const uint32_t p = pbase + q * nt + tid;
            if (p < npairs) {
                pair_of(p, k, pi[q], pj[q]);
            } else {
                pi[q] = pj[q] = 0xFFFFFFFFu;
            }
        }
        for (uint32_t d0 = 0; d0 < a.c.dstride; d0 += kTile) {
            const uint32_t w = min(kTile, a.c.dstride - d0);
            for (uint32_t e = tid; e < k * w; e += nt) {
                const uint32_t r = e / w, col = e % w;
                tile[r * kTileStride + col] = a.c.dense[(uint64_t)cid[r] * a.c.dstride + d0 + col];
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < kMaxPairsPerThread; ++q) {
                if (pi[q] == 0xFFFFFFFFu) continue;
                const float* ri = tile + pi[q] * kTileStride;
                const float* rj = tile + pj[q] * kTileStride;
                double s = acc[q];
                for (uint32_t dd = 0; dd < w; ++dd) s = __fma_rn((double)ri[dd], (double)rj[dd], s);
                acc[q] = s;
            }
            __syncthreads();
        }
#pragma unroll
        for (int q = 0; q < kMaxPairsPerThread; ++q)
            if (pi[q] != 0xFFFFFFFFu) P[pi[q] * k + pj[q]] = acc[q];
#pragma unroll 1
        for (int q = 0; q < kMaxPairsPerThread; ++q) {
            const uint32_t p = pbase + q * nt + tid;
            if (p >= npairs) continue;
            uint32_t i, j;
            pair_of(p, k, i, j);
            const uint64_t x = cid[i], y = cid[j];
            double s = P[i * k + j];
            s = __dadd_rn(s, merge_dot(a.c.l_idx, a.c.l_val, a.c.l_off[x], a.c.l_nnz[x], a.c.l_off[y], a.c.l_nnz[y]));
            s = __dadd_rn(s, merge_dot(a.c.s_idx, a.c.s_val, a.c.s_off[x], a.c.s_nnz[x], a.c.s_off[y], a.c.s_nnz[y]));
            P[i * k + j] = s;
            P[j * k + i] = s;
        }
    }
}

// Even k: the k candidates form k/2 row pairs; thread items are 2x2 blocks of
// row pairs (bi < bj) plus the k/2 diagonal pairs (2m, 2m+1).  The dense rows
// are staged TRANSPOSED as doubles (T[col][row], converted once at staging),
// so one 16-B shared load yields a row pair and each element costs a thread
// two loads for four DFMAs (the old lane-per-pair loop: two loads and two
// F2F conversions per DFMA).  Every output is still its own sequential fp64
// fma chain over the columns in order (= dense_dot, scoring.cpp:10-18).
__device__ __forceinline__ void gram_blocked(const RefineArgs& a, uint32_t k, const uint32_t* cid, double* P,
                                             double* T) {
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    const uint32_t kh = k >> 1, nblk = kh * (kh - 1) / 2;
    const uint32_t S = k + 2;  // doubles per staged column (16-B aligned)
    const double2* T2 = reinterpret_cast<const double2*>(T);
    const uint32_t S2 = S >> 1;
    const uint32_t rounds = max(1u, (nblk + 2 * nt - 1) / (2 * nt));
    for (uint32_t rd = 0; rd < rounds; ++rd) {
        uint32_t bi[2], bj[2];
        bool bv[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const uint32_t b = rd * 2 * nt + q * nt + tid;
            bv[q] = b < nblk;
            if (bv[q]) {
                pair_of(b, kh, bi[q], bj[q]);
            } else {
                bi[q] = bj[q] = 0;
            }
        }
        // diagonal pairs on the last threads of round 0
        const bool sv = rd == 0 && tid >= nt - kh;  // kh <= nt (k <= 160: P fits the SM)
        const uint32_t m = sv ? nt - 1 - tid : 0;
        double acc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
        double accs = 0.0;
        for (uint32_t d0 = 0; d0 < a.c.dstride; d0 += kTileD) {
            const uint32_t w = min(kTileD, a.c.dstride - d0);  // multiple of 4
            const uint32_t w4 = w >> 2;
            for (uint32_t e = tid; e < k * w4; e += nt) {
                const uint32_t r = e / w4, c4 = e % w4;
                const float4 v = __ldg(reinterpret_cast<const float4*>(a.c.dense + (uint64_t)cid[r] * a.c.dstride + d0) + c4);
                double* t = T + (size_t)(4 * c4) * S + r;
                t[0] = (double)v.x;
                t[S] = (double)v.y;
                t[2 * S] = (double)v.z;
                t[3 * S] = (double)v.w;
            }
            __syncthreads();
#pragma unroll 2
            for (uint32_t c = 0; c < w; ++c) {
                const double2* col = T2 + (size_t)c * S2;
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const double2 I = col[bi[q]], J = col[bj[q]];
                    acc[q][0] = __fma_rn(I.x, J.x, acc[q][0]);
                    acc[q][1] = __fma_rn(I.x, J.y, acc[q][1]);
                    acc[q][2] = __fma_rn(I.y, J.x, acc[q][2]);
                    acc[q][3] = __fma_rn(I.y, J.y, acc[q][3]);
                }
                const double2 M = col[m];
                accs = __fma_rn(M.x, M.y, accs);
            }
            __syncthreads();
        }
        // park the dense sums in P (the thread owns these entries), so the
        // sparse merges below do not keep nine fp64 accumulators live
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            if (!bv[q]) continue;
            const uint32_t i0 = 2 * bi[q], j0 = 2 * bj[q];
            P[i0 * k + j0] = acc[q][0];
            P[i0 * k + j0 + 1] = acc[q][1];
            P[(i0 + 1) * k + j0] = acc[q][2];
            P[(i0 + 1) * k + j0 + 1] = acc[q][3];
        }
        if (sv) P[2 * m * k + 2 * m + 1] = accs;
        auto finish = [&](uint32_t i, uint32_t j) {
            const uint64_t x = cid[i], y = cid[j];
            double s = P[i * k + j];
#pragma unroll 1
            for (int path = 0; path < 2; ++path) {  // dense + learned, then + statistical
                const bool l = path == 0;
                s = __dadd_rn(s, merge_dot(l ? a.c.l_idx : a.c.s_idx, l ? a.c.l_val : a.c.s_val,
                                           l ? a.c.l_off[x] : a.c.s_off[x], l ? a.c.l_nnz[x] : a.c.s_nnz[x],
                                           l ? a.c.l_off[y] : a.c.s_off[y], l ? a.c.l_nnz[y] : a.c.s_nnz[y]));
            }
            P[i * k + j] = s;
            P[j * k + i] = s;
        };
#pragma unroll 1
        for (int q = 0; q < 2; ++q) {
            if (!bv[q]) continue;
            const uint32_t i0 = 2 * bi[q], j0 = 2 * bj[q];
#pragma unroll 1
            for (uint32_t e = 0; e < 4; ++e) finish(i0 + (e >> 1), j0 + (e & 1));
        }
        if (sv) finish(2 * m, 2 * m + 1);
    }
}

// ---------------------------------------------------------------------------
// Tensor-core Gram (tcgen05, kind::f16).  The dense part of every candidate
// pair score is computed on the 5th-generation tensor cores as a split-bf16
// product: each fp32 element a = hi + lo (+ r, |r| <= 2^-17 |a|) with
// hi = bf16(a), lo = bf16(a - hi), and
//     dense(x, y) ~= hi_x.hi_y + hi_x.lo_y + lo_x.hi_y
// accumulated in fp32 in TMEM (3 MMAs per 16-wide K step).  The candidates'
// rows are converted while staged (K-chunks of 64, double-buffered, 128-byte
// swizzle), one thread issues M=64 (k <= 64) or M=128 MMAs, N = k rounded to
// 16, and the accumulator is read back with tcgen05.ld.
//
// Certification.  |approx - dense_dot| <= eps * |x| |y| with eps = 2^-10
// (kTcEps): the split drops <= 2^-15.5 |a_i b_i| per product, and 3*K/16 MMA
// accumulations of 17 fp32 terms each lose <= 17 ulps of the running
// magnitude (<= sum|a_i b_i| <= |x||y|) even with truncating alignment:
// 144 * 17 * 2^-23 = 2.9e-4 at d = 768, 3.4x below eps (measured: see
// FGB_REFINE_TC_CHECK and tests/test_gpu_refine_tc.py).  Every pair score
// enters the refinery only through comparisons with four thresholds known up
// front — csc[x], csc[y] (detours, strict <, refine.cpp:35) and sqnorm(x),
// sqnorm(y) (IP prune, >=, refine.cpp:85) — so a pair whose approximate score
// lies within eps of any of them is recomputed with the reference's exact
// sequential fp64 chain (dense_dot, scoring.cpp:10-18) and all others decide
// identically.  The sparse parts are exact merges either way.
constexpr double kTcEps = 0.0009765625;  // 2^-10
constexpr uint32_t kTcMaxItems = 4;      // (M rows x 8 chunks) / 256 threads, M <= 128

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&v);
}

__device__ __forceinline__ void split8(const float4& x0, const float4& x1, uint4& hi, uint4& lo) {
    const float f[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
    float h[8], l[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        h[i] = __bfloat162float(__float2bfloat16_rn(f[i]));
        l[i] = f[i] - h[i];  // exact in fp32
    }
    hi = make_uint4(pack_bf16x2(h[0], h[1]), pack_bf16x2(h[2], h[3]), pack_bf16x2(h[4], h[5]),
                    pack_bf16x2(h[6], h[7]));
    lo = make_uint4(pack_bf16x2(l[0], l[1]), pack_bf16x2(l[2], l[3]), pack_bf16x2(l[4], l[5]),
                    pack_bf16x2(l[6], l[7]));
}

// exact dense_dot (scoring.cpp:10-18): one sequential fp64 chain
__device__ double dense_exact(const DevCorpus& c, uint64_t x, uint64_t y) {
    const float4* A = reinterpret_cast<const float4*>(c.dense + x * c.dstride);
    const float4* B = reinterpret_cast<const float4*>(c.dense + y * c.dstride);
    double acc = 0.0;
    for (uint32_t t = 0; t < (c.dstride >> 2); ++t) {
        const float4 p = __ldg(A + t), q = __ldg(B + t);
        acc = __fma_rn((double)p.x, (double)q.x, acc);
        acc = __fma_rn((double)p.y, (double)q.y, acc);
        acc = __fma_rn((double)p.z, (double)q.z, acc);
        acc = __fma_rn((double)p.w, (double)q.w, acc);
    }
    return acc;
}

// Dense approximation of every candidate pair into P[i*k + j] (i != j); the
// operand stages alias P (they are dead before the epilogue writes it).
__device__ void gram_tc_dense(const RefineArgs& a, uint32_t k, const uint32_t* cid, double* P,
                              unsigned char* U, uint64_t* bar, uint32_t* tmem_slot) {
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t M = k <= 64 ? 64 : 128;
    const uint32_t N = (k + 15) & ~15u;
    const uint32_t ncols = N <= 32 ? 32 : N <= 64 ? 64 : 128;
    const uint32_t tile = M * 128;  // bytes of one operand tile (M rows x 64 bf16)
    const uint32_t nk = (a.c.dstride + 63) >> 6;
    const uint32_t items = M * 8 / kRefineThreads;
    const uint32_t idesc = idesc_bf16_f32(M, N);
    if (warp == 0) {
        tmem_alloc(tmem_slot, ncols);
        tmem_relinquish();
    }
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_proxy_async();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;

    float4 buf[kTcMaxItems][2];
    auto load = [&](uint32_t kc) {
#pragma unroll
        for (uint32_t it = 0; it < kTcMaxItems; ++it) {
            if (it >= items) break;
            const uint32_t q = tid + it * kRefineThreads, r = q >> 3, c = q & 7;
            const uint32_t col = kc * 64 + c * 8;
            float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0;
            if (r < k && col < a.c.dstride) {
                const float4* src = reinterpret_cast<const float4*>(a.c.dense + (uint64_t)cid[r] * a.c.dstride + col);
                v0 = __ldg(src);
                if (col + 4 < a.c.dstride) v1 = __ldg(src + 1);
            }
            buf[it][0] = v0;
            buf[it][1] = v1;
        }
    };
    auto store = [&](uint32_t st) {
        unsigned char* hi_t = U + st * 2 * tile;
        unsigned char* lo_t = hi_t + tile;
#pragma unroll
        for (uint32_t it = 0; it < kTcMaxItems; ++it) {
            if (it >= items) break;
            const uint32_t q = tid + it * kRefineThreads, r = q >> 3, c = q & 7;
            const uint32_t off = (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4);
            uint4 h, l;
            split8(buf[it][0], buf[it][1], h, l);
            *reinterpret_cast<uint4*>(hi_t + off) = h;
            *reinterpret_cast<uint4*>(lo_t + off) = l;
        }
    };
    load(0);
    for (uint32_t kc = 0; kc < nk; ++kc) {
        const uint32_t st = kc & 1;
        if (kc >= 2) mbar_wait(&bar[st], ((kc - 2) >> 1) & 1);  // MMAs of chunk kc-2 done with stage st
        store(st);
        if (kc + 1 < nk) load(kc + 1);  // next chunk's loads in flight across the MMA issue
        fence_proxy_async();            // generic-proxy smem writes -> tensor-core (async proxy) reads
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const unsigned char* hi_t = U + st * 2 * tile;
            const unsigned char* lo_t = hi_t + tile;
#pragma unroll
            for (uint32_t j = 0; j < 4; ++j) {
                const uint64_t dh = sw128_desc(hi_t + 32 * j), dl = sw128_desc(lo_t + 32 * j);
                mma_bf16_ss(tbase, dh, dh, idesc, (kc | j) ? 1u : 0u);
                mma_bf16_ss(tbase, dh, dl, idesc, 1u);
                mma_bf16_ss(tbase, dl, dh, idesc, 1u);
            }
            mma_commit(&bar[st]);
        }
    }
    mbar_wait(&bar[(nk - 1) & 1], ((nk - 1) >> 1) & 1);  // completion is in issue order
    tc_fence_after();
    if (warp < 4) {
        // M=128: row i in TMEM lane i; M=64: rows 16w..16w+15 in lanes 32w..32w+15
        const uint32_t i = M == 128 ? 32 * warp + lane : 16 * warp + lane;
        const bool valid = (M == 128 || lane < 16) && i < k;
        for (uint32_t cb = 0; cb < N; cb += 16) {
            float v[16];
            tmem_ld16(tbase + ((32 * warp) << 16) + cb, v);
            if (valid) {
#pragma unroll
                for (uint32_t c = 0; c < 16; ++c) {
                    const uint32_t j = cb + c;
                    if (j < k && j > i) {
                        P[i * k + j] = (double)v[c];
                        P[j * k + i] = (double)v[c];
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, ncols);
    for (uint32_t j = tid; j < k; j += kRefineThreads) P[j * k + j] = 0.0;
}

// Sparse parts (exact merges) + certification of every pair (see above).
__device__ void gram_tc_finish(const RefineArgs& a, uint32_t k, const uint32_t* cid, const double* csc, double* P) {
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    const uint32_t npairs = k * (k - 1) / 2;
    unsigned long long nres = 0;
    double maxrel = 0.0;
#pragma unroll 1
    for (uint32_t p = tid; p < npairs; p += nt) {
        uint32_t i, j;
        pair_of(p, k, i, j);
        const uint64_t x = cid[i], y = cid[j];
        const double d = P[i * k + j];
        const double l = merge_dot(a.c.l_idx, a.c.l_val, a.c.l_off[x], a.c.l_nnz[x], a.c.l_off[y], a.c.l_nnz[y]);
        const double t = merge_dot(a.c.s_idx, a.c.s_val, a.c.s_off[x], a.c.s_nnz[x], a.c.s_off[y], a.c.s_nnz[y]);
        double s = __dadd_rn(__dadd_rn(d, l), t);
        const double e = a.tc_eps * a.c.dnorm[x] * a.c.dnorm[y] * (1.0 + 1e-9) +
                         1e-13 * (fabs(d) + fabs(l) + fabs(t));
        const bool unc = fabs(s - csc[i]) <= e || fabs(s - csc[j]) <= e || fabs(s - a.c.sqnorm[x]) <= e ||
                         fabs(s - a.c.sqnorm[y]) <= e;
        if (unc || a.tc_check) {
            const double dx = dense_exact(a.c, x, y);
            if (a.tc_check) {
                const double nn = a.c.dnorm[x] * a.c.dnorm[y];
                if (nn > 0) maxrel = fmax(maxrel, fabs(d - dx) / nn);
            }
            s = __dadd_rn(__dadd_rn(dx, l), t);
            nres += unc;
        }
        P[i * k + j] = s;
        P[j * k + i] = s;
    }
    if (a.tc_stats) {
        const unsigned long long np = (tid < npairs) ? (npairs - tid + nt - 1) / nt : 0;
        atomicAdd(&a.tc_stats[0], np);
        if (nres) atomicAdd(&a.tc_stats[1], nres);
        if (maxrel > 0) atomicMax(&a.tc_stats[2], (unsigned long long)__double_as_longlong(maxrel));
    }
}

__global__ void __launch_bounds__(kRefineThreads) refine_node_kernel(RefineArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t tc_bar[2];
    __shared__ uint32_t tc_tmem;
    const uint32_t k = a.k;
    const uint64_t u = a.lo + blockIdx.x;
    const uint64_t ur = u - a.row0;  // row of u in the list / output arrays
    const uint32_t tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    // tensor-core path: P and the swizzled operand stages share a 1024-B aligned union
    unsigned char* smem = smem_raw;
    if (a.tc) smem += (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
    double* P = reinterpret_cast<double*>(smem);             // k*k
    double* csc = reinterpret_cast<double*>(smem + (a.tc ? a.tc_union : k * k * 8));  // k
    float* tile = reinterpret_cast<float*>(csc + k);         // k * kTileStride (SIMT Gram only)
    uint32_t* cid = reinterpret_cast<uint32_t*>(tile + (a.tc ? 0 : tile_floats(k)));
    uint32_t* det = cid + k;
    uint32_t* order = det + k;   // rank -> candidate index
    uint32_t* kp = order + k;    // kept ranked positions
    uint32_t* rec = kp + k;      // recycled ids
    uint32_t* kwset = rec + k;   // kept-keyword hash
    uint32_t* ukw = kwset + a.kwcap;
    __shared__ uint32_t nkept, nrec;

    for (uint32_t j = tid; j < k; j += nt) {
        cid[j] = a.L_ids[ur * k + j];
        csc[j] = a.L_sc[ur * k + j];
        if (!a.tc) P[j * k + j] = 0.0;
    }
    for (uint32_t j = tid; j < a.kwcap; j += nt) kwset[j] = kEmpty;
    const uint64_t ub = a.c.kw_ptr[u], ue = a.c.kw_ptr[u + 1];
    const uint32_t nukw = static_cast<uint32_t>(ue - ub);
    for (uint32_t j = tid; j < nukw; j += nt) ukw[j] = a.c.kw_idx[ub + j];
    __syncthreads();

    // ---- candidate Gram (refine.cpp:11-23)
    if (a.tc) {
        gram_tc_dense(a, k, cid, P, smem, tc_bar, &tc_tmem);
        __syncthreads();
        gram_tc_finish(a, k, cid, csc, P);
    } else if ((k & 1) == 0) {
        gram_blocked(a, k, cid, P, reinterpret_cast<double*>(tile));
    } else {
        gram_pairs(a, k, cid, P, tile);
    }
    __syncthreads();

    // ---- detours (strict <) and rank (refine.cpp:25-65)
    for (uint32_t v = tid; v < k; v += nt) {
        const double dis_uv = -csc[v];
        uint32_t cnt = 0;
        for (uint32_t x = 0; x < k; ++x) {
            if (x == v) continue;
            const double dis_ux = -csc[x];
            const double dis_xv = -P[x * k + v];
            cnt += fmax(dis_ux, dis_xv) < dis_uv;
        }
        det[v] = cnt;
    }
    __syncthreads();
    for (uint32_t v = tid; v < k; v += nt) {
        uint32_t r = 0;
        for (uint32_t w = 0; w < k; ++w) {
            const bool before = det[w] != det[v]   ? det[w] < det[v]
                                : csc[w] != csc[v] ? csc[w] > csc[v]
                                                   : cid[w] < cid[v];
            r += before;
        }
        order[r] = v;
    }
    __syncthreads();
    for (uint32_t r = tid; r < k; r += nt) {
        const uint32_t v = order[r];
        a.ordered[ur * k + r] = cid[v];
        a.ordered_sc[ur * k + r] = csc[v];
        a.detours[ur * k + r] = det[v];
    }

    // ---- IP prune walk + keyword recycling (refine.cpp:67-118), one warp
    if (warp == 0) {
        const uint32_t kwmask = a.kwcap - 1;
        auto kw_insert = [&](uint32_t node) {
            const uint64_t b = a.c.kw_ptr[node], e = a.c.kw_ptr[node + 1];
            for (uint64_t t = b + lane; t < e; t += 32) {
                const uint32_t key = a.c.kw_idx[t];
                uint32_t s = hslot(key, kwmask);
                while (true) {
                    const uint32_t prev = atomicCAS(&kwset[s], kEmpty, key);
                    if (prev == kEmpty || prev == key) break;
                    s = (s + 1) & kwmask;
                }
            }
            __syncwarp();
        };
        auto kw_has = [&](uint32_t key) {
            uint32_t s = hslot(key, kwmask);
            while (true) {
                const uint32_t kk = kwset[s];
                if (kk == key) return true;
                if (kk == kEmpty) return false;
                s = (s + 1) & kwmask;
            }
        };
        uint32_t nk = 0, nr = 0;
        if (k > 0) {
            if (lane == 0) kp[0] = 0;
            nk = 1;
            __syncwarp();
            kw_insert(cid[order[0]]);
        }
        for (uint32_t r = 1; r < k; ++r) {
            const uint32_t v = order[r];
            const uint32_t vid = cid[v];
            const double self_ip = a.c.sqnorm[vid];
            int pruner = -1;  // index into kp
            for (uint32_t b = 0; b < nk && pruner < 0; b += 32) {
                const uint32_t i = b + lane;
                const bool hit = i < nk && P[order[kp[i]] * k + v] >= self_ip;
                const uint32_t m = __ballot_sync(0xFFFFFFFFu, hit);
                if (m) pruner = static_cast<int>(b + __ffs(m) - 1);
            }
            if (pruner < 0 && nk < a.degree) {
                if (lane == 0) kp[nk] = r;
                ++nk;
                __syncwarp();
                kw_insert(vid);
                continue;
            }
            // dropped: recycle when shared keywords are not covered
            const uint64_t vb = a.c.kw_ptr[vid], ve = a.c.kw_ptr[vid + 1];
            const bool per = a.per_neighbour && pruner >= 0;
            uint64_t pb = 0, pe = 0;
            if (per) {
                const uint32_t pid = cid[order[kp[pruner]]];
                pb = a.c.kw_ptr[pid];
                pe = a.c.kw_ptr[pid + 1];
            }
            bool any_shared = false, uncovered = false;
            for (uint64_t t = vb + lane; t < ve; t += 32) {
                const uint32_t key = a.c.kw_idx[t];
                // sorted_intersection(node_kw, doc_kw) membership
                uint32_t lo = 0, hi = nukw;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (ukw[mid] < key)
                        lo = mid + 1;
                    else
                        hi = mid;
                }
                if (lo < nukw && ukw[lo] == key) {
                    any_shared = true;
                    const bool cov = per ? sorted_contains(a.c.kw_idx, pb, pe, key) : kw_has(key);
                    uncovered |= !cov;
                }
            }
            any_shared = __any_sync(0xFFFFFFFFu, any_shared);
            uncovered = __any_sync(0xFFFFFFFFu, uncovered);
            if (any_shared && uncovered) {
                if (lane == 0) rec[nr] = vid;
                ++nr;
            }
        }
        __syncwarp();
        for (uint32_t i = lane; i < nk; i += 32) a.kept[ur * a.degree + i] = cid[order[kp[i]]];
        for (uint32_t i = lane; i < nr; i += 32) a.recycled[ur * k + i] = rec[i];
        if (lane == 0) {
            a.kept_count[ur] = nk;
            a.rec_count[ur] = nr;
        }
    }
}

// (position, keeper) entries of every kept edge, keyed for the stable sorts.
__global__ void keeper_keys_kernel(uint64_t n, uint32_t degree, const uint32_t* kept,
                                   const uint32_t* kept_count, uint32_t* pos_key,
                                   uint32_t* vals, uint32_t* cnt) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= n * degree) return;
    const uint64_t w = t / degree;
    const uint32_t p = static_cast<uint32_t>(t % degree);
    vals[t] = static_cast<uint32_t>(t);
    if (p < kept_count[w]) {
        pos_key[t] = p;
        atomicAdd(&cnt[kept[t]], 1u);
    } else {
        pos_key[t] = 0xFFFFFFFFu;  // invalid: sorts last
    }
}

__global__ void target_key_kernel(uint64_t n, uint32_t degree, const uint32_t* kept,
                                  const uint32_t* kept_count, const uint32_t* order,
                                  uint32_t* tkey) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= n * degree) return;
    const uint32_t e = order[t];
    const uint64_t w = e / degree;
    const uint32_t p = e % degree;
    tkey[t] = p < kept_count[w] ? kept[e] : static_cast<uint32_t>(n);
}

// merge_reverse_edges for node u (warp per node) + keyword disjointness.
__global__ void merge_reverse_kernel(uint64_t n, uint32_t k, uint32_t degree, const uint32_t* kept,
                                     const uint32_t* kept_count, const uint32_t* keepers,
                                     const uint32_t* kstart, const uint32_t* kcnt,
                                     const uint32_t* ordered, uint32_t* semantic,
                                     uint32_t* recycled, uint32_t* rec_count) {
    extern __shared__ uint32_t lists[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t u = blockIdx.x * (uint64_t)(blockDim.x >> 5) + warp;
    if (u >= n) return;
    uint32_t* list = lists + warp * degree;
    const uint32_t half = degree / 2;
    const uint32_t kc = kept_count[u];
    const uint32_t fwd = min(half, kc);
    for (uint32_t i = lane; i < fwd; i += 32) list[i] = kept[u * degree + i];
    uint32_t size = fwd;
    __syncwarp();
    auto has = [&](uint32_t id) {
        bool hit = false;
        for (uint32_t i = lane; i < size; i += 32) hit |= list[i] == id;
        return __any_sync(0xFFFFFFFFu, hit);
    };
    auto push = [&](uint32_t id) {
        if (lane == 0) list[size] = id;
        ++size;
        __syncwarp();
    };
    const uint32_t rb = kstart[u], rn = kcnt[u];
    for (uint32_t i = 0; i < rn; ++i) {
        if (size >= fwd + half) break;
        const uint32_t e = keepers[rb + i];
        const uint32_t w = e / degree;
        if (!has(w)) push(w);
    }
    for (uint32_t i = fwd; i < kc && size < degree; ++i) {
        const uint32_t id = kept[u * degree + i];
        if (!has(id)) push(id);
    }
    for (uint32_t i = 0; i < k && size < degree; ++i) {
        const uint32_t id = ordered[u * k + i];
        if (!has(id)) push(id);
    }
    for (uint32_t i = lane; i < size; i += 32) semantic[u * degree + i] = list[i];
    // keyword lists stay disjoint from the semantic list (refine.cpp:207-215)
    const uint32_t nr = rec_count[u];
    uint32_t out = 0;
    for (uint32_t i = 0; i < nr; ++i) {
        const uint32_t id = recycled[u * k + i];
        if (!has(id)) {
            if (lane == 0) recycled[u * k + out] = id;
            ++out;
        }
    }
    if (lane == 0) rec_count[u] = out;
}

}  // namespace

// Diagnostics of the tensor-core Gram (FGB_REFINE_TC_STATS=1 or
// FGB_REFINE_TC_CHECK=1): counters on the current device, read through
// fg_refine_tc_stats.
unsigned long long* g_tc_stats = nullptr;
int g_tc_stats_dev = -1;
unsigned long long* refine_tc_stats_ptr() {
    const char* se = std::getenv("FGB_REFINE_TC_STATS");
    const char* ce = std::getenv("FGB_REFINE_TC_CHECK");
    if (!((se && se[0] == '1') || (ce && ce[0] == '1'))) return nullptr;
    int dev = 0;
    FGB_CUDA(cudaGetDevice(&dev));
    if (!g_tc_stats || g_tc_stats_dev != dev) {
        FGB_CUDA(cudaMalloc(&g_tc_stats, 4 * sizeof(unsigned long long)));
        FGB_CUDA(cudaMemset(g_tc_stats, 0, 4 * sizeof(unsigned long long)));
        g_tc_stats_dev = dev;
    }
    return g_tc_stats;
}

void refine_alloc(const DevKnn& g, uint32_t degree, RefineOut& out, cudaStream_t s) {
    const uint64_t n = g.n;
    const uint32_t k = g.k;
    if (degree == 0) throw Error("invalid-k", "degree must be positive");
    if (k < 2) throw Error("invalid-k", "refinery needs at least two candidates");
    if (static_cast<uint64_t>(k) * (k - 1) / 2 > static_cast<uint64_t>(kRefineThreads) * kMaxPairsPerThread * 64)
        throw Error("invalid-k", "knn_k too large for the refinery kernel");
    out.degree = degree;
    out.k = k;
    out.semantic.alloc(n * degree);
    out.keyword.alloc(n * k);
    out.kw_count.alloc(n);
    out.ordered.alloc(n * k);
    out.ordered_sc.alloc(n * k);
    out.detours.alloc(n * k);
    out.kept.alloc(n * degree);
    out.kept_count.alloc(n);
    FGB_CUDA(cudaMemsetAsync(out.semantic.get(), 0xFF, n * degree * 4, s));
}

void refine_nodes(const fg_corpus& c, const DevKnn& g, bool per_neighbour, uint64_t lo, uint64_t hi,
                  RefineOut& out, cudaStream_t s, uint64_t row0) {
    if (hi <= lo) return;
    const uint32_t k = g.k, degree = out.degree;
    uint32_t max_kw = 0;
    for (size_t i = 0; i < c.keywords.rows(); ++i)
        max_kw = std::max<uint32_t>(max_kw, static_cast<uint32_t>(c.keywords.len(i)));
    uint32_t kwcap = 32;
    while (kwcap < 2ull * max_kw * std::min(degree, k)) kwcap <<= 1;
    RefineArgs a{c.dc, k, degree, per_neighbour ? 1 : 0, g.ids.get(), g.scores.get(),
                 out.ordered.get(), out.ordered_sc.get(), out.detours.get(), out.kept.get(),
                 out.kept_count.get(), out.keyword.get(), out.kw_count.get(), kwcap, max_kw, lo, row0};
    // dense Gram on the tensor cores (gram_tc_dense) for k <= 128;
    // FGB_REFINE_TC=0 keeps the exact fp64 SIMT Gram (A/B and fallback tests)
    const char* te = std::getenv("FGB_REFINE_TC");
    a.tc = (!te || te[0] != '0') && k <= 128 && c.dc.dnorm != nullptr;
    const uint32_t tc_m = k <= 64 ? 64 : 128;
    a.tc_union = static_cast<uint32_t>(std::max<size_t>(static_cast<size_t>(k) * k * 8, 4ull * tc_m * 128));
    a.tc_eps = kTcEps;
    if (const char* e = std::getenv("FGB_REFINE_TC_EPS_SCALE")) a.tc_eps *= std::max(1.0, std::atof(e));
    const char* ce = std::getenv("FGB_REFINE_TC_CHECK");
    a.tc_check = ce && ce[0] == '1';
    a.tc_stats = refine_tc_stats_ptr();
    const size_t body = a.tc ? 1024 + a.tc_union + k * 8 : static_cast<size_t>(k) * k * 8 + k * 8 +
                                                            static_cast<size_t>(tile_floats(k)) * 4;
    const size_t sm = body + 5 * k * 4 + static_cast<size_t>(kwcap) * 4 + static_cast<size_t>(max_kw) * 4 + 16;
    if (sm > 227 * 1024)
        throw Error("invalid-k", "refinery shared memory exceeds the SM (" + std::to_string(sm) + " B)");
    FGB_CUDA(cudaFuncSetAttribute(refine_node_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    refine_node_kernel<<<(unsigned)(hi - lo), kRefineThreads, sm, s>>>(a);
    FGB_LAUNCH("refine_node_kernel");
}

void refine_merge(uint64_t n, RefineOut& out, cudaStream_t s) {
    const uint32_t k = out.k, degree = out.degree;
    // ---- keepers sorted by (target, position, keeper) (refine.cpp:127-133)
    const uint64_t m = n * degree;
    // CUB's sorts/scans take int item counts; keeper_keys_kernel packs the
    // entry index in 32 bits
    if (m >= 0x7FFFFFFFull || n >= 0x7FFFFFFFull)
        throw Error("invalid-argument", "n*degree exceeds 2^31-1 edge entries");
    DevBuf<uint32_t> pos_a(m), pos_b(m), vals_a(m), vals_b(m), tkey_a(m), tkey_b(m), cnt(n + 1),
        start(n + 1);
    cnt.zero(s);
    const unsigned gb = (unsigned)((m + 255) / 256);
    keeper_keys_kernel<<<gb, 256, 0, s>>>(n, degree, out.kept.get(), out.kept_count.get(),
                                          pos_a.get(), vals_a.get(), cnt.get());
    FGB_LAUNCH("keeper_keys_kernel");
    int tbits = 1;
    while ((1ull << tbits) <= n) ++tbits;
    size_t t1 = 0, t2 = 0, t3 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, pos_a.get(), pos_b.get(), vals_a.get(), vals_b.get(), (int)m, 0, 32, s);
    cub::DeviceRadixSort::SortPairs(nullptr, t2, tkey_a.get(), tkey_b.get(), vals_b.get(), vals_a.get(), (int)m, 0, tbits, s);
    cub::DeviceScan::ExclusiveSum(nullptr, t3, cnt.get(), start.get(), (int)n, s);
    DevBuf<unsigned char> temp(std::max({t1, t2, t3, size_t(16)}));
    size_t tb = temp.size();
    FGB_CUDA(cub::DeviceRadixSort::SortPairs(temp.get(), tb, pos_a.get(), pos_b.get(), vals_a.get(),
                                             vals_b.get(), (int)m, 0, 32, s));
    target_key_kernel<<<gb, 256, 0, s>>>(n, degree, out.kept.get(), out.kept_count.get(),
                                         vals_b.get(), tkey_a.get());
    FGB_LAUNCH("target_key_kernel");
    tb = temp.size();
    FGB_CUDA(cub::DeviceRadixSort::SortPairs(temp.get(), tb, tkey_a.get(), tkey_b.get(), vals_b.get(),
                                             vals_a.get(), (int)m, 0, tbits, s));
    tb = temp.size();
    FGB_CUDA(cub::DeviceScan::ExclusiveSum(temp.get(), tb, cnt.get(), start.get(), (int)n, s));
    const int warps = 8;
    merge_reverse_kernel<<<(unsigned)((n + warps - 1) / warps), warps * 32, warps * degree * 4, s>>>(
        n, k, degree, out.kept.get(), out.kept_count.get(), vals_a.get(), start.get(), cnt.get(),
        out.ordered.get(), out.semantic.get(), out.keyword.get(), out.kw_count.get());
    FGB_LAUNCH("merge_reverse_kernel");
    FGB_CUDA(cudaStreamSynchronize(s));
}

void refine_device(const fg_corpus& c, const DevKnn& g, uint32_t degree, bool per_neighbour,
                   RefineOut& out, cudaStream_t s) {
    HostTimer ht("refine");
    refine_alloc(g, degree, out, s);
    ht.mark("alloc");
    refine_nodes(c, g, per_neighbour, 0, g.n, out, s);
    ht.mark("nodes");
    refine_merge(g.n, out, s);
    ht.mark("merge");
}

}  // namespace fgb

using namespace fgb;

extern "C" {

int fg_refine(const fg_corpus* c, const fg_knn_lists* knn, const fg_refine_params* p,
              fg_refined* out, fg_refine_trace* trace) {
    return guarded([&] {
        if (!c || !knn || !p || !out) throw Error("invalid-argument", "null pointer");
        if (knn->n != c->n) throw Error("invalid-argument", "list count differs from corpus");
        if (out->keyword_cap < knn->k) throw Error("invalid-argument", "keyword_cap < k");
        FGB_CUDA(cudaSetDevice(c->device));
        cudaStream_t s = c->stream;
        DevKnn g;
        g.alloc(knn->n, knn->k);
        g.ids.upload(knn->ids, knn->n * knn->k, s);
        g.scores.upload(knn->scores, knn->n * knn->k, s);
        g.fresh.upload(knn->fresh, knn->n * knn->k, s);
        RefineOut r;
        refine_device(*c, g, p->degree, p->per_neighbour_keyword_check != 0, r, s);
        const uint64_t n = knn->n;
        const uint32_t k = knn->k;
        r.semantic.download(out->semantic, n * p->degree, s);
        std::vector<uint32_t> kw(n * k);
        r.keyword.download(kw.data(), n * k, s);
        r.kw_count.download(out->keyword_count, n, s);
        if (trace) {
            if (trace->ordered_ids) r.ordered.download(trace->ordered_ids, n * k, s);
            if (trace->ordered_scores) r.ordered_sc.download(trace->ordered_scores, n * k, s);
            if (trace->detours) r.detours.download(trace->detours, n * k, s);
            if (trace->kept) r.kept.download(trace->kept, n * p->degree, s);
            if (trace->kept_count) r.kept_count.download(trace->kept_count, n, s);
        }
        FGB_CUDA(cudaStreamSynchronize(s));
        for (uint64_t u = 0; u < n; ++u)
            std::copy(kw.begin() + u * k, kw.begin() + u * k + out->keyword_count[u],
                      out->keyword + u * out->keyword_cap);
    });
}

}  // extern "C"

extern "C" int fg_refine_tc_stats(uint64_t* pairs, uint64_t* resolved, double* max_rel_err, int reset) {
    return fgb::guarded([&] {
        unsigned long long h[4] = {0, 0, 0, 0};
        if (fgb::g_tc_stats) {
            FGB_CUDA(cudaDeviceSynchronize());
            FGB_CUDA(cudaMemcpy(h, fgb::g_tc_stats, sizeof(h), cudaMemcpyDeviceToHost));
            if (reset) FGB_CUDA(cudaMemset(fgb::g_tc_stats, 0, sizeof(h)));
        }
        if (pairs) *pairs = h[0];
        if (resolved) *resolved = h[1];
        if (max_rel_err) {
            double d;
            std::memcpy(&d, &h[2], 8);
            *max_rel_err = d;
        }
    });
}
