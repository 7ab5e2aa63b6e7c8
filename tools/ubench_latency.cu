// Microbenchmark: dependent-load latency of the access patterns the search
// uses, on DRAM-resident rows (pointer chase over a random cycle), at W warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2511_00855_b200/csrc -o tools/ubench_latency tools/ubench_latency.cu
// mode 0: one coalesced 512-B warp load (LDG.128) per step; the next row id is in the row
// mode 1: same, plus a bulk L2 prefetch of the row two steps ahead (known one step early)
// mode 2: TMA bulk copy of the 3 KB row to smem + mbarrier wait per step
// mode 3: 16-B load per lane from 32 different rows (lane-per-row), next ids from lane 0's row
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

#include "tma.cuh"

using namespace fgb;
constexpr int D = 768;

__device__ __forceinline__ void l2pf(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// row r holds next[r] in word 0 and next[next[r]] in word 1
template <int MODE>
__global__ void lat(const float* __restrict__ rows, long long* cyc, int steps, unsigned start_stride,
                    unsigned* sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm) + warp;
    float* slot = reinterpret_cast<float*>(sm + 16 * 64) + warp * D;
    if (lane == 0) mbar_init(bar, 1);
    fence_proxy_async();
    __syncthreads();
    const int gw = blockIdx.x * nw + warp;
    unsigned r = gw * start_stride;
    uint32_t phase = 0;
    unsigned acc = 0;
    long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        const float* row = rows + (size_t)r * D;
        if (MODE == 0 || MODE == 1) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(row) + lane);
            const unsigned nx = __shfl_sync(0xffffffffu, v.x, 0);
            if (MODE == 1 && lane == 0) l2pf(rows + (size_t)__shfl_sync(0x1u, v.y, 0) * D, D * 4);
            acc += v.z;
            r = nx;
        } else if (MODE == 2) {
            if (lane == 0) {
                mbar_arrive_expect_tx(bar, D * 4);
                bulk_g2s(slot, row, D * 4, bar);
            }
            mbar_wait(bar, phase);
            phase ^= 1;
            r = reinterpret_cast<const unsigned*>(slot)[0];
            acc += reinterpret_cast<const unsigned*>(slot)[lane + 2];
            __syncwarp();
        } else {
            // lane-per-row: lane l reads 16 B of row next^l(r)... use row r + lane*7919 (random-ish)
            const unsigned rl = lane == 0 ? r : __ldg(reinterpret_cast<const unsigned*>(rows + (size_t)r * D) + 2 + lane);
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(rows + (size_t)rl * D));
            r = __shfl_sync(0xffffffffu, v.x, 0);
            acc += v.z;
        }
    }
    long long t1 = clock64();
    if (lane == 0) cyc[gw] = t1 - t0;
    if (acc == 0xdeadbeef) sink[0] = acc;
}

int main() {
    const unsigned big = 400000;  // 1.2 GB of rows
    std::vector<unsigned> perm(big);
    for (unsigned i = 0; i < big; ++i) perm[i] = i;
    std::mt19937 g(7);
    std::shuffle(perm.begin(), perm.end(), g);
    std::vector<unsigned> nxt(big);
    for (unsigned i = 0; i < big; ++i) nxt[perm[i]] = perm[(i + 1) % big];  // one random cycle
    std::vector<float> host((size_t)big * D);
    for (unsigned i = 0; i < big; ++i) {
        unsigned* w = reinterpret_cast<unsigned*>(&host[(size_t)i * D]);
        w[0] = nxt[i];
        w[1] = nxt[nxt[i]];
        for (int j = 2; j < D; ++j) w[j] = (i * 2654435761u) ^ (j * 40503u);  // incompressible-ish, ids for mode 3
        for (int j = 2; j < 34; ++j) w[j] = (i * 2654435761u + j * 97u) % big;
    }
    float* rows;
    long long* cyc;
    unsigned* sink;
    cudaMalloc(&rows, sizeof(float) * (size_t)big * D);
    cudaMemcpy(rows, host.data(), sizeof(float) * (size_t)big * D, cudaMemcpyHostToDevice);
    cudaMalloc(&cyc, sizeof(long long) * 148 * 64);
    cudaMalloc(&sink, 4);
    const char* names[] = {"coalesced 512B LDG", "LDG + L2 bulk prefetch ahead", "TMA 3KB -> smem", "lane-per-row 16B LDG"};
    for (int mode = 0; mode < 4; ++mode)
        for (int W : {1, 4, 16, 32}) {
            const size_t smem = 16 * 64 + (size_t)W * D * 4;
            const int steps = 300;
            const unsigned stride = big / (148 * W) ;
            for (int it = 0; it < 2; ++it) {
                switch (mode) {
                    case 0: cudaFuncSetAttribute(lat<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); lat<0><<<148, 32 * W, smem>>>(rows, cyc, steps, stride, sink); break;
                    case 1: cudaFuncSetAttribute(lat<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); lat<1><<<148, 32 * W, smem>>>(rows, cyc, steps, stride, sink); break;
                    case 2: cudaFuncSetAttribute(lat<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); lat<2><<<148, 32 * W, smem>>>(rows, cyc, steps, stride, sink); break;
                    case 3: cudaFuncSetAttribute(lat<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); lat<3><<<148, 32 * W, smem>>>(rows, cyc, steps, stride, sink); break;
                }
            }
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("%s W=%d: %s\n", names[mode], W, cudaGetErrorString(e)); return 1; }
            long long hc[148 * 32];
            cudaMemcpy(hc, cyc, sizeof(long long) * 148 * W, cudaMemcpyDeviceToHost);
            double s = 0;
            for (int i = 0; i < 148 * W; ++i) s += hc[i];
            s /= 148 * W;
            printf("%-30s warps/SM %2d: %6.0f cycles/step\n", names[mode], W, s / steps);
        }
    return 0;
}
