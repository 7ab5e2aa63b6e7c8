// Microbenchmark: dependent-load latency of the access patterns the search
// uses, on DRAM-resident rows, at W warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2511_00855_b200/csrc -o tools/ubench_latency tools/ubench_latency.cu
// mode 0: one coalesced 512-B warp load (LDG.128) per step, row chosen from the previous load
// mode 1: same, but the row was bulk-prefetched into L2 one step earlier
// mode 2: TMA bulk copy of a 3 KB row to smem + mbarrier wait per step
// mode 3: one 16-B load per lane from 32 different rows (lane-per-row)
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "tma.cuh"

using namespace fgb;
constexpr int D = 768;

__device__ __forceinline__ void l2pf(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <int MODE>
__global__ void lat(const float* __restrict__ rows, long long* cyc, int steps, int nrows, unsigned* sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm) + warp;
    float* slot = reinterpret_cast<float*>(sm + 16 * 64) + warp * D;
    if (lane == 0) mbar_init(bar, 1);
    fence_proxy_async();
    __syncthreads();
    const int gw = blockIdx.x * nw + warp;
    unsigned h = gw * 2654435761u + 12345u;
    unsigned nxt = (h * 747796405u) % nrows;
    uint32_t phase = 0;
    unsigned acc = 0;
    long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        const unsigned r = nxt;
        if (MODE == 0 || MODE == 1) {
            if (MODE == 1 && lane == 0) {
                // prefetch the row after next (independent of this step's data)
                const unsigned r2 = ((r ^ 0x5bd1e995u) * 747796405u) % nrows;
                l2pf(rows + (size_t)r2 * D, D * 4);
            }
            const float4 v = __ldg(reinterpret_cast<const float4*>(rows + (size_t)r * D) + lane);
            acc += __float_as_uint(v.x) + __float_as_uint(v.w);
            const unsigned dep = __reduce_or_sync(0xffffffffu, __float_as_uint(v.y) & 1u);  // data dependence
            nxt = MODE == 1 ? ((r ^ 0x5bd1e995u) * 747796405u + dep) % nrows : (r * 747796405u + 1u + dep) % nrows;
        } else if (MODE == 2) {
            if (lane == 0) {
                mbar_arrive_expect_tx(bar, D * 4);
                bulk_g2s(slot, rows + (size_t)r * D, D * 4, bar);
            }
            mbar_wait(bar, phase);
            phase ^= 1;
            const unsigned dep = __reduce_or_sync(0xffffffffu, __float_as_uint(slot[lane]) & 1u);
            acc += dep;
            nxt = (r * 747796405u + 1u + dep) % nrows;
            __syncwarp();
        } else {
            const unsigned rl = (r + lane * 7919u) % nrows;
            const float4 v = __ldg(reinterpret_cast<const float4*>(rows + (size_t)rl * D));
            const unsigned dep = __reduce_or_sync(0xffffffffu, __float_as_uint(v.y) & 1u);
            acc += dep;
            nxt = (r * 747796405u + 1u + dep) % nrows;
        }
    }
    long long t1 = clock64();
    if (lane == 0) cyc[gw] = t1 - t0;
    if (acc == 0xdeadbeef) sink[0] = acc;
}

int main() {
    const int big = 400000;
    float* rows;
    long long* cyc;
    unsigned* sink;
    cudaMalloc(&rows, sizeof(float) * (size_t)big * D);
    cudaMemset(rows, 0, sizeof(float) * (size_t)big * D);
    cudaMalloc(&cyc, sizeof(long long) * 148 * 64);
    cudaMalloc(&sink, 4);
    const char* names[] = {"coalesced 512B LDG", "LDG after L2 bulk prefetch", "TMA 3KB -> smem", "lane-per-row 16B LDG"};
    for (int mode = 0; mode < 4; ++mode)
        for (int W : {1, 4, 16, 32}) {
            const size_t smem = 16 * 64 + (size_t)W * D * 4;
            const int steps = 200;
            for (int it = 0; it < 2; ++it) {
                switch (mode) {
                    case 0: cudaFuncSetAttribute(lat<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); lat<0><<<148, 32 * W, smem>>>(rows, cyc, steps, big, sink); break;
                    case 1: cudaFuncSetAttribute(lat<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); lat<1><<<148, 32 * W, smem>>>(rows, cyc, steps, big, sink); break;
                    case 2: cudaFuncSetAttribute(lat<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); lat<2><<<148, 32 * W, smem>>>(rows, cyc, steps, big, sink); break;
                    case 3: cudaFuncSetAttribute(lat<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); lat<3><<<148, 32 * W, smem>>>(rows, cyc, steps, big, sink); break;
                }
            }
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("%s W=%d: %s\n", names[mode], W, cudaGetErrorString(e)); return 1; }
            long long hc[148 * 32];
            cudaMemcpy(hc, cyc, sizeof(long long) * 148 * W, cudaMemcpyDeviceToHost);
            double s = 0;
            for (int i = 0; i < 148 * W; ++i) s += hc[i];
            s /= 148 * W;
            printf("%-28s warps/SM %2d: %6.0f cycles/step\n", names[mode], W, s / steps);
        }
    return 0;
}
