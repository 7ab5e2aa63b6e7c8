// Microbenchmark: TMA-staged rows (cp.async.bulk -> smem) feeding lane-per-row
// bit-exact fp64 chains, vs the register-streamed rows of ubench_chain.cu.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2511_00855_b200/csrc -o tools/ubench_stage tools/ubench_stage.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "tma.cuh"

using namespace fgb;
constexpr int D = 768;
constexpr int SLOT = D + 4;  // words; 4 (mod 32) so 8 lanes' 16-byte reads hit 32 banks

__global__ void staged(const float* __restrict__ rows, const double* __restrict__ qg, double* out,
                       long long* cyc, int reps, int nrows, int R) {
    extern __shared__ __align__(16) unsigned char sm[];
    double* q = reinterpret_cast<double*>(sm);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + D * 8);
    float* slots = reinterpret_cast<float*>(sm + D * 8 + 16 * nw) + (size_t)warp * R * SLOT;
    for (int i = threadIdx.x; i < D; i += blockDim.x) q[i] = qg[i];
    if (lane == 0) mbar_init(&bars[warp], 1);
    fence_proxy_async();
    __syncthreads();
    const int gw = blockIdx.x * nw + warp;
    unsigned long long h = (gw * 32ull + lane + 1) * 0x9E3779B97F4A7C15ull;
    double acc = 0.0;
    uint32_t phase = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        h = h * 6364136223846793005ull + 1442695040888963407ull;
        const float* src = rows + (size_t)((h >> 33) % (unsigned)nrows) * D;
        if (lane == 0) mbar_arrive_expect_tx(&bars[warp], R * D * 4);
        __syncwarp();
        if (lane < R) bulk_g2s(slots + lane * SLOT, src, D * 4, &bars[warp]);
        mbar_wait(&bars[warp], phase);
        phase ^= 1;
        if (lane < R) {
            const float4* r4 = reinterpret_cast<const float4*>(slots + lane * SLOT);
            const double2* q2 = reinterpret_cast<const double2*>(q);
            double a = 0.0;
#pragma unroll 8
            for (int i = 0; i < D / 4; ++i) {
                const float4 d = r4[i];
                const double2 qa = q2[2 * i], qb = q2[2 * i + 1];
                a = __dadd_rn(a, __dmul_rn(qa.x, (double)d.x));
                a = __dadd_rn(a, __dmul_rn(qa.y, (double)d.y));
                a = __dadd_rn(a, __dmul_rn(qb.x, (double)d.z));
                a = __dadd_rn(a, __dmul_rn(qb.y, (double)d.w));
            }
            acc += a;
        }
        __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) cyc[gw] = t1 - t0;
    out[gw * 32 + lane] = acc;
}

int main() {
    const int big = 400000;  // 1.2 GB of rows: DRAM resident
    float* rows;
    double *q, *out;
    long long* cyc;
    cudaMalloc(&rows, sizeof(float) * (size_t)big * D);
    cudaMalloc(&q, sizeof(double) * D);
    cudaMalloc(&out, sizeof(double) * 148 * 64 * 32);
    cudaMalloc(&cyc, sizeof(long long) * 148 * 64);
    cudaMemset(rows, 0, sizeof(float) * (size_t)big * D);
    cudaMemset(q, 0, sizeof(double) * D);
    cudaFuncSetAttribute(staged, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    for (int R : {32, 16, 8, 4})
        for (int W : {1, 2, 4, 8, 16}) {
            const size_t smem = D * 8 + 16 * W + (size_t)W * R * SLOT * 4;
            if (smem > 227 * 1024) continue;
            const int reps = 16;
            for (int it = 0; it < 2; ++it)
                staged<<<148, 32 * W, smem>>>(rows, q, out, cyc, reps, big, R);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("R=%d W=%d: %s\n", R, W, cudaGetErrorString(e));
                return 1;
            }
            long long hc[148 * 16];
            cudaMemcpy(hc, cyc, sizeof(long long) * 148 * W, cudaMemcpyDeviceToHost);
            double s = 0;
            for (int i = 0; i < 148 * W; ++i) s += hc[i];
            s /= 148 * W;
            const double rows_per_clk_sm = (double)W * R * reps / s;
            printf("rows/warp %2d warps/SM %2d smem %6zu B: %7.0f cycles/round, %5.1f cycles/elem, %.2f elem/clk/SM "
                   "(%.0f GB/s at 1.965 GHz)\n",
                   R, W, smem, s / reps, s / (reps * D), rows_per_clk_sm * D,
                   rows_per_clk_sm * D * 4 * 148 * 1.965);
        }
    return 0;
}
