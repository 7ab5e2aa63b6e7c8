// Microbenchmark: latency of the bit-exact fp64 dot chain on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench tools/ubench_chain.cu
// Each lane runs one sequential 768-element chain; reports cycles/element per
// warp for several operand sources, with W warps per SM.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int D = 768;

template <int kStage>
__device__ __forceinline__ double dense_chain(const float* rowp, const double* q) {
    const float4* row = reinterpret_cast<const float4*>(rowp);
    const double2* q2 = reinterpret_cast<const double2*>(q);
    constexpr uint32_t n4 = D / 4;
    double acc = 0.0;
    float4 cur[kStage], nxt[kStage];
#pragma unroll
    for (uint32_t j = 0; j < kStage; ++j) cur[j] = __ldg(row + j);
    for (uint32_t i = 0; i < n4; i += kStage) {
#pragma unroll
        for (uint32_t j = 0; j < kStage; ++j)
            nxt[j] = i + kStage + j < n4 ? __ldg(row + i + kStage + j) : make_float4(0, 0, 0, 0);
#pragma unroll
        for (uint32_t j = 0; j < kStage; ++j) {
            const double2 a = q2[2 * (i + j)], b = q2[2 * (i + j) + 1];
            acc = __fma_rn(a.x, (double)cur[j].x, acc);
            acc = __fma_rn(a.y, (double)cur[j].y, acc);
            acc = __fma_rn(b.x, (double)cur[j].z, acc);
            acc = __fma_rn(b.y, (double)cur[j].w, acc);
        }
#pragma unroll
        for (uint32_t j = 0; j < kStage; ++j) cur[j] = nxt[j];
    }
    return acc;
}

template <int MODE>
__global__ void chain(const float* __restrict__ rows, const double* __restrict__ qg, double* out,
                      long long* cyc, int reps, int nrows) {
    __shared__ double q[D];
    __shared__ float qf[D];
    for (int i = threadIdx.x; i < D; i += blockDim.x) {
        q[i] = qg[i];
        qf[i] = (float)qg[i];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const float* row = rows + (size_t)((gw * 32 + lane) % 4096) * D;
    unsigned long long h = (gw * 32ull + lane) * 0x9E3779B97F4A7C15ull;
    float reg[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) reg[j] = row[j];
    double acc = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (MODE == 0) {  // DFMA chain, operands in registers (pure latency)
            double a = 1.0 + lane;
#pragma unroll 32
            for (int i = 0; i < D; ++i) acc = __fma_rn(a, (double)i, acc);
        } else if (MODE == 1) {  // + F2F per element (float operand in registers)
#pragma unroll
            for (int i = 0; i < D; i += 32)
#pragma unroll
                for (int j = 0; j < 32; ++j) acc = __fma_rn(q[i + j], (double)reg[j], acc);
        } else if (MODE == 2) {  // current: q from smem (fp64), row via 16-B global loads
            const float4* r4 = reinterpret_cast<const float4*>(row);
            const double2* q2 = reinterpret_cast<const double2*>(q);
#pragma unroll 8
            for (int i = 0; i < D / 4; ++i) {
                const float4 d = __ldg(r4 + i);
                const double2 qa = q2[2 * i], qb = q2[2 * i + 1];
                acc = __fma_rn(qa.x, (double)d.x, acc);
                acc = __fma_rn(qa.y, (double)d.y, acc);
                acc = __fma_rn(qb.x, (double)d.z, acc);
                acc = __fma_rn(qb.y, (double)d.w, acc);
            }
        } else if (MODE == 3) {  // DADD chain of exact products computed off-chain
#pragma unroll 32
            for (int i = 0; i < D; ++i) {
                const double p = q[i] * (double)reg[i & 31];
                acc = __dadd_rn(acc, p);
            }
        } else if (MODE == 5 || MODE == 6) {  // explicit double-buffered register stream
            h = h * 6364136223846793005ull + 1442695040888963407ull;
            const float* rp = rows + (size_t)((h >> 33) % (unsigned)nrows) * D;
            acc += MODE == 5 ? dense_chain<8>(rp, q) : dense_chain<16>(rp, q);
        } else if (MODE == 4) {  // products in fp32 pairs? no: F2F-free widening via bit ops
#pragma unroll
            for (int i = 0; i < D; i += 32)
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const unsigned b = __float_as_uint(reg[j]);
                    const unsigned m = b & 0x7fffffffu;
                    const unsigned long long w =
                        m ? ((unsigned long long)(b & 0x80000000u) << 32) |
                                ((unsigned long long)(m + (896u << 23)) << 29)
                          : ((unsigned long long)(b & 0x80000000u) << 32);
                    acc = __fma_rn(q[i + j], __longlong_as_double((long long)w), acc);
                }
        }
    }
    long long t1 = clock64();
    if (lane == 0) cyc[gw] = t1 - t0;
    out[gw * 32 + lane] = acc;
}

int main() {
    float* rows;
    double *q, *out;
    long long* cyc;
    const int big = 200000;  // 614 MB of rows: DRAM resident
    cudaMalloc(&rows, sizeof(float) * (size_t)big * D);
    cudaMalloc(&q, sizeof(double) * D);
    cudaMalloc(&out, sizeof(double) * 148 * 64 * 32);
    cudaMalloc(&cyc, sizeof(long long) * 148 * 64);
    cudaMemset(rows, 0, sizeof(float) * (size_t)big * D);
    cudaMemset(q, 0, sizeof(double) * D);
    const char* names[] = {"dfma-reg", "dfma+f2f smem-q", "dfma ldg row", "dadd exact-prod", "dfma bit-widen",
                           "chain<8> L2rows", "chain<16> L2rows", "chain<8> DRAMrows", "chain<16> DRAMrows"};
    for (int mm = 0; mm < 9; ++mm)
        for (int wps : {1, 4, 12, 16}) {
            const int mode = mm < 7 ? mm : mm - 2;
            const int nrows = mm < 7 ? 4096 : big;
            const int blocks = 148, threads = 32 * wps, reps = 4;
            for (int it = 0; it < 2; ++it) {
                switch (mode) {
                    case 0: chain<0><<<blocks, threads>>>(rows, q, out, cyc, reps, nrows); break;
                    case 1: chain<1><<<blocks, threads>>>(rows, q, out, cyc, reps, nrows); break;
                    case 2: chain<2><<<blocks, threads>>>(rows, q, out, cyc, reps, nrows); break;
                    case 3: chain<3><<<blocks, threads>>>(rows, q, out, cyc, reps, nrows); break;
                    case 4: chain<4><<<blocks, threads>>>(rows, q, out, cyc, reps, nrows); break;
                    case 5: chain<5><<<blocks, threads>>>(rows, q, out, cyc, reps, nrows); break;
                    case 6: chain<6><<<blocks, threads>>>(rows, q, out, cyc, reps, nrows); break;
                }
            }
            cudaDeviceSynchronize();
            long long h[148 * 16];
            cudaMemcpy(h, cyc, sizeof(long long) * blocks * wps, cudaMemcpyDeviceToHost);
            double s = 0;
            for (int i = 0; i < blocks * wps; ++i) s += h[i];
            s /= blocks * wps;
            cudaError_t e = cudaGetLastError();
            if (e != cudaSuccess) { printf("%-18s warps/SM %2d : %s\n", names[mm], wps, cudaGetErrorString(e)); continue; }
            printf("%-18s warps/SM %2d : %6.1f cycles/element/warp (%.2f elem/clk/SM)\n", names[mm], wps,
                   s / (reps * D), wps * 32.0 * reps * D / s);
        }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
