// search_hybrid.cu — host side of the certified hybrid search kernel
// (search_hybrid_kernel.cuh): shared-memory sizing, occupancy and the choice
// among its per-feature instantiations (search_hybrid_{c,r,cr}.cu).
#include <algorithm>
#include <cstdlib>

#include "search_hybrid_kernel.cuh"

namespace fgb {

const void* hybrid_kernel_ptr_c(int nq4, int mode);
const void* hybrid_kernel_ptr_r(int nq4, int mode);
const void* hybrid_kernel_ptr_cr(int nq4, int mode);
void hybrid_launch_c(const HybridLaunch& h, int nq4, uint64_t blocks, size_t smem, cudaStream_t s);
void hybrid_launch_r(const HybridLaunch& h, int nq4, uint64_t blocks, size_t smem, cudaStream_t s);
void hybrid_launch_cr(const HybridLaunch& h, int nq4, uint64_t blocks, size_t smem, cudaStream_t s);

namespace {

int nq4_of(uint32_t dstride) {
    const uint32_t need = ((dstride >> 2) + 31) / 32;
    for (int v : {1, 2, 3, 4, 6, 8})
        if (static_cast<uint32_t>(v) >= need) return v;
    return 0;
}

const void* kernel_for(const HybridLaunch& h) {
    const int v = nq4_of(h.p.c.dstride);
    switch (h.variant) {
        case kHybCtx: return hybrid_kernel_ptr_c(v, h.p.mode);
        case kHybReq: return hybrid_kernel_ptr_r(v, h.p.mode);
        default: return hybrid_kernel_ptr_cr(v, h.p.mode);
    }
}

}  // namespace

size_t hybrid_warp_smem(const HybridLaunch& h) {
    if (nq4_of(h.p.c.dstride) == 0) return 0;
    const size_t b = carve_bytes(h);
    return b <= 227 * 1024 ? b : 0;
}

uint64_t hybrid_slots(const HybridLaunch& h, uint64_t nq, int device) {
    const size_t smem = hybrid_warp_smem(h);
    const void* k = kernel_for(h);
    FGB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0, sms = 0;
    FGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32, smem));
    FGB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    per_sm = std::max(per_sm, 1);
    if (const char* e = std::getenv("FGB_SEARCH_WARPS_PER_SM"))
        per_sm = std::max(1, std::min(per_sm, std::atoi(e)));
    return std::max<uint64_t>(1, std::min<uint64_t>(nq, static_cast<uint64_t>(sms) * per_sm));
}

void launch_search_hybrid(const HybridLaunch& h, uint64_t blocks, cudaStream_t s) {
    const size_t smem = hybrid_warp_smem(h);
    const int v = nq4_of(h.p.c.dstride);
    switch (h.variant) {
        case kHybCtx: hybrid_launch_c(h, v, blocks, smem, s); break;
        case kHybReq: hybrid_launch_r(h, v, blocks, smem, s); break;
        default: hybrid_launch_cr(h, v, blocks, smem, s); break;
    }
    FGB_LAUNCH("search_hybrid_kernel");
}

}  // namespace fgb
