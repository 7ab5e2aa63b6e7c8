// mem_pool.cu — device memory of every DevBuf (fg_cuda.hpp): the device's
// stream-ordered pool, with freed blocks cached for reuse.
#include <cstdint>
#include <map>
#include <mutex>

#include "fg_cuda.hpp"

namespace fgb {

namespace {
struct DevPool {
    cudaMemPool_t pool = nullptr;
    cudaStream_t stream = nullptr;
};
// never destroyed: DevBufs held by static objects of other libraries (the
// drop-in shim's mirror cache) may be released during process exit
std::mutex& pool_mu() {
    static std::mutex* m = new std::mutex;
    return *m;
}
std::map<int, DevPool>& pools() {
    static std::map<int, DevPool>* m = new std::map<int, DevPool>;
    return *m;
}
DevPool& pool_of(int device) {
    std::lock_guard<std::mutex> lock(pool_mu());
    auto it = pools().find(device);
    if (it != pools().end()) return it->second;
    DevPool p;
    FGB_CUDA(cudaDeviceGetDefaultMemPool(&p.pool, device));
    uint64_t keep = UINT64_MAX;  // cache freed blocks instead of returning them to the driver
    FGB_CUDA(cudaMemPoolSetAttribute(p.pool, cudaMemPoolAttrReleaseThreshold, &keep));
    FGB_CUDA(cudaStreamCreateWithFlags(&p.stream, cudaStreamNonBlocking));
    return pools().emplace(device, p).first->second;
}
}  // namespace

void* pool_alloc(size_t bytes, int* device) {
    int dev = 0;
    FGB_CUDA(cudaGetDevice(&dev));
    DevPool& P = pool_of(dev);
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, bytes, P.stream);
    if (e == cudaErrorMemoryAllocation) {  // hand the cached blocks back and retry once
        cudaGetLastError();
        FGB_CUDA(cudaDeviceSynchronize());
        FGB_CUDA(cudaMemPoolTrimTo(P.pool, 0));
        e = cudaMallocAsync(&p, bytes, P.stream);
    }
    FGB_CUDA(e);
    // ordered before any use on the caller's streams
    FGB_CUDA(cudaStreamSynchronize(P.stream));
    *device = dev;
    return p;
}

void pool_free(void* p, int device) noexcept {
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) {
        cudaGetLastError();
        return;  // runtime already unloaded (process exit)
    }
    if (cur != device) cudaSetDevice(device);
    DevPool* P = nullptr;
    {
        std::lock_guard<std::mutex> lock(pool_mu());
        auto it = pools().find(device);
        if (it != pools().end()) P = &it->second;
    }
    if (cudaDeviceSynchronize() == cudaSuccess && P) {
        cudaFreeAsync(p, P->stream);
    } else {
        cudaFree(p);
    }
    cudaGetLastError();
    if (cur != device) cudaSetDevice(cur);
}

}  // namespace fgb
