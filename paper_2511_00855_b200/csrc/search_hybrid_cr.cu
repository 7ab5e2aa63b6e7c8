// search_hybrid_cr.cu — search_hybrid_kernel instantiated for batches mixing both (and forced plain batches).
#include "search_hybrid_kernel.cuh"

namespace fgb {

const void* hybrid_kernel_ptr_cr(int nq4, int mode) { return hybrid_kernel_ptr<true, true>(nq4, mode); }
void hybrid_launch_cr(const HybridLaunch& h, int nq4, uint64_t blocks, size_t smem, cudaStream_t s) {
    hybrid_launch_variant<true, true>(h, nq4, blocks, smem, s);
}

}  // namespace fgb
