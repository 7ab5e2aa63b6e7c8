// search_hybrid_r.cu — search_hybrid_kernel instantiated for required-keyword batches (no entity context).
#include "search_hybrid_kernel.cuh"

namespace fgb {

const void* hybrid_kernel_ptr_r(int nq4, int mode) { return hybrid_kernel_ptr<false, true>(nq4, mode); }
void hybrid_launch_r(const HybridLaunch& h, int nq4, uint64_t blocks, size_t smem, cudaStream_t s) {
    hybrid_launch_variant<false, true>(h, nq4, blocks, smem, s);
}

}  // namespace fgb
