// search_hybrid_c.cu — search_hybrid_kernel instantiated for entity-context batches (no required keywords).
#include "search_hybrid_kernel.cuh"

namespace fgb {

const void* hybrid_kernel_ptr_c(int nq4, int mode) { return hybrid_kernel_ptr<true, false>(nq4, mode); }
void hybrid_launch_c(const HybridLaunch& h, int nq4, uint64_t blocks, size_t smem, cudaStream_t s) {
    hybrid_launch_variant<true, false>(h, nq4, blocks, smem, s);
}

}  // namespace fgb
