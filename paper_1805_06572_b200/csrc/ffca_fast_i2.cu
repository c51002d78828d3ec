// K3 v2 instantiations for I = 2 (separate TU so builds parallelise).
#include "ffca_fast_tma.cuh"

namespace ffca {
template cudaError_t launch_fast2<2, double>(const FastIterParams&, cudaStream_t);
template cudaError_t launch_fast2<2, float>(const FastIterParams&, cudaStream_t);
template int fast2_blocks_per_sm<2, double>();
template int fast2_blocks_per_sm<2, float>();
template int fast_tma_blocks_per_sm<2>();
}  // namespace ffca
