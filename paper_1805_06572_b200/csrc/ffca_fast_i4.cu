// K3 v2 instantiations for I = 4 (separate TU so builds parallelise).
#include "ffca_fast_tma.cuh"

namespace ffca {
template cudaError_t launch_fast2<4, double>(const FastIterParams&, cudaStream_t);
template cudaError_t launch_fast2<4, float>(const FastIterParams&, cudaStream_t);
template int fast2_blocks_per_sm<4, double>();
template int fast2_blocks_per_sm<4, float>();
template int fast_tma_blocks_per_sm<4>();
}  // namespace ffca
