// K3 v2 instantiations for I = 1 (separate TU so builds parallelise).
#include "ffca_fast_tma.cuh"

namespace ffca {
template cudaError_t launch_fast2<1, double>(const FastIterParams&, cudaStream_t);
template cudaError_t launch_fast2<1, float>(const FastIterParams&, cudaStream_t);
template int fast2_blocks_per_sm<1, double>();
template int fast2_blocks_per_sm<1, float>();
template int fast_tma_blocks_per_sm<1>();
}  // namespace ffca
