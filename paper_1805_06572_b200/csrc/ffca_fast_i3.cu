// K3 v2 instantiations for I = 3 (separate TU so builds parallelise).
#include "ffca_fast_tma.cuh"

namespace ffca {
template cudaError_t launch_fast2<3, double>(const FastIterParams&, cudaStream_t);
template cudaError_t launch_fast2<3, float>(const FastIterParams&, cudaStream_t);
template int fast2_blocks_per_sm<3, double>();
template int fast2_blocks_per_sm<3, float>();
template int fast_tma_blocks_per_sm<3>();
}  // namespace ffca
