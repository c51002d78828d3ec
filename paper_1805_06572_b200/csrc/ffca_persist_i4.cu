// KP instantiation for I = 4 (one translation unit per order: parallel builds)
#include "ffca_persist.cuh"

namespace ffca {
template int persist_slots<4>();
template int persist_max_chunks<4>();
template cudaError_t launch_persist<4>(const FastIterParams&, const PencilParams&,
                                       const PersistCtl&, cudaStream_t);
}  // namespace ffca
