// KP instantiation for I = 3 (one translation unit per order: parallel builds)
#include "ffca_persist.cuh"

namespace ffca {
template int persist_slots<3>();
template int persist_max_chunks<3>();
template cudaError_t launch_persist<3>(const FastIterParams&, const PencilParams&,
                                       const PersistCtl&, cudaStream_t);
}  // namespace ffca
