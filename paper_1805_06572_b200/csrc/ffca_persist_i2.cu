// KP instantiation for I = 2 (one translation unit per order: parallel builds)
#include "ffca_persist.cuh"

namespace ffca {
template int persist_slots<2>();
template int persist_max_chunks<2>();
template cudaError_t launch_persist<2>(const FastIterParams&, const PencilParams&,
                                       const PersistCtl&, cudaStream_t);
}  // namespace ffca
