// KP instantiation for I = 1 (one translation unit per order: parallel builds)
#include "ffca_persist.cuh"

namespace ffca {
template int persist_slots<1>();
template int persist_max_chunks<1>();
template cudaError_t launch_persist<1>(const FastIterParams&, const PencilParams&,
                                       const PersistCtl&, cudaStream_t);
}  // namespace ffca
