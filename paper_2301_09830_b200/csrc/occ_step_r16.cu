// occ_step_r16.cu -- the per-phase step kernels for rank 16 (occ_step_impl.cuh).
#include "occ_step_impl.cuh"

namespace occ {
OCC_STEP_INSTANCE(16)
}  // namespace occ
