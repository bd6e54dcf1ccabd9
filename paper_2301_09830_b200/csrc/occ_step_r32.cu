// occ_step_r32.cu -- the per-phase step kernels for rank 32 (occ_step_impl.cuh).
#include "occ_step_impl.cuh"

namespace occ {
OCC_STEP_INSTANCE(32)
}  // namespace occ
