// occ_step_r8.cu -- the per-phase step kernels for rank 8 (occ_step_impl.cuh).
#include "occ_step_impl.cuh"

namespace occ {
OCC_STEP_INSTANCE(8)
}  // namespace occ
