// occ_step_r64.cu -- the per-phase step kernels for rank 64 (occ_step_impl.cuh).
#include "occ_step_impl.cuh"

namespace occ {
OCC_STEP_INSTANCE(64)
}  // namespace occ
