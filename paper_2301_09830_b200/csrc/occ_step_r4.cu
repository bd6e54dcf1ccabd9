// occ_step_r4.cu -- the per-phase step kernels for rank 4 (occ_step_impl.cuh).
#include "occ_step_impl.cuh"

namespace occ {
OCC_STEP_INSTANCE(4)
}  // namespace occ
