// Fused kernels (all drivers, catalog + interpreter) for element type u32,
// reduction kind ACC_VAR (see coot_launch.cuh).
#include "coot_launch.cuh"

namespace coot {
COOT_INSTANTIATE_ACC(uint32_t, ACC_VAR)
}  // namespace coot
