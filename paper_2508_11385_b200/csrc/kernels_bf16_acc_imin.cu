// Fused kernels (all drivers, catalog + interpreter) for element type bf16,
// reduction kind ACC_IMIN (see coot_launch.cuh).
#include "coot_launch.cuh"

namespace coot {
COOT_INSTANTIATE_ACC(bf16, ACC_IMIN)
}  // namespace coot
