// Fused kernels (all drivers, catalog + interpreter) for element type f16,
// reduction kind ACC_SUM (see coot_launch.cuh).
#include "coot_launch.cuh"

namespace coot {
COOT_INSTANTIATE_ACC(f16, ACC_SUM)
}  // namespace coot
