// Fused kernels (all drivers, catalog + interpreter) for element type e4m3,
// reduction kind ACC_SUM (see coot_launch.cuh).
#include "coot_launch.cuh"

namespace coot {
COOT_INSTANTIATE_ACC(e4m3, ACC_SUM)
}  // namespace coot
