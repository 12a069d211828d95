// Fused kernels (all drivers, catalog + interpreter) for element type e5m2,
// reduction kind ACC_IMIN (see coot_launch.cuh).
#include "coot_launch.cuh"

namespace coot {
COOT_INSTANTIATE_ACC(e5m2, ACC_IMIN)
}  // namespace coot
