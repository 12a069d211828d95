// Fused kernels (all drivers, catalog + interpreter) for element type f64,
// reduction kind ACC_NONE (see coot_launch.cuh).
#include "coot_launch.cuh"

namespace coot {
COOT_INSTANTIATE_ACC(double, ACC_NONE)
}  // namespace coot
