// Fused kernels (all drivers, catalog + interpreter) for element type s64,
// reduction kind ACC_SUMSQ (see coot_launch.cuh).
#include "coot_launch.cuh"

namespace coot {
COOT_INSTANTIATE_ACC(s64, ACC_SUMSQ)
}  // namespace coot
