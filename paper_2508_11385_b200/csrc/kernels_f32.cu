// Kernel instantiations for element type f32: launchers, dim sums, combine,
// fill (see coot_launch.cuh); fused kernels live in kernels_f32_acc*.cu.
#include "coot_launch.cuh"

namespace coot {
COOT_EXTERN_ACC(float)
COOT_INSTANTIATE(float)
}  // namespace coot
