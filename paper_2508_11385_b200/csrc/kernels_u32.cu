// Kernel instantiations for element type u32: launchers, dim sums, combine,
// fill (see coot_launch.cuh); fused kernels live in kernels_u32_acc*.cu.
#include "coot_launch.cuh"

namespace coot {
COOT_EXTERN_ACC(uint32_t)
COOT_INSTANTIATE(uint32_t)
}  // namespace coot
