// Kernel instantiations for element type e4m3: launchers, dim sums, combine,
// fill (see coot_launch.cuh); fused kernels live in kernels_e4m3_acc*.cu.
#include "coot_launch.cuh"

namespace coot {
COOT_EXTERN_ACC(e4m3)
COOT_INSTANTIATE(e4m3)
}  // namespace coot
