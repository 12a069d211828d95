// Kernel instantiations for element type e5m2: launchers, dim sums, combine,
// fill (see coot_launch.cuh); fused kernels live in kernels_e5m2_acc*.cu.
#include "coot_launch.cuh"

namespace coot {
COOT_EXTERN_ACC(e5m2)
COOT_INSTANTIATE(e5m2)
}  // namespace coot
