// Kernel instantiations for element type f16: launchers, dim sums, combine,
// fill (see coot_launch.cuh); fused kernels live in kernels_f16_acc*.cu.
#include "coot_launch.cuh"

namespace coot {
COOT_EXTERN_ACC(f16)
COOT_INSTANTIATE(f16)
}  // namespace coot
