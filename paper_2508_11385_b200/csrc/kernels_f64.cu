// Kernel instantiations for element type f64: launchers, dim sums, combine,
// fill (see coot_launch.cuh); fused kernels live in kernels_f64_acc*.cu.
#include "coot_launch.cuh"

namespace coot {
COOT_EXTERN_ACC(double)
COOT_INSTANTIATE(double)
}  // namespace coot
