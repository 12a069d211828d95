// Kernel instantiations for element type s64: launchers, dim sums, combine,
// fill (see coot_launch.cuh); fused kernels live in kernels_s64_acc*.cu.
#include "coot_launch.cuh"

namespace coot {
COOT_EXTERN_ACC(s64)
COOT_INSTANTIATE(s64)
}  // namespace coot
