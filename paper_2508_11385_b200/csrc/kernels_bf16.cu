// Kernel instantiations for element type bf16: launchers, dim sums, combine,
// fill (see coot_launch.cuh); fused kernels live in kernels_bf16_acc*.cu.
#include "coot_launch.cuh"

namespace coot {
COOT_EXTERN_ACC(bf16)
COOT_INSTANTIATE(bf16)
}  // namespace coot
