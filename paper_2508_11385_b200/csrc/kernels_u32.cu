// Kernel instantiations for element type u32 (see coot_launch.cuh).
#include "coot_launch.cuh"

namespace coot {
COOT_INSTANTIATE(uint32_t)
}  // namespace coot
