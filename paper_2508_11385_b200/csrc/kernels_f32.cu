// Kernel instantiations for element type f32 (see coot_launch.cuh).
#include "coot_launch.cuh"

namespace coot {
COOT_INSTANTIATE(float)
}  // namespace coot
