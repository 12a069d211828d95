// Kernel instantiations for element type f64 (see coot_launch.cuh).
#include "coot_launch.cuh"

namespace coot {
COOT_INSTANTIATE(double)
}  // namespace coot
