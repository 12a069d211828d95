// Kernel instantiations for element type s64 (see coot_launch.cuh).
#include "coot_launch.cuh"

namespace coot {
COOT_INSTANTIATE(s64)
}  // namespace coot
