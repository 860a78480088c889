// Kernel instantiations for K_WDTW (see ek_launch.cuh).
#include "ek_launch.cuh"
namespace ekb {
EKB_INSTANTIATE_KIND(K_WDTW)
}  // namespace ekb
