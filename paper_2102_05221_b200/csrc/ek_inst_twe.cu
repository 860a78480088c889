// Kernel instantiations for K_TWE (see ek_launch.cuh).
#include "ek_launch.cuh"
namespace ekb {
EKB_INSTANTIATE_KIND(K_TWE)
}  // namespace ekb
