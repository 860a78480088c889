// Kernel instantiations for K_MSM (see ek_launch.cuh).
#include "ek_launch.cuh"
namespace ekb {
EKB_INSTANTIATE_KIND(K_MSM)
}  // namespace ekb
