// Kernel instantiations for K_DTW (see ek_launch.cuh).
#include "ek_launch.cuh"
namespace ekb {
EKB_INSTANTIATE_KIND(K_DTW)
}  // namespace ekb
