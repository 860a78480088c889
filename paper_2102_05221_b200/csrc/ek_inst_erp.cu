// Kernel instantiations for K_ERP (see ek_launch.cuh).
#include "ek_launch.cuh"
namespace ekb {
EKB_INSTANTIATE_KIND(K_ERP)
}  // namespace ekb
