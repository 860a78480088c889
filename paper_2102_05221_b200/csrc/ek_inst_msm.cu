// Kernel instantiations for K_MSM (see ek_launch.cuh).
#include "ek_launch.cuh"
namespace ekb {
EKB_INSTANTIATE_KIND(K_MSM)
}  // namespace ekb

#ifdef EKB_LIVE
// debug builds: the evaluated / live cell counters of this unit's diagonal engines (reset on read)
extern "C" int ek_debug_live_msm(unsigned long long* out) {
  int e = (int)cudaMemcpyFromSymbol(out, ekb::g_live, 2 * sizeof(unsigned long long));
  const unsigned long long z[2] = {0, 0};
  return e | (int)cudaMemcpyToSymbol(ekb::g_live, z, sizeof z);
}
#endif
