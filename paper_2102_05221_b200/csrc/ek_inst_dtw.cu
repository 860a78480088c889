// Kernel instantiations for K_DTW (see ek_launch.cuh).
#include "ek_launch.cuh"
namespace ekb {
EKB_INSTANTIATE_KIND(K_DTW)
}  // namespace ekb

#ifdef EKB_TRACE
// debug builds: the per-warp timeline of the last dtw k_nn launch (ekb::g_trace of this unit)
extern "C" int ek_debug_trace(unsigned long long* out, int n) {
  if (n > 8192 * 5) n = 8192 * 5;
  return (int)cudaMemcpyFromSymbol(out, ekb::g_trace, sizeof(unsigned long long) * n);
}
#endif
