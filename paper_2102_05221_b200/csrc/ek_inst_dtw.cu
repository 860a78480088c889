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

#ifdef EKB_LIVE
// debug builds: the evaluated / live cell counters of this unit's diagonal engines (reset on read)
extern "C" int ek_debug_live_dtw(unsigned long long* out) {
  int e = (int)cudaMemcpyFromSymbol(out, ekb::g_live, 2 * sizeof(unsigned long long));
  const unsigned long long z[2] = {0, 0};
  return e | (int)cudaMemcpyToSymbol(ekb::g_live, z, sizeof z);
}
#endif
