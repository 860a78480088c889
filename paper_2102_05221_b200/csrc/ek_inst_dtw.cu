// Kernel instantiations for K_DTW (see ek_launch.cuh).
#include <algorithm>
#include "ek_launch.cuh"
#include "ek_nn2.cuh"
namespace ekb {
EKB_INSTANTIATE_KIND(K_DTW)

cudaError_t nn2_pad(int f32, const double* src, const long long* off, int n, int L, int pitch, void* dst,
                    cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((pitch + 255) / 256), (unsigned)n);
  if (f32) k_pad_series<float><<<grid, 256, 0, st>>>(src, off, n, L, pitch, (float*)dst);
  else k_pad_series<double><<<grid, 256, 0, st>>>(src, off, n, L, pitch, (double*)dst);
  return cudaGetLastError();
}

template <int MODE, bool V>
static cudaError_t nn2_go(int nsm, long long warp_units, cudaStream_t st, const void* QP, const void* CP, int pitch,
                          int L, int nq, int ncand, const int* order, int rank_lo, int rank_mid, int rank_hi, int K1,
                          int K2, int w, unsigned long long* cutbits, NNAcc acc, int* qnext, unsigned long long* qdone, const float* skeys,
                          const float2* envq, int lmax, int* qstop) {
  using R = real_t<MODE>;
  auto fn = k_nn2<MODE, V>;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 128, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const long long want = (warp_units + 3) / 4;
  const long long grid = std::min<long long>((long long)nsm * per_sm, std::max<long long>(1, want));
  fn<<<(unsigned)grid, 128, 0, st>>>((const R*)QP, (const R*)CP, pitch, L, nq, ncand, order, rank_lo, rank_mid,
                                     rank_hi, K1, K2, w, cutbits, acc, qnext, qdone, skeys, envq, lmax, qstop);
  return cudaGetLastError();
}

cudaError_t nn2_launch(int mode, bool virt0, int nsm, long long warp_units, cudaStream_t st, const void* QP,
                       const void* CP, int pitch, int L, int nq, int ncand, const int* order, int rank_lo,
                       int rank_mid, int rank_hi, int K1, int K2, int w, unsigned long long* cutbits, NNAcc acc,
                       int* qnext, unsigned long long* qdone, const float* skeys, const float2* envq, int lmax,
                       int* qstop) {
#define EKB_NN2_GO(M, V)                                                                                       \
  return nn2_go<M, V>(nsm, warp_units, st, QP, CP, pitch, L, nq, ncand, order, rank_lo, rank_mid, rank_hi, K1, \
                      K2, w, cutbits, acc, qnext, qdone, skeys, envq, lmax, qstop)
  switch (mode * 2 + (virt0 ? 1 : 0)) {
    case 0: EKB_NN2_GO(0, false);
    case 1: EKB_NN2_GO(0, true);
    case 2: EKB_NN2_GO(1, false);
    case 3: EKB_NN2_GO(1, true);
    case 4: EKB_NN2_GO(2, false);
    case 5: EKB_NN2_GO(2, true);
    case 6: EKB_NN2_GO(3, false);
    case 7: EKB_NN2_GO(3, true);
  }
#undef EKB_NN2_GO
  return cudaErrorInvalidValue;
}
}  // namespace ekb

#ifdef EKB_TRACE
// debug builds: the per-warp timeline of the last dtw k_nn launch (ekb::g_trace of this unit)
extern "C" int ek_debug_trace(unsigned long long* out, int n) {
  if (n > 8192 * 8) n = 8192 * 8;
  return (int)cudaMemcpyFromSymbol(out, ekb::g_trace, sizeof(unsigned long long) * n);
}
// the long pairs of the k_nn2 launches since the last call (count returned, log reset)
extern "C" int ek_debug_plog(unsigned long long* out, int max_rows) {
  unsigned int n = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&n, ekb::g_plog_n, sizeof(n));
  if (n > 32768u) n = 32768u;
  if ((int)n > max_rows) n = (unsigned)max_rows;
  if (n && out) cudaMemcpyFromSymbol(out, ekb::g_plog, sizeof(unsigned long long) * 4 * n);
  const unsigned int z = 0;
  cudaMemcpyToSymbol(ekb::g_plog_n, &z, sizeof(z));
  return (int)n;
}
#endif

#ifdef EKB_LIVE
// debug builds: the evaluated / live cell counters of this unit's diagonal engines (reset on read)
extern "C" int ek_debug_live_dtw(unsigned long long* out) {
  int e = (int)cudaMemcpyFromSymbol(out, ekb::g_live, 2 * sizeof(unsigned long long));
  const unsigned long long z[2] = {0, 0};
  return e | (int)cudaMemcpyToSymbol(ekb::g_live, z, sizeof z);
}
extern "C" int ek_debug_sn_dtw(unsigned long long* out) {
  int e = (int)cudaMemcpyFromSymbol(out, ekb::g_sn, 8 * sizeof(unsigned long long));
  static const unsigned long long z[8] = {};
  return e | (int)cudaMemcpyToSymbol(ekb::g_sn, z, sizeof z);
}
extern "C" int ek_debug_corr_dtw(unsigned long long* out) {
  int e = (int)cudaMemcpyFromSymbol(out, ekb::g_corr, 16 * 33 * sizeof(unsigned long long));
  static const unsigned long long z[16 * 33] = {};
  return e | (int)cudaMemcpyToSymbol(ekb::g_corr, z, sizeof z);
}
#endif
