// Kernel instantiations for subsequence search (dtw/cdtw only; search.py:172-173).
#include "ek_subseq.cuh"

namespace ekb {

#define EKB_SS_CASES(M)                                                   \
  case (M)*16 + E_DIAG4: return k_subseq<M, E_DIAG4>;                     \
  case (M)*16 + E_DIAG8: return k_subseq<M, E_DIAG8>;                     \
  case (M)*16 + E_DIAG16: return k_subseq<M, E_DIAG16>;                   \
  case (M)*16 + E_STR4: return k_subseq<M, E_STR4>;                       \
  case (M)*16 + E_STR8: return k_subseq<M, E_STR8>;                       \
  case (M)*16 + E_STR16: return k_subseq<M, E_STR16>;                     \
  case (M)*16 + E_STRB16: return k_subseq<M, E_STRB16>;                   \
  case (M)*16 + E_STRIP16: return k_subseq<M, E_STRIP16>;                 \
  case (M)*16 + E_STRIPB16: return k_subseq<M, E_STRIPB16>;

SubseqFn get_subseq(int mode, int eng) {
  switch (mode * 16 + eng) {
    EKB_SS_CASES(0)
    EKB_SS_CASES(1)
  }
  return nullptr;
}

SubseqUBFn get_subseq_ub(int mode) { return mode == 0 ? k_subseq_ub<0> : k_subseq_ub<1>; }

SubseqLBFn get_subseq_lb(int mode) { return mode == 0 ? k_subseq_lb<0> : k_subseq_lb<1>; }

}  // namespace ekb
