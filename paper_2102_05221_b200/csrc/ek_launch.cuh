// ek_launch.cuh -- typed kernel-pointer tables, one instantiation unit per distance kind
// (ek_inst_<kind>.cu) so the template expansion compiles in parallel.
#pragma once
#include "ek_kernels.cuh"
#include "ek_refcells.cuh"

namespace ekb {

using PairsFn = void (*)(const double*, const PairDesc*, int, int, Params, double*, int*);
using TriFn = void (*)(const double*, const long long*, const int*, int, int, int, Params, double*, long long,
                      long long, double*, unsigned long long*, int*);
using NNFn = void (*)(const double*, const long long*, const int*, int, const double*, const long long*,
                      const int*, int, const int*, int, int, int, int, int, int, int, Params, int, unsigned long long*,
                      NNAcc, int*, const float*, const float2*, int2*, int*, int*);
using NNFixFn = void (*)(const double*, const long long*, const int*, const double*, const long long*, const int*,
                         int, const int2*, const int*, int, int, Params, unsigned long long*, NNAcc, int*,
                         int2*, int*);
using RefFn = void (*)(const double*, const PairDesc*, int, int, Params, double*, long long*);
using UBFn = void (*)(const double*, const long long*, const int*, int, const double*, const long long*,
                      const int*, int, const int*, int, Params, unsigned long long*, int);

// diagonal_upper_bound (engines.py:87-103): the diagonal then the last column, the
// cost of one admissible path, seeds a query's cutoff.  One warp per query, terms
// summed in parallel and rounded up (k_ub_init).
// (FP32 mode: the same terms in float, from the float-rounded series, as the DP sees them)
template <int KIND, int MODE, class Acc>
__device__ __forceinline__ real_t<MODE> ub_term(const Acc& X, const Acc& Y, int nc, int k, const Params& pp) {
  using R = real_t<MODE>;
  auto xv = [&](int i) -> R { return i < 0 ? pad_before<KIND, R>((R)X[0]) : (R)X[i]; };
  auto yv = [&](int j) -> R { return j < 0 ? pad_before<KIND, R>((R)Y[0]) : (R)Y[j]; };
  if (k <= nc) {  // canonical(k, k)
    const RowD<KIND, R> r = make_row<KIND, MODE>(xv(k - 1), xv(k - 2), pp);
    const R y = yv(k - 1);
    if constexpr (KIND == K_WDTW) return dmul(pcost<MODE>(r.x, y), (R)pp.wt[0]);
    else if constexpr (KIND == K_MSM) return fabs(dsub(r.x, y));
    else if constexpr (KIND == K_TWE)
      return dadd(dadd(pcost<MODE>(r.x, y), pcost<MODE>(k >= 2 ? (R)X[k - 2] : (R)0.0, k >= 2 ? (R)Y[k - 2] : (R)0.0)),
                  dmul((R)pp.nu, dadd((R)0.0, (R)0.0)));
    else return pcost<MODE>(r.x, y);
  }
  // alt_row(k, nc) for the rows below the diagonal's end
  const RowD<KIND, R> r = make_row<KIND, MODE>(xv(k - 1), xv(k - 2), pp);
  const R y = (R)Y[nc - 1];
  if constexpr (KIND == K_WDTW) return dmul(pcost<MODE>(r.x, y), (R)pp.wt[k - nc]);
  else if constexpr (KIND == K_ERP || KIND == K_TWE) return r.ar;
  else if constexpr (KIND == K_MSM) {
    const R e = dsub(r.x, y);
    return msm_alt(sign_bit(e) != r.s, (R)pp.msm_c, r.dr, fabs(e));
  } else return pcost<MODE>(r.x, y);
}

template <int KIND, int MODE>
__global__ void __launch_bounds__(128) k_ub_init(const double* __restrict__ Q, const long long* __restrict__ qoff,
                                                 const int* __restrict__ qlen, int nq, const double* __restrict__ C,
                                                 const long long* __restrict__ coff, const int* __restrict__ clen,
                                                 int ncand, const int* __restrict__ order, int win, Params prm,
                                                 unsigned long long* cutbits, int nseed) {
  // one warp per (query, seed rank); the query's cutoff (prefilled +inf) takes the least
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long wid = (long long)blockIdx.x * 4 + wib;
  const int q = (int)(wid / nseed), rk = (int)(wid % nseed);
  if (q >= nq || rk >= ncand) return;
  const int c = order ? order[(long long)q * ncand + rk] : rk;
  const int lq = qlen[q], lc = clen[c];
  const bool q_rows = lq >= lc;
  const double* X = q_rows ? Q + qoff[q] : C + coff[c];
  const double* Y = q_rows ? C + coff[c] : Q + qoff[q];
  const int nl = q_rows ? lq : lc, nc = q_rows ? lc : lq;
  const int w = win < 0 ? nl : win;
  if (w < nl - nc) return;  // infeasible: +inf, the prefilled value
  const Params pp = pair_params(prm, nl);
  // Every term is >= 0.  Summed in any order with every addition rounded up, the total
  // is >= the exact path cost; one more relative 2^-24 (rounded up) covers the
  // round-to-nearest error of the DP's own in-order sum (<= ~n 2^-53, n < 2^29), so
  // the seed is never below the candidate's DP value -- it stays a valid cutoff.
  //
  // FP32 mode: the float terms are summed exactly as above (rounded up, in double), and
  // the DP's in-order float sum of n of them is at most (1 + 2^-24)^n times their exact
  // sum, covered by (1 + (n+2) 2^-23); the seed is then rounded up to a float.
  double total = 0.0;
  for (int k = 1 + lane; k <= nl; k += 32) total = __dadd_ru(total, (double)ub_term<KIND, MODE>(X, Y, nc, k, pp));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) total = __dadd_ru(total, __shfl_xor_sync(FULL, total, o));
  if constexpr ((MODE & M_F32) != 0) {
    total = __dmul_ru(total, 1.0 + (double)(nl + 2) * 0x1p-23);
    total = (double)__double2float_ru(total);
  } else {
    total = __dmul_ru(total, 1.0 + 0x1p-24);
  }
  if (lane == 0) atomicMin(cutbits + q, (unsigned long long)__double_as_longlong(total));
}

// Single pairs with the reference's own cells_computed (ek_refcells.cuh): one warp per
// pair on the row-stripe engine (S = 16: STR16 / STRB16 / STR16_EA).  pd.pad_ selects
// the count: 1 ea rows, 2 eapruned replay, 3 pruned_only (eapruned replay at the
// diagonal upper bound, computed here in DP order, engines.py:87-118).
__host__ __device__ constexpr int ref_warp_stride(int lmax, int eng) {
  return warp_stride(lmax, eng) + ((lmax + 1) * kRefWords * 2 + (lmax + 1) + 7) / 8;
}

template <int KIND, int MODE, int ENG>
__global__ void __launch_bounds__(32) k_pairs_ref(const double* __restrict__ series,
                                                  const PairDesc* __restrict__ pairs, int npairs, int lmax,
                                                  Params prm, double* __restrict__ out_cost,
                                                  long long* __restrict__ out_cells) {
  extern __shared__ double smem[];
  constexpr int PAD = engine_pad(ENG);
  constexpr bool BANDED = ENG >= E_STRB16;
  constexpr bool EA = ENG == E_STR16_EA;
  const int lane = threadIdx.x & 31;
  double* X = smem + PAD;
  double* Y = X + series_slot(lmax, PAD);
  double* tab = Y - PAD + series_slot(lmax, PAD);
  unsigned short* bits = (unsigned short*)(smem + warp_stride(lmax, ENG));
  unsigned char* vbl = (unsigned char*)(bits + (lmax + 1) * kRefWords);
  __shared__ double terms[32];
  for (int pid = blockIdx.x; pid < npairs; pid += gridDim.x) {
    const PairDesc pd = pairs[pid];
    const Params pp = pair_params(prm, max(pd.nl, pd.nc));
    const int nl = pd.nl, nc = pd.nc, w = pd.w;
    __syncwarp();
    stage_series<KIND>(X, series + pd.xoff, nl, PAD);
    stage_series<KIND>(Y, series + pd.yoff, nc, PAD);
    const int tablen = max(nl, nc) + 1;
    const double* tabe = engine_table<KIND, ENG>(tab, tablen, lmax, pp);
    unsigned* bw = (unsigned*)bits;
    for (int k = lane; k < (nl + 1) * kRefWords / 2; k += 32) bw[k] = 0u;
    for (int k = lane; k <= nl; k += 32) vbl[k] = 0;
    __syncwarp();
    double cut = pd.cut;
    if (pd.pad_ == 3) {  // diagonal_upper_bound, summed in DP order
      double total = 0.0;
      for (int base = 1; base <= nl; base += 32) {
        const int k = base + lane;
        terms[lane] = (k <= nl) ? ub_term<KIND, MODE>((const double*)X, (const double*)Y, nc, k, pp) : 0.0;
        __syncwarp();
        if (lane == 0)
          for (int u = 0; u < min(32, nl - base + 1); ++u) total = dadd(total, terms[u]);
        __syncwarp();
      }
      cut = __shfl_sync(FULL, total, 0);
    }
    const RowBits rec{bits, vbl};
    const StripeResult r = stripe_pair<KIND, MODE, 16, BANDED, false, EA>(SmemSeries{X, nl}, nl, SmemSeries{Y, nc},
                                                                           nc, w, cut, nullptr, tabe, tablen, pp, rec);
    __syncwarp();
    if (lane == 0) {
      long long cells;
      if (pd.pad_ == 1) cells = ea_cells(nl, nc, w, r.ea_row == 0x7fffffff ? nl : r.ea_row);
      else cells = eapruned_cells(bits, vbl, nl, nc, w, KIND == K_ERP);
      out_cost[pid] = r.cost;
      out_cells[pid] = cells;
    }
  }
}

template <int KIND>
RefFn get_pairs_ref(int mode, int eng) {
  switch (mode * 32 + eng) {
    case 0 * 32 + E_STR16: return k_pairs_ref<KIND, 0, E_STR16>;
    case 1 * 32 + E_STR16: return k_pairs_ref<KIND, 1, E_STR16>;
    case 0 * 32 + E_STRB16: return k_pairs_ref<KIND, 0, E_STRB16>;
    case 1 * 32 + E_STRB16: return k_pairs_ref<KIND, 1, E_STRB16>;
    case 0 * 32 + E_STR16_EA: return k_pairs_ref<KIND, 0, E_STR16_EA>;
    case 1 * 32 + E_STR16_EA: return k_pairs_ref<KIND, 1, E_STR16_EA>;
  }
  return nullptr;
}

#define EKB_ENG_CASES(M, FN)                                                                         \
  case (M)*32 + E_DIAG4: return FN<KIND, M, E_DIAG4>;                                               \
  case (M)*32 + E_DIAG8: return FN<KIND, M, E_DIAG8>;                                               \
  case (M)*32 + E_DIAG16: return FN<KIND, M, E_DIAG16>;                                             \
  case (M)*32 + E_STR4: return FN<KIND, M, E_STR4>;                                                 \
  case (M)*32 + E_STR8: return FN<KIND, M, E_STR8>;                                                 \
  case (M)*32 + E_STR16: return FN<KIND, M, E_STR16>;                                               \
  case (M)*32 + E_STRB16: return FN<KIND, M, E_STRB16>;                                             \
  case (M)*32 + E_STRIP16: return FN<KIND, M, E_STRIP16>;                                           \
  case (M)*32 + E_STRIPB16: return FN<KIND, M, E_STRIPB16>;

template <int KIND>
PairsFn get_pairs(int mode, int eng) {
  switch (mode * 32 + eng) {
    EKB_ENG_CASES(0, k_pairs)
    EKB_ENG_CASES(1, k_pairs)
    EKB_ENG_CASES(2, k_pairs)
    EKB_ENG_CASES(3, k_pairs)
    case 0 * 32 + E_STR16_EA: return k_pairs<KIND, 0, E_STR16_EA>;
    case 1 * 32 + E_STR16_EA: return k_pairs<KIND, 1, E_STR16_EA>;
    case 2 * 32 + E_STR16_EA: return k_pairs<KIND, 2, E_STR16_EA>;
    case 3 * 32 + E_STR16_EA: return k_pairs<KIND, 3, E_STR16_EA>;
    case 0 * 32 + E_STRIP16_EA: return k_pairs<KIND, 0, E_STRIP16_EA>;
    case 1 * 32 + E_STRIP16_EA: return k_pairs<KIND, 1, E_STRIP16_EA>;
    case 2 * 32 + E_STRIP16_EA: return k_pairs<KIND, 2, E_STRIP16_EA>;
    case 3 * 32 + E_STRIP16_EA: return k_pairs<KIND, 3, E_STRIP16_EA>;
  }
  return nullptr;
}

template <int KIND>
TriFn get_triangle(int mode, int eng) {
  switch (mode * 32 + eng) {
    EKB_ENG_CASES(0, k_triangle)
    EKB_ENG_CASES(1, k_triangle)
    EKB_ENG_CASES(2, k_triangle)
    EKB_ENG_CASES(3, k_triangle)
    case 0 * 32 + E_STR16H: return k_triangle<KIND, 0, E_STR16H>;
    case 1 * 32 + E_STR16H: return k_triangle<KIND, 1, E_STR16H>;
    case 2 * 32 + E_STR16H: return k_triangle<KIND, 2, E_STR16H>;
    case 3 * 32 + E_STR16H: return k_triangle<KIND, 3, E_STR16H>;
    case 0 * 32 + E_DIAG4H: return k_triangle<KIND, 0, E_DIAG4H>;
    case 1 * 32 + E_DIAG4H: return k_triangle<KIND, 1, E_DIAG4H>;
    case 2 * 32 + E_DIAG4H: return k_triangle<KIND, 2, E_DIAG4H>;
    case 3 * 32 + E_DIAG4H: return k_triangle<KIND, 3, E_DIAG4H>;
    case 0 * 32 + E_DIAG2: return k_triangle<KIND, 0, E_DIAG2>;
    case 1 * 32 + E_DIAG2: return k_triangle<KIND, 1, E_DIAG2>;
    case 2 * 32 + E_DIAG2: return k_triangle<KIND, 2, E_DIAG2>;
    case 3 * 32 + E_DIAG2: return k_triangle<KIND, 3, E_DIAG2>;
  }
  return nullptr;
}

template <int KIND>
NNFn get_nn(int mode, int eng) {
  switch (mode * 32 + eng) {
    EKB_ENG_CASES(0, k_nn)
    EKB_ENG_CASES(1, k_nn)
    EKB_ENG_CASES(2, k_nn)
    EKB_ENG_CASES(3, k_nn)
    case 0 * 32 + E_GDIAG4: return k_nn<KIND, 0, E_GDIAG4>;
    case 1 * 32 + E_GDIAG4: return k_nn<KIND, 1, E_GDIAG4>;
    case 2 * 32 + E_GDIAG4: return k_nn<KIND, 2, E_GDIAG4>;
    case 3 * 32 + E_GDIAG4: return k_nn<KIND, 3, E_GDIAG4>;
    case 0 * 32 + E_GDIAG8: return k_nn<KIND, 0, E_GDIAG8>;
    case 1 * 32 + E_GDIAG8: return k_nn<KIND, 1, E_GDIAG8>;
    case 2 * 32 + E_GDIAG8: return k_nn<KIND, 2, E_GDIAG8>;
    case 3 * 32 + E_GDIAG8: return k_nn<KIND, 3, E_GDIAG8>;
    case 0 * 32 + E_GDIAG16: return k_nn<KIND, 0, E_GDIAG16>;
    case 1 * 32 + E_GDIAG16: return k_nn<KIND, 1, E_GDIAG16>;
    case 2 * 32 + E_GDIAG16: return k_nn<KIND, 2, E_GDIAG16>;
    case 3 * 32 + E_GDIAG16: return k_nn<KIND, 3, E_GDIAG16>;
  }
  return nullptr;
}

// full-band engines that redo guarded-band overflows
template <int KIND>
NNFixFn get_nn_fix(int mode, int eng) {
  switch (mode * 32 + eng) {
    case 0 * 32 + E_GDIAG8: return k_nn_fix<KIND, 0, E_GDIAG8>;
    case 1 * 32 + E_GDIAG8: return k_nn_fix<KIND, 1, E_GDIAG8>;
    case 2 * 32 + E_GDIAG8: return k_nn_fix<KIND, 2, E_GDIAG8>;
    case 3 * 32 + E_GDIAG8: return k_nn_fix<KIND, 3, E_GDIAG8>;
    case 0 * 32 + E_STR4: return k_nn_fix<KIND, 0, E_STR4>;
    case 1 * 32 + E_STR4: return k_nn_fix<KIND, 1, E_STR4>;
    case 0 * 32 + E_STR8: return k_nn_fix<KIND, 0, E_STR8>;
    case 1 * 32 + E_STR8: return k_nn_fix<KIND, 1, E_STR8>;
    case 0 * 32 + E_STR16: return k_nn_fix<KIND, 0, E_STR16>;
    case 1 * 32 + E_STR16: return k_nn_fix<KIND, 1, E_STR16>;
    case 0 * 32 + E_DIAG16: return k_nn_fix<KIND, 0, E_DIAG16>;
    case 1 * 32 + E_DIAG16: return k_nn_fix<KIND, 1, E_DIAG16>;
    case 0 * 32 + E_STRB16: return k_nn_fix<KIND, 0, E_STRB16>;
    case 1 * 32 + E_STRB16: return k_nn_fix<KIND, 1, E_STRB16>;
    case 0 * 32 + E_STRIP16: return k_nn_fix<KIND, 0, E_STRIP16>;
    case 1 * 32 + E_STRIP16: return k_nn_fix<KIND, 1, E_STRIP16>;
    case 0 * 32 + E_STRIPB16: return k_nn_fix<KIND, 0, E_STRIPB16>;
    case 1 * 32 + E_STRIPB16: return k_nn_fix<KIND, 1, E_STRIPB16>;
    case 2 * 32 + E_STR4: return k_nn_fix<KIND, 2, E_STR4>;
    case 3 * 32 + E_STR4: return k_nn_fix<KIND, 3, E_STR4>;
    case 2 * 32 + E_STR8: return k_nn_fix<KIND, 2, E_STR8>;
    case 3 * 32 + E_STR8: return k_nn_fix<KIND, 3, E_STR8>;
    case 2 * 32 + E_STR16: return k_nn_fix<KIND, 2, E_STR16>;
    case 3 * 32 + E_STR16: return k_nn_fix<KIND, 3, E_STR16>;
    case 2 * 32 + E_DIAG16: return k_nn_fix<KIND, 2, E_DIAG16>;
    case 3 * 32 + E_DIAG16: return k_nn_fix<KIND, 3, E_DIAG16>;
    case 2 * 32 + E_STRB16: return k_nn_fix<KIND, 2, E_STRB16>;
    case 3 * 32 + E_STRB16: return k_nn_fix<KIND, 3, E_STRB16>;
    case 2 * 32 + E_STRIP16: return k_nn_fix<KIND, 2, E_STRIP16>;
    case 3 * 32 + E_STRIP16: return k_nn_fix<KIND, 3, E_STRIP16>;
    case 2 * 32 + E_STRIPB16: return k_nn_fix<KIND, 2, E_STRIPB16>;
    case 3 * 32 + E_STRIPB16: return k_nn_fix<KIND, 3, E_STRIPB16>;
  }
  return nullptr;
}

template <int KIND>
UBFn get_ub(int mode) {
  switch (mode) {
    case 0: return k_ub_init<KIND, 0>;
    case 1: return k_ub_init<KIND, 1>;
    case 2: return k_ub_init<KIND, 2>;
    case 3: return k_ub_init<KIND, 3>;
  }
  return nullptr;
}

#define EKB_INSTANTIATE_KIND(K)                  \
  template PairsFn get_pairs<K>(int, int);       \
  template RefFn get_pairs_ref<K>(int, int);     \
  template TriFn get_triangle<K>(int, int);      \
  template NNFn get_nn<K>(int, int);             \
  template NNFixFn get_nn_fix<K>(int, int);      \
  template UBFn get_ub<K>(int);

}  // namespace ekb
