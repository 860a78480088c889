// ek_common.cuh -- per-distance cost semantics for the sm_100a elastic-distance DP.
//
// Every distance is the generic recurrence of the reference
//   cell(i,j) = min(D + canonical(i,j), T + alt_row(i,j), L + alt_col(i,j))
// (pkg/src/elastik/kernels.py:128-277, compiled twin _speedups.pyx:33-94) with
// D = (i-1,j-1), T = (i-1,j), L = (i,j-1).  All arithmetic is IEEE double with
// explicit round-to-nearest intrinsics and no FMA contraction (the library is
// also built with --fmad=false), in the reference's operation order, so every
// finite cell value is bit-identical to the CPU reference.
//
// Per-element data is split into "row data" (a function of the lines series at
// row i: x = l[i-1] and its predecessor) and "column data" (a function of the
// cols series at column j), precomputed once per element as it enters a lane's
// register window, plus per-diagonal constants (WDTW weight w[|i-j|], TWE
// stiffness nu*(|i-j|+|i-j|)).
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <type_traits>

namespace ekb {

enum Kind : int { K_DTW = 0, K_CDTW = 1, K_WDTW = 2, K_ERP = 3, K_MSM = 4, K_TWE = 5 };
enum Mode : int { M_SQ = 0, M_ABS = 1 };

#define EKB_INF (__longlong_as_double(0x7ff0000000000000LL))
#define EKB_DI __device__ __forceinline__

struct Params {
  double gap, msm_c, nu, lam;
  double zero;  // 0.0 supplied at run time (keeps band offsets as full 64-bit registers)
  // WDTW weight tables, host-computed with libm exp (kernels.py:80-92): the table for
  // longest length m (m+1 entries, indexed by |i-j|) starts at wt_all + wt_off[m].
  const double* wt_all;
  const long long* wt_off;
  const double* wt;  // per pair: the table for this pair's longest length
  int wt_len;        // entries available in wt
  // long-series strip engines: per-warp boundary columns (2 x strip_stride doubles per
  // warp, indexed by the global warp id)
  double* strip_buf;
  int strip_stride;
};

// Params for one pair whose longest series has length m.
__device__ __forceinline__ Params pair_params(const Params& p, int m) {
  Params q = p;
  if (p.wt_off != nullptr) {
    q.wt = p.wt_all + p.wt_off[m];
    q.wt_len = m + 1;
  }
  return q;
}

EKB_DI double dadd(double a, double b) { return __dadd_rn(a, b); }
EKB_DI double dsub(double a, double b) { return __dsub_rn(a, b); }
EKB_DI double dmul(double a, double b) { return __dmul_rn(a, b); }
EKB_DI double dmin_ref(double v, double a) { return (a < v) ? a : v; }  // "if a < v: v = a"

// point_cost (kernels.py:70-77; _speedups.pyx:33-38)
template <int MODE>
EKB_DI double pcost(double a, double b) {
  double d = dsub(a, b);
  if (MODE == M_SQ) return dmul(d, d);
  return fabs(d);
}

// IEEE sign bit (0 / 1) of a double
EKB_DI int sign_bit(double v) { return (int)((unsigned)__double2hiint(v) >> 31); }

// ---- row / column data ----
template <int KIND> struct RowD { double x; };
template <int KIND> struct ColD { double y; };
template <> struct RowD<K_ERP> { double x, ar; };
template <> struct ColD<K_ERP> { double y, ac; };
template <> struct RowD<K_TWE> { double x, ar; };
template <> struct ColD<K_TWE> { double y, ac; };
template <> struct RowD<K_MSM> { double x, dr; int s; };  // s: sign bit of x - xprev
template <> struct ColD<K_MSM> { double y, dc; int s; };  // s: sign bit of y - yprev

// x = l[i-1], xp = l[i-2] (pad: MSM uses l[0] at index -1, TWE a phantom 0.0)
template <int KIND, int MODE>
EKB_DI RowD<KIND> make_row(double x, double xp, const Params& p) {
  RowD<KIND> r;
  r.x = x;
  if constexpr (KIND == K_ERP) r.ar = pcost<MODE>(x, p.gap);                 // alt_row: pc(l_i, g)
  if constexpr (KIND == K_TWE) r.ar = dadd(dadd(pcost<MODE>(x, xp), p.nu), p.lam);  // (pc(l_i,l_{i-1})+nu)+lam
  if constexpr (KIND == K_MSM) {
    const double d = dsub(x, xp);
    r.dr = fabs(d);  // fabs(np - x) in msm_cost(l_i, l_{i-1}, c_j)
    r.s = sign_bit(d);
  }
  return r;
}

template <int KIND, int MODE>
EKB_DI ColD<KIND> make_col(double y, double yp, const Params& p) {
  ColD<KIND> c;
  c.y = y;
  if constexpr (KIND == K_ERP) c.ac = pcost<MODE>(p.gap, y);                 // alt_col: pc(g, c_j)
  if constexpr (KIND == K_TWE) c.ac = dadd(dadd(pcost<MODE>(y, yp), p.nu), p.lam);
  if constexpr (KIND == K_MSM) {
    const double d = dsub(y, yp);
    c.dc = fabs(d);  // fabs(np - y) in msm_cost(c_j, l_i, c_{j-1})
    c.s = sign_bit(d);
  }
  return c;
}

// ---- per-diagonal constant and per-slot state ----
// off: +inf for a diagonal outside the band (its cells must stay +inf), 0.0 inside;
// the DTW family adds it to the move cost, which replaces two selects per cell.
template <int KIND> struct DiagK { double off; };
template <> struct DiagK<K_WDTW> { double w, off; };
template <> struct DiagK<K_TWE> { double tw; };
template <int KIND> struct SlotS {};
template <> struct SlotS<K_TWE> { double pcp; };  // pc(l_{i-2}, c_{j-2}) = previous cell's pc on this diagonal

template <int KIND>
EKB_DI DiagK<KIND> make_diag(int d, const Params& p, bool in_band = true) {
  DiagK<KIND> k;
  int ad = d < 0 ? -d : d;
  if constexpr (KIND == K_DTW || KIND == K_CDTW || KIND == K_WDTW || KIND == K_ERP || KIND == K_MSM)
    k.off = in_band ? p.zero : EKB_INF;
  if constexpr (KIND == K_WDTW) k.w = (ad < p.wt_len) ? p.wt[ad] : 0.0;  // wt[|i-j|]
  if constexpr (KIND == K_TWE) {
    double dij = (double)ad;
    k.tw = dmul(p.nu, dadd(dij, dij));  // nu * (dij + dij)
  }
  return k;
}

// MSM split/merge alternative (kernels.py:95-105; _speedups.pyx:41-47), given the
// shared |l_i - c_j| and the between-test already decided.
//
// Between-tests from sign bits: with e = l_i - c_j and dr = l_i - l_{i-1},
// "l_{i-1} <= l_i <= c_j or l_{i-1} >= l_i >= c_j" holds iff e and dr do not have the
// same strict sign, and the column test (l_i <= c_j <= c_{j-1} or ...) iff e and
// dc = c_j - c_{j-1} do.  Reading "strict sign" as the IEEE sign bit only misclassifies
// a zero (e or dr / dc == +0: an exact difference is never -0), and then both outcomes
// give the same value: c, or c + min(|d|, 0) = c + 0 = c.
EKB_DI double msm_alt(bool between, double c, double dother, double de) {
  double m = (dother < de) ? dother : de;  // "d1 if d1 < d2 else d2" (value-identical)
  return between ? c : dadd(c, m);
}

// One cell.  D, T, L are the dependency values; the result is the reference's
// value bit-for-bit whenever the dependencies are.  (For the DTW family the
// band offset k.off is folded into the cost: cost + 0.0 == cost exactly.)
template <int KIND, int MODE, bool OFF = true>
EKB_DI double cell(double D, double T, double L, const RowD<KIND>& r, const ColD<KIND>& c,
                   const DiagK<KIND>& k, SlotS<KIND>& st, const Params& p) {
  if constexpr (KIND == K_DTW || KIND == K_CDTW || KIND == K_WDTW) {
    // all three move costs are equal: min(D+c, T+c, L+c) == min(D,T,L)+c (monotone rounding)
    double cost = pcost<MODE>(r.x, c.y);
    if constexpr (KIND == K_WDTW) cost = dmul(cost, k.w);
    if constexpr (OFF) cost = dadd(cost, k.off);  // +0.0 in band (exact), +inf outside
    double m = dmin_ref(D, T);
    m = dmin_ref(m, L);
    return dadd(m, cost);
  } else if constexpr (KIND == K_ERP) {
    double v = dadd(D, pcost<MODE>(r.x, c.y));
    v = dmin_ref(v, dadd(T, r.ar));
    return dmin_ref(v, dadd(L, c.ac));
  } else if constexpr (KIND == K_TWE) {
    double pc = pcost<MODE>(r.x, c.y);
    double canon = dadd(dadd(pc, st.pcp), k.tw);  // (pc(l_i,c_j) + pc(l_{i-1},c_{j-1})) + nu*(d+d)
    st.pcp = pc;
    double v = dadd(D, canon);
    v = dmin_ref(v, dadd(T, r.ar));
    return dmin_ref(v, dadd(L, c.ac));
  } else {  // MSM: canonical |l_i - c_j| regardless of cost mode
    double e = dsub(r.x, c.y);
    double de = fabs(e);
    const int se = sign_bit(e);
    bool brow = se != r.s;  // l_{i-1}<=l_i<=c_j or l_{i-1}>=l_i>=c_j (see msm_alt)
    bool bcol = se == c.s;  // l_i<=c_j<=c_{j-1} or l_i>=c_j>=c_{j-1}
    double ar = msm_alt(brow, p.msm_c, r.dr, de);
    double ac = msm_alt(bcol, p.msm_c, c.dc, de);
    double v = dadd(D, de);
    v = dmin_ref(v, dadd(T, ar));
    return dmin_ref(v, dadd(L, ac));
  }
}

// Pads around a series in shared memory: index -1 and index n.  Index -1 is the
// "previous" of the first element (MSM: the point itself; TWE: phantom 0.0);
// index n is +inf so cells past the end of the matrix evaluate to +inf.
template <int KIND>
EKB_DI double pad_before(double first) {
  return KIND == K_MSM ? first : 0.0;
}

}  // namespace ekb
