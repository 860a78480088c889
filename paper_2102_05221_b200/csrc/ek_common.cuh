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
enum Mode : int { M_SQ = 0, M_ABS = 1, M_F32 = 2 };
// MODE = cost mode (bit 0) | M_F32 (bit 1).  The FP32 mode (not the reference's
// arithmetic: an optional faster mode, within 1e-5 relative of it) runs the same
// engines on float values staged from the float64 inputs.
template <int MODE> using real_t = typename std::conditional<(MODE & M_F32) != 0, float, double>::type;

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
  // k_nn, non-LB path on dense even-length float64 batches with a diagonal engine: stage
  // each candidate with one bulk asynchronous copy (TMA), one pair ahead, into a second
  // per-warp candidate slot (see ek_tma.cuh); 0 = synchronous staging
  int bulk;
  // k_triangle on equal lengths with a row-stripe engine that reads an |i-j| table (WDTW,
  // TWE): one table per block instead of one per pair slot (every pair has the same one)
  int shared_tab;
  // k_triangle on equal lengths with the half-warp diagonal engine (E_DIAG4H): pads of this
  // many elements around each staged series instead of the engine's general pad (0 = that).
  // 16 lanes x P = 4 with series of one length n read indices in [-32, n + 30] only
  // (diag_pair: i = (t + d) / 2, t <= 2n - 2 at the last load, |d| <= 62), so 40 elements
  // do, against the 72 that unequal lengths need (C3 ERP: 4 -> 5 resident blocks).
  int compact_pad;
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
EKB_DI float dadd(float a, float b) { return __fadd_rn(a, b); }
EKB_DI float dsub(float a, float b) { return __fsub_rn(a, b); }
EKB_DI float dmul(float a, float b) { return __fmul_rn(a, b); }
template <class R>
EKB_DI R dmin_ref(R v, R a) { return (a < v) ? a : v; }  // "if a < v: v = a"
template <class R> EKB_DI R rinf();
template <> EKB_DI double rinf<double>() { return EKB_INF; }
template <> EKB_DI float rinf<float>() { return __int_as_float(0x7f800000); }

// point_cost (kernels.py:70-77; _speedups.pyx:33-38)
template <int MODE>
EKB_DI real_t<MODE> pcost(real_t<MODE> a, real_t<MODE> b) {
  real_t<MODE> d = dsub(a, b);
  if ((MODE & 1) == M_SQ) return dmul(d, d);
  return fabs(d);
}

// IEEE sign bit (0 / 1)
EKB_DI int sign_bit(double v) { return (int)((unsigned)__double2hiint(v) >> 31); }
EKB_DI int sign_bit(float v) { return (int)(__float_as_uint(v) >> 31); }

// ---- row / column data ----
template <int KIND, class R = double> struct RowD { R x; };
template <int KIND, class R = double> struct ColD { R y; };
template <class R> struct RowD<K_ERP, R> { R x, ar; };
template <class R> struct ColD<K_ERP, R> { R y, ac; };
template <class R> struct RowD<K_TWE, R> { R x, ar; };
template <class R> struct ColD<K_TWE, R> { R y, ac; };
template <class R> struct RowD<K_MSM, R> { R x, dr; int s; };  // s: sign bit of x - xprev
template <class R> struct ColD<K_MSM, R> { R y, dc; int s; };  // s: sign bit of y - yprev

// x = l[i-1], xp = l[i-2] (pad: MSM uses l[0] at index -1, TWE a phantom 0.0)
template <int KIND, int MODE>
EKB_DI RowD<KIND, real_t<MODE>> make_row(real_t<MODE> x, real_t<MODE> xp, const Params& p) {
  using R = real_t<MODE>;
  RowD<KIND, R> r;
  r.x = x;
  if constexpr (KIND == K_ERP) r.ar = pcost<MODE>(x, (R)p.gap);                 // alt_row: pc(l_i, g)
  if constexpr (KIND == K_TWE) r.ar = dadd(dadd(pcost<MODE>(x, xp), (R)p.nu), (R)p.lam);  // (pc(l_i,l_{i-1})+nu)+lam
  if constexpr (KIND == K_MSM) {
    const R d = dsub(x, xp);
    r.dr = fabs(d);  // fabs(np - x) in msm_cost(l_i, l_{i-1}, c_j)
    r.s = sign_bit(d);
  }
  return r;
}

template <int KIND, int MODE>
EKB_DI ColD<KIND, real_t<MODE>> make_col(real_t<MODE> y, real_t<MODE> yp, const Params& p) {
  using R = real_t<MODE>;
  ColD<KIND, R> c;
  c.y = y;
  if constexpr (KIND == K_ERP) c.ac = pcost<MODE>((R)p.gap, y);                 // alt_col: pc(g, c_j)
  if constexpr (KIND == K_TWE) c.ac = dadd(dadd(pcost<MODE>(y, yp), (R)p.nu), (R)p.lam);
  if constexpr (KIND == K_MSM) {
    const R d = dsub(y, yp);
    c.dc = fabs(d);  // fabs(np - y) in msm_cost(c_j, l_i, c_{j-1})
    c.s = sign_bit(d);
  }
  return c;
}

// ---- per-diagonal constant and per-slot state ----
// off: +inf for a diagonal outside the band (its cells must stay +inf), 0.0 inside;
// the DTW family adds it to the move cost, which replaces two selects per cell.
template <int KIND, class R = double> struct DiagK { R off; };
template <class R> struct DiagK<K_WDTW, R> { R w, off; };
template <class R> struct DiagK<K_TWE, R> { R tw; };
template <int KIND, class R = double> struct SlotS {};
template <class R> struct SlotS<K_TWE, R> { R pcp; };  // pc(l_{i-2}, c_{j-2}) = previous cell's pc on this diagonal

// FP32 mode: the WDTW weight is the host table's value rounded to float; TWE's
// nu*(d+d) is evaluated in float.
template <int KIND, class R = double>
EKB_DI DiagK<KIND, R> make_diag(int d, const Params& p, bool in_band = true) {
  DiagK<KIND, R> k;
  int ad = d < 0 ? -d : d;
  if constexpr (KIND == K_DTW || KIND == K_CDTW || KIND == K_WDTW || KIND == K_ERP || KIND == K_MSM)
    k.off = in_band ? (R)p.zero : rinf<R>();
  if constexpr (KIND == K_WDTW) k.w = (ad < p.wt_len) ? (R)p.wt[ad] : (R)0.0;  // wt[|i-j|]
  if constexpr (KIND == K_TWE) {
    R dij = (R)ad;
    k.tw = dmul((R)p.nu, dadd(dij, dij));  // nu * (dij + dij)
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
template <class R>
EKB_DI R msm_alt(bool between, R c, R dother, R de) {
  R m = (dother < de) ? dother : de;  // "d1 if d1 < d2 else d2" (value-identical)
  return between ? c : dadd(c, m);
}
// The same value with the choice folded into one fused multiply-add: fma(m, f, c) with
// f = 0.0 (between) or 1.0 is RN(c + m * f) = c or RN(c + m), since m * f is exact (m is a
// finite difference).  A one-word select builds f, and the FMA replaces the add and the
// 64-bit select (two ALU selects) -- the MSM cell is ALU-pipe bound.
EKB_DI double msm_alt_fma(bool between, double c, double dother, double de) {
  const double m = (dother < de) ? dother : de;
  const double f = __hiloint2double(between ? 0 : 0x3ff00000, 0);
  return __fma_rn(m, f, c);
}
EKB_DI float msm_alt_fma(bool between, float c, float dother, float de) {
  const float m = (dother < de) ? dother : de;
  return __fmaf_rn(m, between ? 0.f : 1.f, c);
}
// The factor from the sign bits without a compare and a select: nb = 1 when the point is NOT
// between (0 / 1, one logic op on the two sign bits), and the factor's high word
// nb * 0x3ff00000 comes from the FMA pipe's integer multiply-add, which these cells leave
// idle while the select (ALU) pipe bounds them.
EKB_DI double msm_alt_fma_nb(int nb, double c, double dother, double de) {
  const double m = (dother < de) ? dother : de;
  int hi;
  asm("mad.lo.s32 %0, %1, 0x3ff00000, 0;" : "=r"(hi) : "r"(nb));
  return __fma_rn(m, __hiloint2double(hi, 0), c);
}
EKB_DI float msm_alt_fma_nb(int nb, float c, float dother, float de) {
  const float m = (dother < de) ? dother : de;
  return __fmaf_rn(m, (float)nb, c);
}
#ifndef EKB_MSM_FMA
#define EKB_MSM_FMA 2  // 2: msm_alt_fma_nb, 1: msm_alt_fma, 0: msm_alt
#endif

// One cell.  D, T, L are the dependency values; the result is the reference's
// value bit-for-bit whenever the dependencies are.  (For the DTW family the
// band offset k.off is folded into the cost: cost + 0.0 == cost exactly.)
// T_LAST: take the T operand last (the diagonal engine's shuffled operand, so its latency
// overlaps the first minimum).  The minimum of the three is the same value either way: the
// first operand D is never NaN for a cell inside the band, values are >= +0 or +inf, and
// "if a < v" never selects a NaN second operand.
template <int KIND, int MODE, bool OFF = true, bool T_LAST = false, class R = real_t<MODE>>
EKB_DI R cell(R D, R T, R L, const RowD<KIND, R>& r, const ColD<KIND, R>& c, const DiagK<KIND, R>& k,
              SlotS<KIND, R>& st, const Params& p) {
  if constexpr (KIND == K_DTW || KIND == K_CDTW || KIND == K_WDTW) {
    // all three move costs are equal: min(D+c, T+c, L+c) == min(D,T,L)+c (monotone rounding)
    R cost = pcost<MODE>(r.x, c.y);
    if constexpr (KIND == K_WDTW) cost = dmul(cost, k.w);
    if constexpr (OFF) cost = dadd(cost, k.off);  // +0.0 in band (exact), +inf outside
    R m = dmin_ref(D, T_LAST ? L : T);
    m = dmin_ref(m, T_LAST ? T : L);
    return dadd(m, cost);
  } else if constexpr (KIND == K_ERP) {
    R v = dadd(D, pcost<MODE>(r.x, c.y));
    v = dmin_ref(v, dadd(T, r.ar));
    return dmin_ref(v, dadd(L, c.ac));
  } else if constexpr (KIND == K_TWE) {
    R pc = pcost<MODE>(r.x, c.y);
    R canon = dadd(dadd(pc, st.pcp), k.tw);  // (pc(l_i,c_j) + pc(l_{i-1},c_{j-1})) + nu*(d+d)
    st.pcp = pc;
    R v = dadd(D, canon);
    v = dmin_ref(v, dadd(T, r.ar));
    return dmin_ref(v, dadd(L, c.ac));
  } else {  // MSM: canonical |l_i - c_j| regardless of cost mode
    R e = dsub(r.x, c.y);
    R de = fabs(e);
    const int se = sign_bit(e);
    bool brow = se != r.s;  // l_{i-1}<=l_i<=c_j or l_{i-1}>=l_i>=c_j (see msm_alt)
    bool bcol = se == c.s;  // l_i<=c_j<=c_{j-1} or l_i>=c_j>=c_{j-1}
    R ar, ac;
    if constexpr (EKB_MSM_FMA == 2) {  // not between: the row test's signs equal, the column test's differ
      ar = msm_alt_fma_nb(se ^ r.s ^ 1, (R)p.msm_c, r.dr, de);
      ac = msm_alt_fma_nb(se ^ c.s, (R)p.msm_c, c.dc, de);
    } else {
      ar = EKB_MSM_FMA ? msm_alt_fma(brow, (R)p.msm_c, r.dr, de) : msm_alt(brow, (R)p.msm_c, r.dr, de);
      ac = EKB_MSM_FMA ? msm_alt_fma(bcol, (R)p.msm_c, c.dc, de) : msm_alt(bcol, (R)p.msm_c, c.dc, de);
    }
    R v = dadd(D, de);
    v = dmin_ref(v, dadd(T, ar));
    return dmin_ref(v, dadd(L, ac));
  }
}

// Pads around a series in shared memory: index -1 and index n.  Index -1 is the
// "previous" of the first element (MSM: the point itself; TWE: phantom 0.0);
// index n is +inf so cells past the end of the matrix evaluate to +inf.
template <int KIND, class R = double>
EKB_DI R pad_before(R first) {
  return KIND == K_MSM ? first : (R)0.0;
}

// LB pre-tests (ek_lb.cuh) and the diagonal-distance liveness bound (ek_diag.cuh): a bound
// above lb_threshold(cut) proves the DP value exceeds cut.
// bound > cutoff * (1 + 2^-32) proves the DP value exceeds the cutoff (see header).
// FP32 mode: the bound is exact for the float-rounded series the DP sees (rounding is
// monotone, so the outward float envelope still encloses them), and the float DP value
// of any path is >= its exact cost * (1 - u)^(2n+3), u = 2^-24 (each term passes
// through <= 2n+3 roundings); hence the wider margin (1 + (2n+8) 2^-24), rounded up.
template <int MODE>
__device__ __forceinline__ double lb_threshold(double cut, int n) {
  if constexpr ((MODE & M_F32) != 0) return __dmul_ru(cut, 1.0 + (double)(2 * n + 8) * 0x1p-24);
  return cut * (1.0 + 2.3283064365386963e-10);
}
__device__ __forceinline__ double lb_threshold(double cut) { return lb_threshold<0>(cut, 0); }

}  // namespace ekb
