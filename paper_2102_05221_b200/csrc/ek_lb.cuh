// ek_lb.cuh -- LB_Keogh pre-tests for dtw/cdtw 1-NN: the rounding
// rules and the warp-cooperative reverse bound; the forward bound of every pair is
// k_lb_matrix (ek_misc.cu), which uses the same rounding.
//
// Reference: lower_bounds.build_envelope / lb_keogh (pkg/src/elastik/lower_bounds.py:23-84)
// and their use as a skip test in search.nn_search (search.py:104-112).  Here the
// bound is a *scheduling* filter: a candidate is dropped only when its bound
// proves the DP result would be +inf anyway, so the 1-NN answer is unchanged
// (result invariance across lb modes: pkg/tests/test_search.py:59-76).
//
// Soundness in floating point: every alignment path in the band matches each
// query point i with some candidate point j, |i-j| <= w, so its cost is at
// least sum_i dist(q_i, [L_i, U_i]).  Envelopes are stored as floats rounded
// outward (upper up, lower down), which only widens them, and the per-pair bound
// is summed in FP32 rounding toward -inf (lb_lane_terms, totals in fixed point: lb_reduce), so it never exceeds the exact
// bound.  The DP value carries at most ~2n ulps of relative error (n <= 2^13 terms
// of non-negative sums), so a candidate is skipped only when the bound exceeds
// cutoff * (1 + 2^-32), far above that error.
// (k_envelope, which builds the envelopes, lives in ek_misc.cu.)
#pragma once
#include "ek_common.cuh"
#include "ek_diag.cuh"

namespace ekb {

// Warp-cooperative lb_keogh(q, env(c)) test with early exit.  Points are taken in
// batches of LB_BATCH x 32 (lane = point within a 32-point chunk); the first batch
// arrives prefetched, later batches are loaded together so their latency overlaps.
constexpr int LB_BATCH = 4;

// One batch of LB_Keogh terms in FP32 with every operation rounded toward -inf, so
// the sum is a guaranteed lower bound of the exact bound: q is widened to
// [RD(q), RU(q)], the distances to the (outward-rounded) envelope are rounded down,
// squared and summed rounding down.  Returns this lane's partial sum.
// FP32 mode (R = float): the staged values are floats already, the interval is a point.
template <int MODE, class R>
__device__ __forceinline__ float lb_lane_terms(const R* qs, int base, int L, const float2 (&e)[LB_BATCH]) {
  const int lane = threadIdx.x & 31;
  float t = 0.f;
#pragma unroll
  for (int b = 0; b < LB_BATCH; ++b) {
    const int k = base + b * 32 + lane;
    float qlo, qhi;
    if constexpr (std::is_same<R, float>::value) {
      qlo = qhi = k < L ? qs[k] : 0.f;
    } else {
      const double qi = k < L ? qs[k] : 0.0;
      qlo = __double2float_rd(qi);
      qhi = __double2float_ru(qi);
    }
    // distance to [lower, upper] (upper >= lower), branch-free; neutral interval -> 0
    const float d = fmaxf(fmaxf(__fsub_rd(qlo, e[b].x), __fsub_rd(e[b].y, qhi)), 0.f);
    t = __fadd_rd(t, (MODE & 1) == 0 ? __fmul_rd(d, d) : d);
  }
  return t;
}

// Warp totals in fixed point: each lane's partial is scaled by a power of two s and
// truncated (clamped at 2^26, so 32 lanes cannot overflow), then one integer
// __reduce_add_sync replaces the five-step float butterfly.  s puts the threshold in
// [2^20, 2^21): T = ceil(RU(thr) * s) exactly, every other step rounds down, so a total
// above T proves the exact bound exceeds thr; truncation only weakens the bound.
struct LBScale {
  float s;     // multiplier (0: never prune)
  unsigned T;  // scaled threshold
  bool all;    // thr < 0: every pair is pruned (nothing is <= a negative cutoff)
};
__device__ __forceinline__ LBScale lb_scale(double thr) {
  LBScale r;
  r.all = thr < 0.0;
  const float tf = __double2float_ru(thr);
  const int ex = ((__float_as_int(tf) >> 23) & 0xff) - 127;  // tf in [2^ex, 2^(ex+1)) for normal tf
  if (!(thr >= 0.0) || !(tf < __int_as_float(0x7f800000))) {
    r.s = 0.f;  // +inf / NaN threshold: never prune
    r.T = 0xffffffffu;
  } else if (tf < 0x1p-100f) {  // (near) zero threshold: any term above 2^-100 prunes
    r.s = 0x1p100f;
    r.T = 0u;
  } else {
    r.s = __int_as_float((147 - ex) << 23);  // 2^(20 - ex)
    r.T = __float2uint_ru(tf * r.s);         // exact product, in [2^20, 2^21)
  }
  return r;
}
__device__ __forceinline__ unsigned lb_reduce(float t, const LBScale& sc) {
  const unsigned q = __float2uint_rd(fminf(__fmul_rd(t, sc.s), 67108864.0f));  // 2^26
  return __reduce_add_sync(FULL, q);
}

// out-of-range points load the neutral interval [-inf, +inf]
__device__ __forceinline__ void lb_load(const float2* __restrict__ env, int base, int L, float2 (&e)[LB_BATCH]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int b = 0; b < LB_BATCH; ++b) {
    const int k = base + b * 32 + lane;
    e[b] = k < L ? __ldg(env + k) : make_float2(__int_as_float(0x7f800000), __int_as_float(0xff800000));
  }
}

// The reverse bound LB_Keogh(candidate, envelope(query)) (lb_keogh2's second order,
// lower_bounds.py:87-98) over a candidate staged in shared memory; the query
// envelope comes from global memory.  true when the pair must still be evaluated.
template <int MODE, class R>
__device__ __forceinline__ bool warp_lb_reverse(const R* cs, const float2* __restrict__ envq, int L,
                                                const LBScale& sc) {
  unsigned total = 0;
  for (int base = 0; base < L; base += 32 * LB_BATCH) {
    float2 e[LB_BATCH];
    lb_load(envq, base, L, e);
    total += lb_reduce(lb_lane_terms<MODE>(cs, base, L, e), sc);
    if (total > sc.T) return false;
  }
  return true;
}

// lb_threshold (the pre-tests' cutoff margin) lives in ek_common.cuh

}  // namespace ekb
