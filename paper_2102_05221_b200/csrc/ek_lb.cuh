// ek_lb.cuh -- LB_Keogh pre-test for dtw/cdtw 1-NN.
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
// is summed in FP32 rounding toward -inf (lb_terms), so it never exceeds the exact
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
// squared and summed rounding down.  The warp total (xor butterfly, so every lane holds
// the same value) is exact-or-below; lb_threshold's margin covers the DP's rounding.
template <int MODE>
__device__ __forceinline__ float lb_terms(const double* qs, int base, int L, const float2 (&e)[LB_BATCH]) {
  const int lane = threadIdx.x & 31;
  float t = 0.f;
#pragma unroll
  for (int b = 0; b < LB_BATCH; ++b) {
    const int k = base + b * 32 + lane;
    const double qi = k < L ? qs[k] : 0.0;
    const float qlo = __double2float_rd(qi), qhi = __double2float_ru(qi);
    // distance to [lower, upper] (upper >= lower), branch-free; neutral interval -> 0
    const float d = fmaxf(fmaxf(__fsub_rd(qlo, e[b].x), __fsub_rd(e[b].y, qhi)), 0.f);
    t = __fadd_rd(t, MODE == 0 ? __fmul_rd(d, d) : d);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) t = __fadd_rd(t, __shfl_xor_sync(FULL, t, o));
  return t;
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

// Continues the test past the prefetched first batch (running total `total`).
// Returns true when the candidate must still be evaluated.
template <int MODE>
__device__ __forceinline__ bool warp_lb_rest(const double* qs, const float2* __restrict__ env, int L, double thr,
                                             float total) {
  for (int base = 32 * LB_BATCH; base < L; base += 32 * LB_BATCH) {
    float2 e[LB_BATCH];
    lb_load(env, base, L, e);
    total = __fadd_rd(total, lb_terms<MODE>(qs, base, L, e));
    if ((double)total > thr) return false;
  }
  return true;
}

// The reverse bound LB_Keogh(candidate, envelope(query)) (lb_keogh2's second order,
// lower_bounds.py:87-98) over a candidate staged in shared memory; the query
// envelope comes from global memory.  true when the pair must still be evaluated.
template <int MODE>
__device__ __forceinline__ bool warp_lb_reverse(const double* cs, const float2* __restrict__ envq, int L,
                                                double thr) {
  float total = 0.f;
  for (int base = 0; base < L; base += 32 * LB_BATCH) {
    float2 e[LB_BATCH];
    lb_load(envq, base, L, e);
    total = __fadd_rd(total, lb_terms<MODE>(cs, base, L, e));
    if ((double)total > thr) return false;
  }
  return true;
}

// bound > cutoff * (1 + 2^-32) proves the DP value exceeds the cutoff (see header)
__device__ __forceinline__ double lb_threshold(double cut) { return cut * (1.0 + 2.3283064365386963e-10); }

}  // namespace ekb
