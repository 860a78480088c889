// ek_diag.cuh -- warp-per-pair anti-diagonal wavefront for banded elastic DPs.
//
// Layout ("diagonal slots"): lane l owns P consecutive diagonals d = i - j,
// d = dbase + l*P + p.  Cell (i,j) sits on diagonal d at time t = i + j; its
// dependencies are its own diagonal at t-2 (D), diagonal d-1 at t-1 (T) and
// diagonal d+1 at t-1 (L).  One "double step" advances every diagonal by one
// cell: even slots at time t, odd slots at time t+1.  Inside a lane all
// dependencies are registers; the only exchange is one 64-bit shuffle per
// half step across the lane boundary.  The Sakoe-Chiba band maps to a
// contiguous range of slots, so a band of width 2w+1 costs ~(2w+3)/32 slots
// per lane instead of a full row.
//
// Borders: the corner is diagonal 0 at t=0; border cells (i,0)/(0,j) are the
// first cells of diagonals +i/-j (t=|d|).  For ERP they follow from the
// recurrence itself -- (d,0) = (d-1,0) + pc(l_d, g) is exactly the sequential
// prefix of _erp_border (kernels.py:280-289) -- and every other kind has +inf
// borders, which also fall out once diagonals +-1 are seeded at t=1.  The two
// "virtual" diagonals just outside the band hold their border value at their
// border time and +inf otherwise, which reproduces the reference's window
// (hborder for j <= w+1, vborder while jstart == 1; _speedups.pyx:137-148).
// Cells before a diagonal's border time evaluate to +inf (their inputs are
// +inf and the padded series values are finite); cells past the end of the
// matrix are never read by a cell inside it.
//
// Pruning/abandoning: every path crosses one of any two consecutive
// anti-diagonals, so when no cell of (t, t+1) is <= cutoff the pair is
// abandoned (+inf).  A pair whose exact cost is <= cutoff never abandons (all
// cells on its optimal path are <= cost), so the observable contract is the
// reference eapruned's: exact when cost <= cutoff, +inf otherwise
// (engines.py:72-84).  With a shared cutoff that only tightens,
// the same argument holds against the final cutoff.  The liveness test compares
// the high 32-bit words of the IEEE images (values are >= +0 or +inf, the
// cutoff is canonicalised by the host: NaN -> -inf, -0.0 -> +0.0), which is
// conservative -- it can only keep a pair alive longer, never change a result.
#pragma once
#include "ek_common.cuh"

namespace ekb {

constexpr unsigned FULL = 0xffffffffu;

#ifdef EKB_LIVE
// debug builds: in-matrix band cells the diagonal engine evaluated, and those of them that
// were live (value <= the cutoff in force) -- the share EAPruned's column pruning would skip
__device__ unsigned long long g_live[2];
// and the live corridor at each vote: the span of lanes holding a live cell (first..last),
// histogrammed per 64 anti-diagonals of t (16 x 33 bins)
__device__ unsigned long long g_corr[16 * 33];
// narrow-window simulation (a 16-lane = 64-diagonal window, 2-lane guards, re-centred when a
// guard lane is live and the corridor fits 12 lanes, else overflow): pairs, narrowed pairs,
// overflowed pairs, votes, narrow votes, narrow votes of overflowed pairs, re-centrings
__device__ unsigned long long g_sn[8];
#endif

#ifndef EKB_DBOUND
#define EKB_DBOUND 1  // MSM / TWE diagonal-distance bound in the liveness test
#endif
#ifndef EKB_ROT_MAX_H
#define EKB_ROT_MAX_H 2  // register windows rotate at compile time up to H = P/2 = 2 (U = 6 unrolled steps)
#endif

struct DiagResult {
  double cost;   // exact, or +inf when abandoned / above cutoff
  int t_end;     // last anti-diagonal processed
  bool ovf;      // guarded band: a cell <= cutoff reached a guard lane (cost meaningless)
};

// The shared cutoff as one warp-uniform value.  Lanes of a warp are not
// guaranteed to execute a load together (independent thread scheduling), so a
// per-lane load can observe two different values around another warp's atomicMin;
// every decision taken on the cutoff must be the same in all 32 lanes, hence lane
// 0's value is broadcast.  Call from converged code only.
// Split form: ld_cut_raw issues lane 0's load, bcast_cut broadcasts it; placing the
// broadcast well after the load hides its latency.
__device__ __forceinline__ unsigned long long ld_cut_raw(const unsigned long long* p) {
  unsigned long long v = 0;
  if ((threadIdx.x & 31) == 0) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double bcast_cut(unsigned long long v) {
  return __longlong_as_double((long long)__shfl_sync(0xffffffffu, v, 0));
}
__device__ __forceinline__ double ld_cut(const unsigned long long* p) { return bcast_cut(ld_cut_raw(p)); }

__device__ __forceinline__ int hi_word(double v) { return __double2hiint(v); }
// FP32 mode: the whole image (values are >= +0 or +inf, so the bits order as integers)
__device__ __forceinline__ int hi_word(float v) { return __float_as_int(v); }

// A cutoff in the engine's precision.  FP32 keep-if-<= against a float64 cutoff c:
// a float v satisfies v <= c iff v <= RD(c), so the cutoff is rounded down.
template <class R> __device__ __forceinline__ R to_cut(double c);
template <> __device__ __forceinline__ double to_cut<double>(double c) { return c; }
template <> __device__ __forceinline__ float to_cut<float>(double c) { return __double2float_rd(c); }

// Loader protocol: next_t(dlo, dhi, H) = first double-step time at which the
// engine needs data beyond what is staged; ensure(t, dlo, dhi, H) stages more.
struct NoLoader {
  __device__ __forceinline__ int next_t(int, int, int) const { return 0x7fffffff; }
  __device__ __forceinline__ void ensure(int, int, int, int) {}
};

// Padding (elements) the diagonal engine may read beyond either end of a
// series, for P slots per lane: i = (t + d)/2 ranges over [-16P-2, n + 16P + 2].
__host__ __device__ constexpr int diag_pad(int P) { return 16 * P + 8; }

// Series accessor over shared memory padded on both sides (see stage_series):
// index -1 holds the kind's "previous of the first element", indices < -1 hold
// 0.0, indices >= n hold +inf.
template <class R>
struct SmemSeriesT {
  const R* p;
  int n;
  __device__ __forceinline__ R at(int k) const {
#ifdef EKB_BOUNDS
    if (k < -EKB_BOUNDS || k >= n + EKB_BOUNDS) {
      printf("SmemSeries OOB k=%d n=%d block=%d warp=%d\n", k, n, blockIdx.x, threadIdx.x >> 5);
      __trap();
    }
#endif
    return p[k];
  }
};
using SmemSeries = SmemSeriesT<double>;

// Runs f(integral_constant<S>) for S = S0 .. U-1 until one returns true.
template <int S0, int U, class F>
__device__ __forceinline__ bool unrolled_steps(F& f) {
  if constexpr (S0 == U) {
    return false;
  } else {
    if (f(std::integral_constant<int, S0>{})) return true;
    return unrolled_steps<S0 + 1, U>(f);
  }
}

// X: lines accessor (nl >= nc), Y: cols accessor.  w: effective window
// (w >= nl - nc, checked by the caller).
//
// guard != 0 (a lane mask) runs the band [-w, w] as a stand-in for a wider true band:
// cells outside it count as +inf.  That is exact under the keep-if-<=-cutoff contract
// as long as no cell <= cutoff ever appears in a guard lane (the lanes holding the
// band's narrowed edges).  A path of cost <= cutoff has all its prefixes <= cutoff
// (costs are >= 0) and moves one diagonal at a time, so before it could leave the
// band it would put a live cell, computed exactly, in a guard lane; the cutoff only
// decreases, so a path <= the final cutoff is live at every check.  On that event the
// pair stops with ovf set and the caller redoes it with a full-band engine.
//
// VIRT0 (DTW family): the caller guarantees both virtual diagonals dlo - 1 and dhi + 1 sit in
// slot 0 of their lanes (a symmetric band with w odd).  Only slot 0 then adds the +inf band
// offset.  Every other out-of-band slot lies beyond a virtual diagonal, starts at +inf and
// only ever sees +inf / NaN inputs (NaN from the +inf pads), so it stays +inf or NaN, which
// is dead for the liveness test and never selected by an in-band cell: the "if a < v"
// minimum never picks a NaN second argument, and an in-band cell's first argument is its
// own diagonal.
//
// W = 16: two pairs per warp, one per half (lanes 0-15 / 16-31), run in lockstep.  The
// caller guarantees both halves have the same shape (nl, nc, w) and passes no cutoff (the
// all-pairs engine): the loop bounds are then warp-uniform and nothing is ever abandoned,
// so the liveness vote is compiled out; shuffles stay inside a half (width 16).
template <int KIND, int MODE, int P, bool SHARED_CUT, bool GUARD = false, bool VIRT0 = false, int W = 32,
          class XAcc, class YAcc, class Loader>
__device__ DiagResult diag_pair(const XAcc& X, int nl, const YAcc& Y, int nc, int w, double cut64,
                                const unsigned long long* cutp, const Params& prm, Loader& ld,
                                unsigned guard = 0u) {
  static_assert(P % 2 == 0 && P >= 2, "P must be even");
  static_assert(W == 32 || (W == 16 && !SHARED_CUT && !GUARD), "half-warp pairs never abandon");
  using R = real_t<MODE>;
  const R INF = rinf<R>();
  R cut = to_cut<R>(cut64);
  constexpr int H = P / 2;
  constexpr bool BORDERED = (KIND == K_ERP);
  // the DTW family masks out-of-band diagonals through their cost (+inf offset)
  constexpr bool COST_MASK = (KIND == K_DTW || KIND == K_CDTW || KIND == K_WDTW);
  // MSM / TWE with VIRT0 (the guarded bands: both virtual diagonals in slot 0 of their lanes):
  // only slot 0 is masked, through its result: v + 0.0 == v exactly inside the band (v >= +0,
  // +inf or NaN), v + inf == +inf on a virtual diagonal (or NaN where v is: beyond the
  // matrix, never selected by an in-band cell).  Every other out-of-band slot lies beyond a
  // virtual diagonal, starts at +inf and only sees +inf / NaN inputs (as for the DTW family
  // above).  One FP64 add per lane and double step replaces the two selects per cell of
  // "upd ? v : INF": these cells are bound by the select (ALU) pipe.
  constexpr bool RES_MASK = (KIND == K_MSM || KIND == K_TWE) && VIRT0;
  const int lane = threadIdx.x & (W - 1);
  const int dlo = max(-w, 1 - nc), dhi = min(w, nl - 1);
  const int dbase = (dlo - 1) & ~1;  // floor to even, includes the lower virtual diagonal
  const int d0 = dbase + lane * P;

  int t_load = ld.next_t(dlo, dhi, H);
  if (t_load <= 2) {
    ld.ensure(2, dlo, dhi, H);
    t_load = ld.next_t(dlo, dhi, H);
  }
  R val[P];
  bool upd[P];
  int tb[P];  // ERP: border time of a virtual diagonal, else -1
  DiagK<KIND, R> kk[P];
  SlotS<KIND, R> st[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const int d = d0 + p;
    upd[p] = (d >= dlo) && (d <= dhi);
    tb[p] = (BORDERED && (d == dlo - 1 || d == dhi + 1)) ? (d < 0 ? -d : d) : -1;
    kk[p] = make_diag<KIND, R>(d, prm, upd[p] || !COST_MASK);
    val[p] = INF;
    if constexpr (KIND == K_TWE) st[p].pcp = (R)0.0;
    if (d == 0) val[p] = (R)0.0;  // corner, t = 0
    if (d == 1) {              // border cell (1,0) at t = 1
      if constexpr (BORDERED) val[p] = dadd((R)0.0, pcost<MODE>(X.at(0), (R)prm.gap));
      if constexpr (KIND == K_TWE) st[p].pcp = pcost<MODE>(X.at(0), (R)0.0);
    }
    if (d == -1) {             // border cell (0,1) at t = 1
      if constexpr (BORDERED) val[p] = dadd((R)0.0, pcost<MODE>((R)prm.gap, Y.at(0)));
      if constexpr (KIND == K_TWE) st[p].pcp = pcost<MODE>((R)0.0, Y.at(0));
    }
  }

  const R off0 = upd[0] ? (R)0.0 : INF;  // RES_MASK: slot 0's mask
  int t = 2;
  int I0 = (t + d0) >> 1, J0 = (t - d0) >> 1;
  RowD<KIND, R> xw[H + 1];
  ColD<KIND, R> yw[H];
#pragma unroll
  for (int k = 0; k <= H; ++k) xw[k] = make_row<KIND, MODE>(X.at(I0 + k - 1), X.at(I0 + k - 2), prm);
#pragma unroll
  for (int m = 0; m < H; ++m) yw[m] = make_col<KIND, MODE>(Y.at(J0 - m - 1), Y.at(J0 - m - 2), prm);

  const int Tf = nl + nc;
  int cut_hi = hi_word(cut);
  // MSM / TWE: a cell on diagonal d still needs |d - (nl - nc)| diagonal-changing moves to
  // reach the last cell, and each costs at least cmin (MSM: the split/merge cost c; TWE:
  // nu + lambda, a deletion's least cost).  Its path's final value is then at least
  // val + |d - dfin| cmin (less the rounding of the remaining additions, which the pre-test
  // margin of lb_threshold covers), so the cell is alive only while val <= cut' - k cmin:
  // one threshold per slot (its diagonal is fixed), refreshed with the cutoff.
  constexpr bool DBOUND = (KIND == K_MSM || KIND == K_TWE) && EKB_DBOUND;
  int thr_hi[DBOUND ? P : 1];
  double cmin = 0.0;
  if constexpr (DBOUND) cmin = KIND == K_MSM ? prm.msm_c : __dadd_rd(prm.nu, prm.lam);
  auto set_thr = [&](double c64) {
    if constexpr (DBOUND) {
      const double cm = lb_threshold<MODE>(c64, Tf);
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int k = abs(d0 + p - (nl - nc));
        thr_hi[p] = hi_word(to_cut<R>(__dsub_ru(cm, __dmul_rd((double)k, cmin))));
      }
    }
  };
  set_thr(cut64);
  bool dead = false;
  bool ovf = false;
#ifdef EKB_LIVE
  unsigned long long lv_ev = 0, lv_n = 0;
  bool sn_narrow = false, sn_ovf = false, sn_ever = false;
  int sn_wlo = 0;
  unsigned long long sn_votes = 0, sn_nvotes = 0, sn_shifts = 0;
  const int sn_lanes = (dhi + 2 - dbase + P - 1) / P;  // lanes holding the band
#endif

  // One double step.  With ROT the register windows are rings whose rotation
  // (rx for xw, ry for yw) is a compile-time function of the unrolled step S,
  // so sliding costs no register moves; otherwise the windows shift in place.
  constexpr bool ROT = (H <= EKB_ROT_MAX_H);
  constexpr int U = ROT ? H * (H + 1) : 1;
  // liveness accumulates over two double steps and is voted on every second one:
  // four consecutive dead anti-diagonals still cut every path, and the warp vote
  // (and the guard test: a path needs >= P/2 double steps to cross a P-diagonal guard
  // lane) runs half as often
  bool alive = false;
  // One double step evaluates two whole consecutive anti-diagonals (even slots at t, odd
  // slots at t+1: d = i - j has the parity of t = i + j), which every path crosses, so the
  // liveness of every second double step suffices: it is taken in the voting step only
  // (abandoning moves by at most one double step).  Guards: a path crossing a guard lane
  // visits its P >= 4 diagonals at >= 4 distinct anti-diagonals, and consecutive cells of
  // a path are at most 2 anti-diagonals apart, so it has a live cell in the lane in >= 2
  // consecutive double steps, one of which votes.
  auto live_step = [&](int S) { return ROT ? (S & 1) == 1 : ((t >> 1) & 1) == 1; };
  // ROT: the block's series loads address one base per block with compile-time offsets
  const R* xblk = X.p + I0;
  const R* yblk = Y.p + J0;
  // CHK: test for the end of the matrix after the step (only the block that can reach it)
  auto dstep = [&](auto S_, auto CHK_) -> bool {
    constexpr int S = decltype(S_)::value;
    constexpr bool CHK = decltype(CHK_)::value;
    constexpr int rx = ROT ? S % (H + 1) : 0;
    constexpr int ry = ROT ? (H - S % H) % H : 0;
    const bool lv = live_step(S);
    auto XW = [&](int k) -> RowD<KIND, R>& { return xw[(k + rx) % (H + 1)]; };
    auto YW = [&](int m) -> ColD<KIND, R>& { return yw[(m + ry) % H]; };
    // ---- half step A: time t, even slots; cell (I0+m, J0-m) ----
    R tin = __shfl_up_sync(FULL, val[P - 1], 1, W);
    if constexpr (BORDERED) {
      if (lane == 0) tin = INF;
    }
#pragma unroll
    for (int m = 0; m < H; ++m) {
      const int p = 2 * m;
      const R T = (m == 0) ? tin : val[p - 1];
      // slot 0's T arrives by shuffle: it enters its cell's minimum last
      const R v = (VIRT0 && p != 0) ? cell<KIND, MODE, false>(val[p], T, val[p + 1], XW(m), YW(m), kk[p], st[p], prm)
                                    : cell<KIND, MODE, true, true>(val[p], T, val[p + 1], XW(m), YW(m), kk[p], st[p], prm);
      if constexpr (BORDERED) {
        val[p] = (upd[p] || tb[p] == t) ? v : INF;
      } else if constexpr (COST_MASK) {
        val[p] = v;
      } else if constexpr (RES_MASK) {
        val[p] = (p == 0) ? dadd(v, off0) : v;
      } else {
        val[p] = upd[p] ? v : INF;
      }
      if (lv) alive |= hi_word(val[p]) <= (DBOUND ? thr_hi[DBOUND ? p : 0] : cut_hi);
#ifdef EKB_LIVE
      if (upd[p] && I0 + m >= 1 && I0 + m <= nl && J0 - m >= 1 && J0 - m <= nc) {
        ++lv_ev;
        lv_n += val[p] <= cut;
      }
#endif
    }
    // ---- half step B: time t+1, odd slots; cell (I0+m+1, J0-m) ----
    R lin = __shfl_down_sync(FULL, val[0], 1, W);
    if constexpr (BORDERED) {
      if (lane == W - 1) lin = INF;
    }
#pragma unroll
    for (int m = 0; m < H; ++m) {
      const int p = 2 * m + 1;
      const R L = (p == P - 1) ? lin : val[p + 1];
      const R v = VIRT0 ? cell<KIND, MODE, false>(val[p], val[p - 1], L, XW(m + 1), YW(m), kk[p], st[p], prm)
                        : cell<KIND, MODE>(val[p], val[p - 1], L, XW(m + 1), YW(m), kk[p], st[p], prm);
      if constexpr (BORDERED) {
        val[p] = (upd[p] || tb[p] == t + 1) ? v : INF;
      } else if constexpr (COST_MASK) {
        val[p] = v;
      } else if constexpr (RES_MASK) {
        val[p] = v;
      } else {
        val[p] = upd[p] ? v : INF;
      }
      if (lv) alive |= hi_word(val[p]) <= (DBOUND ? thr_hi[DBOUND ? p : 0] : cut_hi);
#ifdef EKB_LIVE
      if (upd[p] && I0 + m + 1 >= 1 && I0 + m + 1 <= nl && J0 - m >= 1 && J0 - m <= nc) {
        ++lv_ev;
        lv_n += val[p] <= cut;
      }
#endif
    }
    // the final cell (nl, nc) is on anti-diagonal Tf: if Tf == t it sits in an even
    // slot, which half step B (odd slots) leaves untouched
    if (CHK && t + 1 >= Tf) return true;
    const bool vote = W == 32 && (ROT ? (S & 1) == 1 : ((t >> 1) & 1) == 1);
    if (vote) {
#ifdef EKB_LIVE
      if constexpr (!GUARD && W == 32) {
        const unsigned m = __ballot_sync(FULL, alive);
        if (lane == 0) {
          const int span = m ? (32 - __clz(m)) - (__ffs(m) - 1) : 0;
          atomicAdd(&g_corr[min(t >> 6, 15) * 33 + span], 1ull);
          if (m && sn_lanes > 16) {
            const int lo = __ffs(m) - 1, hi = 31 - __clz(m);
            ++sn_votes;
            if (!sn_narrow) {
              if (hi - lo + 1 <= 12) {
                sn_narrow = sn_ever = true;
                sn_wlo = max(0, min(lo - 2, sn_lanes - 16));
              }
            } else if (sn_narrow) {
              ++sn_nvotes;
              const bool blo = lo < sn_wlo + 2 && sn_wlo > 0;
              const bool bhi = hi > sn_wlo + 13 && sn_wlo + 16 < sn_lanes;
              if (blo || bhi) {
                if (hi - lo + 1 <= 12) {
                  sn_wlo = max(0, min(lo - 2, sn_lanes - 16));
                  ++sn_shifts;
                } else {  // expand in place (counted per expansion)
                  sn_ovf = true;
                  sn_narrow = false;
                  atomicAdd(&g_sn[7], 1ull);
                }
              }
            }
          }
        }
      }
#endif
      if constexpr (GUARD) {
        const unsigned live = __ballot_sync(FULL, alive);
        if (!live) {
          dead = true;
          return true;
        }
        if (live & guard) {
          ovf = true;
          return true;
        }
      } else if (!__any_sync(FULL, alive)) {
        dead = true;
        return true;
      }
      alive = false;
    }
    // ---- slide the register windows by one element ----
    t += 2;
    ++I0;
    ++J0;
    if constexpr (!ROT) {
      if (t >= t_load) {
        ld.ensure(t, dlo, dhi, H);
        t_load = ld.next_t(dlo, dhi, H);
      }
    }
    if constexpr (ROT) {
      // logical xw[H] of the next step is ring slot rx; logical yw[0] is ring slot (ry+H-1)%H
      // (I0 / J0 are the block's base + S + 1 here)
      const R xprev = XW(H).x;
      const R yprev = YW(0).y;
#ifdef EKB_BOUNDS
      (void)X.at(I0 + H - 1);
      (void)Y.at(J0 - 1);
#endif
      xw[rx] = make_row<KIND, MODE>(xblk[S + H], xprev, prm);
      yw[(ry + H - 1) % H] = make_col<KIND, MODE>(yblk[S], yprev, prm);
    } else {
#pragma unroll
      for (int k = 0; k < H; ++k) xw[k] = xw[k + 1];
      xw[H] = make_row<KIND, MODE>(X.at(I0 + H - 1), xw[H - 1].x, prm);
#pragma unroll
      for (int m = H - 1; m > 0; --m) yw[m] = yw[m - 1];
      yw[0] = make_col<KIND, MODE>(Y.at(J0 - 1), yw[0].y, prm);
    }
    return false;
  };
  constexpr int REP = (U >= 16) ? 1 : 16 / U;  // unrolled blocks between cutoff refreshes
  bool finished = false;
  while (!finished) {
    unsigned long long nextcut = 0;
    if constexpr (SHARED_CUT) nextcut = ld_cut_raw(cutp);  // broadcast after this block of double steps
#pragma unroll 1
    for (int b = 0; b < REP && !finished; ++b) {
      if constexpr (ROT) {  // stage series data for the whole unrolled block at once
        if (t + 2 * U >= t_load) {
          ld.ensure(t + 2 * U, dlo, dhi, H);
          t_load = ld.next_t(dlo, dhi, H);
        }
      }
      xblk = X.p + I0;
      yblk = Y.p + J0;
      // blocks that end before anti-diagonal Tf skip the per-step end test
      if (t + 2 * U + 1 < Tf) {
        auto fast = [&](auto S_) { return dstep(S_, std::false_type{}); };
        finished = unrolled_steps<0, U>(fast);
      } else {
        auto last = [&](auto S_) { return dstep(S_, std::true_type{}); };
        finished = unrolled_steps<0, U>(last);
      }
    }
    if constexpr (SHARED_CUT) {
      const double c64 = bcast_cut(nextcut);
      cut = fmin(cut, to_cut<R>(c64));
      cut_hi = hi_word(cut);
      if constexpr (DBOUND) {
        cut64 = fmin(cut64, c64);
        set_thr(cut64);
      }
    }
  }

#ifdef EKB_LIVE
  for (int o = W / 2; o; o >>= 1) {
    lv_ev += __shfl_xor_sync(FULL, lv_ev, o, W);
    lv_n += __shfl_xor_sync(FULL, lv_n, o, W);
  }
  if (lane == 0) {
    atomicAdd(&g_live[0], lv_ev);
    atomicAdd(&g_live[1], lv_n);
    if (sn_votes) {
      atomicAdd(&g_sn[0], 1ull);
      atomicAdd(&g_sn[1], sn_ever ? 1ull : 0ull);
      atomicAdd(&g_sn[2], sn_ovf ? 1ull : 0ull);
      atomicAdd(&g_sn[3], sn_votes);
      atomicAdd(&g_sn[4], sn_nvotes);
      atomicAdd(&g_sn[5], sn_ovf ? sn_nvotes : 0ull);
      atomicAdd(&g_sn[6], sn_shifts);
    }
  }
#endif
  DiagResult res;
  res.t_end = (dead || ovf) ? t + 1 : Tf;  // last anti-diagonal evaluated
  res.ovf = ovf;
  if (dead || ovf) {
    res.cost = EKB_INF;
    return res;
  }
  if constexpr (SHARED_CUT) cut = fmin(cut, to_cut<R>(ld_cut(cutp)));
  const int sf = (nl - nc) - dbase;
  const int pf = sf % P;
  R r = val[0];
#pragma unroll
  for (int p = 1; p < P; ++p)
    if (p == pf) r = val[p];
  r = __shfl_sync(FULL, r, sf / P, W);
  res.cost = (r <= cut) ? (double)r : EKB_INF;
  return res;
}

// Slots needed by diag_pair for this band: the lanes must cover [dbase, dhi+1].
__host__ __device__ inline int diag_slots_needed(int nl, int nc, int w) {
  int dlo = (-w > 1 - nc) ? -w : 1 - nc;
  int dhi = (w < nl - 1) ? w : nl - 1;
  int dbase = (dlo - 1) & ~1;
  return dhi + 2 - dbase;
}

}  // namespace ekb
