// ek_stripe.cuh -- warp-per-pair row wavefront over column stripes, for wide or
// unconstrained bands and for the row-based "ea" variant.
//
// Lane l owns columns (l*S, (l+1)*S] (1-based) and keeps the previous row's
// values for them in registers; at step t it evaluates row i = r0 + t - l, so
// lane l-1 hands over the value of its last column for row i (one shuffle per
// row per lane).  Rows stream from shared memory; the S column records are
// loaded once per pair.  Out-of-band cells (|i-j| > w) are +inf, exactly the
// reference's windowed engines (_speedups.pyx:129-271), and the left border
// (i,0) / top border row 0 follow kernels.py:244-262 (ERP: sequential prefixes,
// evaluated here by the recurrence itself along row 0 / by lane 0 down column 0).
//
// Abandoning: cells evaluated at steps t-1 and t form a cut of every alignment
// path (a move advances the step by at most 2), so "no cell <= cutoff in two
// consecutive steps" abandons with the eapruned contract (exact iff <= cutoff).
// With EA=true the engine instead reproduces the reference's classic row
// abandoning (_speedups.pyx:129-162): the running row minimum (border cell
// included) travels along with the hand-over value, the lane holding the last
// column of the row sees the complete minimum, and any row minimum > cutoff
// makes the result +inf; otherwise the exact cost is returned even if > cutoff.
#pragma once
#include "ek_common.cuh"
#include "ek_diag.cuh"

namespace ekb {

struct StripeResult {
  double cost;
  int t_end;  // steps executed
};

// tab: per-pair |i-j| table in shared memory (WDTW: weights; TWE: nu*(d+d)); len >= max(nl,nc)+1.
template <int KIND, int MODE, int S, bool BANDED, bool SHARED_CUT, bool EA, class XAcc, class YAcc>
__device__ StripeResult stripe_pair(const XAcc& X, int nl, const YAcc& Y, int nc, int w, double cut,
                                    const unsigned long long* cutp, const double* tab, int tablen,
                                    const Params& prm) {
  const int lane = threadIdx.x & 31;
  constexpr bool BORDERED = (KIND == K_ERP);
  constexpr bool TWE = (KIND == K_TWE);
  const int r0 = BORDERED ? 0 : 1;  // ERP evaluates the top border row through the recurrence
  const int jbase = lane * S;       // columns jbase+1 .. jbase+S
  const int lf = (nc - 1) / S;      // lane holding column nc
  const bool lane_on = jbase < nc;

  auto cy = [&](int k) { return Y.at(min(max(k, -1), nc)); };  // column records: once per pair
  auto cx = [&](int k) { return X.at(k); };                      // rows: padded by >= 40

  ColD<KIND> cols[S];
  double val[S];
  double pcr[TWE ? S : 1];  // TWE: pc of the previous row per column
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int j = jbase + 1 + s;
    cols[s] = make_col<KIND, MODE>(cy(j - 1), cy(j - 2), prm);
    val[s] = EKB_INF;
    if constexpr (TWE) pcr[s] = pcost<MODE>(cx(r0 - 2), cols[s].y);
  }
  // hand-over state from the left neighbour (value of column jbase for the previous row)
  double dg = EKB_INF;     // (i-1, jbase)
  double dgpc = 0.0;       // TWE: pc at (i-1, jbase)
  double xprev = cx(r0 - 2);
  double vb = 0.0;         // lane 0: ERP left border accumulator
  const double ycol0 = cy(jbase - 1);  // c_{jbase} for the column-0 pc of lane 0 / TWE hand-over
  if (lane == 0) {
    dg = BORDERED ? EKB_INF : 0.0;  // (r0-1, 0): ERP starts at row 0 (nothing above); else corner (0,0)
    if constexpr (TWE) dgpc = pcost<MODE>(cx(r0 - 2), ycol0);
  }
  if constexpr (TWE) {
    if (lane != 0) dgpc = pcost<MODE>(cx(r0 - 2), ycol0);
  }

  const int nsteps = nl - r0 + lf + 1;  // the last lane that matters finishes row nl
  bool alive2 = false;                  // alive over the previous step
  bool ea_flag = false;                 // EA: some row minimum exceeded the cutoff
  double nextcut = cut;
  int t = 0;
  bool dead = false;
  double lastv = EKB_INF;  // value of the lane's last column for the current row
  double lastpc = 0.0;
  double rowmin_out = EKB_INF;
  for (t = 0; t < nsteps; ++t) {
    if constexpr (SHARED_CUT) {
      if ((t & 31) == 0) nextcut = ld_cut(cutp);
      if ((t & 31) == 24) cut = fmin(cut, nextcut);
    }
    const int i = r0 + t - lane;  // this lane's row
    // receive the left neighbour's last column for row i (computed at step t-1)
    double lb = __shfl_up_sync(FULL, lastv, 1);
    double lbpc = TWE ? __shfl_up_sync(FULL, lastpc, 1) : 0.0;
    double rmin = EA ? __shfl_up_sync(FULL, rowmin_out, 1) : EKB_INF;
    const double x = cx(i - 1);
    const RowD<KIND> rd = make_row<KIND, MODE>(x, xprev, prm);
    xprev = x;
    if (lane == 0) {
      // border cell (i, 0)
      if constexpr (BORDERED) {
        if (i == 0) vb = 0.0;
        else vb = dadd(vb, rd.ar);  // vb[i] = vb[i-1] + pc(l_i, g)
        lb = (i <= w + 1) ? vb : EKB_INF;
      } else {
        lb = (i == 0) ? 0.0 : EKB_INF;
      }
      if constexpr (TWE) lbpc = pcost<MODE>(x, 0.0);  // pc(l_i, c_0 := 0) of the border cell
      rmin = (i >= 1) ? lb : EKB_INF;                 // ea: the border cell joins the row minimum
    }
    const bool row_ok = (i >= r0) && (i <= nl);
    bool alive = row_ok && lane == 0 && (lb <= cut);
    // band of row i within this stripe: slots [a, b]
    int a = 0, b = S - 1;
    if constexpr (BANDED) {
      const int hi = (i == 0) ? w + 1 : i + w;  // row 0 keeps hborder up to j = w+1
      a = i - w - jbase - 1;
      b = hi - jbase - 1;
    }
    double dgl = dg, lft = lb, dpc = dgpc;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int j = jbase + 1 + s;
      const double up = val[s];
      DiagK<KIND> k{};  // off = 0.0: the stripe engine masks the band itself
      if constexpr (KIND == K_WDTW) k.w = tab[min(abs(i - j), tablen - 1)];
      if constexpr (TWE) k.tw = tab[min(abs(i - j), tablen - 1)];
      SlotS<KIND> stt;
      double upc = 0.0;
      if constexpr (TWE) {
        stt.pcp = dpc;
        upc = pcr[s];
      }
      double v = cell<KIND, MODE, false>(dgl, up, lft, rd, cols[s], k, stt, prm);
      if constexpr (BANDED) v = (s >= a && s <= b) ? v : EKB_INF;
      if constexpr (TWE) {
        pcr[s] = stt.pcp;  // pc(l_i, c_j) for the next row
        dpc = upc;
      }
      val[s] = v;
      dgl = up;
      lft = v;
      alive |= row_ok && (j <= nc) && (v <= cut);
      if constexpr (EA) rmin = (v < rmin) ? v : rmin;
    }
    dg = lb;
    dgpc = lbpc;
    lastv = val[S - 1];
    if constexpr (TWE) lastpc = pcr[S - 1];
    if constexpr (EA) {
      rowmin_out = rmin;
      if (lane == lf && row_ok && i >= 1 && rmin > cut) ea_flag = true;
    }
    if constexpr (!EA) {
      if (t & 1) {
        if (!__any_sync(FULL, alive || alive2)) { dead = true; break; }
      }
      alive2 = alive;
    } else {
      if ((t & 31) == 31 && __any_sync(FULL, ea_flag)) { dead = true; break; }
    }
  }
  (void)lane_on;
  StripeResult res;
  res.t_end = dead ? t + 1 : nsteps;
  if (dead) {
    res.cost = EKB_INF;
    return res;
  }
  // cell (nl, nc) lives in lane lf, slot (nc-1) % S, computed at its last step
  const int sf = (nc - 1) % S;
  double r = val[0];
#pragma unroll
  for (int s = 1; s < S; ++s)
    if (s == sf) r = val[s];
  r = __shfl_sync(FULL, r, lf);
  if constexpr (EA) {
    const bool flagged = __any_sync(FULL, ea_flag);
    res.cost = flagged ? EKB_INF : r;
  } else {
    if constexpr (SHARED_CUT) cut = fmin(cut, ld_cut(cutp));
    res.cost = (r <= cut) ? r : EKB_INF;
  }
  return res;
}

}  // namespace ekb
