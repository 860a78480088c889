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
  int t_end;   // steps executed
  int ea_row;  // EA: first row whose minimum exceeded the cutoff (0x7fffffff if none)
};

// Row recorder: the default records nothing.  RowBits (ek_refcells.cuh) keeps each
// row's "value <= cutoff" bits so the reference's own cell count can be replayed.
struct NoRec {
  static constexpr bool on = false;
  __device__ __forceinline__ void row(int, int, unsigned) const {}
  __device__ __forceinline__ void vb(int, bool) const {}
};

// tab: the entry d = i - j = 0 of the two-sided |i-j| table in shared memory (stage_table2;
// WDTW: weights; TWE: nu*(d+d)), covering d in [-(nc + 2S), nl + S].
// W = 16: two pairs per warp (one per half-warp) in lockstep, all-pairs only (no cutoff,
// no ea rows, no recorder): the caller guarantees equal shapes, so the step count is
// warp-uniform and the abandon vote is compiled out; shuffles stay inside a half.
template <int KIND, int MODE, int S, bool BANDED, bool SHARED_CUT, bool EA, class XAcc, class YAcc,
          class Rec = NoRec, int W = 32>
__device__ StripeResult stripe_pair(const XAcc& X, int nl, const YAcc& Y, int nc, int w, double cut64,
                                    const unsigned long long* cutp, const real_t<MODE>* tab, int tablen,
                                    const Params& prm, const Rec& rec = Rec{}) {
  static_assert(W == 32 || (W == 16 && !SHARED_CUT && !EA && !Rec::on), "half-warp pairs never abandon");
  using R = real_t<MODE>;
  const R INF = rinf<R>();
  R cut = to_cut<R>(cut64);
  const int lane = threadIdx.x & (W - 1);
  constexpr bool BORDERED = (KIND == K_ERP);
  constexpr bool TWE = (KIND == K_TWE);
  const int r0 = BORDERED ? 0 : 1;  // ERP evaluates the top border row through the recurrence
  const int jbase = lane * S;       // columns jbase+1 .. jbase+S
  const int lf = (nc - 1) / S;      // lane holding column nc
  const bool lane_on = jbase < nc;

  auto cy = [&](int k) { return Y.at(min(max(k, -1), nc)); };  // column records: once per pair
  // rows: lanes run up to 62 rows ahead of / behind the matrix; clamp to the pads (the
  // +inf pad past the end, a finite one before it) so those rows stay +inf
  auto cx = [&](int k) { return X.at(min(max(k, -1), nl)); };

  ColD<KIND, R> cols[S];
  R val[S];
  R pcr[TWE ? S : 1];  // TWE: pc of the previous row per column
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int j = jbase + 1 + s;
    cols[s] = make_col<KIND, MODE>(cy(j - 1), cy(j - 2), prm);
    val[s] = INF;
    if constexpr (TWE) pcr[s] = pcost<MODE>(cx(r0 - 2), cols[s].y);
  }
  // hand-over state from the left neighbour (value of column jbase for the previous row)
  R dg = INF;     // (i-1, jbase)
  R dgpc = R(0);       // TWE: pc at (i-1, jbase)
  R xprev = cx(r0 - 2);
  R vb = R(0);         // lane 0: ERP left border accumulator
  const R ycol0 = cy(jbase - 1);  // c_{jbase} for the column-0 pc of lane 0 / TWE hand-over
  if (lane == 0) {
    dg = BORDERED ? INF : R(0);  // (r0-1, 0): ERP starts at row 0 (nothing above); else corner (0,0)
    if constexpr (TWE) dgpc = pcost<MODE>(cx(r0 - 2), ycol0);
  }
  if constexpr (TWE) {
    if (lane != 0) dgpc = pcost<MODE>(cx(r0 - 2), ycol0);
  }

  // Two rows per step: lane l evaluates rows i0 = r0 + 2(t-l) and i1 = i0 + 1.  Row i1
  // trails row i0 by one column inside the lane, so the two dependency chains
  // interleave (the compiler schedules the fully unrolled straight-line code).
  const int nsteps = lf + (nl - r0) / 2 + 1;  // lane lf reaches row nl in its last step
  const bool last_is_i0 = ((nl - r0) & 1) == 0;
  bool alive2 = false;   // alive over the previous step
  bool ea_flag = false;  // EA: some row minimum exceeded the cutoff
  R nextcut = cut;
  int cut_hi = hi_word(cut);
  int t = 0;
  bool dead = false;
  R last0 = INF, last1 = INF;  // this lane's last column for rows i0 / i1
  R lastpc0 = R(0), lastpc1 = R(0);
  R rmo0 = INF, rmo1 = INF;
  R fin = INF;  // final cell when row nl is an i0 row
  const int sf = (nc - 1) % S;

  // one row over this lane's S columns; prev[] holds row i-1 on entry, row i on exit
  int ea_row = 0x7fffffff;
  auto row_pass = [&](int i, const RowD<KIND, R>& rd, R lft, R dgl, R dpc, R& rmin,
                      R (&row)[S], bool& alive) {
    unsigned live_bits = 0;
    int a = 0, b = S - 1;
    if constexpr (BANDED) {
      const int hi = (i == 0) ? w + 1 : i + w;  // row 0 keeps hborder up to j = w+1
      a = i - w - jbase - 1;
      b = hi - jbase - 1;
    }
    // tab points at d = i - j = 0 of a two-sided table (stage_table2): this row's base,
    // clamped so garbage rows / lanes stay inside it (cells of the matrix never clamp)
    const R* trow = tab + min(max(i - jbase - 1, -(nc + S)), nl + S);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int j = jbase + 1 + s;
      const R up = row[s];
      DiagK<KIND, R> k{};  // off = 0.0: the stripe engine masks the band itself
      if constexpr (KIND == K_WDTW) k.w = trow[-s];
      if constexpr (TWE) k.tw = trow[-s];
      SlotS<KIND, R> stt;
      R upc = R(0);
      if constexpr (TWE) {
        stt.pcp = dpc;
        upc = pcr[s];
      }
      R v = cell<KIND, MODE, false>(dgl, up, lft, rd, cols[s], k, stt, prm);
      if constexpr (BANDED) v = (s >= a && s <= b) ? v : INF;
      if constexpr (TWE) {
        pcr[s] = stt.pcp;  // pc(l_i, c_j) for the next row
        dpc = upc;
      }
      row[s] = v;
      dgl = up;
      lft = v;
      // garbage cells (before the first row, past the last row or column) are +inf
      // or only delay abandoning; the hi-word test is conservative (ek_diag.cuh)
      alive |= hi_word(v) <= cut_hi;
      if constexpr (EA) rmin = (v < rmin) ? v : rmin;
      if constexpr (Rec::on) live_bits |= (unsigned)(j <= nc && v <= cut) << s;
    }
    if constexpr (Rec::on) {
      if (i >= 0 && i <= nl) rec.row(i, lane, live_bits);
    }
  };

  for (t = 0; t < nsteps; ++t) {
    if constexpr (SHARED_CUT) {
      if ((t & 15) == 0) nextcut = to_cut<R>(ld_cut(cutp));
      if ((t & 15) == 12) {
        cut = fmin(cut, nextcut);
        cut_hi = hi_word(cut);
      }
    }
    const int i0 = r0 + 2 * (t - lane), i1 = i0 + 1;
    // the left neighbour's last column for rows i0, i1 (computed at step t-1)
    R lb0 = __shfl_up_sync(FULL, last0, 1, W);
    R lb1 = __shfl_up_sync(FULL, last1, 1, W);
    R lbpc0 = TWE ? __shfl_up_sync(FULL, lastpc0, 1, W) : R(0);
    R lbpc1 = TWE ? __shfl_up_sync(FULL, lastpc1, 1, W) : R(0);
    R rm0 = EA ? __shfl_up_sync(FULL, rmo0, 1, W) : INF;
    R rm1 = EA ? __shfl_up_sync(FULL, rmo1, 1, W) : INF;
    const R x0 = cx(i0 - 1), x1 = cx(i1 - 1);
    const RowD<KIND, R> rd0 = make_row<KIND, MODE>(x0, xprev, prm);
    const RowD<KIND, R> rd1 = make_row<KIND, MODE>(x1, x0, prm);
    xprev = x1;
    if (lane == 0) {
      // border cells (i0, 0), (i1, 0)
      if constexpr (BORDERED) {
        vb = (i0 == 0) ? R(0) : dadd(vb, rd0.ar);  // vb[i] = vb[i-1] + pc(l_i, g)
        lb0 = (i0 <= w + 1) ? vb : INF;
        vb = dadd(vb, rd1.ar);
        lb1 = (i1 <= w + 1) ? vb : INF;
      } else {
        lb0 = (i0 == 0) ? R(0) : INF;
        lb1 = INF;
      }
      if constexpr (TWE) {
        lbpc0 = pcost<MODE>(x0, R(0));  // pc(l_i, c_0 := 0) of the border cell
        lbpc1 = pcost<MODE>(x1, R(0));
      }
      rm0 = (i0 >= 1) ? lb0 : INF;  // ea: the border cell joins the row minimum
      rm1 = (i1 >= 1) ? lb1 : INF;
      if constexpr (Rec::on) {
        if (i0 >= 1 && i0 <= nl) rec.vb(i0, lb0 <= cut);
        if (i1 >= 1 && i1 <= nl) rec.vb(i1, lb1 <= cut);
      }
    }
    bool alive = lane == 0 && (hi_word(lb0) <= cut_hi || hi_word(lb1) <= cut_hi);
    R row0[S];
#pragma unroll
    for (int s2 = 0; s2 < S; ++s2) row0[s2] = val[s2];
    // row i0: diagonal input (i0-1, jbase) is the left neighbour's row i1 of step t-1
    row_pass(i0, rd0, lb0, dg, dgpc, rm0, row0, alive);
    if constexpr (TWE) lastpc0 = pcr[S - 1];
    if (t == nsteps - 1 && last_is_i0) {
#pragma unroll
      for (int s2 = 0; s2 < S; ++s2)
        if (s2 == sf) fin = row0[s2];
    }
#pragma unroll
    for (int s2 = 0; s2 < S; ++s2) val[s2] = row0[s2];
    // row i1: diagonal input (i0, jbase) = lb0
    row_pass(i1, rd1, lb1, lb0, lbpc0, rm1, val, alive);
    if constexpr (TWE) lastpc1 = pcr[S - 1];
    dg = lb1;
    dgpc = lbpc1;
    last0 = row0[S - 1];
    last1 = val[S - 1];
    if constexpr (EA) {
      rmo0 = rm0;
      rmo1 = rm1;
      if (lane == lf) {
        if (i0 >= 1 && i0 <= nl && rm0 > cut) {
          ea_flag = true;
          ea_row = min(ea_row, i0);
        }
        if (i1 >= 1 && i1 <= nl && rm1 > cut) {
          ea_flag = true;
          ea_row = min(ea_row, i1);
        }
      }
    }
    if constexpr (!EA) {
      if (W == 32 && (t & 1)) {
        if (!__any_sync(FULL, alive || alive2)) { dead = true; break; }
      }
      alive2 = alive;
    } else {
      if ((t & 15) == 15 && __any_sync(FULL, ea_flag)) { dead = true; break; }
    }
  }
  (void)lane_on;
  StripeResult res;
  res.t_end = dead ? t + 1 : nsteps;
  res.ea_row = EA ? __shfl_sync(FULL, ea_row, lf) : 0x7fffffff;
  if (dead) {
    res.cost = EKB_INF;
    return res;
  }
  // cell (nl, nc) lives in lane lf, slot (nc-1) % S, computed at its last step
  R r = val[0];
#pragma unroll
  for (int s = 1; s < S; ++s)
    if (s == sf) r = val[s];
  if (last_is_i0) r = fin;
  r = __shfl_sync(FULL, r, lf, W);
  if constexpr (EA) {
    const bool flagged = __any_sync(FULL, ea_flag);
    res.cost = flagged ? INF : r;
  } else {
    if constexpr (SHARED_CUT) cut = fmin(cut, to_cut<R>(ld_cut(cutp)));
    res.cost = (r <= cut) ? r : INF;
  }
  return res;
}

}  // namespace ekb

namespace ekb {

// Long series (more than 32 x 16 columns): the row-stripe engine over vertical strips of
// 512 columns, one after another.  Strip k reads its left boundary column (column 512k,
// rows 0..nl) from `bin` and writes its own last column to `bout` for strip k + 1; the
// two buffers (nl + 1 doubles each, per warp) swap between strips.  Inside strip 0 the
// two-dead-steps cut is valid as in stripe_pair; later strips can be re-entered from
// their left boundary, so they only stop the pair when a whole boundary column is dead
// (every path crosses every column).  The same cells, borders and band masks as
// stripe_pair, so values are bit-identical.  EA (`ea` with a finite cutoff): a row's
// minimum spans every strip, so nothing is abandoned; each strip folds its row minima
// (border cell included, _speedups.pyx:147-160) into `rmin` and the result is +inf if
// any row minimum exceeds the cutoff, else the exact cost.
template <int KIND, int MODE, bool BANDED, bool SHARED_CUT, bool EA, class XAcc, class YAcc>
__device__ StripeResult strip_pair(const XAcc& X, int nl, const YAcc& Y, int nc, int w, double cut64,
                                   const unsigned long long* cutp, const real_t<MODE>* tab, int tablen,
                                   const Params& prm, real_t<MODE>* bin, real_t<MODE>* bout, real_t<MODE>* rmin) {
  using R = real_t<MODE>;
  const R INF = rinf<R>();
  R cut = to_cut<R>(cut64);
  constexpr int S = 16;
  constexpr int STRIP = 32 * S;
  const int lane = threadIdx.x & 31;
  constexpr bool BORDERED = (KIND == K_ERP);
  constexpr bool TWE = (KIND == K_TWE);
  const int r0 = BORDERED ? 0 : 1;
  const int nstrips = (nc + STRIP - 1) / STRIP;
  auto cy = [&](int k) { return Y.at(min(max(k, -1), nc)); };
  auto cx = [&](int k) { return X.at(min(max(k, -1), nl)); };  // see stripe_pair
  R nextcut = cut;
  int cut_hi = hi_word(cut);
  int steps_done = 0;
  R result = INF;
  bool dead = false;
  if constexpr (EA) {
    for (int i = lane; i <= nl; i += 32) rmin[i] = INF;
    __syncwarp();
  }

  for (int sk = 0; sk < nstrips && !dead; ++sk) {
    const int jbase = sk * STRIP + lane * S;
    const bool last_strip = sk == nstrips - 1;
    const int lf = last_strip ? (nc - 1 - sk * STRIP) / S : 31;
    const int sf = (nc - 1) % S;
    ColD<KIND, R> cols[S];
    R val[S];
    R pcr[TWE ? S : 1];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int j = jbase + 1 + s;
      cols[s] = make_col<KIND, MODE>(cy(j - 1), cy(j - 2), prm);
      val[s] = INF;
      if constexpr (TWE) pcr[s] = pcost<MODE>(cx(r0 - 2), cols[s].y);
    }
    R dg = INF, dgpc = R(0);
    R xprev = cx(r0 - 2);
    R vb = R(0);
    const R ycol0 = cy(jbase - 1);
    if (lane == 0 && sk == 0) dg = BORDERED ? INF : R(0);
    if constexpr (TWE) dgpc = pcost<MODE>(cx(r0 - 2), ycol0);
    const int nsteps = lf + (nl - r0) / 2 + 1;
    const bool last_is_i0 = ((nl - r0) & 1) == 0;
    bool alive2 = false;
    R last0 = INF, last1 = INF, lastpc0 = R(0), lastpc1 = R(0);
    R rmo0 = INF, rmo1 = INF;
    R fin = INF;

    auto row_pass = [&](int i, const RowD<KIND, R>& rd, R lft, R dgl, R dpc, R (&row)[S],
                        bool& alive, R& rm) {
      int a = 0, b = S - 1;
      if constexpr (BANDED) {
        const int hi = (i == 0) ? w + 1 : i + w;
        a = i - w - jbase - 1;
        b = hi - jbase - 1;
      }
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int j = jbase + 1 + s;
        const R up = row[s];
        DiagK<KIND, R> k{};
        if constexpr (KIND == K_WDTW) k.w = tab[min(abs(i - j), tablen - 1)];
        if constexpr (TWE) k.tw = tab[min(abs(i - j), tablen - 1)];
        SlotS<KIND, R> stt;
        R upc = R(0);
        if constexpr (TWE) {
          stt.pcp = dpc;
          upc = pcr[s];
        }
        R v = cell<KIND, MODE, false>(dgl, up, lft, rd, cols[s], k, stt, prm);
        if constexpr (BANDED) v = (s >= a && s <= b) ? v : INF;
        if constexpr (TWE) {
          pcr[s] = stt.pcp;
          dpc = upc;
        }
        row[s] = v;
        dgl = up;
        lft = v;
        alive |= hi_word(v) <= cut_hi;
        if constexpr (EA) rm = (v < rm) ? v : rm;
      }
    };

    int t = 0;
    for (t = 0; t < nsteps; ++t) {
      if constexpr (SHARED_CUT) {
        if ((t & 15) == 0) nextcut = to_cut<R>(ld_cut(cutp));
        if ((t & 15) == 12) {
          cut = fmin(cut, nextcut);
          cut_hi = hi_word(cut);
        }
      }
      const int i0 = r0 + 2 * (t - lane), i1 = i0 + 1;
      R lb0 = __shfl_up_sync(FULL, last0, 1);
      R lb1 = __shfl_up_sync(FULL, last1, 1);
      R lbpc0 = TWE ? __shfl_up_sync(FULL, lastpc0, 1) : R(0);
      R lbpc1 = TWE ? __shfl_up_sync(FULL, lastpc1, 1) : R(0);
      R rm0 = EA ? __shfl_up_sync(FULL, rmo0, 1) : INF;
      R rm1 = EA ? __shfl_up_sync(FULL, rmo1, 1) : INF;
      const R x0 = cx(i0 - 1), x1 = cx(i1 - 1);
      const RowD<KIND, R> rd0 = make_row<KIND, MODE>(x0, xprev, prm);
      const RowD<KIND, R> rd1 = make_row<KIND, MODE>(x1, x0, prm);
      xprev = x1;
      if (lane == 0) {
        if (sk == 0) {  // the matrix border (stripe_pair's lane 0)
          if constexpr (BORDERED) {
            vb = (i0 == 0) ? R(0) : dadd(vb, rd0.ar);
            lb0 = (i0 <= w + 1) ? vb : INF;
            vb = dadd(vb, rd1.ar);
            lb1 = (i1 <= w + 1) ? vb : INF;
          } else {
            lb0 = (i0 == 0) ? R(0) : INF;
            lb1 = INF;
          }
          if constexpr (TWE) {
            lbpc0 = pcost<MODE>(x0, R(0));
            lbpc1 = pcost<MODE>(x1, R(0));
          }
          rm0 = (i0 >= 1) ? lb0 : INF;  // ea: the border cell joins the row minimum
          rm1 = (i1 >= 1) ? lb1 : INF;
        } else {  // the previous strip's last column (already in the previous strip's minimum)
          rm0 = INF;
          rm1 = INF;
          lb0 = (i0 >= 0 && i0 <= nl) ? bin[i0] : INF;
          lb1 = (i1 >= 0 && i1 <= nl) ? bin[i1] : INF;
          if constexpr (TWE) {
            lbpc0 = pcost<MODE>(x0, ycol0);
            lbpc1 = pcost<MODE>(x1, ycol0);
          }
        }
      }
      bool alive = lane == 0 && (hi_word(lb0) <= cut_hi || hi_word(lb1) <= cut_hi);
      R row0[S];
#pragma unroll
      for (int s2 = 0; s2 < S; ++s2) row0[s2] = val[s2];
      row_pass(i0, rd0, lb0, dg, dgpc, row0, alive, rm0);
      if constexpr (TWE) lastpc0 = pcr[S - 1];
      if (t == nsteps - 1 && last_is_i0) {
#pragma unroll
        for (int s2 = 0; s2 < S; ++s2)
          if (s2 == sf) fin = row0[s2];
      }
#pragma unroll
      for (int s2 = 0; s2 < S; ++s2) val[s2] = row0[s2];
      row_pass(i1, rd1, lb1, lb0, lbpc0, val, alive, rm1);
      if constexpr (TWE) lastpc1 = pcr[S - 1];
      dg = lb1;
      dgpc = lbpc1;
      last0 = row0[S - 1];
      last1 = val[S - 1];
      if (!last_strip && lane == 31) {  // this strip's last column for the next strip
        if (i0 >= 0 && i0 <= nl) bout[i0] = last0;
        if (i1 >= 0 && i1 <= nl) bout[i1] = last1;
      }
      if constexpr (EA) {
        rmo0 = rm0;
        rmo1 = rm1;
        if (lane == lf) {  // the strip's row minima (lane lf holds column nc in the last strip)
          if (i0 >= 1 && i0 <= nl) rmin[i0] = fmin(rmin[i0], rm0);
          if (i1 >= 1 && i1 <= nl) rmin[i1] = fmin(rmin[i1], rm1);
        }
      }
      if (nstrips == 1 && !EA) {  // a cut of every path only when the strip spans all columns
        if (t & 1) {
          if (!__any_sync(FULL, alive || alive2)) {
            dead = true;
            break;
          }
        }
        alive2 = alive;
      }
    }
    steps_done += dead ? t + 1 : nsteps;
    if (dead) break;
    if (!last_strip) {
      __syncwarp();
      bool any = EA;  // a dead boundary column ends every path
      for (int i = r0 + lane; i <= nl; i += 32) any |= hi_word(bout[i]) <= cut_hi;
      if (!__any_sync(FULL, any)) {
        dead = true;
        break;
      }
      R* tmp = bin;
      bin = bout;
      bout = tmp;
      __syncwarp();
    } else {
      R r = val[0];
#pragma unroll
      for (int s = 1; s < S; ++s)
        if (s == sf) r = val[s];
      if (last_is_i0) r = fin;
      result = __shfl_sync(FULL, r, lf);
    }
  }
  StripeResult res;
  res.t_end = steps_done;
  res.ea_row = 0x7fffffff;
  if (dead) {
    res.cost = EKB_INF;
    return res;
  }
  if constexpr (EA) {  // _ea: +inf iff some row minimum exceeds the cutoff, else the exact cost
    __syncwarp();
    bool over = false;
    for (int i = 1 + lane; i <= nl; i += 32) over |= rmin[i] > cut;
    res.cost = __any_sync(FULL, over) ? INF : result;
    return res;
  }
  if constexpr (SHARED_CUT) cut = fmin(cut, to_cut<R>(ld_cut(cutp)));
  res.cost = (result <= cut) ? result : INF;
  return res;
}

}  // namespace ekb
