// ek_kernels.cuh -- driver kernels around the two DP engines.
//
//   k_pairs     : one elastic distance per (pair, cutoff); replaces a loop of
//                 _speedups.run / engines.distance (engines.py:121-147)
//   k_triangle  : the all-pairs upper triangle, mirrored
//   k_nn        : 1-NN search with a per-query shared cutoff (search.py:81-160)
//   (k_subseq in ek_subseq.cuh, the 1-NN result pick k_nn_pick / k_nn_final in ek_misc.cu)
//
// All kernels are warp-per-pair and persistent (grid = SM count x resident
// blocks, work claimed with an atomic counter).  Series are staged into padded
// per-warp shared-memory buffers with coalesced loads; the 1-NN kernel stages a
// candidate lazily in 128-element chunks (most pairs are abandoned within the
// first few anti-diagonals) and prefetches the next candidate's first chunk into
// registers while the current pair runs.
#pragma once
#include "ek_common.cuh"
#include "ek_diag.cuh"
#include "ek_stripe.cuh"
#include "ek_lb.cuh"
#include "ek_tma.cuh"

namespace ekb {

#ifdef EKB_TRACE
// per-warp timeline of the last k_nn launch (debug builds only): start, end, DP ns, items, DPs
__device__ unsigned long long g_trace[8192 * 8];
#endif

// Engine codes: 0..2 diagonal P=4/8/16; 3..5 stripe S=4/8/16 (unbanded);
// 6 stripe S=16 banded; 7 stripe S=16 banded with row abandoning ("ea");
// 8..9 guarded diagonal P=8/16: a band narrower than the pair's own, valid as long as
// no cell <= cutoff reaches the band's edge lanes (else the pair is redone; see
// diag_pair's GUARD) -- EAPruned's pruned columns, skipped wholesale.
enum Engine : int {
  E_DIAG4 = 0, E_DIAG8 = 1, E_DIAG16 = 2,
  E_STR4 = 3, E_STR8 = 4, E_STR16 = 5,
  E_STRB16 = 6,
  E_STR16_EA = 7,
  E_GDIAG8 = 8, E_GDIAG16 = 9,
  E_DIAG2 = 10,  // narrow bands (<= 64 slots) in the all-pairs kernel: twice the lanes of P=4
  E_STRIP16 = 11, E_STRIPB16 = 12,  // long series: 512-column strips (unbanded / banded)
  E_STRIP16_EA = 13,                // long series, ea rows (full computation + row minima)
  E_DIAG4H = 14,  // all-pairs, bands <= 64 slots: P=4 on 16 lanes, two lockstep pairs per warp
  E_STR16H = 15,  // all-pairs, unbanded, <= 256 columns: S=16 on 16 lanes, two pairs per warp
  E_GDIAG4 = 16,  // guarded diagonal P=4 (+-62)
  E_COUNT = 17
};
__host__ __device__ constexpr int engine_W(int e) { return (e == E_DIAG4H || e == E_STR16H) ? 16 : 32; }
__host__ __device__ constexpr int engine_is_strip(int e) {
  return e == E_STRIP16 || e == E_STRIPB16 || e == E_STRIP16_EA;
}
constexpr int kStripDone = 0x40000000;  // strip engines' t_end for a completed pair

__host__ __device__ constexpr int engine_is_diag(int e) {
  return e <= E_DIAG16 || e == E_GDIAG8 || e == E_GDIAG16 || e == E_DIAG2 || e == E_DIAG4H || e == E_GDIAG4;
}
__host__ __device__ constexpr int engine_guarded(int e) { return e == E_GDIAG8 || e == E_GDIAG16 || e == E_GDIAG4; }
__host__ __device__ constexpr int engine_P(int e) {
  return e == E_DIAG2 ? 2 : (e == E_DIAG4 || e == E_DIAG4H || e == E_GDIAG4) ? 4 : (e == E_DIAG8 || e == E_GDIAG8) ? 8 : 16;
}
__host__ __device__ constexpr int engine_S(int e) { return e == E_STR4 ? 4 : e == E_STR8 ? 8 : 16; }
// elements an engine may read beyond either end of a staged series (stripe: rows stream past
// the ends by < 2 W)
__host__ __device__ constexpr int engine_pad(int e) {
  return engine_is_diag(e) ? diag_pad(engine_P(e)) : 40;  // stripe: rows stream past the ends by < 32
}
// per-warp shared-memory layout: [pad | X lmax | pad][pad | Y lmax | pad][|i-j| table]; the
// table is one-sided (lmax + 1 entries) for the strip engines, two-sided for the row-stripe
// engines: 2 (lmax + kTabPad) + 1 entries around d = i - j = 0 (stage_table2), so a lane
// addresses a row's weights from one per-row base with compile-time offsets
constexpr int kTabPad = 48;  // > 2 S - 1 + the clamp margin S (ek_stripe.cuh), S <= 16
__host__ __device__ constexpr int series_slot(int lmax, int pad) { return lmax + 2 * pad; }
__host__ __device__ constexpr int warp_stride(int lmax, int e) {  // (W = 16: two such blocks)
  return (32 / engine_W(e)) * (2 * series_slot(lmax, engine_pad(e)) +
                               (engine_is_diag(e) ? 0 : engine_is_strip(e) ? lmax + 1 : 2 * (lmax + kTabPad) + 1));
}

struct PairDesc {
  long long xoff, yoff;  // lines / cols offsets into the series buffer
  int nl, nc;            // nl >= nc (orientation done by the host, ties keep s on the rows)
  int w;                 // effective window (>= nl - nc, else the host already returned +inf)
  int pad_;
  double cut;
};

// ---- staging helpers -------------------------------------------------------

// pads: index -1 = the kind's predecessor of element 0, [-pad, -2] = 0.0, [n, n+pad) = +inf
// R = float (FP32 mode) stages the float64 inputs rounded to nearest.
template <int KIND, class R, int W = 32>
__device__ __forceinline__ void stage_pads(R* dst, int n, int pad, double first) {
  const int lane = threadIdx.x & (W - 1);
  for (int k = lane + 1; k <= pad; k += W) {
    dst[-k] = (k == 1) ? pad_before<KIND, R>((R)first) : (R)0.0;
    dst[n + k - 1] = rinf<R>();
  }
}

// W: the lanes staging the series (16: a half-warp pair, E_DIAG4H)
template <int KIND, class R, int W = 32>
__device__ __forceinline__ void stage_series(R* dst, const double* __restrict__ src, int n, int pad) {
  const int lane = threadIdx.x & (W - 1);
  int k = lane;
  for (; k + 7 * W < n; k += 8 * W) {  // eight loads in flight per lane before the stores
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(src + k + W * u);
#pragma unroll
    for (int u = 0; u < 8; ++u) dst[k + W * u] = (R)v[u];
  }
  for (; k < n; k += W) dst[k] = (R)__ldg(src + k);
  stage_pads<KIND, R, W>(dst, n, pad, __ldg(src));
}

template <int KIND, class R>
__device__ __forceinline__ void stage_table(R* tab, int len, const Params& prm) {
  const int lane = threadIdx.x & 31;
  if constexpr (KIND == K_WDTW) {
    for (int k = lane; k < len; k += 32) tab[k] = (k < prm.wt_len) ? (R)prm.wt[k] : (R)0.0;
  } else if constexpr (KIND == K_TWE) {
    for (int k = lane; k < len; k += 32) {
      R dij = (R)k;
      tab[k] = dmul((R)prm.nu, dadd(dij, dij));
    }
  }
}

// two-sided form: tab[k] = the entry for |d| = min(|k - half|, len - 1), k in [0, 2 half]
template <int KIND, class R, int W = 32>
__device__ __forceinline__ void stage_table2(R* tab, int len, int half, const Params& prm) {
  const int lane = threadIdx.x & (W - 1);
  if constexpr (KIND == K_WDTW) {
    for (int k = lane; k <= 2 * half; k += W) {
      const int d = min(abs(k - half), len - 1);
      tab[k] = (d < prm.wt_len) ? (R)prm.wt[d] : (R)0.0;
    }
  } else if constexpr (KIND == K_TWE) {
    for (int k = lane; k <= 2 * half; k += W) {
      R dij = (R)min(abs(k - half), len - 1);
      tab[k] = dmul((R)prm.nu, dadd(dij, dij));
    }
  }
}
// the engines' |i-j| table: staged for ENG, returns what run_engine / stripe_pair take
// (the strip engines: the one-sided table; the row-stripe engines: the entry of d = 0)
template <int KIND, int ENG, class R>
__device__ __forceinline__ const R* stage_engine_table(R* tab, int len, int lmax, const Params& prm) {
  if constexpr (engine_is_strip(ENG)) {
    stage_table<KIND>(tab, len, prm);
    return tab;
  } else {
    stage_table2<KIND, R, engine_W(ENG)>(tab, len, lmax + kTabPad, prm);
    return tab + lmax + kTabPad;
  }
}
template <int KIND, int ENG, class R>
__device__ __forceinline__ const R* engine_table(R* tab, int len, int lmax, const Params& prm) {
  if constexpr (engine_is_diag(ENG)) return tab;  // the diagonal engines keep per-diagonal registers
  else return stage_engine_table<KIND, ENG>(tab, len, lmax, prm);
}

// The band an engine actually runs: guarded engines narrow it to what 32 lanes of P
// slots hold (the widest w with diag_slots_needed <= 32P).
template <int ENG, int KIND = K_DTW>
__device__ __forceinline__ int engine_band(int nl, int nc, int w) {
  if constexpr (engine_guarded(ENG)) {
    constexpr int P = engine_P(ENG);
    int wg = min(w, 16 * P - 2);
    while (wg > 0 && diag_slots_needed(nl, nc, wg) > 32 * P) --wg;
    // MSM / TWE: the band whose two virtual diagonals both fall in slot 0 of their lanes
    // (diag_pair's VIRT0: wg + 1 a multiple of P / 2), so only slot 0 is ever masked
    if constexpr (KIND == K_MSM || KIND == K_TWE)
      while (wg > 0 && (wg + 1) % (P / 2) != 0) --wg;
    return wg;
  } else {
    return w;
  }
}

template <int KIND, int MODE, int ENG, bool SHARED_CUT, class XAcc, class YAcc, class Loader>
__device__ __forceinline__ void run_engine(const XAcc& X, int nl, const YAcc& Y, int nc, int w, double cut,
                                           const unsigned long long* cutp, const real_t<MODE>* tab, int tablen,
                                           const Params& prm, Loader& ld, double& cost, int& tend) {
  if constexpr (engine_guarded(ENG)) {
    // the widest band that fits 32 lanes of P slots; guard the sides it narrows
    constexpr int P = engine_P(ENG);
    const int wg = engine_band<ENG, KIND>(nl, nc, w);
    const int dlo_t = max(-w, 1 - nc), dhi_t = min(w, nl - 1);
    const int dlo_g = max(-wg, 1 - nc), dhi_g = min(wg, nl - 1);
    const int dbase = (dlo_g - 1) & ~1;
    // MSM / TWE run the slot-0-masked form only: its alignment holds whenever the series are
    // longer than the band (what a guarded engine is chosen for); anything else is redone
    constexpr bool V0 = (KIND == K_MSM || KIND == K_TWE);
    const bool aligned = !V0 || (wg > 0 && dlo_g - 1 == dbase && (dhi_g + 1 - dbase) % P == 0);
    if (wg < nl - nc || !aligned) {  // the final cell would fall outside: redo with the full engine
      cost = __longlong_as_double(0x7ff8000000000000LL);
      tend = -1;
      return;
    }
    const unsigned guard = (dlo_g > dlo_t ? 1u : 0u) | (dhi_g < dhi_t ? 1u << ((dhi_g - dbase) / P) : 0u);
    DiagResult r = diag_pair<KIND, MODE, P, SHARED_CUT, true, V0>(X, nl, Y, nc, wg, cut, cutp, prm, ld, guard);
    cost = r.cost;
    tend = r.t_end;
    if (r.ovf) {
      cost = __longlong_as_double(0x7ff8000000000000LL);
      tend = -1;
    }
  } else if constexpr (engine_is_diag(ENG)) {
    constexpr int P = engine_P(ENG);
    DiagResult r;
    if constexpr (KIND == K_DTW || KIND == K_CDTW || KIND == K_WDTW) {
      // both virtual diagonals in slot 0 of their lanes: only slot 0 needs the band offset
      const int dlo = max(-w, 1 - nc), dhi = min(w, nl - 1), dbase = (dlo - 1) & ~1;
      if (dlo - 1 == dbase && (dhi + 1 - dbase) % P == 0)
        r = diag_pair<KIND, MODE, P, SHARED_CUT, false, true, engine_W(ENG)>(X, nl, Y, nc, w, cut, cutp, prm, ld);
      else
        r = diag_pair<KIND, MODE, P, SHARED_CUT, false, false, engine_W(ENG)>(X, nl, Y, nc, w, cut, cutp, prm, ld);
    } else {
      r = diag_pair<KIND, MODE, P, SHARED_CUT, false, false, engine_W(ENG)>(X, nl, Y, nc, w, cut, cutp, prm, ld);
    }
    cost = r.cost;
    tend = r.t_end;
  } else if constexpr (engine_is_strip(ENG)) {
    real_t<MODE>* sb = (real_t<MODE>*)prm.strip_buf +
                       (size_t)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 3 * prm.strip_stride;
    StripeResult r = strip_pair<KIND, MODE, ENG != E_STRIP16, SHARED_CUT, ENG == E_STRIP16_EA>(
        X, nl, Y, nc, w, cut, cutp, tab, tablen, prm, sb, sb + prm.strip_stride, sb + 2 * prm.strip_stride);
    cost = r.cost;
    tend = (r.cost < EKB_INF) ? kStripDone : r.t_end;  // warp_cells: the band, or steps x 1024 cells
  } else {
    constexpr bool BANDED = ENG == E_STRB16 || ENG == E_STR16_EA;
    constexpr bool EA = ENG == E_STR16_EA;
    StripeResult r = stripe_pair<KIND, MODE, engine_S(ENG), BANDED, SHARED_CUT, EA, XAcc, YAcc, NoRec, engine_W(ENG)>(
        X, nl, Y, nc, w, cut, cutp,
                                                                                     tab, tablen, prm);
    cost = r.cost;
    tend = r.t_end;
  }
}

// Band cells an engine evaluated before it stopped at t_end (warp-parallel; every
// lane returns the total): the diagonal engine evaluates each band cell with
// i + j <= t_end; the stripe engine (two rows per step) evaluates row i of lane l
// while r0 + 2(t_end-1-l) + 1 >= i.
template <int ENG>
__device__ __forceinline__ int warp_cells(int nl, int nc, int w, int tend, int r0) {
  const int lane = threadIdx.x & 31;
  constexpr bool DIAG = engine_is_diag(ENG);
  constexpr int S = engine_S(ENG);
  if constexpr (engine_is_strip(ENG)) {  // whole band when completed, else ~1024 cells per step
    int c = 0;
    for (int i = 1 + lane; i <= nl; i += 32) c += max(0, min(nc, i + w) - max(1, i - w) + 1);
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
    return tend >= kStripDone ? c : min(c, tend * 1024);
  }
  const int imax = DIAG ? min(nl, tend - 1) : min(nl, r0 + 2 * tend - 1);
  int c = 0;
  for (int i = 1 + lane; i <= imax; i += 32) {
    const int jlo = max(1, i - w);
    int jhi = min(nc, i + w);
    jhi = DIAG ? min(jhi, tend - i) : min(jhi, ((r0 + 2 * tend - 1 - i) / 2 + 1) * S);
    c += max(0, jhi - jlo + 1);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
  return c;
}

// ---- generic pair list ------------------------------------------------------

template <int KIND, int MODE, int ENG>
__global__ void __launch_bounds__(128) k_pairs(const double* __restrict__ series, const PairDesc* __restrict__ pairs,
                                               int npairs, int lmax, Params prm, double* __restrict__ out_cost,
                                               int* __restrict__ out_tend) {
  extern __shared__ double smem[];
  constexpr int PAD = engine_pad(ENG);
  const int wib = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  using R = real_t<MODE>;
  R* X = (R*)smem + wib * warp_stride(lmax, ENG) + PAD;
  R* Y = X + series_slot(lmax, PAD);
  R* tab = Y - PAD + series_slot(lmax, PAD);
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  NoLoader ld;
  for (int pid = blockIdx.x * (blockDim.x >> 5) + wib; pid < npairs; pid += nwarps) {
    const PairDesc pd = pairs[pid];
    const Params pp = pair_params(prm, max(pd.nl, pd.nc));
    __syncwarp();
    stage_series<KIND>(X, series + pd.xoff, pd.nl, PAD);
    stage_series<KIND>(Y, series + pd.yoff, pd.nc, PAD);
    const int tablen = max(pd.nl, pd.nc) + 1;
    const R* tabe = engine_table<KIND, ENG>(tab, tablen, lmax, pp);
    __syncwarp();
    double cost;
    int tend;
    run_engine<KIND, MODE, ENG, false>(SmemSeriesT<R>{X, pd.nl}, pd.nl, SmemSeriesT<R>{Y, pd.nc}, pd.nc, pd.w, pd.cut,
                                       nullptr, tabe, tablen, pp, ld, cost, tend);
    const int cells = warp_cells<ENG>(pd.nl, pd.nc, pd.w, tend, KIND == K_ERP ? 0 : 1);
    if (lane == 0) {
      out_cost[pid] = cost;
      out_tend[pid] = cells;
    }
  }
}

// ---- all-pairs upper triangle ---------------------------------------------------
// pair index p in [0, n(n-1)/2) -> (i, j), i < j; D[i][j] = D[j][i] = distance(X_i, X_j).

__device__ __forceinline__ void tri_index(long long p, int n, int& i, int& j) {
  // row i holds n-1-i pairs; solve the largest i with i*(2n-i-1)/2 <= p
  double nn = (double)n;
  double disc = (2.0 * nn - 1.0) * (2.0 * nn - 1.0) - 8.0 * (double)p;
  int ii = (int)floor(((2.0 * nn - 1.0) - sqrt(disc)) * 0.5);
  ii = max(0, min(ii, n - 2));
  auto start = [&](long long r) { return r * (2LL * n - r - 1) / 2; };
  while (ii > 0 && start(ii) > p) --ii;
  while (ii < n - 2 && start(ii + 1) <= p) ++ii;
  i = ii;
  j = (int)(p - start(ii)) + ii + 1;
}

template <int KIND, int MODE, int ENG>
__global__ void __launch_bounds__(128) k_triangle(const double* __restrict__ series, const long long* __restrict__ off,
                                                  const int* __restrict__ len, int n, int win, int lmax, Params prm,
                                                  double* __restrict__ D, long long plo, long long phi,
                                                  double* __restrict__ Dvec,
                                                  unsigned long long* __restrict__ cells_total,
                                                  int* __restrict__ counter) {
  // pairs [plo, phi) of the upper triangle (row-major, np.triu_indices order); Dvec != null
  // writes cost p to Dvec[p - plo] (a rank's shard, ek_pairwise_range), else both cells of D
  extern __shared__ double smem[];
  constexpr int PAD = engine_pad(ENG);
  const int wib = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  using R = real_t<MODE>;
  // prm.shared_tab (all series of length lmax): the warps' slots hold only the series, and
  // one two-sided |i-j| table after them serves the whole block
  constexpr bool TABLED = (KIND == K_WDTW || KIND == K_TWE) && !engine_is_diag(ENG) && !engine_is_strip(ENG);
  const bool shtab = TABLED && prm.shared_tab != 0;
  const int wst = shtab ? (32 / engine_W(ENG)) * 2 * series_slot(lmax, PAD) : warp_stride(lmax, ENG);
  R* X = (R*)smem + wib * wst + PAD;
  R* Y = X + series_slot(lmax, PAD);
  R* tab = Y - PAD + series_slot(lmax, PAD);
  const R* btab = (R*)smem + (blockDim.x >> 5) * wst + lmax + kTabPad;  // its d = 0 entry
  if (shtab) {
    R* bt = (R*)smem + (blockDim.x >> 5) * wst;
    const Params pp = pair_params(prm, lmax);
    const int half = lmax + kTabPad;
    for (int k = threadIdx.x; k <= 2 * half; k += blockDim.x) {
      const int d = min(abs(k - half), lmax);
      if constexpr (KIND == K_WDTW) {
        bt[k] = (d < pp.wt_len) ? (R)pp.wt[d] : (R)0.0;
      } else {
        const R dij = (R)d;
        bt[k] = dmul((R)pp.nu, dadd(dij, dij));
      }
    }
    __syncthreads();
  }
  const long long npairs = phi;
  NoLoader ld;
  unsigned long long my_cells = 0;
  if constexpr (engine_W(ENG) == 16) {
    // two pairs per claim, one per half-warp, in lockstep when their shapes match; a pair
    // of different shapes runs in two passes with both halves on the same pair
    const int half = (threadIdx.x >> 4) & 1, hl = threadIdx.x & 15;
    // each half: [X][Y][|i-j| table (unless shared)]; equal lengths on the diagonal engine:
    // compact pads (Params.compact_pad), no table
    const bool cpad = engine_is_diag(ENG) && prm.compact_pad > 0;
    const int pad = cpad ? prm.compact_pad : PAD;
    const int hst = cpad ? 2 * series_slot(lmax, pad) : wst / 2;
    R* Xh = cpad ? (R*)smem + (wib * 2 + half) * hst + pad : X + half * hst;
    R* Yh = Xh + series_slot(lmax, pad);
    R* tabh = Yh - pad + series_slot(lmax, pad);
    for (;;) {
      long long p = 0;
      if (lane == 0) p = plo + (long long)atomicAdd((unsigned long long*)counter, 2ULL);
      p = __shfl_sync(FULL, p, 0);
      if (p >= npairs) break;
      int pa[2], pb[2], ps[2], pt[2];
      const int np = p + 1 < npairs ? 2 : 1;
      for (int k = 0; k < np; ++k) {
        tri_index(p + k, n, pa[k], pb[k]);
        ps[k] = pa[k];  // make_recurrence orientation (ties keep a on the rows)
        pt[k] = pb[k];
        if (len[pb[k]] > len[pa[k]]) {
          ps[k] = pb[k];
          pt[k] = pa[k];
        }
      }
      const bool same = np == 2 && len[ps[0]] == len[ps[1]] && len[pt[0]] == len[pt[1]];
      for (int pass = 0; pass < (same ? 1 : np); ++pass) {
        const int k = same ? half : pass;  // this half's pair
        const int s = ps[k], t = pt[k];
        const int nl = len[s], nc = len[t];
        const int w = win < 0 ? nl : win;
        double cost = EKB_INF;
        int tend = 0;
        if (w >= nl - nc) {  // the same for both halves (same shape)
          const Params pp = pair_params(prm, nl);
          __syncwarp();
          stage_series<KIND, R, 16>(Xh, series + off[s], nl, pad);
          stage_series<KIND, R, 16>(Yh, series + off[t], nc, pad);
          const int tablen = max(nl, nc) + 1;
          const R* tabe = shtab ? btab : engine_table<KIND, ENG>(tabh, tablen, lmax, pp);
          __syncwarp();
          run_engine<KIND, MODE, ENG, false>(SmemSeriesT<R>{Xh, nl}, nl, SmemSeriesT<R>{Yh, nc}, nc, w, EKB_INF,
                                             nullptr, tabe, tablen, pp, ld, cost, tend);
          // nothing abandons here (no cutoff): the whole band of this shape, summed over the
          // warp (x2 when both halves ran a pair of it)
          my_cells += (unsigned long long)warp_cells<E_DIAG4>(nl, nc, w, nl + nc, KIND == K_ERP ? 0 : 1) *
                      (same ? 2u : 1u);
        }
        if (hl == 0 && (same || half == 0)) {
          if (Dvec) {
            Dvec[p + k - plo] = cost;
          } else {
            D[(long long)pa[k] * n + pb[k]] = cost;
            D[(long long)pb[k] * n + pa[k]] = cost;
          }
        }
      }
    }
    if (lane == 0 && cells_total) atomicAdd(cells_total, my_cells);
    return;
  }
  for (;;) {
    long long p = 0;
    if (lane == 0) p = plo + (long long)atomicAdd((unsigned long long*)counter, 1ULL);
    p = __shfl_sync(FULL, p, 0);
    if (p >= npairs) break;
    int a, b;
    tri_index(p, n, a, b);
    // make_recurrence orientation: lines = longer, ties keep the first argument (a) on the rows
    int s = a, t = b;
    if (len[b] > len[a]) { s = b; t = a; }
    const int nl = len[s], nc = len[t];
    const int w = win < 0 ? nl : win;
    double cost = EKB_INF;
    int tend = 0;
    if (w >= nl - nc) {
      const Params pp = pair_params(prm, nl);
      __syncwarp();
      stage_series<KIND>(X, series + off[s], nl, PAD);
      stage_series<KIND>(Y, series + off[t], nc, PAD);
      const int tablen = max(nl, nc) + 1;
      const R* tabe = shtab ? btab : engine_table<KIND, ENG>(tab, tablen, lmax, pp);
      __syncwarp();
      run_engine<KIND, MODE, ENG, false>(SmemSeriesT<R>{X, nl}, nl, SmemSeriesT<R>{Y, nc}, nc, w, EKB_INF, nullptr, tabe,
                                         tablen, pp, ld, cost, tend);
      my_cells += (unsigned long long)warp_cells<ENG>(nl, nc, w, tend, KIND == K_ERP ? 0 : 1);
    }
    if (lane == 0) {
      if (Dvec) {
        Dvec[p - plo] = cost;
      } else {
        D[(long long)a * n + b] = cost;
        D[(long long)b * n + a] = cost;
      }
    }
  }
  if (lane == 0 && cells_total) atomicAdd(cells_total, my_cells);
}

// ---- 1-NN with a shared per-query cutoff -----------------------------------------

// 1-NN results, accumulated on the fly instead of a per-pair Q x C matrix: per query the
// least finite cost (IEEE image: values are >= +0, so the bits order as integers), the
// count of finite results and the evaluated cells; the finite results themselves go to an
// append-only list, from which the lowest index among equal minima is picked after the
// search (k_nn_pick / k_nn_final, ek_misc.cu).  Every result with cost <= the final cutoff
// is exact, so that is nn_search's answer (strict "<", lowest index) whatever the schedule.
struct NNAcc {
  unsigned long long* best;  // [nq]
  long long* cells;          // [nq]
  int* computed;             // [nq]
  int* idx;                  // [nq] lowest index of the least cost (k_nn_pick)
  long long* fin;            // [cap] q << 32 | c of each finite result
  double* fin_cost;          // [cap]
  int* fin_count;
};
// lane 0: one pair's result
__device__ __forceinline__ void nn_publish(const NNAcc& a, int q, int c, double cost) {
  if (cost < EKB_INF) {
    atomicMin(a.best + q, (unsigned long long)__double_as_longlong(cost));
    const int k = atomicAdd(a.fin_count, 1);
    a.fin[k] = ((long long)q << 32) | (unsigned)c;
    a.fin_cost[k] = cost;
    atomicAdd(a.computed + q, 1);
  }
}

constexpr int kChunk = 128;  // candidate staging granule (4 doubles per lane)
constexpr int kNnCounters = 8;  // k_nn work counters (64-bit each)

// Lazily staged candidate; the first chunk arrives prefetched.
template <class R>
struct LazyCand {
  R* buf;
  const double* src;
  int n, loaded;
  bool is_x;  // backs the lines series (else the cols series)
  __device__ __forceinline__ void load_to(int need) {
    need = min(need, n);
    const int lane = threadIdx.x & 31;
    while (loaded < need) {
      const int base = loaded;
#pragma unroll
      for (int u = 0; u < kChunk / 32; ++u) {
        const int k = base + u * 32 + lane;
        if (k < n) buf[k] = (R)__ldg(src + k);
      }
      loaded = min(base + kChunk, n);
    }
    __syncwarp();
  }
  // diag engine protocol (see ek_diag.cuh): data needed by the double step at t
  // and the window slide after it: lines up to (t+dhi+3)/2+1+H, cols up to (t+3-dlo)/2+2.
  __device__ __forceinline__ int next_t(int dlo, int dhi, int H) const {
    if (loaded >= n) return 0x7fffffff;
    return is_x ? 2 * (loaded - 2 - H) - dhi - 5 : 2 * (loaded - 3) + dlo - 5;
  }
  __device__ __forceinline__ void ensure(int t, int dlo, int dhi, int H) {
    const int ahead = t + 2 * kChunk;  // stage one chunk ahead of the wavefront
    load_to(is_x ? (ahead + dhi + 3) / 2 + 2 + H : (ahead + 3 - dlo) / 2 + 3);
  }
};

#ifndef EKB_NN_DTW_MINB
#define EKB_NN_DTW_MINB 5  // measured: 96 registers without spills, C2 phase B -1%
#endif
// min resident blocks for the dtw/cdtw diagonal 1-NN kernels (0: the compiler's choice)
#ifndef EKB_NN_GUARD_MINB
#define EKB_NN_GUARD_MINB 3  // MSM / TWE guarded P=4 band (C4 phase B): 3 blocks (TWE -3%, MSM without spills)
#endif
// (the FP32 kernels keep the compiler's choice: forcing 3 blocks there let them grow past
// 4 blocks' worth of registers, C4 FP32 TWE 23.8 -> 27.0 ms)
__host__ __device__ constexpr int nn_minb(int kind, int eng, int mode) {
  return (kind == K_DTW && eng == E_DIAG4) ? EKB_NN_DTW_MINB
         : ((kind == K_MSM || kind == K_TWE) && eng == E_GDIAG4 && (mode & M_F32) == 0) ? EKB_NN_GUARD_MINB : 0;
}

template <int KIND, int MODE, int ENG>
__global__ void __launch_bounds__(128, nn_minb(KIND, ENG, MODE)) k_nn(const double* __restrict__ Q, const long long* __restrict__ qoff,
                                            const int* __restrict__ qlen, int nq, const double* __restrict__ C,
                                            const long long* __restrict__ coff, const int* __restrict__ clen,
                                            int ncand, const int* __restrict__ order, int rank_lo, int rank_mid,
                                            int rank_hi, int K1, int K2, int win, int lmax, Params prm, int share,
                                            unsigned long long* cutbits, NNAcc acc, int* __restrict__ counter,
                                            const float* __restrict__ skeys, const float2* __restrict__ envq,
                                            int2* __restrict__ ovf_list, int* __restrict__ ovf_count,
                                            int* __restrict__ qstop) {
  extern __shared__ double smem[];
  constexpr int PAD = engine_pad(ENG);
  constexpr int PF = kChunk / 32;
  const int wib = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  using R = real_t<MODE>;
  // prm.bulk: a second candidate slot after the warp's usual layout (diagonal engines have
  // no table, so both slots stay 16-byte aligned), filled by bulk copies one pair ahead
  const bool bulk = (MODE & M_F32) == 0 && engine_is_diag(ENG) && skeys == nullptr && prm.bulk != 0;
  const int wstride = warp_stride(lmax, ENG) + (prm.bulk ? series_slot(lmax, PAD) : 0);
  R* QB = (R*)smem + wib * wstride + PAD;
  R* CB = QB + series_slot(lmax, PAD);
  R* tab = CB - PAD + series_slot(lmax, PAD);
  R* const CB2 = (R*)smem + wib * wstride + warp_stride(lmax, ENG) + PAD;
  __shared__ unsigned long long nn_bar[4][2];  // per warp (blockDim <= 128): one mbarrier per slot
  unsigned bphase = 0;                          // bit b: parity of slot b's next completion
  int bcur = 0;                                 // slot of the pair about to run
  if (bulk) {
    if (lane == 0) {
      mbar_init(&nn_bar[wib][0], 1);
      mbar_init(&nn_bar[wib][1], 1);
      mbar_init_fence();
    }
    __syncwarp();
  }
  // two segments in one launch: ranks [rank_lo, rank_mid) in items of K1, then
  // [rank_mid, rank_hi) in items of K2, each round-major over the queries, so warps
  // that finish the first segment's tail start on the second at once.  Only the
  // dtw/cdtw LB path uses a second segment; the other kinds keep the one-segment item
  // logic (rank_mid == rank_hi), whose code they are register-tuned on.
  constexpr bool TWO_SEG = (KIND == K_DTW);
  const long long items1 = (long long)((rank_mid - rank_lo + K1 - 1) / K1) * nq;
  const long long nitems = TWO_SEG ? items1 + (long long)((rank_hi - rank_mid + K2 - 1) / K2) * nq : items1;
  // LB path (dtw/cdtw, equal lengths): skeys[q * ncand + rank] = LB_Keogh(q, env(c)) of the
  // rank's candidate, rounded down (k_lb_matrix; the ranks are ordered by it).  Pairs whose
  // key exceeds the cutoff are never visited (their outputs are prefilled: +inf, 0 cells).
  const bool use_lb = skeys != nullptr;
  int staged_q = -1, cb_len = -1;
  unsigned long long* const ctr = (unsigned long long*)counter;
  // Items are claimed from kNnCounters interleaved counters (item = local * kNnCounters
  // + k), starting at the warp's own: one counter would serialise ~10^5..10^6 claims at
  // L2.  (Claiming one item ahead measured slower: a claimed item waits behind the
  // current one's DPs, which unbalances the tail.)
  int ck = (int)((blockIdx.x * (blockDim.x >> 5) + wib) % kNnCounters), ctr_left = kNnCounters;
  // LB path: the ranks are sorted by the keys' top 16 bits (k_rank_radix; truncation rounds
  // a positive float down), so once a rank's truncated key exceeds the threshold of the
  // query's cutoff, every later rank fails its key test too: qstop[q] is the least such
  // rank, items at or past it are skipped unread, and qstop[nq] counts the queries that
  // have one -- when it reaches nq no item can hold a pair to visit and the warps leave
  // without claiming the rest (the cutoff only decreases, so a stop stays valid).
  const bool stops = use_lb && qstop != nullptr;
  // Leaving once every query has a stop is sound only when all the items of a query come
  // from one counter, claimed in increasing rank: item it is on counter it % kNnCounters, and
  // it = (segment base) + r nq + q, so that needs nq % kNnCounters == 0.  Otherwise an item
  // below a stop could still sit unclaimed on a lagging counter; the per-item test remains.
  const bool stop_exit = stops && nq % kNnCounters == 0;
#ifdef EKB_TRACE
  unsigned long long tr_t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_t0));
  unsigned long long tr_dp = 0, tr_items = 0, tr_dps = 0;
#endif
  for (;;) {
    long long it = -1;
    if (lane == 0 && !(stop_exit && *(volatile int*)(qstop + nq) >= nq)) {
      while (ctr_left > 0) {
        const long long cand = (long long)atomicAdd(ctr + ck, 1ULL) * kNnCounters + ck;
        if (cand < nitems) {
          it = cand;
          break;
        }
        ck = (ck + 1) % kNnCounters;  // counter ck is exhausted: the next one
        --ctr_left;
      }
    }
    it = __shfl_sync(FULL, it, 0);
    if (it < 0) break;
#ifdef EKB_TRACE
    ++tr_items;
#endif
    const bool first_seg = !TWO_SEG || it < items1;
    const long long is = first_seg ? it : it - items1;
    const int q = (int)(is % nq);
    const int r = (int)(is / nq);
    const int lq = qlen[q];
    const int K = first_seg ? K1 : K2;
    const int k_lo = (first_seg ? rank_lo : rank_mid) + r * K;
    const int k_hi = min(k_lo + K, first_seg ? rank_mid : rank_hi);
    const int cnt = k_hi - k_lo;
    double cut = ld_cut(cutbits + q);
    // this item's pairs to visit: all of them, or (LB path) those whose key passes the cutoff
    unsigned todo = cnt >= 32 ? FULL : (1u << cnt) - 1u;
    float key = 0.f;
    double pf[PF];
    if (use_lb) {
      if (stops && __shfl_sync(FULL, lane == 0 ? *(volatile int*)(qstop + q) : 0, 0) <= k_lo) continue;
      key = lane < cnt ? skeys[(long long)q * ncand + k_lo + lane] : 0.f;
      const double thr = lb_threshold<MODE>(cut, lq);
      todo = __ballot_sync(FULL, lane < cnt && (double)key <= thr);
      if (stops) {
        const float kt = __uint_as_float(__float_as_uint(key) & 0xffff0000u);  // the sort key, <= key
        const unsigned past = __ballot_sync(FULL, lane < cnt && (double)kt > thr);
        if (past && lane == 0) {
          const int r0 = k_lo + __ffs(past) - 1;
          if (atomicMin(qstop + q, r0) >= ncand) atomicAdd(qstop + nq, 1);
        }
      }
      if (!todo) continue;  // nothing to visit: the query is not even staged
    }
    // this item's candidates and their metadata, one per lane (K <= 32)
    const int ord = lane < cnt ? order[(long long)q * ncand + k_lo + lane] : 0;
#ifdef EKB_BOUNDS
    if (ord < 0 || ord >= ncand || q < 0 || q >= nq || k_lo < 0 || k_hi > ncand || cnt > 32) {
      printf("k_nn bad item q=%d ord=%d k_lo=%d k_hi=%d cnt=%d it=%lld\n", q, ord, k_lo, k_hi, cnt, it);
      __trap();
    }
#endif
    const int olen = clen[ord];
    const long long ooff = coff[ord];
#ifdef EKB_BOUNDS
    if (olen < 0 || olen > lmax || qlen[q] > lmax) {
      printf("k_nn bad len olen=%d lq=%d lmax=%d\n", olen, qlen[q], lmax);
      __trap();
    }
#endif
    if (q != staged_q) {
      __syncwarp();
      stage_series<KIND>(QB, Q + qoff[q], lq, PAD);
      staged_q = q;
    }
    if (bulk) {  // the first pair's candidate, whole, into the current slot
      const double* s = C + __shfl_sync(FULL, ooff, 0);
      const int lc = __shfl_sync(FULL, olen, 0);
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async();
        bulk_g2s(bcur ? CB2 : CB, s, 8u * (unsigned)lc, &nn_bar[wib][bcur]);
      }
    } else if (!use_lb) {  // the first pair's first data chunk
      const double* s = C + __shfl_sync(FULL, ooff, 0);
      const int lc = __shfl_sync(FULL, olen, 0);
#pragma unroll
      for (int u = 0; u < PF; ++u) pf[u] = (u * 32 + lane < lc) ? __ldg(s + u * 32 + lane) : 0.0;
    }
    __syncwarp();
    long long icells = 0;  // this item's evaluated cells (one atomic per item)
    while (todo) {
      const int i = __ffs(todo) - 1;
      todo &= todo - 1;
      const int c = __shfl_sync(FULL, ord, i);
      const int lc = __shfl_sync(FULL, olen, i);
      const double* csrc = C + __shfl_sync(FULL, ooff, i);
      // orientation (kernels.py:168-171): query is s, candidate is t
      const bool q_rows = lq >= lc;
      const int nl = q_rows ? lq : lc, nc = q_rows ? lc : lq;
      const int w = win < 0 ? nl : win;
      bool evaluate = w >= nl - nc;
      int staged = min(kChunk, lc);  // candidate elements already in CB
      R* CBc = CB;                    // the slot holding this pair's candidate
      if (bulk) {
        // this pair's copy has landed: request the next pair's into the other slot (its last
        // readers finished with the previous pair: __syncwarp, then the proxy fence), and
        // write the pads around this one
        mbar_wait(&nn_bar[wib][bcur], (bphase >> bcur) & 1u);
        bphase ^= 1u << bcur;
        CBc = bcur ? CB2 : CB;
        const double* ns = C + __shfl_sync(FULL, ooff, min(i + 1, 31));
        const int nl2 = __shfl_sync(FULL, olen, min(i + 1, 31));
        __syncwarp();
        if (i + 1 < cnt && lane == 0) {
          fence_proxy_async();
          bulk_g2s(bcur ? CB : CB2, ns, 8u * (unsigned)nl2, &nn_bar[wib][bcur ^ 1]);
        }
        stage_pads<KIND>(CBc, lc, PAD, (double)CBc[0]);
        staged = lc;
        bcur ^= 1;
        __syncwarp();
      } else if (use_lb) {
        // the key against the current (tighter) cutoff, then the reverse bound
        const double thr = lb_threshold<MODE>(cut, nl);
        evaluate = evaluate && (double)__shfl_sync(FULL, key, i) <= thr;
        if (evaluate) {  // survivor: stage the whole candidate, then the reverse bound
          __syncwarp();
          stage_series<KIND>(CB, csrc, lc, PAD);
          cb_len = lc;
          staged = lc;
          __syncwarp();
          evaluate = warp_lb_reverse<MODE>(CB, envq + (long long)q * lmax, lc, lb_scale(thr));
        }
      } else {
        __syncwarp();
#pragma unroll
        for (int u = 0; u < PF; ++u)
          if (u * 32 + lane < lc) CB[u * 32 + lane] = (R)pf[u];
        const double first = __shfl_sync(FULL, pf[0], 0);
        if (lc != cb_len || KIND == K_MSM) {
          stage_pads<KIND>(CB, lc, PAD, first);
          cb_len = lc;
        }
        if (i + 1 < cnt) {  // prefetch the next candidate's first chunk (todo holds every pair)
          const double* s = C + __shfl_sync(FULL, ooff, i + 1);
          const int ln = __shfl_sync(FULL, olen, i + 1);
#pragma unroll
          for (int u = 0; u < PF; ++u) pf[u] = (u * 32 + lane < ln) ? __ldg(s + u * 32 + lane) : 0.0;
        }
      }
      double cost = EKB_INF;
      int tend = 0;
      if (evaluate) {
        const Params pp = pair_params(prm, nl);
        LazyCand<R> ld{CBc, csrc, lc, staged, !q_rows};
        const int tablen = max(nl, nc) + 1;
        if constexpr (!engine_is_diag(ENG)) ld.load_to(lc);  // the stripe engine reads all columns up front
        const R* tabe = engine_table<KIND, ENG>(tab, tablen, lmax, pp);
        __syncwarp();
        const SmemSeriesT<R> X{q_rows ? QB : CBc, nl};
        const SmemSeriesT<R> Y{q_rows ? CBc : QB, nc};
#ifdef EKB_TRACE
        unsigned long long tr_a, tr_b;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_a));
#endif
        run_engine<KIND, MODE, ENG, true>(X, nl, Y, nc, w, cut, cutbits + q, tabe, tablen, pp, ld, cost, tend);
#ifdef EKB_TRACE
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_b));
        tr_dp += tr_b - tr_a;
        ++tr_dps;
#endif
        if (share && lane == 0 && cost < EKB_INF) {
          // values are >= 0 (or +inf), so IEEE bits order as unsigned integers
          atomicMin(cutbits + q, (unsigned long long)__double_as_longlong(cost));
        }
        if (share) cut = fmin(cut, fmin(cost, ld_cut(cutbits + q)));
      }
      const int cells = tend > 0 ? warp_cells<ENG>(nl, nc, engine_band<ENG, KIND>(nl, nc, w), tend, KIND == K_ERP ? 0 : 1) : 0;
      if (lane == 0) {
        if (tend < 0) {  // guarded band overflowed: the pair is redone by k_nn_fix
          ovf_list[atomicAdd(ovf_count, 1)] = make_int2(q, c);
          cost = EKB_INF;
        }
        nn_publish(acc, q, c, cost);
        icells += cells;
      }
    }
    if (lane == 0 && icells) atomicAdd((unsigned long long*)acc.cells + q, (unsigned long long)icells);
  }
#ifdef EKB_TRACE
  if (lane == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    const int gw = blockIdx.x * (blockDim.x >> 5) + wib;
    if (gw < 8192) {
      g_trace[gw * 8 + 0] = tr_t0;
      g_trace[gw * 8 + 1] = t1;
      g_trace[gw * 8 + 2] = tr_dp;
      g_trace[gw * 8 + 3] = tr_items;
      g_trace[gw * 8 + 4] = tr_dps;
    }
  }
#endif
}

// Redo of the pairs a guarded band gave up on (`list`, *count of them) with a wider engine
// and the query's shared cutoff: a wider guarded band, whose own overflows go to ovf_list /
// ovf_count for the next redo, or the full band.
template <int KIND, int MODE, int ENG>
__global__ void __launch_bounds__(128) k_nn_fix(const double* __restrict__ Q, const long long* __restrict__ qoff,
                                                const int* __restrict__ qlen, const double* __restrict__ C,
                                                const long long* __restrict__ coff, const int* __restrict__ clen,
                                                int ncand, const int2* __restrict__ list,
                                                const int* __restrict__ count, int win, int lmax, Params prm,
                                                unsigned long long* cutbits, NNAcc acc, int* __restrict__ counter,
                                                int2* __restrict__ ovf_list, int* __restrict__ ovf_count) {
  extern __shared__ double smem[];
  constexpr int PAD = engine_pad(ENG);
  const int wib = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  using R = real_t<MODE>;
  R* X = (R*)smem + wib * warp_stride(lmax, ENG) + PAD;
  R* Y = X + series_slot(lmax, PAD);
  R* tab = Y - PAD + series_slot(lmax, PAD);
  const int n = *count;
  NoLoader ld;
  for (;;) {
    int e = 0;
    if (lane == 0) e = atomicAdd(counter, 1);
    e = __shfl_sync(FULL, e, 0);
    if (e >= n) break;
    const int2 pc = list[e];
    const int q = pc.x, c = pc.y;
    const int lq = qlen[q], lc = clen[c];
    const bool q_rows = lq >= lc;  // orientation (kernels.py:168-171)
    const int nl = q_rows ? lq : lc, nc = q_rows ? lc : lq;
    const int w = win < 0 ? nl : win;
    const Params pp = pair_params(prm, nl);
    __syncwarp();
    stage_series<KIND>(X, q_rows ? Q + qoff[q] : C + coff[c], nl, PAD);
    stage_series<KIND>(Y, q_rows ? C + coff[c] : Q + qoff[q], nc, PAD);
    const int tablen = max(nl, nc) + 1;
    const R* tabe = engine_table<KIND, ENG>(tab, tablen, lmax, pp);
    __syncwarp();
    const double cut = ld_cut(cutbits + q);
    double cost;
    int tend;
    run_engine<KIND, MODE, ENG, true>(SmemSeriesT<R>{X, nl}, nl, SmemSeriesT<R>{Y, nc}, nc, w, cut, cutbits + q, tabe, tablen,
                                      pp, ld, cost, tend);
    const int cells = tend > 0 ? warp_cells<ENG>(nl, nc, engine_band<ENG, KIND>(nl, nc, w), tend, KIND == K_ERP ? 0 : 1) : 0;
    if (lane == 0) {
      if (tend < 0) {  // a guarded redo overflowed too: the next, wider engine takes it
        ovf_list[atomicAdd(ovf_count, 1)] = make_int2(q, c);
        cost = EKB_INF;
      }
      if (cost < EKB_INF) atomicMin(cutbits + q, (unsigned long long)__double_as_longlong(cost));
      nn_publish(acc, q, c, cost);
      if (cells) atomicAdd((unsigned long long*)acc.cells + q, (unsigned long long)cells);
    }
  }
}

}  // namespace ekb
