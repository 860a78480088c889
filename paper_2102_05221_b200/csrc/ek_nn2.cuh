// ek_nn2.cuh -- phase B of the 1-NN LB path (dtw/cdtw, equal lengths, a band of at most 128
// diagonal slots, e.g. C2's cdtw w=51 on 512 points: 105 slots): two pairs per warp.
//
// Each half-warp runs one (query, candidate) pair on the diagonal wavefront of ek_diag.cuh
// with P = 8 slots on 16 lanes (the 128 slots one pair has on 32 lanes x P = 4 in k_nn).
// Per double step a lane evaluates 8 cells instead of 4 for the same two 64-bit shuffles,
// two series loads, liveness vote and loop control, and its two half steps each hold four
// independent cell chains instead of two.
//
// The halves run in lockstep through blocks of U = 10 double steps (the period of the
// register rings, an even number so votes fall on odd steps).  A half whose pair abandons
// (four consecutive dead anti-diagonals, as in diag_pair) or reaches its last cell stops
// updating its result and idles to the block's end; between blocks every idle half
// publishes its result and is refilled with the next survivor, which starts at phase 0 of
// the rings.  Survivors come from the same work items as k_nn (query, rank range; the LB
// keys tested lane-parallel against the query's shared cutoff, the reverse bound
// warp-wide), claimed from kNnCounters interleaved counters with the per-query stop ranks.
//
// No staging: queries and candidates are read through L1 from padded copies in HBM
// (k_pad_series: 0.0 before a series, +inf after it, like the shared-memory pads of
// stage_series), so a refill costs no shared-memory traffic and the kernel's occupancy is
// set by registers alone.
//
// Exactness is diag_pair's: the same cells (cell<K_DTW, ...>, the VIRT0 band offsets), the
// same four-anti-diagonal abandoning argument per pair, the same final test r <= cutoff and
// atomicMin publication; the 1-NN pick is unchanged (k_nn_pick / k_nn_final).
#pragma once
#include "ek_kernels.cuh"

namespace ekb {

#ifdef EKB_TRACE
// long pairs of the last k_nn2 launch: (start ns, end ns, query, key / threshold * 1e6, rank-ordered claim index)
__device__ unsigned long long g_plog[32768 * 4];
__device__ unsigned int g_plog_n;
#endif

constexpr int kPadG = 96;  // elements of padding on each side of a padded series (>= 92, see below)

// dst[s * pitch + kPadG + k], k in [-kPadG, L + kPadG): the series (rounded to R), 0.0 before
// it (the DTW family's pad_before), +inf after it.  The engine reads indices in
// [-66, L + 88] for any band of <= 128 slots (t in [2, 2L + 2U + 2], windows H + U ahead).
template <class R>
__global__ void k_pad_series(const double* __restrict__ src, const long long* __restrict__ off, int n, int L,
                             int pitch, R* __restrict__ dst) {
  // grid (ceil(pitch / blockDim), n): one block per 256 elements of one padded series
  const int s = blockIdx.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x - kPadG;
  if (k >= L + kPadG) return;
  const double* p = src + off[s];
  dst[(long long)s * pitch + kPadG + k] = k < 0 ? (R)0.0 : k >= L ? rinf<R>() : (R)__ldg(p + k);
}

#ifndef EKB_NN2_MINB
#define EKB_NN2_MINB 4
#endif

template <int MODE, bool VIRT0>
__global__ void __launch_bounds__(128, EKB_NN2_MINB)
    k_nn2(const real_t<MODE>* __restrict__ QP, const real_t<MODE>* __restrict__ CP, int pitch, int L, int nq,
          int ncand, const int* __restrict__ order, int rank_lo, int rank_mid, int rank_hi, int K1, int K2, int w,
          unsigned long long* cutbits, NNAcc acc, int* __restrict__ qnext, unsigned long long* qdone,
          const float* __restrict__ skeys, const float2* __restrict__ envq, int lmax, int* __restrict__ qstop) {
  using R = real_t<MODE>;
  constexpr int P = 8, H = P / 2;
  constexpr int RX = H + 1, RY = H + 1;  // register rings (y keeps one spare slot: both rings have period 5)
  constexpr int U = 2 * RX;              // double steps per block
  const R INF = rinf<R>();
  const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  const unsigned hmask = 0xffffu << (16 * half);
  const int dlo = max(-w, 1 - L), dhi = min(w, L - 1);
  const int dbase = (dlo - 1) & ~1;
  const int d0 = dbase + hl * P;
  const int Tf = 2 * L;
  const int lf = (-dbase) / P, pf = (-dbase) % P;  // the final cell (L, L) is on diagonal 0
  const Params prm{};                              // (the DTW cell reads no parameters)
  DiagK<K_DTW, R> kk[VIRT0 ? 1 : P];
#pragma unroll
  for (int p = 0; p < (VIRT0 ? 1 : P); ++p) kk[p].off = (d0 + p >= dlo && d0 + p <= dhi) ? (R)0.0 : INF;
  SlotS<K_DTW, R> ss;

  // ---- this half's pair (every value is uniform within the half) ----
  R val[P], xw[RX], yw[RY];
#pragma unroll
  for (int p = 0; p < P; ++p) val[p] = INF;
#pragma unroll
  for (int k = 0; k < RX; ++k) xw[k] = yw[k] = (R)0.0;
  int t = 2, I0 = 0, J0 = 0;
  const R* xp = QP;
  const R* yp = CP;
  R cut = INF;
  int cut_hi = hi_word(cut);
  int pq = 0, pc = 0;
  bool run = false;  // the half is evaluating a pair
  int st = 0;        // 0: nothing to publish, 1: finished (res), 2: abandoned
  R res = INF;
  int tend = 0;
  bool alive = false;

  // ---- work source (warp-uniform): per-query item counters ----
  // Item j of query q covers ranks [rank_lo + j K1, +K1) for j < n1, then items of K2 up to
  // rank_hi.  A warp walks the queries round robin, claiming each one's next item from its
  // counter qnext[q]; a query is marked done in the bitmask qdone once an item starts at or
  // past its stop rank (the ranks are sorted by the truncated keys: every later item fails
  // its key test) or past rank_hi.  Every item below a query's stop is claimed by some warp,
  // because its counter only grows; the launch ends when every query is done.
  const int nw = (nq + 63) >> 6;
  const int n1 = (rank_mid - rank_lo + K1 - 1) / K1;
  const bool stops = qstop != nullptr;
  int qc = (int)(((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % nq);
  int it_q = 0, ord = 0;
  unsigned todo = 0;
  float key = 0.f;
  bool exhausted = false;
  auto mark_done = [&](int q) {
    if (lane == 0) atomicOr(qdone + (q >> 6), 1ull << (q & 63));
  };
  // the first query not done at or after `from` in circular order, or -1
  auto find_q = [&](int from) -> int {
    const int w0 = from >> 6;
    for (int g = 0; g <= nw; g += 32) {
      const int l = g + lane;  // word w0 + l; l == nw re-reads word w0 for the bits below `from`
      unsigned long long fb = 0;
      if (l <= nw) {
        const int wi = (w0 + l) % nw;
        unsigned long long bits;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(bits) : "l"(qdone + wi));
        fb = ~bits;
        if (wi == nw - 1 && (nq & 63)) fb &= (1ull << (nq & 63)) - 1;
        if (l == 0) fb &= ~0ull << (from & 63);
      }
      const unsigned hit = __ballot_sync(FULL, fb != 0);
      if (hit) {
        const int src = __ffs(hit) - 1;
        const unsigned long long f = __shfl_sync(FULL, fb, src);
        return ((w0 + g + src) % nw) * 64 + __ffsll((long long)f) - 1;
      }
    }
    return -1;
  };

#ifdef EKB_TRACE
  unsigned long long tr_ratio = 0, tr_pst = 0, tr_prat = 0;
#endif
  auto next_pair = [&](int& oq, int& oc) -> bool {
    for (;;) {
      while (todo) {
        const int i = __ffs(todo) - 1;
        todo &= todo - 1;
        const int c = __shfl_sync(FULL, ord, i);
        const float k = __shfl_sync(FULL, key, i);
        // the key against the query's current (tighter) cutoff, then the reverse bound
        const double thr = lb_threshold<MODE>(ld_cut(cutbits + it_q), L);
        if ((double)k > thr) continue;
        if (!warp_lb_reverse<MODE>(CP + (long long)c * pitch + kPadG, envq + (long long)it_q * lmax, L,
                                   lb_scale(thr)))
          continue;
#ifdef EKB_TRACE
        tr_ratio = (unsigned long long)(1e6 * (double)k / thr);
#endif
        oq = it_q;
        oc = c;
        return true;
      }
      if (exhausted) return false;
      const int q = find_q(qc);
      if (q < 0) {
        exhausted = true;
        return false;
      }
      int j = 0;
      if (lane == 0) j = atomicAdd(qnext + q, 1);
      j = __shfl_sync(FULL, j, 0);
      qc = q + 1 == nq ? 0 : q + 1;  // round robin over the queries
      int k_lo, k_hi;
      if (j < n1) {
        k_lo = rank_lo + j * K1;
        k_hi = min(k_lo + K1, rank_mid);
      } else {
        k_lo = rank_mid + (j - n1) * K2;
        k_hi = min(k_lo + K2, rank_hi);
      }
      if (k_lo >= rank_hi) {
        mark_done(q);
        continue;
      }
      const int cnt = k_hi - k_lo;
      // the item's stop rank, cutoff, keys and candidates, loaded together
      int stop_q = 0;
      unsigned long long cbits = 0;
      if (lane == 0) {
        if (stops) stop_q = *(volatile int*)(qstop + q);
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(cbits) : "l"(cutbits + q));
      }
      key = lane < cnt ? skeys[(long long)q * ncand + k_lo + lane] : 0.f;
      ord = lane < cnt ? order[(long long)q * ncand + k_lo + lane] : 0;
      if (stops && __shfl_sync(FULL, stop_q, 0) <= k_lo) {
        mark_done(q);
        continue;
      }
      const double thr = lb_threshold<MODE>(bcast_cut(cbits), L);
      todo = __ballot_sync(FULL, lane < cnt && (double)key <= thr);
      if (stops) {  // the ranks are sorted by the keys' top 16 bits (see k_nn)
        const float kt = __uint_as_float(__float_as_uint(key) & 0xffff0000u);
        const unsigned past = __ballot_sync(FULL, lane < cnt && (double)kt > thr);
        if (past && lane == 0) {
          atomicMin(qstop + q, k_lo + __ffs(past) - 1);
          mark_done(q);  // every later item of q starts past the stop
        }
      }
      if (!todo) continue;
      it_q = q;
    }
  };

  // one finished pair of half h: the result (exact iff <= the cutoff, as diag_pair) and the
  // evaluated band cells; warp-wide
  auto publish = [&](int h) {
    const int s_ = __shfl_sync(FULL, st, 16 * h);
    const int q_ = __shfl_sync(FULL, pq, 16 * h), c_ = __shfl_sync(FULL, pc, 16 * h);
    const int te = __shfl_sync(FULL, tend, 16 * h);
    const R r_ = __shfl_sync(FULL, res, 16 * h + lf);
    const R ch = __shfl_sync(FULL, cut, 16 * h);
    const int cells = warp_cells<E_DIAG4>(L, L, w, te, 1);
#ifdef EKB_TRACE
    {
      const unsigned long long ps = __shfl_sync(FULL, tr_pst, 16 * h), pr = __shfl_sync(FULL, tr_prat, 16 * h);
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (lane == 0 && te >= 400) {
        const unsigned k = atomicAdd(&g_plog_n, 1u);
        if (k < 32768) {
          g_plog[k * 4 + 0] = ps;
          g_plog[k * 4 + 1] = now;
          g_plog[k * 4 + 2] = ((unsigned long long)q_ << 32) | (unsigned)te;
          g_plog[k * 4 + 3] = pr;
        }
      }
    }
#endif
    const double cq = ld_cut(cutbits + q_);
    if (lane == 0) {
      double cost = EKB_INF;
      if (s_ == 1) {
        const R c = fmin(ch, to_cut<R>(cq));
        cost = (r_ <= c) ? (double)r_ : EKB_INF;
        if (cost < EKB_INF) atomicMin(cutbits + q_, (unsigned long long)__double_as_longlong(cost));
      }
      nn_publish(acc, q_, c_, cost);
      atomicAdd((unsigned long long*)acc.cells + q_, (unsigned long long)cells);
    }
  };

  auto dstep = [&](auto S_, auto CHK_, const R* xblk, const R* yblk) {
    constexpr int S = decltype(S_)::value;
    constexpr bool CHK = decltype(CHK_)::value;
    constexpr int rx = S % RX;
    constexpr int ry = (RY - S % RY) % RY;
    constexpr bool VOTE = (S & 1) == 1;
    auto XW = [&](int k) -> R { return xw[(k + rx) % RX]; };
    auto YW = [&](int m) -> R { return yw[(m + ry) % RY]; };
    // ---- half step A: time t, even slots ----
    const R tin = __shfl_up_sync(FULL, val[P - 1], 1, 16);
#pragma unroll
    for (int m = 0; m < H; ++m) {
      const int p = 2 * m;
      const R T = (m == 0) ? tin : val[p - 1];
      const RowD<K_DTW, R> rr{XW(m)};
      const ColD<K_DTW, R> cc{YW(m)};
      R v;
      if (VIRT0 && p != 0) v = cell<K_DTW, MODE, false>(val[p], T, val[p + 1], rr, cc, kk[0], ss, prm);
      else v = cell<K_DTW, MODE, true, true>(val[p], T, val[p + 1], rr, cc, kk[VIRT0 ? 0 : p], ss, prm);
      val[p] = v;
      if (VOTE) alive |= hi_word(v) <= cut_hi;
    }
    // ---- half step B: time t + 1, odd slots ----
    const R lin = __shfl_down_sync(FULL, val[0], 1, 16);
#pragma unroll
    for (int m = 0; m < H; ++m) {
      const int p = 2 * m + 1;
      const R Lv = (p == P - 1) ? lin : val[p + 1];
      const RowD<K_DTW, R> rr{XW(m + 1)};
      const ColD<K_DTW, R> cc{YW(m)};
      R v;
      if (VIRT0) v = cell<K_DTW, MODE, false>(val[p], val[p - 1], Lv, rr, cc, kk[0], ss, prm);
      else v = cell<K_DTW, MODE>(val[p], val[p - 1], Lv, rr, cc, kk[VIRT0 ? 0 : p], ss, prm);
      val[p] = v;
      if (VOTE) alive |= hi_word(v) <= cut_hi;
    }
    if (CHK) {  // the final cell sits in an even slot at t == Tf (half step B leaves it alone)
      if (run && t + 1 >= Tf) {
        R r = val[0];
#pragma unroll
        for (int p = 1; p < P; ++p)
          if (p == pf) r = val[p];
        res = r;
        st = 1;
        tend = Tf;
        run = false;
      }
    }
    if (VOTE) {  // every path crosses one of the four anti-diagonals since the last vote
      const unsigned m = __ballot_sync(FULL, alive);
      if (run && !(m & hmask)) {
        st = 2;
        tend = t + 1;
        run = false;
      }
      alive = false;
    }
    t += 2;
    ++I0;
    ++J0;
    // slide: the new logical xw[H] goes to ring slot rx, the new logical yw[0] to ry(S + 1)
    xw[rx] = xblk[S + H];
    yw[(RY - (S + 1) % RY) % RY] = yblk[S];
  };

#ifdef EKB_TRACE
  unsigned long long tr_t0, tr_blocks = 0, tr_busy = 0, tr_pairs = 0, tr_exh = 0, tr_last_pair = 0, tr_maxblk = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_t0));
#endif
  for (;;) {
    // ---- publish and refill the idle halves (warp-uniform) ----
    const unsigned idle = __ballot_sync(FULL, !run);
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      if (!(idle & (1u << (16 * h)))) continue;
      if (__shfl_sync(FULL, st, 16 * h) != 0) {
        publish(h);
        if (half == h) st = 0;
      }
      int q = 0, c = 0;
      if (!next_pair(q, c)) {
#ifdef EKB_TRACE
        if (!tr_exh) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_exh));
#endif
        continue;
      }
#ifdef EKB_TRACE
      ++tr_pairs;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr_last_pair));
      if (half == h) {
        tr_pst = tr_last_pair;
        tr_prat = tr_ratio;
      }
#endif
      const double cq = ld_cut(cutbits + q);
      if (half == h) {
        pq = q;
        pc = c;
        xp = QP + (long long)q * pitch + kPadG;
        yp = CP + (long long)c * pitch + kPadG;
        t = 2;
        I0 = (2 + d0) >> 1;
        J0 = (2 - d0) >> 1;
#pragma unroll
        for (int p = 0; p < P; ++p) val[p] = (d0 + p == 0) ? (R)0.0 : INF;  // the corner (t = 0)
#pragma unroll
        for (int k = 0; k <= H; ++k) xw[k] = xp[I0 + k - 1];
#pragma unroll
        for (int m = 0; m < H; ++m) yw[m] = yp[J0 - m - 1];
        cut = to_cut<R>(cq);
        cut_hi = hi_word(cut);
        run = true;
        alive = false;
      }
    }
    if (!__any_sync(FULL, run)) break;
#ifdef EKB_TRACE
    {
      const unsigned rb = __ballot_sync(FULL, run);
      ++tr_blocks;
      tr_busy += ((rb & 1u) ? 1 : 0) + ((rb >> 16) & 1u ? 1 : 0);
    }
#endif
    // ---- one block of U double steps for both halves ----
    // every lane loads its half's cutoff (pq is always a valid query): no merge of a
    // conditional load, so nothing waits for it before the block's end
    unsigned long long nextcut;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(nextcut) : "l"(cutbits + pq));
    const bool chk = __any_sync(FULL, run && t + 2 * U + 1 >= Tf);
    if (!run) {  // an idle half's indices would keep advancing past its last series' pads
      I0 = 0;
      J0 = 0;
    }
    const R* xblk = xp + I0;
    const R* yblk = yp + J0;
    // After step RX - 1 the rings are back at phase 0: a half that stopped at the block's
    // first votes is refilled there (half a block sooner) when there is work left.  (Votes
    // are self-contained cut tests of their own double step, so their spacing may change.)
    auto brk = [&](auto S_) -> bool {
      constexpr int S = decltype(S_)::value;
      if constexpr (S == RX - 1) return !exhausted && __ballot_sync(FULL, !run) != 0u;
      return false;
    };
    if (!chk) {
      auto fast = [&](auto S_) {
        dstep(S_, std::false_type{}, xblk, yblk);
        return brk(S_);
      };
      unrolled_steps<0, U>(fast);
    } else {
      auto last = [&](auto S_) {
        dstep(S_, std::true_type{}, xblk, yblk);
        return brk(S_);
      };
      unrolled_steps<0, U>(last);
    }
    const double c64 = __longlong_as_double((long long)__shfl_sync(FULL, nextcut, 16 * half));
    if (run) {
      cut = fmin(cut, to_cut<R>(c64));
      cut_hi = hi_word(cut);
    }
  }
#ifdef EKB_TRACE
  if (lane == 0) {  // per warp: start, end, busy half-blocks, blocks, pairs (tools/trace_nn.py)
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (gw < 8192) {
      g_trace[gw * 8 + 0] = tr_t0;
      g_trace[gw * 8 + 1] = t1;
      g_trace[gw * 8 + 2] = tr_busy;
      g_trace[gw * 8 + 3] = tr_blocks;
      g_trace[gw * 8 + 4] = tr_pairs;
      g_trace[gw * 8 + 5] = tr_exh;
      g_trace[gw * 8 + 6] = tr_last_pair;
    }
  }
#endif
}

}  // namespace ekb

namespace ekb {
// host side (ek_inst_dtw.cu): pad series for k_nn2 (f32: float copies), and launch it
// persistently (occupancy-sized grid); both return the CUDA status of the launch
cudaError_t nn2_pad(int f32, const double* src, const long long* off, int n, int L, int pitch, void* dst,
                    cudaStream_t st);
cudaError_t nn2_launch(int mode, bool virt0, int nsm, long long warp_units, cudaStream_t st, const void* QP,
                       const void* CP, int pitch, int L, int nq, int ncand, const int* order, int rank_lo,
                       int rank_mid, int rank_hi, int K1, int K2, int w, unsigned long long* cutbits, NNAcc acc,
                       int* qnext, unsigned long long* qdone, const float* skeys, const float2* envq, int lmax,
                       int* qstop);
}  // namespace ekb
