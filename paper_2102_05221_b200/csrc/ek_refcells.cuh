// ek_refcells.cuh -- the reference's own cells_computed for single-pair distance()
// (SURVEY 8(f)#3), so EngineResult(cost, cells) equals the reference's for every
// variant, not only for base.
//
// The GPU engines evaluate a superset of the cells the reference touches, in
// another order, so their own counts differ.  The reference's count is a pure
// function of which cells are <= cutoff:
//   * _ea (_speedups.pyx:129-162) computes whole band rows and stops after the
//     first row whose minimum (left border included) exceeds the cutoff;
//   * _eapruned (_speedups.pyx:165-271) walks each row through its five stages,
//     driven only by "value <= cutoff" tests on cells it computed.  The cells it
//     computes carry the true DP value whenever that value is <= cutoff (every
//     dependency it drops is one it has proven > cutoff), and the unpruned DP value
//     is <= cutoff exactly when the pruned one is.  So the live masks of the
//     plain DP drive an exact replay of its control flow.
// The row-stripe engine records those masks (RowBits: 16 columns per lane, one
// 16-bit word per lane per row), then lane 0 replays the stages.  Rows the engine
// never reached (it stops once two steps are dead) are dead, as the bitmap's
// zeros say.
#pragma once
#include "ek_kernels.cuh"

namespace ekb {

constexpr int kRefMaxCols = 512;              // 32 lanes x 16 columns
constexpr int kRefWords = kRefMaxCols / 16;   // 16-bit words per row

struct RowBits {
  static constexpr bool on = true;
  unsigned short* bits;  // [(nl+1) x kRefWords]: bit s of word l = column 16*l + s + 1
  unsigned char* vbl;    // [nl+1]: left border (i, 0) <= cutoff
  __device__ __forceinline__ void row(int i, int lane, unsigned m) const {
    bits[i * kRefWords + lane] = (unsigned short)m;
  }
  __device__ __forceinline__ void vb(int i, bool live) const { vbl[i] = live; }
};

__device__ __forceinline__ bool live_at(const unsigned short* row, int j) {  // column j >= 1
  return (row[(j - 1) >> 4] >> ((j - 1) & 15)) & 1;
}
// first live column in [a, b] (b >= a), or -1
__device__ __forceinline__ int first_live(const unsigned short* row, int a, int b) {
  for (int j = a; j <= b;) {
    const int w = (j - 1) >> 4, o = (j - 1) & 15;
    const unsigned m = (unsigned)row[w] >> o;
    if (m) {
      const int f = j + __ffs(m) - 1;
      return f <= b ? f : -1;
    }
    j += 16 - o;
  }
  return -1;
}
// last live column in [a, b], or -1
__device__ __forceinline__ int last_live(const unsigned short* row, int a, int b) {
  for (int j = b; j >= a;) {
    const int w = (j - 1) >> 4, o = (j - 1) & 15;
    const unsigned m = (unsigned)row[w] & ((2u << o) - 1u);
    if (m) {
      const int f = 16 * w + 31 - __clz(m) + 1;
      return f >= a ? f : -1;
    }
    j -= o + 1;
  }
  return -1;
}
// first dead column in [a, b], or -1
__device__ __forceinline__ int first_dead(const unsigned short* row, int a, int b) {
  for (int j = a; j <= b;) {
    const int w = (j - 1) >> 4, o = (j - 1) & 15;
    const unsigned m = (~(unsigned)row[w] & 0xffffu) >> o;
    if (m) {
      const int f = j + __ffs(m) - 1;
      return f <= b ? f : -1;
    }
    j += 16 - o;
  }
  return -1;
}

// _eapruned's cells_computed (_speedups.pyx:165-271) from the live masks.
// bits row 0 = hborder (ERP), vbl[i] = vborder(i) <= cutoff; w >= nl - nc.
__device__ __forceinline__ long long eapruned_cells(const unsigned short* bits, const unsigned char* vbl, int nl, int nc, int w,
                                    bool bordered) {
  long long cells = 0;
  int npp = 1;
  if (bordered) {  // row 0: hborder(j) for j <= min(w + 1, nc)
    const int l = last_live(bits, 1, min(w + 1, nc));
    if (l > 0) npp = l + 1;
  }
  int next_start = 1, pp = npp, j = 1;
  for (int i = 1; i <= nl; ++i) {
    const unsigned short* row = bits + i * kRefWords;
    const int jstart = max(i - w, next_start), jstop = min(i + w, nc);
    j = jstart;
    const bool left_live = jstart == 1 && vbl[i];
    bool alive = left_live;
    // stage 2: discard points while the left neighbour is dead
    if (!left_live && j <= pp - 1 && j == next_start) {
      const int f = first_live(row, j, pp - 1);
      if (f > 0) {
        cells += f - j + 1;
        npp = f + 1;
        alive = true;
        next_start = f;
        j = f + 1;
      } else {
        cells += pp - j;
        next_start = pp;
        j = pp;
      }
    }
    // stage 3: full cells up to the pruning point
    if (j <= pp - 1) {
      cells += pp - j;
      const int l = last_live(row, j, pp - 1);
      if (l > 0) {
        npp = l + 1;
        alive = true;
      }
      j = pp;
    }
    // stage 4: the pruning point
    if (j <= jstop) {
      const bool left_dead = (j - 1 < jstart) ? !left_live : !live_at(row, j - 1);
      cells += 1;
      const bool lv = live_at(row, j);
      if (j == next_start && left_dead) {
        if (!lv) return cells;  // abandoned
      }
      if (lv) {
        npp = j + 1;
        alive = true;
      }
      ++j;
    } else if (j == next_start) {
      return cells;  // abandoned
    }
    // stage 5: left-only tail while the previous cell is live
    if (j <= jstop && j == npp) {
      const int d = first_dead(row, j, jstop);
      if (d > 0) {
        cells += d - j + 1;
        if (d > j) alive = true;
        npp = d;
        j = d + 1;
      } else {
        cells += jstop - j + 1;
        alive = true;
        npp = jstop + 1;
        j = jstop + 1;
      }
    }
    if (!alive) return cells;
    pp = npp;
  }
  return cells;
}

// _ea's count: whole band rows through the first failing row (or all rows).
__device__ __forceinline__ long long ea_cells(int nl, int nc, int w, int rows) {
  long long c = 0;
  for (int i = 1; i <= min(rows, nl); ++i) c += min(i + w, nc) - max(i - w, 1) + 1;
  return c;
}

}  // namespace ekb
