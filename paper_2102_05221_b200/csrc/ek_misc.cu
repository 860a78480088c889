// ek_misc.cu -- kind-independent kernels of the 1-NN path: candidate ranking
// (a scheduling heuristic only -- it never decides a result), the per-query
// lexicographic (distance, index) reduction, and computed-cell accounting.
#include "ek_misc.cuh"
#include <cub/block/block_radix_sort.cuh>
#include <algorithm>
#include <type_traits>

namespace ekb {

// Piecewise aggregate approximation for the ranking: dst[s * D + k] = sum of series s
// over points [kR, kR + R) (zero past its end), in FP32.  Ranking only.
__global__ void k_paa(const double* __restrict__ src, const long long* __restrict__ off,
                      const int* __restrict__ len, int n, int R, int D, float* __restrict__ dst) {
  const long long total = (long long)n * D;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(e / D), k = (int)(e % D);
    const int L = len[s];
    const double* x = src + off[s];
    float acc = 0.f;
    for (int r = 0; r < R; ++r) {
      const int i = k * R + r;
      if (i < L) acc += (float)x[i];
    }
    dst[e] = acc;
  }
}

// Squared Euclidean distance between PAA rows (FP32), 32x64 (query, candidate) tile per
// block (enough blocks to fill 148 SMs at 256 x 4096), 2x4 per thread, D in chunks of
// 16 through shared memory.  Ranking only.
__global__ void __launch_bounds__(256) k_rank_paa(const float* __restrict__ Qp, int nq, const float* __restrict__ Cp,
                                                  int ncand, int D, float* __restrict__ out) {
  __shared__ float qs[16][33];
  __shared__ float cs[16][65];
  const int q0 = blockIdx.y * 32, c0 = blockIdx.x * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[2][4] = {};
  for (int kb = 0; kb < D; kb += 16) {
    for (int e = threadIdx.x; e < 64 * 16; e += 256) {
      const int r = e >> 4, k = e & 15;
      const int c = c0 + r, kk = kb + k;
      cs[k][r] = (c < ncand && kk < D) ? Cp[(long long)c * D + kk] : 0.f;
      if (r < 32) {
        const int q = q0 + r;
        qs[k][r] = (q < nq && kk < D) ? Qp[(long long)q * D + kk] : 0.f;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      float a[2], b[4];
#pragma unroll
      for (int u = 0; u < 2; ++u) a[u] = qs[k][ty + 16 * u];
#pragma unroll
      for (int v = 0; v < 4; ++v) b[v] = cs[k][tx + 16 * v];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const float d = a[u] - b[v];
          acc[u][v] = fmaf(d, d, acc[u][v]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int q = q0 + ty + 16 * u, c = c0 + tx + 16 * v;
      if (q < nq && c < ncand) out[(long long)q * ncand + c] = acc[u][v];
    }
}

// LB_Keogh(q, env(c)) of every (query, candidate) pair of a dense batch (all series of
// length L), as a tiled matrix: 32 queries x 64 candidates per 128-thread block (enough
// blocks to keep every SM busy at 256 x 4096), 4 x 4 per thread, points in chunks of 32
// through shared memory.  Every operation rounds toward -inf (the query point widened to
// [RD(q), RU(q)], distances to the outward-rounded float envelope rounded down, squared
// and accumulated with fma.rm), so each value is a guaranteed lower bound of the exact
// LB_Keogh and hence of the DP value (ek_lb.cuh).  FP32 mode (MODE & M_F32): the query
// point is the float the DP stages.  Two candidates per packed FADD2 / FFMA2 (sm_100):
// per (query, candidate, point) 2.5 instructions.  These keys order the 1-NN candidates
// and drop pairs whose bound exceeds the running cutoff.
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk2(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(u64 v, float& a, float& b) { asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ u64 add2_rd(u64 a, u64 b) {
  u64 r;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 fma2_rd(u64 a, u64 b, u64 c) {
  u64 r;
  asm("fma.rm.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// qt[k * nq + q] = (RD(q), -RU(q)) (FP32 mode: (q, -q)): the queries point-major
template <int MODE>
__global__ void k_lb_qprep(const double* __restrict__ Q, const long long* __restrict__ qoff, int nq, int L,
                           float2* __restrict__ qt) {
  const long long n = (long long)nq * L;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(e / L), k = (int)(e % L);
    const double x = Q[qoff[q] + k];
    float lo, hi;
    if constexpr ((MODE & M_F32) != 0) {
      lo = hi = (float)x;
    } else {
      lo = __double2float_rd(x);
      hi = __double2float_ru(x);
    }
    qt[(long long)k * nq + q] = make_float2(lo, -hi);
  }
}

// Two 128-thread groups per block split the points (group g takes chunks g, g + 2, ...,
// syncing on its own named barrier) and combine their sums at the end (rounded down):
// twice the warps of a one-group tile for the same work, which hides the fill latency.
template <int MODE>
__global__ void __launch_bounds__(256) k_lb_matrix(const float2* __restrict__ qt, int nq, const float2* __restrict__ envp,
                                                   int ncand, int c_begin, int c_end, int L, float* __restrict__ out) {
  constexpr int KP = 16;
  __shared__ __align__(16) float2 qs_[2][KP][32];  // (RD(q), -RU(q))
  __shared__ __align__(16) float nus_[2][KP][64];  // -upper
  __shared__ __align__(16) float los_[2][KP][64];  // lower
  const int g = threadIdx.x >> 7, t = threadIdx.x & 127;
  float2 (&qs)[KP][32] = qs_[g];
  float (&nus)[KP][64] = nus_[g];
  float (&los)[KP][64] = los_[g];
  auto gsync = [&]() {
    if (g == 0) asm volatile("bar.sync 1, 128;" ::: "memory");
    else asm volatile("bar.sync 2, 128;" ::: "memory");
  };
  const int q0 = blockIdx.y * 32, c0 = c_begin + blockIdx.x * 64;
  const int tx = t & 15, ty = t >> 4;
  u64 acc[4][2] = {};
  const float NINF = __int_as_float(0xff800000);
  // fills (point-major sources, consecutive threads = consecutive candidates / queries:
  // coalesced loads, conflict-free stores): candidates cc = t % 64 at points t / 64 + 2 i,
  // queries qq = t % 32 at points t / 32 + 4 i; all of a chunk's loads are issued first
  const int cc = t & 63, kc = t >> 6, qq = t & 31, kq = t >> 5;
  const bool c_ok = c0 + cc < c_end, q_ok = q0 + qq < nq;
  for (int k0 = g * KP; k0 < L; k0 += 2 * KP) {
    float2 ev[KP / 2], qv[KP / 4];
#pragma unroll
    for (int i = 0; i < KP / 2; ++i) {
      const int k = k0 + kc + 2 * i;
      ev[i] = (c_ok && k < L) ? envp[(long long)k * ncand + c0 + cc] : make_float2(NINF, NINF);  // neutral
    }
#pragma unroll
    for (int i = 0; i < KP / 4; ++i) {
      const int k = k0 + kq + 4 * i;
      qv[i] = (q_ok && k < L) ? qt[(long long)k * nq + q0 + qq] : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < KP / 2; ++i) {
      nus[kc + 2 * i][cc] = ev[i].x;
      los[kc + 2 * i][cc] = ev[i].y;
    }
#pragma unroll
    for (int i = 0; i < KP / 4; ++i) qs[kq + 4 * i][qq] = qv[i];
    gsync();
#pragma unroll 4
    for (int k = 0; k < KP; ++k) {
      const float4 nu = *reinterpret_cast<const float4*>(&nus[k][tx * 4]);
      const float4 lo = *reinterpret_cast<const float4*>(&los[k][tx * 4]);
      const float4 qa = *reinterpret_cast<const float4*>(&qs[k][ty * 4]);
      const float4 qb = *reinterpret_cast<const float4*>(&qs[k][ty * 4 + 2]);
      const u64 nU[2] = {pk2(nu.x, nu.y), pk2(nu.z, nu.w)}, Lo[2] = {pk2(lo.x, lo.y), pk2(lo.z, lo.w)};
      const float ql[4] = {qa.x, qa.z, qb.x, qb.z}, nqh[4] = {qa.y, qa.w, qb.y, qb.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const u64 l2 = pk2(ql[u], ql[u]), h2 = pk2(nqh[u], nqh[u]);  // scalar operands broadcast (.F32)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          float a0, a1, b0, b1;
          upk2(add2_rd(l2, nU[v]), a0, a1);  // RD(q) - upper
          upk2(add2_rd(Lo[v], h2), b0, b1);  // lower - RU(q)
          const u64 d = pk2(fmaxf(fmaxf(a0, b0), 0.f), fmaxf(fmaxf(a1, b1), 0.f));
          acc[u][v] = (MODE & 1) == 0 ? fma2_rd(d, d, acc[u][v]) : add2_rd(acc[u][v], d);
        }
      }
    }
    gsync();
  }
  // group 1 hands its sums to group 0 through the (then idle) tiles: 128 threads x 8 sums
  // = 8 KB from nus_[1] into los_[0], so both groups must be done with them
  u64* const part = reinterpret_cast<u64*>(&nus_[1][0][0]);
  __syncthreads();
  if (g == 1) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v) part[(u * 2 + v) * 128 + t] = acc[u][v];
  }
  __syncthreads();
  if (g == 1) return;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int q = q0 + ty * 4 + u;
    if (q >= nq) continue;
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      float a, b, a1, b1;
      upk2(acc[u][v], a, b);
      upk2(part[(u * 2 + v) * 128 + t], a1, b1);
      const int c = c0 + tx * 4 + 2 * v;
      if (c < c_end) out[(long long)q * ncand + c] = __fadd_rd(a, a1);
      if (c + 1 < c_end) out[(long long)q * ncand + c + 1] = __fadd_rd(b, b1);
    }
  }
}

cudaError_t lb_qprep(int mode, const double* Q, const long long* qoff, int nq, int L, float2* qt, cudaStream_t st) {
  const unsigned pb = (unsigned)std::min<long long>(1024, ((long long)nq * L + 255) / 256);
  switch (mode) {
    case 0: k_lb_qprep<0><<<pb, 256, 0, st>>>(Q, qoff, nq, L, qt); break;
    case 1: k_lb_qprep<1><<<pb, 256, 0, st>>>(Q, qoff, nq, L, qt); break;
    case 2: k_lb_qprep<2><<<pb, 256, 0, st>>>(Q, qoff, nq, L, qt); break;
    default: k_lb_qprep<3><<<pb, 256, 0, st>>>(Q, qoff, nq, L, qt); break;
  }
  return cudaGetLastError();
}
cudaError_t lb_matrix(int mode, const float2* qt, int nq, const float2* envp, int ncand, int c_begin, int c_end, int L,
                      float* out, cudaStream_t st) {
  if (c_end <= c_begin) return cudaSuccess;
  const dim3 grid((unsigned)((c_end - c_begin + 63) / 64), (unsigned)((nq + 31) / 32));
  switch (mode) {
    case 0: k_lb_matrix<0><<<grid, 256, 0, st>>>(qt, nq, envp, ncand, c_begin, c_end, L, out); break;
    case 1: k_lb_matrix<1><<<grid, 256, 0, st>>>(qt, nq, envp, ncand, c_begin, c_end, L, out); break;
    case 2: k_lb_matrix<2><<<grid, 256, 0, st>>>(qt, nq, envp, ncand, c_begin, c_end, L, out); break;
    default: k_lb_matrix<3><<<grid, 256, 0, st>>>(qt, nq, envp, ncand, c_begin, c_end, L, out); break;
  }
  return cudaGetLastError();
}

// Per query: stable block radix sort of (key, candidate) -> ranked candidate order
// (ties keep index order).  THREADS x ITEMS >= ncand; padding sorts last.
template <int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS) k_rank_radix(const float* __restrict__ keys, int ncand,
                                                        int* __restrict__ order, int lo_bit,
                                                        float* __restrict__ skeys) {
  using Sort = cub::BlockRadixSort<float, THREADS, ITEMS, int>;
  extern __shared__ __align__(16) unsigned char rank_sm[];
  auto& tmp = *reinterpret_cast<typename Sort::TempStorage*>(rank_sm);
  const int q = blockIdx.x;
  const float* row = keys + (long long)q * ncand;
  float k[ITEMS];
  int v[ITEMS];
#pragma unroll
  for (int u = 0; u < ITEMS; ++u) {
    const int i = threadIdx.x * ITEMS + u;  // blocked arrangement
    const float key = i < ncand ? row[i] : __int_as_float(0x7f800000);
    k[u] = key != key ? __int_as_float(0x7f800000) : key;  // NaN ranks last
    v[u] = i;
  }
  Sort(tmp).Sort(k, v, lo_bit, 32);
#pragma unroll
  for (int u = 0; u < ITEMS; ++u) {
    const int i = threadIdx.x * ITEMS + u;
    if (i < ncand) {
      order[(long long)q * ncand + i] = v[u];
      if (skeys) skeys[(long long)q * ncand + i] = k[u];  // the keys in rank order
    }
  }
}
// launched from this unit (a template kernel's host stub must live with its definition)
cudaError_t rank_radix(const float* keys, int nq, int ncand, int* order, cudaStream_t st, float* skeys) {
  const int lo_bit = 16;  // top 16 key bits (~1% buckets): the order is a schedule only
  if (ncand <= 128 * 8) {
    using Sort = cub::BlockRadixSort<float, 128, 8, int>;
    k_rank_radix<128, 8><<<nq, 128, sizeof(typename Sort::TempStorage), st>>>(keys, ncand, order, lo_bit, skeys);
  } else if (ncand <= 256 * 16) {
    using Sort = cub::BlockRadixSort<float, 256, 16, int>;
    k_rank_radix<256, 16><<<nq, 256, sizeof(typename Sort::TempStorage), st>>>(keys, ncand, order, lo_bit, skeys);
  } else {
    using Sort = cub::BlockRadixSort<float, 1024, 16, int>;
    const size_t sm = sizeof(typename Sort::TempStorage);
    cudaError_t e = cudaFuncSetAttribute((const void*)k_rank_radix<1024, 16>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    k_rank_radix<1024, 16><<<nq, 1024, sm, st>>>(keys, ncand, order, lo_bit, skeys);
  }
  return cudaGetLastError();
}

// Per query: bitonic sort of (key, candidate) in shared memory -> ranked candidate order.
__global__ void __launch_bounds__(1024) k_rank_sort(const float* __restrict__ keys, int ncand, int npow2,
                                                    int* __restrict__ order) {
  extern __shared__ unsigned char sm_raw[];
  float* k = reinterpret_cast<float*>(sm_raw);
  int* v = reinterpret_cast<int*>(k + npow2);
  const int q = blockIdx.x;
  for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
    k[i] = i < ncand ? keys[(long long)q * ncand + i] : __int_as_float(0x7f800000);
    v[i] = i;
  }
  __syncthreads();
  for (int size = 2; size <= npow2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < npow2 / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const float a = k[lo], b = k[hi];
        const int va = v[lo], vb = v[hi];
        // ascending by (key, index) so equal keys keep index order
        const bool gt = (a > b) || (a == b && va > vb);
        if (gt == up) {
          k[lo] = b; k[hi] = a;
          v[lo] = vb; v[hi] = va;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < ncand; i += blockDim.x) order[(long long)q * ncand + i] = v[i];
}

__global__ void k_identity_order(int nq, int ncand, int* __restrict__ order) {
  const long long n = (long long)nq * ncand;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    order[i] = (int)(i % ncand);
}

// nn_search's outcome per query (search.py:101-123) from the accumulators of k_nn
// (NNAcc): the lowest index among the finite results equal to the query's least cost --
// the serial scan's strict "<" keeps the first one.
__global__ void k_nn_pick(NNAcc a) {
  const int n = *a.fin_count;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const long long qc = a.fin[k];
    const int q = (int)(qc >> 32), c = (int)(qc & 0xffffffffLL);
    if ((unsigned long long)__double_as_longlong(a.fin_cost[k]) == a.best[q]) atomicMin(a.idx + q, c);
  }
}
__global__ void k_nn_final(NNAcc a, int nq, int ncand, long long* __restrict__ nn_idx, double* __restrict__ nn_dist,
                           long long* __restrict__ cells, long long* __restrict__ computed,
                           long long* __restrict__ abandoned) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
    const int i = a.idx[q];
    nn_idx[q] = i == 0x7fffffff ? -1 : i;
    nn_dist[q] = __longlong_as_double((long long)a.best[q]);
    cells[q] = a.cells[q];
    computed[q] = a.computed[q];
    abandoned[q] = ncand - a.computed[q];
  }
}
__global__ void k_nn_acc_init(NNAcc a, int nq) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
    a.best[q] = 0x7ff0000000000000ULL;
    a.cells[q] = 0;
    a.computed[q] = 0;
    a.idx[q] = 0x7fffffff;
    if (q == 0) *a.fin_count = 0;
  }
}

// Sliding max/min over [k-w, k+w] (build_envelope, lower_bounds.py:23-57) for every
// series, row-major (env[c * L + k] = (upper, lower)) so a warp reads 32 consecutive
// points; stored as floats rounded outward (upper up, lower down).  Rounding is
// monotone, so it is applied first and the tables hold floats.
//
// Sparse table per series: level p holds max/min of x[k .. k + 2^p - 1].  A clipped
// window [a, b] of length n is covered by two level-floor(log2 n) runs,
// max(T[a], T[b - 2^p + 1]).  Window lengths lie in [min(w+1, L), min(2w+1, L)], a
// factor-of-two range, so only levels pmin and pmin + 1 are needed: level pmin is
// built in place (rows processed in increasing chunks of the block, each read before
// any write of its chunk), level pmin + 1 goes to a second pair of rows.  16 L bytes
// per series: shared memory, or the global `scratch` rows (16 L bytes per block) when
// L is too long for it.  Blocks stride over the series.
template <class T>
__device__ __forceinline__ T tmax(T a, T b) { return a > b ? a : b; }  // no NaNs here (finite inputs)
template <class T>
__device__ __forceinline__ T tmin(T a, T b) { return a < b ? a : b; }

// FMT (EnvFmt): kEnvPlain float2 (upper, lower); kEnvExact double tables,
// build_envelope's upper / lower.  GLOBAL: table
// rows in `scratch` (a compile-time choice, so shared-memory accesses stay LDS/STS).
template <int FMT, bool GLOBAL>
__global__ void __launch_bounds__(kEnvThreads) k_envelope(const double* __restrict__ C,
                                                          const long long* __restrict__ coff, int L, int nser, int w,
                                                          float2* __restrict__ env, double* __restrict__ up, double* __restrict__ dn,
                                                          void* __restrict__ scratch, int pm_stride) {
  constexpr bool EXACT = FMT == kEnvExact;
  using T = typename std::conditional<EXACT, double, float>::type;
  extern __shared__ __align__(16) unsigned char env_sm[];
  T* hi;
  if constexpr (GLOBAL) hi = static_cast<T*>(scratch) + (size_t)blockIdx.x * 4 * L;
  else hi = reinterpret_cast<T*>(env_sm);
  T* const lo = hi + L;
  T* const hi2 = hi + 2 * L;
  T* const lo2 = hi + 3 * L;
  const int W = min(w, L - 1);
  const int pmin = 31 - __clz(min(W + 1, L)), pmax = 31 - __clz(min(2 * W + 1, L));
  constexpr int R = 4, CH = kEnvThreads * R;
  for (int c = blockIdx.x; c < nser; c += gridDim.x) {
    const double* src = C + coff[c];
    for (int k = threadIdx.x; k < L; k += kEnvThreads) {
      const double x = src[k];
      if constexpr (EXACT) {
        hi[k] = x;
        lo[k] = x;
      } else {
        hi[k] = __double2float_ru(x);
        lo[k] = __double2float_rd(x);
      }
    }
    for (int p = 1; p <= pmax; ++p) {
      const int s = 1 << (p - 1), n = L - (1 << p) + 1;  // entries of level p
      const bool inplace = p <= pmin;
      T* const dh = inplace ? hi : hi2;
      T* const dl = inplace ? lo : lo2;
      for (int base = 0; base < n; base += CH) {
        T vh[R], vl[R];
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int k = base + r * kEnvThreads + threadIdx.x;
          if (k < n) {
            vh[r] = tmax(hi[k], hi[k + s]);
            vl[r] = tmin(lo[k], lo[k + s]);
          }
        }
        if (inplace) __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int k = base + r * kEnvThreads + threadIdx.x;
          if (k < n) {
            dh[k] = vh[r];
            dl[k] = vl[r];
          }
        }
      }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < L; k += kEnvThreads) {
      const int a = max(k - W, 0), b = min(k + W, L - 1);
      const int p = 31 - __clz(b - a + 1);
      const T* th = p == pmin ? hi : hi2;
      const T* tl = p == pmin ? lo : lo2;
      const int b2 = b - (1 << p) + 1;
      const long long o = FMT == kEnvPointMajor ? (long long)k * pm_stride + c : (long long)c * L + k;
      const T u = tmax(th[a], th[b2]), l = tmin(tl[a], tl[b2]);
      if constexpr (EXACT) {
        up[o] = u;
        dn[o] = l;
      } else if constexpr (FMT == kEnvPointMajor) {
        env[o] = make_float2(-u, l);
      } else {
        env[o] = make_float2(u, l);
      }
    }
    __syncthreads();
  }
}

size_t env_smem_bytes(int L, bool exact) { return (exact ? 32 : 16) * (size_t)L; }
size_t env_scratch_bytes(int L, bool exact) {
  return env_smem_bytes(L, exact) > kEnvSmemMax ? env_smem_bytes(L, exact) * kEnvScratchBlocks : 0;
}

template <int FMT>
static cudaError_t envelope_launch(const double* C, const long long* coff, int L, int nser, int w, float2* env,
                                   double* up, double* dn, void* scratch, cudaStream_t st, int pm_stride = 0) {
  if (nser <= 0 || L <= 0) return cudaSuccess;
  constexpr bool EXACT = FMT == kEnvExact;
  const size_t sm = env_smem_bytes(L, EXACT);
  if (env_scratch_bytes(L, EXACT)) {
    if (!scratch) return cudaErrorInvalidValue;
    k_envelope<FMT, true><<<(unsigned)std::min(nser, kEnvScratchBlocks), kEnvThreads, 0, st>>>(
        C, coff, L, nser, w, env, up, dn, scratch, pm_stride);
  } else {
    if (sm > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute((const void*)k_envelope<FMT, false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      if (e != cudaSuccess) return e;
    }
    k_envelope<FMT, false><<<(unsigned)nser, kEnvThreads, sm, st>>>(C, coff, L, nser, w, env, up, dn, nullptr, pm_stride);
  }
  return cudaGetLastError();
}
cudaError_t envelope(const double* C, const long long* coff, int L, int nser, int w, float2* env, void* scratch,
                     cudaStream_t st) {
  return envelope_launch<kEnvPlain>(C, coff, L, nser, w, env, nullptr, nullptr, scratch, st);
}
// Point-major candidate envelopes for the LB keys, warp per series, eight series per block:
// each warp builds its series' sparse table in its own shared-memory rows (the same levels
// and clipped windows as k_envelope, so the same floats), and the block writes its eight
// series' envelopes transposed, eight consecutive candidates per point (k_envelope's
// block-per-series writes land one 8-byte value per 32-byte sector).  With `padded`, the
// warp also writes the padded copy k_nn2 reads (kPadG_ elements of 0.0 before the series, of
// +inf after it; float in the FP32 mode): one pass over the candidates instead of two.
constexpr int kEnvPmSeries = 8;
template <class R>
__global__ void __launch_bounds__(256) k_envelope_pm8(const double* __restrict__ C, const long long* __restrict__ coff,
                                                       int L, int nser, int w, float2* __restrict__ env, int stride,
                                                       R* __restrict__ padded, int pitch, int padg) {
  extern __shared__ __align__(16) unsigned char envpm_sm[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float2* const tile = reinterpret_cast<float2*>(envpm_sm);          // [L][8]
  float* const hi = reinterpret_cast<float*>(tile + (size_t)L * kEnvPmSeries) + (size_t)wib * 4 * L;
  float* const lo = hi + L;
  float* const hi2 = hi + 2 * L;
  float* const lo2 = hi + 3 * L;
  const int W = min(w, L - 1);
  const int pmin = 31 - __clz(min(W + 1, L)), pmax = 31 - __clz(min(2 * W + 1, L));
  const int c0 = blockIdx.x * kEnvPmSeries;
  const int c = c0 + wib;
  if (c < nser) {
    const double* src = C + coff[c];
    R* pc = padded ? padded + (long long)c * pitch : nullptr;
    for (int k = lane; k < L; k += 32) {
      const double x = src[k];
      hi[k] = __double2float_ru(x);
      lo[k] = __double2float_rd(x);
      if (pc) pc[padg + k] = (R)x;
    }
    if (pc) {
      for (int k = lane; k < padg; k += 32) {
        pc[k] = (R)0.0;
        pc[padg + L + k] = rinf<R>();
      }
    }
    __syncwarp();
    for (int p = 1; p <= pmax; ++p) {
      const int sh = 1 << (p - 1), n = L - (1 << p) + 1;
      const bool inplace = p <= pmin;
      float* const dh = inplace ? hi : hi2;
      float* const dl = inplace ? lo : lo2;
      for (int base = 0; base < n; base += 128) {  // four values per lane read before any write
        float vh[4], vl[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int k = base + r * 32 + lane;
          if (k < n) {
            vh[r] = tmax(hi[k], hi[k + sh]);
            vl[r] = tmin(lo[k], lo[k + sh]);
          }
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int k = base + r * 32 + lane;
          if (k < n) {
            dh[k] = vh[r];
            dl[k] = vl[r];
          }
        }
        __syncwarp();
      }
    }
    for (int k = lane; k < L; k += 32) {
      const int a = max(k - W, 0), b = min(k + W, L - 1);
      const int p = 31 - __clz(b - a + 1);
      const float* th = p == pmin ? hi : hi2;
      const float* tl = p == pmin ? lo : lo2;
      const int b2 = b - (1 << p) + 1;
      tile[k * kEnvPmSeries + wib] = make_float2(-tmax(th[a], th[b2]), tmin(tl[a], tl[b2]));
    }
  }
  __syncthreads();
  const int ns = min(kEnvPmSeries, nser - c0);
  for (int i = threadIdx.x; i < L * kEnvPmSeries; i += blockDim.x) {
    const int k = i / kEnvPmSeries, sidx = i % kEnvPmSeries;
    if (sidx < ns) env[(long long)k * stride + c0 + sidx] = tile[i];
  }
}

size_t env_pm8_smem(int L) { return (size_t)L * kEnvPmSeries * (sizeof(float2) + 4 * sizeof(float)); }

cudaError_t envelope_pm(const double* C, const long long* coff, int L, int nser, int w, float2* env, void* scratch,
                        cudaStream_t st, int stride, void* padded, int padded_f32, int pitch, int padg) {
  const size_t sm = env_pm8_smem(L);
  if (nser > 0 && L > 0 && sm <= 200 * 1024) {
    const unsigned grid = (unsigned)((nser + kEnvPmSeries - 1) / kEnvPmSeries);
    cudaError_t e;
    if (padded_f32) {
      if (sm > 48 * 1024 && (e = cudaFuncSetAttribute((const void*)k_envelope_pm8<float>,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)) != cudaSuccess)
        return e;
      k_envelope_pm8<float><<<grid, 256, sm, st>>>(C, coff, L, nser, w, env, stride, (float*)padded, pitch, padg);
    } else {
      if (sm > 48 * 1024 && (e = cudaFuncSetAttribute((const void*)k_envelope_pm8<double>,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)) != cudaSuccess)
        return e;
      k_envelope_pm8<double><<<grid, 256, sm, st>>>(C, coff, L, nser, w, env, stride, (double*)padded, pitch, padg);
    }
    return cudaGetLastError();
  }
  if (padded) return cudaErrorInvalidValue;  // (long series: the caller pads separately)
  return envelope_launch<kEnvPointMajor>(C, coff, L, nser, w, env, nullptr, nullptr, scratch, st, stride);
}
cudaError_t envelope_exact(const double* C, const long long* coff, int L, int nser, int w, double* up, double* dn,
                           void* scratch, cudaStream_t st) {
  return envelope_launch<kEnvExact>(C, coff, L, nser, w, nullptr, up, dn, scratch, st);
}

}  // namespace ekb
