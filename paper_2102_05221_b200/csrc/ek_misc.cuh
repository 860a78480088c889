// ek_misc.cuh -- declarations of the kind-independent kernels (ek_misc.cu).
#pragma once
#include "ek_kernels.cuh"

namespace ekb {

// Cells of the band evaluated by an engine that stopped at t_end: the diagonal
// engine evaluates every band cell with i + j <= t_end, the stripe engine row i of
// lane l while l <= r0 + t_end - 1 - i.
__device__ inline long long cells_done(int eng_diag, int S, int r0, int nl, int nc, int w, int tend) {
  long long cells = 0;
  const int imax = eng_diag ? min(nl, tend - 1) : min(nl, r0 + tend - 1);
  for (int i = 1; i <= imax; ++i) {
    const int jlo = max(1, i - w);
    int jhi = min(nc, i + w);
    jhi = eng_diag ? min(jhi, tend - i) : min(jhi, (r0 + tend - i) * S);
    if (jhi >= jlo) cells += jhi - jlo + 1;
  }
  return cells;
}

__global__ void k_rank_dist(const double* Q, const long long* qoff, const int* qlen, int nq, const double* C,
                            const long long* coff, const int* clen, int ncand, float* out);
__global__ void k_rank_sort(const float* keys, int ncand, int npow2, int* order);
__global__ void k_identity_order(int nq, int ncand, int* order);
__global__ void k_nn_reduce(const double* dist, const int* tend, const int* qlen, int nq, const int* clen, int ncand,
                            int win, int eng_diag, int S, int r0, long long* nn_idx, double* nn_dist,
                            long long* cells, long long* computed, long long* abandoned);
__global__ void k_cells_pairs(const PairDesc* pairs, const int* tend, int npairs, int eng_diag, int S, int r0,
                              long long* out);
__global__ void k_cells_triangle(const int* len, int n, int win, const int* tend, int eng_diag, int S, int r0,
                                 unsigned long long* total);

}  // namespace ekb
