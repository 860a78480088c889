// ek_misc.cuh -- declarations of the kind-independent kernels (ek_misc.cu).
#pragma once
#include "ek_kernels.cuh"

namespace ekb {

__global__ void k_envelope(const double* C, const long long* coff, int L, int ncand, int w, float2* env);

__global__ void k_rank_dist(const double* Q, const long long* qoff, const int* qlen, int nq, const double* C,
                            const long long* coff, const int* clen, int ncand, float* out);
__global__ void k_rank_sort(const float* keys, int ncand, int npow2, int* order);
// per-query stable radix sort of the rank keys (ncand <= 16384); launches k_rank_radix
cudaError_t rank_radix(const float* keys, int nq, int ncand, int* order, cudaStream_t st);
__global__ void k_paa(const double* src, const long long* off, const int* len, int n, int R, int D, float* dst);
__global__ void k_rank_paa(const float* Qp, int nq, const float* Cp, int ncand, int D, float* out);
__global__ void k_identity_order(int nq, int ncand, int* order);
__global__ void k_nn_reduce(const double* dist, const int* tend, const int* qlen, int nq, const int* clen, int ncand,
                            int win, int eng_diag, int S, int r0, long long* nn_idx, double* nn_dist,
                            long long* cells, long long* computed, long long* abandoned);

}  // namespace ekb
