// ek_misc.cuh -- declarations of the kind-independent kernels (ek_misc.cu).
#pragma once
#include <vector>
#include "ek_kernels.cuh"

namespace ekb {

// Envelopes (k_envelope): sparse-table rows in shared memory up to kEnvSmemMax bytes
// per series, else global scratch rows (env_scratch_bytes(L, exact); kEnvScratchBlocks
// blocks).  envelope(): float2 (upper rounded up, lower rounded down) for the LB
// kernels; envelope_exact(): build_envelope's double upper / lower.
enum EnvFmt { kEnvPlain = 0, kEnvPointMajor = 1, kEnvExact = 2 };
constexpr int kEnvThreads = 128;
constexpr int kEnvScratchBlocks = 592;  // 4 x 148 SMs
constexpr size_t kEnvSmemMax = 192 * 1024;
size_t env_smem_bytes(int L, bool exact);
size_t env_scratch_bytes(int L, bool exact);
cudaError_t envelope(const double* C, const long long* coff, int L, int nser, int w, float2* env, void* scratch,
                     cudaStream_t st);
// point-major float2 (-upper, lower) at env[k * nser + c]: the layout k_lb_matrix reads
// (stride: the row stride of env, >= nser; a chunk of candidates passes env + its first index)
// padded != null (k_nn2's padded copies, float when padded_f32): written in the same pass;
// env_pm8_smem(L) > 200 KB (very long series) takes the block-per-series kernel, without padding
cudaError_t envelope_pm(const double* C, const long long* coff, int L, int nser, int w, float2* env, void* scratch,
                        cudaStream_t st, int stride, void* padded = nullptr, int padded_f32 = 0, int pitch = 0,
                        int padg = 0);
size_t env_pm8_smem(int L);
cudaError_t envelope_exact(const double* C, const long long* coff, int L, int nser, int w, double* up, double* dn,
                           void* scratch, cudaStream_t st);

__global__ void k_rank_sort(const float* keys, int ncand, int npow2, int* order);
// per-query stable radix sort of the rank keys (ncand <= 16384); launches k_rank_radix
cudaError_t rank_radix(const float* keys, int nq, int ncand, int* order, cudaStream_t st, float* skeys = nullptr);
// LB_Keogh(q, env(c)) for all pairs of a dense batch, rounded down (keys of the LB path)
// lb_qprep: the queries point-major, qt[k * nq + q] = (RD(q), -RU(q)); lb_matrix: the keys of
// candidates [c_begin, c_end) (envp: envelope_pm of the candidates, row stride ncand)
cudaError_t lb_qprep(int mode, const double* Q, const long long* qoff, int nq, int L, float2* qt, cudaStream_t st);
cudaError_t lb_matrix(int mode, const float2* qt, int nq, const float2* envp, int ncand, int c_begin, int c_end, int L,
                      float* out, cudaStream_t st);
// out[i] = +inf, tend[i] = 0 (pairs the LB path never visits)
__global__ void k_paa(const double* src, const long long* off, const int* len, int n, int R, int D, float* dst);
__global__ void k_rank_paa(const float* Qp, int nq, const float* Cp, int ncand, int D, float* out);
__global__ void k_identity_order(int nq, int ncand, int* order);
__global__ void k_nn_pick(NNAcc a);
__global__ void k_nn_final(NNAcc a, int nq, int ncand, long long* nn_idx, double* nn_dist, long long* cells,
                           long long* computed, long long* abandoned);
__global__ void k_nn_acc_init(NNAcc a, int nq);

// ingestion (ek_ingest.cu): numpy pairwise-sum plans, and the series transforms on the device
void np_plan_build(int start, int n, std::vector<int2>& leaves, std::vector<int>& ops);
cudaError_t derivative_dev(const double* in, const long long* off, const int* len, long long n, double* out,
                           const long long* ooff, cudaStream_t st);
cudaError_t znormalize_dev(const double* in, const long long* off, const int* len, const int* hl, long long n,
                           double* out, const long long* ooff, cudaStream_t st);

}  // namespace ekb
