// ek_ingest.cu -- ingestion: UCR text files parsed natively into the packed
// layout every entry point takes (one flat float64 buffer, int64 offsets, lengths; the
// Python side places it in page-locked memory), and the per-series transforms of
// series.py on the device, bit-identical to the reference's numpy:
//   derivative  (pkg/src/elastik/series.py:134-144)
//   znormalize  (pkg/src/elastik/series.py:118-131; numpy's pairwise sums, ek_subseq.cuh)
#include <clocale>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/elastik_b200.h"
#include "ek_misc.cuh"
#include "ek_subseq.cuh"

namespace ekb {

// numpy pairwise-sum plan for a series of n elements starting at `start` (see ek_subseq.cuh):
// leaves of <= 128 elements in recursion order, ops in post order (k >= 0: leaf k, -1: add)
void np_plan_build(int start, int n, std::vector<int2>& leaves, std::vector<int>& ops) {
  if (n <= 128) {
    ops.push_back((int)leaves.size());
    leaves.push_back(make_int2(start, n));
    return;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  np_plan_build(start, n2, leaves, ops);
  np_plan_build(start + n2, n - n2, leaves, ops);
  ops.push_back(-1);
}

// out[i] = ((s[i+1] - s[i]) + (s[i+2] - s[i]) / 2) / 2 (x / 2 and x * 0.5 are the same
// correctly rounded value); one block per series
__global__ void k_derivative(const double* __restrict__ in, const long long* __restrict__ off,
                             const int* __restrict__ len, long long n, double* __restrict__ out,
                             const long long* __restrict__ ooff) {
  for (long long s = blockIdx.x; s < n; s += gridDim.x) {
    const double* x = in + off[s];
    double* y = out + ooff[s];
    const int m = len[s] - 2;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      const double a = x[i], b = x[i + 1], c = x[i + 2];
      y[i] = __dmul_rn(__dadd_rn(__dsub_rn(b, a), __dmul_rn(__dsub_rn(c, a), 0.5)), 0.5);
    }
  }
}

// znormalize of every series, one warp per series: numpy's mean / std (warp_znorm_stats with
// the pairwise-sum plan of the series' length), std < 1e-12 -> zeros, else (s - mean) / std
__global__ void __launch_bounds__(32) k_znorm_batch(const double* __restrict__ in, const long long* __restrict__ off,
                                                    const int* __restrict__ len, long long n,
                                                    double* __restrict__ out, const long long* __restrict__ ooff,
                                                    const int2* __restrict__ leaves, const int* __restrict__ ops,
                                                    const int4* __restrict__ plans, const int* __restrict__ plan_of) {
  extern __shared__ double scratch[];
  const int lane = threadIdx.x & 31;
  for (long long s = blockIdx.x; s < n; s += gridDim.x) {
    const int4 pd = plans[plan_of[s]];
    const NpPlan plan{leaves + pd.x, pd.y, ops + pd.z, pd.w};
    const double* x = in + off[s];
    const int m = len[s];
    const WinStats st = warp_znorm_stats(x, m, plan, scratch);
    double* y = out + ooff[s];
    for (int k = lane; k < m; k += 32) y[k] = st.zero ? 0.0 : __ddiv_rn(dsub(x[k], st.mean), st.sd);
    __syncwarp();
  }
}

cudaError_t derivative_dev(const double* in, const long long* off, const int* len, long long n, double* out,
                           const long long* ooff, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const unsigned blocks = (unsigned)std::min<long long>(n, 148LL * 16);
  k_derivative<<<blocks, 128, 0, st>>>(in, off, len, n, out, ooff);
  return cudaGetLastError();
}

// plans: one per distinct length (host lengths hl); launches k_znorm_batch
cudaError_t znormalize_dev(const double* in, const long long* off, const int* len, const int* hl, long long n,
                           double* out, const long long* ooff, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  std::vector<int2> leaves;
  std::vector<int> ops, plan_of((size_t)n);
  std::vector<int4> plans;
  std::vector<std::pair<int, int>> seen;  // (length, plan index)
  int max_leaves = 0;
  for (long long s = 0; s < n; ++s) {
    int idx = -1;
    for (auto& p : seen)
      if (p.first == hl[s]) idx = p.second;
    if (idx < 0) {
      // each plan on its own (its ops index its own leaves), then appended
      std::vector<int2> lv;
      std::vector<int> ov;
      np_plan_build(0, hl[s], lv, ov);
      plans.push_back(make_int4((int)leaves.size(), (int)lv.size(), (int)ops.size(), (int)ov.size()));
      leaves.insert(leaves.end(), lv.begin(), lv.end());
      ops.insert(ops.end(), ov.begin(), ov.end());
      max_leaves = std::max(max_leaves, (int)lv.size());
      idx = (int)plans.size() - 1;
      seen.push_back({hl[s], idx});
    }
    plan_of[(size_t)s] = idx;
  }
  const size_t smem = sizeof(double) * (size_t)(max_leaves + 16);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  void* buf = nullptr;
  const size_t bl = sizeof(int2) * leaves.size(), bo = sizeof(int) * ops.size(), bp = sizeof(int4) * plans.size(),
               bq = sizeof(int) * plan_of.size();
  cudaError_t e = cudaMallocAsync(&buf, bl + bo + bp + bq + 64, st);
  if (e != cudaSuccess) return e;
  char* b = (char*)buf;
  int4* dplans = (int4*)b;
  int2* dleaves = (int2*)(b + bp);
  int* dops = (int*)(b + bp + bl);
  int* dof = (int*)(b + bp + bl + bo);
  if ((e = cudaMemcpyAsync(dplans, plans.data(), bp, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
      (e = cudaMemcpyAsync(dleaves, leaves.data(), bl, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
      (e = cudaMemcpyAsync(dops, ops.data(), bo, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
      (e = cudaMemcpyAsync(dof, plan_of.data(), bq, cudaMemcpyHostToDevice, st)) != cudaSuccess) {
    cudaFreeAsync(buf, st);
    return e;
  }
  if (smem > 48 * 1024) cudaFuncSetAttribute((const void*)k_znorm_batch, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
  const unsigned blocks = (unsigned)std::min<long long>(n, 148LL * 32);
  k_znorm_batch<<<blocks, 32, smem, st>>>(in, off, len, n, out, ooff, dleaves, dops, dplans, dof);
  e = cudaGetLastError();
  // the host vectors above were copied by stream-ordered memcpys from pageable memory, which
  // return only after the source is consumed; the plan buffer is freed in stream order
  cudaFreeAsync(buf, st);
  return e;
}

}  // namespace ekb

// ---- UCR text parsing (host) ---------------------------------------------------------
namespace {

// Python's str.isspace for ASCII (str.strip / float() trim these)
inline bool py_space(unsigned char c) {
  return c == ' ' || (c >= '\t' && c <= '\r') || (c >= 0x1c && c <= 0x1f);
}

// The decimal subset of Python's float(): [ws] [+-] (d+ [. d*] | . d+) [(e|E) [+-] d+] [ws].
// Anything else (underscores, inf / nan words, non-ASCII digits, ...) is left to the
// reference loader, as is a value that overflows to +-inf.  strtod (correctly rounded in
// the C locale) then gives Python's value.
bool parse_number(const char* p, long long n, double* out) {
  long long a = 0, b = n;
  while (a < b && py_space((unsigned char)p[a])) ++a;
  while (b > a && py_space((unsigned char)p[b - 1])) --b;
  if (b - a <= 0 || b - a > 400) return false;
  long long k = a;
  if (p[k] == '+' || p[k] == '-') ++k;
  long long digits = 0;
  while (k < b && p[k] >= '0' && p[k] <= '9') ++k, ++digits;
  if (k < b && p[k] == '.') {
    ++k;
    while (k < b && p[k] >= '0' && p[k] <= '9') ++k, ++digits;
  }
  if (digits == 0) return false;
  if (k < b && (p[k] == 'e' || p[k] == 'E')) {
    ++k;
    if (k < b && (p[k] == '+' || p[k] == '-')) ++k;
    long long ed = 0;
    while (k < b && p[k] >= '0' && p[k] <= '9') ++k, ++ed;
    if (ed == 0) return false;
  }
  if (k != b) return false;
  char buf[416];
  std::memcpy(buf, p + a, (size_t)(b - a));
  buf[b - a] = '\0';
  static locale_t c_loc = newlocale(LC_NUMERIC_MASK, "C", (locale_t)0);
  char* end = nullptr;
  const double v = c_loc ? strtod_l(buf, &end, c_loc) : strtod(buf, &end);
  if (end != buf + (b - a) || !std::isfinite(v)) return false;
  *out = v;
  return true;
}

}  // namespace

extern "C" int ek_parse_tsv(const char* text, int64_t len, int32_t sep, int64_t* n_series, int64_t* n_values,
                            int64_t* labels, int64_t* offsets, int64_t* lengths, double* values,
                            int64_t* bad_line) {
  if ((!text && len > 0) || len < 0 || !n_series || !n_values || sep <= 0 || sep > 127 || sep == '\n' ||
      sep == '\r')
    return -1;
  const bool fill = values != nullptr;
  if (fill && (!labels || !offsets || !lengths)) return -1;
  if (bad_line) *bad_line = 0;
  long long ns = 0, nv = 0, line = 0, i = 0;
  auto fallback = [&](long long ln) {
    if (bad_line) *bad_line = ln;
    *n_series = ns;
    *n_values = nv;
    return 1;
  };
  while (i < len) {
    // universal newlines (text-mode iteration): \n, \r\n and a lone \r all end a line
    long long e = i;
    while (e < len && text[e] != '\n' && text[e] != '\r') ++e;
    long long nxt = e;
    if (nxt < len) nxt += (text[nxt] == '\r' && nxt + 1 < len && text[nxt + 1] == '\n') ? 2 : 1;
    ++line;
    bool blank = true;
    for (long long k = i; k < e; ++k) {
      const unsigned char c = (unsigned char)text[k];
      if (c >= 0x80) return fallback(line);  // non-ASCII: the reference loader decides
      if (!py_space(c)) blank = false;
    }
    if (blank) {  // line.strip() is empty
      i = nxt;
      continue;
    }
    long long fstart = i, cnt = 0;
    int col = 0;
    for (long long k = i; k <= e; ++k) {
      if (k < e && text[k] != (char)sep) continue;
      ++col;
      double v;
      if (!parse_number(text + fstart, k - fstart, &v)) return fallback(line);
      if (col == 1) {
        if (!(std::fabs(v) < 9.2e18)) return fallback(line);  // int(label) beyond int64
        if (fill) labels[ns] = (int64_t)v;                     // truncation, as int(float)
      } else {
        if (fill) values[nv + cnt] = v;
        ++cnt;
      }
      fstart = k + 1;
    }
    if (col < 2) return fallback(line);  // "expected a label and at least one value"
    if (fill) {
      offsets[ns] = nv;
      lengths[ns] = cnt;
    }
    nv += cnt;
    ++ns;
    i = nxt;
  }
  *n_series = ns;
  *n_values = nv;
  return ns == 0 ? 1 : 0;  // an empty dataset: the reference's EmptyDatasetError
}
