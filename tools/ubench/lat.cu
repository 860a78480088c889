// Dependent-chain latencies on sm_100a (clock64 around 256-long chains, one warp).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  double x = a, y = b;
  long long t0, t1;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
  t1 = clock64(); cyc[0] = t1 - t0; out[0] = x;
  // DMUL chain
  x = a; t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dmul_rn(x, y);
  t1 = clock64(); cyc[1] = t1 - t0; out[1] = x;
  // min chain: x = (y < x) ? y : x  with y dependent on x
  x = a; t0 = clock64();
  for (int i = 0; i < n; ++i) { double z = __dadd_rn(x, y); x = (z < x) ? z : x; x = __dadd_rn(x, b); }
  t1 = clock64(); cyc[2] = t1 - t0; out[2] = x;
  // shuffle chain (64-bit)
  x = a; t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffff, x, 1);
  t1 = clock64(); cyc[3] = t1 - t0; out[3] = x;
  // float min chain
  float fx = (float)a, fy = (float)b; t0 = clock64();
  for (int i = 0; i < n; ++i) { float z = __fadd_rn(fx, fy); fx = fminf(z, fx); fx = __fadd_rn(fx, fy); }
  t1 = clock64(); cyc[4] = t1 - t0; out[4] = fx;
  // shuffle 32-bit chain
  int ix = (int)a; t0 = clock64();
  for (int i = 0; i < n; ++i) ix = __shfl_xor_sync(0xffffffff, ix, 1);
  t1 = clock64(); cyc[5] = t1 - t0; out[5] = ix;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64); cudaMalloc(&c, 64);
  const int n = 1024;
  k<<<1, 32>>>(o, c, 1.0, 1e-9, n); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 1.0, 1e-9, n); cudaDeviceSynchronize();
  long long h[6]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  const char* nm[6] = {"DADD", "DMUL", "DADD+DMIN(DSETP+2FSEL)+DADD", "SHFL64", "FADD+FMNMX+FADD", "SHFL32"};
  for (int i = 0; i < 6; ++i) printf("%-30s %.1f cyc/iter\n", nm[i], (double)h[i] / n);
  return 0;
}
