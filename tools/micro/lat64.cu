// Dependent-chain latencies (cycles) of the FP64 operations on the critical
// path of the small factorizations (development aid).
#include <cstdio>
__global__ void k(double* out, long long* cyc, int n, double seed) {
  double x = seed + threadIdx.x * 1e-9, y = 1.0000001;
  long long t0, t1;
  __shared__ double sm[64];
  sm[threadIdx.x] = x;
  __syncwarp();
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-12);
  t1 = clock64();
  cyc[0] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x) + 0.5;
  t1 = clock64();
  cyc[1] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / x + 0.5;
  t1 = clock64();
  cyc[2] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) * 1.0000001;
  t1 = clock64();
  cyc[3] = t1 - t0;
  t0 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < n; ++i) { x = sm[idx & 31] + x; idx = (int)x & 31; }
  t1 = clock64();
  cyc[4] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x) + 0.5;
  t1 = clock64();
  cyc[5] = t1 - t0;
  t0 = clock64();
  unsigned u = (unsigned)x;
  for (int i = 0; i < n; ++i) u = __reduce_max_sync(0xffffffffu, u + threadIdx.x);
  t1 = clock64();
  cyc[6] = t1 - t0;
  out[threadIdx.x] = x + u;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 64);
  const int n = 1000;
  k<<<1, 32>>>(o, c, n, 1.5);
  k<<<1, 32>>>(o, c, n, 1.5);
  long long h[8]; cudaMemcpy(h, c, 56, cudaMemcpyDeviceToHost);
  const char* nm[7] = {"dfma", "sqrt+dadd", "rcp+dadd", "shfl.f64+dmul", "lds.64+dadd+cvt", "rsqrt+dadd", "redux.max"};
  for (int i = 0; i < 7; ++i) printf("%-18s %.1f cyc/iter\n", nm[i], (double)h[i] / n);
}
