// Dependent-issue latency of DMMA m8n8k4 (cycles, one warp): accumulator chain
// (D -> C of the next), operand chain (D -> A of the next) and DFMA / DADD for
// comparison.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a dmma_lat.cu -o dmma_lat
#include <cstdio>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
__global__ void k(double* out, long long* cyc, int n) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1e-3;
  double c[2] = {0.0, 0.0};
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) dmma(c, a, b);
  long long t1 = clock64();
  cyc[0] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {  // D -> A
    double d[2] = {0.0, 0.0};
    dmma(d, a, b);
    a = d[0];
  }
  t1 = clock64();
  cyc[1] = t1 - t0;
  double x = a;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 1.0000001, 1e-12);
  t1 = clock64();
  cyc[2] = t1 - t0;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x + 1e-12;
  t1 = clock64();
  cyc[3] = t1 - t0;
  // 3 independent accumulator chains interleaved (the solver's n-tiles)
  double c0[2] = {0, 0}, c1[2] = {0, 0}, c2[2] = {0, 0};
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    dmma(c0, a, b);
    dmma(c1, a, b);
    dmma(c2, a, b);
  }
  t1 = clock64();
  cyc[4] = t1 - t0;
  out[threadIdx.x] = c[0] + c[1] + x + c0[0] + c1[0] + c2[0];
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 64);
  const int n = 2000;
  k<<<1, 32>>>(o, c, n);
  k<<<1, 32>>>(o, c, n);
  long long h[8]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
  const char* nm[5] = {"dmma D->C chain", "dmma D->A chain", "dfma chain", "dadd chain", "3 interleaved dmma chains (per triple)"};
  for (int i = 0; i < 5; ++i) printf("%-40s %.1f cyc/iter\n", nm[i], (double)h[i] / n);
  return 0;
}
