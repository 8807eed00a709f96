// Latency microbenchmarks (one warp): dependent chains of mma.sync / shfl / fadd.
#include <cstdio>
#include <cstdint>
__global__ void k(float* out, long long* cyc, int n) {
  float c[4] = {threadIdx.x * 1e-3f, 0.f, 0.f, 0.f};
  uint32_t a[4] = {0x3f800000u, 0x3f800000u, 0x3f800000u, 0x3f800000u}, b0 = 0x3f000000u, b1 = 0x3f000000u;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  long long t1 = clock64();
  double d[2] = {threadIdx.x * 1e-3, 0.0};
  double da = 1.0, db = 0.5;
  for (int i = 0; i < n; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d[0]), "+d"(d[1]) : "d"(da), "d"(db));
  long long t2 = clock64();
  float x = c[0];
  for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
  long long t3 = clock64();
  float y = x;
  for (int i = 0; i < n; ++i) asm volatile("add.f32 %0, %0, %1;" : "+f"(y) : "f"(x));
  long long t4 = clock64();
  // independent HMMA throughput: 4 chains
  float e[4][4] = {};
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(e[u][0]), "+f"(e[u][1]), "+f"(e[u][2]), "+f"(e[u][3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  long long t5 = clock64();
  volatile __shared__ int flag;
  flag = 0;
  int z = 0;
  for (int i = 0; i < n; ++i) z += flag + z;
  long long t6 = clock64();
  out[threadIdx.x] = c[0] + c[1] + c[2] + c[3] + (float)d[0] + (float)d[1] + y + e[0][0] + e[1][1] + e[2][2] + e[3][3] + z;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 4096); cudaMallocManaged(&c, 64);
  int n = 1000;
  k<<<1, 32>>>(o, c, n); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, n); cudaDeviceSynchronize();
  const char* names[] = {"HMMA tf32 dep chain", "DMMA f64 dep chain", "SHFL+FADD dep", "FADD dep", "HMMA x4 indep (per mma)", "LDS volatile dep"};
  for (int i = 0; i < 6; ++i) printf("%-26s %.1f cycles\n", names[i], (double)c[i] / n / (i == 4 ? 4 : 1));
  return 0;
}
