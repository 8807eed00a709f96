// Dependent-chain latency of the legacy warp MMAs and a few ALU ops on sm_100a
// (development aid for the inner solver's per-iteration critical path).
#include <cstdio>
#include <cstdint>
__global__ void k(float* out, long long* cyc, int n) {
  float c[4] = {0.f, 0.f, 0.f, 0.f};
  uint32_t a[4] = {threadIdx.x, 1u, 2u, 3u}, b[2] = {5u, 7u};
  float x = threadIdx.x * 1e-3f;
  long long t0, t1;
  // TF32 m16n8k8 chain
  t0 = clock64();
  for (int i = 0; i < n; ++i)
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  // BF16 m16n8k16 chain
  t0 = clock64();
  for (int i = 0; i < n; ++i)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
  // TF32 chain through the A operand (accumulator -> A, like the solver's iteration)
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    a[0] = __float_as_uint(c[0]) & 0xffffe000u;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
  // 3 independent accumulators interleaved (throughput of the chain pattern)
  float d[4] = {0, 0, 0, 0}, e[4] = {0, 0, 0, 0};
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(e[0]), "+f"(e[1]), "+f"(e[2]), "+f"(e[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = t1 - t0;
  // FFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fmaf(x, 0.999f, 1e-3f);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = t1 - t0;
  // SHFL chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = t1 - t0;
  // DMMA f64 m8n8k4 chain
  double dc[2] = {0, 0}, da = threadIdx.x, db = 1.0;
  t0 = clock64();
  for (int i = 0; i < n; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(dc[0]), "+d"(dc[1]) : "d"(da), "d"(db));
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = t1 - t0;
  out[threadIdx.x] = c[0] + c[1] + c[2] + c[3] + d[0] + e[1] + x + (float)dc[0] + (float)dc[1];
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 64 * 8);
  const int n = 1000;
  k<<<1, 32>>>(o, c, n);
  k<<<1, 32>>>(o, c, n);
  long long h[7]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  const char* names[7] = {"tf32 m16n8k8 acc chain", "bf16 m16n8k16 acc chain", "tf32 acc->A chain (+LOP)",
                          "3 interleaved tf32 chains (per step)", "ffma chain", "shfl+fadd chain", "dmma m8n8k4 chain"};
  for (int i = 0; i < 7; ++i) printf("%-40s %.1f cycles\n", names[i], (double)h[i] / n);
  return 0;
}
