// Cycles of the inner solver's MMA block (3 accumulator chains: 9 BF16 m16n8k16
// then 9 TF32 m16n8k8, as in one half-iteration) and of pure-type blocks.
#include <cstdio>
#include <cstdint>
#define BF(c, a, b)                                                                                         \
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};" \
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]))
#define TF(c, a, b)                                                                                         \
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};" \
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]))
__global__ void k(float* out, long long* cyc, int n, int mode) {
  float c0[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0}, c2[4] = {0, 0, 0, 0};
  uint32_t a[4] = {threadIdx.x, 1u, 2u, 3u}, b[2] = {5u, 7u};
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (mode == 0) {
#pragma unroll
      for (int kt = 0; kt < 3; ++kt) { BF(c0, a, b); BF(c1, a, b); BF(c2, a, b); }
#pragma unroll
      for (int kt = 0; kt < 3; ++kt) { TF(c0, a, b); TF(c1, a, b); TF(c2, a, b); }
    } else if (mode == 1) {
#pragma unroll
      for (int kt = 0; kt < 6; ++kt) { TF(c0, a, b); TF(c1, a, b); TF(c2, a, b); }
    } else if (mode == 2) {
#pragma unroll
      for (int kt = 0; kt < 6; ++kt) { BF(c0, a, b); BF(c1, a, b); BF(c2, a, b); }
    } else {
      // block, then a dependent feed of the results into the next block's A (the solver's loop)
#pragma unroll
      for (int kt = 0; kt < 3; ++kt) { BF(c0, a, b); BF(c1, a, b); BF(c2, a, b); }
#pragma unroll
      for (int kt = 0; kt < 3; ++kt) { TF(c0, a, b); TF(c1, a, b); TF(c2, a, b); }
      a[0] = __float_as_uint(c0[0] + c1[1]) & 0xffffe000u;
      a[1] = __float_as_uint(c2[2]);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[mode] = t1 - t0;
  out[threadIdx.x + 32 * mode] = c0[0] + c1[1] + c2[2] + c0[3];
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 64 * 8);
  const int n = 200;
  const char* names[4] = {"9 bf16 + 9 tf32 (3 chains)", "18 tf32 (3 chains)", "18 bf16 (3 chains)", "mixed + dependent A feed"};
  for (int rep = 0; rep < 2; ++rep)
    for (int m = 0; m < 4; ++m) k<<<1, 32>>>(o, c, n, m);
  long long h[4]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  for (int m = 0; m < 4; ++m) printf("%-32s %.1f cycles per block of 18\n", names[m], (double)h[m] / n);
  // two warps on one SMSP (warps 0 and 4 of a 5-warp block)
  for (int rep = 0; rep < 2; ++rep) k<<<1, 160>>>(o, c, n, 3);
  cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  printf("%-32s %.1f cycles per block of 18 (5 warps/SM)\n", names[3], (double)h[3] / n);
  return 0;
}
