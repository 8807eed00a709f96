// Pure compute chain of one solver iteration (fp32, NT=3, 16 columns per warp),
// no resolver: cycles per iteration for 1..8 warps per CTA.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t hi_(float x) { return __float_as_uint(x) & 0xffffe000u; }
__device__ __forceinline__ uint32_t lo_(float x, uint32_t h) { return __float_as_uint(x - __uint_as_float(h)); }
__device__ __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <int NT, int MODE>
__global__ void k(const float* W, float* out, long long* cyc, int iters) {
  constexpr int NE = 4 * NT;
  const int lane = threadIdx.x & 31, gq = lane >> 2, tq = lane & 3;
  __shared__ double pp[64 * 16 * 3];
  uint32_t bhi[NT][NT][2], blo[NT][NT][2];
  for (int kt = 0; kt < NT; ++kt)
    for (int nt = 0; nt < NT; ++nt)
      for (int h = 0; h < 2; ++h) {
        float w = W[(8 * nt + gq) * 24 + 8 * kt + 2 * tq + h];
        bhi[kt][nt][h] = hi_(w);
        blo[kt][nt][h] = lo_(w, bhi[kt][nt][h]);
      }
  float ua[NE], ub[NE], fa[NE], vv[NE];
  for (int e = 0; e < NE; ++e) { ua[e] = 0.01f * (e + lane); ub[e] = ua[e]; vv[e] = 0.5f; fa[e] = 0; }
  const float rnegL = -0.1f;
  float ps0 = 0, ps1 = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float w = 0.5f + 1e-6f * it;
    float fo[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) fo[e] = fmaxf(fmaf(ua[e] - ub[e], w, ua[e]), 0.f);
    float g[NE];
    uint32_t ahi[NT][4], alo[NT][4];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const float v4[4] = {fo[4 * t], fo[4 * t + 2], fo[4 * t + 1], fo[4 * t + 3]};
#pragma unroll
      for (int r = 0; r < 4; ++r) { ahi[t][r] = hi_(v4[r]); alo[t][r] = lo_(v4[r], ahi[t][r]); }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      float cc[4] = {-vv[4 * nt], -vv[4 * nt + 1], -vv[4 * nt + 2], -vv[4 * nt + 3]};
      if (MODE != 2) {
#pragma unroll
        for (int kt = 0; kt < NT; ++kt) {
          mma(cc, alo[kt], bhi[kt][nt][0], bhi[kt][nt][1]);
          mma(cc, ahi[kt], blo[kt][nt][0], blo[kt][nt][1]);
        }
      }
#pragma unroll
      for (int kt = 0; kt < NT; ++kt) mma(cc, ahi[kt], bhi[kt][nt][0], bhi[kt][nt][1]);
#pragma unroll
      for (int r = 0; r < 4; ++r) g[4 * nt + r] = cc[r];
    }
    if (MODE != 1) {
      float s0 = ps0, s1 = ps1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) { s0 += __shfl_xor_sync(0xffffffffu, s0, o); s1 += __shfl_xor_sync(0xffffffffu, s1, o); }
      if (lane == 0) { double* q = pp + ((it % 64) * 16 + (threadIdx.x >> 5)) * 3; q[0] = s0; q[1] = s1; }
    }
    ps0 = ps1 = 0;
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      ub[e] = fmaf(g[e], rnegL, fo[e]);
      const float pgv = fo[e] > 0.f ? g[e] : fminf(g[e], 0.f);
      ps0 = fmaf(pgv, pgv, ps0);
      ps1 = fmaf(fo[e], g[e] - vv[e], ps1);
    }
#pragma unroll
    for (int e = 0; e < NE; ++e) { float t = ua[e]; ua[e] = ub[e]; ub[e] = t; }
  }
  long long t1 = clock64();
  float acc = ps0 + ps1;
  for (int e = 0; e < NE; ++e) acc += ua[e];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + pp[lane];
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int NT, int MODE>
void run(const char* name, float* W, float* o, long long* c) {
  int iters = 2000;
  for (int nw : {1, 2, 4, 5, 8}) {
    k<NT, MODE><<<148, 32 * nw>>>(W, o, c, iters); cudaDeviceSynchronize();
    k<NT, MODE><<<148, 32 * nw>>>(W, o, c, iters); cudaDeviceSynchronize();
    printf("%-22s warps/CTA %d: %.0f cycles/iter\n", name, nw, (double)*c / iters);
  }
}
int main() {
  float *W, *o; long long* c;
  cudaMalloc(&W, 24 * 24 * 4); cudaMemset(W, 0, 24 * 24 * 4); cudaMalloc(&o, 148 * 512 * 4); cudaMallocManaged(&c, 8);
  run<3, 0>("full (3xTF32+post)", W, o, c);
  run<3, 1>("no post/shuffles", W, o, c);
  run<3, 2>("1xTF32 + post", W, o, c);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
