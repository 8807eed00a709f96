// FP64 compute peaks of this B200 (sm_100a): the DMMA tensor pipe
// (mma.sync m8n8k4 f64, 512 flops per warp instruction) and the CUDA-core
// DFMA pipe, all SMs, independent accumulator chains, CUDA-event timing.
// Prints one JSON line; bench.py's fp64 roofline divides by the DMMA figure
// (stored in profiles/fp64_peak.json).  nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a fp64_peak.cu -o fp64_peak
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int CH = 8;  // independent chains per warp

__global__ void __launch_bounds__(256) k_dmma(double* out, int iters) {
  double c[CH][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int j = 0; j < CH; ++j) c[j][0] = c[j][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters) {
  double c[CH];
  const double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
#pragma unroll
  for (int j = 0; j < CH; ++j) c[j] = j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j) c[j] = fma(c[j], b, a);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += c[j];
  if (s == 12345.678) out[0] = s;
}

// distinct operand registers per chain (a real kernel's DMMAs do not share operands)
__global__ void __launch_bounds__(256) k_dmma_var(double* out, int iters) {
  double c[CH][2], a[CH], b[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    c[j][0] = c[j][1] = 0.0;
    a[j] = 1.0 + (threadIdx.x + j) * 1e-9;
    b[j] = 1.0 - (threadIdx.x + 3 * j) * 1e-9;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1])
                   : "d"(a[j]), "d"(b[j]));
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[0] = s;
}

// operands from shared memory, the X-pass pattern: per k-step 2 X fragments and
// 4 skinny fragments (LDS.64 each) feed 8 DMMAs; 16 k-steps per "tile"
__global__ void __launch_bounds__(256) k_dmma_lds(double* out, int tiles) {
  __shared__ double xs[64 * 68 + 24 * 68];
  for (int i = threadIdx.x; i < 88 * 68; i += blockDim.x) xs[i] = 1.0 + i * 1e-9;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = (threadIdx.x >> 5) & 3, gq = lane >> 2, tq = lane & 3;
  double c[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int b = 0; b < 4; ++b) c[i][b][0] = c[i][b][1] = 0.0;
  const double* x0 = xs + (16 * w + gq) * 68 + tq;
  const double* a0 = xs + 64 * 68 + gq * 68 + tq;
  for (int t = 0; t < tiles; ++t) {
#pragma unroll
    for (int ks = 0; ks < 16; ++ks) {
      const double xa0 = x0[4 * ks], xa1 = x0[8 * 68 + 4 * ks];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const double sk = a0[(8 * b % 24) * 68 + 4 * ks];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[0][b][0]), "+d"(c[0][b][1])
                     : "d"(xa0), "d"(sk));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[1][b][0]), "+d"(c[1][b][1])
                     : "d"(xa1), "d"(sk));
      }
    }
    asm volatile("" ::: "memory");
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int b = 0; b < 4; ++b) s += c[i][b][0] + c[i][b][1];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
static double time_kernel(K kern, int blocks, int threads, double* out, int iters, double flops_per_iter_warp,
                          cudaEvent_t e0, cudaEvent_t e1) {
  double best = 0;
  for (int rep = 0; rep < 4; ++rep) {
    kern<<<blocks, threads>>>(out, 10);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = (double)blocks * (threads / 32) * iters * flops_per_iter_warp;
    if (fl / (ms * 1e-3) / 1e12 > best) best = fl / (ms * 1e-3) / 1e12;
  }
  return best;
}

static double run_dmma(int blocks, int threads, double* out, cudaEvent_t e0, cudaEvent_t e1) {
  double best = 0;
  for (int rep = 0; rep < 4; ++rep) {
    const int iters = 20000;
    k_dmma<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = (double)blocks * (threads / 32) * iters * CH * 512.0;
    if (fl / (ms * 1e-3) / 1e12 > best) best = fl / (ms * 1e-3) / 1e12;
  }
  return best;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 256;
  double best_mma = 0, best_fma = 0;
  for (int rep = 0; rep < 6; ++rep) {
    const int iters = 20000;
    k_dmma<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = (double)blocks * (threads / 32) * iters * CH * 512.0;
    if (fl / (ms * 1e-3) / 1e12 > best_mma) best_mma = fl / (ms * 1e-3) / 1e12;
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double ff = (double)blocks * threads * iters * CH * 2.0;
    if (ff / (ms * 1e-3) / 1e12 > best_fma) best_fma = ff / (ms * 1e-3) / 1e12;
  }
  if (getenv("FP64_VAR") != nullptr) {
    fprintf(stderr, "distinct operands, %d CTAs x 256: %.2f TF/s\n", blocks,
            time_kernel(k_dmma_var, blocks, 256, out, 20000, CH * 512.0, e0, e1));
    for (int wps : {4, 8, 16})
      fprintf(stderr, "distinct operands, %d warps/SM: %.2f TF/s\n", wps,
              time_kernel(k_dmma_var, sms * (wps <= 8 ? 1 : wps / 8), wps <= 8 ? 32 * wps : 256, out, 20000, CH * 512.0,
                          e0, e1));
    for (int wps : {4, 8, 16})
      fprintf(stderr, "LDS-fed X-pass pattern, %d warps/SM: %.2f TF/s\n", wps,
              time_kernel(k_dmma_lds, sms * (wps <= 8 ? 1 : wps / 8), wps <= 8 ? 32 * wps : 256, out, 2000,
                          128 * 512.0, e0, e1));
  }
  if (getenv("FP64_OCC") != nullptr) {
    for (int wps : {4, 8, 16, 32}) {
      const int threads = wps <= 8 ? 32 * wps : 256, per = wps <= 8 ? 1 : wps / 8;
      fprintf(stderr, "warps/SM %2d: %.2f TF/s\n", wps, run_dmma(sms * per, threads, out, e0, e1));
    }
  }
  printf("{\"fp64_dmma_tflops\": %.3f, \"fp64_dfma_tflops\": %.3f, \"sms\": %d, \"clock_khz\": %d, "
         "\"how\": \"tools/micro/fp64_peak.cu: %d CTAs x 256 threads, %d independent chains per warp, best of 6, "
         "CUDA events\", \"err\": \"%s\"}\n",
         best_mma, best_fma, sms, clk, blocks, CH, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
