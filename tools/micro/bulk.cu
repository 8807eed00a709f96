// Micro-benchmark: HBM read throughput of a persistent 1-D bulk-copy stream
// (cp.async.bulk -> smem ring of NST stages, consumer releases immediately).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk bulk.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(su(b)), "r"(ph) : "memory");
}
template <int NST>
__global__ void __launch_bounds__(64, 1) k(const uint8_t* src, int64_t per_cta, int stage_bytes, int pieces, int order) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int64_t nt = per_cta / stage_bytes;
  if (tid == 0) {
    for (int64_t t = 0; t < nt; ++t) {
      int s = t % NST;
      wait(&empty[s], ((t / NST) & 1) ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(stage_bytes));
      // order 0: each CTA streams its own contiguous region; 1: interleaved (tile t of CTA b at (t*grid+b))
      const uint8_t* g = order == 0 ? src + (int64_t)blockIdx.x * per_cta + t * stage_bytes
                                    : src + (t * gridDim.x + blockIdx.x) * (int64_t)stage_bytes;
      int pb = stage_bytes / pieces;
      for (int p = 0; p < pieces; ++p)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su(sm + (size_t)s * stage_bytes + p * pb)), "l"(g + p * pb), "r"(pb), "r"(su(&full[s])) : "memory");
    }
  } else if (tid == 32) {
    for (int64_t t = 0; t < nt; ++t) {
      int s = t % NST;
      wait(&full[s], (t / NST) & 1);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
    }
  }
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t total = 400ll << 20;
  uint8_t* buf; cudaMalloc(&buf, total + (64 << 20));
  cudaMemset(buf, 1, total);
  uint8_t* flush; cudaMalloc(&flush, 256 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int stages[] = {2, 3, 4, 6, 8};
  int sizes[] = {16384, 32768, 65536, 81920, 98304};
  for (int order = 0; order < 2; ++order)
  for (int sz : sizes) for (int nst : stages) for (int pieces : {1, 4, 32, 128}) {
    if (pieces > 4 && !(sz == 65536 && nst == 3)) continue;
    if ((size_t)nst * sz > 220 * 1024) continue;
    int grid = sms;
    int64_t per_cta = total / grid / sz * sz;
    size_t smem = (size_t)nst * sz;
    void (*f)(const uint8_t*, int64_t, int, int, int) = nst == 2 ? k<2> : nst == 3 ? k<3> : nst == 4 ? k<4> : nst == 6 ? k<6> : k<8>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float best = 1e9;
    for (int r = 0; r < 4; ++r) {
      cudaMemsetAsync(flush, r, 256 << 20);
      cudaEventRecord(a);
      f<<<grid, 64, smem>>>(buf, per_cta, sz, pieces, order);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("order %d stage %6d B x %d  pieces %d : %7.1f GB/s %s\n", order, sz, nst, pieces,
           (double)per_cta * grid / best / 1e6, e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
