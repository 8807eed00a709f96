// Development aid: per-phase timing of the fused CholeskyQR2 (qr.cu k_cholqr2)
// on two cfg2-shaped panels (k = 30, 10^4 rows each), from CTA 0's globaltimer
// stamps.  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a
//   -I../../paper_1812_04315_b200/csrc -I../../include qr_phases.cu -o qr_phases
#include "../../paper_1812_04315_b200/csrc/qr.cu"
#include <cstdio>
#include <vector>
namespace nenmf {
unsigned long long launch_counter_add(unsigned long long) { return 0; }
cudaError_t set_smem_attr(const void* fn, size_t bytes) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}
}
using namespace nenmf;
int main(int argc, char** argv) {
  const int k = argc > 1 ? atoi(argv[1]) : 30;
  const int64_t rows = argc > 2 ? atol(argv[2]) : 10000;
  std::vector<float> h((size_t)k * rows);
  uint64_t x = 88172645463325252ull;
  for (auto& v : h) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    v = (float)((x >> 11) * (1.0 / 9007199254740992.0)) - 0.5f;
  }
  float *p0, *p1;
  cudaMalloc(&p0, h.size() * 4);
  cudaMalloc(&p1, h.size() * 4);
  nenmf_device_status* st;
  cudaMalloc(&st, 64);
  cudaMemset(st, 0, 64);
  size_t wsb = 64 << 20;
  void* ws;
  cudaMalloc(&ws, wsb);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(p0, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(p1, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    Arena a(ws, wsb);
    cudaEventRecord(e0);
    int rc = orthonormalize_pair<float>(a, p0, rows, p1, rows, k, st, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long t[24];
    cudaMemcpyFromSymbol(t, g_qr_phase, sizeof(t));
    printf("rc %d  %.1f us | ", rc, ms * 1e3);
    const char* names[11] = {"A gram", "bar1", "B reduce", "bar2", "C factor", "C trsm+gram", "bar3", "D reduce", "bar4", "E factor", "E trsm"};
    for (int i = 0; i < 11; ++i) printf("%s %.1f  ", names[i], (t[i + 1] - t[i]) * 1e-3);
    printf("| A.dmma %.1f A.acc %.1f (stamps 12/13 are from phase C's gram) C.pre-trsm %.1f C.trsm %.1f ",
           (t[12] - t[0]) * 1e-3, (t[13] - t[12]) * 1e-3, (t[14] - t[4]) * 1e-3, (t[15] - t[14]) * 1e-3);
    long long cy[24];
    cudaMemcpyFromSymbol(cy, g_qr_cyc, sizeof(cy));
    printf("| SM MHz over the kernel %.0f ", (double)(cy[11] - cy[0]) / (double)(t[11] - t[0]) * 1e3);
    printf("| err %s\n", cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
