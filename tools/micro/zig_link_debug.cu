// Debug aid: runs the device draw pipeline of rng.cu on cfg2's draw count and
// reports how many chunks the parallel link rejects (and where).
#include "../../paper_1812_04315_b200/csrc/rng.cu"
#include <cstdio>
namespace nenmf { unsigned long long launch_counter_add(unsigned long long) { return 0; } }
#include <vector>
using namespace nenmf;
using namespace nenmf::zig;
int main() {
  std::vector<uint64_t> tab(768);
  FILE* f = fopen("tools/micro/zig_tables.bin", "rb");
  if (fread(tab.data(), 8, 768, f) != 768) return 1;
  fclose(f);
  void* dT;
  cudaMalloc(&dT, 768 * 8);
  cudaMemcpy(dT, tab.data(), 768 * 8, cudaMemcpyHostToDevice);
  const int64_t need = 600000;
  int S = 64;
  const int64_t nchunks = (int64_t)((double)need * 1.03 / S) + 8;
  ChunkScan* sc;
  cudaMalloc(&sc, nchunks * sizeof(ChunkScan));
  // arbitrary PCG64 state
  uint64_t s_lo = 0x123456789abcdefull, s_hi = 0xfedcba987654321ull, i_lo = 0x1111111111111111ull | 1, i_hi = 0x2222;
  k_zig_scan<<<(unsigned)((nchunks + 63) / 64), 64>>>((const Tables*)dT, s_lo, s_hi, i_lo, i_hi, nchunks, S, sc);
  std::vector<ChunkScan> h(nchunks);
  cudaMemcpy(h.data(), sc, nchunks * sizeof(ChunkScan), cudaMemcpyDeviceToHost);
  int bad = 0, maxexit = 0;
  for (int64_t c = 1; c < nchunks; ++c) {
    const int e = h[c - 1].exit;
    if (e > maxexit) maxexit = e;
    if (e != 0 && !(e < 64 && ((h[c].mask >> e) & 1ull))) {
      if (bad < 5) printf("bad chunk %ld: e=%d mask=%016llx count=%d exit=%d\n", (long)c, e, h[c].mask, h[c].count, h[c].exit);
      ++bad;
    }
  }
  printf("nchunks %ld bad %d maxexit %d err %s\n", (long)nchunks, bad, maxexit, cudaGetErrorString(cudaGetLastError()));
  for (int c = 0; c < 4; ++c) printf("chunk %d mask %016llx count %d exit %d\n", c, h[c].mask, h[c].count, h[c].exit);
}
