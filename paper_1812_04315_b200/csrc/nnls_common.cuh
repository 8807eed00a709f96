// Shared declarations of the persistent NNLS solver (nnls.cu + nnls_k_*.cu).
#pragma once
#include "common.cuh"
#include <climits>
#include <cstdlib>

namespace nenmf {

// -------------------------------------------------------------- helpers ----
__device__ __forceinline__ double alpha_next_d(double a) {
  // (1 + sqrt(4*a*a + 1)) / 2 with NumPy's rounding sequence (nnls.py:68-69)
  return __ddiv_rn(__dadd_rn(1.0, sqrt(__dadd_rn(__dmul_rn(__dmul_rn(4.0, a), a), 1.0))), 2.0);
}

__device__ __forceinline__ bool finite_d(double x) { return isfinite(x); }

__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// a grid that stops making progress for this long aborts with NENMF_ERR_CUDA
// (iteration -2) instead of hanging the device
constexpr unsigned long long NN_WATCHDOG_NS = 5000000000ull;

// optional per-iteration timeline (NENMF_NNLS_TRACE=1): [0] CTA 0 compute
// warp 0 posts, [1] CTA 0 publishes, [2] CTA 0 resolves, [3] last CTA posts
constexpr int NN_TRACE_LEN = 4096;

constexpr int NW_WIN = 32;             // iterations per window
constexpr int NW_FLIGHT = 4;           // windows computed ahead of decisions
constexpr int NW_SNAP = NW_FLIGHT + 2; // rotating snapshot slots (+1 best slot)
constexpr int NW_SLOTS = NW_FLIGHT + 3;// window-record ring
constexpr int NW_MAXW = 16;            // warps per CTA incl. resolver
constexpr int NW_PPD = (NW_FLIGHT + 2) * NW_WIN;  // per-iteration warp-sum ring

struct __align__(16) WinRec {
  double v[NW_WIN][3];     // per iteration: ||PG||^2, <F,g>, <F,V>
  unsigned long long tag;  // window index + 1 once v is valid
  unsigned long long pad;
};

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// ------------------------------------------------------------------- plan
struct NnlsPlan {
  int grid = 1, threads = 64, tpc = 1, rmax = 1, ldS = 0, ldW = 0;
  int64_t cpb = 1;
  bool smem_state = false;
  size_t smem = 0;
};

template <typename T>
static NnlsPlan plan_nnls(int64_t p, int64_t c) {
  NnlsPlan pl;
  int sms = sm_count();
  if (sms <= 0) sms = 148;
  pl.grid = (int)imax(1, imin(sms, cdiv(c, 32)));
  if (const char* e = getenv("NENMF_NNLS_GRID")) pl.grid = (int)imax(1, imin(sms, atoi(e)));
  pl.cpb = cdiv(c, pl.grid);
  // TPC: smallest power of two with ceil(p / TPC) <= 8
  int tpc = 1;
  while (cdiv(p, tpc) > 8) tpc *= 2;
  pl.tpc = tpc;
  pl.rmax = (int)cdiv(p, tpc);
  if (tpc > 1 && pl.rmax < 5) pl.rmax = 5;  // instantiated shapes: TPC=1 x 1..8, TPC>1 x 5..8
  const int vw = 16 / (int)sizeof(T);
  pl.ldW = (int)(cdiv(tpc * pl.rmax, vw) * vw);
  int64_t nct = imin(32 * (NW_MAXW - 1), cdiv(pl.cpb * tpc, 32) * 32);
  pl.threads = (int)nct + 32;
  size_t base = (((size_t)tpc * pl.rmax * pl.ldW * sizeof(T) + 15) / 16) * 16 +
                (size_t)NW_PPD * NW_MAXW * 3 * sizeof(double);
  // ldS: per-column block stride (5 buffers of PMV entries), padded so that
  // the 16-byte loads of the warp's columns fall into distinct bank groups
  const int pmv = (int)(cdiv(tpc * pl.rmax, vw) * vw);
  int64_t ld = 5 * pmv;
  if (sizeof(T) == 4) {
    while (ld % 32 != 4) ++ld;
  } else {
    while (ld % 16 != 2) ++ld;
  }
  size_t st_bytes = (size_t)pl.cpb * ld * sizeof(T);
  if (base + st_bytes <= 200 * 1024) {
    pl.smem_state = true;
    pl.ldS = (int)ld;
    pl.smem = base + st_bytes;
  } else {
    pl.smem = base;
  }
  return pl;
}


template <typename T, int TPC>
int launch_nnls_tpc(const NnlsPlan& pl, const T* W, const T* V, const T* F0, T* Fout, T* snaps, double* salpha,
                    T* gstate, int p, int64_t c, const double* Lptr, int max_iter, double grad_tol, WinRec* recs,
                    WinRec* results, nenmf_device_status* st, unsigned long long* tracebuf, cudaStream_t s);

}  // namespace nenmf
