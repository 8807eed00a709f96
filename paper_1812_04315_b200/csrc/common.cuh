// Shared device/host helpers of libnenmf_b200 (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <math.h>

#include "../../include/nenmf_b200.h"

namespace nenmf {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// host-side error plumbing
// ---------------------------------------------------------------------------
#define NENMF_CUDA_TRY(expr)                                   \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return NENMF_ERR_CUDA;              \
  } while (0)

// every kernel launch site is followed by NENMF_LAUNCH_CHECK(), which also
// bumps a diagnostic launch counter (nenmf_launch_count, read by bench.py)
unsigned long long launch_counter_add(unsigned long long n);
#define NENMF_LAUNCH_CHECK()            \
  do {                                  \
    nenmf::launch_counter_add(1);       \
    NENMF_CUDA_TRY(cudaGetLastError()); \
  } while (0)

#define NENMF_TRY(expr)                                        \
  do {                                                         \
    int _s = (expr);                                           \
    if (_s != NENMF_OK) return _s;                             \
  } while (0)

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Bump allocator over a caller-provided workspace.  Sizing functions run the
// same carve sequence with base == nullptr to obtain the byte count.
struct Arena {
  char* base;
  size_t cap;
  size_t used = 0;
  bool ok = true;
  Arena(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <typename T>
  T* take(size_t count) {
    size_t off = align_up(used);
    used = off + align_up(count * sizeof(T));
    if (base == nullptr) return nullptr;
    if (used > cap) { ok = false; return nullptr; }
    return reinterpret_cast<T*>(base + off);
  }
};

inline int sm_count() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return sms;
}

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size
// (the call is expensive relative to a launch; results are cached)
cudaError_t set_smem_attr(const void* fn, size_t bytes);
template <typename K>
inline cudaError_t set_smem(K* fn, size_t bytes) {
  return set_smem_attr(reinterpret_cast<const void*>(fn), bytes);
}
__host__ __device__ __forceinline__ int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------

// IEEE ops without FMA contraction, matching NumPy's separately rounded ufuncs.
__device__ __forceinline__ double op_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float op_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double op_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float op_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double op_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float op_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double op_div(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float op_div(float a, float b) { return __fdiv_rn(a, b); }

__device__ __forceinline__ double fma_acc(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float fma_acc(float a, float b, float c) { return fmaf(a, b, c); }

// np.maximum(x, 0) keeping NaN (numpy propagates NaN; fmax would not)
template <typename T>
__device__ __forceinline__ T relu_nan(T x) { return (x >= T(0) || x != x) ? x : T(0); }
// max(x, 0) propagating NaN in one instruction (the sign of a zero may differ)
__device__ __forceinline__ float relu_nan_fast(float x) {
  float r;
  asm("max.NaN.f32 %0, %1, 0f00000000;" : "=f"(r) : "f"(x));
  return r;
}
// FP64: the same by the sign bit on the integer pipe (the FP64 pipe is the
// bound of the FP64 solver; DSETP compares ran on it).  A negative-signed NaN
// becomes 0 here, but a NaN only reaches this point from an iterate whose
// sums were already non-finite (the failure is decided there).
__device__ __forceinline__ double relu_nan_fast(double x) {
  const int hi = __double2hiint(x), lo = __double2loint(x);
  const int keep = ~(hi >> 31);  // 0 for a set sign bit, all ones otherwise
  return __hiloint2double(hi & keep, lo & keep);
}
// PG entry (nnls.py:89-107): g where f > 0, else min(g, 0), on the integer
// pipe: f > 0 is "f's bit pattern is a positive int64" (exact for every
// non-NaN f, -0.0 included), min(g, 0) zeroes a g without sign bit (a
// positive NaN g also makes <f, g> non-finite, which fails the iteration as
// the reference does).
__device__ __forceinline__ double pg_entry_fast(double f, double g) {
  const int gh = __double2hiint(g), gl = __double2loint(g);
  const int keep = (__double_as_longlong(f) > 0) ? -1 : (gh >> 31);
  return __hiloint2double(gh & keep, gl & keep);
}
// np.minimum(x, 0) keeping NaN
template <typename T>
__device__ __forceinline__ T min0_nan(T x) { return (x <= T(0) || x != x) ? x : T(0); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order block reduction (deterministic): warp xor-trees, then warp 0
// adds the per-warp values in warp order.  Result valid in all threads.
// `scratch` must hold >= 33 doubles.  Contains __syncthreads.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += scratch[w];
    scratch[32] = s;
  }
  __syncthreads();
  return scratch[32];
}

// record the first failure only
__device__ __forceinline__ void status_fail(nenmf_device_status* st, int code, int iteration) {
  if (st == nullptr) return;
  if (atomicCAS(&st->code, 0, code) == 0) st->iteration = iteration;
}

__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename T>
struct DT;
template <>
struct DT<double> {
  static constexpr int code = NENMF_F64;
};
template <>
struct DT<float> {
  static constexpr int code = NENMF_F32;
};

}  // namespace nenmf

// dtype dispatch: calls BODY with `scalar_t` bound to double / float
#define NENMF_DISPATCH(dtype, ...)                         \
  [&]() -> int {                                           \
    if ((dtype) == NENMF_F64) {                            \
      using scalar_t = double;                             \
      return __VA_ARGS__();                                \
    } else if ((dtype) == NENMF_F32) {                     \
      using scalar_t = float;                              \
      return __VA_ARGS__();                                \
    }                                                      \
    return NENMF_ERR_VALUE;                                \
  }()
