// Device side of the NMFB loader (matrix.py:180-214): the
// file's little-endian float64 payload arrives in pinned chunks; each chunk is
// converted on the device to the working dtype while the host reads the next
// one, and non-finite values are flagged (read_nmfb's require_finite).
#include "common.cuh"

namespace nenmf {

template <typename T>
__global__ void k_convert_f64(const double* __restrict__ src, int64_t count, T* __restrict__ dst,
                              int* __restrict__ nonfinite) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool bad = false;
  const int64_t n2 = count / 2;
  const double2* s2 = reinterpret_cast<const double2*>(src);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
    const double2 v = __ldcs(&s2[i]);  // streamed once
    bad |= !isfinite(v.x) || !isfinite(v.y);
    dst[2 * i] = (T)v.x;
    dst[2 * i + 1] = (T)v.y;
  }
  if ((count & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const double v = src[count - 1];
    bad |= !isfinite(v);
    dst[count - 1] = (T)v;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *nonfinite = 1;
}

}  // namespace nenmf

using namespace nenmf;

extern "C" int nenmf_convert_f64(int dtype, const double* src, int64_t count, void* dst, int* nonfinite,
                                 void* stream) {
  if (count < 0 || (count > 0 && (src == nullptr || dst == nullptr || nonfinite == nullptr))) return NENMF_ERR_VALUE;
  if (count == 0) return NENMF_OK;
  if ((reinterpret_cast<uintptr_t>(src) & 15) != 0) return NENMF_ERR_VALUE;  // double2 loads
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int sms = sm_count();
  if (sms <= 0) sms = 148;
  const unsigned grid = (unsigned)imax(1, imin(cdiv(count / 2, 256), (int64_t)sms * 8));
  if (dtype == NENMF_F32) {
    k_convert_f64<float><<<grid, 256, 0, s>>>(src, count, static_cast<float*>(dst), nonfinite);
  } else if (dtype == NENMF_F64) {
    k_convert_f64<double><<<grid, 256, 0, s>>>(src, count, static_cast<double*>(dst), nonfinite);
  } else {
    return NENMF_ERR_VALUE;
  }
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}
