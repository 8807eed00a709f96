// The exact-SNR problem generator's arithmetic (synthetic.py:62-81) fused on
// the device: X = G F + s N with s = ||G F|| 10^(-snr/20) / ||N||.
//   k_gen_norms: ||G F||^2 (G F formed on the fly, fp64, never stored) and
//                ||N||^2 in ONE read of N; fixed-order partials.
//   k_gen_write: X = G F + s N in the working dtype (G F recomputed: p FMAs
//                per element instead of an n x m round trip through HBM).
// G (n x p) and F (p x m) are fp64, N fp64 n x m (the bit-identical NumPy
// normal stream), X fp64 or fp32.  Replaces a cuBLAS DGEMM, three norm
// passes and four elementwise passes (~80 B/element) by ~24 B/element.
#include "common.cuh"

namespace nenmf {

constexpr int GEN_THREADS = 256;
constexpr int GEN_PMAX = 1 << 20;  // the kernels loop over p; no structural limit

// one thread per (row, 4-column group); the CTA stages F's 4-column slabs
__global__ void __launch_bounds__(GEN_THREADS)
k_gen_norms(const double* __restrict__ G, const double* __restrict__ F, const double* __restrict__ N, int64_t n,
            int64_t m, int p, double* __restrict__ part) {
  __shared__ double red[33];
  double c2 = 0.0, n2 = 0.0;
  const int64_t total = n * m;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t i = e / m, j = e - i * m;
    double v = 0.0;
    for (int a = 0; a < p; ++a) v = fma(G[i * p + a], F[(int64_t)a * m + j], v);
    c2 = fma(v, v, c2);
    const double z = N[e];
    n2 = fma(z, z, n2);
  }
  c2 = block_sum(c2, red);
  n2 = block_sum(n2, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = c2;
    part[2 * blockIdx.x + 1] = n2;
  }
}

__global__ void k_gen_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double red[33];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    a += part[2 * i];
    b += part[2 * i + 1];
  }
  a = block_sum(a, red);
  b = block_sum(b, red);
  if (threadIdx.x == 0) {
    out[0] = a;
    out[1] = b;
  }
}

template <typename TO>
__global__ void __launch_bounds__(GEN_THREADS)
k_gen_write(const double* __restrict__ G, const double* __restrict__ F, const double* __restrict__ N, int64_t n,
            int64_t m, int p, double scale, TO* __restrict__ X) {
  const int64_t total = n * m;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t i = e / m, j = e - i * m;
    double v = 0.0;
    for (int a = 0; a < p; ++a) v = fma(G[i * p + a], F[(int64_t)a * m + j], v);
    X[e] = (TO)(N != nullptr ? __dadd_rn(v, __dmul_rn(N[e], scale)) : v);
  }
}

}  // namespace nenmf

extern "C" {

size_t nenmf_generate_workspace_bytes(void) { return (size_t)2 * 4 * 148 * 8 * sizeof(double) + 512; }

int nenmf_generate_norms(const double* G, const double* F, const double* N, int64_t n, int64_t m, int64_t p,
                         double* out2, void* ws, size_t ws_bytes, void* stream) {
  using namespace nenmf;
  if (G == nullptr || F == nullptr || N == nullptr || out2 == nullptr || ws == nullptr) return NENMF_ERR_VALUE;
  if (n < 1 || m < 1 || p < 1 || p > GEN_PMAX) return NENMF_ERR_DIM;
  int sms = sm_count();
  if (sms <= 0) sms = 148;
  const unsigned grid = (unsigned)imax(1, imin((int64_t)sms * 8, cdiv(n * m, GEN_THREADS)));
  if (ws_bytes < (size_t)grid * 2 * sizeof(double)) return NENMF_ERR_WORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* part = static_cast<double*>(ws);
  k_gen_norms<<<grid, GEN_THREADS, 0, s>>>(G, F, N, n, m, (int)p, part);
  NENMF_LAUNCH_CHECK();
  k_gen_final<<<1, 256, 0, s>>>(part, (int)grid, out2);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

int nenmf_generate_write(int dtype, const double* G, const double* F, const double* N, int64_t n, int64_t m,
                         int64_t p, double scale, void* X, void* stream) {
  using namespace nenmf;
  if (G == nullptr || F == nullptr || X == nullptr) return NENMF_ERR_VALUE;
  if (n < 1 || m < 1 || p < 1 || p > GEN_PMAX) return NENMF_ERR_DIM;
  int sms = sm_count();
  if (sms <= 0) sms = 148;
  const unsigned grid = (unsigned)imax(1, imin((int64_t)sms * 8, cdiv(n * m, GEN_THREADS)));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == NENMF_F64)
    k_gen_write<double><<<grid, GEN_THREADS, 0, s>>>(G, F, N, n, m, (int)p, scale, static_cast<double*>(X));
  else if (dtype == NENMF_F32)
    k_gen_write<float><<<grid, GEN_THREADS, 0, s>>>(G, F, N, n, m, (int)p, scale, static_cast<float*>(X));
  else
    return NENMF_ERR_VALUE;
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

}  // extern "C"
