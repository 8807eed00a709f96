// Orthonormal basis of a tall panel (the role of np.linalg.qr in
// compression.py:88-106) by rank-revealing CholeskyQR2, all on the device.
//
//   G1 = P^T P (fp64, fixed-order split-K)                   gram_d
//   pivoted Cholesky of G1 -> rank r, P Pi = Q1 R11          k_factor     (1 CTA)
//   Q1 = P Pi R11^{-1} (row-parallel triangular solves);      k_trsm_apply
//        columns r..k-1 replaced by fixed pseudo-random
//        vectors (the reference's trailing Householder columns of a
//        rank-deficient panel are rounding noise; any orthonormal completion
//        spans the same determined subspace)
//   G2 = Q1^T Q1, Cholesky R2 (no pivoting)                  k_factor     (1 CTA)
//   Q  = Q1 R2^{-1}                                          k_trsm_apply
//
// Cost: four streaming passes over the panel plus two one-CTA k x k
// factorisations, instead of a k-step Householder sweep.  The compressed
// problem is invariant to the choice of orthonormal basis of the subspace
// (W = F_R F_R^T and V = F_R X_R^T are unchanged by R -> R U), and RSI's
// subspace evolution is basis independent, so only the subspace is pinned
// against the reference (tests/test_gpu_rsi_factorize.py).
// Failure semantics follow compression.py:97-105: a non-finite panel or a
// panel with no usable direction raises NumericalCollapseError.
#include "rsi.cuh"
#include "skinny.cuh"

#include <cooperative_groups.h>

namespace nenmf {

constexpr int QC_KMAX = 32;  // the register-row factorisation holds k <= 32

// (Pivoted) Cholesky of a k x k Gram matrix, right-looking, by ONE warp:
// lane a keeps row a of the Schur complement in registers (k <= 32), the
// pivot row is exchanged with shuffles; no block barriers.  Rows of R are
// produced in pivot order with columns in the original index space:
// P[:, perm] = Q R11 (R11[j][l] = R[j*k + perm[l]]).  Without pivoting perm is
// the identity.  Pivots <= rel_tol * max(diag) end it (rank).  S (k*k) holds
// the Gram matrix; R (k*k) is shared scratch.  Only warp 0 works.
__device__ void block_factor(double* S, double* R, int k, int pivot, double rel_tol, double* __restrict__ Rout,
                             int* __restrict__ meta, nenmf_device_status* st) {
  __shared__ int perm[QC_KMAX];
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const unsigned FULL = 0xffffffffu;
    double row[32];
#pragma unroll
    for (int b = 0; b < 32; ++b) row[b] = (lane < k && b < k) ? S[lane * k + b] : 0.0;
    bool rem = lane < k;
    bool bad = false;
#pragma unroll
    for (int b = 0; b < 32; ++b) bad |= !isfinite(row[b]);
    bad = __any_sync(FULL, bad);
    double diag = 0.0;
#pragma unroll
    for (int b = 0; b < 32; ++b)
      if (b == lane) diag = row[b];
    double mx = rem ? diag : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
    for (int e = lane; e < k * k; e += 32) R[e] = 0.0;
    int rank = k;
    if (bad || !(mx > 0.0)) {
      rank = 0;
      if (lane == 0) status_fail(st, NENMF_ERR_NUMERICAL_COLLAPSE, -1);
    } else {
      const double tau = rel_tol * mx;
      for (int j = 0; j < k; ++j) {
        int best;
        double bv;
        if (pivot) {
          bv = rem ? diag : -1.0;
          best = rem ? lane : -1;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(FULL, bv, o);
            const int oi = __shfl_xor_sync(FULL, best, o);
            if (ov > bv || (ov == bv && oi >= 0 && (best < 0 || oi < best))) {
              bv = ov;
              best = oi;
            }
          }
        } else {
          best = j;
          bv = __shfl_sync(FULL, diag, j);
        }
        if (!(bv > tau)) {
          rank = j;
          break;
        }
        const int pj = best;
        if (lane == pj) rem = false;
        if (lane == 0) perm[j] = pj;
        const double rjj = sqrt(bv), inv = 1.0 / rjj;
        // R[j][a] = S[a][pj] / rjj for remaining rows a (column pj of my row)
        double sap = 0.0;
#pragma unroll
        for (int b = 0; b < 32; ++b)
          if (b == pj) sap = row[b];
        const double ra = rem ? sap * inv : (lane == pj ? rjj : 0.0);
        if (lane < k) R[j * k + lane] = ra;
        const double rself = rem ? ra : 0.0;
        // Schur update of my row: row[b] -= R[j][a] R[j][b]
#pragma unroll
        for (int b = 0; b < 32; ++b) {
          const double rb = __shfl_sync(FULL, rem ? ra : 0.0, b);
          row[b] = fma(-rself, rb, row[b]);
        }
#pragma unroll
        for (int b = 0; b < 32; ++b)
          if (b == lane) diag = row[b];
      }
    }
    __syncwarp();
    for (int e = lane; e < k * k; e += 32) Rout[e] = R[e];
    for (int i = lane; i < k; i += 32) meta[1 + i] = i < rank ? perm[i] : -1;
    if (lane == 0) {
      meta[0] = rank;
      if (!pivot && rank < k) status_fail(st, NENMF_ERR_NUMERICAL_COLLAPSE, -1);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ double hash_uniform(uint64_t a, uint64_t b) {
  uint64_t z = a * 0x9E3779B97F4A7C15ull + b * 0xD1B54A32D192ED03ull + 0x632BE59BD9B4E019ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

// row i of the panel: solve q R11 = z with z_l = in[perm[l]] (l < rank), i.e.
// Q = P[:, perm] R11^{-1}; columns l >= rank get fixed pseudo-random values.
template <typename T, int KM>
__device__ __forceinline__ void trsm_row(const T* __restrict__ in_t, int64_t rows, int k, const double* Rs,
                                         const int* perm, const double* rdiag_inv, int r, int64_t i,
                                         T* __restrict__ out_t) {
  double q[KM];
  // all loads first (independent), then the dependent substitution
#pragma unroll
  for (int l = 0; l < KM; ++l) q[l] = l < r ? (double)in_t[(int64_t)perm[l] * rows + i] : 0.0;
#pragma unroll
  for (int l = 0; l < KM; ++l) {
    if (l < r) {
      double z = q[l];
      const double* rc = Rs + perm[l];
#pragma unroll
      for (int j = 0; j < KM; ++j)
        if (j < l) z = fma(-q[j], rc[j * k], z);
      q[l] = z * rdiag_inv[l];
    }
  }
#pragma unroll
  for (int l = 0; l < KM; ++l)
    if (l < k) out_t[(int64_t)l * rows + i] = (T)(l < r ? q[l] : hash_uniform((uint64_t)i, (uint64_t)l));
}

// Gram partial sum_{i in [r0, r1)} p_i p_i^T of a short-major panel -> out (k*k)
template <typename T>
__device__ void block_gram(const T* __restrict__ Pt, int64_t rows, int k, int64_t r0, int64_t r1, double* tile,
                           double* __restrict__ out) {
  constexpr int RS = 128;
  const int kk = k * k;
  double acc[QC_KMAX * QC_KMAX / 256];
#pragma unroll
  for (int t = 0; t < QC_KMAX * QC_KMAX / 256; ++t) acc[t] = 0.0;
  for (int64_t base = r0; base < r1; base += RS) {
    const int nr = (int)imin(RS, r1 - base);
    __syncthreads();
    for (int idx = threadIdx.x; idx < k * RS; idx += blockDim.x) {
      const int a = idx / RS, rr = idx - a * RS;
      tile[a * (RS + 1) + rr] = rr < nr ? (double)Pt[(int64_t)a * rows + base + rr] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < QC_KMAX * QC_KMAX / 256; ++t) {
      const int e = threadIdx.x + 256 * t;
      if (e < kk) {
        const int a = e / k, b = e - a * k;
        const double* pa = tile + a * (RS + 1);
        const double* pb = tile + b * (RS + 1);
        double s = acc[t];
        for (int rr = 0; rr < nr; ++rr) s = fma(pa[rr], pb[rr], s);
        acc[t] = s;
      }
    }
  }
#pragma unroll
  for (int t = 0; t < QC_KMAX * QC_KMAX / 256; ++t) {
    const int e = threadIdx.x + 256 * t;
    if (e < kk) out[e] = acc[t];
  }
}

template <typename T>
struct QrPanel {
  T* Pt;
  int64_t rows;
  nenmf_device_status* st;
  double* part;  // [ncta][k*k]
  double* R;     // k*k
  int* meta;     // 1 + k
  T* Q1;         // k * rows
  int cta0, ncta;
};

// Rank-revealing CholeskyQR2 of one or two panels in ONE cooperative launch:
// Gram partials | leader: reduce + pivoted Cholesky | triangular solves +
// Gram partials of Q1 | leader: reduce + Cholesky | triangular solves.
__device__ unsigned long long g_qr_trace[16];
__device__ __forceinline__ void qr_stamp(int i) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_qr_trace[i] = t;
  }
}

// grid-wide barrier over co-resident CTAs (cooperative launch): monotone
// counter, barrier number `gen` completes at gen * gridDim.x arrivals
__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    const unsigned target = gen * gridDim.x;
    while (true) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
      __nanosleep(20);
    }
  }
  __syncthreads();
}

template <typename T, int KM>
__global__ void __launch_bounds__(256) k_qr2(QrPanel<T> P0, QrPanel<T> P1, int npanels, int k, unsigned* bar) {
  extern __shared__ double qsm[];
  double* S = qsm;                    // k*k
  double* R = S + k * k;              // k*k
  double* tile = R + k * k;           // k * 129
  __shared__ int perm[QC_KMAX];
  __shared__ double rdinv[QC_KMAX];
  const bool second = npanels > 1 && (int)blockIdx.x >= P1.cta0;
  const QrPanel<T>& P = second ? P1 : P0;
  const int local = (int)blockIdx.x - P.cta0;
  const int64_t r0 = (int64_t)local * P.rows / P.ncta, r1 = (int64_t)(local + 1) * P.rows / P.ncta;
  const int kk = k * k;

  auto reduce_factor = [&](int pivot, double tol) {
    if (local == 0) {
      for (int e = threadIdx.x; e < kk; e += blockDim.x) {
        double s = 0.0;
        for (int c = 0; c < P.ncta; ++c) s += P.part[(int64_t)c * kk + e];
        S[e] = s;
      }
      __syncthreads();
      block_factor(S, R, k, pivot, tol, P.R, P.meta, P.st);
    }
  };
  auto solve_rows = [&](const T* in_t, T* out_t) {
    for (int e = threadIdx.x; e < kk; e += blockDim.x) R[e] = P.R[e];
    for (int i = threadIdx.x; i < k; i += blockDim.x) perm[i] = P.meta[1 + i];
    __syncthreads();
    const int r = P.meta[0];
    for (int i = threadIdx.x; i < r; i += blockDim.x) rdinv[i] = 1.0 / R[i * k + perm[i]];
    __syncthreads();
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x)
      trsm_row<T, KM>(in_t, P.rows, k, R, perm, rdinv, r, i, out_t);
    __syncthreads();
  };

  qr_stamp(0);
  block_gram<T>(P.Pt, P.rows, k, r0, r1, tile, P.part + (int64_t)local * kk);  // G1 partials
  qr_stamp(1);
  grid_barrier(bar, 1);
  qr_stamp(2);
  reduce_factor(1, 1e-14);  // rank-revealing pass
  qr_stamp(3);
  grid_barrier(bar, 2);
  qr_stamp(4);
  const bool ok = P.meta[0] > 0;
  if (ok) {
    solve_rows(P.Pt, P.Q1);
    qr_stamp(5);
    __threadfence_block();
    block_gram<T>(P.Q1, P.rows, k, r0, r1, tile, P.part + (int64_t)local * kk);  // G2 partials
  }
  qr_stamp(6);
  grid_barrier(bar, 3);
  qr_stamp(7);
  if (ok) reduce_factor(0, 1e-300);  // CholeskyQR2 second pass
  qr_stamp(8);
  grid_barrier(bar, 4);
  qr_stamp(9);
  if (ok && P.meta[0] == k) solve_rows(P.Q1, P.Pt);
  qr_stamp(10);
}

template <typename T>
int orthonormalize_pair(Arena& ws, T* P0t, int64_t rows0, T* P1t, int64_t rows1, int64_t k,
                        nenmf_device_status* st, cudaStream_t s) {
  if (k < 1 || k > QC_KMAX || rows0 < k || (P1t != nullptr && rows1 < k)) return k > QC_KMAX ? NENMF_ERR_UNSUPPORTED : NENMF_ERR_DIM;
  const int npan = P1t != nullptr ? 2 : 1;
  auto ctas = [](int64_t rows) { return (int)imax(1, imin(32, cdiv(rows, 64))); };
  QrPanel<T> Q[2];
  const int64_t rowsv[2] = {rows0, rows1};
  T* ptv[2] = {P0t, P1t};
  int cta0 = 0;
  for (int i = 0; i < npan; ++i) {
    Q[i].Pt = ptv[i];
    Q[i].rows = rowsv[i];
    Q[i].st = st;
    Q[i].ncta = ctas(rowsv[i]);
    Q[i].cta0 = cta0;
    cta0 += Q[i].ncta;
    Q[i].part = ws.take<double>((size_t)Q[i].ncta * k * k);
    Q[i].R = ws.take<double>((size_t)k * k);
    Q[i].meta = ws.take<int>((size_t)k + 4);
    Q[i].Q1 = ws.take<T>((size_t)k * rowsv[i]);
  }
  if (npan == 1) Q[1] = Q[0];
  unsigned* bar = ws.take<unsigned>(64);
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  NENMF_CUDA_TRY(cudaMemsetAsync(bar, 0, sizeof(unsigned), s));
  const size_t smem = ((size_t)2 * k * k + (size_t)k * 129) * sizeof(double);
  int kint = (int)k;
  void* args[] = {(void*)&Q[0], (void*)&Q[1], (void*)&npan, (void*)&kint, (void*)&bar};
  NENMF_CUDA_TRY(set_smem(k_qr2<T, 32>, smem));
  NENMF_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_qr2<T, 32>, dim3(cta0), dim3(256), args, smem, s));
  launch_counter_add(1);
  return NENMF_OK;
}

template <typename T>
int orthonormalize_cholqr(Arena& ws, T* Pt, int64_t rows, int64_t k, nenmf_device_status* st, cudaStream_t s) {
  if (rows < 1 || k < 1 || k > rows) return NENMF_ERR_DIM;
  return orthonormalize_pair<T>(ws, Pt, rows, nullptr, 0, k, st, s);
}

template int orthonormalize_pair<double>(Arena&, double*, int64_t, double*, int64_t, int64_t, nenmf_device_status*,
                                         cudaStream_t);
template int orthonormalize_pair<float>(Arena&, float*, int64_t, float*, int64_t, int64_t, nenmf_device_status*,
                                        cudaStream_t);
template int orthonormalize_cholqr<double>(Arena&, double*, int64_t, int64_t, nenmf_device_status*, cudaStream_t);
template int orthonormalize_cholqr<float>(Arena&, float*, int64_t, int64_t, nenmf_device_status*, cudaStream_t);

}  // namespace nenmf

extern "C" int nenmf_debug_qr_trace(unsigned long long* host_out) {
  return cudaMemcpyFromSymbol(host_out, nenmf::g_qr_trace, sizeof(unsigned long long) * 16) == cudaSuccess ? 0 : 6;
}
