// Randomized subspace iteration (compression.py:120-188) on sm_100a.
//
//   k_dual         one streaming pass over X producing BOTH X @ A and X^T @ B
//                  (compression.py:134-139,188 issue them as separate GEMMs
//                  and re-read X for each; here the L-chain and R-chain share
//                  every read of X: 2q+2 passes instead of 4q+4)
//   TSQR           reduced Householder QR of a tall panel (compression.py:101,
//                  np.linalg.qr = LAPACK dgeqrf + dorgqr): blocks of rows are
//                  factored in shared memory, their R factors stacked and
//                  factored again until one block remains; Q is formed top
//                  down.  Rank deficiency is tolerated (Householder Q is always
//                  orthonormal); non-finite input or an all-zero diag(R) is a
//                  NumericalCollapseError (compression.py:97-105).
//
// Skinny panels are stored short-major (Pt = P^T, k x rows), so a panel is a
// column-major tall matrix and every Householder column is contiguous.
#include "rsi.cuh"

#include <cstdlib>
#include "skinny.cuh"

namespace nenmf {

// ================================================================ dual ====
constexpr int DU_TR = 32;       // rows per sub-tile
constexpr int DU_TC = 64;       // cols per sub-tile
constexpr int DU_BR = 256;      // rows per CTA block
constexpr int DU_BCMAX = 256;   // cols per CTA block (runtime, multiple of DU_TC)
constexpr int DU_THREADS = 256;
constexpr int DU_KMAX = 128;
constexpr size_t DU_SMEM_BUDGET = 200 * 1024;

template <typename T>
inline int dual_block_cols(int64_t k) {
  size_t tiles = ((size_t)DU_TR * (DU_TC + 1) + (size_t)k * (DU_TC + 1) + (size_t)k * (DU_TR + 1)) * sizeof(T);
  int64_t bc = (int64_t)((DU_SMEM_BUDGET - tiles) / ((size_t)k * sizeof(T))) / DU_TC * DU_TC;
  return (int)imax(DU_TC, imin(DU_BCMAX, bc));
}

// Yt = At X^T (k x n) and Zt = Bt X (k x m) over the CTA's X block; partial
// sums over column blocks (Y) / row blocks (Z) go to Ypart / Zpart unless the
// grid has a single block along that axis, in which case they are final.
template <typename T>
__global__ void __launch_bounds__(DU_THREADS)
k_dual(const T* __restrict__ X, int64_t n, int64_t m, int64_t ldx, const T* __restrict__ At,
       const T* __restrict__ Bt, int k, int BC, T* __restrict__ Yout, T* __restrict__ Zout) {
  extern __shared__ double smem_d[];
  T* Xs = reinterpret_cast<T*>(smem_d);                 // [TR][TC+1]
  T* Ats = Xs + DU_TR * (DU_TC + 1);                     // [k][TC+1]
  T* Bts = Ats + k * (DU_TC + 1);                        // [k][TR+1]
  T* Zacc = Bts + k * (DU_TR + 1);                       // [k][BC]
  const int DU_BC = BC;
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * DU_BR, c0 = (int64_t)blockIdx.x * DU_BC;
  const int64_t r1 = min(n, r0 + DU_BR), c1 = min(m, c0 + DU_BC);
  const bool doY = At != nullptr, doZ = Bt != nullptr;
  // Y mapping: row yi of the band, a = yag + 8 s
  const int yi = tid & 31, yag = tid >> 5;
  // Z mapping: column zj of the tile, a = zag + 4 s
  const int zj = tid & 63, zag = tid >> 6;
  if (doZ)
    for (int i = tid; i < k * BC; i += DU_THREADS) Zacc[i] = T(0);

  for (int64_t rb = r0; rb < r1; rb += DU_TR) {
    const int nr = (int)imin(DU_TR, r1 - rb);
    T yacc[DU_KMAX / 8];
#pragma unroll
    for (int s = 0; s < DU_KMAX / 8; ++s) yacc[s] = T(0);
    for (int64_t cb = c0; cb < c1; cb += DU_TC) {
      const int nc = (int)imin(DU_TC, c1 - cb);
      __syncthreads();
      for (int idx = tid; idx < DU_TR * DU_TC; idx += DU_THREADS) {
        int i = idx / DU_TC, j = idx % DU_TC;
        Xs[i * (DU_TC + 1) + j] = (i < nr && j < nc) ? X[(rb + i) * ldx + cb + j] : T(0);
      }
      if (doY)
        for (int idx = tid; idx < k * DU_TC; idx += DU_THREADS) {
          int a = idx / DU_TC, j = idx % DU_TC;
          Ats[a * (DU_TC + 1) + j] = j < nc ? At[(int64_t)a * m + cb + j] : T(0);
        }
      if (doZ)
        for (int idx = tid; idx < k * DU_TR; idx += DU_THREADS) {
          int a = idx / DU_TR, i = idx % DU_TR;
          Bts[a * (DU_TR + 1) + i] = i < nr ? Bt[(int64_t)a * n + rb + i] : T(0);
        }
      __syncthreads();
      if (doY && yi < nr) {
        for (int j = 0; j < nc; ++j) {
          const T x = Xs[yi * (DU_TC + 1) + j];
#pragma unroll
          for (int s = 0; s < DU_KMAX / 8; ++s) {
            int a = yag + 8 * s;
            if (a < k) yacc[s] = fma_acc(Ats[a * (DU_TC + 1) + j], x, yacc[s]);
          }
        }
      }
      if (doZ && zj < nc) {
        T zacc[DU_KMAX / 4];
#pragma unroll
        for (int s = 0; s < DU_KMAX / 4; ++s) zacc[s] = T(0);
        for (int i = 0; i < nr; ++i) {
          const T x = Xs[i * (DU_TC + 1) + zj];
#pragma unroll
          for (int s = 0; s < DU_KMAX / 4; ++s) {
            int a = zag + 4 * s;
            if (a < k) zacc[s] = fma_acc(Bts[a * (DU_TR + 1) + i], x, zacc[s]);
          }
        }
        const int jo = (int)(cb - c0) + zj;
#pragma unroll
        for (int s = 0; s < DU_KMAX / 4; ++s) {
          int a = zag + 4 * s;
          if (a < k) Zacc[a * DU_BC + jo] += zacc[s];
        }
      }
    }
    if (doY && yi < nr) {
      T* dst = Yout + (int64_t)blockIdx.x * k * n;  // partial slab of this column block
#pragma unroll
      for (int s = 0; s < DU_KMAX / 8; ++s) {
        int a = yag + 8 * s;
        if (a < k) dst[(int64_t)a * n + rb + yi] = yacc[s];
      }
    }
  }
  if (doZ) {
    __syncthreads();
    T* dst = Zout + (int64_t)blockIdx.y * k * m;
    for (int idx = tid; idx < k * DU_BC; idx += DU_THREADS) {
      int a = idx / DU_BC, j = idx % DU_BC;
      if (c0 + j < c1) dst[(int64_t)a * m + c0 + j] = Zacc[idx];
    }
  }
}

template <typename T>
__global__ void k_slab_reduce(const T* __restrict__ part, int nslab, int64_t count, T* __restrict__ out) {
  int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= count) return;
  T s = part[o];
  for (int c = 1; c < nslab; ++c) s += part[(int64_t)c * count + o];
  out[o] = s;
}

int dual_pass_tc(Arena& ws, const float* X, int64_t n, int64_t m, int64_t ldx, const float* At, const float* Bt,
                 int64_t k, float* Yt, float* Zt, cudaStream_t s);
int dual_pass_f64(Arena& ws, const double* X, int64_t n, int64_t m, int64_t ldx, const double* At,
                  const double* Bt, int64_t k, double* Yt, double* Zt, cudaStream_t s);

template <typename T>
int dual_pass(Arena& ws, const T* X, int64_t n, int64_t m, int64_t ldx, const T* At, const T* Bt, int64_t k,
              T* Yt, T* Zt, cudaStream_t s) {
  if (n < 1 || m < 1 || k < 1) return NENMF_ERR_DIM;
  {
    // wide sketches (any nu, compression.py:109-117): row blocks of the short-major skinny
    // operands, one X stream per block (FP64: 32 rows, the DMMA pass; FP32: 128)
    const int64_t kblk = sizeof(T) == 4 ? 128 : 32;
    if (k > kblk) {
      const bool dry = ws.base == nullptr;
      size_t need = 0;
      for (int64_t k0 = 0; k0 < k; k0 += kblk) {
        const int64_t kc = imin(kblk, k - k0);
        Arena a = dry ? Arena(nullptr, 0) : ws;
        NENMF_TRY(dual_pass<T>(a, X, n, m, ldx, At != nullptr ? At + k0 * m : nullptr,
                               Bt != nullptr ? Bt + k0 * n : nullptr, kc, Yt != nullptr ? Yt + k0 * n : nullptr,
                               Zt != nullptr ? Zt + k0 * m : nullptr, s));
        if (a.used - (dry ? 0 : ws.used) > need) need = a.used - (dry ? 0 : ws.used);
      }
      if (dry) ws.take<char>(need);
      return NENMF_OK;
    }
  }
  if constexpr (sizeof(T) == 4) {
    // FP32 data: tcgen05 BF16x3 pass when the shape fits (dual_tc.cu)
    int rc = dual_pass_tc(ws, reinterpret_cast<const float*>(X), n, m, ldx, reinterpret_cast<const float*>(At),
                          reinterpret_cast<const float*>(Bt), k, reinterpret_cast<float*>(Yt),
                          reinterpret_cast<float*>(Zt), s);
    if (rc != NENMF_ERR_UNSUPPORTED) return rc;
  }
  if constexpr (sizeof(T) == 8) {
    // FP64: both products from one read of X on the FP64 tensor pipe (dual64.cu)
    if (getenv("NENMF_DUAL_SIMT") == nullptr) {
      Arena a = ws;
      const int rc = dual_pass_f64(a, reinterpret_cast<const double*>(X), n, m, ldx,
                                   reinterpret_cast<const double*>(At), reinterpret_cast<const double*>(Bt), k,
                                   reinterpret_cast<double*>(Yt), reinterpret_cast<double*>(Zt), s);
      if (rc != NENMF_ERR_UNSUPPORTED) {
        ws = a;
        return rc;
      }
    }
    // otherwise the two products separately (skinny.cu ab -> k_xv64 / k_ux64),
    // one X stream each: Yt = At X^T (B = X^T), Zt = Bt X (B = X)
    if (k <= 32 && getenv("NENMF_DUAL_SIMT") == nullptr) {
      Arena a0 = ws;
      if (At != nullptr) NENMF_TRY(ab<T>(a0, At, k, m, X, n, ldx, true, Yt, s));
      Arena a1 = ws;
      if (Bt != nullptr) NENMF_TRY(ab<T>(a1, Bt, k, n, X, m, ldx, false, Zt, s));
      ws.used = a0.used > a1.used ? a0.used : a1.used;
      if (!ws.ok || !a0.ok || !a1.ok) ws.ok = false;
      return ws.base == nullptr || ws.ok ? NENMF_OK : NENMF_ERR_WORKSPACE;
    }
  }
  if (k > DU_KMAX) return NENMF_ERR_UNSUPPORTED;
  const int BC = dual_block_cols<T>(k);
  const int64_t gx = cdiv(m, BC), gy = cdiv(n, DU_BR);
  T* Ypart = (At != nullptr && gx > 1) ? ws.take<T>((size_t)gx * k * n) : nullptr;
  T* Zpart = (Bt != nullptr && gy > 1) ? ws.take<T>((size_t)gy * k * m) : nullptr;
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  size_t smem = ((size_t)DU_TR * (DU_TC + 1) + (size_t)k * (DU_TC + 1) + (size_t)k * (DU_TR + 1) +
                 (size_t)k * BC) * sizeof(T);
  NENMF_CUDA_TRY(set_smem(k_dual<T>, smem));
  dim3 grid((unsigned)gx, (unsigned)gy);
  k_dual<T><<<grid, DU_THREADS, smem, s>>>(X, n, m, ldx, At, Bt, (int)k, BC, Ypart ? Ypart : Yt, Zpart ? Zpart : Zt);
  NENMF_LAUNCH_CHECK();
  if (Ypart) {
    k_slab_reduce<T><<<(unsigned)cdiv(k * n, 256), 256, 0, s>>>(Ypart, (int)gx, k * n, Yt);
    NENMF_LAUNCH_CHECK();
  }
  if (Zpart) {
    k_slab_reduce<T><<<(unsigned)cdiv(k * m, 256), 256, 0, s>>>(Zpart, (int)gy, k * m, Zt);
    NENMF_LAUNCH_CHECK();
  }
  return NENMF_OK;
}

// ================================================================ TSQR ====
constexpr int QR_THREADS = 512;
constexpr size_t QR_SMEM_BUDGET = 200 * 1024;

inline int qr_block_rows(int64_t k) {
  int64_t hb = (int64_t)(QR_SMEM_BUDGET / sizeof(double)) / k;
  hb = imin(hb, 1024);
  hb = hb / 32 * 32;
  return (int)imax(hb, 2 * k);
}

__device__ __forceinline__ int64_t blk_start(int64_t rows, int nb, int b) { return (int64_t)b * rows / nb; }

// Householder QR of each row block of M (rows x k, column-major with leading
// dimension ldm).  Writes the reflectors (block-local column-major h x k,
// LAPACK layout with implicit unit diagonal) and tau, and R_b into rows
// [b k, b k + k) of Mnext (column-major, leading dimension ldn).  When nb == 1
// and top != 0, checks diag(R) for total collapse.
template <typename TIN>
__global__ void __launch_bounds__(QR_THREADS)
k_qr_block(const TIN* __restrict__ M, int64_t ldm, int64_t rows, int k, int nb, double* __restrict__ Vbuf,
           double* __restrict__ tau, double* __restrict__ Mnext, int64_t ldn, int top, int check_finite,
           nenmf_device_status* st) {
  extern __shared__ double C[];  // [k][h]
  __shared__ double sh[4];
  __shared__ int bad;
  const int b = blockIdx.x;
  const int64_t s0 = blk_start(rows, nb, b);
  const int h = (int)(blk_start(rows, nb, b + 1) - s0);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int idx = tid; idx < k * h; idx += blockDim.x) {
    int c = idx / h, i = idx % h;
    double v = (double)M[(int64_t)c * ldm + s0 + i];
    if (check_finite && !isfinite(v)) bad = 1;
    C[c * h + i] = v;
  }
  __syncthreads();
  if (bad) {
    if (tid == 0) status_fail(st, NENMF_ERR_NUMERICAL_COLLAPSE, -1);
    return;
  }
  for (int j = 0; j < k; ++j) {
    double* cj = C + j * h;
    if (wid == 0) {
      // dlarfg on C[j:h, j]
      double x2 = 0.0;
      for (int i = j + 1 + lane; i < h; i += 32) x2 = fma(cj[i], cj[i], x2);
      x2 = warp_sum(x2);
      const double alpha = cj[j];
      const double xnorm = sqrt(x2);
      double beta, t, scal;
      if (xnorm == 0.0) {
        beta = alpha;
        t = 0.0;
        scal = 0.0;
      } else {
        beta = -copysign(hypot(alpha, xnorm), alpha);
        t = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      if (xnorm != 0.0)
        for (int i = j + 1 + lane; i < h; i += 32) cj[i] *= scal;
      if (lane == 0) {
        sh[0] = t;
        cj[j] = beta;  // R_jj
      }
    }
    __syncthreads();
    const double t = sh[0];
    if (t != 0.0) {
      for (int c = j + 1 + wid; c < k; c += nw) {
        double* cc = C + c * h;
        double d = 0.0;
        for (int i = j + 1 + lane; i < h; i += 32) d = fma(cj[i], cc[i], d);
        d = warp_sum(d) + cc[j];
        const double td = t * d;
        if (lane == 0) cc[j] -= td;
        for (int i = j + 1 + lane; i < h; i += 32) cc[i] = fma(-td, cj[i], cc[i]);
      }
    }
    if (tid == 0) tau[(int64_t)b * k + j] = t;
    __syncthreads();
  }
  // reflectors out (whole block, LAPACK layout; upper part holds R)
  double* vb = Vbuf + s0 * k;
  for (int idx = tid; idx < k * h; idx += blockDim.x) vb[idx] = C[idx];
  // R_b -> next level stack
  if (Mnext != nullptr)
    for (int idx = tid; idx < k * k; idx += blockDim.x) {
      int c = idx / k, r = idx % k;
      Mnext[(int64_t)c * ldn + (int64_t)b * k + r] = r <= c ? C[c * h + r] : 0.0;
    }
  if (top && tid == 0) {
    bool any = false;
    for (int j = 0; j < k; ++j) any |= (C[j * h + j] != 0.0);
    if (!any) status_fail(st, NENMF_ERR_NUMERICAL_COLLAPSE, -1);
  }
}

// Q_b = H_1 ... H_k [S_b; 0] for each block (LAPACK dorgqr semantics), with
// S_b rows [b k, b k + k) of the level above's Q (or I at the top level).
template <typename TOUT>
__global__ void __launch_bounds__(QR_THREADS)
k_qr_apply(const double* __restrict__ Vbuf, const double* __restrict__ tau, int64_t rows, int k, int nb,
           const double* __restrict__ Qup, int64_t ldu, TOUT* __restrict__ Q, int64_t ldq,
           const nenmf_device_status* __restrict__ st) {
  if (st != nullptr && st->code != 0) return;
  extern __shared__ double C[];  // [k][h]
  const int b = blockIdx.x;
  const int64_t s0 = blk_start(rows, nb, b);
  const int h = (int)(blk_start(rows, nb, b + 1) - s0);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const double* vb = Vbuf + s0 * k;
  for (int idx = tid; idx < k * h; idx += blockDim.x) {
    int c = idx / h, i = idx % h;
    double v = 0.0;
    if (i < k) v = Qup != nullptr ? Qup[(int64_t)c * ldu + (int64_t)b * k + i] : (i == c ? 1.0 : 0.0);
    C[idx] = v;
  }
  __syncthreads();
  for (int j = k - 1; j >= 0; --j) {
    const double t = tau[(int64_t)b * k + j];
    if (t != 0.0) {
      const double* vj = vb + (int64_t)j * h;
      for (int c = wid; c < k; c += nw) {
        double* cc = C + c * h;
        double d = 0.0;
        for (int i = j + 1 + lane; i < h; i += 32) d = fma(__ldg(vj + i), cc[i], d);
        d = warp_sum(d) + cc[j];
        const double td = t * d;
        if (lane == 0) cc[j] -= td;
        for (int i = j + 1 + lane; i < h; i += 32) cc[i] = fma(-td, __ldg(vj + i), cc[i]);
      }
    }
    __syncthreads();
  }
  for (int idx = tid; idx < k * h; idx += blockDim.x) {
    int c = idx / h, i = idx % h;
    Q[(int64_t)c * ldq + s0 + i] = (TOUT)C[idx];
  }
}

struct QrPlan {
  int levels = 0;
  int64_t rows[16];
  int nb[16];
};

inline int plan_qr(int64_t rows, int64_t k, QrPlan& pl) {
  const int hb = qr_block_rows(k);
  int64_t r = rows;
  pl.levels = 0;
  while (true) {
    if (pl.levels >= 16) return NENMF_ERR_UNSUPPORTED;
    pl.rows[pl.levels] = r;
    if (r <= hb) {
      pl.nb[pl.levels] = 1;
      pl.levels++;
      break;
    }
    int nb = (int)cdiv(r, hb);
    pl.nb[pl.levels] = nb;
    pl.levels++;
    r = (int64_t)nb * k;
  }
  return NENMF_OK;
}

template <typename T>
int orthonormalize_cholqr(Arena& ws, T* Pt, int64_t rows, int64_t k, nenmf_device_status* st, cudaStream_t s);
template <typename T>
int orthonormalize_pair(Arena& ws, T* P0t, int64_t rows0, T* P1t, int64_t rows1, int64_t k,
                        nenmf_device_status* st, cudaStream_t s);

// Householder TSQR (kept as the reference-faithful alternative: NENMF_QR=tsqr)
template <typename T>
int orthonormalize_tsqr(Arena& ws, T* Pt, int64_t rows, int64_t k, nenmf_device_status* st, cudaStream_t s) {
  if (rows < 1 || k < 1 || k > rows) return NENMF_ERR_DIM;
  if (k > 64) return NENMF_ERR_UNSUPPORTED;
  QrPlan pl;
  NENMF_TRY(plan_qr(rows, k, pl));
  double* V[16];
  double* tau[16];
  double* Mst[16];  // Mst[l] = input of level l (l >= 1), column-major k x rows[l]
  double* Qb[16];   // Q of level l (l >= 1)
  for (int l = 0; l < pl.levels; ++l) {
    V[l] = ws.take<double>((size_t)pl.rows[l] * k);
    tau[l] = ws.take<double>((size_t)pl.nb[l] * k);
    Mst[l] = l >= 1 ? ws.take<double>((size_t)pl.rows[l] * k) : nullptr;
    Qb[l] = l >= 1 ? ws.take<double>((size_t)pl.rows[l] * k) : nullptr;
  }
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  const int hb = qr_block_rows(k);
  size_t smem = (size_t)k * (hb + 1) * sizeof(double);
  NENMF_CUDA_TRY(set_smem(k_qr_block<T>, smem));
  NENMF_CUDA_TRY(set_smem(k_qr_block<double>, smem));
  NENMF_CUDA_TRY(set_smem(k_qr_apply<T>, smem));
  NENMF_CUDA_TRY(set_smem(k_qr_apply<double>, smem));
  // forward: factor every level
  for (int l = 0; l < pl.levels; ++l) {
    const bool top = l == pl.levels - 1;
    double* next = top ? nullptr : Mst[l + 1];
    int64_t ldn = top ? 0 : pl.rows[l + 1];
    if (l == 0)
      k_qr_block<T><<<pl.nb[0], QR_THREADS, smem, s>>>(Pt, rows, rows, (int)k, pl.nb[0], V[0], tau[0], next, ldn,
                                                        top ? 1 : 0, 1, st);
    else
      k_qr_block<double><<<pl.nb[l], QR_THREADS, smem, s>>>(Mst[l], pl.rows[l], pl.rows[l], (int)k, pl.nb[l], V[l],
                                                             tau[l], next, ldn, top ? 1 : 0, 0, st);
    NENMF_LAUNCH_CHECK();
  }
  // backward: form Q top-down
  for (int l = pl.levels - 1; l >= 0; --l) {
    const bool top = l == pl.levels - 1;
    const double* up = top ? nullptr : Qb[l + 1];
    int64_t ldu = top ? 0 : pl.rows[l + 1];
    if (l == 0)
      k_qr_apply<T><<<pl.nb[0], QR_THREADS, smem, s>>>(V[0], tau[0], rows, (int)k, pl.nb[0], up, ldu, Pt, rows, st);
    else
      k_qr_apply<double><<<pl.nb[l], QR_THREADS, smem, s>>>(V[l], tau[l], pl.rows[l], (int)k, pl.nb[l], up, ldu,
                                                             Qb[l], pl.rows[l], st);
    NENMF_LAUNCH_CHECK();
  }
  return NENMF_OK;
}

template <typename T>
__global__ void k_sub_inplace(T* __restrict__ a, const T* __restrict__ b, int64_t count) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) a[i] -= b[i];
}

// Panels wider than the 64 columns the one-launch factorizations hold (the
// reference takes any nu <= min(n, m), compression.py:109-117): block
// Gram-Schmidt over column blocks of 64.  Every block is projected against
// the finished blocks (C = P_b Q_j^T, P_b -= C Q_j, block by block) and made
// orthonormal by the rank-revealing CholeskyQR2; the sweep runs twice, so the
// rounding of the first projection and the random completion directions of a
// rank-deficient block are orthogonal to the earlier blocks as well.
template <typename T>
static int orthonormalize_blocked(Arena& ws, T* Pt, int64_t rows, int64_t k, nenmf_device_status* st,
                                  cudaStream_t s) {
  if (rows < 1 || k < 1 || k > rows) return NENMF_ERR_DIM;
  constexpr int64_t KB = 64;
  const bool dry = ws.base == nullptr;
  T* C = ws.take<T>((size_t)KB * KB);
  T* V = ws.take<T>((size_t)KB * rows);
  if (!dry && !ws.ok) return NENMF_ERR_WORKSPACE;
  size_t need = 0;
  auto sub = [&](auto&& fn) -> int {  // a sub-step with its own view of the remaining scratch
    Arena a = ws;
    const int rc = fn(a);
    if (a.used - ws.used > need) need = a.used - ws.used;
    if (rc == NENMF_OK && !dry && !a.ok) return NENMF_ERR_WORKSPACE;
    return rc;
  };
  for (int64_t k0 = 0; k0 < k; k0 += KB) {
    const int64_t kb = imin(KB, k - k0);
    T* Pb = dry ? nullptr : Pt + k0 * rows;
    for (int sweep = 0; sweep < 2; ++sweep) {
      for (int64_t j0 = 0; j0 < k0; j0 += KB) {
        const T* Qj = dry ? nullptr : Pt + j0 * rows;
        NENMF_TRY(sub([&](Arena& a) { return abt<T>(a, Pb, kb, Qj, KB, rows, C, s); }));
        NENMF_TRY(sub([&](Arena& a) { return ab<T>(a, C, kb, KB, Qj, rows, rows, false, V, s); }));
        if (!dry) {
          k_sub_inplace<T><<<(unsigned)imin(cdiv(kb * rows, 256), 2368), 256, 0, s>>>(Pb, V, kb * rows);
          NENMF_LAUNCH_CHECK();
        }
      }
      if (sweep == 1 && k0 == 0) break;  // the first block has nothing to be projected against
      NENMF_TRY(sub([&](Arena& a) { return orthonormalize_cholqr<T>(a, Pb, rows, kb, st, s); }));
    }
  }
  if (dry) ws.take<char>(need);
  return NENMF_OK;
}

template <typename T>
int orthonormalize(Arena& ws, T* Pt, int64_t rows, int64_t k, nenmf_device_status* st, cudaStream_t s) {
  const char* e = getenv("NENMF_QR");
  if (k > 64) return orthonormalize_blocked<T>(ws, Pt, rows, k, st, s);
  if (e != nullptr && e[0] == 't') return orthonormalize_tsqr<T>(ws, Pt, rows, k, st, s);
  return orthonormalize_cholqr<T>(ws, Pt, rows, k, st, s);
}

// ====================================================== power iteration ====
// compression.py:144-176 keeps the raw power iterates and checks them for
// overflow after every step.  FP64 runs that arithmetic as is (finiteness
// check per step).  FP32 rescales every iterate by a power of two after each
// pass (exact; the subspace is unchanged) and tracks the exponent per chain,
// so the reference's fp64 overflow is reproduced: step k collapses when an
// iterate's magnitude reaches 2^1024.
struct PowerChains {
  unsigned maxbits[4];  // |x| max of the two panels of the current pass (float bits)
  int bad;              // a non-finite value was seen
  int exp[2];           // accumulated exponents: [0] L-chain (Y), [1] R-chain (Z)
};

__global__ void k_power_stats(const float* __restrict__ P0, int64_t c0, const float* __restrict__ P1, int64_t c1,
                              PowerChains* pc) {
  __shared__ unsigned sm[2];
  __shared__ int sbad;
  if (threadIdx.x < 2) sm[threadIdx.x] = 0u;
  if (threadIdx.x == 0) sbad = 0;
  __syncthreads();
  unsigned m0 = 0u, m1 = 0u;
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c0 + c1; i += stride) {
    const float v = i < c0 ? P0[i] : P1[i - c0];
    bad |= !isfinite(v);
    const unsigned b = __float_as_uint(fabsf(v));
    if (i < c0) m0 = b > m0 ? b : m0;
    else m1 = b > m1 ? b : m1;
  }
  atomicMax(&sm[0], m0);
  atomicMax(&sm[1], m1);
  if (bad) sbad = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicMax(&pc->maxbits[0], sm[0]);
    atomicMax(&pc->maxbits[1], sm[1]);
    if (sbad) atomicExch(&pc->bad, 1);
  }
}

// scale panel i by 2^-e_i (e_i = exponent of its max), add e_i to its chain;
// block 0 / thread 0 also applies the emulated fp64 overflow rule
__global__ void k_power_scale(float* __restrict__ P0, int64_t c0, int chain0, float* __restrict__ P1, int64_t c1,
                              int chain1, PowerChains* pc, int step, nenmf_device_status* st) {
  const float mx0 = __uint_as_float(pc->maxbits[0]), mx1 = __uint_as_float(pc->maxbits[1]);
  const int e0 = mx0 > 0.f ? ilogbf(mx0) : 0, e1 = mx1 > 0.f ? ilogbf(mx1) : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c0 + c1; i += stride) {
    if (i < c0) P0[i] = ldexpf(P0[i], -e0);
    else P1[i - c0] = ldexpf(P1[i - c0], -e1);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int E0 = pc->exp[chain0] + e0, E1 = pc->exp[chain1] + e1;
    pc->exp[chain0] = E0;
    pc->exp[chain1] = E1;
    if (pc->bad || E0 >= 1024 || E1 >= 1024) status_fail(st, NENMF_ERR_NUMERICAL_COLLAPSE, step);
    pc->maxbits[0] = pc->maxbits[1] = 0u;
    pc->bad = 0;
  }
}

template <typename T>
__global__ void k_power_finite(const T* __restrict__ P0, int64_t c0, const T* __restrict__ P1, int64_t c1, int step,
                               nenmf_device_status* st) {
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c0 + c1; i += stride)
    bad |= !isfinite(i < c0 ? P0[i] : P1[i - c0]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) status_fail(st, NENMF_ERR_NUMERICAL_COLLAPSE, step);
}

// a panel column (row of the short-major storage) that is entirely zero
template <typename T>
__global__ void k_zero_rows(const T* __restrict__ P0, int64_t len0, const T* __restrict__ P1, int64_t len1, int k,
                            int step, nenmf_device_status* st) {
  if (st != nullptr && st->code != 0) return;
  const int b = blockIdx.x;
  const T* row = b < k ? P0 + (int64_t)b * len0 : P1 + (int64_t)(b - k) * len1;
  const int64_t len = b < k ? len0 : len1;
  bool any = false;
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) any |= row[i] != T(0);
  if (!__syncthreads_or(any) && threadIdx.x == 0) status_fail(st, NENMF_ERR_NUMERICAL_COLLAPSE, step);
}

// ================================================================= RSI ====
template <typename T>
int rsi(Arena& ws, const T* X, int64_t n, int64_t m, int64_t ldx, const T* omega_l_t, const T* omega_r, int64_t nu,
        int q, T* L, T* Rt, nenmf_device_status* st, cudaStream_t s, const uint8_t* Xpre, int power) {
  if (nu < 1 || nu > min(n, m)) return NENMF_ERR_DIM;
  if (q < 1) return NENMF_ERR_VALUE;
  const bool dry = ws.base == nullptr;
  // FP32: X is split once into the tile-major bf16 hi/lo form every
  // tensor-core pass of the sketch streams (dual_tc.cu)
  bool pre = false;
  if constexpr (sizeof(T) == 4) pre = tc_pass_eligible(n, m, nu);
  // (a caller-prepared copy, nenmf_prepare_x, is used as is)
  const bool own = pre && Xpre == nullptr;
  uint8_t* Xs = own ? ws.take<uint8_t>(tc_presplit_bytes(n, m)) : const_cast<uint8_t*>(Xpre);
  T* tcol = ws.take<T>((size_t)nu * m);  // Q~ of the L-chain (m x nu panel)
  T* trow = ws.take<T>((size_t)nu * n);  // Q~ of the R-chain (n x nu panel)
  PowerChains* pchains = power ? ws.take<PowerChains>(1) : nullptr;
  if (!dry && !ws.ok) return NENMF_ERR_WORKSPACE;
  auto pass = [&](Arena& a, const T* At, const T* Bt, T* Yt, T* Zt) -> int {
    if constexpr (sizeof(T) == 4) {
      if (pre)
        return dual_pass_tc_pre(a, dry ? reinterpret_cast<const uint8_t*>(16) : Xs, n, m,
                                reinterpret_cast<const float*>(At), reinterpret_cast<const float*>(Bt), nu,
                                reinterpret_cast<float*>(Yt), reinterpret_cast<float*>(Zt), s);
    }
    return dual_pass<T>(a, X, n, m, ldx, At, Bt, nu, Yt, Zt, s);
  };
  // scratch of the passes and QRs is reused stage after stage
  Arena scratch = ws;
  size_t need = 0;
  {
    // sizing dry runs: non-null sentinels so both pass outputs are counted
    const T* sent = reinterpret_cast<const T*>(alignof(T));
    Arena a(nullptr, 0);
    if (pre) {
      dual_pass_tc_pre(a, reinterpret_cast<const uint8_t*>(16), n, m, reinterpret_cast<const float*>(sent),
                       reinterpret_cast<const float*>(sent), nu, nullptr, nullptr, s);
    } else {
      dual_pass<T>(a, sent, n, m, ldx, sent, sent, nu, nullptr, nullptr, s);
    }
    need = max(need, a.used);
    Arena b(nullptr, 0);
    orthonormalize<T>(b, L, n, nu, st, s);
    need = max(need, b.used);
    Arena c(nullptr, 0);
    orthonormalize<T>(c, L, m, nu, st, s);
    need = max(need, c.used);
    Arena d(nullptr, 0);
    orthonormalize_pair<T>(d, const_cast<T*>(sent), n, const_cast<T*>(sent), m, nu, st, s);  // both panels counted
    need = max(need, d.used);
    if (power) {
      Arena e1(nullptr, 0), e2(nullptr, 0);
      orthonormalize_tsqr<T>(e1, L, n, nu, st, s);
      orthonormalize_tsqr<T>(e2, L, m, nu, st, s);
      need = max(need, max(e1.used, e2.used));
    }
  }
  char* sbase = scratch.take<char>(need);
  if (dry) {
    ws = scratch;
    return NENMF_OK;
  }
  if (!scratch.ok) return NENMF_ERR_WORKSPACE;
  auto fresh = [&]() { return Arena(sbase, need); };
  if constexpr (sizeof(T) == 4) {
    if (own) NENMF_TRY(tc_presplit(reinterpret_cast<const float*>(X), n, m, ldx, Xs, s));
  }
  // start: Y = X Omega_L -> L (as Q_col^T), Z = X^T Omega_R^T -> Rt (compression.py:134-135)
  { Arena a = fresh(); NENMF_TRY(pass(a, omega_l_t, omega_r, L, Rt)); }
  auto qr2 = [&](T* A, int64_t ra, T* B, int64_t rb) -> int {
    Arena a = fresh();
    const char* e = getenv("NENMF_QR");
    if ((e != nullptr && e[0] == 't') || nu > 64) {  // CholeskyQR2 path holds k <= 64
      NENMF_TRY(orthonormalize<T>(a, A, ra, nu, st, s));
      Arena b = fresh();
      return orthonormalize<T>(b, B, rb, nu, st, s);
    }
    return orthonormalize_pair<T>(a, A, ra, B, rb, nu, st, s);  // both chains in one launch
  };
  // power iteration (compression.py:144-176): no QR between products
  const unsigned eg = (unsigned)imin(1184, cdiv(nu * (n + m), 256));
  auto pscale = [&](T* Yc, int64_t ny, int cy, T* Zc, int64_t nz, int cz, int step) -> int {
    if constexpr (sizeof(T) == 4) {
      k_power_stats<<<eg, 256, 0, s>>>(reinterpret_cast<const float*>(Yc), nu * ny, reinterpret_cast<const float*>(Zc),
                                       nu * nz, pchains);
      NENMF_LAUNCH_CHECK();
      k_power_scale<<<eg, 256, 0, s>>>(reinterpret_cast<float*>(Yc), nu * ny, cy, reinterpret_cast<float*>(Zc),
                                       nu * nz, cz, pchains, step, st);
      NENMF_LAUNCH_CHECK();
    }
    return NENMF_OK;
  };
  if (power) {
    NENMF_CUDA_TRY(cudaMemsetAsync(pchains, 0, sizeof(PowerChains), s));
    NENMF_TRY(pscale(L, n, 0, Rt, m, 1, 1));
  } else {
    NENMF_TRY(qr2(L, n, Rt, m));
  }
  for (int it = 1; it <= q; ++it) {
    // pass a: X^T Q_col (-> tcol, m x nu) and X Q_row (-> trow, n x nu)  (compression.py:138-139)
    { Arena a = fresh(); NENMF_TRY(pass(a, Rt, L, trow, tcol)); }
    if (power) NENMF_TRY(pscale(tcol, m, 0, trow, n, 1, it));
    else NENMF_TRY(qr2(tcol, m, trow, n));
    // pass b: X Q~_col (-> L) and X^T Q~_row (-> Rt)
    { Arena a = fresh(); NENMF_TRY(pass(a, tcol, trow, L, Rt)); }
    if (power) {
      if constexpr (sizeof(T) == 4) NENMF_TRY(pscale(L, n, 0, Rt, m, 1, it));
      else {
        k_power_finite<T><<<eg, 256, 0, s>>>(L, nu * n, Rt, nu * m, it, st);  // compression.py:164-168
        NENMF_LAUNCH_CHECK();
      }
    } else {
      NENMF_TRY(qr2(L, n, Rt, m));
    }
  }
  if (power) {
    // zero column on either side after q steps (compression.py:169-174), then one QR
    // each: Householder TSQR (the raw power iterate has condition ~ (s1/sk)^(2q+1),
    // beyond what a Gram-based QR resolves)
    k_zero_rows<T><<<(unsigned)(2 * nu), 256, 0, s>>>(L, n, Rt, m, (int)nu, q, st);
    NENMF_LAUNCH_CHECK();
    { Arena a = fresh(); NENMF_TRY(orthonormalize_tsqr<T>(a, L, n, nu, st, s)); }
    { Arena a = fresh(); NENMF_TRY(orthonormalize_tsqr<T>(a, Rt, m, nu, st, s)); }
  }
  return NENMF_OK;
}

template <typename T>
int compress(Arena& ws, const T* X, int64_t n, int64_t m, int64_t ldx, const T* L, const T* Rt, int64_t nu, T* XL,
             T* XRt, cudaStream_t s, const uint8_t* Xpre) {
  // X_R^T = Rt X^T (Y side with At = Rt); X_L = L X (Z side with Bt = L)
  if constexpr (sizeof(T) == 4) {
    if (Xpre != nullptr && tc_pass_eligible(n, m, nu))
      return dual_pass_tc_pre(ws, Xpre, n, m, reinterpret_cast<const float*>(Rt), reinterpret_cast<const float*>(L),
                              nu, reinterpret_cast<float*>(XRt), reinterpret_cast<float*>(XL), s);
  }
  return dual_pass<T>(ws, X, n, m, ldx, Rt, L, nu, XRt, XL, s);
}

#define NENMF_INST_RSI(T)                                                                                   \
  template int dual_pass<T>(Arena&, const T*, int64_t, int64_t, int64_t, const T*, const T*, int64_t, T*,   \
                            T*, cudaStream_t);                                                              \
  template int orthonormalize<T>(Arena&, T*, int64_t, int64_t, nenmf_device_status*, cudaStream_t);         \
  template int rsi<T>(Arena&, const T*, int64_t, int64_t, int64_t, const T*, const T*, int64_t, int, T*, T*, \
                      nenmf_device_status*, cudaStream_t, const uint8_t*, int);                             \
  template int compress<T>(Arena&, const T*, int64_t, int64_t, int64_t, const T*, const T*, int64_t, T*, T*, \
                           cudaStream_t, const uint8_t*);
NENMF_INST_RSI(double)
NENMF_INST_RSI(float)

}  // namespace nenmf
