// Orthonormal basis of a tall panel (the role of np.linalg.qr in
// compression.py:88-106) by rank-revealing CholeskyQR2, all on the device.
//
//   G1 = P^T P (fp64, fixed-order split-K)                   k_gram_part  (all SMs)
//   pivoted Cholesky of G1 -> rank r, P Pi = Q1 R11          k_gram_factor (1 CTA)
//   Q1 = P Pi R11^{-1} (row-parallel triangular solves);      k_trsm
//        columns r..k-1 replaced by fixed pseudo-random
//        vectors (the reference's trailing Householder columns of a
//        rank-deficient panel are rounding noise; any orthonormal completion
//        spans the same determined subspace)
//   G2 = Q1^T Q1, Cholesky R2 (no pivoting)                  k_gram_factor (1 CTA)
//   Q  = Q1 R2^{-1}                                          k_trsm
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


namespace nenmf {

constexpr int QC_KMAX = 64;  // panels of up to 64 columns (BASELINE cfg3's p' = 60)

// (Pivoted) Cholesky of a k x k Gram matrix (k <= 32), right-looking, by the
// whole CTA: the Schur complement stays in shared memory S; per step the
// pivot is chosen by warp 0 (largest remaining diagonal, compared on its
// leading 32 bits, lowest index among equals: deterministic), the pivot
// column of R is formed by k threads and the rank-1 update of the remaining
// block by all threads.  Rows of R are produced in pivot order with columns in
// the original index space: P[:, perm] = Q R11 (R11[j][l] = R[j*k + perm[l]]).
// Without pivoting perm is the identity.  A pivot <= rel_tol * max(diag) ends
// it (rank).  R (k*k) is shared scratch.
__device__ void block_factor(double* S_in, int k, int pivot, double rel_tol, double* __restrict__ Rout,
                             int* __restrict__ meta, nenmf_device_status* st) {
  // row stride 64 inside: element (a, b) at a * 64 + b, no integer division
  constexpr int KS = QC_KMAX;
  __shared__ double S[KS * KS];
  __shared__ double Rc[KS];  // the current column of R (remaining rows)
  __shared__ int perm[KS];
  __shared__ int rem[KS];
  __shared__ int s_piv, s_stop, s_bad;
  __shared__ double s_rjj, s_inv, s_tau;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarp = blockDim.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const int kk = k * k;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  for (int a = wid; a < KS; a += nwarp)
    for (int b = lane; b < KS; b += 32) {
      const double v = (a < k && b < k) ? S_in[a * k + b] : 0.0;
      S[a * KS + b] = v;
      if (!isfinite(v)) s_bad = 1;
    }
  for (int e = tid; e < kk; e += blockDim.x) Rout[e] = 0.0;
  if (tid < KS) rem[tid] = tid < k ? 1 : 0;
  __syncthreads();
  if (tid < 32) {
    double mx = fmax(lane < k ? S[lane * (KS + 1)] : 0.0, lane + 32 < k ? S[(lane + 32) * (KS + 1)] : 0.0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
    if (lane == 0) {
      if (!(mx > 0.0)) s_bad = 1;
      s_tau = rel_tol * mx;
    }
  }
  __syncthreads();
  int rank = k;
  if (s_bad) {
    rank = 0;
    if (tid == 0) status_fail(st, NENMF_ERR_NUMERICAL_COLLAPSE, -1);
  } else {
    for (int j = 0; j < k; ++j) {
      if (tid < 32) {
        // lane holds candidate rows lane and lane + 32
        const bool live0 = lane < k && rem[lane], live1 = lane + 32 < k && rem[lane + 32];
        const double d0 = live0 ? S[lane * (KS + 1)] : -1.0;
        const double d1 = live1 ? S[(lane + 32) * (KS + 1)] : -1.0;
        int pj;
        if (pivot) {
          // positive doubles order like their bit patterns: compare the top 32 bits
          const unsigned k0 = d0 > 0.0 ? (unsigned)(__double_as_longlong(d0) >> 32) : 0u;
          const unsigned k1 = d1 > 0.0 ? (unsigned)(__double_as_longlong(d1) >> 32) : 0u;
          const unsigned best = __reduce_max_sync(FULL, k0 > k1 ? k0 : k1);
          const unsigned c0 = __ballot_sync(FULL, live0 && k0 == best);
          const unsigned c1 = __ballot_sync(FULL, live1 && k1 == best);
          pj = c0 ? __ffs(c0) - 1 : (c1 ? 32 + __ffs(c1) - 1 : j);
        } else {
          pj = j;
        }
        const double bv = S[pj * (KS + 1)];
        const bool stop = !(bv > s_tau);
        double rjj = 0.0, inv = 0.0;
        if (!stop) {
          rjj = sqrt(bv);
          inv = 1.0 / rjj;
        }
        // R[j][a] = S[a][pj] / rjj for the remaining rows, rjj at the pivot
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int a = lane + 32 * h;
          const bool live = h == 0 ? live0 : live1;
          const bool other = live && a != pj;
          const double ra = other ? S[a * KS + pj] * inv : (a == pj ? rjj : 0.0);
          if (!stop) {
            Rc[a] = other ? ra : 0.0;
            if (a < k) Rout[j * k + a] = ra;
          }
        }
        if (lane == 0) {
          s_stop = stop;
          s_piv = pj;
          perm[j] = pj;
        }
      }
      __syncthreads();
      if (s_stop) {
        rank = j;
        break;
      }
      if (tid == s_piv) rem[tid] = 0;
      // rank-1 update of the remaining block (Rc is 0 outside it)
      {
        const double rb0 = Rc[lane], rb1 = Rc[lane + 32];
        for (int a = wid; a < k; a += nwarp) {
          const double ra = Rc[a];
          if (ra != 0.0) {
            if (rb0 != 0.0) S[a * KS + lane] = fma(-ra, rb0, S[a * KS + lane]);
            if (rb1 != 0.0) S[a * KS + lane + 32] = fma(-ra, rb1, S[a * KS + lane + 32]);
          }
        }
      }
      __syncthreads();
    }
  }
  __syncthreads();
  for (int i = tid; i < k; i += blockDim.x) meta[1 + i] = i < rank ? perm[i] : -1;
  if (tid == 0) {
    meta[0] = rank;
    if (!pivot && rank < k) status_fail(st, NENMF_ERR_NUMERICAL_COLLAPSE, -1);
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
                                         T* __restrict__ out_t, int64_t row0 = 0) {
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
    if (l < k) out_t[(int64_t)l * rows + i] = (T)(l < r ? q[l] : hash_uniform((uint64_t)(i + row0), (uint64_t)l));
}

// ---------------------------------------------------------------------------
// Decomposed CholeskyQR2: every stage is its own launch so that the Gram
// matrices can be all-reduced between ranks when the panel is row-sharded
// (SURVEY 8(e)); on one GPU the same sequence runs back to back.
//   k_gram_part   Gram partials of row blocks, all SMs      (fixed CTA split)
//   k_gram_factor fixed-order reduction of the partials (+ optional extra
//                 all-reduced input) and the one-warp (pivoted) Cholesky
//   k_trsm        row-parallel triangular solves (+ random completion)
// Up to two panels per launch (the L- and R-chains of RSI).
struct PanelSet {
  const void* in[2];   // short-major panels k x rows[i]
  void* out[2];
  int64_t rows[2];
  int64_t row0[2];     // global index of the first row (random completion hash)
  int cta0[2], ncta[2];
  double* part[2];     // [ncta][k*k]
  double* G[2];        // reduced Gram (k*k); input of the factor when `gin`
  double* R[2];        // k*k
  int* meta[2];        // 1 + k: rank, perm
  int npan;
};

// Gram partials on the FP64 tensor pipe: G = P^T P with DMMA m8n8k4, the
// row block of the CTA split over its 8 warps in 4-row steps.  The A fragment
// (8 columns x 4 rows) and the B fragment of the same column block hold the
// same values, so one fp32->fp64 load per column block feeds both; only the
// upper-triangle tiles are formed and mirrored (G is exactly symmetric).
// Warp partials are summed in warp order (deterministic).
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

template <typename T, int NB>
__global__ void __launch_bounds__(256) k_gram_part(PanelSet P, int k) {
  constexpr int NT = NB * (NB + 1) / 2;  // upper-triangle 8 x 8 tiles
  constexpr int KS = 8 * NB;
  extern __shared__ double qsm[];        // [KS][KS]: the CTA's partial, warps added in order
  const int pi = (P.npan > 1 && (int)blockIdx.x >= P.cta0[1]) ? 1 : 0;
  const int local = (int)blockIdx.x - P.cta0[pi];
  const int64_t rows = P.rows[pi];
  const int64_t r0 = (int64_t)local * rows / P.ncta[pi], r1 = (int64_t)(local + 1) * rows / P.ncta[pi];
  const T* __restrict__ Pt = reinterpret_cast<const T*>(P.in[pi]);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, gq = lane >> 2, tq = lane & 3;
  const int nb = (k + 7) >> 3;  // 8-column blocks in use
  double acc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
  auto load = [&](int64_t r, double (&f)[NB]) {
    const int64_t row = r + tq;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int col = 8 * b + gq;
      f[b] = (b < nb && col < k && row < r1) ? (double)__ldg(&Pt[(int64_t)col * rows + row]) : 0.0;
    }
  };
  double fn[NB];
  load(r0 + 4 * wid, fn);  // software pipelined: the next step's loads are in flight during the DMMAs
  for (int64_t r = r0 + 4 * wid; r < r1; r += 32) {
    double f[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) f[b] = fn[b];
    if (r + 32 < r1) load(r + 32, fn);
    int t = 0;
#pragma unroll
    for (int ma = 0; ma < NB; ++ma)
#pragma unroll
      for (int na = ma; na < NB; ++na, ++t)
        if (na < nb) dmma(acc[t], f[ma], f[na]);
  }
  for (int e = threadIdx.x; e < KS * KS; e += blockDim.x) qsm[e] = 0.0;
  for (int w = 0; w < 8; ++w) {
    __syncthreads();
    if (wid == w) {
      int t = 0;
#pragma unroll
      for (int ma = 0; ma < NB; ++ma)
#pragma unroll
        for (int na = ma; na < NB; ++na, ++t) {
          if (na >= nb) continue;
          const int i = 8 * ma + gq, j = 8 * na + 2 * tq;
          qsm[i * KS + j] += acc[t][0];
          qsm[i * KS + j + 1] += acc[t][1];
          if (ma != na) {  // mirror (G is exactly symmetric)
            qsm[j * KS + i] += acc[t][0];
            qsm[(j + 1) * KS + i] += acc[t][1];
          }
        }
    }
  }
  __syncthreads();
  double* out = P.part[pi] + (int64_t)local * k * k;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int a = e / k, b = e - a * k;
    out[e] = qsm[a * KS + b];
  }
}

// one CTA per panel: G = sum of partials in CTA order (then written to P.G),
// or G read from P.G when the partials were reduced elsewhere (gin);
// factorisation into P.R / P.meta
constexpr int GF_THREADS = 1024;  // more loads in flight for the partial reduction
__global__ void __launch_bounds__(GF_THREADS) k_gram_factor(PanelSet P, int k, int pivot, double tol, int gin,
                                                     nenmf_device_status* st) {
  extern __shared__ double qsm[];
  double* S = qsm;
  const int pi = blockIdx.x;
  const int kk = k * k;
  if (st != nullptr && st->code != 0) {
    if (threadIdx.x == 0) P.meta[pi][0] = 0;
    return;
  }
  if (gin) {
    for (int e = threadIdx.x; e < kk; e += blockDim.x) S[e] = P.G[pi][e];
  } else {
    const double* part = P.part[pi];
    const int nc = P.ncta[pi];
    // 8 independent loads in flight per thread; fixed order (deterministic)
    for (int e = threadIdx.x; e < kk; e += blockDim.x) {
      double sv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) sv[u] = 0.0;
      int c = 0;
      for (; c + 8 <= nc; c += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(part + (int64_t)(c + u) * kk + e);
#pragma unroll
        for (int u = 0; u < 8; ++u) sv[u] += v[u];
      }
      for (; c < nc; ++c) sv[0] += __ldcg(part + (int64_t)c * kk + e);
      S[e] = ((sv[0] + sv[1]) + (sv[2] + sv[3])) + ((sv[4] + sv[5]) + (sv[6] + sv[7]));
      if (P.G[pi] != nullptr) P.G[pi][e] = S[e];
    }
  }
  __syncthreads();
  if (pivot < 0) return;
  block_factor(S, k, pivot, tol, P.R[pi], P.meta[pi], st);
}

template <typename T, int KM>
__global__ void __launch_bounds__(256) k_trsm(PanelSet P, int k, int full_only) {
  __shared__ double R[QC_KMAX * QC_KMAX];
  __shared__ int perm[QC_KMAX];
  __shared__ double rdinv[QC_KMAX];
  const int pi = (P.npan > 1 && (int)blockIdx.x >= P.cta0[1]) ? 1 : 0;
  const int local = (int)blockIdx.x - P.cta0[pi];
  const int r = P.meta[pi][0];
  if (r <= 0 || (full_only && r < k)) return;
  const int kk = k * k;
  for (int e = threadIdx.x; e < kk; e += blockDim.x) R[e] = P.R[pi][e];
  for (int i = threadIdx.x; i < k; i += blockDim.x) perm[i] = P.meta[pi][1 + i];
  __syncthreads();
  for (int i = threadIdx.x; i < r; i += blockDim.x) rdinv[i] = 1.0 / R[i * k + perm[i]];
  __syncthreads();
  const int64_t rows = P.rows[pi];
  const int64_t r0 = (int64_t)local * rows / P.ncta[pi], r1 = (int64_t)(local + 1) * rows / P.ncta[pi];
  const T* in_t = reinterpret_cast<const T*>(P.in[pi]);
  T* out_t = reinterpret_cast<T*>(P.out[pi]);
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x)
    trsm_row<T, KM>(in_t, rows, k, R, perm, rdinv, r, i, out_t, P.row0[pi]);
}

inline size_t gram_smem(int k) { return (size_t)(k <= 32 ? 32 * 32 : 64 * 64) * sizeof(double); }
inline size_t factor_smem(int k) { return (size_t)k * k * sizeof(double); }

// CTAs per panel: the whole GPU shared by the panels, >= 256 rows per CTA
// (the one-CTA factor kernel reduces the per-CTA Gram partials)
inline void split_ctas(PanelSet& P) {
  int sms = sm_count();
  if (sms <= 0) sms = 148;
  int64_t tot = 0;
  for (int i = 0; i < P.npan; ++i) tot += P.rows[i];
  int c0 = 0;
  for (int i = 0; i < P.npan; ++i) {
    static const int64_t min_rows = [] {
      const char* e = getenv("NENMF_QR_ROWS");  // development knob (timing experiments)
      return (int64_t)(e != nullptr ? atoi(e) : 256);
    }();
    const int64_t want = imax(1, imin(cdiv(P.rows[i], min_rows), (int64_t)sms * P.rows[i] / imax(tot, 1)));
    P.ncta[i] = (int)imax(1, want);
    P.cta0[i] = c0;
    c0 += P.ncta[i];
  }
}

template <typename T>
int launch_gram_part(PanelSet& P, int k, cudaStream_t s) {
  const size_t smem = gram_smem(k);
  const unsigned grid = P.cta0[P.npan - 1] + P.ncta[P.npan - 1];
  if (k <= 32) {
    NENMF_CUDA_TRY(set_smem(k_gram_part<T, 4>, smem));
    k_gram_part<T, 4><<<grid, 256, smem, s>>>(P, k);
  } else {
    NENMF_CUDA_TRY(set_smem(k_gram_part<T, 8>, smem));
    k_gram_part<T, 8><<<grid, 256, smem, s>>>(P, k);
  }
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

int launch_gram_factor(PanelSet& P, int k, int pivot, double tol, int gin, nenmf_device_status* st,
                       cudaStream_t s) {
  NENMF_CUDA_TRY(set_smem(k_gram_factor, factor_smem(k)));
  k_gram_factor<<<P.npan, GF_THREADS, factor_smem(k), s>>>(P, k, pivot, tol, gin, st);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

template <typename T>
int launch_trsm(PanelSet& P, int k, int full_only, cudaStream_t s) {
  const unsigned grid = P.cta0[P.npan - 1] + P.ncta[P.npan - 1];
  if (k <= 32) k_trsm<T, 32><<<grid, 256, 0, s>>>(P, k, full_only);
  else k_trsm<T, 64><<<grid, 256, 0, s>>>(P, k, full_only);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

template <typename T>
int orthonormalize_pair(Arena& ws, T* P0t, int64_t rows0, T* P1t, int64_t rows1, int64_t k,
                        nenmf_device_status* st, cudaStream_t s) {
  if (k < 1 || k > QC_KMAX || rows0 < k || (P1t != nullptr && rows1 < k)) return k > QC_KMAX ? NENMF_ERR_UNSUPPORTED : NENMF_ERR_DIM;
  PanelSet P{};
  P.npan = P1t != nullptr ? 2 : 1;
  T* ptv[2] = {P0t, P1t};
  const int64_t rowsv[2] = {rows0, rows1};
  T* q1[2] = {nullptr, nullptr};
  for (int i = 0; i < P.npan; ++i) {
    P.rows[i] = rowsv[i];
    P.row0[i] = 0;
  }
  split_ctas(P);
  for (int i = 0; i < P.npan; ++i) {
    P.part[i] = ws.take<double>((size_t)P.ncta[i] * k * k);
    P.R[i] = ws.take<double>((size_t)k * k);
    P.meta[i] = ws.take<int>((size_t)k + 4);
    q1[i] = ws.take<T>((size_t)k * rowsv[i]);
    P.G[i] = nullptr;
  }
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  const int kint = (int)k;
  // pass 1: rank-revealing pivoted Cholesky of P^T P, Q1 = P Pi R11^-1 (+ completion)
  for (int i = 0; i < P.npan; ++i) {
    P.in[i] = ptv[i];
    P.out[i] = q1[i];
  }
  NENMF_TRY(launch_gram_part<T>(P, kint, s));
  NENMF_TRY(launch_gram_factor(P, kint, 1, 1e-14, 0, st, s));
  NENMF_TRY(launch_trsm<T>(P, kint, 0, s));
  // pass 2: Cholesky of Q1^T Q1 (no pivoting), Q = Q1 R2^-1 back into the panel
  for (int i = 0; i < P.npan; ++i) {
    P.in[i] = q1[i];
    P.out[i] = ptv[i];
  }
  NENMF_TRY(launch_gram_part<T>(P, kint, s));
  NENMF_TRY(launch_gram_factor(P, kint, 0, 1e-300, 0, st, s));
  NENMF_TRY(launch_trsm<T>(P, kint, 1, s));
  return NENMF_OK;
}

// ---- sharded building blocks (C ABI: nenmf_panel_*) ----------------------
template <typename T>
int panel_gram(Arena& ws, const T* Pt, int64_t rows, int64_t k, double* G, cudaStream_t s) {
  if (k < 1 || k > QC_KMAX || rows < 1) return k > QC_KMAX ? NENMF_ERR_UNSUPPORTED : NENMF_ERR_DIM;
  PanelSet P{};
  P.npan = 1;
  P.rows[0] = rows;
  split_ctas(P);
  P.part[0] = ws.take<double>((size_t)P.ncta[0] * k * k);
  P.R[0] = ws.take<double>((size_t)k * k);
  P.meta[0] = ws.take<int>((size_t)k + 4);
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  P.in[0] = Pt;
  P.G[0] = G;
  NENMF_TRY(launch_gram_part<T>(P, (int)k, s));
  // reduce only (the factorisation runs after the cross-rank all-reduce):
  // k_gram_factor with pivot = -1 stops after writing G
  NENMF_CUDA_TRY(set_smem(k_gram_factor, factor_smem((int)k)));
  k_gram_factor<<<1, GF_THREADS, factor_smem((int)k), s>>>(P, (int)k, -1, 0.0, 0, nullptr);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

int panel_factor(const double* G, int64_t k, int pivot, double* R, int* meta, nenmf_device_status* st,
                 cudaStream_t s) {
  if (k < 1 || k > QC_KMAX) return k > QC_KMAX ? NENMF_ERR_UNSUPPORTED : NENMF_ERR_DIM;
  PanelSet P{};
  P.npan = 1;
  P.G[0] = const_cast<double*>(G);
  P.R[0] = R;
  P.meta[0] = meta;
  return launch_gram_factor(P, (int)k, pivot, pivot ? 1e-14 : 1e-300, 1, st, s);
}

template <typename T>
int panel_trsm(const T* Pin_t, int64_t rows, int64_t k, const double* R, const int* meta, T* Pout_t, int64_t row0,
               int full_only, cudaStream_t s) {
  if (k < 1 || k > QC_KMAX || rows < 1) return k > QC_KMAX ? NENMF_ERR_UNSUPPORTED : NENMF_ERR_DIM;
  PanelSet P{};
  P.npan = 1;
  P.rows[0] = rows;
  P.row0[0] = row0;
  split_ctas(P);
  P.in[0] = Pin_t;
  P.out[0] = Pout_t;
  P.R[0] = const_cast<double*>(R);
  P.meta[0] = const_cast<int*>(meta);
  return launch_trsm<T>(P, (int)k, full_only, s);
}

template int panel_gram<double>(Arena&, const double*, int64_t, int64_t, double*, cudaStream_t);
template int panel_gram<float>(Arena&, const float*, int64_t, int64_t, double*, cudaStream_t);
template int panel_trsm<double>(const double*, int64_t, int64_t, const double*, const int*, double*, int64_t, int,
                                cudaStream_t);
template int panel_trsm<float>(const float*, int64_t, int64_t, const double*, const int*, float*, int64_t, int,
                               cudaStream_t);

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


