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

// (Pivoted) Cholesky of a k x k Gram matrix (k <= 64), right-looking, by ONE
// warp of the CTA (the others wait at the closing barrier): the Schur
// complement stays in shared memory S (row stride 65: conflict-free column
// reads), lane l owns rows l and l + 32 and keeps their current diagonal in
// registers.  Per step: the pivot is the largest remaining diagonal, compared
// on its leading 32 bits, lowest index among equals (deterministic); the
// pivot column of R comes from one shared-memory read per row; the rank-1
// update of the remaining block broadcasts the column with warp shuffles.
// No CTA barrier inside the k-step loop (a CTA-wide version spent ~1 us per
// step in its two barriers).  Rows of R are produced in pivot order with
// columns in the original index space: P[:, perm] = Q R11 (R11[j][l] =
// R[j*k + perm[l]]).  Without pivoting perm is the identity.  A pivot <=
// rel_tol * max(diag) ends it (rank).  Rout (k*k) and meta may be shared or
// global memory.
__device__ void block_factor(double* S_in, int k, int pivot, double rel_tol, double* __restrict__ Rout,
                             int* __restrict__ meta, nenmf_device_status* st) {
  constexpr int KS = QC_KMAX;
  constexpr int LD = KS + 1;
  __shared__ double S[KS * LD];
  __shared__ int perm[KS];
  __shared__ int s_rank, s_bad;
  const int tid = threadIdx.x, lane = tid & 31;
  const unsigned FULL = 0xffffffffu;
  const int kk = k * k;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  bool nonfinite = false;
  for (int e = tid; e < KS * KS; e += blockDim.x) {
    const int a = e >> 6, b = e & (KS - 1);
    const double v = (a < k && b < k) ? S_in[a * k + b] : 0.0;
    S[a * LD + b] = v;
    nonfinite |= !isfinite(v);
  }
  if (nonfinite) s_bad = 1;
  for (int e = tid; e < kk; e += blockDim.x) Rout[e] = 0.0;
  __syncthreads();
  if (tid < 32 && k <= 32) {
    // k <= 32: lane a holds row a of the Schur complement in registers; the
    // pivot column entry is selected by an unrolled compare (no dynamic
    // register index) and the update broadcasts the column by shuffles
    double row[32];
#pragma unroll
    for (int bcol = 0; bcol < 32; ++bcol) row[bcol] = S[lane * LD + bcol];
    bool live = lane < k;
    double dg = live ? row[0] : 0.0;
#pragma unroll
    for (int bcol = 1; bcol < 32; ++bcol)
      if (bcol == lane) dg = row[bcol];
    if (!live) dg = 0.0;
    double mx = dg;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
    const bool bad = s_bad || !(mx > 0.0);
    const double tau = rel_tol * mx;
    int rank = k;
    if (bad) {
      rank = 0;
    } else {
      for (int j = 0; j < k; ++j) {
        int pj;
        if (pivot) {
          const unsigned k0 = live && dg > 0.0 ? (unsigned)(__double_as_longlong(dg) >> 32) : 0u;
          const unsigned best = __reduce_max_sync(FULL, k0);
          const unsigned c0 = __ballot_sync(FULL, live && k0 == best);
          pj = c0 ? __ffs(c0) - 1 : j;
        } else {
          pj = j;
        }
        const double bv = __shfl_sync(FULL, dg, pj);
        if (!(bv > tau)) {
          rank = j;
          break;
        }
        // inv and rjj from one reciprocal square root (instead of sqrt then a
        // division on the step's critical path)
        const double inv = rsqrt(bv), rjj = bv * inv;
        // row[pj] by a 5-level select tree (pj is warp-uniform)
        double v16[16], v8[8], v4[4], v2[2];
#pragma unroll
        for (int u = 0; u < 16; ++u) v16[u] = (pj & 1) ? row[2 * u + 1] : row[2 * u];
#pragma unroll
        for (int u = 0; u < 8; ++u) v8[u] = (pj & 2) ? v16[2 * u + 1] : v16[2 * u];
#pragma unroll
        for (int u = 0; u < 4; ++u) v4[u] = (pj & 4) ? v8[2 * u + 1] : v8[2 * u];
#pragma unroll
        for (int u = 0; u < 2; ++u) v2[u] = (pj & 8) ? v4[2 * u + 1] : v4[2 * u];
        const double sp = (pj & 16) ? v2[1] : v2[0];
        const double ra = live ? (lane == pj ? rjj : sp * inv) : 0.0;
        if (lane < k) Rout[j * k + lane] = ra;
        if (lane == 0) perm[j] = pj;
        if (lane == pj) live = false;
        const double rc = live ? ra : 0.0;
        // rank-1 update (rc = 0 outside the remaining block leaves rows unchanged)
#pragma unroll
        for (int bcol = 0; bcol < 32; ++bcol) row[bcol] = fma(-rc, __shfl_sync(FULL, rc, bcol), row[bcol]);
        dg = fma(-rc, rc, dg);
      }
    }
    if (lane == 0) {
      s_rank = rank;
      if (bad) s_bad = 1;
    }
  } else if (k > 32 && tid < 64) {
    // 32 < k <= 64: two warps, lane l of warp w holds row 32 w + l in
    // registers (64 doubles); per step the warps exchange their pivot
    // candidates and their pivot-column entries through shared memory
    // (named barrier 1, 64 threads)
    __shared__ unsigned s_key[2];
    __shared__ int s_idx[2];
    __shared__ double rcv[64];
    const int w = tid >> 5, a = tid;
    double row[64];
#pragma unroll
    for (int bcol = 0; bcol < 64; ++bcol) row[bcol] = S[a * LD + bcol];
    bool live = a < k;
    double dg = live ? S[a * LD + a] : 0.0;
    double mx = dg;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
    if (lane == 0) rcv[w] = mx;
    asm volatile("bar.sync 1, 64;" ::: "memory");
    mx = fmax(rcv[0], rcv[1]);
    const bool bad = s_bad || !(mx > 0.0);
    const double tau = rel_tol * mx;
    int rank = k;
    if (bad) {
      rank = 0;
    } else {
      for (int j = 0; j < k; ++j) {
        int pj;
        if (pivot) {
          const unsigned kk0 = live && dg > 0.0 ? (unsigned)(__double_as_longlong(dg) >> 32) : 0u;
          const unsigned best = __reduce_max_sync(FULL, kk0);
          const unsigned c0 = __ballot_sync(FULL, live && kk0 == best);
          asm volatile("bar.sync 1, 64;" ::: "memory");  // previous step's readers are done
          if (lane == 0) {
            s_key[w] = best;
            s_idx[w] = c0 ? 32 * w + __ffs(c0) - 1 : 1 << 30;
          }
          asm volatile("bar.sync 1, 64;" ::: "memory");
          // larger key wins; equal keys: the lower index (warp 0 first)
          pj = s_key[1] > s_key[0] ? s_idx[1] : (s_key[0] > s_key[1] ? s_idx[0] : min(s_idx[0], s_idx[1]));
          if (pj >= (1 << 30)) pj = j;
        } else {
          pj = j;
        }
        // the pivot's diagonal, from its owner
        asm volatile("bar.sync 1, 64;" ::: "memory");
        if (a == pj) rcv[0] = dg;
        asm volatile("bar.sync 1, 64;" ::: "memory");
        const double bv = rcv[0];
        if (!(bv > tau)) {
          rank = j;
          break;
        }
        const double inv = rsqrt(bv), rjj = bv * inv;
        double v32[32], v16[16], v8[8], v4[4], v2[2];
#pragma unroll
        for (int u = 0; u < 32; ++u) v32[u] = (pj & 1) ? row[2 * u + 1] : row[2 * u];
#pragma unroll
        for (int u = 0; u < 16; ++u) v16[u] = (pj & 2) ? v32[2 * u + 1] : v32[2 * u];
#pragma unroll
        for (int u = 0; u < 8; ++u) v8[u] = (pj & 4) ? v16[2 * u + 1] : v16[2 * u];
#pragma unroll
        for (int u = 0; u < 4; ++u) v4[u] = (pj & 8) ? v8[2 * u + 1] : v8[2 * u];
#pragma unroll
        for (int u = 0; u < 2; ++u) v2[u] = (pj & 16) ? v4[2 * u + 1] : v4[2 * u];
        const double sp = (pj & 32) ? v2[1] : v2[0];
        const double ra = live ? (a == pj ? rjj : sp * inv) : 0.0;
        if (a < k) Rout[j * k + a] = ra;
        if (tid == 0) perm[j] = pj;
        if (a == pj) live = false;
        const double rc = live ? ra : 0.0;
        asm volatile("bar.sync 1, 64;" ::: "memory");  // everyone has read rcv[0]
        rcv[a] = rc;
        asm volatile("bar.sync 1, 64;" ::: "memory");
#pragma unroll
        for (int bcol = 0; bcol < 64; ++bcol) row[bcol] = fma(-rc, rcv[bcol], row[bcol]);
        dg = fma(-rc, rc, dg);
      }
    }
    if (tid == 0) {
      s_rank = rank;
      if (bad) s_bad = 1;
    }
  }
  __syncthreads();
  const int rank = s_rank;
  for (int i = tid; i < k; i += blockDim.x) meta[1 + i] = i < rank ? perm[i] : -1;
  if (tid == 0) {
    meta[0] = rank;
    if (s_bad) status_fail(st, NENMF_ERR_NUMERICAL_COLLAPSE, -1);
    else if (!pivot && rank < k) status_fail(st, NENMF_ERR_NUMERICAL_COLLAPSE, -1);
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
// Rows [r0, r1) of the panel: solve q R11 = z with z_l = in[perm[l]] (l < r),
// i.e. Q = P[:, perm] R11^{-1}; columns l >= r get fixed pseudo-random
// values.  Rp is R11 already permuted into pivot order (Rp[j][l] =
// R[j][perm[l]], row stride KM, shared memory).  Each thread solves one row
// at a time, its entries kept in a column of zs ([KM][TPR] shared doubles,
// conflict-free).  Blocked by 8 columns: a block's 8 entries sit in
// registers, take the contributions of all earlier entries (8 independent
// FMAs per earlier entry, broadcast loads of R), then the 8 x 8 triangle is
// solved in registers.  The loops over blocks and earlier entries stay
// rolled (a fully unrolled solve made the kernel miss in the instruction
// cache: ncu showed 31 % no_inst stalls).
template <typename T, int KM, int TPR>
__device__ void solve_rows(const T* __restrict__ in_t, int64_t rows, int k, const double* __restrict__ Rp,
                           const int* __restrict__ perm, const double* __restrict__ rdinv, int r, int64_t r0,
                           int64_t r1, T* __restrict__ out_t, int64_t row0, double* __restrict__ zs) {
  const int t = threadIdx.x;
  if (t >= TPR) return;
  double* __restrict__ z = zs + t;
  for (int64_t i = r0 + t; i < r1; i += TPR) {
    // all loads of the row in flight at once (a load-convert-store loop
    // waited one memory latency per entry)
    {
      T v[KM];
#pragma unroll
      for (int l = 0; l < KM; ++l) v[l] = l < r ? in_t[(int64_t)perm[l] * rows + i] : T(0);
#pragma unroll
      for (int l = 0; l < KM; ++l)
        if (l < r) z[l * TPR] = (double)v[l];
    }
    for (int c0 = 0; c0 < r; c0 += 8) {
      double acc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] = c0 + u < r ? z[(c0 + u) * TPR] : 0.0;
      for (int j = 0; j < c0; ++j) {
        const double qj = z[j * TPR];
        const double2* rj = reinterpret_cast<const double2*>(Rp + j * KM + c0);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double2 rv = rj[u];
          acc[2 * u] = fma(-qj, rv.x, acc[2 * u]);
          acc[2 * u + 1] = fma(-qj, rv.y, acc[2 * u + 1]);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (c0 + u < r) {
          acc[u] *= rdinv[c0 + u];
#pragma unroll
          for (int v = u + 1; v < 8; ++v) acc[v] = fma(-acc[u], Rp[(c0 + u) * KM + c0 + v], acc[v]);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (c0 + u < r) z[(c0 + u) * TPR] = acc[u];
    }
    for (int l = 0; l < k; ++l)
      out_t[(int64_t)l * rows + i] = (T)(l < r ? z[l * TPR] : hash_uniform((uint64_t)(i + row0), (uint64_t)l));
  }
}

// Rp (KM x KM, pivot order) and 1 / diag from the factor's R (k x k rows in
// pivot order, columns in the original index space) and perm
__device__ __forceinline__ void permute_r(const double* R, const int* perm, int k, int r, int KM, double* Rp,
                                          double* rdinv) {
  for (int e = threadIdx.x; e < KM * KM; e += blockDim.x) {
    const int j = e / KM, l = e - j * KM;
    Rp[e] = (j < r && l < r) ? R[j * k + perm[l]] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < r; i += blockDim.x) rdinv[i] = 1.0 / Rp[i * KM + i];
  __syncthreads();
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

// phase timestamps of CTA 0's last launch (development aid: tools/micro/qr_phases.cu)
__device__ unsigned long long g_qr_phase[24];
__device__ long long g_qr_cyc[24];
__device__ __forceinline__ void qr_stamp(int i) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_qr_phase[i] = t;
    g_qr_cyc[i] = clock64();
  }
}

// The Gram partial of rows [r0, r1) of a short-major panel (k x rows) by the
// whole CTA (256 threads) into out (k x k); qsm: (8 NB)^2 doubles of shared
// memory.
template <typename T, int NB>
__device__ __forceinline__ void gram_partial_block(const T* __restrict__ Pt, int64_t rows, int64_t r0, int64_t r1,
                                                   int k, double* qsm, double* __restrict__ out) {
  constexpr int NT = NB * (NB + 1) / 2;  // upper-triangle 8 x 8 tiles
  constexpr int KS = 8 * NB;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, gq = lane >> 2, tq = lane & 3;
  const int nb = (k + 7) >> 3;  // 8-column blocks in use
  double acc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
  // raw values stay in their storage type until used, so no conversion makes
  // the warp wait for a load issued ahead of time
  auto load = [&](int64_t r, T (&f)[NB]) {
    const int64_t row = r + tq;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int col = 8 * b + gq;
      f[b] = (b < nb && col < k && row < r1) ? __ldcg(&Pt[(int64_t)col * rows + row]) : T(0);
    }
  };
  // software pipeline PD steps deep: the loads of the next PD - 1 row steps
  // are in flight during a step's DMMAs (one step ahead left every step
  // waiting a memory latency)
  constexpr int PD = NB <= 4 ? 4 : 2;
  T fn[PD][NB];
#pragma unroll
  for (int d = 0; d < PD; ++d) load(r0 + 4 * wid + 32 * d, fn[d]);
  for (int64_t r = r0 + 4 * wid; r < r1; r += 32 * PD) {
#pragma unroll
    for (int d = 0; d < PD; ++d) {
      double f[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) f[b] = (double)fn[d][b];
      load(r + 32 * (d + PD), fn[d]);
      int t = 0;
#pragma unroll
      for (int ma = 0; ma < NB; ++ma)
#pragma unroll
        for (int na = ma; na < NB; ++na, ++t)
          if (na < nb) dmma(acc[t], f[ma], f[na]);
    }
  }
  // cross-warp sum in fixed warp order (0 + w0 + w1 + ... + w7): every warp
  // stores its fragments (no read-modify-write chains in shared memory), then
  // every output entry is summed independently; NB = 8 in two rounds of 4 warps
  constexpr int WPR = NB <= 4 ? 8 : 4;  // warps per round
  double* frag = qsm;                    // [WPR][NT][64]
  double sum[(KS * KS + 255) / 256];
#pragma unroll
  for (int u = 0; u < (KS * KS + 255) / 256; ++u) sum[u] = 0.0;
#pragma unroll
  for (int round = 0; round < 8 / WPR; ++round) {
    __syncthreads();
    if (wid / WPR == round) {
      double* fw = frag + (size_t)(wid % WPR) * NT * 64;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        fw[t * 64 + gq * 8 + 2 * tq] = acc[t][0];
        fw[t * 64 + gq * 8 + 2 * tq + 1] = acc[t][1];
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < (KS * KS + 255) / 256; ++u) {
      const int e = u * 256 + threadIdx.x;
      if (e < k * k) {
        const int a = e / k, b = e - a * k;
        const int i = a <= b ? a : b, j = a <= b ? b : a;
        const int ma = i >> 3, na = j >> 3;
        const int t = ma * NB - ma * (ma - 1) / 2 + (na - ma);
        // diagonal tiles hold both triangles; off-diagonal ones the upper block
        const int el = (ma == na) ? (a & 7) * 8 + (b & 7) : (i & 7) * 8 + (j & 7);
#pragma unroll
        for (int w = 0; w < WPR; ++w) sum[u] += frag[((size_t)w * NT + t) * 64 + el];
      }
    }
  }
#pragma unroll
  for (int u = 0; u < (KS * KS + 255) / 256; ++u) {
    const int e = u * 256 + threadIdx.x;
    if (e < k * k) out[e] = sum[u];
  }
  __syncthreads();
}

template <typename T, int NB>
__global__ void __launch_bounds__(256) k_gram_part(PanelSet P, int k) {
  extern __shared__ double qsm[];        // [KS][KS]: the CTA's partial, warps added in order
  const int pi = (P.npan > 1 && (int)blockIdx.x >= P.cta0[1]) ? 1 : 0;
  const int local = (int)blockIdx.x - P.cta0[pi];
  const int64_t rows = P.rows[pi];
  const int64_t r0 = (int64_t)local * rows / P.ncta[pi], r1 = (int64_t)(local + 1) * rows / P.ncta[pi];
  gram_partial_block<T, NB>(reinterpret_cast<const T*>(P.in[pi]), rows, r0, r1, k, qsm,
                            P.part[pi] + (int64_t)local * k * k);
}

// fixed-order sum of the ncta Gram partials of one entry (8 independent loads
// in flight; the order of k_gram_factor)
__device__ __forceinline__ double reduce_partials(const double* __restrict__ part, int nc, int kk, int e) {
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
  return ((sv[0] + sv[1]) + (sv[2] + sv[3])) + ((sv[4] + sv[5]) + (sv[6] + sv[7]));
}

// one CTA per panel: G = sum of partials in CTA order (then written to P.G),
// or G read from P.G when the partials were reduced elsewhere (gin);
// factorisation into P.R / P.meta
constexpr int GF_THREADS = 256;  // the factor runs in registers of one warp (<= 255 per thread)
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
      S[e] = reduce_partials(part, nc, kk, e);
      if (P.G[pi] != nullptr) P.G[pi][e] = S[e];
    }
  }
  __syncthreads();
  if (pivot < 0) return;
  block_factor(S, k, pivot, tol, P.R[pi], P.meta[pi], st);
}

template <typename T, int KM>
__global__ void __launch_bounds__(256) k_trsm(PanelSet P, int k, int full_only) {
  constexpr int TPR = KM <= 32 ? 256 : 128;
  extern __shared__ double tsm[];  // R [KM*KM] | Rp [KM*KM] | zs [KM][TPR]
  __shared__ int perm[QC_KMAX];
  __shared__ double rdinv[QC_KMAX];
  double* R = tsm;
  double* Rp = tsm + KM * KM;
  double* zs = Rp + KM * KM;
  const int pi = (P.npan > 1 && (int)blockIdx.x >= P.cta0[1]) ? 1 : 0;
  const int local = (int)blockIdx.x - P.cta0[pi];
  const int r = P.meta[pi][0];
  if (r <= 0 || (full_only && r < k)) return;
  const int kk = k * k;
  for (int e = threadIdx.x; e < kk; e += blockDim.x) R[e] = P.R[pi][e];
  for (int i = threadIdx.x; i < k; i += blockDim.x) perm[i] = P.meta[pi][1 + i];
  __syncthreads();
  permute_r(R, perm, k, r, KM, Rp, rdinv);
  const int64_t rows = P.rows[pi];
  const int64_t r0 = (int64_t)local * rows / P.ncta[pi], r1 = (int64_t)(local + 1) * rows / P.ncta[pi];
  solve_rows<T, KM, TPR>(reinterpret_cast<const T*>(P.in[pi]), rows, k, Rp, perm, rdinv, r, r0, r1,
                         reinterpret_cast<T*>(P.out[pi]), P.row0[pi], zs);
}

template <int KM>
constexpr size_t trsm_smem() {
  return (2 * (size_t)KM * KM + (size_t)KM * (KM <= 32 ? 256 : 128)) * sizeof(double);
}

// per-warp Gram fragments (gram_partial_block): 8 warps x 10 tiles (k <= 32)
// or 4 warps x 36 tiles (k <= 64) of 64 doubles
inline size_t gram_smem(int k) { return (size_t)(k <= 32 ? 8 * 10 * 64 : 4 * 36 * 64) * sizeof(double); }
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
    const int64_t want = imax(1, imin(cdiv(P.rows[i], min_rows), (int64_t)(sms - P.npan + 1) * P.rows[i] / imax(tot, 1)));
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
  if (k <= 32) {
    NENMF_CUDA_TRY(set_smem(k_trsm<T, 32>, trsm_smem<32>()));
    k_trsm<T, 32><<<grid, 256, trsm_smem<32>(), s>>>(P, k, full_only);
  } else {
    NENMF_CUDA_TRY(set_smem(k_trsm<T, 64>, trsm_smem<64>()));
    k_trsm<T, 64><<<grid, 256, trsm_smem<64>(), s>>>(P, k, full_only);
  }
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

// ---------------------------------------------------------------------------
// CholeskyQR2 of up to two panels in ONE cooperative launch (one CTA per SM,
// the panels' row blocks split over the grid as above).  The stages are the
// ones of the decomposed path, separated by grid barriers instead of launches:
//   A  Gram partials of the CTA's rows                          (all CTAs)
//   B  fixed-order reduction of the partials, entries split over the panel's CTAs
//   C  every CTA factors the reduced Gram itself (pivoted, rank-revealing;
//      the same input and code give the same R in every CTA), solves its rows
//      into Q1 (+ the random completion), then forms the Gram partial of its
//      rows of Q1
//   D  reduction as B
//   E  every CTA factors Q1^T Q1 (no pivoting) and solves its rows of Q into
//      the panel
// Four grid barriers replace six launches, two of them one-CTA factor kernels
// (the RSI passes' main fixed cost before).  Results equal the decomposed
// path's bit for bit (same partials, same reduction order, same factor).
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

template <typename T, int NB>
__global__ void __launch_bounds__(256) k_cholqr2(PanelSet P, int k, unsigned* bar, nenmf_device_status* st) {
  constexpr int KM = 8 * NB;
  constexpr int TPR = KM <= 32 ? 256 : 128;
  // Gram fragments (phases A, C) | later: factor input [KM*KM] | Rs [KM*KM] | Rp [KM*KM] | zs [KM][TPR]
  extern __shared__ double qsm[];
  double* Rs = qsm + KM * KM;
  double* Rp = Rs + KM * KM;
  double* zs = Rp + KM * KM;
  __shared__ int meta[KM + 4];
  __shared__ int ident[KM];
  __shared__ double rdinv[KM];
  for (int i = threadIdx.x; i < KM; i += blockDim.x) ident[i] = i;
  const unsigned G = gridDim.x;
  const int pi = (P.npan > 1 && (int)blockIdx.x >= P.cta0[1]) ? 1 : 0;
  const int local = (int)blockIdx.x - P.cta0[pi];
  const int nc = P.ncta[pi];
  const int64_t rows = P.rows[pi];
  const int64_t r0 = (int64_t)local * rows / nc, r1 = (int64_t)(local + 1) * rows / nc;
  const int kk = k * k;
  T* panel = reinterpret_cast<T*>(P.out[pi]);
  T* q1 = reinterpret_cast<T*>(const_cast<void*>(P.in[pi]));  // scratch Q1 (k x rows)
  double* part = P.part[pi];
  double* Gr = P.G[pi];
  const bool skip = st != nullptr && st->code != 0;  // an earlier stage failed: leave the panel alone
  qr_stamp(0);
  // A
  if (!skip) gram_partial_block<T, NB>(panel, rows, r0, r1, k, qsm, part + (int64_t)local * kk);
  qr_stamp(1);
  grid_barrier(bar, G);
  qr_stamp(2);
  // B
  if (!skip)
    for (int e = local * 256 + threadIdx.x; e < kk; e += nc * 256) Gr[e] = reduce_partials(part, nc, kk, e);
  qr_stamp(3);
  grid_barrier(bar, 2 * G);
  qr_stamp(4);
  // C
  int rank = 0;
  if (!skip) {
    for (int e = threadIdx.x; e < kk; e += blockDim.x) qsm[e] = __ldcg(&Gr[e]);
    __syncthreads();
    block_factor(qsm, k, 1, 1e-14, Rs, meta, blockIdx.x == 0 ? st : nullptr);
    qr_stamp(5);
    rank = meta[0];
    if (rank > 0) {
      permute_r(Rs, meta + 1, k, rank, KM, Rp, rdinv);
      qr_stamp(14);
      solve_rows<T, KM, TPR>(panel, rows, k, Rp, meta + 1, rdinv, rank, r0, r1, q1, P.row0[pi], zs);
      __syncthreads();
      qr_stamp(15);
      gram_partial_block<T, NB>(q1, rows, r0, r1, k, qsm, part + (int64_t)local * kk);
    }
  }
  qr_stamp(6);
  grid_barrier(bar, 3 * G);
  qr_stamp(7);
  // D
  if (rank > 0)
    for (int e = local * 256 + threadIdx.x; e < kk; e += nc * 256) Gr[e] = reduce_partials(part, nc, kk, e);
  qr_stamp(8);
  grid_barrier(bar, 4 * G);
  qr_stamp(9);
  // E
  if (rank > 0) {
    for (int e = threadIdx.x; e < kk; e += blockDim.x) qsm[e] = __ldcg(&Gr[e]);
    __syncthreads();
    block_factor(qsm, k, 0, 1e-300, Rs, meta, blockIdx.x == 0 ? st : nullptr);
    qr_stamp(10);
    if (meta[0] == k) {
      permute_r(Rs, ident, k, k, KM, Rp, rdinv);
      solve_rows<T, KM, TPR>(q1, rows, k, Rp, ident, rdinv, k, r0, r1, panel, P.row0[pi], zs);
    }
  }
  qr_stamp(11);
}

template <typename T>
int launch_cholqr2(PanelSet& P, int k, unsigned* bar, nenmf_device_status* st, cudaStream_t s) {
  const unsigned grid = P.cta0[P.npan - 1] + P.ncta[P.npan - 1];
  const size_t smem = std::max(gram_smem(k), k <= 32 ? (3 * 32 * 32 + 32 * 256) * sizeof(double)
                                                     : (3 * 64 * 64 + 64 * 128) * sizeof(double));
  NENMF_CUDA_TRY(cudaMemsetAsync(bar, 0, sizeof(unsigned), s));
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (k <= 32) {
    NENMF_CUDA_TRY(set_smem(k_cholqr2<T, 4>, smem));
    NENMF_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_cholqr2<T, 4>, P, k, bar, st));
  } else {
    NENMF_CUDA_TRY(set_smem(k_cholqr2<T, 8>, smem));
    NENMF_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_cholqr2<T, 8>, P, k, bar, st));
  }
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
  unsigned* bar = ws.take<unsigned>(4);
  double* gred[2] = {ws.take<double>((size_t)k * k), P.npan > 1 ? ws.take<double>((size_t)k * k) : nullptr};
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  const int kint = (int)k;
  static const bool staged = [] {
    const char* e = getenv("NENMF_QR");  // development switch: the decomposed launches
    return e != nullptr && e[0] == 's';
  }();
  if (!staged) {
    for (int i = 0; i < P.npan; ++i) {
      P.in[i] = q1[i];  // scratch Q1
      P.out[i] = ptv[i];
      P.G[i] = gred[i];
    }
    return launch_cholqr2<T>(P, kint, bar, st, s);
  }
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


