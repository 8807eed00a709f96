// Compressed / vanilla NeNMF inner solver on sm_100a.
//
// Restates nnls.py:119-227 (solve_nnls) and matrix.py:131-174 (Lipschitz
// constant by power iteration) as:
//
//   abt  W = A^T A               (skinny.cu)
//   ab   V = A^T B               (skinny.cu; B may be a transposed view of X)
//   k_power                      lambda_max(Gram) with the reference's seeded
//                                start vectors, 1.01 inflation, zero check
//   k_nnls  (persistent, cooperative)  the whole inner loop in ONE launch
//   resid + k_decide + k_select  _true_objective tie-break (nnls.py:219-227)
//
// k_nnls: every CTA owns a slab of columns of F (columns are independent
// except for the two global sums per iteration that drive the stop/best
// decisions, nnls.py:194-203).  Iterates are computed speculatively up to D
// iterations ahead of those decisions: each CTA publishes its per-iteration
// partial sums to a tagged slot ring and resolves iteration j once every CTA
// has published j, in fixed CTA order (deterministic, identical in all CTAs).
// The barrier latency of a grid-wide reduction is thereby overlapped with the
// next D iterations instead of being paid every iteration.  A ring of the last
// D+2 iterates lets a late "iteration j is the new best" decision still copy
// F_j; a late "stop at j" discards the speculative iterates after j.
#include "nnls.cuh"
#include "skinny.cuh"

#include <cooperative_groups.h>

namespace nenmf {

struct __align__(32) Slot {
  double pg2, fg, fv;
  unsigned long long tag;
};

constexpr int NN_D = 8;               // speculation depth
constexpr int NN_RING = NN_D + 2;     // iterate ring slots
constexpr int NN_SLOTS = 2 * NN_D + 2;

// -------------------------------------------------------------- helpers ----
__device__ __forceinline__ double alpha_next_d(double a) {
  // (1 + sqrt(4*a*a + 1)) / 2 with NumPy's rounding sequence (nnls.py:68-69)
  return __ddiv_rn(__dadd_rn(1.0, sqrt(__dadd_rn(__dmul_rn(__dmul_rn(4.0, a), a), 1.0))), 2.0);
}

__device__ __forceinline__ bool finite_d(double x) { return isfinite(x); }

// -------------------------------------------------------- gram (r < p) ----
template <typename T>
__global__ void k_gram_rows(const T* __restrict__ At, int p, int r, T* __restrict__ G) {
  // G (r x r) = A A^T with A = At^T (matrix.py:170, the cols > rows branch)
  for (int o = threadIdx.x; o < r * r; o += blockDim.x) {
    int s = o / r, t = o % r;
    double acc = 0.0;
    for (int a = 0; a < p; ++a) acc = fma((double)At[(int64_t)a * r + s], (double)At[(int64_t)a * r + t], acc);
    G[o] = (T)acc;
  }
}

// ---------------------------------------------------------------- power ----
// matrix.py:131-155 in double: v from the seeded stream, w = G v, nw = ||w||,
// restart from the next stream vector if nw == 0, stop on relative change,
// x1.01 if max_iters ran out; then *= safety; est == 0 -> ZeroMatrixError.
template <typename T>
__global__ void __launch_bounds__(128)
k_power(const T* __restrict__ G, int k, const double* __restrict__ vecs, int count, double tol,
        int max_iters, double safety, double* __restrict__ Lout, nenmf_device_status* st) {
  extern __shared__ double sm[];
  double* Gs = sm;              // k*k
  double* v = Gs + k * k;       // k
  double* w = v + k;            // k
  __shared__ double red[33];
  for (int i = threadIdx.x; i < k * k; i += blockDim.x) Gs[i] = (double)G[i];
  for (int i = threadIdx.x; i < k; i += blockDim.x) v[i] = vecs[i];
  __syncthreads();
  int draw = 1;
  double est = 0.0;
  bool converged = false;
  for (int it = 0; it < max_iters; ++it) {
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
      double acc = 0.0;
      for (int l = 0; l < k; ++l) acc = fma(Gs[i * k + l], v[l], acc);
      w[i] = acc;
    }
    __syncthreads();
    double part = 0.0;
    for (int i = threadIdx.x; i < k; i += blockDim.x) part = fma(w[i], w[i], part);
    const double nw = sqrt(block_sum(part, red));
    if (nw == 0.0) {
      // the reference re-draws a fresh start vector (matrix.py:146-149)
      for (int i = threadIdx.x; i < k; i += blockDim.x) v[i] = draw < count ? vecs[(int64_t)draw * k + i] : 0.0;
      ++draw;
      __syncthreads();
      continue;
    }
    const bool conv = fabs(nw - est) <= tol * nw;
    est = nw;
    for (int i = threadIdx.x; i < k; i += blockDim.x) v[i] = __ddiv_rn(w[i], nw);
    __syncthreads();
    if (conv) {
      converged = true;
      break;
    }
  }
  if (!converged) est = est * 1.01;
  if (threadIdx.x == 0) {
    const double L = safety * est;
    *Lout = L;
    if (st != nullptr) st->lipschitz = L;
    if (est == 0.0) status_fail(st, NENMF_ERR_ZERO_MATRIX, 0);
  }
}

// ------------------------------------------------------------- solver ----
template <typename T, int PMAX>
__global__ void __launch_bounds__(256, 1)
k_nnls(const T* __restrict__ W, const T* __restrict__ V, const T* __restrict__ F0, T* __restrict__ Fbest,
       T* __restrict__ ring, T* __restrict__ g2, int p, int64_t c, int64_t cpb, const double* __restrict__ Lptr,
       int max_iter, double grad_tol, Slot* __restrict__ slots, nenmf_device_status* st) {
  __shared__ T Ws[PMAX * PMAX];
  __shared__ double red[3][33];
  __shared__ double bc[3];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  const int G = gridDim.x;
  const int64_t j0 = (int64_t)blockIdx.x * cpb;
  const int64_t j1 = min(c, j0 + cpb);
  const int64_t pc = (int64_t)p * c;

  for (int i = tid; i < p * p; i += blockDim.x) Ws[i] = W[i];
  if (st->code != 0) return;  // an earlier stage failed (uniform across CTAs)
  const double L = *Lptr;
  const T negL = (T)(-L);
  __syncthreads();

  // fixed-order CTA reduction of three doubles -> slot (tag = j + 2)
  auto publish = [&](int j, double a0, double a1, double a2) {
    a0 = warp_sum(a0);
    a1 = warp_sum(a1);
    a2 = warp_sum(a2);
    if (lane == 0) {
      red[0][wid] = a0;
      red[1][wid] = a1;
      red[2][wid] = a2;
    }
    __syncthreads();
    if (tid == 0) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      for (int w = 0; w < nwarps; ++w) {
        s0 += red[0][w];
        s1 += red[1][w];
        s2 += red[2][w];
      }
      Slot* sl = slots + (int64_t)((j + 1) % NN_SLOTS) * G + blockIdx.x;
      sl->pg2 = s0;
      sl->fg = s1;
      sl->fv = s2;
      st_release_u64(reinterpret_cast<uint64_t*>(&sl->tag), (uint64_t)(j + 2));
    }
    __syncthreads();
  };

  // --- start point: g = W F0 - V; pg_ref and partial_start (nnls.py:163-178)
  {
    double apg = 0.0, afg = 0.0, afv = 0.0;
    for (int64_t j = j0 + tid; j < j1; j += blockDim.x) {
      T f[PMAX];
#pragma unroll
      for (int l = 0; l < PMAX; ++l) f[l] = l < p ? F0[(int64_t)l * c + j] : T(0);
      for (int i = 0; i < p; ++i) {
        T acc = T(0);
#pragma unroll
        for (int l = 0; l < PMAX; ++l)
          if (l < p) acc = fma_acc(Ws[i * p + l], f[l], acc);
        const T vv = V[(int64_t)i * c + j];
        const T g = op_sub(acc, vv);
        g2[(int64_t)i * c + j] = g;
        g2[pc + (int64_t)i * c + j] = g;
        T fi = F0[(int64_t)i * c + j];
        const double pgv = (double)(fi > T(0) ? g : min0_nan(g));
        apg += pgv * pgv;
        afg += (double)fi * (double)g;
        afv += (double)fi * (double)vv;
      }
    }
    publish(-1, apg, afg, afv);
  }

  // --- decision state (identical in every CTA)
  int resolved = -2;    // last resolved iteration (-1 = start point)
  int best_j = -1;
  double best_part = 0.0, pg_ref = 0.0;
  int stop_at = -1;     // iteration whose pg met the tolerance
  bool halted = false;  // stop or failure

  auto resolve = [&](int j) {
    if (wid == 0) {
      const Slot* row = slots + (int64_t)((j + 1) % NN_SLOTS) * G;
      const uint64_t want = (uint64_t)(j + 2);
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      for (int b = lane; b < G; b += 32) {
        const Slot* sl = row + b;
        while (ld_acquire_u64(reinterpret_cast<const uint64_t*>(&sl->tag)) != want) {
        }
        s0 += sl->pg2;
        s1 += sl->fg;
        s2 += sl->fv;
      }
      s0 = warp_sum(s0);
      s1 = warp_sum(s1);
      s2 = warp_sum(s2);
      if (lane == 0) {
        bc[0] = s0;
        bc[1] = s1;
        bc[2] = s2;
      }
    }
    __syncthreads();
    const double pg = sqrt(bc[0]);
    const double part = 0.5 * (bc[1] - bc[2]);
    __syncthreads();
    resolved = j;
    if (j < 0) {
      pg_ref = pg;
      best_part = part;
      if (!(finite_d(part) && finite_d(pg) && finite_d(L))) {
        if (blockIdx.x == 0 && tid == 0) status_fail(st, NENMF_ERR_NUMERICAL_FAILURE, 0);
        halted = true;
      }
      return;
    }
    if (!(finite_d(pg) && finite_d(part))) {
      if (blockIdx.x == 0 && tid == 0) status_fail(st, NENMF_ERR_NUMERICAL_FAILURE, j);
      halted = true;
      return;
    }
    if (part < best_part) {
      best_part = part;
      best_j = j;
      const T* src = ring + (int64_t)(j % NN_RING) * pc;
      for (int64_t jj = j0 + tid; jj < j1; jj += blockDim.x)
        for (int l = 0; l < p; ++l) Fbest[(int64_t)l * c + jj] = src[(int64_t)l * c + jj];
    }
    if (pg <= grad_tol * pg_ref) {
      stop_at = j;
      halted = true;
    }
  };

  double alpha = 1.0, w_prev = 0.0;  // w_{k-1}; w_{-1} = 0 gives Y_0 = F0
  int k = 0;
  for (; k < max_iter; ++k) {
    while (!halted && resolved < k - 1 - NN_D) resolve(resolved + 1);
    if (halted) break;
    const T* F1 = k >= 1 ? ring + (int64_t)((k - 1) % NN_RING) * pc : F0;
    const T* F2 = k >= 2 ? ring + (int64_t)((k - 2) % NN_RING) * pc : F0;
    const T* G1 = g2 + (int64_t)((k - 1) & 1) * pc;
    T* G2 = g2 + (int64_t)(k & 1) * pc;  // holds g_{k-2}; receives g_k
    T* Fk = ring + (int64_t)(k % NN_RING) * pc;
    const T w = (T)w_prev;
    double apg = 0.0, afg = 0.0, afv = 0.0;
    for (int64_t j = j0 + tid; j < j1; j += blockDim.x) {
      T f[PMAX];
#pragma unroll
      for (int l = 0; l < PMAX; ++l) {
        if (l < p) {
          const int64_t o = (int64_t)l * c + j;
          const T f1 = F1[o], f2 = F2[o], q1 = G1[o], q2 = G2[o];
          // Y = (F_{k-1} - F_{k-2}) w + F_{k-1};  grad_Y likewise (nnls.py:208-213)
          const T y = op_add(op_mul(op_sub(f1, f2), w), f1);
          const T gy = op_add(op_mul(op_sub(q1, q2), w), q1);
          // F_k = max(0, Y + grad_Y / (-L))  (nnls.py:189-191)
          f[l] = relu_nan(op_add(op_div(gy, negL), y));
          Fk[o] = f[l];
        } else {
          f[l] = T(0);
        }
      }
#pragma unroll
      for (int i = 0; i < PMAX; ++i) {
        if (i >= p) break;
        T acc = T(0);
#pragma unroll
        for (int l = 0; l < PMAX; ++l)
          if (l < p) acc = fma_acc(Ws[i * p + l], f[l], acc);
        const int64_t o = (int64_t)i * c + j;
        const T vv = V[o];
        const T g = op_sub(acc, vv);  // g_k = W F_k - V (nnls.py:192-193)
        G2[o] = g;
        const T fi = f[i];
        const double pgv = (double)(fi > T(0) ? g : min0_nan(g));
        apg += pgv * pgv;
        afg += (double)fi * (double)g;
        afv += (double)fi * (double)vv;
      }
    }
    publish(k, apg, afg, afv);
    const double a1 = alpha_next_d(alpha);
    w_prev = __ddiv_rn(alpha - 1.0, a1);
    alpha = a1;
  }
  while (!halted && resolved < k - 1) resolve(resolved + 1);

  if (blockIdx.x == 0 && tid == 0) {
    st->inner_iters = stop_at >= 0 ? stop_at + 1 : (st->code != 0 ? st->iteration : max_iter);
    st->returned_best = best_j >= 0 ? 1 : 0;
    st->best_partial = best_part;
    st->pg_ref = pg_ref;
  }
}

// the explicit-residual tie-break (nnls.py:219-227): best unless
// 1/2||A best - B||^2 > 1/2||A start - B||^2 (each as float(norm)**2 / 2)
__global__ void k_decide(const double* __restrict__ r2, nenmf_device_status* st) {
  if (st->returned_best == 0) return;
  const double nb = sqrt(r2[0]), ns = sqrt(r2[1]);
  const double tb = 0.5 * (nb * nb), ts = 0.5 * (ns * ns);
  st->resid[0] = tb;
  st->resid[1] = ts;
  if (!(tb <= ts)) st->returned_best = 0;
}

template <typename T>
__global__ void k_select(const T* __restrict__ F0, T* __restrict__ Fout, int64_t count,
                         const nenmf_device_status* __restrict__ st) {
  if (st->code != 0 || st->returned_best != 0) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) Fout[i] = F0[i];
}

// ------------------------------------------------------------- drivers ----
template <typename T>
static int lipschitz(Arena& ws, const T* At, int64_t r, int64_t p, const T* W, const double* pvec, int pcount,
                     int pmax, double ptol, double safety, double* Lout, nenmf_device_status* st, cudaStream_t s) {
  const int64_t k = min(r, p);
  if (k > 64) return NENMF_ERR_UNSUPPORTED;
  const T* gram = W;
  T* gsmall = nullptr;
  if (p > r) gsmall = ws.take<T>((size_t)k * k);
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  if (p > r) {
    k_gram_rows<T><<<1, 256, 0, s>>>(At, (int)p, (int)r, gsmall);
    NENMF_LAUNCH_CHECK();
    gram = gsmall;
  }
  size_t smem = ((size_t)k * k + 2 * k) * sizeof(double);
  NENMF_CUDA_TRY(cudaFuncSetAttribute(k_power<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_power<T><<<1, 128, smem, s>>>(gram, (int)k, pvec, pcount, ptol, pmax, safety, Lout, st);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

template <typename T, int PMAX>
static int launch_nnls(const T* W, const T* V, const T* F0, T* Fbest, T* ring, T* g2, int p, int64_t c,
                       const double* Lptr, int max_iter, double grad_tol, Slot* slots,
                       nenmf_device_status* st, int grid, int threads, cudaStream_t s) {
  int64_t cpb = cdiv(c, grid);
  void* args[] = {(void*)&W, (void*)&V, (void*)&F0, (void*)&Fbest, (void*)&ring, (void*)&g2, (void*)&p,
                  (void*)&c, (void*)&cpb, (void*)&Lptr, (void*)&max_iter, (void*)&grad_tol, (void*)&slots,
                  (void*)&st};
  NENMF_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_nnls<T, PMAX>, dim3(grid), dim3(threads), args, 0, s));
  launch_counter_add(1);
  return NENMF_OK;
}

template <typename T>
static int nnls_grid(int64_t c, int& grid, int& threads) {
  int sms = sm_count();
  if (sms <= 0) sms = 148;
  grid = (int)imax(1, imin(sms, cdiv(c, 32)));
  int64_t cpb = cdiv(c, grid);
  threads = (int)imin(256, imax(32, cdiv(cpb, 32) * 32));
  return NENMF_OK;
}

template <typename T>
int solve_nnls(Arena& ws, const T* At, int64_t r, int64_t p, const T* B, int64_t c, int64_t ldb, bool trans,
               const T* F0, T* Fout, int max_iter, double grad_tol, double safety, const double* pvec,
               int pcount, int pmax, double ptol, nenmf_device_status* st, cudaStream_t s) {
  if (r < 1 || p < 1 || c < 1) return NENMF_ERR_DIM;
  if (p > 64) return NENMF_ERR_UNSUPPORTED;
  if (max_iter < 1 || pcount < 1) return NENMF_ERR_VALUE;
  const bool dry = ws.base == nullptr;
  int grid = 1, threads = 32;
  nnls_grid<T>(c, grid, threads);
  const int64_t pc = p * c;
  T* W = ws.take<T>((size_t)p * p);
  T* V = ws.take<T>((size_t)pc);
  double* Lbuf = ws.take<double>(4);
  T* ring = ws.take<T>((size_t)NN_RING * pc);
  T* g2 = ws.take<T>((size_t)2 * pc);
  Slot* slots = ws.take<Slot>((size_t)NN_SLOTS * grid);
  if (!dry && !ws.ok) return NENMF_ERR_WORKSPACE;
  NENMF_TRY(abt<T>(ws, At, p, At, p, r, W, s));                       // W = A^T A   (nnls.py:157)
  NENMF_TRY(ab<T>(ws, At, p, r, B, c, ldb, trans, V, s));             // V = A^T B   (nnls.py:158)
  NENMF_TRY(lipschitz<T>(ws, At, r, p, W, pvec, pcount, pmax, ptol, safety, Lbuf, st, s));  // (nnls.py:159)
  if (!dry) {
    NENMF_CUDA_TRY(cudaMemsetAsync(slots, 0, sizeof(Slot) * NN_SLOTS * grid, s));
    if (p <= 8) NENMF_TRY((launch_nnls<T, 8>(W, V, F0, Fout, ring, g2, (int)p, c, Lbuf, max_iter, grad_tol, slots, st, grid, threads, s)));
    else if (p <= 16) NENMF_TRY((launch_nnls<T, 16>(W, V, F0, Fout, ring, g2, (int)p, c, Lbuf, max_iter, grad_tol, slots, st, grid, threads, s)));
    else if (p <= 32) NENMF_TRY((launch_nnls<T, 32>(W, V, F0, Fout, ring, g2, (int)p, c, Lbuf, max_iter, grad_tol, slots, st, grid, threads, s)));
    else NENMF_TRY((launch_nnls<T, 64>(W, V, F0, Fout, ring, g2, (int)p, c, Lbuf, max_iter, grad_tol, slots, st, grid, threads, s)));
  }
  // explicit residuals of best and start, only when an iterate improved (nnls.py:219-227)
  NENMF_TRY(resid<T>(ws, At, p, r, B, c, ldb, trans, Fout, F0, Lbuf + 2, &st->returned_best, s));
  if (dry) return NENMF_OK;
  k_decide<<<1, 1, 0, s>>>(Lbuf + 2, st);
  NENMF_LAUNCH_CHECK();
  k_select<T><<<(unsigned)imin(cdiv(pc, 256), 1184), 256, 0, s>>>(F0, Fout, pc, st);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

template <typename T>
int spectral_norm_sq(Arena& ws, const T* At, int64_t r, int64_t p, const double* pvec, int pcount, int pmax,
                     double tol, double* out, nenmf_device_status* st, cudaStream_t s) {
  if (r < 1 || p < 1) return NENMF_ERR_DIM;
  if (min(r, p) > 64) return NENMF_ERR_UNSUPPORTED;
  T* W = p <= r ? ws.take<T>((size_t)p * p) : nullptr;
  if (ws.base != nullptr && !ws.ok) return NENMF_ERR_WORKSPACE;
  if (p <= r) NENMF_TRY(abt<T>(ws, At, p, At, p, r, W, s));
  return lipschitz<T>(ws, At, r, p, W, pvec, pcount, pmax, tol, 1.0, out, st, s);
}

template <typename T>
int gradient(Arena& ws, const T* At, int64_t r, int64_t p, const T* B, int64_t c, int64_t ldb, bool trans,
             const T* F, T* grad, cudaStream_t s) {
  if (r < 1 || p < 1 || c < 1) return NENMF_ERR_DIM;
  T* W = ws.take<T>((size_t)p * p);
  T* V = ws.take<T>((size_t)p * c);
  if (ws.base != nullptr && !ws.ok) return NENMF_ERR_WORKSPACE;
  NENMF_TRY(abt<T>(ws, At, p, At, p, r, W, s));
  NENMF_TRY(ab<T>(ws, At, p, r, B, c, ldb, trans, V, s));
  if (ws.base == nullptr) return NENMF_OK;
  return wf_minus_v<T>(W, p, F, c, V, grad, s);
}

#define NENMF_INST_NNLS(T)                                                                                    \
  template int solve_nnls<T>(Arena&, const T*, int64_t, int64_t, const T*, int64_t, int64_t, bool, const T*,  \
                             T*, int, double, double, const double*, int, int, double, nenmf_device_status*,   \
                             cudaStream_t);                                                                  \
  template int spectral_norm_sq<T>(Arena&, const T*, int64_t, int64_t, const double*, int, int, double, double*, \
                                   nenmf_device_status*, cudaStream_t);                                      \
  template int gradient<T>(Arena&, const T*, int64_t, int64_t, const T*, int64_t, int64_t, bool, const T*,    \
                           T*, cudaStream_t);
NENMF_INST_NNLS(double)
NENMF_INST_NNLS(float)

}  // namespace nenmf
