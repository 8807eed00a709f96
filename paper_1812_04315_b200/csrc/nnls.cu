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
// Block = NCW compute warps + 1 resolver warp.
//
// Compute warps: TPC threads per column (same warp).  Per iteration k each
// thread forms its share of F_k = max(0, Y + grad_Y / (-L)) from F_{k-1},
// F_{k-2}, g_{k-1}, g_{k-2} (nnls.py:189-191,208-213), the column's TPC
// threads exchange F_k through the state buffer, then each computes its rows
// of g_k = W F_k - V (nnls.py:192-193) and its part of the three sums
// ||PG||^2, <F,g>, <F,V> (nnls.py:194-195).  Thread 0 of the compute group
// publishes the CTA's sums for k (slot + release-increment of a counter) and
// throttles the group to stay at most D iterations ahead of the decisions.
// State (two F and two g buffers) lives in shared memory when it fits, else
// in global memory; F_k also goes to a global ring of R = D + 2 iterates.
//
// Resolver warp: polls the per-iteration counters of up to 32 iterations at
// once, sums every CTA's slot in fixed order (identical in all CTAs), and
// applies the reference's decisions in order: finiteness (nnls.py:177,196),
// strict-improvement best tracking (:198-201), KKT stop (:202-203).  It
// publishes best_j / resolved / halt through shared memory.  Before a ring
// slot is overwritten, a column whose iterate is the current best copies it to
// F_out (lazy best copy: the common "best moves forward" case costs nothing).
template <typename T, int PMAX, int TPC, bool SMEM>
__global__ void __launch_bounds__(1024, 1)
k_nnls(const T* __restrict__ W, const T* __restrict__ V, const T* __restrict__ F0, T* __restrict__ Fout,
       T* __restrict__ ring, T* __restrict__ gstate, int p, int64_t c, int64_t cpb, int ldS,
       const double* __restrict__ Lptr, int max_iter, double grad_tol, Slot* __restrict__ slots,
       unsigned int* __restrict__ counts, nenmf_device_status* st) {
  extern __shared__ double smem_d[];
  T* Ws = reinterpret_cast<T*>(smem_d);                                   // p*p
  double* part = smem_d + (((size_t)PMAX * PMAX * sizeof(T) + 7) / 8);    // [2][32][3]
  T* Sbase = reinterpret_cast<T*>(part + 2 * 32 * 3);                    // SMEM: [4][p][ldS]
  __shared__ volatile int s_resolved, s_best_j, s_halt, s_go;
  __shared__ int s_stop_at, s_fail_at, s_kdone;
  __shared__ double s_best_part, s_pg_ref;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ncw = (blockDim.x >> 5) - 1;  // compute warps
  const int nct = ncw * 32;
  const bool resolver = wid == ncw;
  const int G = gridDim.x;
  const int64_t j0 = (int64_t)blockIdx.x * cpb;
  const int64_t ncols = imin(c, j0 + cpb) - j0;
  const int64_t pc = (int64_t)p * c;

  for (int i = tid; i < p * p; i += blockDim.x) Ws[i] = W[i];
  if (tid == 0) {
    s_resolved = -2;
    s_best_j = -1;
    s_halt = 0;
    s_go = 1;
    s_stop_at = -1;
    s_fail_at = -1;
    s_best_part = 0.0;
    s_pg_ref = 0.0;
  }
  __syncthreads();
  if (st->code != 0) return;  // an earlier stage failed (uniform across CTAs)
  const double L = *Lptr;
  const T negL = (T)(-L);

  // state buffers: b = 0,1 -> F parity buffers, b = 2,3 -> g parity buffers
  // element (l, col) of buffer b; col is CTA-local in SMEM mode, global otherwise
  auto sref = [&](int b, int l, int64_t cl) -> T& {
    if (SMEM) return Sbase[((size_t)b * p + l) * ldS + cl];
    return gstate[(int64_t)b * pc + (int64_t)l * c + j0 + cl];
  };

  if (!resolver) {
    // ---------------------------------------------------------- compute warps
    const int sub = tid % TPC;           // row share of this thread
    const int64_t cstride = nct / TPC;   // columns handled per sweep
    const int64_t c_first = tid / TPC;
    double apg = 0.0, afg = 0.0, afv = 0.0;

    // start point: g = W F0 - V, pg_ref and partial objective (nnls.py:163-178)
    for (int64_t cl = c_first; cl < ncols; cl += cstride) {
      const int64_t j = j0 + cl;
      for (int l = sub; l < p; l += TPC) {
        const T f = F0[(int64_t)l * c + j];
        sref(0, l, cl) = f;
        sref(1, l, cl) = f;
      }
      __syncwarp();
      T f[PMAX];
#pragma unroll
      for (int l = 0; l < PMAX; ++l) f[l] = l < p ? sref(1, l, cl) : T(0);
      for (int i = sub; i < p; i += TPC) {
        T acc = T(0);
#pragma unroll
        for (int l = 0; l < PMAX; ++l)
          if (l < p) acc = fma_acc(Ws[i * p + l], f[l], acc);
        const T vv = __ldg(V + (int64_t)i * c + j);
        const T g = op_sub(acc, vv);
        sref(2, i, cl) = g;
        sref(3, i, cl) = g;
        const T fi = sref(1, i, cl);
        const double pgv = (double)(fi > T(0) ? g : min0_nan(g));
        apg += pgv * pgv;
        afg += (double)fi * (double)g;
        afv += (double)fi * (double)vv;
      }
    }

    auto publish = [&](int j) {
      double a0 = warp_sum(apg), a1 = warp_sum(afg), a2 = warp_sum(afv);
      double* pp = part + (size_t)((j + 2) & 1) * 96;
      if (lane == 0) {
        pp[wid * 3 + 0] = a0;
        pp[wid * 3 + 1] = a1;
        pp[wid * 3 + 2] = a2;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(nct) : "memory");
      if (tid == 0) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
        for (int w = 0; w < ncw; ++w) {
          s0 += pp[w * 3 + 0];
          s1 += pp[w * 3 + 1];
          s2 += pp[w * 3 + 2];
        }
        const int slot = (j + 1) % NN_SLOTS;
        Slot* sl = slots + (int64_t)slot * G + blockIdx.x;
        sl->pg2 = s0;
        sl->fg = s1;
        sl->fv = s2;
        __threadfence();
        atomicAdd(counts + slot, 1u);
        // throttle: iteration j+1 may start once j+1 - D - 1 is resolved
        while (s_resolved < j - NN_D && !s_halt) __nanosleep(20);
        s_go = s_halt ? 0 : 1;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(nct) : "memory");
    };
    publish(-1);

    double alpha = 1.0, w_prev = 0.0;  // w_{-1} = 0: Y_0 = F0, grad_Y_0 = g(F0)
    int k = 0;
    for (; k < max_iter && s_go; ++k) {
      const int cur = k & 1, prv = cur ^ 1;   // F/g parity buffers: prv = k-1, cur = k-2 -> k
      T* rk = ring + (int64_t)(k % NN_RING) * pc;
      const int evict = k - NN_RING;           // iterate leaving the ring
      const bool save_best = evict >= 0 && s_best_j == evict;
      const T w = (T)w_prev;
      apg = afg = afv = 0.0;
      for (int64_t cl = c_first; cl < ncols; cl += cstride) {
        const int64_t j = j0 + cl;
        if (save_best)
          for (int l = sub; l < p; l += TPC) Fout[(int64_t)l * c + j] = rk[(int64_t)l * c + j];
        for (int l = sub; l < p; l += TPC) {
          const T f1 = sref(prv, l, cl), f2 = sref(cur, l, cl);
          const T q1 = sref(2 + prv, l, cl), q2 = sref(2 + cur, l, cl);
          // Y = (F_{k-1} - F_{k-2}) w + F_{k-1};  grad_Y likewise (nnls.py:208-213)
          const T y = op_add(op_mul(op_sub(f1, f2), w), f1);
          const T gy = op_add(op_mul(op_sub(q1, q2), w), q1);
          const T fk = relu_nan(op_add(op_div(gy, negL), y));  // nnls.py:189-191
          sref(cur, l, cl) = fk;
          rk[(int64_t)l * c + j] = fk;
        }
        __syncwarp();
        T f[PMAX];
#pragma unroll
        for (int l = 0; l < PMAX; ++l) f[l] = l < p ? sref(cur, l, cl) : T(0);
        for (int i = sub; i < p; i += TPC) {
          T acc = T(0);
#pragma unroll
          for (int l = 0; l < PMAX; ++l)
            if (l < p) acc = fma_acc(Ws[i * p + l], f[l], acc);
          const T vv = __ldg(V + (int64_t)i * c + j);
          const T g = op_sub(acc, vv);  // g_k = W F_k - V
          sref(2 + cur, i, cl) = g;
          const T fi = sref(cur, i, cl);  // written by this thread above (i == sub mod TPC)
          const double pgv = (double)(fi > T(0) ? g : min0_nan(g));
          apg += pgv * pgv;
          afg += (double)fi * (double)g;
          afv += (double)fi * (double)vv;
        }
        __syncwarp();
      }
      publish(k);
      const double a1 = alpha_next_d(alpha);
      w_prev = __ddiv_rn(alpha - 1.0, a1);
      alpha = a1;
    }
    if (tid == 0) s_kdone = k;  // iterations computed by this CTA (uniform)
  } else {
    // ---------------------------------------------------------- resolver warp
    int resolved = -2, best_j = -1, stop_at = -1, fail_at = -1;
    double best_part = 0.0, pg_ref = 0.0;
    bool halt = false;
    while (!halt && resolved < max_iter - 1) {
      const int jb = resolved + 1;
      const int jj = jb + lane;
      bool ready = false;
      if (jj <= max_iter - 1) {
        const int slot = (jj + 1) % NN_SLOTS;
        const unsigned target = (unsigned)G * (unsigned)((jj + 1) / NN_SLOTS + 1);
        unsigned v;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counts + slot) : "memory");
        ready = v >= target;
      }
      const unsigned mask = __ballot_sync(0xffffffffu, ready);
      const int nready = (~mask == 0u) ? 32 : (__ffs(~mask) - 1);
      if (nready == 0) {
        __nanosleep(32);
        continue;
      }
      __threadfence();
      for (int t = 0; t < nready && !halt; ++t) {
        const int j = jb + t;
        const Slot* row = slots + (int64_t)((j + 1) % NN_SLOTS) * G;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
        for (int b = lane; b < G; b += 32) {
          s0 += __ldcg(&row[b].pg2);
          s1 += __ldcg(&row[b].fg);
          s2 += __ldcg(&row[b].fv);
        }
        s0 = warp_sum(s0);
        s1 = warp_sum(s1);
        s2 = warp_sum(s2);
        const double pg = sqrt(s0);
        const double partial = 0.5 * (s1 - s2);
        if (j < 0) {
          pg_ref = pg;
          best_part = partial;
          if (!(isfinite(partial) && isfinite(pg) && isfinite(L))) {
            fail_at = 0;
            halt = true;
          }
        } else if (!(isfinite(pg) && isfinite(partial))) {
          fail_at = j;
          halt = true;
        } else {
          if (partial < best_part) {
            best_part = partial;
            best_j = j;
          }
          if (pg <= grad_tol * pg_ref) {
            stop_at = j;
            halt = true;
          }
        }
        resolved = j;
      }
      if (lane == 0) {
        s_best_j = best_j;
        __threadfence_block();
        s_resolved = resolved;
        if (halt) s_halt = 1;
      }
      __syncwarp();
    }
    if (lane == 0) {
      s_best_j = best_j;
      s_stop_at = stop_at;
      s_fail_at = fail_at;
      s_best_part = best_part;
      s_pg_ref = pg_ref;
      __threadfence_block();
      s_resolved = resolved;
      s_halt = 1;
    }
  }
  __syncthreads();  // compute warps done, resolver's decisions final
  if (!resolver) {
    // the best iterate is still in the ring unless it was evicted (then F_out has it)
    const int bj = s_best_j;
    const int k_last = s_kdone - 1;
    if (bj >= 0 && bj + NN_RING > k_last) {
      const T* src = ring + (int64_t)(bj % NN_RING) * pc;
      const int sub = tid % TPC;
      for (int64_t cl = tid / TPC; cl < ncols; cl += nct / TPC)
        for (int l = sub; l < p; l += TPC) Fout[(int64_t)l * c + j0 + cl] = src[(int64_t)l * c + j0 + cl];
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    if (s_fail_at >= 0) status_fail(st, NENMF_ERR_NUMERICAL_FAILURE, s_fail_at);
    st->inner_iters = s_stop_at >= 0 ? s_stop_at + 1 : (s_fail_at >= 0 ? s_fail_at : max_iter);
    st->returned_best = s_best_j >= 0 ? 1 : 0;
    st->best_partial = s_best_part;
    st->pg_ref = s_pg_ref;
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

struct NnlsPlan {
  int grid = 1, threads = 64, tpc = 1, ldS = 0;
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
  pl.cpb = cdiv(c, pl.grid);
  int tpc = 1;
  while (tpc < 8 && tpc * 2 <= p && pl.cpb * tpc * 2 <= 512) tpc *= 2;
  pl.tpc = tpc;
  int64_t nct = imin(992, cdiv(pl.cpb * tpc, 32) * 32);
  pl.threads = (int)nct + 32;
  int pmax = p <= 8 ? 8 : p <= 16 ? 16 : p <= 32 ? 32 : 64;
  size_t base = (((size_t)pmax * pmax * sizeof(T) + 7) / 8) * 8 + 2 * 32 * 3 * sizeof(double);
  int64_t ld = cdiv(pl.cpb, 32) * 32 + (sizeof(T) == 4 ? 8 : 4);
  size_t st_bytes = (size_t)4 * p * ld * sizeof(T);
  if (base + st_bytes <= 200 * 1024) {
    pl.smem_state = true;
    pl.ldS = (int)ld;
    pl.smem = base + st_bytes;
  } else {
    pl.smem = base;
  }
  return pl;
}

template <typename T, int PMAX, int TPC, bool SM>
static int launch_nnls_t(const NnlsPlan& pl, const T* W, const T* V, const T* F0, T* Fout, T* ring, T* gstate, int p,
                         int64_t c, const double* Lptr, int max_iter, double grad_tol, Slot* slots, unsigned* counts,
                         nenmf_device_status* st, cudaStream_t s) {
  auto fn = k_nnls<T, PMAX, TPC, SM>;
  NENMF_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
  int64_t cpb = pl.cpb;
  int ldS = pl.ldS;
  void* args[] = {(void*)&W, (void*)&V, (void*)&F0, (void*)&Fout, (void*)&ring, (void*)&gstate, (void*)&p,
                  (void*)&c, (void*)&cpb, (void*)&ldS, (void*)&Lptr, (void*)&max_iter, (void*)&grad_tol,
                  (void*)&slots, (void*)&counts, (void*)&st};
  NENMF_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)fn, dim3(pl.grid), dim3(pl.threads), args, pl.smem, s));
  launch_counter_add(1);
  return NENMF_OK;
}

template <typename T, int PMAX, int TPC>
static int launch_nnls_s(const NnlsPlan& pl, const T* W, const T* V, const T* F0, T* Fout, T* ring, T* gstate, int p,
                         int64_t c, const double* Lptr, int max_iter, double grad_tol, Slot* slots, unsigned* counts,
                         nenmf_device_status* st, cudaStream_t s) {
  if (pl.smem_state)
    return launch_nnls_t<T, PMAX, TPC, true>(pl, W, V, F0, Fout, ring, gstate, p, c, Lptr, max_iter, grad_tol, slots,
                                             counts, st, s);
  return launch_nnls_t<T, PMAX, TPC, false>(pl, W, V, F0, Fout, ring, gstate, p, c, Lptr, max_iter, grad_tol, slots,
                                            counts, st, s);
}

template <typename T, int PMAX>
static int launch_nnls_p(const NnlsPlan& pl, const T* W, const T* V, const T* F0, T* Fout, T* ring, T* gstate, int p,
                         int64_t c, const double* Lptr, int max_iter, double grad_tol, Slot* slots, unsigned* counts,
                         nenmf_device_status* st, cudaStream_t s) {
  switch (pl.tpc) {
    case 1: return launch_nnls_s<T, PMAX, 1>(pl, W, V, F0, Fout, ring, gstate, p, c, Lptr, max_iter, grad_tol, slots, counts, st, s);
    case 2: return launch_nnls_s<T, PMAX, 2>(pl, W, V, F0, Fout, ring, gstate, p, c, Lptr, max_iter, grad_tol, slots, counts, st, s);
    case 4: return launch_nnls_s<T, PMAX, 4>(pl, W, V, F0, Fout, ring, gstate, p, c, Lptr, max_iter, grad_tol, slots, counts, st, s);
    default: return launch_nnls_s<T, PMAX, 8>(pl, W, V, F0, Fout, ring, gstate, p, c, Lptr, max_iter, grad_tol, slots, counts, st, s);
  }
}

template <typename T>
int solve_nnls(Arena& ws, const T* At, int64_t r, int64_t p, const T* B, int64_t c, int64_t ldb, bool trans,
               const T* F0, T* Fout, int max_iter, double grad_tol, double safety, const double* pvec,
               int pcount, int pmax, double ptol, nenmf_device_status* st, cudaStream_t s) {
  if (r < 1 || p < 1 || c < 1) return NENMF_ERR_DIM;
  if (p > 64) return NENMF_ERR_UNSUPPORTED;
  if (max_iter < 1 || pcount < 1) return NENMF_ERR_VALUE;
  const bool dry = ws.base == nullptr;
  const NnlsPlan pl = plan_nnls<T>(p, c);
  const int64_t pc = p * c;
  T* W = ws.take<T>((size_t)p * p);
  T* V = ws.take<T>((size_t)pc);
  double* Lbuf = ws.take<double>(4);
  T* ring = ws.take<T>((size_t)NN_RING * pc);
  T* gstate = pl.smem_state ? nullptr : ws.take<T>((size_t)4 * pc);
  Slot* slots = ws.take<Slot>((size_t)NN_SLOTS * pl.grid);
  unsigned* counts = ws.take<unsigned>(NN_SLOTS);
  if (!dry && !ws.ok) return NENMF_ERR_WORKSPACE;
  NENMF_TRY(abt<T>(ws, At, p, At, p, r, W, s));                       // W = A^T A   (nnls.py:157)
  NENMF_TRY(ab<T>(ws, At, p, r, B, c, ldb, trans, V, s));             // V = A^T B   (nnls.py:158)
  NENMF_TRY(lipschitz<T>(ws, At, r, p, W, pvec, pcount, pmax, ptol, safety, Lbuf, st, s));  // (nnls.py:159)
  if (!dry) {
    // slots and counters are contiguous: one memset
    size_t zbytes = (size_t)((char*)(counts + NN_SLOTS) - (char*)slots);
    NENMF_CUDA_TRY(cudaMemsetAsync(slots, 0, zbytes, s));
    if (p <= 8) NENMF_TRY((launch_nnls_p<T, 8>(pl, W, V, F0, Fout, ring, gstate, (int)p, c, Lbuf, max_iter, grad_tol, slots, counts, st, s)));
    else if (p <= 16) NENMF_TRY((launch_nnls_p<T, 16>(pl, W, V, F0, Fout, ring, gstate, (int)p, c, Lbuf, max_iter, grad_tol, slots, counts, st, s)));
    else if (p <= 32) NENMF_TRY((launch_nnls_p<T, 32>(pl, W, V, F0, Fout, ring, gstate, (int)p, c, Lbuf, max_iter, grad_tol, slots, counts, st, s)));
    else NENMF_TRY((launch_nnls_p<T, 64>(pl, W, V, F0, Fout, ring, gstate, (int)p, c, Lbuf, max_iter, grad_tol, slots, counts, st, s)));
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
