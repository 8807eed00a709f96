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
//                                (nnls_kernel.cuh, instantiated by nnls_k_*.cu)
//   resid + k_decide + k_select  _true_objective tie-break (nnls.py:219-227)
//
// k_nnls: every CTA owns a slab of columns of F (columns are independent
// except for the two global sums per iteration that drive the stop/best
// decisions, nnls.py:194-203).  Iterations run in windows of 32 with no
// cross-CTA synchronisation inside a window; per-window sums are exchanged
// through tagged records and added in fixed CTA order, so every CTA takes the
// same decisions; the best iterate is recomputed from a window snapshot when
// it is no longer live.  See nnls_kernel.cuh.
#include "nnls.cuh"
#include "rsi.cuh"
#include "nnls_common.cuh"
#include "skinny.cuh"

#include <cooperative_groups.h>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <mutex>

namespace nenmf {

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
  if (k > 160) return NENMF_ERR_UNSUPPORTED;  // the Gram and two vectors in shared memory
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
  NENMF_CUDA_TRY(set_smem(k_power<T>, smem));
  k_power<T><<<1, 128, smem, s>>>(gram, (int)k, pvec, pcount, ptol, pmax, safety, Lout, st);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

__device__ unsigned long long g_nnls_trace[4][NN_TRACE_LEN];

// Momentum weights w_k = (alpha_k - 1) / alpha_{k+1} depend only on k
// (nnls.py:68-69, 213): computed once per device on the host with the same
// IEEE rounding sequence as alpha_next_d and kept in device memory, so the
// solver loop carries no sqrt/div on its critical path.
constexpr int NN_WTAB_LEN = 1 << 16;
__device__ double g_wtab[NN_WTAB_LEN];

static const double* momentum_table(int max_iter) {
  if (max_iter > NN_WTAB_LEN) return nullptr;
  static std::mutex mu;
  static bool ready[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!ready[dev]) {
    static double host[NN_WTAB_LEN];
    volatile double alpha = 1.0;
    for (int k = 0; k < NN_WTAB_LEN; ++k) {
      volatile double t = 4.0 * alpha;
      t = t * alpha;
      t = t + 1.0;
      volatile double sq = std::sqrt((double)t);
      volatile double a1 = (1.0 + sq) / 2.0;
      host[k] = (alpha - 1.0) / a1;
      alpha = a1;
    }
    if (cudaMemcpyToSymbol(g_wtab, host, sizeof(host)) != cudaSuccess) return nullptr;
    ready[dev] = true;
  }
  void* ptr = nullptr;
  if (cudaGetSymbolAddress(&ptr, g_wtab) != cudaSuccess) return nullptr;
  return static_cast<const double*>(ptr);
}

template <typename T>
static int launch_nnls(const NnlsPlan& pl, const T* W, const T* V, const T* F0, T* Fout, T* snaps, double* salpha,
                       T* gstate, int p, int64_t c, const double* Lptr, int max_iter, double grad_tol, WinRec* recs,
                       WinRec* results, nenmf_device_status* st, cudaStream_t s) {
  unsigned long long* tracebuf = nullptr;
  if (getenv("NENMF_NNLS_TRACE") != nullptr) NENMF_CUDA_TRY(cudaGetSymbolAddress((void**)&tracebuf, g_nnls_trace));
#define NN_DARGS pl, W, V, F0, Fout, snaps, salpha, gstate, p, c, Lptr, max_iter, grad_tol, recs, results, st, tracebuf, s
  switch (pl.tpc) {
    case 1: return launch_nnls_tpc<T, 1>(NN_DARGS);
    case 2: return launch_nnls_tpc<T, 2>(NN_DARGS);
    case 4: return launch_nnls_tpc<T, 4>(NN_DARGS);
    case 8: return launch_nnls_tpc<T, 8>(NN_DARGS);
    case 16: return launch_nnls_tpc<T, 16>(NN_DARGS);
  }
#undef NN_DARGS
  return NENMF_ERR_UNSUPPORTED;
}

unsigned long long nn_watchdog_ns() {
  static const unsigned long long ns = [] {
    const char* e = getenv("NENMF_WATCHDOG_S");
    const double sec = e != nullptr ? atof(e) : 0.0;
    return sec > 0.0 ? (unsigned long long)(sec * 1e9) : NN_WATCHDOG_NS_DEFAULT;
  }();
  return ns;
}

template <typename T>
int solve_nnls(Arena& ws, const T* At, int64_t r, int64_t p, const T* B, int64_t c, int64_t ldb, bool trans,
               const T* F0, T* Fout, int max_iter, double grad_tol, double safety, const double* pvec,
               int pcount, int pmax, double ptol, nenmf_device_status* st, cudaStream_t s, const T* Pt,
               int64_t nup, T* Pout, const uint8_t* Xpre, const GroupHost* grp) {
  if (r < 1 || p < 1 || c < 1) return NENMF_ERR_DIM;
  if (Pt != nullptr && (nup < 1 || Pout == nullptr)) return NENMF_ERR_VALUE;
  if (p > 128) return NENMF_ERR_UNSUPPORTED;  // the CUDA-core solver holds 16 threads x 8 entries per column
  if (max_iter < 1 || pcount < 1) return NENMF_ERR_VALUE;
  const bool dry = ws.base == nullptr;
  const NnlsPlan pl = plan_nnls<T>(p, c);
  const int64_t pc = p * c;
  // tensor-core solver: p <= 32 and at most 15 blocks of 8 columns per CTA
  int sms = sm_count();
  if (sms <= 0) sms = 148;
  const bool grouped = grp != nullptr && grp->ranks > 1;
  int mgrid = (int)imax(1, imin(sms, cdiv(c, nnls_mma_col_block<T>())));
  int64_t mcpb = cdiv(c, mgrid);
  int grid_r = mgrid;
  if (grouped) {
    // a rank group: nvr virtual ranks of grid_r CTAs each in this
    // launch (nvr = 1 on a real multi-GPU run); columns per CTA = the largest
    // rank's share
    if (grp->ranks > NG_MAXR || grp->nvr < 1 || grp->nvr > grp->ranks || grp->rank0 < 0 ||
        grp->rank0 + grp->nvr > grp->ranks || grp->col0[0] != 0 || grp->col0[grp->nvr] != c || grp->epoch == 0 ||
        grp->epoch >= (1ull << 40))
      return NENMF_ERR_VALUE;
    int64_t cmax = 1;
    for (int v = 0; v < grp->nvr; ++v) {
      if (grp->col0[v + 1] < grp->col0[v]) return NENMF_ERR_VALUE;
      cmax = imax(cmax, grp->col0[v + 1] - grp->col0[v]);
    }
    grid_r = (int)imax(1, imin(sms / grp->nvr, cdiv(cmax, nnls_mma_col_block<T>())));
    mgrid = grid_r * grp->nvr;
    mcpb = cdiv(cmax, grid_r);
  }
  const bool use_mma = p <= 32 && mcpb <= nnls_mma_max_cols<T>((int)p) && max_iter <= NN_WTAB_LEN &&
                       getenv("NENMF_NNLS_SIMT") == nullptr;
  // FP32, p <= 32, too many columns for the register-resident solver: the
  // streamed tensor-core solver (nnls_stream.cuh) keeps u_k in HBM
  const bool use_stream = !use_mma && sizeof(T) == 4 && p <= 64 && max_iter <= NN_WTAB_LEN &&
                          getenv("NENMF_NNLS_SIMT") == nullptr;
  // streamed solver: column blocks of whole 16-column tiles (16-byte aligned rows for cp.async)
  const int64_t scpb = cdiv(cdiv(c, imax(1, imin(sms, cdiv(c, 16)))), 16) * 16;
  const int sgrid = (int)imax(1, cdiv(c, scpb));
  const int grid_used = use_mma ? mgrid : (use_stream ? sgrid : pl.grid);
  // fused prologue/epilogue (W, V, L and the tie-break inside the solver
  // launch) for the compressed problems' short operands
  const int cbm = nnls_mma_col_block<T>();
  const bool fused = use_mma && r <= NN_FUSE_RMAX && getenv("NENMF_NNLS_UNFUSED") == nullptr &&
                     (size_t)NW_PPD * NW_MAXW * 3 * sizeof(double) +
                             fused_smem_bytes(sizeof(T), (int)p, r, (int)cdiv(mcpb, cbm), cbm, mcpb) <=
                         227 * 1024;
  // the next product inside the launch when its tiles fit too
  const bool fused_next = fused && Pt != nullptr &&
                          (size_t)NW_PPD * NW_MAXW * 3 * sizeof(double) +
                                  fused_smem_bytes(sizeof(T), (int)p, r, (int)cdiv(mcpb, cbm), cbm, mcpb) +
                                  (size_t)(p + nup) * mcpb * sizeof(T) <=
                              227 * 1024;
  // a group solve runs only on the fused tensor-core path (its exchange lives
  // in that kernel): other shapes are the caller's to replicate
  if (grouped && !(fused && (Pt == nullptr || fused_next))) return NENMF_ERR_UNSUPPORTED;
  T* W = fused ? nullptr : ws.take<T>((size_t)p * p);
  T* V = fused ? nullptr : ws.take<T>((size_t)pc);
  double* Lbuf = ws.take<double>(4);
  T* snaps = ws.take<T>((size_t)(NW_SNAP + 1) * 4 * pc);
  T* ustate = use_stream ? ws.take<T>((size_t)2 * pc) : nullptr;
  double* salpha = use_mma ? nullptr : ws.take<double>((size_t)pl.grid * NW_MAXW * (NW_SNAP + 1) * 2);
  T* gstate = (use_mma || use_stream || pl.smem_state) ? nullptr : ws.take<T>((size_t)4 * pc);
  double* rpart = fused ? ws.take<double>((size_t)2 * grid_used) : nullptr;
  double* npart = fused_next ? ws.take<double>((size_t)grid_used * 2 * p * nup) : nullptr;  // [grid][best, start]
  // window records + (fused) the grid-barrier counter, zeroed together
  const size_t rec_bytes = sizeof(WinRec) * ((size_t)NW_SLOTS * grid_used + NW_SLOTS) + 64;
  unsigned char* recmem = ws.take<unsigned char>(rec_bytes);
  WinRec* recs = reinterpret_cast<WinRec*>(recmem);
  WinRec* results = recs + (size_t)NW_SLOTS * grid_used;
  unsigned int* bar = reinterpret_cast<unsigned int*>(results + NW_SLOTS);
  if (!dry && !ws.ok) return NENMF_ERR_WORKSPACE;
  if (!fused) {
    NENMF_TRY(abt<T>(ws, At, p, At, p, r, W, s));                       // W = A^T A   (nnls.py:157)
    bool vdone = false;
    if constexpr (sizeof(T) == 4) {
      // V = A^T B from one tensor-core pass over the prepared X: the Y side when
      // B = X^T (X is c x r), the Z side when B = X (r x c); the other side of
      // the pass is discarded
      const int64_t nx = trans ? c : r, mx = trans ? r : c;
      if (Xpre != nullptr && tc_pass_eligible(nx, mx, p)) {
        float* junk = ws.take<float>((size_t)p * (trans ? r : r));
        const float* A_f = reinterpret_cast<const float*>(At);
        const float* F0_f = reinterpret_cast<const float*>(F0);
        float* V_f = reinterpret_cast<float*>(V);
        if (trans)  // Y (p x nx = c) = At X^T with At (p x mx = r); Z side fed F0 (p x c)
          NENMF_TRY(dual_pass_tc_pre(ws, Xpre, nx, mx, A_f, dry ? A_f : F0_f, p, V_f, junk, s));
        else        // Z (p x mx = c) = At X with At (p x nx = r); Y side fed F0 (p x c)
          NENMF_TRY(dual_pass_tc_pre(ws, Xpre, nx, mx, dry ? A_f : F0_f, A_f, p, junk, V_f, s));
        vdone = true;
      }
    }
    if (!vdone) NENMF_TRY(ab<T>(ws, At, p, r, B, c, ldb, trans, V, s));  // V = A^T B   (nnls.py:158)
    NENMF_TRY(lipschitz<T>(ws, At, r, p, W, pvec, pcount, pmax, ptol, safety, Lbuf, st, s));  // (nnls.py:159)
  }
  if (!dry) {
    NENMF_CUDA_TRY(cudaMemsetAsync(recmem, 0, rec_bytes, s));
    if (use_mma) {
      const double* wtab = momentum_table(max_iter);
      if (wtab == nullptr) return NENMF_ERR_CUDA;
      MmaArgs<T> a{};
      a.W = W;
      a.V = V;
      a.L = Lbuf;
      a.At = At;
      a.B = B;
      a.r = r;
      a.ldb = ldb;
      a.trans = trans ? 1 : 0;
      a.fused = fused ? 1 : 0;
      a.pvec = pvec;
      a.pcount = pcount;
      a.pmax = pmax;
      a.ptol = ptol;
      a.safety = safety;
      a.F0 = F0;
      a.Fout = Fout;
      a.snaps = snaps;
      a.p = (int)p;
      a.c = c;
      a.cpb = mcpb;
      a.max_iter = max_iter;
      a.grad_tol = grad_tol;
      a.recs = recs;
      a.results = results;
      a.st = st;
      a.tracebuf = nullptr;
      if (getenv("NENMF_NNLS_TRACE") != nullptr) NENMF_CUDA_TRY(cudaGetSymbolAddress((void**)&a.tracebuf, g_nnls_trace));
      a.wtab = wtab;
      // NENMF_NNLS_DBG (timing experiments only; results are not valid):
      // 1 = no resolver, 2 = no snapshots, 4 = no per-iteration sums
      const char* dbg_env = getenv("NENMF_NNLS_DBG");
      a.dbg = dbg_env != nullptr ? atoi(dbg_env) : 0;
      a.rpart = rpart;
      a.bar = bar;
      a.Pt = fused_next ? Pt : nullptr;
      a.nup = fused_next ? nup : 0;
      a.Pout = fused_next ? Pout : nullptr;
      a.npart = npart;
      a.watchdog_ns = nn_watchdog_ns();
      a.grp.ranks = 1;
      if (grouped) {
        if (grp->watchdog_s > 0) a.watchdog_ns = (unsigned long long)grp->watchdog_s * 1000000000ull;
        a.grp.ranks = grp->ranks;
        a.grp.rank0 = grp->rank0;
        a.grp.nvr = grp->nvr;
        a.grp.grid_r = grid_r;
        for (int v = 0; v <= grp->nvr; ++v) a.grp.col0[v] = grp->col0[v];
        for (int d = 0; d < grp->ranks; ++d) a.grp.xch[d] = static_cast<XchBuf*>(grp->xch[d]);
        a.grp.epoch = grp->epoch;
      }
      NENMF_TRY(launch_nnls_mma<T>(a, mgrid, s));
      if (fused) {
        if (Pt != nullptr && !fused_next) NENMF_TRY(abt<T>(ws, Fout, p, Pt, nup, c, Pout, s));
        return NENMF_OK;
      }
    } else if (use_stream) {
      if constexpr (sizeof(T) == 4) {
        const double* wtab = momentum_table(max_iter);
        if (wtab == nullptr) return NENMF_ERR_CUDA;
        StreamArgs a{};
        a.W = W;
        a.V = V;
        a.L = Lbuf;
        a.F0 = F0;
        a.Fout = Fout;
        a.U = ustate;
        a.snaps = snaps;
        a.p = (int)p;
        a.c = c;
        a.cpb = scpb;
        a.max_iter = max_iter;
        a.grad_tol = grad_tol;
        a.wtab = wtab;
        a.recs = recs;
        a.results = results;
        a.st = st;
        a.watchdog_ns = nn_watchdog_ns();
        NENMF_TRY(launch_nnls_stream(a, sgrid, s));
      }
    } else {
      NENMF_TRY(launch_nnls<T>(pl, W, V, F0, Fout, snaps, salpha, gstate, (int)p, c, Lbuf, max_iter, grad_tol, recs,
                               results, st, s));
    }
  }
  if (fused) return (Pt != nullptr && !fused_next) ? abt<T>(ws, Fout, p, Pt, nup, c, Pout, s) : NENMF_OK;
  // explicit residuals of best and start, only when an iterate improved (nnls.py:219-227);
  // FP32 with a prepared X: both in one tensor-core pass (k_resid_bulk)
  bool rdone = false;
  if constexpr (sizeof(T) == 4) {
    const int64_t nx = trans ? c : r, mx = trans ? r : c;
    if (Xpre != nullptr && p <= 32 && tc_pass_eligible(nx, mx, p)) {
      const float* A_f = reinterpret_cast<const float*>(At);
      const float* F1 = reinterpret_cast<const float*>(Fout);
      const float* F2 = reinterpret_cast<const float*>(F0);
      const int rc = trans ? resid_tc_pre(ws, Xpre, nx, mx, F1, A_f, p, Lbuf + 2, s, F2, 1, &st->returned_best)
                           : resid_tc_pre(ws, Xpre, nx, mx, A_f, F1, p, Lbuf + 2, s, F2, 2, &st->returned_best);
      if (rc != NENMF_ERR_UNSUPPORTED) {
        NENMF_TRY(rc);
        rdone = true;
      }
    }
  }
  if (!rdone) NENMF_TRY(resid<T>(ws, At, p, r, B, c, ldb, trans, Fout, F0, Lbuf + 2, &st->returned_best, s));
  if (!dry) {
    k_decide<<<1, 1, 0, s>>>(Lbuf + 2, st);
    NENMF_LAUNCH_CHECK();
    k_select<T><<<(unsigned)imin(cdiv(pc, 256), 1184), 256, 0, s>>>(F0, Fout, pc, st);
    NENMF_LAUNCH_CHECK();
  }
  if (Pt != nullptr) NENMF_TRY(abt<T>(ws, Fout, p, Pt, nup, c, Pout, s));
  return NENMF_OK;
}

template <typename T>
int spectral_norm_sq(Arena& ws, const T* At, int64_t r, int64_t p, const double* pvec, int pcount, int pmax,
                     double tol, double* out, nenmf_device_status* st, cudaStream_t s) {
  if (r < 1 || p < 1) return NENMF_ERR_DIM;
  if (min(r, p) > 160) return NENMF_ERR_UNSUPPORTED;
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

}  // namespace nenmf

extern "C" int nenmf_debug_nnls_trace(unsigned long long* host_out, int count) {
  if (count > 4 * nenmf::NN_TRACE_LEN) count = 4 * nenmf::NN_TRACE_LEN;
  return cudaMemcpyFromSymbol(host_out, nenmf::g_nnls_trace, sizeof(unsigned long long) * count) == cudaSuccess ? 0 : 6;
}

namespace nenmf {
#define NENMF_INST_NNLS(T)                                                                                    \
  template int solve_nnls<T>(Arena&, const T*, int64_t, int64_t, const T*, int64_t, int64_t, bool, const T*,  \
                             T*, int, double, double, const double*, int, int, double, nenmf_device_status*,   \
                             cudaStream_t, const T*, int64_t, T*, const uint8_t*, const GroupHost*);         \
  template int spectral_norm_sq<T>(Arena&, const T*, int64_t, int64_t, const double*, int, int, double, double*, \
                                   nenmf_device_status*, cudaStream_t);                                      \
  template int gradient<T>(Arena&, const T*, int64_t, int64_t, const T*, int64_t, int64_t, bool, const T*,    \
                           T*, cudaStream_t);
NENMF_INST_NNLS(double)
NENMF_INST_NNLS(float)

}  // namespace nenmf
