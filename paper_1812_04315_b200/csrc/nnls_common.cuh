// Shared declarations of the persistent NNLS solver (nnls.cu + nnls_k_*.cu).
#pragma once
#include "common.cuh"
#include <climits>
#include <cstdlib>

namespace nenmf {

// -------------------------------------------------------------- helpers ----
__device__ __forceinline__ double alpha_next_d(double a) {
  // (1 + sqrt(4*a*a + 1)) / 2 with NumPy's rounding sequence (nnls.py:68-69)
  return __ddiv_rn(__dadd_rn(1.0, sqrt(__dadd_rn(__dmul_rn(__dmul_rn(4.0, a), a), 1.0))), 2.0);
}

__device__ __forceinline__ bool finite_d(double x) { return isfinite(x); }

__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// a grid that stops making progress for this long aborts with
// NENMF_ERR_WATCHDOG instead of hanging the device; the host passes the limit
// (NENMF_WATCHDOG_S, default 60 s: long enough for preemption, a debugger or
// compute-sanitizer, and for the ranks of a group to reach the same solve)
constexpr unsigned long long NN_WATCHDOG_NS_DEFAULT = 60000000000ull;
unsigned long long nn_watchdog_ns();

// optional per-iteration timeline (NENMF_NNLS_TRACE=1): [0] CTA 0 compute
// warp 0 posts, [1] CTA 0 publishes, [2] CTA 0 resolves, [3] last CTA posts
constexpr int NN_TRACE_LEN = 4096;

constexpr int NW_WIN = 32;             // iterations per window
constexpr int NW_FLIGHT = 8;           // windows computed ahead of decisions
constexpr int NW_SNAP = NW_FLIGHT + 2; // rotating snapshot slots (+1 best slot)
constexpr int NW_SLOTS = NW_FLIGHT + 3;// window-record ring
constexpr int NW_MAXW = 16;            // warps per CTA incl. resolver
constexpr int NW_PPD = (NW_FLIGHT + 2) * NW_WIN;  // per-iteration warp-sum ring

struct __align__(16) WinRec {
  double v[NW_WIN][3];     // per iteration: ||PG||^2, <F,g>, <F,V>
  unsigned long long tag;  // window index + 1 once v is valid
  unsigned long long pad;
};

// ------------------------------------------------ rank groups
// A solve whose columns are split over R ranks (one process per GPU, or R
// "virtual ranks" emulated by one launch on one GPU for tests).  Every rank
// runs the same persistent solver on its own columns; the per-iteration sums
// of the decision protocol and the tie-break residuals are exchanged through
// an exchange buffer on every rank (peer-mapped over NVLink; st.sys + release
// tags), summed in rank order, so every rank takes the same decisions and the
// same result as one GPU up to the summation order.
constexpr int NG_MAXR = 8;
constexpr int NG_XSLOTS = 2 * NW_FLIGHT + 4;  // window ring: a rank can run 2 x NW_FLIGHT windows ahead of a peer's reads
struct __align__(16) XWin {
  double v[NW_WIN][3];
  unsigned long long tag[NW_WIN];  // (epoch << 20) | (window + 2) per iteration entry
};
struct __align__(16) XTie {
  double b0, b1;
  unsigned long long tag;  // epoch
  unsigned long long pad;
};
struct __align__(16) XchBuf {
  XWin win[NG_XSLOTS][NG_MAXR];  // [slot][source rank]
  XTie tie[NG_MAXR];             // [source rank]
};
struct GroupDev {
  int ranks;     // R (1: no group)
  int rank0;     // rank of this launch's first virtual rank
  int nvr;       // virtual ranks in this launch (1 per GPU; R when emulated)
  int grid_r;    // CTAs per virtual rank
  int64_t col0[NG_MAXR + 1];  // first column of each virtual rank in this launch's arrays
  XchBuf* xch[NG_MAXR];       // every rank's exchange buffer
  unsigned long long epoch;   // identical on all ranks, unique per solve
};
__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ unsigned long long xwin_tag(unsigned long long epoch, int w) {
  return (epoch << 20) | (unsigned long long)(w + 2);
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// ------------------------------------------------------------------- plan
struct NnlsPlan {
  int grid = 1, threads = 64, tpc = 1, rmax = 1, ldS = 0, ldW = 0;
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
  if (const char* e = getenv("NENMF_NNLS_GRID")) pl.grid = (int)imax(1, imin(sms, atoi(e)));
  pl.cpb = cdiv(c, pl.grid);
  // TPC: smallest power of two with ceil(p / TPC) <= 8
  int tpc = 1;
  while (cdiv(p, tpc) > 8) tpc *= 2;
  pl.tpc = tpc;
  pl.rmax = (int)cdiv(p, tpc);
  if (tpc > 1 && pl.rmax < 5) pl.rmax = 5;  // instantiated shapes: TPC=1 x 1..8, TPC>1 x 5..8
  const int vw = 16 / (int)sizeof(T);
  pl.ldW = (int)(cdiv(tpc * pl.rmax, vw) * vw);
  int64_t nct = imin(32 * (NW_MAXW - 1), cdiv(pl.cpb * tpc, 32) * 32);
  pl.threads = (int)nct + 32;
  size_t base = (((size_t)tpc * pl.rmax * pl.ldW * sizeof(T) + 15) / 16) * 16 +
                (size_t)NW_PPD * NW_MAXW * 3 * sizeof(double);
  // ldS: per-column block stride (5 buffers of PMV entries), padded so that
  // the 16-byte loads of the warp's columns fall into distinct bank groups
  const int pmv = (int)(cdiv(tpc * pl.rmax, vw) * vw);
  int64_t ld = 5 * pmv;
  if (sizeof(T) == 4) {
    while (ld % 32 != 4) ++ld;
  } else {
    while (ld % 16 != 2) ++ld;
  }
  size_t st_bytes = (size_t)pl.cpb * ld * sizeof(T);
  if (base + st_bytes <= 200 * 1024) {
    pl.smem_state = true;
    pl.ldS = (int)ld;
    pl.smem = base + st_bytes;
  } else {
    pl.smem = base;
  }
  return pl;
}



struct SolverShared {
  volatile int resolved, best_j, halt;
  volatile int prep_done;  // fused: the resolver staged the start point's tie-break inputs
  volatile int posted[NW_MAXW];
  int kdone[NW_MAXW], bsw[NW_MAXW];  // per warp: iterations done, window held in the best slot
  int stop_at, fail_at;
  double best_part, pg_ref;
};

__device__ __forceinline__ void solver_shared_init(SolverShared& sh) {
  if (threadIdx.x < NW_MAXW) {
    sh.posted[threadIdx.x] = -3;
    sh.kdone[threadIdx.x] = 0;
    sh.bsw[threadIdx.x] = -1;
  }
  if (threadIdx.x == 0) {
    sh.resolved = -2;
    sh.best_j = -1;
    sh.halt = 0;
    sh.prep_done = 0;
    sh.stop_at = -1;
    sh.fail_at = -1;
    sh.best_part = 0.0;
    sh.pg_ref = 0.0;
  }
}

// The resolver warp of a persistent solver CTA (see nnls_kernel.cuh):
// publishes this CTA's window records, summarizes the windows it owns and
// applies the reference's per-iteration decisions (nnls.py:177,196-203) in
// order.  `pp` holds the compute warps' per-iteration sums [PPD][MAXW][3].
static __device__ void resolver_warp(SolverShared& sh, const double* pp, int ncw, int max_iter, double grad_tol, double L,
                              WinRec* __restrict__ recs, WinRec* __restrict__ results,
                              unsigned long long* __restrict__ tracebuf, int ppw = NW_MAXW,
                              const GroupDev* grp = nullptr, unsigned long long watchdog_ns = NN_WATCHDOG_NS_DEFAULT) {
  const int lane = threadIdx.x & 31;
  const int G = gridDim.x;
  // group: this CTA's virtual rank and its CTA range; summarised windows go to
  // every rank's exchange buffer instead of `results`
  const bool grouped = grp != nullptr && grp->ranks > 1;
  const int Gr = grouped ? grp->grid_r : G;
  const int vr = grouped ? (int)blockIdx.x / Gr : 0;
  const int lb = grouped ? (int)blockIdx.x % Gr : (int)blockIdx.x;
  const int b_lo = vr * Gr, b_hi = b_lo + Gr;
  const int myrank = grouped ? grp->rank0 + vr : 0;
  auto xslot = [&](int w) { return (w + 1 + NG_XSLOTS) % NG_XSLOTS; };
  const bool trace = tracebuf != nullptr;
  auto g_nnls_trace = [&](int row) { return tracebuf + (size_t)row * NN_TRACE_LEN; };
    const int nwin = (max_iter + NW_WIN - 1) / NW_WIN;
    const int nq = (nwin + 1) * NW_WIN;  // pairs of windows -1 .. nwin-1
    int pubw = -1;                       // next window to publish (-1: the start point)
    int sumq = lb;                       // next owned (window, iteration) pair to summarize
    int ready_w = -2;                    // window whose records were all seen published
    int resw = -1;                       // next window to resolve
    int best_j = -1, stop_at = -1, fail_at = -1;
    double best_part = 0.0, pg_ref = 0.0;
    bool halt = false;
    unsigned long long t_prog = gtimer_ns();
    auto rec_idx = [&](int w) { return (w + 1 + NW_SLOTS) % NW_SLOTS; };
    auto win_first = [&](int w) { return w < 0 ? -1 : w * NW_WIN; };
    auto win_last = [&](int w) { return w < 0 ? -1 : min(max_iter - 1, w * NW_WIN + NW_WIN - 1); };
    while (!halt && resw < nwin) {
      bool progress = false;
      // A. publish this CTA's record of window pubw once every compute warp posted it
      if (pubw < nwin) {
        const int last = win_last(pubw);
        const int posted = lane < ncw ? sh.posted[lane] : INT_MAX;
        if (__all_sync(0xffffffffu, posted >= last)) {
          __threadfence_block();
          WinRec* rec = recs + (int64_t)rec_idx(pubw) * G + blockIdx.x;
          const int j = win_first(pubw) + lane;
          if (j <= last) {
            const double* q = pp + (size_t)((j + NW_PPD) % NW_PPD) * ppw * 3;
            double v0 = 0.0, v1 = 0.0, v2 = 0.0;
            for (int w = 0; w < ncw; ++w) {
              v0 += q[w * 3 + 0];
              v1 += q[w * 3 + 1];
              v2 += q[w * 3 + 2];
            }
            rec->v[lane][0] = v0;
            rec->v[lane][1] = v1;
            rec->v[lane][2] = v2;
          }
          __syncwarp();
          if (lane == 0) {
            fence_gpu();
            st_relaxed_u64(&rec->tag, (unsigned long long)(pubw + 2));
          }
          __syncwarp();
          if (trace && blockIdx.x == 0 && lane == 0 && pubw + 1 < NN_TRACE_LEN)
            g_nnls_trace(1)[pubw + 1] = gtimer_ns();
          if (trace && lane == 0 && pubw == nwin - 1 && blockIdx.x < 512) g_nnls_trace(0)[512 + blockIdx.x] = gtimer_ns();
          ++pubw;
          progress = true;
        }
      }
      // B. summarize the owned (window, iteration) pairs: pair q = 32 (w + 1) + j
      //    is summed over all CTAs' records by CTA q mod G (lane-strided over
      //    CTAs, fixed butterfly: deterministic) and counted into results[w].
      if (sumq < nq) {
        const int w = sumq / NW_WIN - 1, j = sumq % NW_WIN;
        const WinRec* row = recs + (int64_t)rec_idx(w) * G;
        const unsigned long long want = (unsigned long long)(w + 2);
        bool ok = w == ready_w;
        if (!ok) {
          ok = true;
          for (int b = b_lo + lane; b < b_hi; b += 32) ok &= ld_relaxed_u64(&row[b].tag) == want;
          ok = __all_sync(0xffffffffu, ok);
          if (ok) ready_w = w;
        }
        if (ok) {
          fence_gpu();
          double v0 = 0.0, v1 = 0.0, v2 = 0.0;
          const int it = w < 0 ? (j == 0 ? -1 : INT_MAX) : w * NW_WIN + j;
          if (it <= win_last(w)) {
            for (int b = b_lo + lane; b < b_hi; b += 32) {
              v0 += __ldcg(&row[b].v[j][0]);
              v1 += __ldcg(&row[b].v[j][1]);
              v2 += __ldcg(&row[b].v[j][2]);
            }
            v0 = warp_sum(v0);
            v1 = warp_sum(v1);
            v2 = warp_sum(v2);
          }
          if (!grouped) {
            if (lane == 0) {
              WinRec* res = results + rec_idx(w);
              res->v[j][0] = v0;
              res->v[j][1] = v1;
              res->v[j][2] = v2;
              __threadfence();
              atomicAdd(&res->tag, 1ull);
              if (trace && w + 1 < 1024 && j == 0) g_nnls_trace(3)[3072 + w + 1] = gtimer_ns();
            }
          } else if (lane < grp->ranks) {
            // this rank's sums of (w, j) into every rank's exchange buffer (lane d -> rank d)
            XWin* xw = &grp->xch[lane]->win[xslot(w)][myrank];
            xw->v[j][0] = v0;
            xw->v[j][1] = v1;
            xw->v[j][2] = v2;
            fence_sys();
            st_relaxed_sys_u64(&xw->tag[j], xwin_tag(grp->epoch, w));
          }
          __syncwarp();
          sumq += Gr;
          progress = true;
        }
      }
      // C. resolve window resw
      {
        const WinRec* res = results + rec_idx(resw);
        bool ready;
        if (!grouped) {
          // results of a ring slot count 32 per use: window resw is the
          // ((resw + 1) / NW_SLOTS)-th use of its slot
          const unsigned long long want = (unsigned long long)NW_WIN * ((resw + 1) / NW_SLOTS + 1);
          ready = ld_relaxed_u64(&res->tag) >= want;  // same address in all lanes
        } else {
          // every source rank's entry of this lane's iteration
          const XWin* xr = grp->xch[myrank]->win[xslot(resw)];
          const unsigned long long want = xwin_tag(grp->epoch, resw);
          bool mine = true;
          for (int src = 0; src < grp->ranks; ++src) mine &= ld_relaxed_sys_u64(&xr[src].tag[lane]) == want;
          ready = __all_sync(0xffffffffu, mine);
        }
        if (ready) {
          double r0, r1, r2;
          if (!grouped) {
            fence_gpu();
            r0 = __ldcg(&res->v[lane][0]);
            r1 = __ldcg(&res->v[lane][1]);
            r2 = __ldcg(&res->v[lane][2]);
          } else {
            fence_sys();
            // summed in rank order: the same value on every rank
            const XWin* xr = grp->xch[myrank]->win[xslot(resw)];
            r0 = __ldcv(&xr[0].v[lane][0]);
            r1 = __ldcv(&xr[0].v[lane][1]);
            r2 = __ldcv(&xr[0].v[lane][2]);
            for (int src = 1; src < grp->ranks; ++src) {
              r0 += __ldcv(&xr[src].v[lane][0]);
              r1 += __ldcv(&xr[src].v[lane][1]);
              r2 += __ldcv(&xr[src].v[lane][2]);
            }
          }
          const int first = win_first(resw), last = win_last(resw);
          if (resw < 0) {
            // the start point (nnls.py:178-181)
            pg_ref = sqrt(r0);
            best_part = 0.5 * (r1 - r2);
            pg_ref = __shfl_sync(0xffffffffu, pg_ref, 0);
            best_part = __shfl_sync(0xffffffffu, best_part, 0);
            if (!(isfinite(best_part) && isfinite(pg_ref) && isfinite(L))) {
              fail_at = 0;
              halt = true;
            }
          } else {
            // the window's iterations in parallel, one per lane; the same
            // decisions as the sequential scan of nnls.py:196-203: the first
            // non-finite iteration fails, the first with pg <= tol * pg_ref
            // stops (after the best-update of its own iteration), and best is
            // the earliest strict minimum of the partial objective before that
            const int j = first + lane;
            const bool valid = j <= last;
            const double pg = sqrt(r0), partial = 0.5 * (r1 - r2);
            const bool bad = valid && !(isfinite(pg) && isfinite(partial));
            const bool stp = valid && !bad && pg <= grad_tol * pg_ref;
            const unsigned ev = __ballot_sync(0xffffffffu, bad || stp);
            const int e = ev ? __ffs(ev) - 1 : 32;
            const bool e_bad = ev ? ((__ballot_sync(0xffffffffu, bad) >> e) & 1u) != 0 : false;
            // candidates for best: valid lanes before the event, and the event itself when it is a stop
            const bool cand = valid && !bad && (lane < e || (lane == e && !e_bad));
            double mv = cand ? partial : __longlong_as_double(0x7ff0000000000000ll);  // +inf
            int mi = cand ? lane : 32;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              const double ov = __shfl_xor_sync(0xffffffffu, mv, o);
              const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
              if (ov < mv || (ov == mv && oi < mi)) {
                mv = ov;
                mi = oi;
              }
            }
            if (mi < 32 && mv < best_part) {
              best_part = mv;
              best_j = first + mi;
            }
            if (e < 32) {
              if (e_bad) {
                fail_at = first + e;
              } else {
                stop_at = first + e;
              }
              halt = true;
            }
            if (trace && blockIdx.x == 0 && valid && j + 1 < NN_TRACE_LEN) g_nnls_trace(2)[j + 1] = gtimer_ns();
          }
          if (lane == 0) {
            sh.best_j = best_j;
            __threadfence_block();
            sh.resolved = last;
            if (halt) sh.halt = 1;
          }
          __syncwarp();
          ++resw;
          progress = true;
        }
      }
      if (progress) {
        t_prog = gtimer_ns();
      } else {
        __nanosleep(32);
        if (gtimer_ns() - t_prog > watchdog_ns) {
          fail_at = -2;
          halt = true;
        }
      }
    }
    if (trace && lane == 0 && blockIdx.x < 512) g_nnls_trace(0)[1024 + blockIdx.x] = gtimer_ns();
    if (lane == 0) {
      sh.best_j = best_j;
      sh.stop_at = stop_at;
      sh.fail_at = fail_at;
      sh.best_part = best_part;
      sh.pg_ref = pg_ref;
      __threadfence_block();
      sh.halt = 1;
    }
  }

// Arguments of the tensor-core solver.  Unfused: W = A^T A, V = A^T B and L
// are precomputed by separate kernels.  Fused (r <= NN_FUSE_RMAX): every CTA
// forms W, its own columns of V and L (the reference's power iteration) from
// At and B itself, and the explicit-residual tie-break plus the final select
// (nnls.py:219-227) run inside the same launch.
constexpr int NN_FUSE_RMAX = 64;
// extra dynamic smem of the fused mode (after the [PPD][MAXW][3] sum ring):
// At [p][r] | W [32][32] | gram [32][32] double | pv [64] double |
// ftile [ncw][2][32][cb] | Bs [r][cpb]
inline size_t fused_smem_bytes(size_t ts, int p, int64_t r, int ncw, int cb, int64_t cpb) {
  return ((size_t)p * r + 3) / 4 * 4 * ts + 32 * 32 * ts + 32 * 32 * sizeof(double) + 64 * sizeof(double) +
         (size_t)ncw * 2 * 32 * cb * ts + (size_t)r * cpb * ts + 64;
}
template <typename T>
struct MmaArgs {
  const T* W;
  const T* V;
  double* L;  // unfused: input L; fused: output [L, r_best, r_start]
  const T* At;
  const T* B;
  int64_t r, ldb;
  int trans, fused;
  const double* pvec;
  int pcount, pmax;
  double ptol, safety;
  const T* F0;
  T* Fout;
  T* snaps;
  int p;
  int64_t c, cpb;
  int max_iter;
  double grad_tol;
  WinRec* recs;
  WinRec* results;
  nenmf_device_status* st;
  unsigned long long* tracebuf;
  const double* wtab;
  int dbg;
  double* rpart;      // fused: [grid][2] per-CTA residual partials
  unsigned int* bar;  // fused: grid barrier counters [2] (zeroed with recs)
  const T* Pt;        // fused next product Pout (p x nup) = F_out Pt^T, Pt (nup x c)
  int64_t nup;
  T* Pout;
  double* npart;      // [grid][p][nup] per-CTA partials
  GroupDev grp;       // rank group (grp.ranks == 1: a single-GPU solve)
  unsigned long long watchdog_ns;
};
template <typename T>
int launch_nnls_mma(const MmaArgs<T>& a, int grid, cudaStream_t s);

// Arguments of the streamed tensor-core solver (nnls_stream.cuh, FP32).
struct StreamArgs {
  const float* W;   // p x p
  const float* V;   // p x c
  const double* L;  // [0] = Lipschitz constant
  const float* F0;  // p x c
  float* Fout;      // p x c
  float* U;         // 2 x p x c: u_k lives in slot k & 1 (u_{-1}: slot 1)
  float* snaps;     // (NW_SNAP + 1) x 2 x p x c
  int p;
  int64_t c, cpb;
  int max_iter;
  double grad_tol;
  const double* wtab;
  WinRec* recs;
  WinRec* results;
  nenmf_device_status* st;
  int resident;     // 1: u_k and V of the CTA's columns stay in shared memory (set by the launcher)
  unsigned long long watchdog_ns;
};

// 1 when the launch keeps its state in shared memory (the CTA's columns fit)
int launch_nnls_stream(StreamArgs& a, int grid, cudaStream_t s);

template <typename T>
int nnls_mma_max_cols(int p);  // columns one CTA of the tensor-core solver can hold
template <typename T>
int nnls_mma_col_block();      // columns per compute warp of the tensor-core solver

template <typename T, int TPC>
int launch_nnls_tpc(const NnlsPlan& pl, const T* W, const T* V, const T* F0, T* Fout, T* snaps, double* salpha,
                    T* gstate, int p, int64_t c, const double* Lptr, int max_iter, double grad_tol, WinRec* recs,
                    WinRec* results, nenmf_device_status* st, unsigned long long* tracebuf, cudaStream_t s);

}  // namespace nenmf
