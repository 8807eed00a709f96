// The persistent inner-solver kernel (included by nnls.cu).
//
// Restates the inner loop of nnls.py:161-227 as ONE cooperative launch.
//
// Work split.  Columns of F are independent except for the two global sums per
// iteration (||PG||_F and the Gram-form objective, nnls.py:194-195) that drive
// the stop rule, the best-iterate rule and the non-finite check
// (nnls.py:196-203).  Every CTA owns a slab of columns; TPC threads of one
// warp own a column, each holding RMAX consecutive entries of the column
// (elementwise update) and the same RMAX rows of g = W F - V (matvec).
//
// Windows.  Iterations run in windows of WIN = 32 without any cross-CTA
// synchronisation.  At each window start a CTA snapshots its columns' state
// (F_{k-1}, F_{k-2}, g_{k-1}, g_{k-2}).  Per-iteration, per-warp sums go to
// shared memory; at the end of a window the CTA's resolver warp adds them in
// warp order and publishes one 32-iteration record.  The CTA that owns the
// window (w mod G) adds all CTAs' records in CTA order and publishes the
// window result; every resolver reads it and applies the reference's
// decisions iteration by iteration, in order, so all CTAs agree bit for bit.
// Compute warps may run NWIN windows ahead of the decisions.  After a stop at
// j the speculative iterations past j are discarded; the returned best
// iterate is recomputed from the snapshot of its window (deterministic, the
// same arithmetic), unless it is still in the live state buffers.
#pragma once
#include "nnls_common.cuh"

namespace nenmf {

template <typename T, int TPC, int RMAX, bool SMEM>
__global__ void __launch_bounds__(512, 1)
k_nnls(const T* __restrict__ W, const T* __restrict__ V, const T* __restrict__ F0, T* __restrict__ Fout,
       T* __restrict__ snaps, double* __restrict__ snap_alpha, T* __restrict__ gstate, int p, int64_t c,
       int64_t cpb, int ldS, int ldW, const double* __restrict__ Lptr, int max_iter, double grad_tol,
       WinRec* __restrict__ recs, WinRec* __restrict__ results, nenmf_device_status* st,
       unsigned long long* __restrict__ tracebuf) {
  const bool trace = tracebuf != nullptr;
  auto g_nnls_trace = [&](int row) { return tracebuf + (size_t)row * NN_TRACE_LEN; };
  constexpr int PM = TPC * RMAX;               // padded column length handled by a column group
  constexpr int VW = 16 / sizeof(T);           // elements per 16-byte shared load
  constexpr int PMV = (PM + VW - 1) / VW * VW;  // f register length (vector-padded)
  extern __shared__ __align__(16) double smem_d[];
  T* Ws = reinterpret_cast<T*>(smem_d);                                       // [PM][ldW], zero padded
  double* pp = smem_d + (((size_t)PM * ldW * sizeof(T) + 15) / 16) * 2;        // [PPD][MAXW][3]
  T* Sb = reinterpret_cast<T*>(pp + (size_t)NW_PPD * NW_MAXW * 3);            // [5][p][ldS]
  __shared__ SolverShared sh;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ncw = (blockDim.x >> 5) - 1;
  const int nct = ncw * 32;
  const bool resolver = wid == ncw;
  const int G = gridDim.x;
  const int64_t j0 = (int64_t)blockIdx.x * cpb;
  const int ncols = (int)(imin(c, j0 + cpb) - j0);
  const int64_t pc = (int64_t)p * c;

  for (int i = tid; i < PM * ldW; i += blockDim.x) {
    const int r = i / ldW, l = i % ldW;
    Ws[i] = (r < p && l < p) ? W[r * p + l] : T(0);
  }
  solver_shared_init(sh);
  __syncthreads();
  if (st->code != 0) return;  // an earlier stage failed (uniform)
  const double L = *Lptr;
  const T rnegL = (T)(-1.0 / L);

  // state: b = 0,1 F parity buffers, 2,3 g parity buffers, 4 V (SMEM only).
  // SMEM: column-major blocks of ldS elements per column ([b][PMV] inside),
  // so a column's entries are contiguous (16-byte loads, compile-time offsets)
  // and ldS is chosen so the warp's lanes hit distinct banks.
  // GLOBAL: [b][p][c] (coalesced across the warp's columns).
  auto sref = [&](int b, int i, int cl) -> T& {
    if (SMEM) return Sb[(size_t)cl * ldS + b * PMV + i];
    return gstate[(int64_t)b * pc + (int64_t)i * c + j0 + cl];
  };
  auto vref = [&](int i, int cl) -> T {
    if (SMEM) return Sb[(size_t)cl * ldS + 4 * PMV + i];
    return __ldg(V + (int64_t)i * c + j0 + cl);
  };
  // snapshot slot s (NW_SNAP = best slot): [4][p][c]
  auto snref = [&](int s, int b, int i, int cl) -> T& {
    return snaps[(((int64_t)s * 4 + b) * p + i) * c + j0 + cl];
  };

  const int sub = tid % TPC;
  const int ibase = sub * RMAX;                 // first entry/row owned by this thread
  const int cstride = nct / TPC;
  const int cfirst = tid / TPC;
  const int wfirst = (wid * 32) / TPC;          // column loops are warp-uniform

  // one iteration k for column cl: F_k into buffer cur, g_k into 2+cur.
  // Returns the thread's share of the three sums in (a0, a1, a2) when STATS.
  auto step = [&](int cl, int cur, int prv, T w, double& a0, double& a1, double& a2, bool stats) {
    // SMEM mode runs every PM entry: rows/entries >= p are zero-padded in W,
    // V and the state, stay exactly zero and add nothing to the sums.
    T fmine[RMAX];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      const int i = ibase + r;
      fmine[r] = T(0);
      if (SMEM || i < p) {
        const T f1 = sref(prv, i, cl), f2 = sref(cur, i, cl);
        const T q1 = sref(2 + prv, i, cl), q2 = sref(2 + cur, i, cl);
        // Y = (F_{k-1} - F_{k-2}) w + F_{k-1};  grad_Y likewise (nnls.py:208-213)
        const T y = op_add(op_mul(op_sub(f1, f2), w), f1);
        const T gy = op_add(op_mul(op_sub(q1, q2), w), q1);
        // F_k = max(0, Y + grad_Y / (-L)) (nnls.py:189-191); the division is a
        // multiplication by the rounded reciprocal (<= 1 ulp from the reference)
        const T fk = relu_nan(op_add(op_mul(gy, rnegL), y));
        sref(cur, i, cl) = fk;
        fmine[r] = fk;
      }
    }
    __syncwarp();
    T f[PMV];
    if constexpr (SMEM) {
      const T* cp = Sb + (size_t)cl * ldS + cur * PMV;
#pragma unroll
      for (int l0 = 0; l0 < PMV; l0 += VW) {
        if constexpr (VW == 4) {
          const float4 v = *reinterpret_cast<const float4*>(cp + l0);
          f[l0] = (T)v.x;
          f[l0 + 1] = (T)v.y;
          f[l0 + 2] = (T)v.z;
          f[l0 + 3] = (T)v.w;
        } else {
          const double2 v = *reinterpret_cast<const double2*>(cp + l0);
          f[l0] = (T)v.x;
          f[l0 + 1] = (T)v.y;
        }
      }
    } else {
#pragma unroll
      for (int l = 0; l < PMV; ++l) f[l] = l < p ? sref(cur, l, cl) : T(0);
    }
    T acc[RMAX];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) acc[r] = T(0);
#pragma unroll
    for (int l0 = 0; l0 < PMV; l0 += VW) {
      if (SMEM || l0 < p) {
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
          const int i = ibase + r;
          if (SMEM || i < p) {
            if constexpr (VW == 4) {
              const float4 wv = *reinterpret_cast<const float4*>(Ws + i * ldW + l0);
              acc[r] = fma_acc((T)wv.x, f[l0 + 0], acc[r]);
              acc[r] = fma_acc((T)wv.y, f[l0 + 1], acc[r]);
              acc[r] = fma_acc((T)wv.z, f[l0 + 2], acc[r]);
              acc[r] = fma_acc((T)wv.w, f[l0 + 3], acc[r]);
            } else {
              const double2 wv = *reinterpret_cast<const double2*>(Ws + i * ldW + l0);
              acc[r] = fma_acc((T)wv.x, f[l0 + 0], acc[r]);
              acc[r] = fma_acc((T)wv.y, f[l0 + 1], acc[r]);
            }
          }
        }
      }
    }
    // per-thread partial sums in T (the thread's RMAX entries), then double
    T s0 = T(0), s1 = T(0), s2 = T(0);
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      const int i = ibase + r;
      if (SMEM || i < p) {
        const T vv = vref(i, cl);
        const T g = op_sub(acc[r], vv);  // g_k = W F_k - V (nnls.py:192-193)
        sref(2 + cur, i, cl) = g;
        const T fi = fmine[r];
        const T pgv = fi > T(0) ? g : min0_nan(g);
        s0 = fma_acc(pgv, pgv, s0);
        s1 = fma_acc(fi, g, s1);
        s2 = fma_acc(fi, vv, s2);
      }
    }
    if (stats) {
      a0 += (double)s0;
      a1 += (double)s1;
      a2 += (double)s2;
    }
    __syncwarp();
  };

  if (!resolver) {
    // ------------------------------------------------------------ compute
    auto post = [&](int j, double a0, double a1, double a2) {
      a0 = warp_sum(a0);
      a1 = warp_sum(a1);
      a2 = warp_sum(a2);
      if (lane == 0) {
        double* q = pp + ((size_t)((j + NW_PPD) % NW_PPD) * NW_MAXW + wid) * 3;
        q[0] = a0;
        q[1] = a1;
        q[2] = a2;
      }
    };
    auto post_flag = [&](int j) {
      if (lane == 0) {
        __threadfence_block();
        sh.posted[wid] = j;
      }
    };

    // start point: g(F0) = W F0 - V; pg_ref, partial_start (nnls.py:163-178)
    {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      for (int base = 0; wfirst + base < ncols; base += cstride) {
        const int cl = cfirst + base;
        const bool act = cl < ncols;
        const int64_t j = j0 + cl;
        if (act) {
          if (SMEM)
            for (int e = sub; e < ldS; e += TPC) Sb[(size_t)cl * ldS + e] = T(0);
          __syncwarp();
#pragma unroll
          for (int r = 0; r < RMAX; ++r) {
            const int i = ibase + r;
            if (i < p) {
              const T f = F0[(int64_t)i * c + j];
              sref(0, i, cl) = f;
              sref(1, i, cl) = f;
              if (SMEM) Sb[(size_t)cl * ldS + 4 * PMV + i] = V[(int64_t)i * c + j];
            }
          }
        } else {
          __syncwarp();
        }
        __syncwarp();
        if (act) {
          T f[PM];
#pragma unroll
          for (int l = 0; l < PM; ++l) f[l] = l < p ? sref(1, l, cl) : T(0);
#pragma unroll
          for (int r = 0; r < RMAX; ++r) {
            const int i = ibase + r;
            if (i < p) {
              T acc = T(0);
#pragma unroll
              for (int l = 0; l < PM; ++l)
                if (l < p) acc = fma_acc(Ws[i * ldW + l], f[l], acc);
              const T vv = vref(i, cl);
              const T g = op_sub(acc, vv);
              sref(2, i, cl) = g;
              sref(3, i, cl) = g;
              const T fi = f[i];
              const double pgv = (double)(fi > T(0) ? g : min0_nan(g));
              a0 += pgv * pgv;
              a1 += (double)fi * (double)g;
              a2 += (double)fi * (double)vv;
            }
          }
        }
        __syncwarp();
      }
      post(-1, a0, a1, a2);
      post_flag(-1);
    }

    double alpha = 1.0, w_prev = 0.0;  // w_{-1} = 0: Y_0 = F0, grad_Y_0 = g(F0)
    int k = 0;
    bool go = true;
    for (; k < max_iter && go; ++k) {
      if (k % NW_WIN == 0) {
        const int w = k / NW_WIN;
        // throttle: windows <= w - NW_FLIGHT - 1 must be resolved
        int ok = 1;
        if (lane == 0) {
          const int need = (w - NW_FLIGHT) * NW_WIN - 1;
          while (sh.resolved < need && !sh.halt) __nanosleep(64);
          ok = sh.halt ? 0 : 1;
        }
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (!ok) break;
        // snapshot slot w % NW_SNAP; if it still holds the best window, save it first
        const int slot = w % NW_SNAP;
        const int evicted = w - NW_SNAP;
        const int bj = sh.best_j;
        const bool save = evicted >= 0 && bj >= 0 && bj / NW_WIN == evicted;
        for (int base = 0; wfirst + base < ncols; base += cstride) {
          const int cl = cfirst + base;
          if (cl >= ncols) continue;
#pragma unroll
          for (int r = 0; r < RMAX; ++r) {
            const int i = ibase + r;
            if (i < p) {
              if (save)
                for (int b = 0; b < 4; ++b) snref(NW_SNAP, b, i, cl) = snref(slot, b, i, cl);
              // buffer roles at iteration k: prv = (k-1)&1 holds F_{k-1}, cur = k&1 holds F_{k-2}
              const int cur = k & 1, prv = cur ^ 1;
              snref(slot, 0, i, cl) = sref(prv, i, cl);
              snref(slot, 1, i, cl) = sref(cur, i, cl);
              snref(slot, 2, i, cl) = sref(2 + prv, i, cl);
              snref(slot, 3, i, cl) = sref(2 + cur, i, cl);
            }
          }
        }
        if (lane == 0) {
          double* sa = snap_alpha + ((int64_t)blockIdx.x * NW_MAXW + wid) * (NW_SNAP + 1) * 2;
          if (save) {
            sa[NW_SNAP * 2 + 0] = sa[slot * 2 + 0];
            sa[NW_SNAP * 2 + 1] = sa[slot * 2 + 1];
            sh.bsw[wid] = evicted;
          }
          sa[slot * 2 + 0] = alpha;
          sa[slot * 2 + 1] = w_prev;
        }
        __syncwarp();
      }
      const int cur = k & 1, prv = cur ^ 1;
      const T w = (T)w_prev;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      for (int base = 0; wfirst + base < ncols; base += cstride) {
        const int cl = cfirst + base;
        if (cl < ncols) {
          step(cl, cur, prv, w, a0, a1, a2, true);
        } else {
          __syncwarp();
          __syncwarp();
        }
      }
      post(k, a0, a1, a2);
      if (k % NW_WIN == NW_WIN - 1 || k == max_iter - 1) post_flag(k);
      if (trace && lane == 0 && wid == 0 && k + 1 < NN_TRACE_LEN) {
        if (blockIdx.x == 0) g_nnls_trace(0)[k + 1] = gtimer_ns();
        if (blockIdx.x == gridDim.x - 1) g_nnls_trace(3)[k + 1] = gtimer_ns();
      }
      const double a1n = alpha_next_d(alpha);
      w_prev = __ddiv_rn(alpha - 1.0, a1n);
      alpha = a1n;
      if (lane == 0 && sh.halt) go = false;
      go = __shfl_sync(0xffffffffu, go ? 1 : 0, 0) != 0;
    }
    if (lane == 0) sh.kdone[wid] = k;  // warps may stop at different k; each keeps its own columns
  } else {
    resolver_warp(sh, pp, ncw, max_iter, grad_tol, L, recs, results, tracebuf, NW_MAXW, nullptr, NN_WATCHDOG_NS_DEFAULT);
  }
  __syncthreads();  // compute warps done; decisions final

  // ---------------------------------------------------------------- output
  const int bj = sh.best_j;
  if (!resolver && bj >= 0 && sh.fail_at < 0) {
    const int kd = sh.kdone[wid];  // iterations this warp computed: 0 .. kd-1
    if (bj == kd - 1 || bj == kd - 2) {
      // still live in a parity buffer
      const int buf = bj & 1;
      for (int base = 0; wfirst + base < ncols; base += cstride) {
        const int cl = cfirst + base;
        if (cl >= ncols) continue;
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
          const int i = ibase + r;
          if (i < p) Fout[(int64_t)i * c + j0 + cl] = sref(buf, i, cl);
        }
      }
    } else {
      // recompute F_bj from the snapshot of its window (same arithmetic)
      const int wb = bj / NW_WIN;
      const int slot = (sh.bsw[wid] == wb && wb + NW_SNAP <= (kd - 1) / NW_WIN) ? NW_SNAP : wb % NW_SNAP;
      const int k0 = wb * NW_WIN;
      const double* sa = snap_alpha + ((int64_t)blockIdx.x * NW_MAXW + wid) * (NW_SNAP + 1) * 2;
      double alpha = sa[slot * 2 + 0];
      double w_prev = sa[slot * 2 + 1];
      for (int base = 0; wfirst + base < ncols; base += cstride) {
        const int cl = cfirst + base;
        if (cl >= ncols) continue;
        const int cur = k0 & 1, prv = cur ^ 1;
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
          const int i = ibase + r;
          if (i < p) {
            sref(prv, i, cl) = snref(slot, 0, i, cl);
            sref(cur, i, cl) = snref(slot, 1, i, cl);
            sref(2 + prv, i, cl) = snref(slot, 2, i, cl);
            sref(2 + cur, i, cl) = snref(slot, 3, i, cl);
          }
        }
      }
      __syncwarp();
      double d0, d1, d2;
      for (int k = k0; k <= bj; ++k) {
        const int cur = k & 1, prv = cur ^ 1;
        const T w = (T)w_prev;
        for (int base = 0; wfirst + base < ncols; base += cstride) {
          const int cl = cfirst + base;
          if (cl < ncols) {
            step(cl, cur, prv, w, d0, d1, d2, false);
          } else {
            __syncwarp();
            __syncwarp();
          }
        }
        const double a1n = alpha_next_d(alpha);
        w_prev = __ddiv_rn(alpha - 1.0, a1n);
        alpha = a1n;
      }
      const int buf = bj & 1;
      for (int base = 0; wfirst + base < ncols; base += cstride) {
        const int cl = cfirst + base;
        if (cl >= ncols) continue;
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
          const int i = ibase + r;
          if (i < p) Fout[(int64_t)i * c + j0 + cl] = sref(buf, i, cl);
        }
      }
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    if (sh.fail_at >= 0) status_fail(st, NENMF_ERR_NUMERICAL_FAILURE, sh.fail_at);
    if (sh.fail_at == -2) status_fail(st, NENMF_ERR_WATCHDOG, -2);
    st->inner_iters = sh.stop_at >= 0 ? sh.stop_at + 1 : (sh.fail_at >= 0 ? sh.fail_at : max_iter);
    st->returned_best = sh.best_j >= 0 ? 1 : 0;
    st->best_partial = sh.best_part;
    st->pg_ref = sh.pg_ref;
  }
}


template <typename T, int TPC, int RMAX, bool SM>
static int launch_nnls_t(const NnlsPlan& pl, const T* W, const T* V, const T* F0, T* Fout, T* snaps, double* salpha,
                         T* gstate, int p, int64_t c, const double* Lptr, int max_iter, double grad_tol, WinRec* recs,
                         WinRec* results, nenmf_device_status* st, unsigned long long* tracebuf, cudaStream_t s) {
  auto fn = k_nnls<T, TPC, RMAX, SM>;
  if (pl.smem > 227 * 1024) return NENMF_ERR_UNSUPPORTED;  // W (padded p x p) + the sum ring: FP64 p <= 112, FP32 p <= 128
  NENMF_CUDA_TRY(set_smem(fn, pl.smem));
  int64_t cpb = pl.cpb;
  int ldS = pl.ldS, ldW = pl.ldW;
  void* args[] = {(void*)&W,    (void*)&V,      (void*)&F0,       (void*)&Fout,     (void*)&snaps, (void*)&salpha,
                  (void*)&gstate, (void*)&p,    (void*)&c,        (void*)&cpb,      (void*)&ldS,   (void*)&ldW,
                  (void*)&Lptr, (void*)&max_iter, (void*)&grad_tol, (void*)&recs,   (void*)&results, (void*)&st,
                  (void*)&tracebuf};
  NENMF_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)fn, dim3(pl.grid), dim3(pl.threads), args, pl.smem, s));
  launch_counter_add(1);
  return NENMF_OK;
}

#define NN_TARGS pl, W, V, F0, Fout, snaps, salpha, gstate, p, c, Lptr, max_iter, grad_tol, recs, results, st, tracebuf, s
template <typename T, int TPC, int RMAX>
static int launch_nnls_r(const NnlsPlan& pl, const T* W, const T* V, const T* F0, T* Fout, T* snaps, double* salpha,
                         T* gstate, int p, int64_t c, const double* Lptr, int max_iter, double grad_tol, WinRec* recs,
                         WinRec* results, nenmf_device_status* st, unsigned long long* tracebuf, cudaStream_t s) {
  if (pl.smem_state) return launch_nnls_t<T, TPC, RMAX, true>(NN_TARGS);
  return launch_nnls_t<T, TPC, RMAX, false>(NN_TARGS);
}

// instantiate launch_nnls_tpc<T, TPC>: RMAX 1..8 for TPC = 1, 5..8 otherwise
#define NENMF_NNLS_TPC_IMPL(T, TPC)                                                                               \
  template <>                                                                                                   \
  int launch_nnls_tpc<T, TPC>(const NnlsPlan& pl, const T* W, const T* V, const T* F0, T* Fout, T* snaps,         \
                              double* salpha, T* gstate, int p, int64_t c, const double* Lptr, int max_iter,       \
                              double grad_tol, WinRec* recs, WinRec* results, nenmf_device_status* st,             \
                              unsigned long long* tracebuf, cudaStream_t s) {                                     \
    switch (pl.rmax) {                                                                                          \
      case 1: if (TPC == 1) return launch_nnls_r<T, TPC, 1>(NN_TARGS); break;                                   \
      case 2: if (TPC == 1) return launch_nnls_r<T, TPC, 2>(NN_TARGS); break;                                   \
      case 3: if (TPC == 1) return launch_nnls_r<T, TPC, 3>(NN_TARGS); break;                                   \
      case 4: if (TPC == 1) return launch_nnls_r<T, TPC, 4>(NN_TARGS); break;                                   \
      case 5: return launch_nnls_r<T, TPC, 5>(NN_TARGS);                                                        \
      case 6: return launch_nnls_r<T, TPC, 6>(NN_TARGS);                                                        \
      case 7: return launch_nnls_r<T, TPC, 7>(NN_TARGS);                                                        \
      case 8: return launch_nnls_r<T, TPC, 8>(NN_TARGS);                                                        \
    }                                                                                                           \
    return NENMF_ERR_UNSUPPORTED;                                                                               \
  }

}  // namespace nenmf
