// Tensor-core variant of the persistent inner solver (included by nnls_m_*.cu).
//
// Same windowed decision protocol as nnls_kernel.cuh (resolver warp, window
// records summed in CTA order, snapshots for the best iterate), but each
// compute warp owns a block of 8 columns and keeps its whole state --
// F_{k-1}, F_{k-2}, g_{k-1}, g_{k-2}, V -- in registers, in the accumulator
// fragment layout of a warp-level MMA.  Per inner iteration:
//   elementwise F_k = max(0, Y + grad_Y / (-L))   (nnls.py:189-191,208-213)
//   F_k -> B fragments through a 1 KB per-warp shared tile
//   g_k = W F_k - V on the tensor pipe           (nnls.py:192-193)
//     FP32: mma m16n8k8 TF32 with the 3xTF32 split (hi*hi + hi*lo + lo*hi),
//           fp32-class accuracy; W's hi/lo fragments stay in registers
//     FP64: mma m8n8k4 F64 (exact fp64 products)
// The cross-warp/CTA sums and all decisions are identical to the SIMT kernel.
#pragma once
#include "nnls_common.cuh"

namespace nenmf {

template <typename T>
struct MmaShape;
template <>
struct MmaShape<float> {
  static constexpr int RM = 16, RK = 8, EPT = 4, BPT = 2;  // rows per M/K tile, C and B elements per thread
};
template <>
struct MmaShape<double> {
  static constexpr int RM = 8, RK = 4, EPT = 2, BPT = 1;
};

// 3xTF32 split by truncation: hi keeps the top 10 mantissa bits (exactly
// representable), lo = x - hi is exact in fp32 and is handed to the MMA raw
// (the tensor core ignores its low 13 bits).  Two instructions per value
// instead of the cvt.rna sequence; the dropped lo*lo term and lo's truncation
// leave a relative error ~2^-20 per product, fp32-class.
__device__ __forceinline__ uint32_t tf32_hi(float x) { return __float_as_uint(x) & 0xffffe000u; }
__device__ __forceinline__ uint32_t tf32_lo(float x, uint32_t hi) { return __float_as_uint(x - __uint_as_float(hi)); }

// Register budget of one compute thread -> CTA size the kernel is compiled for.
// (state: 5 arrays of NE elements; W fragments; fixed overhead, larger for f64)
template <typename T>
__host__ __device__ constexpr int mma_threads(int mt, int kt) {
  return (5 * (sizeof(T) == 4 ? 4 : 2) * mt * (int)(sizeof(T) / 4) + (sizeof(T) == 4 ? 8 : 2) * mt * kt +
          (sizeof(T) == 4 ? 56 : 74)) <= 128
             ? 512
             : ((5 * (sizeof(T) == 4 ? 4 : 2) * mt * (int)(sizeof(T) / 4) + (sizeof(T) == 4 ? 8 : 2) * mt * kt +
                 (sizeof(T) == 4 ? 56 : 74)) <= 170
                    ? 384
                    : 256);
}
template <typename T, int MT, int KT>
struct MmaBudget {
  static constexpr int THREADS = mma_threads<T>(MT, KT);
};

__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_f64(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <typename T, int MT, int KT>
__global__ void __launch_bounds__(MmaBudget<T, MT, KT>::THREADS, 1)
k_nnls_mma(const T* __restrict__ W, const T* __restrict__ V, const T* __restrict__ F0, T* __restrict__ Fout,
           T* __restrict__ snaps, double* __restrict__ snap_alpha, int p, int64_t c, int64_t cpb,
           const double* __restrict__ Lptr, int max_iter, double grad_tol, WinRec* __restrict__ recs,
           WinRec* __restrict__ results, nenmf_device_status* st, unsigned long long* __restrict__ tracebuf,
           const double* __restrict__ wtab) {
  using S = MmaShape<T>;
  constexpr int NE = S::EPT * MT;          // state elements per thread
  constexpr int NROW = S::RM * MT;         // padded rows of the warp's tile
  extern __shared__ __align__(16) double smem_d[];
  double* pp = smem_d;                                            // [PPD][MAXW][3]
  T* stage_all = reinterpret_cast<T*>(pp + (size_t)NW_PPD * NW_MAXW * 3);  // [warps][NROW][8]
  __shared__ SolverShared sh;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ncw = (blockDim.x >> 5) - 1;
  const bool resolver = wid == ncw;
  const int64_t j0 = (int64_t)blockIdx.x * cpb;
  const int ncols = (int)(imin(c, j0 + cpb) - j0);
  const int64_t pc = (int64_t)p * c;
  const int gq = lane >> 2, tq = lane & 3;
  solver_shared_init(sh);
  __syncthreads();
  if (st->code != 0) return;
  const double L = *Lptr;
  const T rnegL = (T)(-1.0 / L);

  // element e of this thread: row / column within the warp's 8-column block
  auto erow = [&](int e) -> int {
    if constexpr (S::EPT == 4) return 16 * (e >> 2) + gq + ((e & 2) ? 8 : 0);
    else return 8 * (e >> 1) + gq;
  };
  auto ecol = [&](int e) -> int { return 2 * tq + (e & 1); };
  const int cblk = 8 * wid;                     // first CTA-local column of this warp
  auto gcol = [&](int e) -> int64_t { return j0 + cblk + ecol(e); };
  auto evalid = [&](int e) -> bool { return erow(e) < p && cblk + ecol(e) < ncols; };
  auto snref = [&](int s, int b, int e) -> T& { return snaps[(((int64_t)s * 4 + b) * p + erow(e)) * c + gcol(e)]; };

  if (!resolver) {
    T* stage = stage_all + (size_t)wid * NROW * 8;
    // W fragments (A operand), resident for the whole solve
    uint32_t ahi[MT][KT][4], alo[MT][KT][4];
    double ad[MT][KT];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        if constexpr (S::EPT == 4) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int i = 16 * mt + gq + ((r & 1) ? 8 : 0);
            const int l = 8 * kt + tq + ((r & 2) ? 4 : 0);
            const float w = (i < p && l < p) ? (float)W[i * p + l] : 0.f;
            ahi[mt][kt][r] = tf32_hi(w);
            alo[mt][kt][r] = tf32_lo(w, ahi[mt][kt][r]);
          }
        } else {
          const int i = 8 * mt + gq, l = 4 * kt + tq;
          ad[mt][kt] = (i < p && l < p) ? (double)W[i * p + l] : 0.0;
        }
      }
    // g = W f for the warp's block: f given in accumulator layout (fe)
    auto matvec = [&](const T (&fe)[NE], T (&acc)[NE]) {
#pragma unroll
      for (int e = 0; e < NE; ++e) stage[erow(e) * 8 + ecol(e)] = fe[e];
      __syncwarp();
      if constexpr (S::EPT == 4) {
        uint32_t bh[KT][2], bl[KT][2];
#pragma unroll
        for (int kt = 0; kt < KT; ++kt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float f = stage[(8 * kt + tq + 4 * h) * 8 + gq];
            bh[kt][h] = tf32_hi(f);
            bl[kt][h] = tf32_lo(f, bh[kt][h]);
          }
        __syncwarp();
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          // three independent accumulation chains (lo*hi, hi*lo, hi*hi), summed small-first
          float c0[4] = {0.f, 0.f, 0.f, 0.f}, c1[4] = {0.f, 0.f, 0.f, 0.f}, c2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int kt = 0; kt < KT; ++kt) {
            mma_tf32(c0, alo[mt][kt], bh[kt][0], bh[kt][1]);
            mma_tf32(c1, ahi[mt][kt], bl[kt][0], bl[kt][1]);
            mma_tf32(c2, ahi[mt][kt], bh[kt][0], bh[kt][1]);
          }
#pragma unroll
          for (int r = 0; r < 4; ++r) acc[4 * mt + r] = (T)((c0[r] + c1[r]) + c2[r]);
        }
      } else {
        double bd[KT];
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) bd[kt] = (double)stage[(4 * kt + tq) * 8 + gq];
        __syncwarp();
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          double cc[2] = {0.0, 0.0};
#pragma unroll
          for (int kt = 0; kt < KT; ++kt) mma_f64(cc, ad[mt][kt], bd[kt]);
          acc[2 * mt] = (T)cc[0];
          acc[2 * mt + 1] = (T)cc[1];
        }
      }
    };

    T f1[NE], f2[NE], q1[NE], q2[NE], vv[NE];
    auto post = [&](int j, T s0, T s1, T s2) {
      // warp-level sums in the working precision, CTA and grid levels in double
      double a0, a1, a2;
      if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          s0 += __shfl_xor_sync(0xffffffffu, s0, o);
          s1 += __shfl_xor_sync(0xffffffffu, s1, o);
          s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        }
        a0 = s0;
        a1 = s1;
        a2 = s2;
      } else {
        a0 = warp_sum((double)s0);
        a1 = warp_sum((double)s1);
        a2 = warp_sum((double)s2);
      }
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
    // one iteration: (f1, f2, q1, q2) -> F_k, g_k; returns the thread's sums
    auto step = [&](T w, T& s0, T& s1, T& s2) {
      T fk[NE], acc[NE];
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        // contracted to FMAs here: the MMA product already fixes a different
        // rounding sequence than the reference's matmul (tolerance parity)
        const T y = fma_acc(op_sub(f1[e], f2[e]), w, f1[e]);
        const T gy = fma_acc(op_sub(q1[e], q2[e]), w, q1[e]);
        fk[e] = relu_nan(fma_acc(gy, rnegL, y));
      }
      matvec(fk, acc);
      s0 = s1 = s2 = T(0);
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const T g = op_sub(acc[e], vv[e]);
        const T pgv = fk[e] > T(0) ? g : min0_nan(g);
        s0 = fma_acc(pgv, pgv, s0);
        s1 = fma_acc(fk[e], g, s1);
        s2 = fma_acc(fk[e], vv[e], s2);
        f2[e] = f1[e];
        f1[e] = fk[e];
        q2[e] = q1[e];
        q1[e] = g;
      }
    };

    // start point (nnls.py:163-178); columns/rows outside the problem stay 0
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const bool ok = evalid(e);
      f1[e] = ok ? F0[(int64_t)erow(e) * c + gcol(e)] : T(0);
      f2[e] = f1[e];
      vv[e] = ok ? V[(int64_t)erow(e) * c + gcol(e)] : T(0);
    }
    {
      T acc[NE];
      matvec(f1, acc);
      T s0 = T(0), s1 = T(0), s2 = T(0);
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const T g = op_sub(acc[e], vv[e]);
        q1[e] = g;
        q2[e] = g;
        const T pgv = f1[e] > T(0) ? g : min0_nan(g);
        s0 = fma_acc(pgv, pgv, s0);
        s1 = fma_acc(f1[e], g, s1);
        s2 = fma_acc(f1[e], vv[e], s2);
      }
      post(-1, s0, s1, s2);
      post_flag(-1);
    }

    double alpha = 1.0, w_prev = 0.0, wwin = 0.0;
    int k = 0;
    bool go = true;
    const bool has_cols = cblk < ncols;
    for (; k < max_iter && go; ++k) {
      if (k % NW_WIN == 0) {
        if (wtab != nullptr) wwin = k + lane < max_iter ? wtab[k + lane] : 0.0;
        const int w = k / NW_WIN;
        int ok = 1;
        if (lane == 0) {
          const int need = (w - NW_FLIGHT) * NW_WIN - 1;
          while (sh.resolved < need && !sh.halt) __nanosleep(64);
          ok = sh.halt ? 0 : 1;
        }
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (!ok) break;
        const int slot = w % NW_SNAP;
        const int evicted = w - NW_SNAP;
        const int bj = sh.best_j;
        const bool save = evicted >= 0 && bj >= 0 && bj / NW_WIN == evicted;
        if (has_cols) {
#pragma unroll
          for (int e = 0; e < NE; ++e)
            if (evalid(e)) {
              if (save)
                for (int b = 0; b < 4; ++b) snref(NW_SNAP, b, e) = snref(slot, b, e);
              snref(slot, 0, e) = f1[e];
              snref(slot, 1, e) = f2[e];
              snref(slot, 2, e) = q1[e];
              snref(slot, 3, e) = q2[e];
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
      const int halt_early = sh.halt;  // consumed at the end of the iteration
      T s0, s1, s2;
      step((T)w_prev, s0, s1, s2);
      post(k, s0, s1, s2);
      if (k % NW_WIN == NW_WIN - 1 || k == max_iter - 1) post_flag(k);
      if (tracebuf != nullptr && lane == 0 && wid == 0 && k + 1 < NN_TRACE_LEN) {
        if (blockIdx.x == 0) tracebuf[k + 1] = gtimer_ns();
        if (blockIdx.x == gridDim.x - 1) tracebuf[3 * NN_TRACE_LEN + k + 1] = gtimer_ns();
      }
      if (wtab != nullptr) {
        w_prev = __shfl_sync(0xffffffffu, wwin, k % NW_WIN);  // w_k = (alpha_k - 1) / alpha_{k+1}
      } else {
        const double a1n = alpha_next_d(alpha);
        w_prev = __ddiv_rn(alpha - 1.0, a1n);
        alpha = a1n;
      }
      go = halt_early == 0;  // one LDS per warp: every lane sees the same value
    }
    if (lane == 0) sh.kdone[wid] = k;
    __syncwarp();

    // -------------------------------------------------------------- output
    // (waits for the resolver's final decision through the block barrier below)
    asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
    const int bj = sh.best_j;
    if (bj >= 0 && sh.fail_at < 0 && has_cols) {
      const int kd = sh.kdone[wid];
      if (bj == kd - 1 || bj == kd - 2) {
#pragma unroll
        for (int e = 0; e < NE; ++e)
          if (evalid(e)) Fout[(int64_t)erow(e) * c + gcol(e)] = bj == kd - 1 ? f1[e] : f2[e];
      } else {
        const int wb = bj / NW_WIN;
        const int slot = (sh.bsw[wid] == wb && wb + NW_SNAP <= (kd - 1) / NW_WIN) ? NW_SNAP : wb % NW_SNAP;
        const double* sa = snap_alpha + ((int64_t)blockIdx.x * NW_MAXW + wid) * (NW_SNAP + 1) * 2;
        double alpha2 = sa[slot * 2 + 0];
        double wp = sa[slot * 2 + 1];
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          const bool ok = evalid(e);
          f1[e] = ok ? snref(slot, 0, e) : T(0);
          f2[e] = ok ? snref(slot, 1, e) : T(0);
          q1[e] = ok ? snref(slot, 2, e) : T(0);
          q2[e] = ok ? snref(slot, 3, e) : T(0);
        }
        for (int kk = wb * NW_WIN; kk <= bj; ++kk) {
          T s0, s1, s2;
          step((T)wp, s0, s1, s2);
          if (wtab != nullptr) {
            wp = wtab[kk];
          } else {
            const double a1n = alpha_next_d(alpha2);
            wp = __ddiv_rn(alpha2 - 1.0, a1n);
            alpha2 = a1n;
          }
        }
#pragma unroll
        for (int e = 0; e < NE; ++e)
          if (evalid(e)) Fout[(int64_t)erow(e) * c + gcol(e)] = f1[e];
      }
    }
  } else {
    resolver_warp(sh, pp, ncw, max_iter, grad_tol, L, recs, results, tracebuf);
    asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
  }
  __syncthreads();
  if (blockIdx.x == 0 && tid == 0) {
    if (sh.fail_at >= 0) status_fail(st, NENMF_ERR_NUMERICAL_FAILURE, sh.fail_at);
    if (sh.fail_at == -2) status_fail(st, NENMF_ERR_CUDA, -2);
    st->inner_iters = sh.stop_at >= 0 ? sh.stop_at + 1 : (sh.fail_at >= 0 ? sh.fail_at : max_iter);
    st->returned_best = sh.best_j >= 0 ? 1 : 0;
    st->best_partial = sh.best_part;
    st->pg_ref = sh.pg_ref;
  }
}

template <typename T, int MT, int KT>
static int launch_nnls_mma_t(const T* W, const T* V, const T* F0, T* Fout, T* snaps, double* salpha, int p, int64_t c,
                             int grid, int64_t cpb, const double* Lptr, int max_iter, double grad_tol, WinRec* recs,
                             WinRec* results, nenmf_device_status* st, unsigned long long* tracebuf,
                             const double* wtab, cudaStream_t s) {
  using S = MmaShape<T>;
  const int ncw = (int)cdiv(cpb, 8);
  const int threads = 32 * (ncw + 1);
  if (threads > MmaBudget<T, MT, KT>::THREADS) return NENMF_ERR_UNSUPPORTED;
  const size_t smem = (size_t)NW_PPD * NW_MAXW * 3 * sizeof(double) + (size_t)ncw * S::RM * MT * 8 * sizeof(T);
  auto fn = k_nnls_mma<T, MT, KT>;
  NENMF_CUDA_TRY(set_smem(fn, smem));
  void* args[] = {(void*)&W,    (void*)&V,        (void*)&F0,       (void*)&Fout,    (void*)&snaps,
                  (void*)&salpha, (void*)&p,      (void*)&c,        (void*)&cpb,     (void*)&Lptr,
                  (void*)&max_iter, (void*)&grad_tol, (void*)&recs, (void*)&results, (void*)&st,
                  (void*)&tracebuf, (void*)&wtab};
  NENMF_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(threads), args, smem, s));
  launch_counter_add(1);
  return NENMF_OK;
}

#define NENMF_NNLS_MMA_IMPL(T)                                                                                       \
  template <>                                                                                                      \
  int nnls_mma_max_cols<T>(int p) {                                                                                \
    using S = MmaShape<T>;                                                                                         \
    const int mt = (int)cdiv(p, S::RM);                                                                            \
    const int kt = mt * (S::RM / S::RK);                                                                           \
    return 8 * (mma_threads<T>(mt, kt) / 32 - 1);                                                                  \
  }                                                                                                                \
  template <>                                                                                                      \
  int launch_nnls_mma<T>(const T* W, const T* V, const T* F0, T* Fout, T* snaps, double* salpha, int p, int64_t c,   \
                         int grid, int64_t cpb, const double* Lptr, int max_iter, double grad_tol, WinRec* recs,     \
                         WinRec* results, nenmf_device_status* st, unsigned long long* tracebuf,                 \
                         const double* wtab, cudaStream_t s) {                                                   \
    using S = MmaShape<T>;                                                                                         \
    const int mt = (int)cdiv(p, S::RM), kt = (int)cdiv(p, S::RK);                                                  \
    const int key = mt * 16 + kt;                                                                                  \
    switch (key) {                                                                                                 \
      NENMF_MMA_CASES(T)                                                                                           \
      default: return NENMF_ERR_UNSUPPORTED;                                                                       \
    }                                                                                                              \
  }

}  // namespace nenmf
