// Tensor-core variant of the persistent inner solver (included by nnls_m_*.cu).
//
// Same windowed decision protocol as nnls_kernel.cuh (resolver warp, window
// records summed in CTA order, snapshots for the best iterate), but each
// compute warp owns a block of columns and keeps its whole state --
// F_{k-1}, F_{k-2}, g_{k-1}, g_{k-2}, V -- in registers, in the accumulator
// fragment layout of a warp-level MMA.  Per inner iteration:
//   elementwise F_k = max(0, Y + grad_Y / (-L))   (nnls.py:189-191,208-213)
//   g_k = W F_k - V on the tensor pipe           (nnls.py:192-193)
// The cross-warp/CTA sums and all decisions are identical to the SIMT kernel.
#pragma once
#include "nnls_common.cuh"

namespace nenmf {

// Data columns are the MMA's M dimension and the solver rows its N and K
// dimensions: g^T (cols x p) = F^T (cols x p) * W^T.  With the K index of
// k-tile t permuted as slot tq -> row 8t+2tq, slot tq+4 -> row 8t+2tq+1, the
// accumulator fragment of n-tile t IS the A fragment of k-tile t, so an
// iteration never leaves registers: elementwise update on the accumulator
// layout -> A fragments -> MMAs -> next accumulator.
//   FP32: 16 columns per warp, 3xTF32: hi*hi, lo*hi and hi*lo on m16n8k8
//         TF32 (relative error ~2^-21 per product; an earlier variant folded
//         the corrections into one BF16 m16n8k16 MMA -- 18 instead of 27 MMAs
//         -- but its 8-bit operands left one-step factors ~1.3e-3 from the
//         fp64 reference, outside the FP32 mode's 1e-3); 27 MMAs per
//         iteration at p <= 24, W^T fragments resident
//   FP64: m8n8k4 F64, 8 columns per warp, exact products
template <typename T>
struct MmaShape;
template <>
struct MmaShape<float> {
  static constexpr int CB = 16, EPT = 4;  // columns per warp, state elements per thread per n-tile
};
template <>
// FP64, NN_F64_WIDE = 1 (compile-time experiment, off): a warp owns TWO 8-column DMMA m-tiles
// (columns gq and gq + 8, the element layout of the fp32 accumulator) and the CTA 5 compute warps
// instead of 9 at cfg2.  Measured slower (1.14 vs 0.88 us per inner iteration): the iteration is
// bound by each warp's own dependent instruction stream, which nine warps hide better than the
// two interleaved column groups of five.
#ifndef NN_F64_WIDE
#define NN_F64_WIDE 0
#endif
struct MmaShape<double> {
#if NN_F64_WIDE
  static constexpr int CB = 16, EPT = 4;
#else
  static constexpr int CB = 8, EPT = 2;
#endif
};

// 3xTF32 split: hi keeps the top 10 mantissa bits by truncation (exactly
// representable), lo = x - hi is exact in fp32 and rounded to nearest TF32;
// the dropped lo*lo term and lo's rounding leave a relative error ~2^-22 per
// product.
__device__ __forceinline__ uint32_t tf32_hi(float x) { return __float_as_uint(x) & 0xffffe000u; }
// FP32 correction terms: false = two TF32 MMAs (lo*hi, hi*lo) per k-tile;
// true = one BF16 m16n8k16 MMA over [F_lo | F_hi] x [W_hi ; W_lo]
#ifndef NN_FP32_BF16_CORR
#define NN_FP32_BF16_CORR 0
#endif
// the residual rounded to nearest TF32 (the tensor core would truncate it)
__device__ __forceinline__ uint32_t tf32_lo(float x, uint32_t hi) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x - __uint_as_float(hi)));
  return r;
}

// CTA size each instantiation is compiled for (register budget per thread:
// 5 state arrays of 4*NT (fp32) / 2*NT doubles, resident W fragments, the
// address/bookkeeping registers); chosen so that ptxas reports no spills.
template <typename T>
__host__ __device__ constexpr int mma_threads(int nt) {
  if (sizeof(T) == 8 && NN_F64_WIDE) return nt <= 1 ? 512 : 256;
  return sizeof(T) == 4 ? (nt <= 2 ? 512 : 256) : (nt <= 1 ? 512 : (nt == 2 ? 384 : (nt == 3 ? 320 : 256)));
}

__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// two fp32 -> packed bf16x2 (round to nearest), first value in the low half
__device__ __forceinline__ uint32_t pack_bf16(float lo_idx, float hi_idx) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_idx), "f"(lo_idx));
  return r;
}
__device__ __forceinline__ void mma_f64(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// smem carve-up of the fused prologue/epilogue (after the pp ring)
template <typename T, int NT>
__global__ void __launch_bounds__(mma_threads<T>(NT), 1)
k_nnls_mma(const __grid_constant__ MmaArgs<T> A) {
  using S = MmaShape<T>;
  constexpr int NE = S::EPT * NT;  // state elements per thread
  const T* __restrict__ F0 = A.F0;
  T* __restrict__ Fout = A.Fout;
  T* __restrict__ snaps = A.snaps;
  const int p = A.p, max_iter = A.max_iter, dbg = A.dbg;
  const int64_t c = A.c, cpb = A.cpb;
  const double* __restrict__ wtab = A.wtab;
  unsigned long long* __restrict__ tracebuf = A.tracebuf;
  nenmf_device_status* st = A.st;
  const bool fused = A.fused != 0;
  const int r = (int)A.r;
  extern __shared__ __align__(16) double smem_d[];
  double* pp = smem_d;  // [PPD][MAXW][3]
  // fused-mode scratch
  T* At_s = reinterpret_cast<T*>(pp + (size_t)NW_PPD * NW_MAXW * 3);  // [p][r]
  T* W_s = At_s + ((size_t)p * r + 3) / 4 * 4;                          // [32][32]
  double* gram = reinterpret_cast<double*>(W_s + 32 * 32);             // [k][k]
  double* pv = gram + 32 * 32;                                          // [64]
  T* ftile_all = reinterpret_cast<T*>(pv + 64);                         // [ncw][32][CB]
  T* Bs = ftile_all + (size_t)((blockDim.x >> 5) - 1) * 2 * 32 * S::CB;  // [r][cpb]: B of this CTA's columns
  __shared__ SolverShared sh;
  __shared__ double s_L, s_red[NW_MAXW][2];
  __shared__ int s_start_wins;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ncw = (blockDim.x >> 5) - 1;
  const bool resolver = wid == ncw;
  // rank group: the launch's CTAs split into virtual ranks of
  // grid_r CTAs; each virtual rank owns the columns [col0[vr], col0[vr + 1])
  const bool grouped = A.grp.ranks > 1;
  const int Gr = grouped ? A.grp.grid_r : (int)gridDim.x;
  const int vr = grouped ? (int)blockIdx.x / Gr : 0;
  const int lb = grouped ? (int)blockIdx.x % Gr : (int)blockIdx.x;
  const int g_lo = vr * Gr, g_hi = g_lo + Gr;
  const int64_t vc0 = grouped ? A.grp.col0[vr] : 0, vc1 = grouped ? A.grp.col0[vr + 1] : c;
  const int64_t vcpb = grouped ? (vc1 - vc0 + Gr - 1) / Gr : cpb;
  const int64_t j0 = vc0 + (int64_t)lb * vcpb;
  const int ncols = (int)imax(0, imin(vc1, j0 + vcpb) - j0);
  const int gq = lane >> 2, tq = lane & 3;
  solver_shared_init(sh);
  __syncthreads();
  if (tracebuf != nullptr && blockIdx.x == 0 && tid == 0) tracebuf[NN_TRACE_LEN + 60 + 0] = gtimer_ns();
  if (tracebuf != nullptr && tid == 0 && blockIdx.x < 512) tracebuf[blockIdx.x] = gtimer_ns();  // per-CTA start
  if (st->code != 0) return;

  // element e of this thread: solver row / CTA-local column
  // FP64 K permutation: the accumulator slot (8-row tile j, slot i = 2 tq + h) is both an output
  // row of g and, one iteration later, a K index of the next product (k-step 2j + h covers the
  // slots i = h, h + 2, h + 4, h + 6).  With p % 8 in 1..4 the last tile's real rows are kept in
  // its even slots (solver row 8j + i / 2), so its odd slots -- one whole k-step -- are padding
  // and that k-step's DMMAs are skipped (p = 20: 15 DMMAs per iteration instead of 18).
  constexpr int PLAST = 8 * (NT - 1);
  const bool kperm = sizeof(T) == 8 && p > PLAST && p - PLAST <= 4;
  auto slot_row = [&](int j, int i) -> int {  // solver row of slot i of tile j
    if (sizeof(T) == 4 || j < NT - 1 || !kperm) return 8 * j + i;
    return PLAST + ((i & 1) ? 4 + (i >> 1) : (i >> 1));
  };
  auto erow = [&](int e) -> int {
    if constexpr (S::EPT == 4) return slot_row(e >> 2, 2 * tq + (e & 1));
    else return slot_row(e >> 1, 2 * tq + (e & 1));
  };
  const int cblk = S::CB * wid;  // first CTA-local column of this warp
  auto ecol = [&](int e) -> int {
    if constexpr (S::EPT == 4) return cblk + gq + ((e & 2) ? 8 : 0);
    else return cblk + gq;
  };
  auto evalid = [&](int e) -> bool { return erow(e) < p && ecol(e) < ncols; };
  // offset of element e in a p x c row-major array: one IMAD per element
  const int64_t pc = (int64_t)p * c;
  const int64_t ebase = (int64_t)(2 * tq) * c + j0 + cblk + gq;
  auto eoff = [&](int e) -> int64_t {
    if constexpr (sizeof(T) == 4) return (int64_t)(8 * (e >> 2) + (e & 1)) * c + ((e & 2) ? 8 : 0) + ebase;
    else return (int64_t)erow(e) * c + j0 + ecol(e);
  };
  auto snref = [&](int s, int b, int e) -> T& { return snaps[(int64_t)(s * 4 + b) * pc + eoff(e)]; };
  // B(t, global column j) of the reference's V = A^T B (B may be a transposed view)
  // B(t, CTA-local column jl) of the reference's V = A^T B, staged in smem
  auto bval = [&](int t, int jl) -> T { return Bs[(size_t)t * cpb + jl]; };
  // explicit residual 1/2||A F - B||^2 of one candidate (0: best, 1: start)
  // over the 16 columns of compute warp w, staged in its ftile slot, into
  // s_red[w][which] (k_resid arithmetic: T products summed over rows in
  // order, double squares); each lane owns one column and a stride of rows t
  auto resid_rows = [&](int w, int which) {
    double acc = 0.0;
    const int cb0 = S::CB * w;
    if (cb0 < ncols) {
      const T* ft = ftile_all + (size_t)w * 2 * 32 * S::CB + (size_t)which * 32 * S::CB;  // [32][CB]
      const int nloc = imin(S::CB, ncols - cb0);
      const int jl = lane % S::CB;
      constexpr int TSTEP = 32 / S::CB;
      if (jl < nloc) {
        const T* fb = ft + jl;
        for (int t = lane / S::CB; t < r; t += TSTEP) {
          T s0 = T(0);
          const T* at = At_s + t;
#pragma unroll 4
          for (int a2 = 0; a2 < p; ++a2) s0 = fma_acc(at[a2 * r], fb[a2 * S::CB], s0);
          const double d0 = (double)(s0 - bval(t, cb0 + jl));
          acc += d0 * d0;
        }
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) s_red[w][which] = acc;
  };
  // compute warps: a candidate held in registers (accumulator layout)
  auto resid_one = [&](const T (&fv)[NE], int which) {
    if (cblk < ncols) {
      T* ft = ftile_all + (size_t)wid * 2 * 32 * S::CB + (size_t)which * 32 * S::CB;
#pragma unroll
      for (int e = 0; e < NE; ++e)
        if (evalid(e)) ft[erow(e) * S::CB + (ecol(e) - cblk)] = fv[e];
    }
    __syncwarp();
    resid_rows(wid, which);
    __syncwarp();
  };
  // resolver warp: the start point of every compute warp's columns, from F0
  auto resid_start_all = [&](int ncw_) {
    for (int w = 0; w < ncw_; ++w) {
      const int cb0 = S::CB * w;
      if (cb0 >= ncols) {
        if (lane == 0) s_red[w][1] = 0.0;
        continue;
      }
      T* ft = ftile_all + (size_t)w * 2 * 32 * S::CB + 32 * S::CB;
      for (int i = lane; i < p * S::CB; i += 32) {
        const int a2 = i / S::CB, jl = i % S::CB;
        ft[a2 * S::CB + jl] = cb0 + jl < ncols ? F0[(int64_t)a2 * c + j0 + cb0 + jl] : T(0);
      }
      __syncwarp();
      resid_rows(w, 1);
      __syncwarp();
    }
  };
  auto stage_pt = [&](int i0, int nthr) {
    T* Ps = Bs + (size_t)r * cpb + (size_t)p * cpb;  // [nup][cpb]
    for (int i = i0; i < (int)A.nup * ncols; i += nthr) {
      const int b = i / ncols, jl = i % ncols;
      Ps[(size_t)b * cpb + jl] = A.Pt[(int64_t)b * c + j0 + jl];
    }
  };

  T nv[NE];  // -V in the accumulator layout (compute warps)
  if (fused) {
    // ---- prologue: At -> smem, W = A^T A (k_abt order: double, t ascending)
    for (int i = tid; i < p * r; i += blockDim.x)
      asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"((uint32_t)__cvta_generic_to_shared(At_s + i)),
                   "l"(A.At + i), "n"((int)sizeof(T))
                   : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    // the power iteration's start vector, loaded while At is staged
    if (resolver && lane < (p <= r ? p : r)) pv[lane] = A.pvec[lane];
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    for (int o = tid; o < p * p; o += blockDim.x) {
      const int a = o / p, b = o % p;
      double acc = 0.0;
      for (int t = 0; t < r; ++t) acc = fma((double)At_s[a * r + t], (double)At_s[b * r + t], acc);
      W_s[a * 32 + b] = (T)acc;
    }
    __syncthreads();
    if (resolver) {
      // L = lambda_max of the smaller Gram (matrix.py:131-174, as k_power):
      // one row per lane, fixed-order warp sums -> identical in every CTA
      const int k = p <= r ? p : r;
      if (p > r) {  // A A^T (r x r), k_gram_rows order
        for (int o = lane; o < r * r; o += 32) {
          const int s2 = o / r, t2 = o % r;
          double acc = 0.0;
          for (int a = 0; a < p; ++a) acc = fma((double)At_s[a * r + s2], (double)At_s[a * r + t2], acc);
          gram[o] = (double)(T)acc;
        }
      } else {
        for (int o = lane; o < k * k; o += 32) gram[o] = (double)W_s[(o / k) * 32 + (o % k)];
      }
      double* v = pv;  // start vector loaded with At above
      __syncwarp();
      // this lane's Gram row in registers (the row reads from shared memory
      // would conflict: rows are k doubles apart); same arithmetic as k_power
      double grow[32];
#pragma unroll
      for (int l = 0; l < 32; ++l) grow[l] = (lane < k && l < k) ? gram[lane * k + l] : 0.0;
      int draw = 1;
      double est = 0.0;
      bool conv_any = false;
      int pits = 0;
      for (int it = 0; it < A.pmax; ++it) {
        ++pits;
        double wi = 0.0;
        if (lane < k) {
#pragma unroll
          for (int l = 0; l < 32; ++l)
            if (l < k) wi = fma(grow[l], v[l], wi);
        }
        const double nw = sqrt(warp_sum(lane < k ? fma(wi, wi, 0.0) : 0.0));
        __syncwarp();
        if (nw == 0.0) {
          if (lane < k) v[lane] = draw < A.pcount ? A.pvec[(int64_t)draw * k + lane] : 0.0;
          ++draw;
          __syncwarp();
          continue;
        }
        const bool conv = fabs(nw - est) <= A.ptol * nw;
        est = nw;
        if (lane < k) v[lane] = __ddiv_rn(wi, nw);
        __syncwarp();
        if (conv) {
          conv_any = true;
          break;
        }
      }
      if (!conv_any) est = est * 1.01;
      if (tracebuf != nullptr && blockIdx.x == 0 && lane == 0) tracebuf[NN_TRACE_LEN + 60 + 15] = (unsigned long long)pits;
      if (tracebuf != nullptr && blockIdx.x == 0 && lane == 0) tracebuf[NN_TRACE_LEN + 60 + 11] = gtimer_ns();
      if (lane == 0) {
        s_L = A.safety * est;
        if (blockIdx.x == 0) {
          A.L[0] = s_L;
          st->lipschitz = s_L;
        }
      }
    } else {
      // B columns of this CTA -> smem (compute warps, overlapping the power
      // iteration; coalesced along B's contiguous dimension)
      if (A.trans) {
        for (int jl = wid; jl < ncols; jl += ncw)
          for (int t = lane; t < r; t += 32) Bs[(size_t)t * cpb + jl] = A.B[(j0 + jl) * A.ldb + t];
      } else {
        // asynchronous element copies: every element of the block in flight at once
        for (int t = wid; t < r; t += ncw)
          for (int jl = lane; jl < ncols; jl += 32)
            asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(Bs + (size_t)t * cpb + jl)),
                         "l"(A.B + (int64_t)t * A.ldb + j0 + jl), "n"((int)sizeof(T))
                         : "memory");
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
      }
      // the start point is read right after the prologue: pull it into L1 now
#pragma unroll
      for (int e = 0; e < NE; ++e)
        if (evalid(e)) asm volatile("prefetch.global.L1 [%0];" ::"l"(F0 + eoff(e)));
      asm volatile("bar.sync 2, %0;" ::"r"(ncw * 32) : "memory");
      // this warp's columns of V = A^T B (k_ab order: T precision, t ascending)
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        T acc = T(0);
        if (evalid(e)) {
          const int a = erow(e), jl = ecol(e);
          for (int t = 0; t < r; ++t) acc = fma_acc(At_s[a * r + t], bval(t, jl), acc);
        }
        nv[e] = -acc;
      }
    }
    __syncthreads();
    if (s_L == 0.0) {  // zero Gram: ZeroMatrixError (matrix.py:172-173)
      if (blockIdx.x == 0 && tid == 0) status_fail(st, NENMF_ERR_ZERO_MATRIX, 0);
      return;
    }
  } else {
    if (tid == 0) s_L = A.L[0];
    __syncthreads();
  }
  const double L = s_L;
  if (tracebuf != nullptr && blockIdx.x == 0 && tid == 0) tracebuf[NN_TRACE_LEN + 60 + 3] = gtimer_ns();
  const T rnegL = (T)(-1.0 / L);
  const T* __restrict__ W = A.W;

  // the final iterate is the best one (the common case: the objective still
  // falls at max_iter) when every warp's last iteration is the decided best
  auto spec_hit = [&](int bj_) -> bool {
    if (!fused || bj_ < 0 || sh.fail_at != -1) return false;
    for (int w = 0; w < ncw; ++w)
      if (sh.kdone[w] - 1 != bj_) return false;
    return true;
  };
  // partials of the next product Pout = F Pt^T (factorize.py:110,113) over this
  // CTA's columns for one candidate (0: the best iterate, staged in ftile; 1:
  // the start point), by threads [0, nthr); sync() orders the smem staging
  auto next_partials = [&](int cand, int nthr, auto&& sync) {
    const int nup = (int)A.nup, no = p * nup;
    T* Fs = Bs + (size_t)r * cpb;  // [p][cpb]
    T* Ps = Fs + (size_t)p * cpb;  // [nup][cpb]
    sync();
    for (int i = tid; i < p * ncols; i += nthr) {
      const int a2 = i / ncols, jl = i % ncols;
      Fs[(size_t)a2 * cpb + jl] = cand == 0 ? ftile_all[(size_t)(jl / S::CB) * 2 * 32 * S::CB + a2 * S::CB + jl % S::CB]
                                            : F0[(int64_t)a2 * c + j0 + jl];
    }
    sync();
    // 2 x 2 output blocks per thread: four independent fp64 chains, each
    // summed over the columns in order
    const int nba = (p + 1) / 2, nbb = (nup + 1) / 2;
    double* dst = A.npart + ((size_t)blockIdx.x * 2 + cand) * no;
    for (int blk = tid; blk < nba * nbb; blk += nthr) {
      const int a0 = 2 * (blk / nbb), b0 = 2 * (blk % nbb);
      const int a1 = imin(a0 + 1, p - 1), b1 = imin(b0 + 1, nup - 1);
      const T* f0 = Fs + (size_t)a0 * cpb;
      const T* f1 = Fs + (size_t)a1 * cpb;
      const T* q0 = Ps + (size_t)b0 * cpb;
      const T* q1 = Ps + (size_t)b1 * cpb;
      double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
      for (int jl = 0; jl < ncols; ++jl) {
        const double x0 = (double)f0[jl], x1 = (double)f1[jl], y0 = (double)q0[jl], y1 = (double)q1[jl];
        c00 = fma(x0, y0, c00);
        c01 = fma(x0, y1, c01);
        c10 = fma(x1, y0, c10);
        c11 = fma(x1, y1, c11);
      }
      dst[a0 * nup + b0] = c00;
      if (b0 + 1 < nup) dst[a0 * nup + b0 + 1] = c01;
      if (a0 + 1 < p) {
        dst[(a0 + 1) * nup + b0] = c10;
        if (b0 + 1 < nup) dst[(a0 + 1) * nup + b0 + 1] = c11;
      }
    }
  };

  if (!resolver) {
    auto wval = [&](int i, int l) -> T {
      return (i < p && l < p) ? (fused ? W_s[i * 32 + l] : W[i * p + l]) : T(0);
    };
    // W^T fragments (B operand), resident for the whole solve; b[kt][nt]:
    // bhi = TF32 hi (m16n8k8), blo = the residual W - W_hi (TF32 correction MMAs)
    uint32_t bhi[NT][NT][2], blo[NT][NT][2];
    double bd[2 * NT][NT];
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int kt = 0; kt < NT; ++kt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float w = (float)wval(8 * nt + gq, 8 * kt + 2 * tq + h);
            bhi[kt][nt][h] = tf32_hi(w);
            blo[kt][nt][h] = tf32_lo(w, bhi[kt][nt][h]);
          }
          if (NN_FP32_BF16_CORR) {
            const float wh0 = __uint_as_float(bhi[kt][nt][0]), wh1 = __uint_as_float(bhi[kt][nt][1]);
            const float w0 = (float)wval(8 * nt + gq, 8 * kt + 2 * tq), w1 = (float)wval(8 * nt + gq, 8 * kt + 2 * tq + 1);
            blo[kt][nt][0] = pack_bf16(wh0, wh1);            // K 2tq, 2tq+1   <-> F_lo rows
            blo[kt][nt][1] = pack_bf16(w0 - wh0, w1 - wh1);  // K 2tq+8, 2tq+9 <-> F_hi rows
          }
        }
    } else {
#pragma unroll
      for (int kk = 0; kk < 2 * NT; ++kk)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) bd[kk][nt] = (double)wval(slot_row(nt, gq), slot_row(kk >> 1, 2 * tq + (kk & 1)));
    }
    // State per element (accumulator layout), with u = F - g / L:
    //   F_k = max(0, Y - grad_Y / L) = max(0, u_{k-1} + w_k (u_{k-1} - u_{k-2}))
    // (Y and grad_Y of nnls.py:189-191,208-213 folded into one affine update)
    T ua[NE], ub[NE], fa[NE], fb[NE];
    // g = W f - V in the accumulator layout (the MMA chain starts from -V)
    auto grad = [&](const T (&fe)[NE], T (&g)[NE]) {
      if constexpr (sizeof(T) == 4) {
        // accumulator element (col, row): c0 (gq, 2tq), c1 (gq, 2tq+1), c2 (gq+8, 2tq), c3 (gq+8, 2tq+1)
        uint32_t ahi[NT][4], alo[NT][4];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const float c0 = (float)fe[4 * t + 0], c1 = (float)fe[4 * t + 1], c2 = (float)fe[4 * t + 2],
                      c3 = (float)fe[4 * t + 3];
          const uint32_t h0 = tf32_hi(c0), h1 = tf32_hi(c1), h2 = tf32_hi(c2), h3 = tf32_hi(c3);
          ahi[t][0] = h0;  // (gq,   K slot tq   -> row 2tq)
          ahi[t][1] = h2;  // (gq+8, K slot tq)
          ahi[t][2] = h1;  // (gq,   K slot tq+4 -> row 2tq+1)
          ahi[t][3] = h3;
          if (NN_FP32_BF16_CORR) {
            const float f0 = __uint_as_float(h0), f1 = __uint_as_float(h1), f2 = __uint_as_float(h2),
                        f3 = __uint_as_float(h3);
            alo[t][0] = pack_bf16(c0 - f0, c1 - f1);  // (gq,   K 2tq, 2tq+1): F_lo
            alo[t][1] = pack_bf16(c2 - f2, c3 - f3);  // (gq+8, K 2tq, 2tq+1)
            alo[t][2] = pack_bf16(f0, f1);            // (gq,   K 2tq+8, 2tq+9): F_hi
            alo[t][3] = pack_bf16(f2, f3);
          } else {
            alo[t][0] = tf32_lo(c0, h0);
            alo[t][1] = tf32_lo(c2, h2);
            alo[t][2] = tf32_lo(c1, h1);
            alo[t][3] = tf32_lo(c3, h3);
          }
        }
        // n-tiles innermost: consecutive MMAs are independent, so the NT
        // accumulation chains overlap in the tensor pipe
        // The tensor core's fp32 accumulation truncates.  A chain started from
        // -V (the large, nearly cancelling term) or summing the hi*hi products
        // of all k-tiles carried that bias into g every iteration, and over
        // 500 accelerated iterations the factors drifted up to ~1.4e-3 from
        // the fp64 reference (NumPy float32: ~2e-5 on the same solve).  So
        // every k-tile's hi*hi product starts from zero and is added with a
        // round-to-nearest fp32 add, the corrections (2^-11 smaller) have
        // their own accumulator, and -V comes last, also rounded to nearest:
        // the same solve is then 1.6e-5 from fp64, like NumPy float32
        // (tools/diag_fp32_iters.py).
        float cc[NT][4], cl[NT][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int r = 0; r < 4; ++r) cc[nt][r] = cl[nt][r] = 0.f;
#pragma unroll
        for (int kt = 0; kt < NT; ++kt)  // correction terms F_lo W_hi + F_hi W_lo
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            if (NN_FP32_BF16_CORR) {
              mma_bf16(cl[nt], alo[kt], blo[kt][nt][0], blo[kt][nt][1]);
            } else {
              mma_tf32(cl[nt], alo[kt], bhi[kt][nt][0], bhi[kt][nt][1]);
              mma_tf32(cl[nt], ahi[kt], blo[kt][nt][0], blo[kt][nt][1]);
            }
          }
#pragma unroll
        for (int kt = 0; kt < NT; ++kt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            // each k-tile's hi*hi product from zero, added with round-to-nearest
            float tk[4] = {0.f, 0.f, 0.f, 0.f};
            mma_tf32(tk, ahi[kt], bhi[kt][nt][0], bhi[kt][nt][1]);
#pragma unroll
            for (int r = 0; r < 4; ++r) cc[nt][r] = __fadd_rn(cc[nt][r], tk[r]);
          }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int r = 0; r < 4; ++r)
            g[4 * nt + r] = (T)__fadd_rn(__fadd_rn(cc[nt][r], cl[nt][r]), (float)nv[4 * nt + r]);
      } else if constexpr (S::EPT == 4) {
        // two m-tiles per warp (column halves hh: gq, gq + 8): element e = 4 nt + 2 hh + h is
        // (row slot 2tq + h of tile nt, column half hh); k-step kk of half hh reads e = 4 (kk >> 1) + 2 hh + (kk & 1)
        double cc[2][NT][2];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            cc[hh][nt][0] = (double)nv[4 * nt + 2 * hh];
            cc[hh][nt][1] = (double)nv[4 * nt + 2 * hh + 1];
          }
#pragma unroll
        for (int kk = 0; kk < 2 * NT; ++kk) {
          if (kk == 2 * NT - 1 && kperm) continue;  // the padding k-step (warp-uniform)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
              mma_f64(cc[hh][nt], (double)fe[4 * (kk >> 1) + 2 * hh + (kk & 1)], bd[kk][nt]);
        }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            g[4 * nt + 2 * hh] = (T)cc[hh][nt][0];
            g[4 * nt + 2 * hh + 1] = (T)cc[hh][nt][1];
          }
      } else {
        double cc[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          cc[nt][0] = (double)nv[2 * nt];
          cc[nt][1] = (double)nv[2 * nt + 1];
        }
#pragma unroll
        for (int kk = 0; kk < 2 * NT; ++kk) {
          if (kk == 2 * NT - 1 && kperm) continue;  // the padding k-step (warp-uniform)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) mma_f64(cc[nt], (double)fe[kk], bd[kk][nt]);
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          g[2 * nt] = (T)cc[nt][0];
          g[2 * nt + 1] = (T)cc[nt][1];
        }
      }
    };

    // per-iteration sums: ||PG||^2 and <F, g - V> (= 2 * partial objective)
    // (FP32: ||PG||^2 in fp32 up to the warp level; the objective sum is carried
    // in double from the element products on -- successive iterates' objectives
    // differ by ~1e-9 relative on ill-conditioned problems and the reference's
    // best-iterate rule, nnls.py:196-203, needs their order)
    auto post = [&](int j, T s0, double s1) {
      double a0, a1;
      if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        a0 = s0;
        a1 = warp_sum(s1);
      } else {
        a0 = warp_sum((double)s0);
        a1 = warp_sum((double)s1);
      }
      if (lane == 0) {
        double* q = pp + ((size_t)((j + NW_PPD) % NW_PPD) * NW_MAXW + wid) * 3;
        q[0] = a0;
        q[1] = a1;
        q[2] = 0.0;
      }
    };
    // the sums of TWO iterations (ja: a0, a1; jb: b0, b1) in one transposed
    // butterfly: 6 shuffles and a 5-level chain for 4 values instead of 20
    // and two 5-level chains; lanes 0 / 8 / 16 / 24 end with a0 / a1 / b0 / b1
    auto post2 = [&](int ja, T a0f, double a1, int jb, T b0f, double b1) {
      const double a0 = (double)a0f, b0 = (double)b0f;
      const bool lo = lane < 16;
      double k0 = lo ? a0 : b0, k1 = lo ? a1 : b1;
      const double x0 = lo ? b0 : a0, x1 = lo ? b1 : a1;
      k0 += __shfl_xor_sync(0xffffffffu, x0, 16);
      k1 += __shfl_xor_sync(0xffffffffu, x1, 16);
      const bool hi8 = (lane & 8) != 0;
      double v = hi8 ? k1 : k0;
      v += __shfl_xor_sync(0xffffffffu, hi8 ? k0 : k1, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if ((lane & 7) == 0) {
        const int j = lo ? ja : jb;
        double* q = pp + ((size_t)((j + NW_PPD) % NW_PPD) * NW_MAXW + wid) * 3;
        q[hi8 ? 1 : 0] = v;
        if (!hi8) q[2] = 0.0;
      }
    };
    auto post_flag = [&](int j) {
      if (lane == 0) {
        __threadfence_block();
        sh.posted[wid] = j;
      }
    };
    // F -> g -> (u, sums); u overwrites uo
    auto finish = [&](const T (&fe)[NE], const T (&g)[NE], T (&uo)[NE], T& s0, double& s1) {
      if constexpr (sizeof(T) == 4) {
        // packed fp32x2 arithmetic (FFMA2/FADD2 on sm_100): elements 2i, 2i+1
        // are two solver rows of one column; the objective products are added in double
        float2 a0 = make_float2(0.f, 0.f);
        double a1 = 0.0;
        const float2 rl = make_float2(rnegL, rnegL);
#pragma unroll
        for (int e = 0; e < NE; e += 4) {
          // four objective products summed in fp32 (their own rounding class), then added in double
          float2 pr = make_float2(0.f, 0.f);
#pragma unroll
          for (int h = 0; h < 4; h += 2) {
            const int i = e + h;
            const float2 f2 = make_float2(fe[i], fe[i + 1]), g2 = make_float2(g[i], g[i + 1]);
            const float2 u2 = __ffma2_rn(g2, rl, f2);
            uo[i] = u2.x;
            uo[i + 1] = u2.y;
            const float2 pg2 =
                make_float2(fe[i] > 0.f ? g[i] : min0_nan(g[i]), fe[i + 1] > 0.f ? g[i + 1] : min0_nan(g[i + 1]));
            a0 = __ffma2_rn(pg2, pg2, a0);
            pr = __ffma2_rn(f2, __fadd2_rn(g2, make_float2(nv[i], nv[i + 1])), pr);
          }
          a1 += (double)(pr.x + pr.y);
        }
        s0 = a0.x + a0.y;
        s1 = a1;
      } else {
        s0 = T(0);
        s1 = 0.0;
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          uo[e] = fma_acc(g[e], rnegL, fe[e]);
          const T pgv = pg_entry_fast(fe[e], g[e]);
          s0 = fma_acc(pgv, pgv, s0);
          s1 = fma_acc((double)fe[e], (double)(g[e] + nv[e]), s1);
        }
      }
    };
    // F_k from (u_{k-1}, u_{k-2}) into fo
    auto extrapolate = [&](const T (&u1)[NE], const T (&u2)[NE], T w, T (&fo)[NE]) {
      if constexpr (sizeof(T) == 4) {
        const float2 w2 = make_float2(w, w), m1 = make_float2(-1.f, -1.f);
#pragma unroll
        for (int e = 0; e < NE; e += 2) {
          const float2 a = make_float2(u1[e], u1[e + 1]), b = make_float2(u2[e], u2[e + 1]);
          const float2 y = __ffma2_rn(__ffma2_rn(b, m1, a), w2, a);  // u1 + w (u1 - u2)
          fo[e] = relu_nan_fast(y.x);
          fo[e + 1] = relu_nan_fast(y.y);
        }
      } else {
#pragma unroll
        for (int e = 0; e < NE; ++e) fo[e] = relu_nan_fast(fma_acc(u1[e] - u2[e], w, u1[e]));
      }
    };

    // start point (nnls.py:163-178); columns/rows outside the problem stay 0
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const bool ok = evalid(e);
      fa[e] = ok ? F0[eoff(e)] : T(0);
      fb[e] = fa[e];
      if (!fused) nv[e] = ok ? -A.V[eoff(e)] : T(0);
    }
    T ps0;  // sums of the last iteration, posted during the next one
    double ps1;
    {
      T g[NE];
      grad(fa, g);
      finish(fa, g, ua, ps0, ps1);
#pragma unroll
      for (int e = 0; e < NE; ++e) ub[e] = ua[e];
      post(-1, ps0, ps1);
      post_flag(-1);
    }

    // w_k of iteration k is wtab[k - 1] (0 for k = 0): lane l of wwin holds
    // wtab[32 w - 1 + l] for the current window w, wnext the next window's
    auto wload = [&](int base) -> double {
      const int i = base - 1 + lane;
      return (i >= 0 && i < max_iter) ? wtab[i] : 0.0;
    };
    if (tracebuf != nullptr && lane == 0 && wid == 0 && blockIdx.x < 512)
      tracebuf[3 * NN_TRACE_LEN + blockIdx.x] = gtimer_ns();  // per-CTA loop start
    if (tracebuf != nullptr && lane == 0 && wid == 0 && blockIdx.x == 0) {
      tracebuf[NN_TRACE_LEN + 52] = clock64();
      tracebuf[NN_TRACE_LEN + 53] = gtimer_ns();
    }
    T wwin = T(0), wnext = (T)wload(0);
    int k = 0;
    bool go = true;
    const bool has_cols = cblk < ncols;
    // one iteration k: F_k into fo, u_k into u2 (which held u_{k-2});
    // the sums of iteration k-1 are reduced and posted while the MMAs run
    // iterations run in pairs (A: even k, B: odd k); B posts the sums of the
    // previous B (k - 2, in ps) and of A (k - 1, in pa) while its MMAs run
    T pa0 = T(0);
    double pa1 = 0.0;
    // momentum weights of the current pair (wA: k, wB: k + 1), fetched one
    // pair ahead so the shuffles are off the iteration's critical path
    T wA = T(0), wB = T(0);
    auto half = [&](T (&u1)[NE], T (&u2)[NE], T (&fo)[NE], bool b_half) {
      extrapolate(u1, u2, b_half ? wB : wA, fo);
      T g[NE];
      grad(fo, g);
      if (b_half) {
        // no branch around the butterfly: its shuffles schedule between the MMAs
        post2(k - 2, ps0, ps1, k - 1, pa0, pa1);
        finish(fo, g, u2, ps0, ps1);
      } else {
        finish(fo, g, u2, pa0, pa1);
      }
      ++k;
    };
    while (true) {
      if (k + 2 > max_iter) break;  // odd tail handled below
      if (k % NW_WIN == 0) {
        const int w = k / NW_WIN;
        wwin = wnext;
        wnext = (T)wload(k + NW_WIN);
        if (k == 0) {
          wA = __shfl_sync(0xffffffffu, wwin, 0);
          wB = __shfl_sync(0xffffffffu, wwin, 1);
        }
        const bool tr = tracebuf != nullptr && lane == 0 && wid == 0 && blockIdx.x == 0 && w < 200;
        if (tr) tracebuf[NN_TRACE_LEN + 100 + 4 * w] = gtimer_ns();
        int ok = 1;
        if (lane == 0) {
          const int need = (w - NW_FLIGHT) * NW_WIN - 1;
          while (!(dbg & 1) && sh.resolved < need && !sh.halt) __nanosleep(64);
          ok = sh.halt ? 0 : 1;
        }
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (!ok) break;
        if (tr) tracebuf[NN_TRACE_LEN + 100 + 4 * w + 1] = gtimer_ns();
        const int slot = w % NW_SNAP;
        const int evicted = w - NW_SNAP;
        const int bj = sh.best_j;
        const bool save = evicted >= 0 && bj >= 0 && bj / NW_WIN == evicted;
        if (has_cols && !(dbg & 2)) {
          T* sp = snaps + (int64_t)(slot * 4) * pc;
          if (save) {
            T* bp = snaps + (int64_t)(NW_SNAP * 4) * pc;
#pragma unroll
            for (int e = 0; e < NE; ++e)
              if (evalid(e))
                for (int b = 0; b < 2; ++b) bp[b * pc + eoff(e)] = sp[b * pc + eoff(e)];
          }
#pragma unroll
          for (int e = 0; e < NE; ++e)
            if (evalid(e)) {
              const int64_t o = eoff(e);
              sp[o] = ua[e];
              sp[pc + o] = ub[e];
            }
        }
        if (lane == 0 && save) sh.bsw[wid] = evicted;
        __syncwarp();
        if (tr) tracebuf[NN_TRACE_LEN + 100 + 4 * w + 2] = gtimer_ns();
      }
      go = sh.halt == 0;  // one LDS per warp: every lane sees the same value
      // the next pair's weights (k + 2 starts the next window when k % 32 == 30)
      const T wsrc = (k + 2) % NW_WIN == 0 ? wnext : wwin;
      const T wA_n = __shfl_sync(0xffffffffu, wsrc, (k + 2) % NW_WIN);
      const T wB_n = __shfl_sync(0xffffffffu, wsrc, (k + 3) % NW_WIN);
      // k is even here (windows have even length): u_{k-1} in ua, F_{k-1} in fa;
      // the pair leaves the roles canonical again, so the loop has no moves
      half(ua, ub, fb, false);
      half(ub, ua, fa, true);
      wA = wA_n;
      wB = wB_n;
      if (k > 2 && (k - 2) % NW_WIN == 0) post_flag(k - 2);  // covers the last iteration of the previous window
      if (k == max_iter || !go) break;
    }
    bool tail = false;
    if (go && k == max_iter - 1) {
      // odd max_iter: the last iteration alone, then the canonical roles back
      // (a snapshot is not needed: a best iterate in this window is F_k itself)
      if (k % NW_WIN == 0) {
        wwin = wnext;
        wA = __shfl_sync(0xffffffffu, wwin, 0);
        if (lane == 0) {
          const int need = (k / NW_WIN - NW_FLIGHT) * NW_WIN - 1;
          while (!(dbg & 1) && sh.resolved < need && !sh.halt) __nanosleep(64);
        }
        __syncwarp();
      }
      half(ua, ub, fb, false);
      tail = true;
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        T t = ua[e];
        ua[e] = ub[e];
        ub[e] = t;
        t = fa[e];
        fa[e] = fb[e];
        fb[e] = t;
      }
    }
    if (tracebuf != nullptr && lane == 0 && blockIdx.x < 512 && wid < 5)
      tracebuf[3 * NN_TRACE_LEN + 512 * (1 + wid) + blockIdx.x] = gtimer_ns();  // per-CTA, per-warp loop end
    if (tracebuf != nullptr && lane == 0 && wid == 0 && blockIdx.x == 0) {
      tracebuf[NN_TRACE_LEN + 50] = clock64();
      tracebuf[NN_TRACE_LEN + 51] = gtimer_ns();
      tracebuf[NN_TRACE_LEN + 54] = k;
    }
    // the last (one or two) iterations' sums and the final window flag
    if (tail) {
      post(k - 2, ps0, ps1);  // the last B (when k - 2 = -1: the start point again, same values)
      post(k - 1, pa0, pa1);  // the odd tail iteration
      post_flag(k - 1);
    } else if (k > 0) {
      post(k - 1, ps0, ps1);
      post_flag(k - 1);
    }
    if (lane == 0) sh.kdone[wid] = k;
    __syncwarp();
    // speculative tie-break work while the resolver decides (nnls.py:219-227):
    // the output, residual and next-product partials of the final iterate
    // (the start point's residual was formed in the prologue)
    if (fused) {
      auto tr = [&](int i) {
        if (tracebuf != nullptr && blockIdx.x == 0 && tid == 0) tracebuf[NN_TRACE_LEN + 90 + i] = gtimer_ns();
      };
      tr(0);
      if (has_cols) {
#pragma unroll
        for (int e = 0; e < NE; ++e)
          if (evalid(e)) Fout[eoff(e)] = fa[e];
      }
      resid_one(fa, 0);
      tr(1);
      if (lane == 0)
        while (!sh.prep_done) __nanosleep(32);
      __syncwarp();
      __threadfence_block();
      if (A.Pt != nullptr) {
        auto csync = [&]() { asm volatile("bar.sync 2, %0;" ::"r"(ncw * 32) : "memory"); };
        next_partials(0, ncw * 32, csync);
      }
      tr(2);
    }

    // -------------------------------------------------------------- output
    // (waits for the resolver's final decision through the block barrier below)
    asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
  if (tracebuf != nullptr && blockIdx.x == 0 && tid == 0) tracebuf[NN_TRACE_LEN + 60 + 6] = gtimer_ns();
    const int bj = sh.best_j;
    const bool ok_best = bj >= 0 && sh.fail_at == -1;
    if (tracebuf != nullptr && blockIdx.x < 512 && lane == 0 && wid < 5) {
      tracebuf[512 * (3 + wid) + blockIdx.x] = gtimer_ns();  // per-warp time past the output barrier
      tracebuf[2 * NN_TRACE_LEN + 512 * (1 + wid) + blockIdx.x] = (unsigned long long)(bj + 1);
    }
    if (tracebuf != nullptr && blockIdx.x == 0 && tid == 0) tracebuf[NN_TRACE_LEN + 60 + 12] = gtimer_ns();
    const bool spec_ok = spec_hit(bj);
    if (ok_best && has_cols && !spec_ok) {
      const int kd = sh.kdone[wid];
      if (tracebuf != nullptr && blockIdx.x == 0 && tid == 0) tracebuf[NN_TRACE_LEN + 60 + 13] = gtimer_ns();
      if (bj == kd - 2) {
#pragma unroll
        for (int e = 0; e < NE; ++e) fa[e] = fb[e];
      } else if (bj != kd - 1) {
        // recompute from the snapshot at the start of the best iterate's window
        const int wb = bj / NW_WIN;
        const int slot = (sh.bsw[wid] == wb && wb + NW_SNAP <= (kd - 1) / NW_WIN) ? NW_SNAP : wb % NW_SNAP;
        const T* sp = snaps + (int64_t)(slot * 4) * pc;
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          const bool ok = evalid(e);
          ua[e] = ok ? sp[eoff(e)] : T(0);
          ub[e] = ok ? sp[pc + eoff(e)] : T(0);
        }
        const T wrec = wload(wb * NW_WIN);  // w of iterations wb*32 .. wb*32+31
        for (int kk = wb * NW_WIN; kk <= bj; ++kk) {
          const T w = __shfl_sync(0xffffffffu, wrec, kk % NW_WIN);
          extrapolate(ua, ub, w, fa);
          T g[NE], d0;
          double d1;
          grad(fa, g);
          finish(fa, g, ub, d0, d1);
#pragma unroll
          for (int e = 0; e < NE; ++e) {
            const T t = ua[e];
            ua[e] = ub[e];
            ub[e] = t;
          }
        }
      }
      if (tracebuf != nullptr && blockIdx.x == 0 && tid == 0) {
        tracebuf[NN_TRACE_LEN + 60 + 4] = gtimer_ns();
        tracebuf[NN_TRACE_LEN + 80] = bj;
        tracebuf[NN_TRACE_LEN + 81] = kd;
      }
      // fa = the best iterate
#pragma unroll
      for (int e = 0; e < NE; ++e)
        if (evalid(e)) Fout[eoff(e)] = fa[e];
    }
    if (fused && ok_best && !spec_ok) resid_one(fa, 0);
  } else {
    if (fused) {
      // while the first windows run: the start point's tie-break residual and
      // Pt staged for the next product (the compute warps wait for prep_done
      // before their end-of-solve use)
      resid_start_all(ncw);
      if (A.Pt != nullptr) stage_pt(lane, 32);
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        sh.prep_done = 1;
      }
      __syncwarp();
    }
    if (!(dbg & 1))
      resolver_warp(sh, pp, ncw, max_iter, A.grad_tol, L, A.recs, A.results, tracebuf, NW_MAXW, &A.grp,
                    A.watchdog_ns);
    if (tracebuf != nullptr && blockIdx.x == 0 && lane == 0) tracebuf[NN_TRACE_LEN + 60 + 14] = gtimer_ns();
    asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
  }
  __syncthreads();
  const int bj = sh.best_j;
  const bool ok_best = bj >= 0 && sh.fail_at == -1;
  if (tracebuf != nullptr && blockIdx.x < 512 && tid == 0) tracebuf[2 * NN_TRACE_LEN + 3072 + blockIdx.x] = (unsigned long long)(bj + 1);
  int start_wins = 0;
  if (tracebuf != nullptr && blockIdx.x == 0 && tid == 0) tracebuf[NN_TRACE_LEN + 60 + 8] = gtimer_ns();
  if (fused && sh.fail_at == -1) {
    // tie-break (nnls.py:219-227) and the next product Pout = F_out Pt^T
    // (factorize.py:110,113) behind one grid barrier: each CTA posts its
    // residual partials of best and start and, for the next product, its
    // partials of the best iterate; after the barrier every CTA reaches the
    // same decision (fixed-order sums) and reduces the chosen candidate's
    // slice (a start-point win adds its partials and a second barrier)
    const bool next = A.Pt != nullptr;
    const int nup = next ? (int)A.nup : 0, no = p * nup;
    if (next && ok_best && !spec_hit(bj)) {
      // the speculation missed: the best iterate's partials
      auto bsync = [&]() { __syncthreads(); };
      next_partials(0, (int)blockDim.x, bsync);
    }
    start_wins = 1;
    if (ok_best || next) {
      __syncthreads();
      if (tid == 0) {
        if (ok_best) {
          double a0 = 0.0, a1 = 0.0;
          for (int w = 0; w < ncw; ++w) {
            a0 += s_red[w][0];
            a1 += s_red[w][1];
          }
          A.rpart[2 * blockIdx.x] = a0;
          A.rpart[2 * blockIdx.x + 1] = a1;
        }
        __threadfence();
        atomicAdd(A.bar + vr, 1u);
        while (ld_acquire_u32(A.bar + vr) < (unsigned)Gr) __nanosleep(32);
      }
      __syncthreads();
    }
    // the best candidate's slice of the next product, reduced by warps 1..
    // while warp 0 reduces the tie-break residuals (same order as below)
    __shared__ double s_pout[32];
    const int nwarps_all = (int)(blockDim.x >> 5);
    const int per_s = next ? (no + Gr - 1) / Gr : 0;
    const int os0 = lb * per_s, os1 = min(no, os0 + per_s);
    const bool pre = next && ok_best && per_s <= 32 && nwarps_all > 1;
    if (pre && wid >= 1) {
      for (int o = os0 + wid - 1; o < os1; o += nwarps_all - 1) {
        double sacc = 0.0;
        for (int g = g_lo + lane; g < g_hi; g += 32) sacc += __ldcg(&A.npart[((size_t)g * 2) * no + o]);
        sacc = warp_sum(sacc);
        if (lane == 0) s_pout[o - os0] = sacc;
      }
    }
    if (ok_best) {
      if (wid == 0) {
        // CTA partials summed lane-strided then by a fixed butterfly: the same
        // order (and value) in every CTA
        double b0 = 0.0, b1 = 0.0;
        for (int g = g_lo + lane; g < g_hi; g += 32) {
          b0 += __ldcg(&A.rpart[2 * g]);
          b1 += __ldcg(&A.rpart[2 * g + 1]);
        }
        b0 = warp_sum(b0);
        b1 = warp_sum(b1);
        if (grouped) {
          // this rank's residual sums to every rank (the rank's first CTA),
          // then every CTA sums all ranks' in rank order
          const int myrank = A.grp.rank0 + vr;
          if (lb == 0 && lane < A.grp.ranks) {
            XTie* xt = &A.grp.xch[lane]->tie[myrank];
            xt->b0 = b0;
            xt->b1 = b1;
            fence_sys();
            st_relaxed_sys_u64(&xt->tag, A.grp.epoch);
          }
          const XTie* xt = A.grp.xch[myrank]->tie;
          const unsigned long long t0 = gtimer_ns();
          for (;;) {
            const bool mine = lane >= A.grp.ranks || ld_relaxed_sys_u64(&xt[lane].tag) == A.grp.epoch;
            if (__all_sync(0xffffffffu, mine)) break;
            __nanosleep(64);
            if (gtimer_ns() - t0 > A.watchdog_ns) {
              if (lane == 0) status_fail(st, NENMF_ERR_WATCHDOG, -2);
              break;
            }
          }
          fence_sys();
          b0 = __ldcv(&xt[0].b0);
          b1 = __ldcv(&xt[0].b1);
          for (int src = 1; src < A.grp.ranks; ++src) {
            b0 += __ldcv(&xt[src].b0);
            b1 += __ldcv(&xt[src].b1);
          }
        }
        if (lane == 0) {
          const double nb = sqrt(b0), ns = sqrt(b1);
          const double tb = 0.5 * (nb * nb), ts = 0.5 * (ns * ns);
          s_start_wins = (tb <= ts) ? 0 : 1;
          if (blockIdx.x == 0) {
            st->resid[0] = tb;
            st->resid[1] = ts;
            A.L[1] = b0;
            A.L[2] = b1;
          }
        }
      }
      __syncthreads();
      start_wins = s_start_wins;
    }
    if (next && start_wins) {
      // the start point won (rare; always without a best iterate): its
      // partials of the next product, then a second grid barrier
      auto bsync = [&]() { __syncthreads(); };
      next_partials(1, (int)blockDim.x, bsync);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(A.bar + vr, 1u);
        while (ld_acquire_u32(A.bar + vr) < 2u * (unsigned)Gr) __nanosleep(32);
      }
      __syncthreads();
    }
    if (start_wins && !resolver && cblk < ncols) {
#pragma unroll
      for (int e = 0; e < NE; ++e)
        if (evalid(e)) Fout[eoff(e)] = F0[eoff(e)];
    }
    // the next product: this (virtual) rank's partial sum over its columns
    // (a group's ranks add theirs with one all-reduce of p x nup afterwards)
    T* Pout_r = next ? A.Pout + (size_t)vr * no : nullptr;
    if (next && pre && !start_wins) {
      for (int i = tid; i < os1 - os0; i += (int)blockDim.x) Pout_r[os0 + i] = (T)s_pout[i];
    } else if (next) {
      const int cand = (ok_best && !start_wins) ? 0 : 1;
      const int per = (no + Gr - 1) / Gr;
      const int o0 = lb * per, o1 = min(no, o0 + per);
      const int nwarps = blockDim.x >> 5;
      for (int o = o0 + wid; o < o1; o += nwarps) {
        double sacc = 0.0;
        for (int g = g_lo + lane; g < g_hi; g += 32) sacc += __ldcg(&A.npart[((size_t)g * 2 + cand) * no + o]);
        sacc = warp_sum(sacc);
        if (lane == 0) Pout_r[o] = (T)sacc;
      }
    }
  }
  if (tracebuf != nullptr && blockIdx.x == 0 && tid == 0) tracebuf[NN_TRACE_LEN + 60 + 10] = gtimer_ns();
  if (blockIdx.x == 0 && tid == 0) {
    if (sh.fail_at >= 0) status_fail(st, NENMF_ERR_NUMERICAL_FAILURE, sh.fail_at);
    if (sh.fail_at == -2) status_fail(st, NENMF_ERR_WATCHDOG, -2);
    st->inner_iters = sh.stop_at >= 0 ? sh.stop_at + 1 : (sh.fail_at >= 0 ? sh.fail_at : max_iter);
    st->returned_best = (bj >= 0 && !start_wins) ? 1 : 0;
    st->best_partial = sh.best_part;
    st->pg_ref = sh.pg_ref;
  }
}

template <typename T, int NT>
static int launch_nnls_mma_t(const MmaArgs<T>& a, int grid, cudaStream_t s) {
  const int ncw = (int)cdiv(a.cpb, MmaShape<T>::CB);
  const int threads = 32 * (ncw + 1);
  if (threads > mma_threads<T>(NT) || ncw >= NW_MAXW) return NENMF_ERR_UNSUPPORTED;
  size_t smem = (size_t)NW_PPD * NW_MAXW * 3 * sizeof(double);
  if (a.fused) smem += fused_smem_bytes(sizeof(T), a.p, a.r, ncw, MmaShape<T>::CB, a.cpb);
  if (a.fused && a.Pt != nullptr) smem += (size_t)(a.p + a.nup) * a.cpb * sizeof(T);
  if (smem > 227 * 1024) return NENMF_ERR_UNSUPPORTED;
  auto fn = k_nnls_mma<T, NT>;
  NENMF_CUDA_TRY(set_smem(fn, smem));
  void* args[] = {(void*)&a};
  NENMF_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(threads), args, smem, s));
  launch_counter_add(1);
  return NENMF_OK;
}

#define NENMF_NNLS_MMA_IMPL(T)                                                                          \
  template <>                                                                                         \
  int nnls_mma_col_block<T>() {                                                                       \
    return MmaShape<T>::CB;                                                                           \
  }                                                                                                   \
  template <>                                                                                         \
  int nnls_mma_max_cols<T>(int p) {                                                                   \
    const int nt = (int)cdiv(p, 8);                                                                   \
    return MmaShape<T>::CB * imin(NW_MAXW - 1, mma_threads<T>(nt) / 32 - 1);                          \
  }                                                                                                   \
  template <>                                                                                         \
  int launch_nnls_mma<T>(const MmaArgs<T>& a, int grid, cudaStream_t s) {                             \
    switch ((int)cdiv(a.p, 8)) {                                                                      \
      case 1: return launch_nnls_mma_t<T, 1>(a, grid, s);                                             \
      case 2: return launch_nnls_mma_t<T, 2>(a, grid, s);                                             \
      case 3: return launch_nnls_mma_t<T, 3>(a, grid, s);                                             \
      case 4: return launch_nnls_mma_t<T, 4>(a, grid, s);                                             \
      default: return NENMF_ERR_UNSUPPORTED;                                                          \
    }                                                                                                 \
  }

}  // namespace nenmf
