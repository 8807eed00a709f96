// Streamed tensor-core inner solver for problems with more columns than the
// register-resident solver holds (BASELINE cfg4's G-half: 400 000 columns,
// cfg5's: 100 000; nnls.py:160-227).
//
// Same arithmetic per 16-column tile as k_nnls_mma (3xTF32: hi x hi plus the
// two TF32 correction MMAs per k-tile, accumulators reused as the next A
// operand) and
// the same windowed decision protocol (resolver warp, window records, fixed
// order sums), but the iterate state lives in HBM: per iteration every warp
// sweeps its tiles, reading u_{k-1}, u_{k-2} and V and writing u_k (16 bytes
// per element and iteration, the streaming floor).  Window snapshots are the
// values already loaded at a window start; the returned best iterate is
// recomputed from its window's snapshot at the end (<= 32 on-chip steps per
// tile).  FP32, p <= 64.
#pragma once
#include "nnls_mma.cuh"

// objective products summed in fp32 in groups of NN_S1_GROUP (a power of two), then in double
#ifndef NN_S1_GROUP
#define NN_S1_GROUP 4
#endif

namespace nenmf {

// 8 (NT <= 3) or 4 compute warps + the resolver.  When the CTA's columns fit
// (BASELINE cfg5) u_{k-1}, u_{k-2} and V stay in shared memory for the whole
// solve; otherwise each compute warp streams its tiles from HBM through a
// shared-memory ring (stage: u_{k-1}, u_{k-2}, V tiles of 8 NT x 16);
// NT <= 4 (p <= 32): 3 stages, W^T fragments in registers; NT 5..8
// (p <= 64, BASELINE cfg3's p = 50): 2 stages, W^T fragments in shared memory.
constexpr int SS_ROW = 20;  // ring / resident tile row stride (floats): conflict-free accumulator reads
template <int NT>
struct SS {
  static constexpr bool WSM = NT > 4;
  // compute warps: 8 (two per SMSP, interleaving their per-tile latency
  // chains) while the rings fit, 4 otherwise; the sum ring has one row per warp
  static constexpr int NCW = NT <= 3 ? 8 : 4;
  static constexpr int PPW = NCW;
  static constexpr int STAGES = WSM ? 2 : 3;
  static constexpr int ARR_F = 8 * NT * SS_ROW;
  static constexpr int STAGE_F = 3 * ARR_F;
  // dynamic shared memory: sum ring, then the per-warp cp.async rings or (resident)
  // [ntiles][3][ARR_F] tiles of U slot 0, U slot 1, V; then the W^T fragments (WSM)
  __host__ __device__ static constexpr size_t state_bytes(bool resident, int ntiles) {
    return resident ? (size_t)ntiles * STAGE_F * sizeof(float) : (size_t)NCW * STAGES * STAGE_F * sizeof(float);
  }
  __host__ __device__ static constexpr size_t smem(bool resident = false, int ntiles = 0) {
    return (size_t)NW_PPD * PPW * 3 * sizeof(double) + state_bytes(resident, ntiles) +
           (WSM ? (size_t)NT * NT * 32 * 16 : 0);
  }
};
template <int NT>
__host__ __device__ constexpr int stream_threads() {
  return (SS<NT>::NCW + 1) * 32;
}

template <int NT>
__global__ void __launch_bounds__(stream_threads<NT>(), 1) k_nnls_stream(const __grid_constant__ StreamArgs A) {
  constexpr int NE = 4 * NT;
  constexpr int CB = 16;
  extern __shared__ __align__(16) double smem_d[];
  double* pp = smem_d;  // [PPD][MAXW][3]
  __shared__ SolverShared sh;
  const int p = A.p, max_iter = A.max_iter;
  const int64_t c = A.c, pc = (int64_t)A.p * A.c;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ncw = (blockDim.x >> 5) - 1;
  const bool resolver = wid == ncw;
  const int64_t j0 = (int64_t)blockIdx.x * A.cpb;
  const int ncols = (int)(imin(c, j0 + A.cpb) - j0);
  const int ntiles = ncols > 0 ? (ncols + CB - 1) / CB : 0;
  const int gq = lane >> 2, tq = lane & 3;
  solver_shared_init(sh);
  __syncthreads();
  if (A.st->code != 0) return;
  const double L = A.L[0];
  const float rnegL = (float)(-1.0 / L);

  if (!resolver) {
    // element e of this thread within a tile: solver row, tile-local column
    auto erow = [&](int e) { return 8 * (e >> 2) + 2 * tq + (e & 1); };
    auto ecol = [&](int e) { return gq + ((e & 2) ? 8 : 0); };
    // W^T fragments, as k_nnls_mma: in registers (NT <= 4) or shared memory
    constexpr bool WSM = SS<NT>::WSM;
    constexpr int NTR = WSM ? 1 : NT;  // register array extent
    uint32_t bhi[NTR][NTR][2], bco[NTR][NTR][2];
    const bool resident = A.resident != 0;
    const int ntiles_cta = (int)((A.cpb + CB - 1) / CB);
    uint4* wf = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(smem_d + (size_t)NW_PPD * SS<NT>::PPW * 3) +
                                         SS<NT>::state_bytes(resident, ntiles_cta));  // [NT][NT][32]
#pragma unroll
    for (int kt = 0; kt < NT; ++kt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        if (WSM && (kt * NT + nt) % ncw != wid) continue;  // fill the shared copy cooperatively
        uint32_t h2[2], l2[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = 8 * nt + gq, l = 8 * kt + 2 * tq + h;
          const float w = (i < p && l < p) ? A.W[i * p + l] : 0.f;
          h2[h] = tf32_hi(w);
          l2[h] = tf32_lo(w, h2[h]);
        }
        const uint32_t c0 = l2[0], c1 = l2[1];  // the W residual (3xTF32 corrections)
        if constexpr (WSM) {
          wf[(kt * NT + nt) * 32 + lane] = make_uint4(h2[0], h2[1], c0, c1);
        } else {
          bhi[kt % NTR][nt % NTR][0] = h2[0];
          bhi[kt % NTR][nt % NTR][1] = h2[1];
          bco[kt % NTR][nt % NTR][0] = c0;
          bco[kt % NTR][nt % NTR][1] = c1;
        }
      }
    if constexpr (WSM) asm volatile("bar.sync 2, %0;" ::"r"(ncw * 32) : "memory");
    auto grad = [&](const float (&fe)[NE], const float (&nv)[NE], float (&g)[NE]) {
      uint32_t ahi[NT][4], aco[NT][4];
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const float c0 = fe[4 * t], c1 = fe[4 * t + 1], c2 = fe[4 * t + 2], c3 = fe[4 * t + 3];
        const uint32_t h0 = tf32_hi(c0), h1 = tf32_hi(c1), h2 = tf32_hi(c2), h3 = tf32_hi(c3);
        ahi[t][0] = h0;
        ahi[t][1] = h2;
        ahi[t][2] = h1;
        ahi[t][3] = h3;
        aco[t][0] = tf32_lo(c0, h0);  // F residual, same slots as ahi
        aco[t][1] = tf32_lo(c2, h2);
        aco[t][2] = tf32_lo(c1, h1);
        aco[t][3] = tf32_lo(c3, h3);
      }
      // zero-started accumulators, -V added with round-to-nearest (see k_nnls_mma)
      float cc[NT][4], cl[NT][4];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int r = 0; r < 4; ++r) cc[nt][r] = cl[nt][r] = 0.f;
      if constexpr (WSM) {
#pragma unroll
        for (int kt = 0; kt < NT; ++kt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const uint4 b = wf[(kt * NT + nt) * 32 + lane];
            mma_tf32(cl[nt], aco[kt], b.x, b.y);  // F_lo W_hi
            mma_tf32(cl[nt], ahi[kt], b.z, b.w);  // F_hi W_lo
            float tk[4] = {0.f, 0.f, 0.f, 0.f};   // hi*hi per k-tile, added with round-to-nearest
            mma_tf32(tk, ahi[kt], b.x, b.y);
#pragma unroll
            for (int r = 0; r < 4; ++r) cc[nt][r] = __fadd_rn(cc[nt][r], tk[r]);
          }
      } else {
#pragma unroll
        for (int kt = 0; kt < NT; ++kt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            mma_tf32(cl[nt], aco[kt], bhi[kt % NTR][nt % NTR][0], bhi[kt % NTR][nt % NTR][1]);
            mma_tf32(cl[nt], ahi[kt], bco[kt % NTR][nt % NTR][0], bco[kt % NTR][nt % NTR][1]);
          }
#pragma unroll
        for (int kt = 0; kt < NT; ++kt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            float tk[4] = {0.f, 0.f, 0.f, 0.f};   // hi*hi per k-tile, added with round-to-nearest
            mma_tf32(tk, ahi[kt], bhi[kt % NTR][nt % NTR][0], bhi[kt % NTR][nt % NTR][1]);
#pragma unroll
            for (int r = 0; r < 4; ++r) cc[nt][r] = __fadd_rn(cc[nt][r], tk[r]);
          }
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int r = 0; r < 4; ++r) g[4 * nt + r] = __fadd_rn(__fadd_rn(cc[nt][r], cl[nt][r]), nv[4 * nt + r]);
    };
    // the objective sum s1 is carried in double from the element products on
    // (nnls_mma.cuh: the best-iterate rule needs the order of objectives that
    // differ by ~1e-9 relative)
    auto post = [&](int j, float s0, double s1) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 = warp_sum(s1);
      if (lane == 0) {
        double* q = pp + ((size_t)((j + NW_PPD) % NW_PPD) * SS<NT>::PPW + wid) * 3;
        q[0] = s0;
        q[1] = s1;
        q[2] = 0.0;
      }
    };
    auto post_flag = [&](int j) {
      if (lane == 0) {
        __threadfence_block();
        sh.posted[wid] = j;
      }
    };
    auto wload = [&](int base) -> double {
      const int i = base - 1 + lane;
      return (i >= 0 && i < max_iter) ? A.wtab[i] : 0.0;
    };
    // one tile of one iteration k (k = -1: the start point), in two halves so
    // that the next tile's loads are in flight while this one computes
    const float* __restrict__ V = A.V;
    const int64_t jend = j0 + ncols;
    auto eoff = [&](int64_t cb, int e) -> int64_t {
      return (int64_t)(8 * (e >> 2) + (e & 1)) * c + ((e & 2) ? 8 : 0) + (int64_t)(2 * tq) * c + cb + gq;
    };
    auto eok = [&](int64_t cb, int e) -> bool {
      return erow(e) < p && cb + ecol(e) < jend;
    };
    // Per-warp 3-stage cp.async ring in shared memory: a stage holds one tile
    // of u_{k-1}, u_{k-2} and V (32 rows x 16 columns each, row stride 20:
    // the accumulator-layout reads are bank-conflict free), two tiles ahead
    // of the one being computed.
    constexpr int SS_STAGES = SS<NT>::STAGES, SS_ARR_F = SS<NT>::ARR_F, SS_STAGE_F = SS<NT>::STAGE_F;
    float* ring = reinterpret_cast<float*>(smem_d + (size_t)NW_PPD * SS<NT>::PPW * 3) +
                  (size_t)wid * SS_STAGES * SS_STAGE_F;
    const bool vec = (c & 3) == 0;  // 16-byte rows: cp.async; otherwise plain loads
    auto issue = [&](int tile, int k, int stg) {
      const int64_t cb = j0 + (int64_t)tile * CB;
      float* st = ring + stg * SS_STAGE_F;
      const float* src[3] = {k < 0 ? A.F0 : A.U + (int64_t)((k + 1) & 1) * pc,  // u_{k-1} (F0 at the start)
                             A.U + (int64_t)(k & 1) * pc,                        // u_{k-2}
                             V};
      const int narr = (k <= 0) ? 1 : 2;  // k <= 0: u_{k-2} := u_{k-1}
      for (int arr = 0; arr < 3; ++arr) {
        if (arr == 1 && narr == 1) continue;
        float* dst = st + arr * SS_ARR_F;
        for (int q = lane; q < 8 * NT * 4; q += 32) {
          const int r = q >> 2, ch = q & 3;
          const int64_t col = cb + 4 * ch;
          const int valid = r < p ? (int)imax(0, imin(4, jend - col)) : 0;
          if (vec) {
            const float* g = src[arr] + (valid ? (int64_t)r * c + col : 0);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(dst + r * SS_ROW + 4 * ch)),
                         "l"(g), "r"(4 * valid)
                         : "memory");
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              dst[r * SS_ROW + 4 * ch + i] = i < valid ? src[arr][(int64_t)r * c + col + i] : 0.f;
          }
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // su1 / su2 / sv: this tile's u_{k-1}, u_{k-2} and V in shared memory (a
    // ring stage, or the resident copy); su_out: where u_k goes in shared
    // memory (resident), else u_k is written to U in HBM
    auto tcompute = [&](int tile, int k, float w, bool snap, int slot, bool save, const float* su1,
                        const float* su2, const float* sv, float* su_out, float& s0, double& s1) {
      const int64_t cb = j0 + (int64_t)tile * CB;
      float u1[NE], u2[NE], nv[NE], fe[NE], g[NE];
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const int sidx = erow(e) * SS_ROW + ecol(e);
        u1[e] = su1[sidx];
        u2[e] = k <= 0 ? u1[e] : su2[sidx];
        nv[e] = -sv[sidx];
      }
      if (k >= 0) {
        if (snap) {
          float* sp = A.snaps + (int64_t)(slot * 2) * pc;
          float* bp = A.snaps + (int64_t)(NW_SNAP * 2) * pc;
#pragma unroll
          for (int e = 0; e < NE; ++e)
            if (eok(cb, e)) {
              const int64_t o = eoff(cb, e);
              if (save) {
                bp[o] = sp[o];
                bp[pc + o] = sp[pc + o];
              }
              sp[o] = u1[e];
              sp[pc + o] = u2[e];
            }
        }
#pragma unroll
        for (int e = 0; e < NE; ++e) fe[e] = relu_nan_fast(fmaf(u1[e] - u2[e], w, u1[e]));
      } else {
#pragma unroll
        for (int e = 0; e < NE; ++e) fe[e] = u1[e];  // F0
      }
      grad(fe, nv, g);
      float* __restrict__ Uo = A.U + (int64_t)(k < 0 ? 1 : (k & 1)) * pc;  // u_{-1} -> slot 1
      float pr4 = 0.f;
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const bool ok = eok(cb, e);
        const float u = fmaf(g[e], rnegL, fe[e]);
        if (su_out != nullptr) {
          su_out[erow(e) * SS_ROW + ecol(e)] = ok ? u : 0.f;
        } else if (ok) {
          Uo[eoff(cb, e)] = u;
        }
        // padded elements are exact zeros (zero-filled loads, zero W rows / V
        // entries): they add nothing to the sums
        const float pgv = fe[e] > 0.f ? g[e] : min0_nan(g[e]);
        s0 = fmaf(pgv, pgv, s0);
        pr4 = fmaf(fe[e], g[e] + nv[e], pr4);  // NN_S1_GROUP products in fp32, then added in double
        if ((e & (NN_S1_GROUP - 1)) == NN_S1_GROUP - 1 || e == NE - 1) {
          s1 += (double)pr4;
          pr4 = 0.f;
        }
      }
    };
    // all of this warp's tiles for iteration k through the ring
    float* res = reinterpret_cast<float*>(smem_d + (size_t)NW_PPD * SS<NT>::PPW * 3);  // resident tiles
    auto sweep = [&](int k, float w, bool snap, int slot, bool save, float& s0, double& s1) {
      __syncwarp();  // this warp's u stores of iteration k - 1 are visible to its reads
      const int nmine = wid < ntiles ? (ntiles - 1 - wid) / ncw + 1 : 0;
      if (resident) {
        // every element is read and rewritten by the same lane: no hazards.
        // Padding (rows >= p, columns past the block) holds exact zeros that
        // stay zero (W's padded rows and V's padded entries are zero), so the
        // sums and stores need no validity tests: same values as the ring path
        const int s1i = k < 0 ? 0 : ((k + 1) & 1), s2i = k & 1, so = k < 0 ? 1 : (k & 1);
        for (int i = 0; i < nmine; ++i) {
          const int t = wid + i * ncw;
          const int ob = t * SS_STAGE_F;
          float u1[NE], u2[NE], nv[NE], fe[NE], g[NE];
#pragma unroll
          for (int e = 0; e < NE; ++e) {
            const int sidx = ob + erow(e) * SS_ROW + ecol(e);
            u1[e] = res[sidx + s1i * SS_ARR_F];
            u2[e] = k <= 0 ? u1[e] : res[sidx + s2i * SS_ARR_F];
            nv[e] = -res[sidx + 2 * SS_ARR_F];
          }
          if (k >= 0) {
            if (snap) {
              const int64_t cb = j0 + (int64_t)t * CB;
              float* sp = A.snaps + (int64_t)(slot * 2) * pc;
              float* bp = A.snaps + (int64_t)(NW_SNAP * 2) * pc;
#pragma unroll
              for (int e = 0; e < NE; ++e)
                if (eok(cb, e)) {
                  const int64_t o = eoff(cb, e);
                  if (save) {
                    bp[o] = sp[o];
                    bp[pc + o] = sp[pc + o];
                  }
                  sp[o] = u1[e];
                  sp[pc + o] = u2[e];
                }
            }
#pragma unroll
            for (int e = 0; e < NE; ++e) fe[e] = relu_nan_fast(fmaf(u1[e] - u2[e], w, u1[e]));
          } else {
#pragma unroll
            for (int e = 0; e < NE; ++e) fe[e] = u1[e];  // F0
          }
          grad(fe, nv, g);
          float pr4 = 0.f;
#pragma unroll
          for (int e = 0; e < NE; ++e) {
            res[ob + erow(e) * SS_ROW + ecol(e) + so * SS_ARR_F] = fmaf(g[e], rnegL, fe[e]);
            const float pgv = fe[e] > 0.f ? g[e] : min0_nan(g[e]);
            s0 = fmaf(pgv, pgv, s0);
            pr4 = fmaf(fe[e], g[e] + nv[e], pr4);  // NN_S1_GROUP products in fp32, then added in double
            if ((e & (NN_S1_GROUP - 1)) == NN_S1_GROUP - 1 || e == NE - 1) {
              s1 += (double)pr4;
              pr4 = 0.f;
            }
          }
        }
        return;
      }
      for (int i = 0; i < SS_STAGES - 1; ++i) {
        if (i < nmine) issue(wid + i * ncw, k, i);
        else asm volatile("cp.async.commit_group;" ::: "memory");
      }
      for (int i = 0; i < nmine; ++i) {
        asm volatile("cp.async.wait_group %0;" ::"n"(SS_STAGES - 2) : "memory");
        __syncwarp();
        const float* st = ring + (i % SS_STAGES) * SS_STAGE_F;
        tcompute(wid + i * ncw, k, w, snap, slot, save, st, st + SS_ARR_F, st + 2 * SS_ARR_F, nullptr, s0, s1);
        __syncwarp();  // the stage is refilled below
        if (i + SS_STAGES - 1 < nmine) issue(wid + (i + SS_STAGES - 1) * ncw, k, (i + SS_STAGES - 1) % SS_STAGES);
        else asm volatile("cp.async.commit_group;" ::: "memory");
      }
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    };
    if (resident) {
      // this warp's tiles of F0 (-> U slot 0, the start point's input) and V,
      // zero-padded past the problem, once
      for (int t = wid; t < ntiles; t += ncw) {
        const int64_t cb = j0 + (int64_t)t * CB;
        float* base = res + (size_t)t * SS_STAGE_F;
        for (int q = lane; q < 8 * NT * CB; q += 32) {
          const int r = q / CB, cc = q % CB;
          const bool ok = r < p && cb + cc < jend;
          const int64_t o = (int64_t)r * c + cb + cc;
          base[r * SS_ROW + cc] = ok ? A.F0[o] : 0.f;
          base[2 * SS_ARR_F + r * SS_ROW + cc] = ok ? V[o] : 0.f;
        }
      }
      __syncwarp();
    }
    // start point (nnls.py:163-178)
    {
      float s0 = 0.f;
      double s1 = 0.0;
      sweep(-1, 0.f, false, 0, false, s0, s1);
      post(-1, s0, s1);
      post_flag(-1);
    }
    double wwin = 0.0, wnext = wload(0);
    int k = 0;
    for (; k < max_iter; ++k) {
      bool snap = false, save = false;
      int slot = 0;
      if (k % NW_WIN == 0) {
        const int w = k / NW_WIN;
        wwin = wnext;
        wnext = wload(k + NW_WIN);
        int ok = 1;
        if (lane == 0) {
          const int need = (w - NW_FLIGHT) * NW_WIN - 1;
          while (sh.resolved < need && !sh.halt) __nanosleep(64);
          ok = sh.halt ? 0 : 1;
        }
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (!ok) break;
        slot = w % NW_SNAP;
        const int evicted = w - NW_SNAP;
        const int bj = sh.best_j;
        save = evicted >= 0 && bj >= 0 && bj / NW_WIN == evicted;
        snap = true;
        if (lane == 0 && save) sh.bsw[wid] = evicted;
        __syncwarp();
      } else if (sh.halt) {
        break;
      }
      const float w = (float)__shfl_sync(0xffffffffu, wwin, k % NW_WIN);
      float s0 = 0.f;
      double s1 = 0.0;
      sweep(k, w, snap, slot, save, s0, s1);
      post(k, s0, s1);
      if ((k + 1) % NW_WIN == 0) post_flag(k);
    }
    if (k > 0) post_flag(k - 1);
    if (lane == 0) sh.kdone[wid] = k;
    __syncwarp();
    asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
    // ---- the best iterate, recomputed from its window's snapshot
    const int bj = sh.best_j;
    if (bj >= 0 && sh.fail_at == -1) {
      const int kd = sh.kdone[wid];
      const int wb = bj / NW_WIN;
      const int slot = (sh.bsw[wid] == wb && wb + NW_SNAP <= (kd - 1) / NW_WIN) ? NW_SNAP : wb % NW_SNAP;
      const float* sp = A.snaps + (int64_t)(slot * 2) * pc;
      const double wrec = wload(wb * NW_WIN);
      for (int t = wid; t < ntiles; t += ncw) {
        const int64_t cb = j0 + (int64_t)t * CB;
        float ua[NE], ub[NE], nv[NE], fe[NE], g[NE];
        int64_t off[NE];
        bool ok[NE];
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          const int r = erow(e);
          const int64_t col = cb + ecol(e);
          ok[e] = r < p && col < j0 + ncols;
          off[e] = (int64_t)r * c + col;
          ua[e] = ok[e] ? sp[off[e]] : 0.f;
          ub[e] = ok[e] ? sp[pc + off[e]] : 0.f;
          nv[e] = ok[e] ? -V[off[e]] : 0.f;
        }
        for (int kk = wb * NW_WIN; kk <= bj; ++kk) {
          const float w = (float)__shfl_sync(0xffffffffu, wrec, kk % NW_WIN);
#pragma unroll
          for (int e = 0; e < NE; ++e) fe[e] = relu_nan_fast(fmaf(ua[e] - ub[e], w, ua[e]));
          grad(fe, nv, g);
#pragma unroll
          for (int e = 0; e < NE; ++e) {
            ub[e] = ua[e];
            ua[e] = fmaf(g[e], rnegL, fe[e]);
          }
        }
#pragma unroll
        for (int e = 0; e < NE; ++e)
          if (ok[e]) A.Fout[off[e]] = fe[e];
      }
    }
  } else {
    resolver_warp(sh, pp, ncw, max_iter, A.grad_tol, L, A.recs, A.results, nullptr, SS<NT>::PPW, nullptr,
                  A.watchdog_ns);
    asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
  }
  __syncthreads();
  if (blockIdx.x == 0 && tid == 0) {
    nenmf_device_status* st = A.st;
    if (sh.fail_at >= 0) status_fail(st, NENMF_ERR_NUMERICAL_FAILURE, sh.fail_at);
    if (sh.fail_at == -2) status_fail(st, NENMF_ERR_WATCHDOG, -2);
    st->inner_iters = sh.stop_at >= 0 ? sh.stop_at + 1 : (sh.fail_at >= 0 ? sh.fail_at : max_iter);
    st->returned_best = sh.best_j >= 0 ? 1 : 0;
    st->best_partial = sh.best_part;
    st->pg_ref = sh.pg_ref;
  }
}

// grid: one CTA per SM (cooperative); returns NENMF_ERR_UNSUPPORTED outside FP32, p <= 32
int launch_nnls_stream(StreamArgs& a, int grid, cudaStream_t s) {
  const int nt = (a.p + 7) / 8;
  const int ntiles = (int)((a.cpb + 15) / 16);
  // the CTA's state stays on chip when its tiles fit (cfg5: 43 tiles of 16 x 16)
  constexpr size_t kSmemCap = 227 * 1024 - 2048;  // leave room for the static shared memory
  void* args[] = {(void*)&a};
  switch (nt) {
#define NENMF_STREAM_CASE(N)                                                                               \
  case N: {                                                                                                \
    const char* env = getenv("NENMF_STREAM_RING");  /* development knob: force the HBM ring */             \
    a.resident = (env == nullptr && SS<N>::smem(true, ntiles) <= kSmemCap) ? 1 : 0;                       \
    const size_t sm = SS<N>::smem(a.resident != 0, ntiles);                                               \
    NENMF_CUDA_TRY(set_smem(k_nnls_stream<N>, sm));                                                        \
    NENMF_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_nnls_stream<N>, dim3(grid),                  \
                                               dim3(stream_threads<N>()), args, sm, s));                   \
    break;                                                                                                 \
  }
    NENMF_STREAM_CASE(1)
    NENMF_STREAM_CASE(2)
    NENMF_STREAM_CASE(3)
    NENMF_STREAM_CASE(4)
    NENMF_STREAM_CASE(5)
    NENMF_STREAM_CASE(6)
    NENMF_STREAM_CASE(7)
    NENMF_STREAM_CASE(8)
#undef NENMF_STREAM_CASE
    default:
      return NENMF_ERR_UNSUPPORTED;
  }
  launch_counter_add(1);
  return NENMF_OK;
}

}  // namespace nenmf
