// FP64 X-pass with ONE read of X for both products (compression.py:134-139,
// 188): Yt = At X^T (k x n) and Zt = Bt X (k x m), k <= 32, on the FP64
// tensor pipe (DMMA m8n8k4, exact fp64 products, fp64 accumulation).
//
// Each 64 x 64 tile of X is staged once in shared memory (cp.async, 3-stage
// ring, with the At slice of its columns and the Bt slice of its rows) and
// feeds both products: warp w owns rows 8w..8w+7 of the tile for Y (the X
// fragment as the A operand) and columns 8w..8w+7 for Z (the X fragment as
// the B operand).  A unit is a band of CT column tiles x a chunk of row
// tiles: Y of the current row tile accumulates over the band's CT tiles in
// registers, Z of the band's CT column tiles over the chunk's row tiles; the
// per-unit partials go to slabs summed in fixed order (deterministic).
//
// The earlier FP64 pass ran the two products as two kernels, each streaming
// X (k_xv64, k_ux64): twice the X traffic and each product's DMMAs waiting
// on its own stream.
#include "rsi.cuh"
#include "skinny.cuh"

#include <cuda.h>

#include <cstdlib>

namespace nenmf {

namespace d64 {
constexpr int T = 64;      // tile rows = tile columns
constexpr int CT = 4;      // column tiles per band
constexpr int XS = 68;     // shared row stride (doubles): conflict-free fragment reads
constexpr int NS = 3;      // stages
constexpr int STAGE = T * XS + 2 * 32 * XS;  // X tile | At slice (32 x 64) | Bt slice (32 x 64), doubles
constexpr int THREADS = 256;

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp16(double* dst, const double* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes)
               : "memory");
}

__global__ void __launch_bounds__(THREADS, 1)
k_dual64(const double* __restrict__ X, int64_t n, int64_t m, int64_t ldx, const double* __restrict__ At,
         const double* __restrict__ Bt, int k, int n_ct, int nbands, int rchunk, int64_t nunits,
         double* __restrict__ Yslab, double* __restrict__ Zslab) {
  extern __shared__ __align__(16) double dsm[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, gq = lane >> 2, tq = lane & 3;
  const int n_rt = (int)((n + T - 1) / T);
  const int ntk = (k + 7) >> 3;  // 8-wide blocks of the skinny dimension in use
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int cb = (int)(u % nbands), rc = (int)(u / nbands);
    const int ct0 = cb * CT, ct1 = min(n_ct, ct0 + CT), nct = ct1 - ct0;
    const int rt0 = rc * rchunk, rt1 = min(n_rt, rt0 + rchunk);
    const int ntl = (rt1 - rt0) * nct;
    auto issue = [&](int t, int stg) {
      double* xs = dsm + (size_t)stg * STAGE;
      double* as = xs + T * XS;
      double* bs = as + 32 * XS;
      const int rt = rt0 + t / nct, ct = ct0 + t % nct;
      const int64_t i0 = (int64_t)rt * T, j0 = (int64_t)ct * T;
      for (int c = tid; c < T * 32; c += THREADS) {  // 64 rows x 32 chunks of 2 doubles
        const int r = c >> 5, ch = c & 31;
        const int64_t i = i0 + r, j = j0 + 2 * ch;
        const int valid = i < n ? (int)imax(0, imin(2, m - j)) : 0;
        cp16(xs + r * XS + 2 * ch, X + (valid ? i * ldx + j : 0), 8 * valid);
      }
      for (int c = tid; c < 2 * 32 * 32; c += THREADS) {  // At (a, cols) and Bt (a, rows) slices
        const bool isA = c < 32 * 32;
        const int cc = isA ? c : c - 32 * 32;
        const int a = cc >> 5, ch = cc & 31;
        const int64_t len = isA ? m : n, base = isA ? j0 : i0;
        const int64_t j = base + 2 * ch;
        const int valid = a < k ? (int)imax(0, imin(2, len - j)) : 0;
        const double* src = isA ? At : Bt;
        cp16((isA ? as : bs) + a * XS + 2 * ch, src + (valid ? (int64_t)a * len + j : 0), 8 * valid);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double accy[4][2], accz[CT][4][2];
#pragma unroll
    for (int b = 0; b < 4; ++b) accy[b][0] = accy[b][1] = 0.0;
#pragma unroll
    for (int c = 0; c < CT; ++c)
#pragma unroll
      for (int b = 0; b < 4; ++b) accz[c][b][0] = accz[c][b][1] = 0.0;
    __syncthreads();
    for (int i = 0; i < NS - 1; ++i) {
      if (i < ntl) issue(i, i);
      else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int t = 0; t < ntl; ++t) {
      asm volatile("cp.async.wait_group %0;" ::"n"(NS - 2) : "memory");
      __syncthreads();
      const double* xs = dsm + (size_t)(t % NS) * STAGE;
      const double* as = xs + T * XS;
      const double* bs = as + 32 * XS;
      const int cc = t % nct;
      // the column tile's Z accumulators into a working set (predicated
      // moves: register arrays cannot be indexed at run time)
      double az[4][2];
#pragma unroll
      for (int b = 0; b < 4; ++b) az[b][0] = az[b][1] = 0.0;
#pragma unroll
      for (int c = 0; c < CT; ++c)
        if (c == cc) {
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            az[b][0] = accz[c][b][0];
            az[b][1] = accz[c][b][1];
          }
        }
      // both products per K step, so eight independent DMMA chains are in
      // flight per warp: Y (rows 8w + gq) += X_tile A with the X fragment as
      // the A operand (K = columns), Z (columns 8w + gq) += Bt X_tile with it
      // as the B operand (K = rows)
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) {
        const double xa = xs[(8 * wid + gq) * XS + 4 * ks + tq];
        const double xb = xs[(4 * ks + tq) * XS + 8 * wid + gq];
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (b < ntk) {
            dmma(accy[b], xa, as[(8 * b + gq) * XS + 4 * ks + tq]);
            dmma(az[b], bs[(8 * b + gq) * XS + 4 * ks + tq], xb);
          }
      }
#pragma unroll
      for (int c = 0; c < CT; ++c)
        if (c == cc) {
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            accz[c][b][0] = az[b][0];
            accz[c][b][1] = az[b][1];
          }
        }
      __syncthreads();
      if (t + NS - 1 < ntl) issue(t + NS - 1, (t + NS - 1) % NS);
      else asm volatile("cp.async.commit_group;" ::: "memory");
      if (cc == nct - 1) {
        // the row tile's Y over this band: C (row, a), row = 8w + gq, a = 8b + 2tq + h
        const int64_t i = (int64_t)(rt0 + t / nct) * T + 8 * wid + gq;
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int a = 8 * b + 2 * tq + h;
            if (a < k && i < n) Yslab[((int64_t)cb * k + a) * n + i] = accy[b][h];
            accy[b][h] = 0.0;
          }
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    // the band's Z over this chunk: C (a, col), a = 8b + gq, col = 8w + 2tq + h
#pragma unroll
    for (int c = 0; c < CT; ++c) {
      if (c >= nct) continue;
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int a = 8 * b + gq;
          const int64_t j = (int64_t)(ct0 + c) * T + 8 * wid + 2 * tq + h;
          if (a < k && j < m) Zslab[((int64_t)rc * k + a) * m + j] = accz[c][b][h];
        }
    }
  }
}

__global__ void k_slab_sum64(const double* __restrict__ py, int ny, int64_t cy, double* __restrict__ oy,
                             const double* __restrict__ pz, int nz, int64_t cz, double* __restrict__ oz) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cy + cz) return;
  const bool isY = i < cy;
  const double* __restrict__ part = isY ? py : pz;
  const int nslab = isY ? ny : nz;
  const int64_t count = isY ? cy : cz, o = isY ? i : i - cy;
  double s = part[o];
  for (int c = 1; c < nslab; ++c) s += part[(int64_t)c * count + o];
  (isY ? oy : oz)[o] = s;
}
}  // namespace d64

// ---------------------------------------------------------------------------
// Warp-specialised version: one producer warp streams the tiles with TMA
// (cp.async.bulk.tensor.2d over tensor maps of X, At and Bt: 12 instructions
// per 64 x 64 tile, out-of-range rows / columns and the skinny rows >= k
// zero-filled by the hardware, completion counted on an mbarrier), eight
// consumer warps issue the DMMAs -- no per-thread copy instructions or CTA
// barriers in the loop.  (Per-row 1-D bulk copies, 128 per tile, were tried
// first: the copy engine retires ~1 small copy per 60 cycles, 2.4 TB/s at
// 512 B, tools/micro/bulk.cu, which bounded the pass at 0.84 ms.)
// Shared-memory tiles are 16-column slabs of 128-byte rows in the 128-byte
// swizzle (16-byte chunk index ^ (row & 7)).  Warps 0-3 own Y (16 rows of the
// tile each: two m-tiles share every skinny fragment), warps 4-7 own Z (16
// columns = one slab each: two n-tiles share every skinny fragment): 6
// shared-memory loads per 8 DMMAs, one Y and one Z warp per scheduler; the
// same loop fed from shared memory reaches the DMMA peak in isolation
// (tools/micro/fp64_peak.cu, FP64_VAR).
namespace d64w {
using d64::dmma;
using d64::T;
constexpr int CT = 4;                      // column tiles per band
constexpr int NS = 4;                      // X stages
constexpr int XB = T * 16 * 8;             // one X slab: 64 rows x 128 B
constexpr int SB = 32 * 16 * 8;            // one skinny slab: 32 rows x 128 B
constexpr int XTILE = 4 * XB;              // 32 KB
constexpr int STILE = 4 * SB;              // a 32 x 64 skinny slice: 16 KB
// shared memory: [At slices of the band's CT column tiles, resident per unit | Bt slice of the
// tile row, double buffered | NS X tiles] = 64 + 32 + 128 KB: a tile costs 32 KB of X plus 4 KB
// of Bt (At once per unit), not 64 KB as with per-tile skinny slices
constexpr int A_OFF = 0, B_OFF = CT * STILE, X_OFF = B_OFF + 2 * STILE;
constexpr int SMEM = X_OFF + NS * XTILE;
constexpr int NCONS = 8;
constexpr int THREADS = 32 * (NCONS + 1);

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}
// shared-space load by 32-bit address (the tile base is rounded up through an integer cast, which
// would otherwise leave the compiler with generic-address loads); volatile: stays below the mbarrier wait
__device__ __forceinline__ double lds(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

__global__ void __launch_bounds__(THREADS, 1)
k_dual64t(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmA,
          const __grid_constant__ CUtensorMap tmB, int64_t n, int64_t m, int k, int n_ct, int nbands, int rchunk,
          int64_t nunits, double* __restrict__ Yslab, double* __restrict__ Zslab, int dbg) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar_full[NS], bar_empty[NS], bar_bfull[2], bar_bempty[2], bar_afull, bar_aempty;
  const int tid = threadIdx.x, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
  const int wid = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int n_rt = (int)((n + T - 1) / T);
  const int ntk = (k + 7) >> 3;  // 8-wide blocks of the skinny dimension in use
  const uint32_t sbase = su32(smem);
  if (tid == 0) {
    auto init = [](uint64_t* b, int cnt) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(cnt) : "memory");
    };
    for (int s = 0; s < NS; ++s) {
      init(&bar_full[s], 1);
      init(&bar_empty[s], NCONS);
    }
    for (int b = 0; b < 2; ++b) {
      init(&bar_bfull[b], 1);
      init(&bar_bempty[b], 4);  // the Z warps
    }
    init(&bar_afull, 1);
    init(&bar_aempty, 4);  // the Y warps
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // Fragment rows within an 8-row block are taken in the order 0,2,4,6,1,3,5,7 (pg): a half-warp
  // (gq 0..3, the unit the 8-byte shared loads are served in) then reads rows whose swizzle keys
  // differ in bits 1-2, so its two 16-byte chunks per row land in 8 distinct chunks: no bank
  // conflict (the natural order folds them onto 4 chunks: 2-way).  The outputs carry the same
  // permutation (emit indices below).
  const int pg = ((gq & 3) << 1) | (gq >> 2);
  // swizzled offset of the thread's 16-byte chunk for k-steps with (ks & 3) = q, rows with (row & 7) = pg
  uint32_t offq[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) offq[q] = (uint32_t)(((2 * q) ^ ((tq >> 1) ^ pg)) << 4);

  if (wid == NCONS) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int t = 0, rowc = 0, uc = 0;
      for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, ++uc) {
        const int cb = (int)(u % nbands), rc = (int)(u / nbands);
        const int ct0 = cb * CT, nct = min(n_ct, ct0 + CT) - ct0;
        const int rt0 = rc * rchunk, rt1 = min(n_rt, rt0 + rchunk);
        mb_wait(&bar_aempty, (uc & 1) ^ 1);
        mb_expect(&bar_afull, (uint32_t)(nct * STILE));
        for (int c = 0; c < nct; ++c)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            tma_2d(smem + A_OFF + c * STILE + q * SB, &tmA, (ct0 + c) * T + 16 * q, 0, &bar_afull);
        for (int rt = rt0; rt < rt1; ++rt, ++rowc) {
          const int rb = rowc & 1, i0 = rt * T;
          mb_wait(&bar_bempty[rb], ((rowc >> 1) & 1) ^ 1);
          mb_expect(&bar_bfull[rb], (uint32_t)STILE);
#pragma unroll
          for (int q = 0; q < 4; ++q) tma_2d(smem + B_OFF + rb * STILE + q * SB, &tmB, i0 + 16 * q, 0, &bar_bfull[rb]);
          for (int c = 0; c < nct; ++c, ++t) {
            const int s = t % NS;
            mb_wait(&bar_empty[s], ((t / NS) & 1) ^ 1);
            mb_expect(&bar_full[s], (uint32_t)XTILE);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              tma_2d(smem + X_OFF + s * XTILE + q * XB, &tmX, (ct0 + c) * T + 16 * q, i0, &bar_full[s]);
          }
        }
      }
    }
  } else if (wid < 4) {
    // ------------------------------------------------------------ Y warps
    const int w = wid;
    const uint32_t xoff = (uint32_t)(X_OFF + (16 * w + pg) * 128 + (tq & 1) * 8);
    const uint32_t aoff = (uint32_t)(A_OFF + pg * 128 + (tq & 1) * 8);
    int t = 0, uc = 0;
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, ++uc) {
      const int cb = (int)(u % nbands), rc = (int)(u / nbands);
      const int ct0 = cb * CT, nct = min(n_ct, ct0 + CT) - ct0;
      const int rt0 = rc * rchunk, rt1 = min(n_rt, rt0 + rchunk);
      mb_wait(&bar_afull, uc & 1);
      for (int rt = rt0; rt < rt1; ++rt) {
        double acc[2][4][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[i][b][0] = acc[i][b][1] = 0.0;
        for (int c = 0; c < nct; ++c, ++t) {
          const int s = t % NS;
          mb_wait(&bar_full[s], (t / NS) & 1);
          const uint32_t xb = sbase + xoff + s * XTILE;
          const uint32_t ab = sbase + aoff + c * STILE;
          if (!(dbg & 1))
#pragma unroll
          for (int ks = 0; ks < 16; ++ks) {
            const uint32_t o = offq[ks & 3];
            const double xa0 = lds(xb + (ks >> 2) * XB + o), xa1 = lds(xb + (ks >> 2) * XB + 1024 + o);
#pragma unroll
            for (int b = 0; b < 4; ++b)
              if (b < ntk) {
                const double sk = lds(ab + (ks >> 2) * SB + b * 1024 + o);
                dmma(acc[0][b], xa0, sk);
                dmma(acc[1][b], xa1, sk);
              }
          }
          __syncwarp();
          if (lane == 0) mb_arrive(&bar_empty[s]);
        }
        // the row tile's Y over this band: C (m slot gq, n slot 2tq + h) = (row 16w + 8i + pg, a = 8b + perm(2tq + h))
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int64_t row = (int64_t)rt * T + 16 * w + 8 * i + pg;
#pragma unroll
          for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int ns = 2 * tq + h;
              const int a = 8 * b + (((ns & 3) << 1) | (ns >> 2));
              if (a < k && row < n) Yslab[((int64_t)cb * k + a) * n + row] = acc[i][b][h];
            }
        }
      }
      __syncwarp();
      if (lane == 0) mb_arrive(&bar_aempty);  // the band's At slices may be replaced
    }
  } else {
    // ------------------------------------------------------------ Z warps
    const int w = wid - 4;
    // X as the B operand (k = row 4ks + tq, n = column 16w + 8j + gq): slab w,
    // chunk (4j + (gq >> 1)) ^ (4 (ks & 1) + tq) = 4 (j ^ (ks & 1)) + ((gq >> 1) ^ tq)
    const uint32_t zoff = (uint32_t)(X_OFF + w * XB + tq * 128 + ((((gq >> 1) ^ tq)) << 4) + (gq & 1) * 8);
    const uint32_t boff = (uint32_t)(B_OFF + pg * 128 + (tq & 1) * 8);
    int t = 0, rowc = 0;
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int cb = (int)(u % nbands), rc = (int)(u / nbands);
      const int ct0 = cb * CT, nct = min(n_ct, ct0 + CT) - ct0;
      const int rt0 = rc * rchunk, rt1 = min(n_rt, rt0 + rchunk);
      double acc[CT][4][2][2];
#pragma unroll
      for (int c = 0; c < CT; ++c)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int j = 0; j < 2; ++j) acc[c][b][j][0] = acc[c][b][j][1] = 0.0;
      for (int rt = rt0; rt < rt1; ++rt, ++rowc) {
        const int rb = rowc & 1;
        mb_wait(&bar_bfull[rb], (rowc >> 1) & 1);
        const uint32_t bb = sbase + boff + rb * STILE;
#pragma unroll
        for (int c = 0; c < CT; ++c) {
          if (c < nct) {
            const int s = t % NS;
            mb_wait(&bar_full[s], (t / NS) & 1);
            const uint32_t zb = sbase + zoff + s * XTILE;
            if (!(dbg & 1))
#pragma unroll
            for (int ks = 0; ks < 16; ++ks) {
              const double xb0 = lds(zb + ks * 512 + ((0 ^ (ks & 1)) << 6));
              const double xb1 = lds(zb + ks * 512 + ((1 ^ (ks & 1)) << 6));
              const uint32_t o = offq[ks & 3];
#pragma unroll
              for (int b = 0; b < 4; ++b)
                if (b < ntk) {
                  const double sk = lds(bb + (ks >> 2) * SB + b * 1024 + o);
                  dmma(acc[c][b][0], sk, xb0);
                  dmma(acc[c][b][1], sk, xb1);
                }
            }
            __syncwarp();
            if (lane == 0) mb_arrive(&bar_empty[s]);
            ++t;
          }
        }
        __syncwarp();
        if (lane == 0) mb_arrive(&bar_bempty[rb]);
      }
      // the band's Z over this chunk: C (m slot gq, n slot 2tq + h) = (a = 8b + pg, col = 16w + 8j + 2tq + h)
#pragma unroll
      for (int c = 0; c < CT; ++c) {
        if (c >= nct) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int a = 8 * b + pg;
              const int64_t col = (int64_t)(ct0 + c) * T + 16 * w + 8 * j + 2 * tq + h;
              if (a < k && col < m) Zslab[((int64_t)rc * k + a) * m + col] = acc[c][b][j][h];
            }
      }
    }
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (the library links no libcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}
// rows x cols row-major fp64 matrix (leading dimension ld), boxes of 16 columns x box_rows rows, 128-byte swizzle
static bool make_map(CUtensorMap* tm, const double* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) return false;
  const cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t gstride[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), gdim, gstride, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace d64w

bool xpass_timing_begin(cudaEvent_t* e0, cudaEvent_t* e1);

int dual_pass_f64(Arena& ws, const double* X, int64_t n, int64_t m, int64_t ldx, const double* At,
                  const double* Bt, int64_t k, double* Yt, double* Zt, cudaStream_t s) {
  using namespace d64;
  // Default: the warp-specialised TMA kernel (one read of X).  NENMF_DUAL64=off: the two one-product
  // kernels (k_xv64 + k_ux64, two reads of X); =v1: the first fused kernel (per-thread cp.async).
  static const char* mode = getenv("NENMF_DUAL64");
  const bool off = mode != nullptr && mode[0] == 'o', v1 = mode != nullptr && mode[0] == 'v';
  if (off || k < 1 || k > 32 || At == nullptr || Bt == nullptr) return NENMF_ERR_UNSUPPORTED;
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (((n | m | ldx) & 1) != 0 || (ws.base != nullptr && (!al16(X) || !al16(At) || !al16(Bt))))
    return NENMF_ERR_UNSUPPORTED;
  int sms = sm_count();
  if (sms <= 0) sms = 148;
  const int n_rt = (int)cdiv(n, T), n_ct = (int)cdiv(m, T);
  const int nbands = (int)cdiv(n_ct, CT);
  int rchunk, nrc_used;
  if (v1) {
    // row chunks: about two units per SM (balance), at least one row tile each
    const int nrc = (int)imax(1, imin(n_rt, cdiv(2 * sms, nbands)));
    rchunk = (int)cdiv(n_rt, nrc);
    nrc_used = (int)cdiv(n_rt, rchunk);
  } else {
    // row chunks: units are dealt round-robin to the persistent CTAs; take the
    // chunking with the smallest heaviest CTA (tiles + the Z slab it costs)
    double best = 1e300;
    rchunk = n_rt;
    for (int rch = 1; rch <= n_rt; ++rch) {
      const int used = (int)cdiv(n_rt, rch);
      const int64_t units = (int64_t)nbands * used;
      if (units > 16 * (int64_t)sms && rch < n_rt) continue;
      const int G = (int)imin(units, (int64_t)sms);
      double mx = 0.0;
      for (int g = 0; g < G; ++g) {
        double load = 0.0;
        for (int64_t u = g; u < units; u += G) {
          const int cb = (int)(u % nbands), rc = (int)(u / nbands);
          const int cols = (int)imin(n_ct, (int64_t)(cb + 1) * CT) - cb * CT;
          const int rows = (int)imin(n_rt, (int64_t)(rc + 1) * rch) - rc * rch;
          load += (double)rows * cols + 0.25 * cols;  // + the unit's Z drain
        }
        mx = load > mx ? load : mx;
      }
      const double slab = (double)used * (double)k * (double)m * 16.0 / G / (T * T * 8.0);
      const double cost = mx + 0.35 * slab;
      if (cost < best) {
        best = cost;
        rchunk = rch;
      }
    }
    nrc_used = (int)cdiv(n_rt, rchunk);
  }
  const int64_t nunits = (int64_t)nbands * nrc_used;
  double* Yslab = ws.take<double>((size_t)nbands * k * n);
  double* Zslab = ws.take<double>((size_t)nrc_used * k * m);
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  const bool timed = xpass_timing_begin(&ev0, &ev1);
  if (timed) cudaEventRecord(ev0, s);
  if (v1) {
    const size_t smem = (size_t)NS * STAGE * sizeof(double);
    NENMF_CUDA_TRY(set_smem(k_dual64, smem));
    k_dual64<<<(unsigned)imin(nunits, (int64_t)sms), THREADS, smem, s>>>(X, n, m, ldx, At, Bt, (int)k, n_ct, nbands,
                                                                          rchunk, nunits, Yslab, Zslab);
  } else {
    CUtensorMap tmX, tmA, tmB;
    if (!d64w::make_map(&tmX, X, n, m, ldx, 64) || !d64w::make_map(&tmA, At, k, m, m, 32) ||
        !d64w::make_map(&tmB, Bt, k, n, n, 32))
      return NENMF_ERR_UNSUPPORTED;  // no tensor-map entry point / unsupported strides: the two-kernel pass
    const size_t smem = (size_t)d64w::SMEM + 1024;
    NENMF_CUDA_TRY(set_smem(d64w::k_dual64t, smem));
    d64w::k_dual64t<<<(unsigned)imin(nunits, (int64_t)sms), d64w::THREADS, smem, s>>>(
        tmX, tmA, tmB, n, m, (int)k, n_ct, nbands, rchunk, nunits, Yslab, Zslab,
        getenv("NENMF_DUAL64_DBG") != nullptr ? atoi(getenv("NENMF_DUAL64_DBG")) : 0);
  }
  NENMF_LAUNCH_CHECK();
  if (timed) cudaEventRecord(ev1, s);
  const int64_t cy = k * n, cz = k * m;
  k_slab_sum64<<<(unsigned)cdiv(cy + cz, 256), 256, 0, s>>>(Yslab, nbands, cy, Yt, Zslab, nrc_used, cz, Zt);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

}  // namespace nenmf
