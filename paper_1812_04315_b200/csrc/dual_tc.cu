// Tensor-core (tcgen05) X-pass for FP32 data: Y^T = A^T X^T and Z^T = B^T X
// from ONE read of X (compression.py:134-139,188), BF16x3 split precision.
//
// Every fp32 element x is split into bf16 hi = rn(x) and lo = rn(x - hi);
// the skinny operands likewise, and x a ~= x_hi a_hi + x_hi a_lo + x_lo a_hi
// (relative error ~1e-5, fp32-class).
//
// X is split ONCE per sketch (k_presplit_x) into "tile-major" form: every
// 128 x 128 tile is one contiguous 64 KB block [hi | lo] already in the
// canonical 128-byte-swizzled K-major shared-memory layout, so a pass is a
// plain stream of 1-D bulk copies (cp.async.bulk, mbarrier complete_tx) into
// shared memory: no producer threads, no register staging.  The pre-split
// copy holds exactly 4 bytes per element, the same bytes as fp32 X, and every
// one of the 2q+2 passes of the sketch (and the compression pass) reads it.
//
// The SAME shared-memory bytes feed both products:
//   Y (rows of X as M, columns as K)  : A = X tile, K-major descriptor
//   Z (columns of X as M, rows as K)  : A = X tile, MN-major descriptor
// Per 16-wide K-chunk three MMAs with N = kpad into one TMEM accumulator:
// x_hi a_hi, x_hi a_lo, x_lo a_hi.
//
// Work: units of (row chunk) x (column block of CT tiles).  Z accumulators of
// the column block live in TMEM for the whole unit; Y accumulators (double
// buffered) for one tile row.  Partial sums per unit are written to global
// slabs and reduced in fixed order (deterministic).  The unit grid is chosen
// on the host to balance tiles per CTA against slab traffic.
//
// Roles (6 warps): 0 bulk-copy producer (one elected thread), 1 MMA issuer +
// TMEM owner, 2-5 epilogue (TMEM -> registers -> global; lane quadrant = warp % 4).
#include "rsi.cuh"

#include <cuda_bf16.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

namespace nenmf {

namespace tc {

constexpr int TILE = 128;
constexpr int PROD_WARP = 0;
constexpr int MMA_WARP = 1;
constexpr int EPI_WARP0 = 2;      // epilogue warps 2..5 (TMEM lane quadrant = warp % 4)
constexpr int NWARPS = 6;
constexpr int NSTAGE = 2;
constexpr int SUB_BYTES = TILE * 128;       // one 128-row x 64-col bf16 sub-tile
constexpr int XTILE_BYTES = 4 * SUB_BYTES;  // [hi sub0 | hi sub1 | lo sub0 | lo sub1] = 64 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// shared-memory matrix descriptor, 128-byte swizzle, sm_100 (version 1)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// The descriptor's address field holds (shared address >> 4) in 14 bits; shared
// memory ends below 256 KB, so moving a descriptor by `bytes` is one 32-bit
// add on its low word.  The MMA warp keeps every descriptor a warp-uniform
// value (uniform registers, no per-MMA register-to-uniform transfers): the
// whole warp computes them and one elected lane issues the instruction.
__device__ __forceinline__ uint32_t sdesc_lo(uint32_t saddr, uint32_t lbo) {
  return ((saddr >> 4) & 0x3FFFu) | (((lbo >> 4) & 0x3FFFu) << 16);
}
constexpr uint32_t SDESC_HI = ((1024u >> 4) & 0x3FFFu) | (1u << 14) | (2u << 29);  // SBO 1024, version 1, 128B swizzle
__device__ __forceinline__ uint64_t sdesc_at(uint32_t lo, uint32_t bytes) {
  return ((uint64_t)SDESC_HI << 32) | (uint64_t)(lo + (bytes >> 4));
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
}
// instruction descriptor: BF16 x BF16 -> F32, M = 128
__host__ __device__ constexpr uint32_t idesc_bf16(int N, bool a_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(TILE >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// shared-space 16-byte load by 32-bit address (the tile base is rounded up through an integer cast,
// which leaves plain dereferences as generic-address loads)
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// 1-D bulk copy global -> shared, completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

struct Units {
  int n_rt, n_ct;       // tiles along rows / columns of X
  int n_cb, n_rc;       // column blocks, row chunks
  int units;
};

__device__ __forceinline__ void unit_bounds(const Units& U, int u, int& rt0, int& rt1, int& ct0, int& ct1, int& rc,
                                            int& cb) {
  rc = u / U.n_cb;
  cb = u % U.n_cb;
  rt0 = (int)((int64_t)rc * U.n_rt / U.n_rc);
  rt1 = (int)((int64_t)(rc + 1) * U.n_rt / U.n_rc);
  ct0 = (int)((int64_t)cb * U.n_ct / U.n_cb);
  ct1 = (int)((int64_t)(cb + 1) * U.n_ct / U.n_cb);
}

// X (n x m fp32, leading dimension ldx) -> tile-major pre-split bf16 hi/lo.
// One thread per (tile, row, 8-column chunk): reads 32 B, writes 16 B of hi
// and 16 B of lo at the swizzled position; padding outside X is zero.
// With `nonzero` set, also raises *nonzero when any element of X is nonzero
// (the X != 0 check of compression.py:109-117, folded into this read of X).
__global__ void k_presplit_x(const float* __restrict__ X, int64_t n, int64_t m, int64_t ldx, int n_ct, int64_t total,
                             uint8_t* __restrict__ Xs, int* __restrict__ nonzero) {
  bool nz = false;
  const bool vec = ((m | ldx) & 3) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c8 = (int)(i & 15);
    const int r = (int)((i >> 4) & 127);
    const int64_t tile = i >> 11;
    const int64_t rt = tile / n_ct, ct = tile % n_ct;
    const int64_t gr = rt * TILE + r, gc = ct * TILE + 8 * c8;
    float v[8];
    if (gr < n && vec && gc + 8 <= m) {
      const float4 a = __ldcs(reinterpret_cast<const float4*>(X + gr * ldx + gc));
      const float4 b = __ldcs(reinterpret_cast<const float4*>(X + gr * ldx + gc + 4));
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = (gr < n && gc + j < m) ? X[gr * ldx + gc + j] : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) nz |= v[j] != 0.f;
    uint32_t hw[4], lw[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
      const float2 f = __bfloat1622float2(h);
      const __nv_bfloat162 l = __floats2bfloat162_rn(v[2 * j] - f.x, v[2 * j + 1] - f.y);
      hw[j] = *reinterpret_cast<const uint32_t*>(&h);
      lw[j] = *reinterpret_cast<const uint32_t*>(&l);
    }
    const int sub = c8 >> 3, ch = c8 & 7;
    const int64_t off = tile * XTILE_BYTES + sub * SUB_BYTES + r * 128 + ((ch ^ (r & 7)) << 4);
    *reinterpret_cast<uint4*>(Xs + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    *reinterpret_cast<uint4*>(Xs + off + 2 * SUB_BYTES) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
  }
  if (nonzero != nullptr && __any_sync(0xffffffffu, nz) && (threadIdx.x & 31) == 0) *nonzero = 1;
}

// Skinny operand S (k x len fp32 row-major) -> per 128-wide K tile:
// [sub0 | sub1], each sub = 2 kpad rows (hi rows 0..kpad, lo rows kpad..2kpad)
// x 128 B, swizzled; rows >= k and columns >= len are zero.
// Both operands of a pass in one launch: items [0, ta) split A, [ta, ta + tb) split B.
__global__ void k_split_skinny(const float* __restrict__ SA, int64_t lenA, int64_t ta, uint8_t* __restrict__ outA,
                               const float* __restrict__ SB, int64_t lenB, int64_t tb, uint8_t* __restrict__ outB,
                               int k, int kpad) {
  for (int64_t ii = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ii < ta + tb;
       ii += (int64_t)gridDim.x * blockDim.x) {
    const bool isA = ii < ta;
    const int64_t i = isA ? ii : ii - ta;
    const float* __restrict__ S = isA ? SA : SB;
    const int64_t len = isA ? lenA : lenB;
    uint8_t* __restrict__ out = isA ? outA : outB;
    const int ch = (int)(i & 7);
    const int64_t rest = i >> 3;
    const int row = (int)(rest % (2 * kpad));
    const int64_t ts = rest / (2 * kpad);  // tile * 2 + sub
    const int sub = (int)(ts & 1);
    const int64_t tile = ts >> 1;
    const int a = row % kpad;
    const bool lo = row >= kpad;
    const int64_t c0 = tile * TILE + sub * 64 + ch * 8;
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float x0 = 0.f, x1 = 0.f;
      if (a < k) {
        if (c0 + 2 * j < len) x0 = S[(int64_t)a * len + c0 + 2 * j];
        if (c0 + 2 * j + 1 < len) x1 = S[(int64_t)a * len + c0 + 2 * j + 1];
      }
      if (lo) {
        x0 -= __bfloat162float(__float2bfloat16_rn(x0));
        x1 -= __bfloat162float(__float2bfloat16_rn(x1));
      }
      const __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
      w[j] = *reinterpret_cast<const uint32_t*>(&h);
    }
    const int64_t off = ts * (int64_t)(2 * kpad) * 128 + row * 128 + ((ch ^ (row & 7)) << 4);
    *reinterpret_cast<uint4*>(out + off) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// NST stages of [X tile | A tile]; NB buffers for the tile row's B tile.
// dbg (development, tools/probe_dual.py): bit 0 skips the MMAs, bit 1 the X copies.
template <int KPAD, int NST, int NB>
__global__ void __launch_bounds__(NWARPS * 32, 1)
k_dual_bulk(const uint8_t* __restrict__ Xs, int64_t n, int64_t m, const uint8_t* __restrict__ A2,
            const uint8_t* __restrict__ B2, int k, Units U, float* __restrict__ Ypart, float* __restrict__ Zpart,
            int dbg) {
  constexpr int SK_SUB = 2 * KPAD * 128;             // skinny sub-tile bytes (hi + lo rows x 128 B)
  constexpr int SK_TILE = 2 * SK_SUB;                // one 128-wide K tile of a skinny operand
  constexpr int STAGE = XTILE_BYTES + SK_TILE;       // X tile | A tile (B: per tile row, below)
  constexpr uint32_t ID_Y = idesc_bf16(KPAD, false), ID_Z = idesc_bf16(KPAD, true);
  constexpr uint32_t LO_OFF = KPAD * 128;            // lo rows of a skinny sub-tile
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* bbuf = smem + (size_t)NST * STAGE;  // [NB][SK_TILE]: B tile of the current (/ next) tile row
  __shared__ __align__(8) uint64_t bar_full[NST], bar_empty[NST], bar_yfull[2], bar_yempty[2], bar_zfull, bar_zempty,
      bar_bfull[NB], bar_bempty[NB];
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, lane = tid & 31;
  const int wid = __shfl_sync(0xffffffffu, tid >> 5, 0);  // warp-uniform for the compiler
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], 1);
    }
    for (int b = 0; b < NB; ++b) {
      mbar_init(&bar_bfull[b], 1);
      mbar_init(&bar_bempty[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar_yfull[b], 1);
      mbar_init(&bar_yempty[b], 128);
    }
    mbar_init(&bar_zfull, 1);
    mbar_init(&bar_zempty, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (wid == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_sh))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // programmatic dependent launch: the slab reduction may be scheduled now
  // (it waits for this grid's completion); this grid's prologue above ran
  // while the skinny-split kernel was finishing
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t tmem = tmem_base_sh;
  // TMEM columns: Y buffers [0, 2 KPAD), Z accumulators [2 KPAD, 2 KPAD + CT KPAD)
  const uint32_t ycol0 = 0, zcol0 = 2 * KPAD;

  if (wid == PROD_WARP) {
    // ------------------------------------------------------------ producer
    // (the whole warp walks the unit; one elected lane issues the copies)
    const bool leader = elect_one();
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the split skinny operands are complete
    const uint64_t pol_x = policy_evict_first(), pol_s = policy_evict_last();
    const bool no_x = (dbg & 2) != 0;
    int t = 0, row_count = 0;
    for (int u = blockIdx.x; u < U.units; u += gridDim.x) {
      int rt0, rt1, ct0, ct1, rc, cb;
      unit_bounds(U, u, rt0, rt1, ct0, ct1, rc, cb);
      for (int rt = rt0; rt < rt1; ++rt, ++row_count) {
        const int rb = row_count % NB;
        mbar_wait(&bar_bempty[rb], ((row_count / NB) & 1) ^ 1);
        if (leader) {
          mbar_expect_tx(&bar_bfull[rb], (uint32_t)SK_TILE);
          bulk_g2s(bbuf + (size_t)rb * SK_TILE, B2 + (int64_t)rt * SK_TILE, SK_TILE, &bar_bfull[rb], pol_s);
        }
        for (int ct = ct0; ct < ct1; ++ct, ++t) {
          const int s = t % NST;
          mbar_wait(&bar_empty[s], ((t / NST) & 1) ^ 1);
          uint8_t* st = smem + (size_t)s * STAGE;
          if (leader) {
            mbar_expect_tx(&bar_full[s], (uint32_t)(no_x ? SK_TILE : STAGE));
            if (!no_x)
              bulk_g2s(st, Xs + ((int64_t)rt * U.n_ct + ct) * XTILE_BYTES, XTILE_BYTES, &bar_full[s], pol_x);
            bulk_g2s(st + XTILE_BYTES, A2 + (int64_t)ct * SK_TILE, SK_TILE, &bar_full[s], pol_s);
          }
        }
      }
    }
  } else if (wid == MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    const bool leader = elect_one();
    const bool no_mma = (dbg & 1) != 0;
    const uint32_t sbase = smem_u32(smem), bbase = smem_u32(bbuf);
    int t = 0, row_count = 0, unit_count = 0;
    for (int u = blockIdx.x; u < U.units; u += gridDim.x, ++unit_count) {
      int rt0, rt1, ct0, ct1, rc, cb;
      unit_bounds(U, u, rt0, rt1, ct0, ct1, rc, cb);
      mbar_wait(&bar_zempty, (unit_count & 1) ^ 1);
      for (int rt = rt0; rt < rt1; ++rt, ++row_count) {
        const int yb = row_count & 1, rb = row_count % NB;
        mbar_wait(&bar_yempty[yb], ((row_count >> 1) & 1) ^ 1);
        mbar_wait(&bar_bfull[rb], (row_count / NB) & 1);
        const uint32_t bk = sdesc_lo(bbase + (uint32_t)rb * SK_TILE, 16);  // B tile, K-major
        const uint32_t dy = tmem + ycol0 + (uint32_t)yb * KPAD;
        for (int ct = ct0; ct < ct1; ++ct, ++t) {
          const int s = t % NST;
          mbar_wait(&bar_full[s], (t / NST) & 1);
          tc_fence_after();
          const uint32_t st = sbase + (uint32_t)s * STAGE;
          const uint32_t xk = sdesc_lo(st, 16);                  // X hi, K-major (Y: K = columns)
          const uint32_t xm = sdesc_lo(st, SUB_BYTES);           // X hi, MN-major (Z: K = rows)
          const uint32_t ak = sdesc_lo(st + XTILE_BYTES, 16);    // A tile, K-major
          const uint32_t dz = tmem + zcol0 + (uint32_t)(ct - ct0) * KPAD;
          const uint32_t acc_y = ct > ct0 ? 1u : 0u, acc_z = rt > rt0 ? 1u : 0u;
          if (leader) {
            if (!no_mma) {
              // Y: K = 128 columns of X = 2 sub-tiles x 4 chunks of 16
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {
                const uint32_t xo = (kk >> 2) * SUB_BYTES + (kk & 3) * 32, so = (kk >> 2) * SK_SUB + (kk & 3) * 32;
                const uint64_t ah = sdesc_at(xk, xo), al = sdesc_at(xk, 2 * SUB_BYTES + xo);
                const uint64_t bh = sdesc_at(ak, so), bl = sdesc_at(ak, so + LO_OFF);
                umma(dy, ah, bh, ID_Y, kk > 0 ? 1u : acc_y);
                umma(dy, ah, bl, ID_Y, 1u);
                umma(dy, al, bh, ID_Y, 1u);
              }
              // Z: K = 128 rows of X = 8 chunks of 16 rows; A is MN-major (LBO = next 64 columns)
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {
                const uint32_t so = (kk >> 2) * SK_SUB + (kk & 3) * 32;
                const uint64_t ah = sdesc_at(xm, kk * 2048), al = sdesc_at(xm, 2 * SUB_BYTES + kk * 2048);
                const uint64_t bh = sdesc_at(bk, so), bl = sdesc_at(bk, so + LO_OFF);
                umma(dz, ah, bh, ID_Z, kk > 0 ? 1u : acc_z);
                umma(dz, ah, bl, ID_Z, 1u);
                umma(dz, al, bh, ID_Z, 1u);
              }
            }
            umma_commit(&bar_empty[s]);
            if (ct == ct1 - 1) {
              umma_commit(&bar_yfull[yb]);
              umma_commit(&bar_bempty[rb]);
              if (rt == rt1 - 1) umma_commit(&bar_zfull);
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (wid >= EPI_WARP0 && wid < EPI_WARP0 + 4) {
    // ------------------------------------------------------------ epilogue
    const int quad = wid & 3;  // TMEM lanes 32 quad .. 32 quad + 31
    const uint32_t lane_base = (uint32_t)(32 * quad) << 16;
    int row_count = 0, unit_count = 0;
    auto emit = [&](uint32_t ta, float* dst, int64_t ld, int64_t idx, bool live) {
#pragma unroll
      for (int h = 0; h < KPAD / 16; ++h) {
        float v[16];
        tmem_ld16(ta + 16 * h, v);
        if (live) {
#pragma unroll
          for (int a = 0; a < 16; ++a)
            if (16 * h + a < k) dst[(int64_t)(16 * h + a) * ld + idx] = v[a];
        }
      }
    };
    for (int u = blockIdx.x; u < U.units; u += gridDim.x, ++unit_count) {
      int rt0, rt1, ct0, ct1, rc, cb;
      unit_bounds(U, u, rt0, rt1, ct0, ct1, rc, cb);
      float* yslab = Ypart + (int64_t)cb * k * n;
      float* zslab = Zpart + (int64_t)rc * k * m;
      for (int rt = rt0; rt < rt1; ++rt, ++row_count) {
        const int yb = row_count & 1;
        mbar_wait(&bar_yfull[yb], (row_count >> 1) & 1);
        tc_fence_after();
        const int64_t row = (int64_t)rt * TILE + 32 * quad + lane;
        emit(tmem + lane_base + ycol0 + (uint32_t)yb * KPAD, yslab, n, row, row < n);
        tc_fence_before();
        mbar_arrive(&bar_yempty[yb]);
      }
      mbar_wait(&bar_zfull, unit_count & 1);
      tc_fence_after();
      for (int ct = ct0; ct < ct1; ++ct) {
        const int64_t col = (int64_t)ct * TILE + 32 * quad + lane;
        emit(tmem + lane_base + zcol0 + (uint32_t)(ct - ct0) * KPAD, zslab, m, col, col < m);
      }
      tc_fence_before();
      mbar_arrive(&bar_zempty);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (wid == MMA_WARP)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// ---------------------------------------------------------------------------
// ||X - U^T V||^2 over the prepared X on the tensor cores (the RRE emit,
// tracing.py:45-57, and the explicit-residual pair of the vanilla tie-break,
// nnls.py:219-227).  Per 128 x 128 tile: P = U[:, rows]^T V[:, cols] by
// tcgen05.mma (BF16x3, fp32 accumulator in TMEM, M = N = 128, K = kpad;
// both operands MN-major: the split skinny tiles of k_split_skinny), then
// the epilogue warps read their row of P from TMEM and of X (hi + lo) from
// the same staged tile and accumulate (x - p)^2 in fp64.  NC = 2: a second
// candidate that differs from the first in ONE operand (W replaces V when
// w_is_v, else U) shares the X tile; its product goes to a second pair of
// TMEM buffers.  The prepared X holds X to 16 significant bits and the
// products carry BF16x3 error (~2^-17 relative); both enter the residual
// norm at second order.
//   warp 0: bulk-copy producer (X tile + U tile + V tile [+ W tile] per stage)
//   warp 1: MMA issuer, TMEM owner (2 buffers x NC accumulators of 128 columns)
//   warps 2-5: epilogue; a stage is free once the MMAs committed AND the
//              epilogue read its X (mbarrier count 1 + 128)
template <int KPAD, int NC>
__global__ void __launch_bounds__(NWARPS * 32, 1)
k_resid_bulk(const uint8_t* __restrict__ Xs, int64_t n, int64_t m, const uint8_t* __restrict__ U2,
             const uint8_t* __restrict__ V2, const uint8_t* __restrict__ W2, int w_is_v, double* __restrict__ part,
             const int* __restrict__ gate) {
  constexpr int SK_SUB = 2 * KPAD * 128;
  constexpr int SK_TILE = 2 * SK_SUB;
  constexpr int STAGE = XTILE_BYTES + (1 + NC) * SK_TILE;  // X tile | U tile | V tile [| W tile]
  constexpr uint32_t LO_OFF = KPAD * 128;
  constexpr uint32_t TCOLS = NC == 1 ? 256 : 512;
  // BF16 x BF16 -> F32, M = N = 128, A and B MN-major
  constexpr uint32_t ID = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(TILE >> 3) << 17) |
                          ((uint32_t)(TILE >> 4) << 24);
  if (gate != nullptr && *gate == 0) return;  // uniform over the grid: nothing allocated yet
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar_full[NSTAGE], bar_empty[NSTAGE], bar_afull[2], bar_aempty[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ double red[33];
  const int tid = threadIdx.x, lane = tid & 31;
  const int wid = __shfl_sync(0xffffffffu, tid >> 5, 0);  // warp-uniform for the compiler
  const int n_ct = (int)((m + TILE - 1) / TILE);
  const int64_t ntiles = (int64_t)((n + TILE - 1) / TILE) * n_ct;
  if (tid == 0) {
    for (int st = 0; st < NSTAGE; ++st) {
      mbar_init(&bar_full[st], 1);
      mbar_init(&bar_empty[st], 1 + 128);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar_afull[b], 1);
      mbar_init(&bar_aempty[b], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (wid == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                 "n"(TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t tmem = tmem_base_sh;
  double acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0.0;
  if (wid == PROD_WARP) {
    const bool leader = elect_one();
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the split operands are complete
    const uint64_t pol_x = policy_evict_first(), pol_s = policy_evict_last();
    int t = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++t) {
      const int rt = (int)(tile / n_ct), ct = (int)(tile % n_ct);
      const int st = t % NSTAGE;
      mbar_wait(&bar_empty[st], ((t / NSTAGE) & 1) ^ 1);
      uint8_t* sp = smem + (size_t)st * STAGE;
      if (leader) {
        mbar_expect_tx(&bar_full[st], (uint32_t)STAGE);
        bulk_g2s(sp, Xs + ((int64_t)rt * n_ct + ct) * XTILE_BYTES, XTILE_BYTES, &bar_full[st], pol_x);
        bulk_g2s(sp + XTILE_BYTES, U2 + (int64_t)rt * SK_TILE, SK_TILE, &bar_full[st], pol_s);
        bulk_g2s(sp + XTILE_BYTES + SK_TILE, V2 + (int64_t)ct * SK_TILE, SK_TILE, &bar_full[st], pol_s);
        if constexpr (NC == 2)
          bulk_g2s(sp + XTILE_BYTES + 2 * SK_TILE, W2 + (int64_t)(w_is_v ? ct : rt) * SK_TILE, SK_TILE, &bar_full[st],
                   pol_s);
      }
    }
  } else if (wid == MMA_WARP) {
    const bool leader = elect_one();
    const uint32_t sbase = smem_u32(smem);
    int t = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++t) {
      const int st = t % NSTAGE, ab = t & 1;
      mbar_wait(&bar_aempty[ab], ((t >> 1) & 1) ^ 1);
      mbar_wait(&bar_full[st], (t / NSTAGE) & 1);
      tc_fence_after();
      const uint32_t sp = sbase + (uint32_t)st * STAGE;
      // skinny tiles, MN-major (LBO = the next 64 of the long dimension)
      const uint32_t u2 = sdesc_lo(sp + XTILE_BYTES, SK_SUB), v2 = sdesc_lo(sp + XTILE_BYTES + SK_TILE, SK_SUB),
                     w2 = sdesc_lo(sp + XTILE_BYTES + 2 * SK_TILE, SK_SUB);
      if (leader) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const uint32_t a = (c == 1 && !w_is_v) ? w2 : u2, b = (c == 1 && w_is_v) ? w2 : v2;
          const uint32_t d = tmem + (uint32_t)(2 * c + ab) * TILE;
#pragma unroll
          for (int kk = 0; kk < KPAD / 16; ++kk) {
            const uint64_t ah = sdesc_at(a, kk * 2048), al = sdesc_at(a, LO_OFF + kk * 2048);
            const uint64_t bh = sdesc_at(b, kk * 2048), bl = sdesc_at(b, LO_OFF + kk * 2048);
            umma(d, ah, bh, ID, kk > 0 ? 1u : 0u);
            umma(d, ah, bl, ID, 1u);
            umma(d, al, bh, ID, 1u);
          }
        }
        umma_commit(&bar_empty[st]);
        umma_commit(&bar_afull[ab]);
      }
      __syncwarp();
    }
  } else if (wid >= EPI_WARP0 && wid < EPI_WARP0 + 4) {
    const int quad = wid & 3;
    const uint32_t lane_base = (uint32_t)(32 * quad) << 16;
    const int r = 32 * quad + lane;  // this thread's row of the tile (TMEM lane)
    int t = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++t) {
      const int st = t % NSTAGE, ab = t & 1;
      const int rt = (int)(tile / n_ct), ct = (int)(tile % n_ct);
      mbar_wait(&bar_full[st], (t / NSTAGE) & 1);  // the X tile (already complete: the MMAs waited on it)
      mbar_wait(&bar_afull[ab], (t >> 1) & 1);
      tc_fence_after();
      const uint32_t sp = smem_u32(smem) + (uint32_t)st * STAGE;
      const bool row_ok = (int64_t)rt * TILE + r < n;
      const int64_t cols = row_ok ? m - (int64_t)ct * TILE : 0;
#pragma unroll
      for (int h = 0; h < 4; ++h) {  // 32 columns at a time, squares summed in fp32 then added in fp64
        float pv[NC][32], sq[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) sq[c] = 0.f;
#pragma unroll
        for (int c = 0; c < NC; ++c) tmem_ld32(tmem + lane_base + (uint32_t)(2 * c + ab) * TILE + 32 * h, pv[c]);
        // X (hi, lo) of this row, columns 32h..32h+31: sub h/2, 16-byte chunks 4(h%2)..4(h%2)+3
        const uint32_t rowp = sp + (h >> 1) * SUB_BYTES + r * 128;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const int chunk = 4 * (h & 1) + q4;
          const int off = (chunk ^ (r & 7)) << 4;
          const uint4 hv = lds128(rowp + off);
          const uint4 lv = lds128(rowp + 2 * SUB_BYTES + off);
          const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w}, lw[4] = {lv.x, lv.y, lv.z, lv.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 hf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hw[q]));
            const float2 lf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&lw[q]));
            const int col = 32 * h + 8 * q4 + 2 * q;
            const float x0 = hf.x + lf.x, x1 = hf.y + lf.y;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              const float d0 = col < cols ? x0 - pv[c][8 * q4 + 2 * q] : 0.f;
              const float d1 = col + 1 < cols ? x1 - pv[c][8 * q4 + 2 * q + 1] : 0.f;
              sq[c] = fmaf(d0, d0, sq[c]);
              sq[c] = fmaf(d1, d1, sq[c]);
            }
          }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] += (double)sq[c];
      }
      tc_fence_before();
      mbar_arrive(&bar_aempty[ab]);
      mbar_arrive(&bar_empty[st]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (wid == MMA_WARP)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS) : "memory");
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const double v = block_sum(acc[c], red);
    if (tid == 0) part[NC * blockIdx.x + c] = v;
  }
}

// fixed-order slab sums of both products in one launch: [0, cy) -> Y, [cy, cy + cz) -> Z
__global__ void k_slabs(const float* __restrict__ py, int ny, int64_t cy, float* __restrict__ oy,
                        const float* __restrict__ pz, int nz, int64_t cz, float* __restrict__ oz) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic launch after the pass kernel
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cy + cz) return;
  const bool isY = i < cy;
  const float* __restrict__ part = isY ? py : pz;
  const int nslab = isY ? ny : nz;
  const int64_t count = isY ? cy : cz, o = isY ? i : i - cy;
  float s = part[o];
  for (int c = 1; c < nslab; ++c) s += part[(int64_t)c * count + o];
  (isY ? oy : oz)[o] = s;
}

// Unit grid: balance tiles per CTA (units are dealt round-robin to the
// persistent CTAs) against the slab traffic of the partial sums.
inline Units choose_units(int64_t n, int64_t m, int64_t k, int ctmax, int sms) {
  static std::mutex mu;
  static std::map<std::tuple<int64_t, int64_t, int64_t, int, int>, Units> cache;
  const auto key = std::make_tuple(n, m, k, ctmax, sms);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  Units best{};
  best.n_rt = (int)cdiv(n, TILE);
  best.n_ct = (int)cdiv(m, TILE);
  double best_cost = 1e300;
  std::vector<double> load;
  for (int n_cb = (int)cdiv(best.n_ct, ctmax); n_cb <= best.n_ct; ++n_cb) {
    for (int n_rc = 1; n_rc <= best.n_rt; ++n_rc) {
      const int units = n_cb * n_rc;
      if (units > 4 * sms) break;
      const int G = units < sms ? units : sms;
      load.assign(G, 0.0);
      for (int u = 0; u < units; ++u) {
        const int rc = u / n_cb, cb = u % n_cb;
        const int64_t rows = (int64_t)(rc + 1) * best.n_rt / n_rc - (int64_t)rc * best.n_rt / n_rc;
        const int64_t cols = (int64_t)(cb + 1) * best.n_ct / n_cb - (int64_t)cb * best.n_ct / n_cb;
        load[u % G] += (double)(rows * cols) + 0.5;  // + per-unit Z drain
      }
      double mx = 0;
      for (double v : load) mx = v > mx ? v : mx;
      // slab bytes (written + read back, mostly L2-resident) per CTA, in tiles of X
      const double slab = (double)((n_cb > 1 ? n_cb * n : 0) + (n_rc > 1 ? n_rc * m : 0)) * k * 4.0 * 2.0;
      const double cost = mx + 0.35 * slab / G / XTILE_BYTES;
      if (cost < best_cost) {
        best_cost = cost;
        best.n_cb = n_cb;
        best.n_rc = n_rc;
        best.units = units;
      }
    }
  }
  std::lock_guard<std::mutex> g(mu);
  cache[key] = best;
  return best;
}

}  // namespace tc

// Measurement hook (bench.py's roofline): while enabled, every k_dual_bulk
// launch is bracketed by CUDA events on its own stream, so the kernel's
// duration is known without the small launches around it.  Debug facility:
// process-wide, guarded by a mutex.
namespace {
std::mutex g_xt_mu;
bool g_xt_on = false;
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_xt_ev;
}  // namespace

bool xpass_timing_begin(cudaEvent_t* e0, cudaEvent_t* e1) {
  std::lock_guard<std::mutex> g(g_xt_mu);
  if (!g_xt_on) return false;
  if (cudaEventCreate(e0) != cudaSuccess || cudaEventCreate(e1) != cudaSuccess) return false;
  g_xt_ev.emplace_back(*e0, *e1);
  return true;
}

bool tc_pass_eligible(int64_t n, int64_t m, int64_t k) {
  if (k < 1 || n < tc::TILE || m < tc::TILE) return false;
  return getenv("NENMF_NO_TC") == nullptr;
}

size_t tc_presplit_bytes(int64_t n, int64_t m) {
  return (size_t)cdiv(n, tc::TILE) * (size_t)cdiv(m, tc::TILE) * tc::XTILE_BYTES;
}

int tc_presplit(const float* X, int64_t n, int64_t m, int64_t ldx, uint8_t* Xs, cudaStream_t s, int* nonzero) {
  using namespace tc;
  const int n_ct = (int)cdiv(m, TILE);
  const int64_t total = cdiv(n, TILE) * n_ct * (int64_t)TILE * 16;
  int sms = sm_count();
  if (sms <= 0) sms = 148;
  k_presplit_x<<<(unsigned)imin(cdiv(total, 256), (int64_t)sms * 8), 256, 0, s>>>(X, n, m, ldx, n_ct, total, Xs,
                                                                                      nonzero);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

static int dual_pass_tc_chunk(Arena& ws, const uint8_t* Xs, int64_t n, int64_t m, const float* At, const float* Bt,
                              int64_t k, float* Yt, float* Zt, cudaStream_t s);

// One pass over a pre-split X (tc_presplit): Yt = At X^T (k x n), Zt = Bt X (k x m).
// k <= 64 reads X once (kpad 16 / 32 / 64: cfg3's p' = 60 and cfg4's 40 run the
// 64-wide instance).  k > 64: the skinny operands are processed in row blocks
// of 64 (short-major storage: a block is a contiguous slice), one X stream per block.
int dual_pass_tc_pre(Arena& ws, const uint8_t* Xs, int64_t n, int64_t m, const float* At, const float* Bt,
                     int64_t k, float* Yt, float* Zt, cudaStream_t s) {
  if (At == nullptr || Bt == nullptr || !tc_pass_eligible(n, m, k)) return NENMF_ERR_UNSUPPORTED;
  static const int64_t kblock = getenv("NENMF_DUAL_K32") != nullptr ? 32 : 64;
  if (k <= kblock) return dual_pass_tc_chunk(ws, Xs, n, m, At, Bt, k, Yt, Zt, s);
  const bool dry = ws.base == nullptr;
  size_t need = 0;
  for (int64_t k0 = 0; k0 < k; k0 += kblock) {
    const int64_t kc = imin(kblock, k - k0);
    Arena a = dry ? Arena(nullptr, 0) : ws;
    NENMF_TRY(dual_pass_tc_chunk(a, Xs, n, m, At + k0 * m, Bt + k0 * n, kc, Yt ? Yt + k0 * n : nullptr,
                                 Zt ? Zt + k0 * m : nullptr, s));
    if (a.used - (dry ? 0 : ws.used) > need) need = a.used - (dry ? 0 : ws.used);
  }
  if (dry) ws.take<char>(need);
  return NENMF_OK;
}

// Shared-memory plan per kpad (227 KB per CTA): stages of [64 KB X tile | A tile] + B buffers.
//   kpad 16: 3 x 72 KB + 1 x  8 KB;  kpad 32: 2 x 80 KB + 2 x 16 KB;  kpad 64: 2 x 96 KB + 1 x 32 KB
template <int KPAD, int NST, int NB>
static int launch_dual(const cudaLaunchConfig_t& base, const uint8_t* Xs, int64_t n, int64_t m, const uint8_t* A2,
                       const uint8_t* B2, int k, const tc::Units& U, float* Yo, float* Zo, int dbg) {
  cudaLaunchConfig_t cfg = base;
  const size_t sk_tile = (size_t)2 * 2 * KPAD * 128;
  cfg.dynamicSmemBytes = NST * (tc::XTILE_BYTES + sk_tile) + NB * sk_tile + 1024;
  NENMF_CUDA_TRY(set_smem(tc::k_dual_bulk<KPAD, NST, NB>, cfg.dynamicSmemBytes));
  NENMF_CUDA_TRY(cudaLaunchKernelEx(&cfg, tc::k_dual_bulk<KPAD, NST, NB>, Xs, n, m, A2, B2, k, U, Yo, Zo, dbg));
  return NENMF_OK;
}

static int dual_pass_tc_chunk(Arena& ws, const uint8_t* Xs, int64_t n, int64_t m, const float* At, const float* Bt,
                              int64_t k, float* Yt, float* Zt, cudaStream_t s) {
  using namespace tc;
  const int kpad = k <= 16 ? 16 : k <= 32 ? 32 : 64;
  const int ctmax = (512 - 2 * kpad) / kpad;
  int sms = sm_count();
  if (sms <= 0) sms = 148;
  const Units U = choose_units(n, m, k, ctmax, sms);
  const int64_t sk_tile = (int64_t)2 * 2 * kpad * 128;
  uint8_t* A2 = ws.take<uint8_t>((size_t)U.n_ct * sk_tile);
  uint8_t* B2 = ws.take<uint8_t>((size_t)U.n_rt * sk_tile);
  float* Ypart = U.n_cb > 1 ? ws.take<float>((size_t)U.n_cb * k * n) : nullptr;
  float* Zpart = U.n_rc > 1 ? ws.take<float>((size_t)U.n_rc * k * m) : nullptr;
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  {
    const int64_t ta = (int64_t)U.n_ct * 2 * 2 * kpad * 8, tb = (int64_t)U.n_rt * 2 * 2 * kpad * 8;
    k_split_skinny<<<(unsigned)imin(cdiv(ta + tb, 256), 2368), 256, 0, s>>>(At, m, ta, A2, Bt, n, tb, B2, (int)k,
                                                                             kpad);
    NENMF_LAUNCH_CHECK();
  }
  const unsigned grid = (unsigned)imin(U.units, sms);
  float* Yo = Ypart ? Ypart : Yt;
  float* Zo = Zpart ? Zpart : Zt;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  const bool timed = xpass_timing_begin(&ev0, &ev1);
  if (timed) cudaEventRecord(ev0, s);
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NWARPS * 32);
  cfg.stream = s;
  cfg.attrs = pdl;
  cfg.numAttrs = 1;
  const char* de = getenv("NENMF_DUAL_DBG");  // development: results invalid when set
  const int dbg = de != nullptr ? atoi(de) : 0;
  if (kpad == 64) NENMF_TRY((launch_dual<64, 2, 1>(cfg, Xs, n, m, A2, B2, (int)k, U, Yo, Zo, dbg)));
  else if (kpad == 32) NENMF_TRY((launch_dual<32, 2, 2>(cfg, Xs, n, m, A2, B2, (int)k, U, Yo, Zo, dbg)));
  else NENMF_TRY((launch_dual<16, 3, 1>(cfg, Xs, n, m, A2, B2, (int)k, U, Yo, Zo, dbg)));
  NENMF_LAUNCH_CHECK();
  if (timed) cudaEventRecord(ev1, s);
  if (Ypart || Zpart) {
    const int64_t cy = Ypart ? k * n : 0, cz = Zpart ? k * m : 0;
    cudaLaunchConfig_t c2 = {};
    c2.gridDim = dim3((unsigned)cdiv(cy + cz, 256));
    c2.blockDim = dim3(256);
    c2.stream = s;
    c2.attrs = pdl;
    c2.numAttrs = 1;
    NENMF_CUDA_TRY(cudaLaunchKernelEx(&c2, k_slabs, (const float*)Ypart, (int)U.n_cb, cy, Yt, (const float*)Zpart,
                                      (int)U.n_rc, cz, Zt));
    NENMF_LAUNCH_CHECK();
  }
  return NENMF_OK;
}

// Stand-alone pass over fp32 X: pre-split into the workspace, then one pass.
// Returns NENMF_ERR_UNSUPPORTED when the shape is outside the fast path (the
// caller then uses the CUDA-core pass).  Needs both operands.
int dual_pass_tc(Arena& ws, const float* X, int64_t n, int64_t m, int64_t ldx, const float* At, const float* Bt,
                 int64_t k, float* Yt, float* Zt, cudaStream_t s) {
  if (At == nullptr || Bt == nullptr || !tc_pass_eligible(n, m, k)) return NENMF_ERR_UNSUPPORTED;
  uint8_t* Xs = ws.take<uint8_t>(tc_presplit_bytes(n, m));
  Arena rest = ws;
  if (ws.base != nullptr && !ws.ok) return NENMF_ERR_WORKSPACE;
  if (ws.base != nullptr) NENMF_TRY(tc_presplit(X, n, m, ldx, Xs, s));
  NENMF_TRY(dual_pass_tc_pre(rest, Xs, n, m, At, Bt, k, Yt, Zt, s));
  ws = rest;
  return NENMF_OK;
}

// ||X - U^T V||^2 over the prepared X (k_resid_bulk): out[0], and with a
// second candidate out[1]: W replaces U (w_side 1) or V (w_side 2); X is
// (n x m), U (k x n), V (k x m) fp32, contiguous.  `gate` (device int, may be
// null): skip everything when zero (the tie-break's returned_best).
// NENMF_ERR_UNSUPPORTED outside k <= 32 / the pass's shapes.
__global__ void k_resid_final(const double* __restrict__ part, int nb, int nc, double* __restrict__ out,
                              const int* __restrict__ gate) {
  if (gate != nullptr && *gate == 0) return;
  __shared__ double red[33];
  for (int c = 0; c < nc; ++c) {
    double a = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) a += part[nc * i + c];
    a = block_sum(a, red);
    if (threadIdx.x == 0) out[c] = a;
    __syncthreads();
  }
}

int resid_tc_pre(Arena& ws, const uint8_t* Xs, int64_t n, int64_t m, const float* U, const float* V, int64_t k,
                 double* out, cudaStream_t s, const float* W, int w_side, const int* gate) {
  using namespace tc;
  if (k < 1 || k > 32 || !tc_pass_eligible(n, m, k) || getenv("NENMF_RESID_NO_TC") != nullptr)
    return NENMF_ERR_UNSUPPORTED;
  const bool pair = w_side != 0;
  const bool w_is_v = w_side == 2;
  const int nc = pair ? 2 : 1;
  const int kpad = k <= 16 ? 16 : 32;
  const int n_rt = (int)cdiv(n, TILE), n_ct = (int)cdiv(m, TILE);
  const int64_t sk_tile = (int64_t)2 * 2 * kpad * 128;
  int sms = sm_count();
  if (sms <= 0) sms = 148;
  const unsigned grid = (unsigned)imin((int64_t)n_rt * n_ct, sms);
  uint8_t* Us = ws.take<uint8_t>((size_t)n_rt * sk_tile);
  uint8_t* Vs = ws.take<uint8_t>((size_t)n_ct * sk_tile);
  uint8_t* Ws = pair ? ws.take<uint8_t>((size_t)(w_is_v ? n_ct : n_rt) * sk_tile) : nullptr;
  double* part = ws.take<double>((size_t)grid * 2);
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  {
    const int64_t ta = (int64_t)n_rt * 2 * 2 * kpad * 8, tb = (int64_t)n_ct * 2 * 2 * kpad * 8;
    k_split_skinny<<<(unsigned)imin(cdiv(ta + tb, 256), 2368), 256, 0, s>>>(U, n, ta, Us, V, m, tb, Vs, (int)k,
                                                                             kpad);
    NENMF_LAUNCH_CHECK();
    if (pair) {
      const int64_t tw = w_is_v ? tb : ta;
      k_split_skinny<<<(unsigned)imin(cdiv(tw, 256), 2368), 256, 0, s>>>(W, w_is_v ? m : n, tw, Ws, W, 0, 0, Ws,
                                                                         (int)k, kpad);
      NENMF_LAUNCH_CHECK();
    }
  }
  const size_t smem = NSTAGE * (XTILE_BYTES + (1 + nc) * (size_t)sk_tile) + 1024;
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NWARPS * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = pdl;
  cfg.numAttrs = 1;
  const int wv = w_is_v ? 1 : 0;
  auto go = [&](auto kern) -> int {
    NENMF_CUDA_TRY(set_smem(kern, smem));
    NENMF_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, Xs, n, m, (const uint8_t*)Us, (const uint8_t*)Vs,
                                      (const uint8_t*)Ws, wv, part, gate));
    return NENMF_OK;
  };
  if (kpad == 32) NENMF_TRY(pair ? go(k_resid_bulk<32, 2>) : go(k_resid_bulk<32, 1>));
  else NENMF_TRY(pair ? go(k_resid_bulk<16, 2>) : go(k_resid_bulk<16, 1>));
  NENMF_LAUNCH_CHECK();
  k_resid_final<<<1, 256, 0, s>>>(part, (int)grid, nc, out, gate);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

}  // namespace nenmf

extern "C" {
void nenmf_debug_xpass_timing(int on) {
  std::lock_guard<std::mutex> g(nenmf::g_xt_mu);
  nenmf::g_xt_on = on != 0;
}

// Total duration (ms) and count of the k_dual_bulk launches timed since the
// last call (waits for them); clears the list.
int nenmf_debug_xpass_ms(double* total_ms) {
  std::lock_guard<std::mutex> g(nenmf::g_xt_mu);
  double tot = 0.0;
  int cnt = 0;
  for (auto& pr : nenmf::g_xt_ev) {
    float ms = 0.f;
    if (cudaEventSynchronize(pr.second) == cudaSuccess && cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) {
      tot += ms;
      ++cnt;
    }
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  nenmf::g_xt_ev.clear();
  if (total_ms != nullptr) *total_ms = tot;
  return cnt;
}
}  // extern "C"
