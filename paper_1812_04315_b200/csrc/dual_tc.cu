// Tensor-core (tcgen05) X-pass for FP32 data: Y^T = A^T X^T and Z^T = B^T X
// from ONE read of X (compression.py:134-139,188), BF16x3 split precision.
//
// Every fp32 element x is split into bf16 hi = rn(x) and lo = rn(x - hi);
// the skinny operands likewise.  Each 128 x 128 tile of X is staged in shared
// memory as hi and lo bf16 tiles in the canonical 128-byte-swizzled layout,
// and the SAME bytes feed both products:
//   Y (rows of X as M, columns as K)  : A = X tile, K-major descriptor
//   Z (columns of X as M, rows as K)  : A = X tile, MN-major descriptor
// Per K-chunk two MMAs per product: [x_hi] x [a_hi | a_lo] (N = 2 kpad) and
// [x_lo] x [a_hi] (N = kpad) into the same TMEM accumulator, so
// x a ~= x_hi a_hi + x_hi a_lo + x_lo a_hi (relative error ~1e-5, fp32-class).
//
// Work: units of (row chunk) x (column block of CT tiles).  Z accumulators of
// the column block live in TMEM for the whole unit; Y accumulators (double
// buffered) for one tile row.  Partial sums per unit are written to global
// slabs and reduced in fixed order (deterministic).
//
// Roles (13 warps): 0-7 producers (global fp32 -> split -> swizzled smem),
// 8 MMA issuer + TMEM owner, 9-12 epilogue (TMEM -> registers -> global).
#include "rsi.cuh"

#include <cuda_bf16.h>

namespace nenmf {

namespace tc {

constexpr int TILE = 128;
constexpr int NPROD = 8;          // producer warps
constexpr int MMA_WARP = 8;
constexpr int EPI_WARP0 = 9;      // epilogue warps 9..12 (TMEM lane quadrant = warp % 4)
constexpr int NWARPS = 13;
constexpr int NSTAGE = 2;
constexpr int SUB_BYTES = TILE * 128;  // one 128-row x 64-col bf16 sub-tile

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

// [hi rows 0..k) | zero | lo rows kpad..kpad+k) | zero], each row ld2 (multiple of 8) bf16
__global__ void k_split_bf16(const float* __restrict__ S, int k, int64_t len, int kpad, int64_t ld2,
                             __nv_bfloat16* __restrict__ out) {
  const int64_t total = (int64_t)2 * kpad * ld2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / ld2, col = i % ld2;
    const int a = (int)(row % kpad);
    const bool lo = row >= kpad;
    float v = 0.f;
    if (a < k && col < len) {
      const float x = S[(int64_t)a * len + col];
      const __nv_bfloat16 h = __float2bfloat16_rn(x);
      v = lo ? (x - __bfloat162float(h)) : x;
    }
    out[i] = __float2bfloat16_rn(v);
  }
}

template <int KPAD>
__global__ void __launch_bounds__(NWARPS * 32, 1)
k_dual_tc(const float* __restrict__ X, int64_t n, int64_t m, int64_t ldx, const __nv_bfloat16* __restrict__ A2,
          int64_t lda2, const __nv_bfloat16* __restrict__ B2, int64_t ldb2, int k, Units U,
          float* __restrict__ Ypart, float* __restrict__ Zpart) {
  constexpr int N2 = 2 * KPAD;                 // [hi | lo] columns
  constexpr int SK_SUB = N2 * 128;             // skinny sub-tile bytes (N2 rows x 128 B)
  constexpr int STAGE = 4 * SUB_BYTES + 4 * SK_SUB;  // Xhi(2 sub) Xlo(2 sub) A2(2 sub) B2(2 sub)
  constexpr uint32_t ID_Y2 = idesc_bf16(N2, false), ID_Y1 = idesc_bf16(KPAD, false);
  constexpr uint32_t ID_Z2 = idesc_bf16(N2, true), ID_Z1 = idesc_bf16(KPAD, true);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar_full[NSTAGE], bar_empty[NSTAGE], bar_yfull[2], bar_yempty[2], bar_zfull,
      bar_zempty;
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&bar_full[s], NPROD * 32);
      mbar_init(&bar_empty[s], 1);
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
  const uint32_t tmem = tmem_base_sh;
  // TMEM columns: Y buffers [0, 2 N2), Z accumulators [2 N2, 2 N2 + CT N2)
  const uint32_t ycol0 = 0, zcol0 = 2 * N2;

  if (wid < NPROD) {
    // ------------------------------------------------------------ producers
    // Each thread owns 16 float4 of every tile.  The loads run one tile ahead
    // in a rolling register queue: slot j is refilled with the next tile's
    // float4 right after it has been split into the current stage, so ~64 KB
    // per SM stay in flight while the producers convert (HBM latency hidden).
    const int ptid = tid;  // 0 .. 255
    constexpr int NQ = TILE * 32 / (NPROD * 32);  // 16 float4 per thread per tile
    int u = blockIdx.x, rt = 0, ct = 0, rt0 = 0, rt1 = 0, ct0 = 0, ct1 = 0, rc_, cb_;
    bool valid = u < U.units;
    if (valid) {
      unit_bounds(U, u, rt0, rt1, ct0, ct1, rc_, cb_);
      rt = rt0;
      ct = ct0;
    }
    auto advance = [&]() {
      if (++ct < ct1) return;
      ct = ct0;
      if (++rt < rt1) return;
      u += gridDim.x;
      valid = u < U.units;
      if (valid) {
        unit_bounds(U, u, rt0, rt1, ct0, ct1, rc_, cb_);
        rt = rt0;
        ct = ct0;
      }
    };
    auto load = [&](int trt, int tct, int j) -> float4 {
      const int q = ptid + j * NPROD * 32;
      const int row = q >> 5, c4 = q & 31;
      const int64_t gr = (int64_t)trt * TILE + row, gc = (int64_t)tct * TILE + 4 * c4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gr < n && gc < m) v = __ldcs(reinterpret_cast<const float4*>(X + gr * ldx + gc));
      return v;
    };
    float4 R[NQ];
    if (valid) {
#pragma unroll
      for (int j = 0; j < NQ; ++j) R[j] = load(rt, ct, j);
    }
    int t = 0;
    while (valid) {
      const int crt = rt, cct = ct;
      advance();  // (rt, ct, valid) now name the next tile
      const int s = t % NSTAGE;
      mbar_wait(&bar_empty[s], ((t / NSTAGE) & 1) ^ 1);
      uint8_t* st = smem + (size_t)s * STAGE;
      uint8_t* xhi = st;
      uint8_t* xlo = st + 2 * SUB_BYTES;
      uint8_t* a2 = st + 4 * SUB_BYTES;
      uint8_t* b2 = a2 + 2 * SK_SUB;
      const int64_t r0 = (int64_t)crt * TILE, c0 = (int64_t)cct * TILE;
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        const float4 v = R[j];
        if (valid) R[j] = load(rt, ct, j);
        const int q = ptid + j * NPROD * 32;
        const int row = q >> 5, c4 = q & 31;
        const __nv_bfloat162 h01 = __floats2bfloat162_rn(v.x, v.y);
        const __nv_bfloat162 h23 = __floats2bfloat162_rn(v.z, v.w);
        const float2 f01 = __bfloat1622float2(h01), f23 = __bfloat1622float2(h23);
        const __nv_bfloat162 l01 = __floats2bfloat162_rn(v.x - f01.x, v.y - f01.y);
        const __nv_bfloat162 l23 = __floats2bfloat162_rn(v.z - f23.x, v.w - f23.y);
        const int sub = c4 >> 4, cc = c4 & 15;
        const uint32_t off = (uint32_t)sub * SUB_BYTES + (uint32_t)row * 128 +
                             ((uint32_t)((cc >> 1) ^ (row & 7)) << 4) + (uint32_t)(cc & 1) * 8;
        uint2 hv, lv;
        hv.x = *reinterpret_cast<const uint32_t*>(&h01);
        hv.y = *reinterpret_cast<const uint32_t*>(&h23);
        lv.x = *reinterpret_cast<const uint32_t*>(&l01);
        lv.y = *reinterpret_cast<const uint32_t*>(&l23);
        *reinterpret_cast<uint2*>(xhi + off) = hv;
        *reinterpret_cast<uint2*>(xlo + off) = lv;
      }
      // skinny tiles: N2 rows x 128 K-elements (bf16) = N2 x 16 chunks of 16 B
      for (int q = ptid; q < N2 * 16; q += NPROD * 32) {
        const int row = q >> 4, ch16 = q & 15, sub = ch16 >> 3, ch = ch16 & 7;
        const uint32_t off = (uint32_t)sub * SK_SUB + (uint32_t)row * 128 + ((uint32_t)(ch ^ (row & 7)) << 4);
        const int64_t ca = c0 + ch16 * 8;
        uint4 va = make_uint4(0, 0, 0, 0), vb = make_uint4(0, 0, 0, 0);
        if (ca < lda2) va = __ldg(reinterpret_cast<const uint4*>(A2 + (int64_t)row * lda2 + ca));
        const int64_t rb = r0 + ch16 * 8;
        if (rb < ldb2) vb = __ldg(reinterpret_cast<const uint4*>(B2 + (int64_t)row * ldb2 + rb));
        *reinterpret_cast<uint4*>(a2 + off) = va;
        *reinterpret_cast<uint4*>(b2 + off) = vb;
      }
      fence_proxy_async();
      mbar_arrive(&bar_full[s]);
      ++t;
    }
  } else if (wid == MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    int t = 0, row_count = 0, unit_count = 0;
    for (int u = blockIdx.x; u < U.units; u += gridDim.x, ++unit_count) {
      int rt0, rt1, ct0, ct1, rc, cb;
      unit_bounds(U, u, rt0, rt1, ct0, ct1, rc, cb);
      if (lane == 0) mbar_wait(&bar_zempty, (unit_count & 1) ^ 1);
      for (int rt = rt0; rt < rt1; ++rt, ++row_count) {
        const int yb = row_count & 1;
        if (lane == 0) mbar_wait(&bar_yempty[yb], ((row_count >> 1) & 1) ^ 1);
        for (int ct = ct0; ct < ct1; ++ct, ++t) {
          const int s = t % NSTAGE;
          if (lane == 0) mbar_wait(&bar_full[s], (t / NSTAGE) & 1);
          __syncwarp();
          tc_fence_after();
          if (lane == 0) {
            const uint32_t st = smem_u32(smem + (size_t)s * STAGE);
            const uint32_t xhi = st, xlo = st + 2 * SUB_BYTES, a2 = st + 4 * SUB_BYTES, b2 = a2 + 2 * SK_SUB;
            const uint32_t dy = tmem + ycol0 + (uint32_t)yb * N2;
            const uint32_t dz = tmem + zcol0 + (uint32_t)(ct - ct0) * N2;
            // Y: K = 128 columns of X = 2 sub-tiles x 4 chunks of 16
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint32_t sub = kk >> 2, koff = (kk & 3) * 32;
              const uint64_t ah = sdesc(xhi + sub * SUB_BYTES + koff, 16, 1024);
              const uint64_t al = sdesc(xlo + sub * SUB_BYTES + koff, 16, 1024);
              const uint64_t bb = sdesc(a2 + sub * SK_SUB + koff, 16, 1024);
              umma(dy, ah, bb, ID_Y2, (ct > ct0 || kk > 0) ? 1u : 0u);
              umma(dy, al, bb, ID_Y1, 1u);
            }
            // Z: K = 128 rows of X = 8 chunks of 16 rows; A is MN-major (LBO = next 64 columns)
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint64_t ah = sdesc(xhi + kk * 2048, SUB_BYTES, 1024);
              const uint64_t al = sdesc(xlo + kk * 2048, SUB_BYTES, 1024);
              const uint64_t bb = sdesc(b2 + (kk >> 2) * SK_SUB + (kk & 3) * 32, 16, 1024);
              umma(dz, ah, bb, ID_Z2, (rt > rt0 || kk > 0) ? 1u : 0u);
              umma(dz, al, bb, ID_Z1, 1u);
            }
            umma_commit(&bar_empty[s]);
            if (ct == ct1 - 1) umma_commit(&bar_yfull[yb]);
            if (ct == ct1 - 1 && rt == rt1 - 1) umma_commit(&bar_zfull);
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
    // hi and lo halves of an accumulator row, 16 columns at a time (keeps the
    // epilogue at 32 live registers)
    auto emit = [&](uint32_t ta, float* dst, int64_t ld, int64_t idx, bool live) {
#pragma unroll
      for (int h = 0; h < KPAD / 16; ++h) {
        float vh[16], vl[16];
        tmem_ld16(ta + 16 * h, vh);
        tmem_ld16(ta + KPAD + 16 * h, vl);
        if (live) {
#pragma unroll
          for (int a = 0; a < 16; ++a)
            if (16 * h + a < k) dst[(int64_t)(16 * h + a) * ld + idx] = vh[a] + vl[a];
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
        emit(tmem + lane_base + ycol0 + (uint32_t)yb * N2, yslab, n, row, row < n);
        tc_fence_before();
        mbar_arrive(&bar_yempty[yb]);
      }
      mbar_wait(&bar_zfull, unit_count & 1);
      tc_fence_after();
      for (int ct = ct0; ct < ct1; ++ct) {
        const int64_t col = (int64_t)ct * TILE + 32 * quad + lane;
        emit(tmem + lane_base + zcol0 + (uint32_t)(ct - ct0) * N2, zslab, m, col, col < m);
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

__global__ void k_slabs(const float* __restrict__ part, int nslab, int64_t count, float* __restrict__ out) {
  int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= count) return;
  float s = part[o];
  for (int c = 1; c < nslab; ++c) s += part[(int64_t)c * count + o];
  out[o] = s;
}

}  // namespace tc

// Returns NENMF_ERR_UNSUPPORTED when the shape is outside the fast path
// (the caller then uses the CUDA-core pass).  Needs both operands.
int dual_pass_tc(Arena& ws, const float* X, int64_t n, int64_t m, int64_t ldx, const float* At, const float* Bt,
                 int64_t k, float* Yt, float* Zt, cudaStream_t s) {
  using namespace tc;
  if (At == nullptr || Bt == nullptr || k < 1 || k > 32) return NENMF_ERR_UNSUPPORTED;
  if (m % 4 != 0 || ldx % 4 != 0 || n < TILE || m < TILE) return NENMF_ERR_UNSUPPORTED;
  if (getenv("NENMF_NO_TC") != nullptr) return NENMF_ERR_UNSUPPORTED;
  const int kpad = k <= 16 ? 16 : 32;
  const int ctmax = (512 - 4 * kpad) / (2 * kpad);
  int sms = sm_count();
  if (sms <= 0) sms = 148;
  Units U;
  U.n_rt = (int)cdiv(n, TILE);
  U.n_ct = (int)cdiv(m, TILE);
  U.n_cb = (int)cdiv(U.n_ct, ctmax);
  U.n_rc = (int)imax(1, imin(U.n_rt, sms / imax(1, U.n_cb)));
  U.units = U.n_cb * U.n_rc;
  const int64_t lda2 = cdiv(m, 8) * 8, ldb2 = cdiv(n, 8) * 8;
  __nv_bfloat16* A2 = ws.take<__nv_bfloat16>((size_t)2 * kpad * lda2);
  __nv_bfloat16* B2 = ws.take<__nv_bfloat16>((size_t)2 * kpad * ldb2);
  float* Ypart = U.n_cb > 1 ? ws.take<float>((size_t)U.n_cb * k * n) : nullptr;
  float* Zpart = U.n_rc > 1 ? ws.take<float>((size_t)U.n_rc * k * m) : nullptr;
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  k_split_bf16<<<(unsigned)imin(1184, cdiv(2 * kpad * lda2, 256)), 256, 0, s>>>(At, (int)k, m, kpad, lda2, A2);
  NENMF_LAUNCH_CHECK();
  k_split_bf16<<<(unsigned)imin(1184, cdiv(2 * kpad * ldb2, 256)), 256, 0, s>>>(Bt, (int)k, n, kpad, ldb2, B2);
  NENMF_LAUNCH_CHECK();
  const size_t stage = 4 * SUB_BYTES + 4 * (size_t)(2 * kpad) * 128;
  const size_t smem = NSTAGE * stage + 1024;
  const unsigned grid = (unsigned)imin(U.units, sms);
  if (kpad == 32) {
    NENMF_CUDA_TRY(set_smem(k_dual_tc<32>, smem));
    k_dual_tc<32><<<grid, NWARPS * 32, smem, s>>>(X, n, m, ldx, A2, lda2, B2, ldb2, (int)k, U, Ypart ? Ypart : Yt,
                                                 Zpart ? Zpart : Zt);
  } else {
    NENMF_CUDA_TRY(set_smem(k_dual_tc<16>, smem));
    k_dual_tc<16><<<grid, NWARPS * 32, smem, s>>>(X, n, m, ldx, A2, lda2, B2, ldb2, (int)k, U, Ypart ? Ypart : Yt,
                                                 Zpart ? Zpart : Zt);
  }
  NENMF_LAUNCH_CHECK();
  if (Ypart) {
    k_slabs<<<(unsigned)cdiv(k * n, 256), 256, 0, s>>>(Ypart, U.n_cb, k * n, Yt);
    NENMF_LAUNCH_CHECK();
  }
  if (Zpart) {
    k_slabs<<<(unsigned)cdiv(k * m, 256), 256, 0, s>>>(Zpart, U.n_rc, k * m, Zt);
    NENMF_LAUNCH_CHECK();
  }
  return NENMF_OK;
}

}  // namespace nenmf
