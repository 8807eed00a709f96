// Skinny products and fixed-order reductions (CUDA cores, sm_100a).
//
//   abt      C = A B^T, long K            F @ R, L @ G, Gram A^T A (factorize.py:110,113; nnls.py:157)
//   ab       V = At B (B or B^T view)     A.T @ B                   (nnls.py:158)
//   resid    sum (At^T F - B)^2, 1-2 F's  _true_objective, emit     (nnls.py:115-116,225; factorize.py:139)
//   sumsq    sum M^2                      frobenius_norm            (matrix.py:177-179)
//   pg_sumsq sum PG(F,g)^2                projected_gradient_norm   (nnls.py:89-107)
//   wfv      W F - V                      gradient (Gram form)      (nnls.py:72-86)
//
// Every reduction is deterministic: K is cut into chunks whose size depends
// only on the shape, each output is one sequential FMA chain per chunk, and
// chunk partials are added in chunk order.  Two calls with the same shapes
// therefore perform bit-identical arithmetic whatever the memory layout of B
// -- which is what makes identity-sketch compressed NeNMF reproduce vanilla
// NeNMF exactly (reference test_factorize.py:161-176).
#include "skinny.cuh"

#include <cstdlib>
#include <utility>

namespace nenmf {

// ----------------------------------------------------------------- abt ----
constexpr int ABT_KT = 32;
constexpr int64_t ABT_KCHUNK = 128;
constexpr int ABT_THREADS = 256;
constexpr int ABT_MAXO = 32;  // outputs per thread: p*q <= 8192

template <typename T, typename TO>
__global__ void __launch_bounds__(ABT_THREADS)
k_abt(const T* __restrict__ A, int p, const T* __restrict__ B, int q, int64_t K,
      int64_t kchunk, double* __restrict__ part, TO* __restrict__ C) {
  extern __shared__ double smem_d[];
  double* As = smem_d;                       // [p][KT+1]
  double* Bs = smem_d + p * (ABT_KT + 1);    // [q][KT+1]
  const int tid = threadIdx.x;
  const int64_t k0 = blockIdx.x * kchunk;
  const int64_t k1 = min(K, k0 + kchunk);
  const int npq = p * q;
  double acc[ABT_MAXO];
#pragma unroll
  for (int s = 0; s < ABT_MAXO; ++s) acc[s] = 0.0;

  for (int64_t kt = k0; kt < k1; kt += ABT_KT) {
    const int nk = (int)imin(ABT_KT, k1 - kt);
    for (int idx = tid; idx < p * ABT_KT; idx += blockDim.x) {
      int a = idx / ABT_KT, kk = idx % ABT_KT;
      As[a * (ABT_KT + 1) + kk] = kk < nk ? (double)A[(int64_t)a * K + kt + kk] : 0.0;
    }
    for (int idx = tid; idx < q * ABT_KT; idx += blockDim.x) {
      int b = idx / ABT_KT, kk = idx % ABT_KT;
      Bs[b * (ABT_KT + 1) + kk] = kk < nk ? (double)B[(int64_t)b * K + kt + kk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < ABT_MAXO; ++s) {
      int o = tid + s * ABT_THREADS;
      if (o < npq) {
        const double* ar = As + (o / q) * (ABT_KT + 1);
        const double* br = Bs + (o % q) * (ABT_KT + 1);
        double a = acc[s];
        for (int kk = 0; kk < nk; ++kk) a = fma(ar[kk], br[kk], a);
        acc[s] = a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int s = 0; s < ABT_MAXO; ++s) {
    int o = tid + s * ABT_THREADS;
    if (o < npq) {
      if (C != nullptr) C[o] = (TO)acc[s];
      else part[(int64_t)blockIdx.x * npq + o] = acc[s];
    }
  }
}

template <typename TO>
__global__ void k_abt_reduce(const double* __restrict__ part, int nchunk, int npq, TO* __restrict__ C) {
  int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= npq) return;
  double s = part[o];
  for (int c = 1; c < nchunk; ++c) s += part[(int64_t)c * npq + o];
  C[o] = (TO)s;
}

template <typename T, typename TO>
int abt_any(Arena& ws, const T* A, int64_t p, const T* B, int64_t q, int64_t K, TO* C, cudaStream_t st) {
  if (p < 1 || q < 1 || K < 1) return NENMF_ERR_DIM;
  if (p * q > ABT_THREADS * ABT_MAXO || p > 512 || q > 512) return NENMF_ERR_UNSUPPORTED;
  const int64_t nchunk = cdiv(K, ABT_KCHUNK);
  double* part = nchunk > 1 ? ws.take<double>((size_t)nchunk * p * q) : nullptr;
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  size_t smem = (size_t)(p + q) * (ABT_KT + 1) * sizeof(double);
  NENMF_CUDA_TRY(cudaFuncSetAttribute(k_abt<T, TO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_abt<T, TO><<<(unsigned)nchunk, ABT_THREADS, smem, st>>>(A, (int)p, B, (int)q, K, ABT_KCHUNK, part,
                                                           nchunk > 1 ? nullptr : C);
  NENMF_LAUNCH_CHECK();
  if (nchunk > 1) {
    int npq = (int)(p * q);
    k_abt_reduce<TO><<<(unsigned)cdiv(npq, 256), 256, 0, st>>>(part, (int)nchunk, npq, C);
    NENMF_LAUNCH_CHECK();
  }
  return NENMF_OK;
}

template <typename T>
int abt(Arena& ws, const T* A, int64_t p, const T* B, int64_t q, int64_t K, T* C, cudaStream_t st) {
  // more outputs than one launch holds (p q > 8192: inner dimensions p or nu above 64): row
  // blocks of A, whose output rows are contiguous in C
  if (p >= 1 && q >= 1 && q <= 512 && p * q > (int64_t)ABT_THREADS * ABT_MAXO) {
    const int64_t pb = imax(1, (int64_t)ABT_THREADS * ABT_MAXO / q);
    const bool dry = ws.base == nullptr;
    size_t need = 0;
    for (int64_t p0 = 0; p0 < p; p0 += pb) {
      Arena a = ws;
      NENMF_TRY((abt_any<T, T>(a, dry ? A : A + p0 * K, imin(pb, p - p0), B, q, K, dry ? C : C + p0 * q, st)));
      if (a.used - ws.used > need) need = a.used - ws.used;
      if (!dry && !a.ok) return NENMF_ERR_WORKSPACE;
    }
    if (dry) ws.take<char>(need);
    return NENMF_OK;
  }
  return abt_any<T, T>(ws, A, p, B, q, K, C, st);
}

template <typename T>
int gram_d(Arena& ws, const T* A, int64_t p, int64_t K, double* G, cudaStream_t st) {
  return abt_any<T, double>(ws, A, p, A, p, K, G, st);
}

// ------------------------------------------------------------------ ab ----
constexpr int AB_CB = 64;        // output columns per CTA
constexpr int AB_RT = 32;        // K rows per smem tile
constexpr int64_t AB_RCHUNK = 1024;
constexpr int AB_THREADS = 256;  // 64 columns x 4 row groups of p
constexpr int AB_MAXA = 16;      // p <= 64

template <typename T, bool TRANS>
__device__ __forceinline__ void load_b_tile(T* Bs, const T* __restrict__ B, int64_t ldb, int64_t r,
                                            int64_t c, int64_t t0, int nt, int64_t j0) {
  // Bs[tt][jj] = B(t0+tt, j0+jj); B(t, j) = TRANS ? Bsrc[j*ldb + t] : Bsrc[t*ldb + j]
  if (!TRANS) {
    for (int idx = threadIdx.x; idx < AB_RT * AB_CB; idx += blockDim.x) {
      int tt = idx / AB_CB, jj = idx % AB_CB;
      int64_t j = j0 + jj;
      Bs[tt * (AB_CB + 1) + jj] = (tt < nt && j < c) ? B[(t0 + tt) * ldb + j] : T(0);
    }
  } else {
    for (int idx = threadIdx.x; idx < AB_RT * AB_CB; idx += blockDim.x) {
      int jj = idx / AB_RT, tt = idx % AB_RT;
      int64_t j = j0 + jj;
      Bs[tt * (AB_CB + 1) + jj] = (tt < nt && j < c) ? B[j * ldb + t0 + tt] : T(0);
    }
  }
}

template <typename T>
__device__ __forceinline__ void load_at_tile(T* Ats, const T* __restrict__ At, int p, int64_t r,
                                             int64_t t0, int nt) {
  for (int idx = threadIdx.x; idx < p * AB_RT; idx += blockDim.x) {
    int a = idx / AB_RT, tt = idx % AB_RT;
    Ats[a * (AB_RT + 1) + tt] = tt < nt ? At[(int64_t)a * r + t0 + tt] : T(0);
  }
}

template <typename T, bool TRANS>
__global__ void __launch_bounds__(AB_THREADS)
k_ab(const T* __restrict__ At, int p, int64_t r, const T* __restrict__ B, int64_t c, int64_t ldb,
     int64_t rchunk, T* __restrict__ part, T* __restrict__ V) {
  extern __shared__ double smem_d[];
  T* Bs = reinterpret_cast<T*>(smem_d);            // [RT][CB+1]
  T* Ats = Bs + AB_RT * (AB_CB + 1);               // [p][RT+1]
  const int jj = threadIdx.x % AB_CB, g = threadIdx.x / AB_CB;
  const int64_t j0 = (int64_t)blockIdx.x * AB_CB;
  const int64_t tc0 = (int64_t)blockIdx.y * rchunk, tc1 = min(r, tc0 + rchunk);
  T acc[AB_MAXA];
#pragma unroll
  for (int s = 0; s < AB_MAXA; ++s) acc[s] = T(0);
  for (int64_t t0 = tc0; t0 < tc1; t0 += AB_RT) {
    const int nt = (int)imin(AB_RT, tc1 - t0);
    load_b_tile<T, TRANS>(Bs, B, ldb, r, c, t0, nt, j0);
    load_at_tile<T>(Ats, At, p, r, t0, nt);
    __syncthreads();
    for (int tt = 0; tt < nt; ++tt) {
      const T b = Bs[tt * (AB_CB + 1) + jj];
#pragma unroll
      for (int s = 0; s < AB_MAXA; ++s) {
        int a = g + 4 * s;
        if (a < p) acc[s] = fma_acc(Ats[a * (AB_RT + 1) + tt], b, acc[s]);
      }
    }
    __syncthreads();
  }
  const int64_t j = j0 + jj;
  if (j >= c) return;
#pragma unroll
  for (int s = 0; s < AB_MAXA; ++s) {
    int a = g + 4 * s;
    if (a < p) {
      if (V != nullptr) V[(int64_t)a * c + j] = acc[s];
      else part[((int64_t)blockIdx.y * p + a) * c + j] = acc[s];
    }
  }
}

template <typename T>
__global__ void k_chunk_reduce(const T* __restrict__ part, int nchunk, int64_t count, T* __restrict__ out) {
  int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= count) return;
  T s = part[o];
  for (int c = 1; c < nchunk; ++c) s += part[(int64_t)c * count + o];
  out[o] = s;
}

__device__ __forceinline__ void mma_tf32_r(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t tf_hi(float x) { return __float_as_uint(x) & 0xffffe000u; }
__device__ __forceinline__ uint32_t tf_lo(float x) { return __float_as_uint(x - __uint_as_float(tf_hi(x))); }

// ---------------------------------------------------------------------------
// FP32 V = A^T B on the tensor pipe (3xTF32 m16n8k8), X streamed through a
// 3-stage cp.async ring, fixed-order partial sums (deterministic).
//   k_ux  ("Z side", B = X):    out (p x mx) = U (p x nx) X (nx x mx); units =
//         (64-column band, row chunk); a warp owns 16 rows of each 128-row
//         tile and accumulates the band's p x 64 partial in registers; the 8
//         warps are summed in order at the end of the unit.
//   k_xv  ("Y side", B = X^T):  out (p x nx) = V (p x mx) X^T; units =
//         (128-row band, column chunk); a warp owns 16 rows and accumulates
//         its 16 x p block over the chunk's 64-column tiles.
// Partials of the chunks go to slabs summed by k_chunk_reduce (chunk order).
constexpr int VP_NS = 3, VP_XS = 72, VP_US = 136, VP_VS = 72;

template <int MT>  // MT = m16 tiles of p (p <= 16 MT)
__global__ void __launch_bounds__(256, 1)
k_ux(const float* __restrict__ X, int64_t nx, int64_t mx, int64_t ldx, const float* __restrict__ U, int p,
     int64_t nbands, int64_t rchunk, int64_t nunits, float* __restrict__ slab) {
  constexpr int KP = 16 * MT;
  constexpr int XB = 128 * VP_XS, UB = KP * VP_US, SF = XB + UB;
  extern __shared__ __align__(16) float vsm[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, gq = lane >> 2, tq = lane & 3;
  float* red = vsm + VP_NS * SF;  // [KP][64] cross-warp sums
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int64_t cb = u % nbands, rc = u / nbands;
    const int64_t j0 = cb * 64, r0 = rc * rchunk, r1 = imin(nx, r0 + rchunk);
    const int ntl = (int)((r1 - r0 + 127) / 128);
    auto issue = [&](int t, int stg) {
      float* xs = vsm + stg * SF;
      float* us = xs + XB;
      const int64_t i0 = r0 + (int64_t)t * 128;
      for (int c = tid; c < 128 * 16; c += 256) {
        const int r = c >> 4, ch = c & 15;
        const int64_t i = i0 + r, j = j0 + 4 * ch;
        const int valid = (i < r1) ? (int)imax(0, imin(4, mx - j)) : 0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(xs + r * VP_XS + 4 * ch)),
                     "l"(X + (valid ? i * ldx + j : 0)), "r"(4 * valid)
                     : "memory");
      }
      for (int c = tid; c < KP * 32; c += 256) {
        const int a = c >> 5, ch = c & 31;
        const int64_t i = i0 + 4 * ch;
        const int valid = a < p ? (int)imax(0, imin(4, r1 - i)) : 0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(us + a * VP_US + 4 * ch)),
                     "l"(U + (valid ? (int64_t)a * nx + i : 0)), "r"(4 * valid)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    float acc[MT][8][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[mt][nt][q] = 0.f;
    __syncthreads();  // the ring is free (previous unit done)
    for (int i = 0; i < VP_NS - 1; ++i) {
      if (i < ntl) issue(i, i);
      else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int t = 0; t < ntl; ++t) {
      asm volatile("cp.async.wait_group %0;" ::"n"(VP_NS - 2) : "memory");
      __syncthreads();
      const float* xs = vsm + (t % VP_NS) * SF;
      const float* us = xs + XB;
#pragma unroll
      for (int kt = 0; kt < 2; ++kt) {
        const int ib = 16 * wid + 8 * kt;  // 8 rows of the tile (K)
        uint32_t ah[MT][4], al[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float v = us[(16 * mt + gq + ((q & 1) ? 8 : 0)) * VP_US + ib + tq + ((q & 2) ? 4 : 0)];
            ah[mt][q] = tf_hi(v);
            al[mt][q] = tf_lo(v);
          }
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          const float b0 = xs[(ib + tq) * VP_XS + 8 * nt + gq], b1 = xs[(ib + tq + 4) * VP_XS + 8 * nt + gq];
          const uint32_t b0h = tf_hi(b0), b1h = tf_hi(b1), b0l = tf_lo(b0), b1l = tf_lo(b1);
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            mma_tf32_r(acc[mt][nt], al[mt], b0h, b1h);
            mma_tf32_r(acc[mt][nt], ah[mt], b0l, b1l);
            mma_tf32_r(acc[mt][nt], ah[mt], b0h, b1h);
          }
        }
      }
      __syncthreads();
      if (t + VP_NS - 1 < ntl) issue(t + VP_NS - 1, (t + VP_NS - 1) % VP_NS);
      else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    // warps summed in order: C (a, j): rows gq / gq+8 of m-tile mt, columns 2tq, 2tq+1 of n-tile nt
    for (int w = 0; w < 8; ++w) {
      __syncthreads();
      if (wid == w) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < 8; ++nt)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int a = 16 * mt + gq + ((q & 2) ? 8 : 0), j = 8 * nt + 2 * tq + (q & 1);
              red[a * 64 + j] = (w == 0 ? 0.f : red[a * 64 + j]) + acc[mt][nt][q];
            }
      }
    }
    __syncthreads();
    for (int e = tid; e < p * 64; e += 256) {
      const int a = e >> 6, j = e & 63;
      if (j0 + j < mx) slab[(rc * p + a) * mx + j0 + j] = red[a * 64 + j];
    }
  }
}

template <int NTP>  // NTP = n8 tiles of p (p <= 8 NTP)
__global__ void __launch_bounds__(256, 1)
k_xv(const float* __restrict__ X, int64_t nx, int64_t mx, int64_t ldx, const float* __restrict__ V, int p,
     int64_t nbands, int64_t cchunk, int64_t nunits, float* __restrict__ slab) {
  constexpr int KP = 8 * NTP;
  constexpr int XB = 128 * VP_XS, VB = KP * VP_VS, SF = XB + VB;
  extern __shared__ __align__(16) float vsm[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, gq = lane >> 2, tq = lane & 3;
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int64_t rb = u % nbands, cc = u / nbands;
    const int64_t i0 = rb * 128, c0 = cc * cchunk, c1 = imin(mx, c0 + cchunk);
    const int ntl = (int)((c1 - c0 + 63) / 64);
    auto issue = [&](int t, int stg) {
      float* xs = vsm + stg * SF;
      float* vs = xs + XB;
      const int64_t j0 = c0 + (int64_t)t * 64;
      for (int c = tid; c < 128 * 16; c += 256) {
        const int r = c >> 4, ch = c & 15;
        const int64_t i = i0 + r, j = j0 + 4 * ch;
        const int valid = (i < nx) ? (int)imax(0, imin(4, c1 - j)) : 0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(xs + r * VP_XS + 4 * ch)),
                     "l"(X + (valid ? i * ldx + j : 0)), "r"(4 * valid)
                     : "memory");
      }
      for (int c = tid; c < KP * 16; c += 256) {
        const int a = c >> 4, ch = c & 15;
        const int64_t j = j0 + 4 * ch;
        const int valid = a < p ? (int)imax(0, imin(4, c1 - j)) : 0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(vs + a * VP_VS + 4 * ch)),
                     "l"(V + (valid ? (int64_t)a * mx + j : 0)), "r"(4 * valid)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    float acc[NTP][4];
#pragma unroll
    for (int nt = 0; nt < NTP; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[nt][q] = 0.f;
    __syncthreads();
    for (int i = 0; i < VP_NS - 1; ++i) {
      if (i < ntl) issue(i, i);
      else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int t = 0; t < ntl; ++t) {
      asm volatile("cp.async.wait_group %0;" ::"n"(VP_NS - 2) : "memory");
      __syncthreads();
      const float* xs = vsm + (t % VP_NS) * SF;
      const float* vs = xs + XB;
      const int rw = 16 * wid;
#pragma unroll
      for (int kt = 0; kt < 8; ++kt) {
        uint32_t ah[4], al[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float v = xs[(rw + gq + ((q & 1) ? 8 : 0)) * VP_XS + 8 * kt + tq + ((q & 2) ? 4 : 0)];
          ah[q] = tf_hi(v);
          al[q] = tf_lo(v);
        }
#pragma unroll
        for (int nt = 0; nt < NTP; ++nt) {
          const float b0 = vs[(8 * nt + gq) * VP_VS + 8 * kt + tq], b1 = vs[(8 * nt + gq) * VP_VS + 8 * kt + tq + 4];
          const uint32_t b0h = tf_hi(b0), b1h = tf_hi(b1), b0l = tf_lo(b0), b1l = tf_lo(b1);
          mma_tf32_r(acc[nt], al, b0h, b1h);
          mma_tf32_r(acc[nt], ah, b0l, b1l);
          mma_tf32_r(acc[nt], ah, b0h, b1h);
        }
      }
      __syncthreads();
      if (t + VP_NS - 1 < ntl) issue(t + VP_NS - 1, (t + VP_NS - 1) % VP_NS);
      else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    // C (row, a): rows gq / gq+8 of the warp's 16, a = 8 nt + 2 tq (+1)
#pragma unroll
    for (int nt = 0; nt < NTP; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int a = 8 * nt + 2 * tq + (q & 1);
        const int64_t i = i0 + 16 * wid + gq + ((q & 2) ? 8 : 0);
        if (a < p && i < nx) slab[(cc * p + a) * nx + i] = acc[nt][q];
      }
  }
}

// ---------------------------------------------------------------------------
// FP64 V = A^T B on the FP64 tensor pipe (DMMA m8n8k4: exact fp64 products),
// the same unit structure as k_ux / k_xv with 64 x 64 tiles of X.
//   k_ux64: warp w owns columns 8w..8w+7 of the band and all 64 rows of each
//           tile (16 k-steps): acc = 4 m-tiles of p x 8 columns
//   k_xv64: warp w owns rows 8w..8w+7 of the band: acc = 8 rows x p
__device__ __forceinline__ void dmma_r(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}
constexpr int VD_NS = 3, VD_XS = 68, VD_OS = 68;  // row strides (doubles)

__global__ void __launch_bounds__(256, 1)
k_ux64(const double* __restrict__ X, int64_t nx, int64_t mx, int64_t ldx, const double* __restrict__ U, int p,
       int64_t nbands, int64_t rchunk, int64_t nunits, double* __restrict__ slab) {
  constexpr int XB = 64 * VD_XS, UB = 32 * VD_OS, SF = XB + UB;
  extern __shared__ __align__(16) double dsm[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, gq = lane >> 2, tq = lane & 3;
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int64_t cb = u % nbands, rc = u / nbands;
    const int64_t j0 = cb * 64, r0 = rc * rchunk, r1 = imin(nx, r0 + rchunk);
    const int ntl = (int)((r1 - r0 + 63) / 64);
    auto issue = [&](int t, int stg) {
      double* xs = dsm + stg * SF;
      double* us = xs + XB;
      const int64_t i0 = r0 + (int64_t)t * 64;
      for (int c = tid; c < 64 * 32; c += 256) {  // 64 rows x 32 chunks of 2 doubles
        const int r = c >> 5, ch = c & 31;
        const int64_t i = i0 + r, j = j0 + 2 * ch;
        const int valid = (i < r1) ? (int)imax(0, imin(2, mx - j)) : 0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(xs + r * VD_XS + 2 * ch)),
                     "l"(X + (valid ? i * ldx + j : 0)), "r"(8 * valid)
                     : "memory");
      }
      for (int c = tid; c < 32 * 32; c += 256) {  // U slice: 32 rows (a) x 64 (i)
        const int a = c >> 5, ch = c & 31;
        const int64_t i = i0 + 2 * ch;
        const int valid = a < p ? (int)imax(0, imin(2, r1 - i)) : 0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(us + a * VD_OS + 2 * ch)),
                     "l"(U + (valid ? (int64_t)a * nx + i : 0)), "r"(8 * valid)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double acc[4][2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
    __syncthreads();
    for (int i = 0; i < VD_NS - 1; ++i) {
      if (i < ntl) issue(i, i);
      else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int t = 0; t < ntl; ++t) {
      asm volatile("cp.async.wait_group %0;" ::"n"(VD_NS - 2) : "memory");
      __syncthreads();
      const double* xs = dsm + (t % VD_NS) * SF;
      const double* us = xs + XB;
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) {
        const double b = xs[(4 * ks + tq) * VD_XS + 8 * wid + gq];  // B (k = row, n = column)
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
          if (8 * mt < p) dmma_r(acc[mt], us[(8 * mt + gq) * VD_OS + 4 * ks + tq], b);
      }
      __syncthreads();
      if (t + VD_NS - 1 < ntl) issue(t + VD_NS - 1, (t + VD_NS - 1) % VD_NS);
      else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    // C (a, j): a = 8 mt + gq, j = 8 w + 2 tq (+1)
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = 8 * mt + gq;
        const int64_t j = j0 + 8 * wid + 2 * tq + h;
        if (a < p && j < mx) slab[(rc * p + a) * mx + j] = acc[mt][h];
      }
  }
}

__global__ void __launch_bounds__(256, 1)
k_xv64(const double* __restrict__ X, int64_t nx, int64_t mx, int64_t ldx, const double* __restrict__ V, int p,
       int64_t nbands, int64_t cchunk, int64_t nunits, double* __restrict__ slab) {
  constexpr int XB = 64 * VD_XS, VB = 32 * VD_OS, SF = XB + VB;
  extern __shared__ __align__(16) double dsm[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, gq = lane >> 2, tq = lane & 3;
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int64_t rb = u % nbands, cc = u / nbands;
    const int64_t i0 = rb * 64, c0 = cc * cchunk, c1 = imin(mx, c0 + cchunk);
    const int ntl = (int)((c1 - c0 + 63) / 64);
    auto issue = [&](int t, int stg) {
      double* xs = dsm + stg * SF;
      double* vs = xs + XB;
      const int64_t j0 = c0 + (int64_t)t * 64;
      for (int c = tid; c < 64 * 32; c += 256) {
        const int r = c >> 5, ch = c & 31;
        const int64_t i = i0 + r, j = j0 + 2 * ch;
        const int valid = (i < nx) ? (int)imax(0, imin(2, c1 - j)) : 0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(xs + r * VD_XS + 2 * ch)),
                     "l"(X + (valid ? i * ldx + j : 0)), "r"(8 * valid)
                     : "memory");
      }
      for (int c = tid; c < 32 * 32; c += 256) {
        const int a = c >> 5, ch = c & 31;
        const int64_t j = j0 + 2 * ch;
        const int valid = a < p ? (int)imax(0, imin(2, c1 - j)) : 0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(vs + a * VD_OS + 2 * ch)),
                     "l"(V + (valid ? (int64_t)a * mx + j : 0)), "r"(8 * valid)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double acc[4][2];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
    __syncthreads();
    for (int i = 0; i < VD_NS - 1; ++i) {
      if (i < ntl) issue(i, i);
      else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int t = 0; t < ntl; ++t) {
      asm volatile("cp.async.wait_group %0;" ::"n"(VD_NS - 2) : "memory");
      __syncthreads();
      const double* xs = dsm + (t % VD_NS) * SF;
      const double* vs = xs + XB;
#pragma unroll
      for (int ks = 0; ks < 16; ++ks) {
        const double a = xs[(8 * wid + gq) * VD_XS + 4 * ks + tq];  // A (m = row, k = column)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
          if (8 * nt < p) dmma_r(acc[nt], a, vs[(8 * nt + gq) * VD_OS + 4 * ks + tq]);
      }
      __syncthreads();
      if (t + VD_NS - 1 < ntl) issue(t + VD_NS - 1, (t + VD_NS - 1) % VD_NS);
      else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    // C (row, a): row = 8 w + gq, a = 8 nt + 2 tq (+1)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a = 8 * nt + 2 * tq + h;
        const int64_t i = i0 + 8 * wid + gq;
        if (a < p && i < nx) slab[(cc * p + a) * nx + i] = acc[nt][h];
      }
  }
}

static int ab_dmma(Arena& ws, const double* At, int64_t p, int64_t r, const double* B, int64_t c, int64_t ldb,
                   bool trans, double* V, cudaStream_t st) {
  if (p > 32 || getenv("NENMF_AB_SIMT") != nullptr) return NENMF_ERR_UNSUPPORTED;
  const int64_t nx = trans ? c : r, mx = trans ? r : c;
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (((nx | mx | ldb) & 1) != 0 || (ws.base != nullptr && (!al16(B) || !al16(At)))) return NENMF_ERR_UNSUPPORTED;
  int sms = sm_count();
  if (sms <= 0) sms = 148;
  auto chunks = [&](int64_t along, int64_t bands) {  // (count, length) of 64-aligned chunks
    int64_t k = imax(1, imin(cdiv(along, 64), cdiv(4 * sms, bands)));
    const int64_t len = cdiv(cdiv(along, k), 64) * 64;
    return std::make_pair(cdiv(along, len), len);
  };
  auto zneed = [&](int64_t zx, int64_t zm) { return chunks(zx, cdiv(zm, 64)).first * p * zm; };
  auto yneed = [&](int64_t yx, int64_t ym) { return chunks(ym, cdiv(yx, 64)).first * p * yx; };
  const int64_t need = imax(imax(zneed(r, c), zneed(c, r)), imax(yneed(c, r), yneed(r, c)));
  double* slab = ws.take<double>((size_t)need);
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  const size_t smem = (size_t)VD_NS * (64 * VD_XS + 32 * VD_OS) * sizeof(double);
  if (!trans) {  // V (p x mx) = At (p x nx) X
    const int64_t nbands = cdiv(mx, 64);
    const auto ch = chunks(nx, nbands);
    const int64_t nunits = nbands * ch.first;
    NENMF_CUDA_TRY(set_smem(k_ux64, smem));
    k_ux64<<<(unsigned)imin(nunits, (int64_t)sms), 256, smem, st>>>(B, nx, mx, ldb, At, (int)p, nbands, ch.second,
                                                                     nunits, slab);
    NENMF_LAUNCH_CHECK();
    k_chunk_reduce<double><<<(unsigned)cdiv(p * mx, 256), 256, 0, st>>>(slab, (int)ch.first, p * mx, V);
    NENMF_LAUNCH_CHECK();
  } else {  // V (p x nx) = At (p x mx) X^T
    const int64_t nbands = cdiv(nx, 64);
    const auto ch = chunks(mx, nbands);
    const int64_t nunits = nbands * ch.first;
    NENMF_CUDA_TRY(set_smem(k_xv64, smem));
    k_xv64<<<(unsigned)imin(nunits, (int64_t)sms), 256, smem, st>>>(B, nx, mx, ldb, At, (int)p, nbands, ch.second,
                                                                     nunits, slab);
    NENMF_LAUNCH_CHECK();
    k_chunk_reduce<double><<<(unsigned)cdiv(p * nx, 256), 256, 0, st>>>(slab, (int)ch.first, p * nx, V);
    NENMF_LAUNCH_CHECK();
  }
  return NENMF_OK;
}

// FP32 tensor-core V = A^T B; NENMF_ERR_UNSUPPORTED outside p <= 32 or
// unaligned operands (the caller then uses the CUDA-core kernel)
static int ab_mma(Arena& ws, const float* At, int64_t p, int64_t r, const float* B, int64_t c, int64_t ldb,
                  bool trans, float* V, cudaStream_t st) {
  if (p > 32 || getenv("NENMF_AB_SIMT") != nullptr) return NENMF_ERR_UNSUPPORTED;
  // X is B (r x c) or, transposed, the c x r matrix whose transpose B is
  const int64_t nx = trans ? c : r, mx = trans ? r : c;
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  // (dry runs size the scratch without seeing the pointers: assume aligned)
  if (((nx | mx | ldb) & 3) != 0 || (ws.base != nullptr && (!al16(B) || !al16(At)))) return NENMF_ERR_UNSUPPORTED;
  int sms = sm_count();
  if (sms <= 0) sms = 148;
  // scratch sized for either orientation of (r, c), so that sizing dry runs
  // (which do not know the orientation of the later call) always suffice
  auto zslab = [&](int64_t zx, int64_t zm) {
    const int64_t nb = cdiv(zm, 64);
    int64_t k = imax(1, imin(cdiv(zx, 128), cdiv(4 * sms, nb)));
    return cdiv(zx, cdiv(cdiv(zx, k), 128) * 128) * p * zm;
  };
  auto yslab = [&](int64_t yx, int64_t ym) {
    const int64_t nb = cdiv(yx, 128);
    int64_t k = imax(1, imin(cdiv(ym, 64), cdiv(4 * sms, nb)));
    return cdiv(ym, cdiv(cdiv(ym, k), 64) * 64) * p * yx;
  };
  const int64_t need = imax(imax(zslab(r, c), zslab(c, r)), imax(yslab(c, r), yslab(r, c)));
  float* slab = ws.take<float>((size_t)need);
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  if (!trans) {
    const int64_t nbands = cdiv(mx, 64);
    // row chunks: ~4 units per SM, chunks of whole 128-row tiles
    int64_t nch = imax(1, imin(cdiv(nx, 128), cdiv(4 * sms, nbands)));
    const int64_t rchunk = cdiv(cdiv(nx, nch), 128) * 128;
    nch = cdiv(nx, rchunk);
    const int mt = (int)cdiv(p, 16);
    const size_t smem = ((size_t)VP_NS * (128 * VP_XS + 16 * mt * VP_US) + (size_t)16 * mt * 64) * sizeof(float);
    const int64_t nunits = nbands * nch;
    const unsigned grid = (unsigned)imin(nunits, (int64_t)sms);
    if (mt == 1) {
      NENMF_CUDA_TRY(set_smem(k_ux<1>, smem));
      k_ux<1><<<grid, 256, smem, st>>>(B, nx, mx, ldb, At, (int)p, nbands, rchunk, nunits, slab);
    } else {
      NENMF_CUDA_TRY(set_smem(k_ux<2>, smem));
      k_ux<2><<<grid, 256, smem, st>>>(B, nx, mx, ldb, At, (int)p, nbands, rchunk, nunits, slab);
    }
    NENMF_LAUNCH_CHECK();
    k_chunk_reduce<float><<<(unsigned)cdiv(p * mx, 256), 256, 0, st>>>(slab, (int)nch, p * mx, V);
    NENMF_LAUNCH_CHECK();
  } else {
    const int64_t nbands = cdiv(nx, 128);
    int64_t nch = imax(1, imin(cdiv(mx, 64), cdiv(4 * sms, nbands)));
    const int64_t cchunk = cdiv(cdiv(mx, nch), 64) * 64;
    nch = cdiv(mx, cchunk);
    const int ntp = (int)cdiv(p, 8);
    const size_t smem = (size_t)VP_NS * (128 * VP_XS + 8 * ntp * VP_VS) * sizeof(float);
    const int64_t nunits = nbands * nch;
    const unsigned grid = (unsigned)imin(nunits, (int64_t)sms);
    auto go = [&](auto kern) -> int {
      NENMF_CUDA_TRY(set_smem(kern, smem));
      kern<<<grid, 256, smem, st>>>(B, nx, mx, ldb, At, (int)p, nbands, cchunk, nunits, slab);
      return NENMF_OK;
    };
    if (ntp == 1) NENMF_TRY(go(k_xv<1>));
    else if (ntp == 2) NENMF_TRY(go(k_xv<2>));
    else if (ntp == 3) NENMF_TRY(go(k_xv<3>));
    else NENMF_TRY(go(k_xv<4>));
    NENMF_LAUNCH_CHECK();
    k_chunk_reduce<float><<<(unsigned)cdiv(p * nx, 256), 256, 0, st>>>(slab, (int)nch, p * nx, V);
    NENMF_LAUNCH_CHECK();
  }
  return NENMF_OK;
}

template <typename T>
static int ab_simt(Arena& ws, const T* At, int64_t p, int64_t r, const T* B, int64_t c, int64_t ldb, bool trans,
                   T* V, cudaStream_t st);

template <typename T>
int ab(Arena& ws, const T* At, int64_t p, int64_t r, const T* B, int64_t c, int64_t ldb, bool trans,
       T* V, cudaStream_t st) {
  if (p < 1 || r < 1 || c < 1) return NENMF_ERR_DIM;
  if (p > 4 * AB_MAXA) {
    // more rows of At than the kernels hold (p > 64): row blocks, whose outputs are contiguous rows of V
    const int64_t pb = 4 * AB_MAXA;
    const bool dry = ws.base == nullptr;
    size_t need = 0;
    for (int64_t p0 = 0; p0 < p; p0 += pb) {
      Arena a = ws;
      NENMF_TRY(ab<T>(a, dry ? At : At + p0 * r, imin(pb, p - p0), r, B, c, ldb, trans, dry ? V : V + p0 * c, st));
      if (a.used - ws.used > need) need = a.used - ws.used;
      if (!dry && !a.ok) return NENMF_ERR_WORKSPACE;
    }
    if (dry) ws.take<char>(need);
    return NENMF_OK;
  }
  {
    // tensor-core path; a dry run sizes it AND the CUDA-core fallback below
    // (the live call may fall back on unaligned operands)
    Arena fast = ws;
    int rc;
    if constexpr (sizeof(T) == 4)
      rc = ab_mma(fast, reinterpret_cast<const float*>(At), p, r, reinterpret_cast<const float*>(B), c, ldb, trans,
                  reinterpret_cast<float*>(V), st);
    else
      rc = ab_dmma(fast, reinterpret_cast<const double*>(At), p, r, reinterpret_cast<const double*>(B), c, ldb,
                   trans, reinterpret_cast<double*>(V), st);
    if (rc != NENMF_ERR_UNSUPPORTED) {
      if (ws.base != nullptr) {
        ws = fast;
        return rc;
      }
      Arena slow = ws;
      const size_t fast_used = fast.used;
      ab_simt<T>(slow, At, p, r, B, c, ldb, trans, V, st);
      ws.used = fast_used > slow.used ? fast_used : slow.used;
      return NENMF_OK;
    }
  }
  return ab_simt<T>(ws, At, p, r, B, c, ldb, trans, V, st);
}

template <typename T>
static int ab_simt(Arena& ws, const T* At, int64_t p, int64_t r, const T* B, int64_t c, int64_t ldb, bool trans,
                   T* V, cudaStream_t st) {
  if (p > 4 * AB_MAXA) return NENMF_ERR_UNSUPPORTED;
  const int64_t nchunk = cdiv(r, AB_RCHUNK);
  T* part = nchunk > 1 ? ws.take<T>((size_t)nchunk * p * c) : nullptr;
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  size_t smem = ((size_t)AB_RT * (AB_CB + 1) + (size_t)p * (AB_RT + 1)) * sizeof(T);
  dim3 grid((unsigned)cdiv(c, AB_CB), (unsigned)nchunk);
  T* direct = nchunk > 1 ? nullptr : V;
  if (trans) {
    NENMF_CUDA_TRY(cudaFuncSetAttribute(k_ab<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_ab<T, true><<<grid, AB_THREADS, smem, st>>>(At, (int)p, r, B, c, ldb, AB_RCHUNK, part, direct);
  } else {
    NENMF_CUDA_TRY(cudaFuncSetAttribute(k_ab<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_ab<T, false><<<grid, AB_THREADS, smem, st>>>(At, (int)p, r, B, c, ldb, AB_RCHUNK, part, direct);
  }
  NENMF_LAUNCH_CHECK();
  if (nchunk > 1) {
    int64_t cnt = p * c;
    k_chunk_reduce<T><<<(unsigned)cdiv(cnt, 256), 256, 0, st>>>(part, (int)nchunk, cnt, V);
    NENMF_LAUNCH_CHECK();
  }
  return NENMF_OK;
}

// --------------------------------------------------------------- resid ----
constexpr int RS_THREADS = 256;  // 64 columns x 4 row groups

// Explicit residual sums ||A F - B||^2 for one or two candidates F (the
// reference's _true_objective, nnls.py:115-116, and the RRE of
// tracing.py:45-57 with A^T = G^T, B = X).  Register-blocked: each thread
// keeps its column of F (p values per candidate) in registers for the whole
// row chunk and reads A^T columns as broadcast 16-byte shared-memory loads,
// so the inner product is FMA-bound and B (X) is streamed once, coalesced.
template <typename T, int PM, bool TRANS>
__global__ void __launch_bounds__(RS_THREADS)
k_resid(const T* __restrict__ At, int p, int64_t r, const T* __restrict__ B, int64_t c, int64_t ldb,
        const T* __restrict__ F1, const T* __restrict__ F2, int64_t rchunk,
        double* __restrict__ part, const int* __restrict__ gate) {
  if (gate != nullptr && *gate == 0) return;
  constexpr int G = RS_THREADS / AB_CB;          // row groups
  constexpr int RPT = AB_RT / G;                 // rows per thread per tile
  constexpr int PS = PM + 4;                     // row stride: 16-byte aligned, fewer store conflicts
  __shared__ __align__(16) T AtT[AB_RT * PS];    // A^T columns of the tile, a contiguous
  __shared__ double red[33];
  const int jj = threadIdx.x % AB_CB, g = threadIdx.x / AB_CB;
  const int64_t j0 = (int64_t)blockIdx.x * AB_CB;
  const int64_t tc0 = (int64_t)blockIdx.y * rchunk, tc1 = min(r, tc0 + rchunk);
  const bool two = F2 != nullptr;
  const int64_t j = j0 + jj;
  const bool live = j < c;
  T f1[PM], f2[PM];
#pragma unroll
  for (int a = 0; a < PM; ++a) {
    f1[a] = (live && a < p) ? F1[(int64_t)a * c + j] : T(0);
    f2[a] = (two && live && a < p) ? F2[(int64_t)a * c + j] : T(0);
  }
  // B(t, j) for this thread's rows g, g + G, ... of a tile, loaded one tile ahead
  auto bload = [&](int64_t t0, T (&v)[RPT]) {
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int64_t t = t0 + g + G * i;
      v[i] = (live && t < tc1) ? (TRANS ? B[j * ldb + t] : __ldcs(&B[t * ldb + j])) : T(0);
    }
  };
  auto dot = [&](const T* w, const T (&f)[PM]) -> T {
    T s = T(0);
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int a = 0; a < PM; a += 4) {
        const float4 w4 = *reinterpret_cast<const float4*>(w + a);
        s = fmaf(w4.x, f[a], s);
        s = fmaf(w4.y, f[a + 1], s);
        s = fmaf(w4.z, f[a + 2], s);
        s = fmaf(w4.w, f[a + 3], s);
      }
    } else {
#pragma unroll
      for (int a = 0; a < PM; a += 2) {
        const double2 w2 = *reinterpret_cast<const double2*>(w + a);
        s = fma(w2.x, f[a], s);
        s = fma(w2.y, f[a + 1], s);
      }
    }
    return s;
  };
  T bc[RPT], bn[RPT];
  bload(tc0, bc);
  double acc0 = 0.0, acc1 = 0.0;
  for (int64_t t0 = tc0; t0 < tc1; t0 += AB_RT) {
    const int nt = (int)imin(AB_RT, tc1 - t0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < AB_RT * PM; idx += blockDim.x) {
      const int a = idx / AB_RT, tt = idx % AB_RT;  // coalesced along the rows of A
      AtT[tt * PS + a] = (tt < nt && a < p) ? At[(int64_t)a * r + t0 + tt] : T(0);
    }
    __syncthreads();
    if (t0 + AB_RT < tc1) bload(t0 + AB_RT, bn);
    if (live) {
      // four rows at a time: four independent FMA chains per candidate
#pragma unroll
      for (int i0 = 0; i0 < RPT; i0 += 4) {
        T s[4] = {T(0), T(0), T(0), T(0)}, s2[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
        for (int a = 0; a < PM; ++a) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const T wa = AtT[(g + G * (i0 + u)) * PS + a];
            s[u] = fma_acc(wa, f1[a], s[u]);
            if (two) s2[u] = fma_acc(wa, f2[a], s2[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (g + G * (i0 + u) < nt) {
            const double d0 = (double)(s[u] - bc[i0 + u]);
            acc0 += d0 * d0;
            if (two) {
              const double d1 = (double)(s2[u] - bc[i0 + u]);
              acc1 += d1 * d1;
            }
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i) bc[i] = bn[i];
  }
  const int64_t bid = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
  double s0 = block_sum(acc0, red);
  double s1 = block_sum(acc1, red);
  if (threadIdx.x == 0) {
    part[bid * 2 + 0] = s0;
    part[bid * 2 + 1] = s1;
  }
}

// FP32 residual sums on the tensor pipe, X-oriented: for X (nx x mx, ld ldx)
// and candidates (U1, V1), (U2, V2) (p x nx and p x mx, p <= 32), part sums
// of ||U^T V - X||^2.  Warp tile 16 rows x 64 columns: the 16 x 8 blocks of
// U^T V come from m16n8k8 TF32 MMAs in 3xTF32 split precision (hi by
// truncation, lo = x - hi raw; relative error ~2^-20), the X values of the
// tile are loaded (two floats per thread per block) before the MMAs so the
// DRAM stream overlaps them.  Row/column tails are masked.

template <int KT>
__global__ void __launch_bounds__(256)
k_resid_mma(const float* __restrict__ X, int64_t nx, int64_t mx, int64_t ldx, int p,
            const float* __restrict__ U1, const float* __restrict__ V1, const float* __restrict__ U2,
            const float* __restrict__ V2, double* __restrict__ part, const int* __restrict__ gate) {
  if (gate != nullptr && *gate == 0) return;
  __shared__ double red[33];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, gq = lane >> 2, tq = lane & 3;
  const bool two = U2 != nullptr;
  const int64_t ntr = (nx + 15) / 16, ntc = (mx + 63) / 64;
  const int64_t tiles = ntr * ntc;
  double acc0 = 0.0, acc1 = 0.0;
  for (int64_t tile = (int64_t)blockIdx.x * 8 + wid; tile < tiles; tile += (int64_t)gridDim.x * 8) {
    const int64_t i0 = (tile / ntc) * 16, j0 = (tile % ntc) * 64;
    // X of the warp tile: rows i0 + gq (+8), columns j0 + 8 nt + 2 tq (+1)
    float2 xv[8][2];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t i = i0 + gq + 8 * h, j = j0 + 8 * nt + 2 * tq;
        float2 v = make_float2(0.f, 0.f);
        if (i < nx) {
          const float* px = X + i * ldx + j;
          if (j + 1 < mx && ((reinterpret_cast<uintptr_t>(px) & 7) == 0)) v = __ldcs(reinterpret_cast<const float2*>(px));
          else {
            if (j < mx) v.x = __ldcs(px);
            if (j + 1 < mx) v.y = __ldcs(px + 1);
          }
        }
        xv[nt][h] = v;
      }
    // A fragments (rows of U^T): a0 (gq, tq), a1 (gq+8, tq), a2 (gq, tq+4), a3 (gq+8, tq+4)
    auto afrag = [&](const float* U, uint32_t (&ah)[KT][4], uint32_t (&al)[KT][4]) {
#pragma unroll
      for (int kt = 0; kt < KT; ++kt)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int a = 8 * kt + tq + ((q & 2) ? 4 : 0);
          const int64_t i = i0 + gq + ((q & 1) ? 8 : 0);
          const float u = (a < p && i < nx) ? __ldg(&U[(int64_t)a * nx + i]) : 0.f;
          ah[kt][q] = tf_hi(u);
          al[kt][q] = tf_lo(u);
        }
    };
    uint32_t a1h[KT][4], a1l[KT][4], a2h[KT][4], a2l[KT][4];
    afrag(U1, a1h, a1l);
    if (two) {
      if (U2 != U1) afrag(U2, a2h, a2l);
      else {
#pragma unroll
        for (int kt = 0; kt < KT; ++kt)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            a2h[kt][q] = a1h[kt][q];
            a2l[kt][q] = a1l[kt][q];
          }
      }
    }
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int64_t jb = j0 + 8 * nt + gq;  // B fragment column
      auto prod = [&](const float* V, const uint32_t (&ah)[KT][4], const uint32_t (&al)[KT][4], float (&c)[4]) {
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const int a0 = 8 * kt + tq, a1 = a0 + 4;
          const float v0 = (a0 < p && jb < mx) ? __ldg(&V[(int64_t)a0 * mx + jb]) : 0.f;
          const float v1 = (a1 < p && jb < mx) ? __ldg(&V[(int64_t)a1 * mx + jb]) : 0.f;
          const uint32_t b0h = tf_hi(v0), b1h = tf_hi(v1), b0l = tf_lo(v0), b1l = tf_lo(v1);
          mma_tf32_r(c, al[kt], b0h, b1h);
          mma_tf32_r(c, ah[kt], b0l, b1l);
          mma_tf32_r(c, ah[kt], b0h, b1h);
        }
      };
      float c1[4] = {0.f, 0.f, 0.f, 0.f};
      prod(V1, a1h, a1l, c1);
      const float d0 = c1[0] - xv[nt][0].x, d1 = c1[1] - xv[nt][0].y, d2 = c1[2] - xv[nt][1].x,
                  d3 = c1[3] - xv[nt][1].y;
      s0 = fmaf(d0, d0, fmaf(d1, d1, fmaf(d2, d2, fmaf(d3, d3, s0))));
      if (two) {
        float c2[4] = {0.f, 0.f, 0.f, 0.f};
        prod(V2, a2h, a2l, c2);
        const float e0 = c2[0] - xv[nt][0].x, e1 = c2[1] - xv[nt][0].y, e2 = c2[2] - xv[nt][1].x,
                    e3 = c2[3] - xv[nt][1].y;
        s1 = fmaf(e0, e0, fmaf(e1, e1, fmaf(e2, e2, fmaf(e3, e3, s1))));
      }
    }
    acc0 += (double)s0;
    acc1 += (double)s1;
  }
  const double b0 = block_sum(acc0, red);
  const double b1 = block_sum(acc1, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = b0;
    part[2 * blockIdx.x + 1] = b1;
  }
}

// Pipelined variant (X, U, V 16-byte aligned, nx, mx, ldx multiples of 4):
// persistent CTAs stream 128 x 64 tiles of X together with the matching
// U (p x 128) and V (p x 64) slices through a 3-stage cp.async ring; the
// 8 warps take 16 rows each; fragments and X values are read from shared
// memory with conflict-free strides.  Same arithmetic as k_resid_mma.
constexpr int RP_NS = 3, RP_XS = 72, RP_US = 136, RP_VS = 72;

__device__ __forceinline__ void cp16(void* dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes)
               : "memory");
}

template <int KT>
__global__ void __launch_bounds__(256, 1)
k_resid_pipe(const float* __restrict__ X, int64_t nx, int64_t mx, int64_t ldx, int p,
             const float* __restrict__ U1, const float* __restrict__ V1, const float* __restrict__ U2,
             const float* __restrict__ V2, double* __restrict__ part, const int* __restrict__ gate) {
  if (gate != nullptr && *gate == 0) return;
  constexpr int KP = 8 * KT;
  constexpr int XB = 128 * RP_XS, UB = KP * RP_US, VB = KP * RP_VS;  // floats per stage section
  extern __shared__ __align__(16) float rsm[];
  __shared__ double red[33];
  const bool two = U2 != nullptr;
  const bool u2s = two && U2 != U1, v2s = two && V2 != V1;  // second-candidate sections
  const int stage_f = XB + UB + VB + (u2s ? UB : 0) + (v2s ? VB : 0);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, gq = lane >> 2, tq = lane & 3;
  const int64_t ntr = (nx + 127) / 128, ntc = (mx + 63) / 64, tiles = ntr * ntc;
  auto issue = [&](int64_t tile, int slot) {
    float* base = rsm + (size_t)slot * stage_f;
    const int64_t i0 = (tile / ntc) * 128, j0 = (tile % ntc) * 64;
    // X: 128 rows x 16 chunks
    for (int c = tid; c < 128 * 16; c += 256) {
      const int r = c >> 4, ch = c & 15;
      const int64_t i = i0 + r, j = j0 + 4 * ch;
      const int valid = (i < nx) ? (int)imax(0, imin(4, mx - j)) : 0;
      cp16(base + r * RP_XS + 4 * ch, X + (valid ? i * ldx + j : 0), 4 * valid);
    }
    auto urows = [&](const float* U, float* dst) {  // p x 128 slice of U (p x nx)
      for (int c = tid; c < KP * 32; c += 256) {
        const int a = c >> 5, ch = c & 31;
        const int64_t i = i0 + 4 * ch;
        const int valid = a < p ? (int)imax(0, imin(4, nx - i)) : 0;
        cp16(dst + a * RP_US + 4 * ch, U + (valid ? (int64_t)a * nx + i : 0), 4 * valid);
      }
    };
    auto vrows = [&](const float* V, float* dst) {  // p x 64 slice of V (p x mx)
      for (int c = tid; c < KP * 16; c += 256) {
        const int a = c >> 4, ch = c & 15;
        const int64_t j = j0 + 4 * ch;
        const int valid = a < p ? (int)imax(0, imin(4, mx - j)) : 0;
        cp16(dst + a * RP_VS + 4 * ch, V + (valid ? (int64_t)a * mx + j : 0), 4 * valid);
      }
    };
    float* us = base + XB;
    float* vs = us + UB;
    urows(U1, us);
    vrows(V1, vs);
    float* extra = vs + VB;
    if (u2s) {
      urows(U2, extra);
      extra += UB;
    }
    if (v2s) vrows(V2, extra);
  };
  const int64_t first = blockIdx.x, step = gridDim.x;
  const int64_t mine = first < tiles ? (tiles - 1 - first) / step + 1 : 0;
#pragma unroll
  for (int sidx = 0; sidx < RP_NS - 1; ++sidx) {
    if (sidx < mine) issue(first + sidx * step, sidx);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  double acc0 = 0.0, acc1 = 0.0;
  for (int64_t it = 0; it < mine; ++it) {
    if (it + RP_NS - 1 < mine) issue(first + (it + RP_NS - 1) * step, (int)((it + RP_NS - 1) % RP_NS));
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(RP_NS - 1) : "memory");
    __syncthreads();
    const float* base = rsm + (size_t)(it % RP_NS) * stage_f;
    const float* xs = base;
    const float* us1 = base + XB;
    const float* vs1 = us1 + UB;
    const float* us2 = u2s ? vs1 + VB : us1;
    const float* vs2 = v2s ? vs1 + VB + (u2s ? UB : 0) : vs1;
    const int rw = 16 * wid;  // this warp's 16 rows of the tile
    auto afr = [&](const float* us, uint32_t (&ah)[KT][4], uint32_t (&al)[KT][4]) {
#pragma unroll
      for (int kt = 0; kt < KT; ++kt)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float u = us[(8 * kt + tq + ((q & 2) ? 4 : 0)) * RP_US + rw + gq + ((q & 1) ? 8 : 0)];
          ah[kt][q] = tf_hi(u);
          al[kt][q] = tf_lo(u);
        }
    };
    uint32_t a1h[KT][4], a1l[KT][4], a2h[KT][4], a2l[KT][4];
    afr(us1, a1h, a1l);
    if (two) afr(us2, a2h, a2l);
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float2 x0 = *reinterpret_cast<const float2*>(xs + (rw + gq) * RP_XS + 8 * nt + 2 * tq);
      const float2 x1 = *reinterpret_cast<const float2*>(xs + (rw + gq + 8) * RP_XS + 8 * nt + 2 * tq);
      auto prod = [&](const float* vs, const uint32_t (&ah)[KT][4], const uint32_t (&al)[KT][4], float (&c)[4]) {
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const float v0 = vs[(8 * kt + tq) * RP_VS + 8 * nt + gq];
          const float v1 = vs[(8 * kt + tq + 4) * RP_VS + 8 * nt + gq];
          const uint32_t b0h = tf_hi(v0), b1h = tf_hi(v1), b0l = tf_lo(v0), b1l = tf_lo(v1);
          mma_tf32_r(c, al[kt], b0h, b1h);
          mma_tf32_r(c, ah[kt], b0l, b1l);
          mma_tf32_r(c, ah[kt], b0h, b1h);
        }
      };
      float c1[4] = {0.f, 0.f, 0.f, 0.f};
      prod(vs1, a1h, a1l, c1);
      const float d0 = c1[0] - x0.x, d1 = c1[1] - x0.y, d2 = c1[2] - x1.x, d3 = c1[3] - x1.y;
      s0 = fmaf(d0, d0, fmaf(d1, d1, fmaf(d2, d2, fmaf(d3, d3, s0))));
      if (two) {
        float c2[4] = {0.f, 0.f, 0.f, 0.f};
        prod(vs2, a2h, a2l, c2);
        const float e0 = c2[0] - x0.x, e1 = c2[1] - x0.y, e2 = c2[2] - x1.x, e3 = c2[3] - x1.y;
        s1 = fmaf(e0, e0, fmaf(e1, e1, fmaf(e2, e2, fmaf(e3, e3, s1))));
      }
    }
    acc0 += (double)s0;
    acc1 += (double)s1;
    __syncthreads();  // the slot is refilled by a later issue
  }
  const double b0 = block_sum(acc0, red);
  const double b1 = block_sum(acc1, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = b0;
    part[2 * blockIdx.x + 1] = b1;
  }
}

// FP64 residuals ||X - U^T V||^2 for one or two candidates on the FP64 tensor
// pipe (the RRE emit, tracing.py:45-57, and the vanilla tie-break pair,
// nnls.py:219-227): X in 64 x 64 tiles through a cp.async ring with the U
// slice of the tile's rows and the V slice(s) of its columns; warp w forms
// the product for rows 8w..8w+7 (DMMA m8n8k4, K = p) and accumulates
// (x - p)^2 straight from the accumulator fragments.  One CTA per SM, tiles
// dealt round-robin, per-CTA partials summed in fixed order.
constexpr int RD_XS = 68;  // shared row stride (doubles)
template <int NC>
__global__ void __launch_bounds__(256, 1)
k_resid64(const double* __restrict__ X, int64_t nx, int64_t mx, int64_t ldx, int p, const double* __restrict__ U1,
          const double* __restrict__ V1, const double* __restrict__ U2, const double* __restrict__ V2,
          double* __restrict__ part, const int* __restrict__ gate) {
  constexpr int NS = NC == 1 ? 3 : 2;
  constexpr int SF = 64 * RD_XS + 2 * NC * 32 * RD_XS;  // X | U1 V1 (| U2 V2), doubles
  extern __shared__ __align__(16) double dsm[];
  __shared__ double red[33];
  if (gate != nullptr && *gate == 0) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, gq = lane >> 2, tq = lane & 3;
  const int64_t nrt = (nx + 63) / 64, nct = (mx + 63) / 64, ntiles = nrt * nct;
  const int nks = (p + 3) >> 2;
  double s1 = 0.0, s2 = 0.0;
  auto issue = [&](int64_t tile, int stg) {
    double* xs = dsm + (size_t)stg * SF;
    const int64_t i0 = (tile / nct) * 64, j0 = (tile % nct) * 64;
    for (int c = tid; c < 64 * 32; c += 256) {
      const int r = c >> 5, ch = c & 31;
      const int64_t i = i0 + r, j = j0 + 2 * ch;
      const int valid = i < nx ? (int)imax(0, imin(2, mx - j)) : 0;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(xs + r * RD_XS + 2 * ch)),
                   "l"(X + (valid ? i * ldx + j : 0)), "r"(8 * valid)
                   : "memory");
    }
    for (int c = tid; c < 2 * NC * 32 * 32; c += 256) {  // [U1 | V1 | U2 | V2] slices, p x 64 each
      const int which = c >> 10, cc = c & 1023, a = cc >> 5, ch = cc & 31;
      const bool isU = (which & 1) == 0;
      const double* src = which == 0 ? U1 : which == 1 ? V1 : which == 2 ? U2 : V2;
      const int64_t len = isU ? nx : mx, base = isU ? i0 : j0, j = base + 2 * ch;
      const int valid = a < p ? (int)imax(0, imin(2, len - j)) : 0;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(
                       xs + 64 * RD_XS + (size_t)which * 32 * RD_XS + a * RD_XS + 2 * ch)),
                   "l"(src + (valid ? (int64_t)a * len + j : 0)), "r"(8 * valid)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int64_t t0 = blockIdx.x;
  for (int i = 0; i < NS - 1; ++i) {
    const int64_t tl = t0 + (int64_t)i * gridDim.x;
    if (tl < ntiles) issue(tl, i);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  int k = 0;
  for (int64_t tile = t0; tile < ntiles; tile += gridDim.x, ++k) {
    asm volatile("cp.async.wait_group %0;" ::"n"(NS - 2) : "memory");
    __syncthreads();
    const double* xs = dsm + (size_t)(k % NS) * SF;
    const int64_t i0 = (tile / nct) * 64, j0 = (tile % nct) * 64;
#pragma unroll
    for (int cand = 0; cand < NC; ++cand) {
      const double* us = xs + 64 * RD_XS + (size_t)(2 * cand) * 32 * RD_XS;
      const double* vs = us + 32 * RD_XS;
      double acc[8][2];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
      for (int ks = 0; ks < nks; ++ks) {
        const double a = us[(4 * ks + tq) * RD_XS + 8 * wid + gq];  // A (row, k) = U[k][row]
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) dmma_r(acc[nt], a, vs[(4 * ks + tq) * RD_XS + 8 * nt + gq]);
      }
      const int r = 8 * wid + gq;
      double sc = 0.0;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = 8 * nt + 2 * tq + h;
          if (i0 + r < nx && j0 + col < mx) {
            const double d = xs[r * RD_XS + col] - acc[nt][h];
            sc = fma(d, d, sc);
          }
        }
      if (cand == 0) s1 += sc;
      else s2 += sc;
    }
    __syncthreads();
    const int64_t nxt = tile + (int64_t)(NS - 1) * gridDim.x;
    if (nxt < ntiles) issue(nxt, (k + NS - 1) % NS);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  s1 = block_sum(s1, red);
  s2 = block_sum(s2, red);
  if (tid == 0) {
    part[2 * blockIdx.x] = s1;
    part[2 * blockIdx.x + 1] = s2;
  }
}

// per-CTA sums of (D - B)^2 over an r x c result D (row-major) against B (r x c with leading
// dimension ldb, or its transpose c x r when trans), into part[2 * block + which]; `zero_other`
// clears the second candidate's slot (one candidate only)
template <typename T>
__global__ void k_diff_sumsq(const T* __restrict__ D, const T* __restrict__ B, int64_t r, int64_t c, int64_t ldb,
                             int trans, double* __restrict__ part, int which, int zero_other) {
  __shared__ double red[33];
  double a = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < r * c; i += stride) {
    const int64_t t = i / c, j = i % c;
    const double d = (double)D[i] - (double)(trans ? B[j * ldb + t] : B[t * ldb + j]);
    a = fma(d, d, a);
  }
  a = block_sum(a, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x + which] = a;
    if (zero_other) part[2 * blockIdx.x + 1 - which] = 0.0;
  }
}

// fixed-order sum of `n` pairs -> out[0..1]; optional gate
__global__ void k_pair_final(const double* __restrict__ part, int64_t n, double* __restrict__ out,
                             const int* __restrict__ gate) {
  if (gate != nullptr && *gate == 0) return;
  __shared__ double red[33];
  double a = 0.0, b = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    a += part[2 * i];
    b += part[2 * i + 1];
  }
  a = block_sum(a, red);
  b = block_sum(b, red);
  if (threadIdx.x == 0) {
    out[0] = a;
    out[1] = b;
  }
}

template <typename T>
int resid(Arena& ws, const T* At, int64_t p, int64_t r, const T* B, int64_t c, int64_t ldb, bool trans,
          const T* F1, const T* F2, double* out2, const int* gate, cudaStream_t st) {
  if (p < 1 || r < 1 || c < 1) return NENMF_ERR_DIM;
  if (p > 64) {
    // inner dimension above the register-blocked kernels (the reference takes any p, nnls.py:119-159):
    // D = A F (r x c) by the CUDA-core product over A = At^T, then sum (D - B)^2 in fixed order
    T* A = ws.take<T>((size_t)r * p);
    T* D = ws.take<T>((size_t)r * c);
    const unsigned grid = (unsigned)imax(1, imin((int64_t)1184, cdiv(r * c, 256)));
    double* part = ws.take<double>((size_t)grid * 2);
    const bool dry = ws.base == nullptr;
    if (!dry && !ws.ok) return NENMF_ERR_WORKSPACE;
    if (!dry) NENMF_TRY(transpose<T>(At, p, r, r, A, st));
    size_t need = 0;
    for (int cand = 0; cand < 2; ++cand) {
      const T* F = cand == 0 ? F1 : F2;
      if (!dry && F == nullptr) break;
      Arena a = ws;
      NENMF_TRY(ab<T>(a, A, r, p, F, c, c, false, D, st));
      if (a.used - ws.used > need) need = a.used - ws.used;
      if (!dry && !a.ok) return NENMF_ERR_WORKSPACE;
      if (!dry) {
        k_diff_sumsq<T><<<grid, 256, 0, st>>>(D, B, r, c, ldb, trans ? 1 : 0, part, cand, F2 == nullptr ? 1 : 0);
        NENMF_LAUNCH_CHECK();
      }
    }
    if (dry) {
      ws.take<char>(need);
      return NENMF_OK;
    }
    k_pair_final<<<1, 256, 0, st>>>(part, (int64_t)grid, out2, nullptr);
    NENMF_LAUNCH_CHECK();
    return NENMF_OK;
  }
  if constexpr (sizeof(T) == 4) {
    if (p <= 32 && getenv("NENMF_RESID_SIMT") == nullptr) {
      // X-oriented tensor-core kernel: B is X (r x c) or, transposed, X (c x r)
      const int64_t nx = trans ? c : r, mx = trans ? r : c;
      const float* U1 = reinterpret_cast<const float*>(trans ? F1 : At);
      const float* U2 = F2 == nullptr ? nullptr : reinterpret_cast<const float*>(trans ? F2 : At);
      const float* V1 = reinterpret_cast<const float*>(trans ? At : F1);
      const float* V2 = F2 == nullptr ? nullptr : reinterpret_cast<const float*>(trans ? At : F2);
      int sms = sm_count();
      if (sms <= 0) sms = 148;
      const int64_t tiles = cdiv(nx, 16) * cdiv(mx, 64);
      const bool pipe_ok = ((nx | mx | ldb) & 3) == 0;
      const unsigned grid = pipe_ok ? (unsigned)imax(1, imin((int64_t)sms, cdiv(nx, 128) * cdiv(mx, 64)))
                                    : (unsigned)imax(1, imin((int64_t)sms * 8, cdiv(tiles, 8)));
      double* part = ws.take<double>((size_t)grid * 2);
      if (ws.base == nullptr) return NENMF_OK;
      if (!ws.ok) return NENMF_ERR_WORKSPACE;
      const float* Xf = reinterpret_cast<const float*>(B);
      const int kt = (int)cdiv(p, 8);
      auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
      if (((nx | mx | ldb) & 3) == 0 && al16(Xf) && al16(U1) && al16(V1) && (U2 == nullptr || al16(U2)) &&
          (V2 == nullptr || al16(V2)) && getenv("NENMF_RESID_V1") == nullptr) {
        const int kp = 8 * kt;
        const size_t stage_f = (size_t)128 * RP_XS + (size_t)kp * RP_US + (size_t)kp * RP_VS +
                               ((U2 != nullptr && U2 != U1) ? (size_t)kp * RP_US : 0) +
                               ((V2 != nullptr && V2 != V1) ? (size_t)kp * RP_VS : 0);
        const size_t smem = stage_f * RP_NS * sizeof(float);
        auto go = [&](auto kern) -> int {
          NENMF_CUDA_TRY(set_smem(kern, smem));
          kern<<<grid, 256, smem, st>>>(Xf, nx, mx, ldb, (int)p, U1, V1, U2, V2, part, gate);
          return NENMF_OK;
        };
        if (kt == 1) NENMF_TRY(go(k_resid_pipe<1>));
        else if (kt == 2) NENMF_TRY(go(k_resid_pipe<2>));
        else if (kt == 3) NENMF_TRY(go(k_resid_pipe<3>));
        else NENMF_TRY(go(k_resid_pipe<4>));
        NENMF_LAUNCH_CHECK();
        k_pair_final<<<1, 256, 0, st>>>(part, (int64_t)grid, out2, gate);
        NENMF_LAUNCH_CHECK();
        return NENMF_OK;
      }
      if (kt == 1) k_resid_mma<1><<<grid, 256, 0, st>>>(Xf, nx, mx, ldb, (int)p, U1, V1, U2, V2, part, gate);
      else if (kt == 2) k_resid_mma<2><<<grid, 256, 0, st>>>(Xf, nx, mx, ldb, (int)p, U1, V1, U2, V2, part, gate);
      else if (kt == 3) k_resid_mma<3><<<grid, 256, 0, st>>>(Xf, nx, mx, ldb, (int)p, U1, V1, U2, V2, part, gate);
      else k_resid_mma<4><<<grid, 256, 0, st>>>(Xf, nx, mx, ldb, (int)p, U1, V1, U2, V2, part, gate);
      NENMF_LAUNCH_CHECK();
      k_pair_final<<<1, 256, 0, st>>>(part, (int64_t)grid, out2, gate);
      NENMF_LAUNCH_CHECK();
      return NENMF_OK;
    }
  }
  if constexpr (sizeof(T) == 8) {
    const int64_t nx = trans ? c : r, mx = trans ? r : c;
    const double* U1 = reinterpret_cast<const double*>(trans ? F1 : At);
    const double* U2 = F2 == nullptr ? nullptr : reinterpret_cast<const double*>(trans ? F2 : At);
    const double* V1 = reinterpret_cast<const double*>(trans ? At : F1);
    const double* V2 = F2 == nullptr ? nullptr : reinterpret_cast<const double*>(trans ? At : F2);
    auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    const bool ok = p <= 32 && ((nx | mx | ldb) & 1) == 0 && getenv("NENMF_RESID_SIMT") == nullptr &&
                    (ws.base == nullptr || (al16(B) && al16(U1) && al16(V1) && (U2 == nullptr || al16(U2)) &&
                                            (V2 == nullptr || al16(V2))));
    if (ok) {
      int sms = sm_count();
      if (sms <= 0) sms = 148;
      const unsigned grid = (unsigned)imax(1, imin((int64_t)sms, cdiv(nx, 64) * cdiv(mx, 64)));
      double* part = ws.take<double>((size_t)grid * 2);
      if (ws.base == nullptr) return NENMF_OK;
      if (!ws.ok) return NENMF_ERR_WORKSPACE;
      const double* Xd = reinterpret_cast<const double*>(B);
      if (F2 == nullptr) {
        const size_t smem = (size_t)3 * (64 * RD_XS + 2 * 32 * RD_XS) * sizeof(double);
        NENMF_CUDA_TRY(set_smem(k_resid64<1>, smem));
        k_resid64<1><<<grid, 256, smem, st>>>(Xd, nx, mx, ldb, (int)p, U1, V1, nullptr, nullptr, part, gate);
      } else {
        const size_t smem = (size_t)2 * (64 * RD_XS + 4 * 32 * RD_XS) * sizeof(double);
        NENMF_CUDA_TRY(set_smem(k_resid64<2>, smem));
        k_resid64<2><<<grid, 256, smem, st>>>(Xd, nx, mx, ldb, (int)p, U1, V1, U2, V2, part, gate);
      }
      NENMF_LAUNCH_CHECK();
      k_pair_final<<<1, 256, 0, st>>>(part, (int64_t)grid, out2, gate);
      NENMF_LAUNCH_CHECK();
      return NENMF_OK;
    }
  }
  const int64_t nchunk = cdiv(r, AB_RCHUNK);
  dim3 grid((unsigned)cdiv(c, AB_CB), (unsigned)nchunk);
  double* part = ws.take<double>((size_t)grid.x * grid.y * 2);
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  auto go = [&](auto kern, int) -> int {
    kern<<<grid, RS_THREADS, 0, st>>>(At, (int)p, r, B, c, ldb, F1, F2, AB_RCHUNK, part, gate);
    return NENMF_OK;
  };
  int rc;
  if (p <= 8) rc = trans ? go(k_resid<T, 8, true>, 8) : go(k_resid<T, 8, false>, 8);
  else if (p <= 16) rc = trans ? go(k_resid<T, 16, true>, 16) : go(k_resid<T, 16, false>, 16);
  else if (p <= 24) rc = trans ? go(k_resid<T, 24, true>, 24) : go(k_resid<T, 24, false>, 24);
  else if (p <= 32) rc = trans ? go(k_resid<T, 32, true>, 32) : go(k_resid<T, 32, false>, 32);
  else rc = trans ? go(k_resid<T, 64, true>, 64) : go(k_resid<T, 64, false>, 64);
  if (rc != NENMF_OK) return rc;
  NENMF_LAUNCH_CHECK();
  k_pair_final<<<1, 256, 0, st>>>(part, (int64_t)grid.x * grid.y, out2, gate);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

// ---------------------------------------------------- sumsq / pg_sumsq ----
constexpr int RED_THREADS = 256;

inline unsigned red_grid(int64_t count) {
  return (unsigned)imax(1, imin(cdiv(count, RED_THREADS * 8), 1184));
}

template <typename T, bool PG>
__global__ void __launch_bounds__(RED_THREADS)
k_sumsq(const T* __restrict__ M, const T* __restrict__ g, int64_t count, double* __restrict__ part) {
  __shared__ double red[33];
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    double v;
    if (PG) {
      T gv = g[i];
      v = (double)(M[i] > T(0) ? gv : min0_nan(gv));
    } else {
      v = (double)M[i];
    }
    acc += v * v;
  }
  double s = block_sum(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_final_sum(const double* __restrict__ part, int64_t n, double* __restrict__ out) {
  __shared__ double red[33];
  double a = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a += part[i];
  a = block_sum(a, red);
  if (threadIdx.x == 0) *out = a;
}

template <typename T>
int sumsq(Arena& ws, const T* M, const T* g, int64_t count, double* out, cudaStream_t st) {
  if (count < 1) return NENMF_ERR_DIM;
  unsigned grid = red_grid(count);
  double* part = ws.take<double>(grid);
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  if (g != nullptr) k_sumsq<T, true><<<grid, RED_THREADS, 0, st>>>(M, g, count, part);
  else k_sumsq<T, false><<<grid, RED_THREADS, 0, st>>>(M, g, count, part);
  NENMF_LAUNCH_CHECK();
  k_final_sum<<<1, 256, 0, st>>>(part, grid, out);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

// ------------------------------------------------------------ scan flags ----
// One read of a (rows x cols, leading dimension ld) matrix: *nonzero = 1 when
// some element is nonzero (compression.py:109-117's X.any()), *negative = 1
// when some element is < 0 (FactorPair's sign check, factorize.py:44-48; NaN
// is not negative there either).  Either flag may be null; they are only
// ever raised, so the caller zeroes them.
template <typename T>
__global__ void __launch_bounds__(RED_THREADS)
k_scan_flags(const T* __restrict__ M, int64_t rows, int64_t cols, int64_t ld, int* __restrict__ nonzero,
             int* __restrict__ negative) {
  bool nz = false, ng = false;
  const int64_t count = rows * cols;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    const int64_t r = ld == cols ? 0 : i / cols;
    const T v = ld == cols ? M[i] : M[r * ld + (i - r * cols)];
    nz |= v != T(0);
    ng |= v < T(0);
  }
  const bool lane0 = (threadIdx.x & 31) == 0;
  if (nonzero != nullptr && __any_sync(0xffffffffu, nz) && lane0) *nonzero = 1;
  if (negative != nullptr && __any_sync(0xffffffffu, ng) && lane0) *negative = 1;
}

template <typename T>
int scan_flags(const T* M, int64_t rows, int64_t cols, int64_t ld, int* nonzero, int* negative, cudaStream_t st) {
  if (rows < 0 || cols < 0 || (rows > 0 && ld < cols)) return NENMF_ERR_DIM;
  if (rows * cols == 0) return NENMF_OK;
  k_scan_flags<T><<<red_grid(rows * cols), RED_THREADS, 0, st>>>(M, rows, cols, ld, nonzero, negative);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

// ------------------------------------------------------------- transpose ----
// dst (cols x rows) = src (rows x cols, leading dimension ld)^T through 32 x 32
// shared-memory tiles (both sides coalesced).  Used to bring factors given as
// n x p into the library's p x n panel layout without a host round trip.
template <typename T>
__global__ void k_transpose(const T* __restrict__ src, int64_t rows, int64_t cols, int64_t ld, T* __restrict__ dst) {
  __shared__ T tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = src[r * ld + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[c * rows + r] = tile[threadIdx.x][i];
  }
}

template <typename T>
int transpose(const T* src, int64_t rows, int64_t cols, int64_t ld, T* dst, cudaStream_t st) {
  if (rows < 0 || cols < 0 || (rows > 0 && ld < cols)) return NENMF_ERR_DIM;
  if (rows * cols == 0) return NENMF_OK;
  if (cdiv(rows, 32) > 65535) return NENMF_ERR_UNSUPPORTED;
  k_transpose<T><<<dim3((unsigned)cdiv(cols, 32), (unsigned)cdiv(rows, 32)), dim3(32, 8), 0, st>>>(src, rows, cols,
                                                                                                   ld, dst);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

// ------------------------------------------------------------------ wfv ----
template <typename T>
__global__ void k_wfv(const T* __restrict__ W, int p, const T* __restrict__ F, int64_t c,
                      const T* __restrict__ V, T* __restrict__ G) {
  extern __shared__ double smem_d[];
  T* Ws = reinterpret_cast<T*>(smem_d);
  for (int i = threadIdx.x; i < p * p; i += blockDim.x) Ws[i] = W[i];
  __syncthreads();
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= c) return;
  for (int i = 0; i < p; ++i) {
    T acc = T(0);
    for (int l = 0; l < p; ++l) acc = fma_acc(Ws[i * p + l], F[(int64_t)l * c + j], acc);
    G[(int64_t)i * c + j] = op_sub(acc, V[(int64_t)i * c + j]);
  }
}

template <typename T>
int wf_minus_v(const T* W, int64_t p, const T* F, int64_t c, const T* V, T* G, cudaStream_t st) {
  size_t smem = (size_t)p * p * sizeof(T);
  if (smem > 200 * 1024) return NENMF_ERR_UNSUPPORTED;
  NENMF_CUDA_TRY(set_smem(k_wfv<T>, smem));
  k_wfv<T><<<(unsigned)cdiv(c, 128), 128, smem, st>>>(W, (int)p, F, c, V, G);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

// explicit instantiations
#define NENMF_INST_SKINNY(T)                                                                              \
  template int abt<T>(Arena&, const T*, int64_t, const T*, int64_t, int64_t, T*, cudaStream_t);           \
  template int gram_d<T>(Arena&, const T*, int64_t, int64_t, double*, cudaStream_t);                      \
  template int ab<T>(Arena&, const T*, int64_t, int64_t, const T*, int64_t, int64_t, bool, T*,            \
                     cudaStream_t);                                                                       \
  template int resid<T>(Arena&, const T*, int64_t, int64_t, const T*, int64_t, int64_t, bool, const T*,   \
                        const T*, double*, const int*, cudaStream_t);                                     \
  template int sumsq<T>(Arena&, const T*, const T*, int64_t, double*, cudaStream_t);                      \
  template int wf_minus_v<T>(const T*, int64_t, const T*, int64_t, const T*, T*, cudaStream_t);           \
  template int scan_flags<T>(const T*, int64_t, int64_t, int64_t, int*, int*, cudaStream_t);              \
  template int transpose<T>(const T*, int64_t, int64_t, int64_t, T*, cudaStream_t);
NENMF_INST_SKINNY(double)
NENMF_INST_SKINNY(float)

}  // namespace nenmf
