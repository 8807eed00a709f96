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

bool xpass_timing_begin(cudaEvent_t* e0, cudaEvent_t* e1);

int dual_pass_f64(Arena& ws, const double* X, int64_t n, int64_t m, int64_t ldx, const double* At,
                  const double* Bt, int64_t k, double* Yt, double* Zt, cudaStream_t s) {
  using namespace d64;
  // opt-in (NENMF_DUAL64_FUSED=1) until it beats the two one-product kernels:
  // measured 0.79-0.81 ms per cfg2 pass (15 TF/s, 41 % of the DMMA peak) vs
  // 0.70 ms for k_xv64 + k_ux64, although it reads X once (DRAM 14 % busy)
  static const bool on = getenv("NENMF_DUAL64_FUSED") != nullptr;
  if (!on || k < 1 || k > 32 || At == nullptr || Bt == nullptr) return NENMF_ERR_UNSUPPORTED;
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (((n | m | ldx) & 1) != 0 || (ws.base != nullptr && (!al16(X) || !al16(At) || !al16(Bt))))
    return NENMF_ERR_UNSUPPORTED;
  int sms = sm_count();
  if (sms <= 0) sms = 148;
  const int n_rt = (int)cdiv(n, T), n_ct = (int)cdiv(m, T);
  const int nbands = (int)cdiv(n_ct, CT);
  // row chunks: about two units per SM (balance), at least one row tile each
  const int nrc = (int)imax(1, imin(n_rt, cdiv(2 * sms, nbands)));
  const int rchunk = (int)cdiv(n_rt, nrc);
  const int nrc_used = (int)cdiv(n_rt, rchunk);
  const int64_t nunits = (int64_t)nbands * nrc_used;
  double* Yslab = ws.take<double>((size_t)nbands * k * n);
  double* Zslab = ws.take<double>((size_t)nrc_used * k * m);
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  const size_t smem = (size_t)NS * STAGE * sizeof(double);
  NENMF_CUDA_TRY(set_smem(k_dual64, smem));
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  const bool timed = xpass_timing_begin(&ev0, &ev1);
  if (timed) cudaEventRecord(ev0, s);
  k_dual64<<<(unsigned)imin(nunits, (int64_t)sms), THREADS, smem, s>>>(X, n, m, ldx, At, Bt, (int)k, n_ct, nbands,
                                                                        rchunk, nunits, Yslab, Zslab);
  NENMF_LAUNCH_CHECK();
  if (timed) cudaEventRecord(ev1, s);
  const int64_t cy = k * n, cz = k * m;
  k_slab_sum64<<<(unsigned)cdiv(cy + cz, 256), 256, 0, s>>>(Yslab, nbands, cy, Yt, Zslab, nrc_used, cz, Zt);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

}  // namespace nenmf
