// The reference's Gaussian sketch draws on the device, bit-identical to NumPy.
//
// compression.py:130-132 draws Omega_L (m x nu) then Omega_R (nu x n) from
// ONE stream: numpy.random.default_rng(seed).standard_normal, i.e. PCG64
// (128-bit LCG, XSL-RR output; numpy/random/src/pcg64) feeding the 256-layer
// ziggurat of random_standard_normal (numpy/random/src/distributions).  The
// restatement here consumes the raw 64-bit stream exactly like NumPy:
//   r = next64; idx = r & 0xff; sign = bit 8; rabs = bits 9..60
//   x = rabs * wi[idx] (negated by sign); accept if rabs < ki[idx]   (~99.3 %)
//   idx == 0: tail loop on two next_double() per attempt
//   else    : accept if (fi[idx-1]-fi[idx]) u + fi[idx] < exp(-x^2/2), else redraw
// The three 256-entry tables are NumPy's own (read from the installed NumPy by
// the host layer and passed in).  The wedge test of the ~0.7 % slow-path
// draws uses CUDA's exp, which agrees with glibc's decisions except within an
// ulp of the boundary (tests: bit-identical); the tail uses glibc_log1p.
//
// Parallelisation of the variable-length stream: the raw positions are cut
// into chunks of S.  k_zig_scan walks every chunk from its first position
// (PCG64 jump-ahead, one thread per chunk) and records which of its first 64
// positions start a draw, how many draws start inside the chunk and where the
// walk leaves it.  k_zig_link (one thread) chains the chunks: a chunk entered
// at a position its own walk also starts a draw at has the same tail (walks
// that meet stay merged), so only entry points off that walk need a re-walk;
// k_zig_link_par does the common case as a parallel scan.
// k_zig_emit walks each chunk again from its true entry and writes draw i to
// Omega_L^T (i < m nu, transposed) or Omega_R; draws from the ziggurat tail
// (~1 in 4000) use glibc_log1p below, the C library's own log1p restated
// operation for operation, so their values (and the accept tests that use
// them) are NumPy's exactly; no host fix-up and no synchronisation.
// A chunk whose re-walk does not merge within 64 positions (never observed)
// sets *ok = 0 and the host redraws with NumPy.
#include "common.cuh"
#include "glibc_log1p.cuh"

namespace nenmf {

namespace zig {

typedef unsigned __int128 u128;
constexpr u128 MULT = ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
constexpr double ZR = 3.6541528853610087963519472518;
constexpr double ZINVR = 0.27366123732975827203338247596;

struct Tables {
  double fi[256], wi[256];
  uint64_t ki[256];
};

// state after `delta` further steps of s' = MULT s + inc
__device__ __forceinline__ u128 advance(u128 s, u128 inc, uint64_t delta) {
  u128 am = 1, ap = 0, cm = MULT, cp = inc;
  while (delta) {
    if (delta & 1) {
      am *= cm;
      ap = ap * cm + cp;
    }
    cp = (cm + 1) * cp;
    cm *= cm;
    delta >>= 1;
  }
  return am * s + ap;
}

struct Stream {
  u128 s, inc;
  __device__ __forceinline__ uint64_t next() {
    s = s * MULT + inc;
    const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    const uint64_t x = hi ^ lo;
    const unsigned rot = (unsigned)(hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __device__ __forceinline__ double next_double() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
};

// one draw starting at the stream's current position; `used` = raw values consumed.
// A draw from the tail (idx 0) reports its accepted 53-bit uniform and sign in
// *tail (u53 << 1 | negative), else *tail = 0 (diagnostics: the tail list).
__device__ __forceinline__ double draw(Stream& g, const Tables& T, int& used, uint64_t* tail = nullptr) {
  used = 0;
  if (tail != nullptr) *tail = 0;
  for (;;) {
    uint64_t r = g.next();
    ++used;
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = (double)rabs * T.wi[idx];
    if (sign) x = -x;
    if (rabs < T.ki[idx]) return x;
    if (idx == 0) {
      for (;;) {
        const uint64_t u53 = g.next() >> 11;
        const double xx = __dmul_rn(-ZINVR, glibc_log1p(-((double)u53 * (1.0 / 9007199254740992.0))));
        const double yy = -glibc_log1p(-g.next_double());
        used += 2;
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
          const bool neg = (rabs >> 8) & 1;
          if (tail != nullptr) *tail = (u53 << 1) | (neg ? 1ull : 0ull) | (1ull << 63);
          return neg ? -__dadd_rn(ZR, xx) : __dadd_rn(ZR, xx);
        }
      }
    } else {
      const double u = g.next_double();
      ++used;
      if (__dadd_rn(__dmul_rn(__dsub_rn(T.fi[idx - 1], T.fi[idx]), u), T.fi[idx]) <
          exp(__dmul_rn(__dmul_rn(-0.5, x), x)))
        return x;
    }
  }
}

struct ChunkScan {
  unsigned long long mask;  // bit e: the walk from the chunk start starts a draw at offset e (< 64)
  int count;                // draws starting in [0, S) on that walk
  int exit;                 // first start offset >= S, minus S
};

__global__ void k_zig_scan(const Tables* __restrict__ T, uint64_t s_lo, uint64_t s_hi, uint64_t i_lo, uint64_t i_hi,
                           int64_t nchunks, int S, ChunkScan* __restrict__ out) {
  __shared__ Tables t;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    t.fi[i] = T->fi[i];
    t.wi[i] = T->wi[i];
    t.ki[i] = T->ki[i];
  }
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  Stream g;
  g.inc = ((u128)i_hi << 64) | i_lo;
  g.s = advance(((u128)s_hi << 64) | s_lo, g.inc, (uint64_t)c * (uint64_t)S);
  unsigned long long mask = 0;
  int pos = 0, count = 0;
  while (pos < S) {
    if (pos < 64) mask |= 1ull << pos;
    int used;
    draw(g, t, used);
    pos += used;
    ++count;
  }
  out[c].mask = mask;
  out[c].count = count;
  out[c].exit = pos - S;
}

// one thread chains the chunks (true entry offset and first draw index of
// each); the block stages the chunk summaries through shared memory so the
// sequential walk reads them at LDS latency
constexpr int LINK_TILE = 2048;
__global__ void __launch_bounds__(256) k_zig_link(const Tables* __restrict__ T, uint64_t s_lo, uint64_t s_hi,
                                                  uint64_t i_lo, uint64_t i_hi, const ChunkScan* __restrict__ sc,
                                                  int64_t nchunks, int S, int64_t need, int* __restrict__ entry,
                                                  int64_t* __restrict__ base, int* __restrict__ ok,
                                                  const int* __restrict__ seq_needed) {
  if (seq_needed != nullptr && *seq_needed == 0) return;  // k_zig_link_par chained every chunk
  __shared__ ChunkScan tile[LINK_TILE];
  __shared__ int s_e, s_good;
  __shared__ long long s_b;
  if (threadIdx.x == 0) {
    s_e = 0;
    s_b = 0;
    s_good = 1;
  }
  for (int64_t t0 = 0; t0 < nchunks; t0 += LINK_TILE) {
    const int nt = (int)imin(LINK_TILE, nchunks - t0);
    __syncthreads();
    for (int i = threadIdx.x; i < nt; i += blockDim.x) tile[i] = sc[t0 + i];
    __syncthreads();
    if (threadIdx.x != 0 || !s_good) continue;
    int e = s_e;
    int64_t b = s_b;
    int good = 1;
    for (int i = 0; i < nt; ++i) {
      const int64_t c = t0 + i;
      const ChunkScan s = tile[i];
      entry[c] = e;
      base[c] = b;
      if (e == 0) {  // the common case: the chunk's own walk
        b += s.count;
        e = s.exit;
        continue;
      }
      if (e < 64 && ((s.mask >> e) & 1ull)) {  // merged with the chunk's walk
        b += s.count - __popcll(s.mask & ((1ull << e) - 1ull));
        e = s.exit;
        continue;
      }
      // re-walk from the true entry until it meets the chunk's walk (rare)
      Stream g;
      g.inc = ((u128)i_hi << 64) | i_lo;
      g.s = advance(((u128)s_hi << 64) | s_lo, g.inc, (uint64_t)c * (uint64_t)S + (uint64_t)e);
      int pos = e, extra = 0;
      while (pos < S && !(pos < 64 && ((s.mask >> pos) & 1ull))) {
        if (pos >= 64) break;
        int used;
        draw(g, *T, used);
        pos += used;
        ++extra;
      }
      if (pos >= S) {  // the whole chunk walked from the entry
        b += extra;
        e = pos - S;
      } else if (pos < 64 && ((s.mask >> pos) & 1ull)) {
        b += extra + s.count - __popcll(s.mask & ((1ull << pos) - 1ull));
        e = s.exit;
      } else {
        good = 0;
        break;
      }
    }
    s_e = e;
    s_b = b;
    s_good = good;
  }
  __syncthreads();
  if (threadIdx.x == 0) *ok = (s_good && s_b >= need) ? 1 : 0;
}

// The chaining above is a scan in disguise: a chunk entered at an offset
// its own walk also starts a draw at contributes count - (draws of its walk
// before the entry) and leaves at its own exit, whatever happened before; a
// chunk entered off its walk is re-walked from the entry until the two walks
// meet (about one chunk boundary in 10^4) and then leaves at its own exit
// too.  So with every chunk's entry taken as its predecessor's own exit, all
// chunks are counted in parallel (one block, a prefix sum for the first draw
// indices).  Only a re-walk that leaves the chunk before meeting its walk
// (never observed) changes an exit; then the sequential k_zig_link redoes
// the chaining after this kernel.
constexpr int LINKP_THREADS = 1024;
__device__ __forceinline__ int chunk_contribution(const Tables& T, uint64_t s_lo, uint64_t s_hi, uint64_t i_lo,
                                                  uint64_t i_hi, int64_t c, int S, int e, const ChunkScan& s,
                                                  bool& exit_changed) {
  if (e == 0) return s.count;
  if (e < 64 && ((s.mask >> e) & 1ull)) return s.count - __popcll(s.mask & ((1ull << e) - 1ull));
  Stream g;
  g.inc = ((u128)i_hi << 64) | i_lo;
  g.s = advance(((u128)s_hi << 64) | s_lo, g.inc, (uint64_t)c * (uint64_t)S + (uint64_t)e);
  int pos = e, extra = 0;
  while (pos < S && pos < 64 && !((s.mask >> pos) & 1ull)) {
    int used;
    draw(g, T, used);
    pos += used;
    ++extra;
  }
  if (pos < 64 && pos < S && ((s.mask >> pos) & 1ull)) return extra + s.count - __popcll(s.mask & ((1ull << pos) - 1ull));
  exit_changed = true;
  return 0;
}

__global__ void __launch_bounds__(LINKP_THREADS) k_zig_link_par(const Tables* __restrict__ T, uint64_t s_lo,
                                                                uint64_t s_hi, uint64_t i_lo, uint64_t i_hi,
                                                                const ChunkScan* __restrict__ sc, int64_t nchunks,
                                                                int S, int64_t need, int* __restrict__ entry,
                                                                int64_t* __restrict__ base, int* __restrict__ ok,
                                                                int* __restrict__ seq_needed) {
  __shared__ Tables tb;
  __shared__ long long wsum[LINKP_THREADS / 32];
  __shared__ int s_bad;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  for (int i = t; i < 256; i += blockDim.x) {
    tb.fi[i] = T->fi[i];
    tb.wi[i] = T->wi[i];
    tb.ki[i] = T->ki[i];
  }
  if (t == 0) s_bad = 0;
  __syncthreads();
  const int64_t per = (nchunks + LINKP_THREADS - 1) / LINKP_THREADS;
  const int64_t c0 = min(nchunks, (int64_t)t * per), c1 = min(nchunks, c0 + per);
  long long mine = 0;
  bool bad = false;
  for (int64_t c = c0; c < c1; ++c) {
    const int e = c == 0 ? 0 : sc[c - 1].exit;
    mine += chunk_contribution(tb, s_lo, s_hi, i_lo, i_hi, c, S, e, sc[c], bad);
  }
  if (bad) s_bad = 1;
  // block-wide exclusive scan of the per-thread counts (thread order = chunk order)
  long long incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    long long v = wsum[lane], w = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long u = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += u;
    }
    wsum[lane] = w - v;  // exclusive
  }
  __syncthreads();
  long long b = wsum[wid] + incl - mine;
  if (s_bad) {
    if (t == 0) *seq_needed = 1;
    return;
  }
  for (int64_t c = c0; c < c1; ++c) {
    const int e = c == 0 ? 0 : sc[c - 1].exit;
    entry[c] = e;
    base[c] = b;
    b += chunk_contribution(tb, s_lo, s_hi, i_lo, i_hi, c, S, e, sc[c], bad);
  }
  if (t == LINKP_THREADS - 1) {
    *seq_needed = 0;
    *ok = b >= need ? 1 : 0;
  }
}

template <typename TO>
__global__ void k_zig_emit(const Tables* __restrict__ T, uint64_t s_lo, uint64_t s_hi, uint64_t i_lo, uint64_t i_hi,
                           int64_t nchunks, int S, const int* __restrict__ entry, const int64_t* __restrict__ base,
                           int* __restrict__ ok, int64_t n, int64_t m, int64_t nu, TO* __restrict__ olt,
                           TO* __restrict__ orr, unsigned long long* __restrict__ tails, int cap) {
  __shared__ Tables t;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    t.fi[i] = T->fi[i];
    t.wi[i] = T->wi[i];
    t.ki[i] = T->ki[i];
  }
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks || *ok == 0) return;
  const int64_t nl = m * nu, need = nl + nu * n;
  int64_t i = base[c];
  if (i >= need) return;
  Stream g;
  g.inc = ((u128)i_hi << 64) | i_lo;
  int pos = entry[c];
  g.s = advance(((u128)s_hi << 64) | s_lo, g.inc, (uint64_t)c * (uint64_t)S + (uint64_t)pos);
  while (pos < S && i < need) {
    int used;
    uint64_t tl;
    const double x = draw(g, t, used, &tl);
    pos += used;
    if (tl != 0) {  // [count][(index, u53 << 1 | neg) pairs]
      const unsigned long long slot = atomicAdd(&tails[0], 1ull);
      if (slot < (unsigned long long)cap) {
        tails[1 + 2 * slot] = (unsigned long long)i;
        tails[2 + 2 * slot] = tl & ~(1ull << 63);
      } else {
        *ok = 0;
      }
    }
    if (i < nl) {
      const int64_t row = i / nu, col = i - row * nu;  // Omega_L (m x nu) -> Omega_L^T (nu x m)
      olt[col * m + row] = (TO)x;
    } else {
      orr[i - nl] = (TO)x;
    }
    ++i;
  }
}

}  // namespace zig

int sketch_tail_capacity(int64_t n, int64_t m, int64_t nu) { return (int)((m + n) * nu / 512 + 256); }

int sketch_draws_device(int dtype, const void* tables, uint64_t s_lo, uint64_t s_hi, uint64_t i_lo, uint64_t i_hi,
                        int64_t n, int64_t m, int64_t nu, void* olt, void* orr, int* ok, unsigned long long* tails,
                        Arena& ws, cudaStream_t s) {
  using namespace zig;
  if (n < 1 || m < 1 || nu < 1) return NENMF_ERR_DIM;
  const int64_t need = (m + n) * nu;
  // chunk length: short walks (latency of the scan and emit passes), at
  // most ~64 K chunks for the parallel link; >= 64 so that an entry offset
  // (a few positions) always lies inside the chunk's start mask
  int S = 64;
  while (S < 4096 && need / S > 65536) S *= 2;
  const int64_t nchunks = (int64_t)((double)need * 1.03 / S) + 8;
  ChunkScan* sc = ws.take<ChunkScan>((size_t)nchunks);
  int* entry = ws.take<int>((size_t)nchunks);
  int64_t* base = ws.take<int64_t>((size_t)nchunks);
  int* seq = ws.take<int>(4);
  if (ws.base == nullptr) return NENMF_OK;
  if (!ws.ok) return NENMF_ERR_WORKSPACE;
  const Tables* T = static_cast<const Tables*>(tables);
  const int cap = sketch_tail_capacity(n, m, nu);
  NENMF_CUDA_TRY(cudaMemsetAsync(tails, 0, sizeof(unsigned long long), s));
  const unsigned blocks = (unsigned)cdiv(nchunks, 64);
  k_zig_scan<<<blocks, 64, 0, s>>>(T, s_lo, s_hi, i_lo, i_hi, nchunks, S, sc);
  NENMF_LAUNCH_CHECK();
  k_zig_link_par<<<1, LINKP_THREADS, 0, s>>>(T, s_lo, s_hi, i_lo, i_hi, sc, nchunks, S, need, entry, base, ok,
                                              seq);
  NENMF_LAUNCH_CHECK();
  k_zig_link<<<1, 256, 0, s>>>(T, s_lo, s_hi, i_lo, i_hi, sc, nchunks, S, need, entry, base, ok, seq);
  NENMF_LAUNCH_CHECK();
  if (dtype == NENMF_F64)
    k_zig_emit<double><<<blocks, 64, 0, s>>>(T, s_lo, s_hi, i_lo, i_hi, nchunks, S, entry, base, ok, n, m, nu,
                                             static_cast<double*>(olt), static_cast<double*>(orr), tails, cap);
  else
    k_zig_emit<float><<<blocks, 64, 0, s>>>(T, s_lo, s_hi, i_lo, i_hi, nchunks, S, entry, base, ok, n, m, nu,
                                            static_cast<float*>(olt), static_cast<float*>(orr), tails, cap);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

// NumPy's Generator.random (float64): one raw value per draw, (r >> 11) 2^-53.
// Thread t owns draws [t CH, (t + 1) CH): one jump-ahead, then sequential.
constexpr int UNI_CH = 32;
__global__ void k_uniform(uint64_t s_lo, uint64_t s_hi, uint64_t i_lo, uint64_t i_hi, int64_t count,
                          double* __restrict__ out, int* __restrict__ zero) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i0 = t * UNI_CH;
  if (i0 >= count) return;
  const zig::u128 inc = ((zig::u128)i_hi << 64) | i_lo;
  zig::Stream g{zig::advance(((zig::u128)s_hi << 64) | s_lo, inc, (uint64_t)i0), inc};
  const int64_t i1 = i0 + UNI_CH < count ? i0 + UNI_CH : count;
  bool z = false;
  for (int64_t i = i0; i < i1; ++i) {
    const double v = g.next_double();
    z |= v == 0.0;
    out[i] = v;
  }
  if (z) *zero = 1;
}

}  // namespace nenmf

extern "C" {

int nenmf_uniform_draws(uint64_t state_lo, uint64_t state_hi, uint64_t inc_lo, uint64_t inc_hi, int64_t count,
                        double* out, int* zero, void* stream) {
  if (count < 0 || (count > 0 && (out == nullptr || zero == nullptr))) return NENMF_ERR_VALUE;
  if (count == 0) return NENMF_OK;
  const int64_t threads = (count + nenmf::UNI_CH - 1) / nenmf::UNI_CH;
  nenmf::k_uniform<<<(unsigned)((threads + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      state_lo, state_hi, inc_lo, inc_hi, count, out, zero);
  NENMF_LAUNCH_CHECK();
  return NENMF_OK;
}

size_t nenmf_sketch_draws_workspace_bytes(int64_t n, int64_t m, int64_t nu) {
  nenmf::Arena a(nullptr, 0);
  nenmf::sketch_draws_device(NENMF_F64, nullptr, 0, 0, 0, 0, n, m, nu, nullptr, nullptr, nullptr, nullptr, a,
                             nullptr);
  return a.used + 256;
}

int64_t nenmf_sketch_tail_capacity(int64_t n, int64_t m, int64_t nu) { return nenmf::sketch_tail_capacity(n, m, nu); }

int nenmf_sketch_draws(int dtype, const void* tables, uint64_t state_lo, uint64_t state_hi, uint64_t inc_lo,
                       uint64_t inc_hi, int64_t n, int64_t m, int64_t nu, void* omega_l_t, void* omega_r, int* ok,
                       unsigned long long* tails, void* ws, size_t ws_bytes, void* stream) {
  if (tables == nullptr || omega_l_t == nullptr || omega_r == nullptr || ok == nullptr || tails == nullptr ||
      ws == nullptr)
    return NENMF_ERR_VALUE;
  if (dtype != NENMF_F64 && dtype != NENMF_F32) return NENMF_ERR_VALUE;
  nenmf::Arena a(ws, ws_bytes);
  return nenmf::sketch_draws_device(dtype, tables, state_lo, state_hi, inc_lo, inc_hi, n, m, nu, omega_l_t, omega_r,
                                    ok, tails, a, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
