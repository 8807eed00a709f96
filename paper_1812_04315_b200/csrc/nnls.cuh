// Internal entry points of the inner solver (nnls.cu).
#pragma once
#include "common.cuh"

namespace nenmf {

struct GroupDev;
// Host view of a rank group (C ABI nenmf_group, include/nenmf_b200.h).
struct GroupHost {
  int ranks, rank0, nvr, watchdog_s;
  int64_t col0[9];
  void* xch[8];
  unsigned long long epoch;
};

// Whole solve_nnls (nnls.py:119-227).  F_out receives the returned iterate;
// F0 and F_out must not alias.  The caller zeroes *st before the first use.
// Optional next product (Pt != nullptr): Pout (p x nup) = F_out Pt^T with Pt
// (nup x c) -- the operand of the next half-step (F R or L G,
// factorize.py:110,113), formed inside the solver launch when it is fused.
// Optional Xpre (FP32): the prepared copy (nenmf_prepare_x) of the X that B
// is (or whose transpose B is); V = A^T B then comes from one tensor-core
// pass over it (the vanilla half-steps, factorize.py:94-98).
template <typename T>
int solve_nnls(Arena& ws, const T* At, int64_t r, int64_t p, const T* B, int64_t c, int64_t ldb, bool trans,
               const T* F0, T* Fout, int max_iter, double grad_tol, double safety, const double* pvec,
               int pcount, int pmax, double ptol, nenmf_device_status* st, cudaStream_t s,
               const T* Pt = nullptr, int64_t nup = 0, T* Pout = nullptr, const uint8_t* Xpre = nullptr,
               const GroupHost* grp = nullptr);

template <typename T>
int spectral_norm_sq(Arena& ws, const T* At, int64_t r, int64_t p, const double* pvec, int pcount, int pmax,
                     double tol, double* out, nenmf_device_status* st, cudaStream_t s);

template <typename T>
int gradient(Arena& ws, const T* At, int64_t r, int64_t p, const T* B, int64_t c, int64_t ldb, bool trans,
             const T* F, T* grad, cudaStream_t s);

}  // namespace nenmf
