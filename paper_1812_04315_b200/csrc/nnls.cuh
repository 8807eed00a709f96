// Internal entry points of the inner solver (nnls.cu).
#pragma once
#include "common.cuh"

namespace nenmf {

// Whole solve_nnls (nnls.py:119-227).  F_out receives the returned iterate;
// F0 and F_out must not alias.  The caller zeroes *st before the first use.
template <typename T>
int solve_nnls(Arena& ws, const T* At, int64_t r, int64_t p, const T* B, int64_t c, int64_t ldb, bool trans,
               const T* F0, T* Fout, int max_iter, double grad_tol, double safety, const double* pvec,
               int pcount, int pmax, double ptol, nenmf_device_status* st, cudaStream_t s);

template <typename T>
int spectral_norm_sq(Arena& ws, const T* At, int64_t r, int64_t p, const double* pvec, int pcount, int pmax,
                     double tol, double* out, nenmf_device_status* st, cudaStream_t s);

template <typename T>
int gradient(Arena& ws, const T* At, int64_t r, int64_t p, const T* B, int64_t c, int64_t ldb, bool trans,
             const T* F, T* grad, cudaStream_t s);

}  // namespace nenmf
