// Internal entry points of the randomized-subspace-iteration kernels (rsi.cu).
#pragma once
#include "common.cuh"

namespace nenmf {

template <typename T>
int dual_pass(Arena& ws, const T* X, int64_t n, int64_t m, int64_t ldx, const T* At, const T* Bt, int64_t k,
              T* Yt, T* Zt, cudaStream_t s);

template <typename T>
int orthonormalize(Arena& ws, T* Pt, int64_t rows, int64_t k, nenmf_device_status* st, cudaStream_t s);

template <typename T>
int rsi(Arena& ws, const T* X, int64_t n, int64_t m, int64_t ldx, const T* omega_l_t, const T* omega_r, int64_t nu,
        int q, T* L, T* Rt, nenmf_device_status* st, cudaStream_t s);

template <typename T>
int compress(Arena& ws, const T* X, int64_t n, int64_t m, int64_t ldx, const T* L, const T* Rt, int64_t nu, T* XL,
             T* XRt, cudaStream_t s);

}  // namespace nenmf
