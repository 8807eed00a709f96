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
        int q, T* L, T* Rt, nenmf_device_status* st, cudaStream_t s, const uint8_t* Xpre = nullptr,
        int power = 0);

template <typename T>
int compress(Arena& ws, const T* X, int64_t n, int64_t m, int64_t ldx, const T* L, const T* Rt, int64_t nu, T* XL,
             T* XRt, cudaStream_t s, const uint8_t* Xpre = nullptr);

// decomposed CholeskyQR2 stages (qr.cu) for row-sharded panels
template <typename T>
int panel_gram(Arena& ws, const T* Pt, int64_t rows, int64_t k, double* G, cudaStream_t s);
int panel_factor(const double* G, int64_t k, int pivot, double* R, int* meta, nenmf_device_status* st,
                 cudaStream_t s);
template <typename T>
int panel_trsm(const T* Pin_t, int64_t rows, int64_t k, const double* R, const int* meta, T* Pout_t, int64_t row0,
               int full_only, cudaStream_t s);

// FP32 tensor-core pass over a pre-split X (dual_tc.cu)
bool tc_pass_eligible(int64_t n, int64_t m, int64_t k);
size_t tc_presplit_bytes(int64_t n, int64_t m);
int tc_presplit(const float* X, int64_t n, int64_t m, int64_t ldx, uint8_t* Xs, cudaStream_t s,
                int* nonzero = nullptr);
int dual_pass_tc_pre(Arena& ws, const uint8_t* Xs, int64_t n, int64_t m, const float* At, const float* Bt,
                     int64_t k, float* Yt, float* Zt, cudaStream_t s);
// ||X - U^T V||^2 over the prepared X on the tensor cores (U: k x n, V: k x m)
// -> out[0]; with a second candidate -> out[1]: W replaces U (w_side 1) or V (w_side 2)
int resid_tc_pre(Arena& ws, const uint8_t* Xs, int64_t n, int64_t m, const float* U, const float* V, int64_t k,
                 double* out, cudaStream_t s, const float* W = nullptr, int w_side = 0, const int* gate = nullptr);

}  // namespace nenmf
