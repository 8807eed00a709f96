// Internal (C++) entry points of the skinny-product and reduction kernels.
// Every function carves its scratch from `ws`; called with ws.base == nullptr
// it only sizes the scratch (dry run, no launch).
#pragma once
#include "common.cuh"

namespace nenmf {

template <typename T>
int abt(Arena& ws, const T* A, int64_t p, const T* B, int64_t q, int64_t K, T* C, cudaStream_t st);

// G (p x p, double) = A A^T for A (p x K): Gram of a short-major panel
template <typename T>
int gram_d(Arena& ws, const T* A, int64_t p, int64_t K, double* G, cudaStream_t st);

template <typename T>
int ab(Arena& ws, const T* At, int64_t p, int64_t r, const T* B, int64_t c, int64_t ldb, bool trans,
       T* V, cudaStream_t st);

// out2[0] = sum (At^T F1 - B)^2, out2[1] = same for F2 (0 if F2 == nullptr);
// the kernels return immediately when gate != nullptr && *gate == 0.
template <typename T>
int resid(Arena& ws, const T* At, int64_t p, int64_t r, const T* B, int64_t c, int64_t ldb, bool trans,
          const T* F1, const T* F2, double* out2, const int* gate, cudaStream_t st);

// sum M^2 (g == nullptr) or sum PG(M, g)^2 -> *out
template <typename T>
int sumsq(Arena& ws, const T* M, const T* g, int64_t count, double* out, cudaStream_t st);
template <typename T>
int scan_flags(const T* M, int64_t rows, int64_t cols, int64_t ld, int* nonzero, int* negative, cudaStream_t st);
template <typename T>
int transpose(const T* src, int64_t rows, int64_t cols, int64_t ld, T* dst, cudaStream_t st);

template <typename T>
int wf_minus_v(const T* W, int64_t p, const T* F, int64_t c, const T* V, T* G, cudaStream_t st);

}  // namespace nenmf
