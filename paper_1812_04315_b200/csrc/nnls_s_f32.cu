// Instantiates the streamed tensor-core solver (FP32, p <= 32).
#include "nnls_stream.cuh"
