// Instantiates the tensor-core persistent solver for double (f64 mma).
#include "nnls_mma.cuh"

namespace nenmf {
NENMF_NNLS_MMA_IMPL(double)
}  // namespace nenmf
