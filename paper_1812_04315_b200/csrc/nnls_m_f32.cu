// Instantiates the tensor-core persistent solver for float (3xTF32 mma).
#include "nnls_mma.cuh"

namespace nenmf {
NENMF_NNLS_MMA_IMPL(float)
}  // namespace nenmf
