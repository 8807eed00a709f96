// Instantiates the persistent solver for float, 16 thread(s) per column.
#include "nnls_kernel.cuh"

namespace nenmf {
NENMF_NNLS_TPC_IMPL(float, 16)
}  // namespace nenmf
