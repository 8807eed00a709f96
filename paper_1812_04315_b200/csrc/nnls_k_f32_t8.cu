// Instantiates the persistent solver for float, 8 thread(s) per column.
#include "nnls_kernel.cuh"

namespace nenmf {
NENMF_NNLS_TPC_IMPL(float, 8)
}  // namespace nenmf
