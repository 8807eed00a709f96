// Instantiates the persistent solver for float, 4 thread(s) per column.
#include "nnls_kernel.cuh"

namespace nenmf {
NENMF_NNLS_TPC_IMPL(float, 4)
}  // namespace nenmf
