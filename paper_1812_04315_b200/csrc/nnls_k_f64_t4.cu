// Instantiates the persistent solver for double, 4 thread(s) per column.
#include "nnls_kernel.cuh"

namespace nenmf {
NENMF_NNLS_TPC_IMPL(double, 4)
}  // namespace nenmf
