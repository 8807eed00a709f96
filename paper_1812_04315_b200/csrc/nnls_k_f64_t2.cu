// Instantiates the persistent solver for double, 2 thread(s) per column.
#include "nnls_kernel.cuh"

namespace nenmf {
NENMF_NNLS_TPC_IMPL(double, 2)
}  // namespace nenmf
