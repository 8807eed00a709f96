// Instantiates the persistent solver for double, 16 thread(s) per column.
#include "nnls_kernel.cuh"

namespace nenmf {
NENMF_NNLS_TPC_IMPL(double, 16)
}  // namespace nenmf
