// Instantiates the tensor-core persistent solver for float (3xTF32 mma).
#include "nnls_mma.cuh"

namespace nenmf {
#define NENMF_MMA_CASES(T) case 17: return launch_nnls_mma_t<T, 1, 1>(W, V, F0, Fout, snaps, salpha, p, c, grid, cpb, Lptr, max_iter, grad_tol, recs, results, st, tracebuf, wtab, s); case 18: return launch_nnls_mma_t<T, 1, 2>(W, V, F0, Fout, snaps, salpha, p, c, grid, cpb, Lptr, max_iter, grad_tol, recs, results, st, tracebuf, wtab, s); case 35: return launch_nnls_mma_t<T, 2, 3>(W, V, F0, Fout, snaps, salpha, p, c, grid, cpb, Lptr, max_iter, grad_tol, recs, results, st, tracebuf, wtab, s); case 36: return launch_nnls_mma_t<T, 2, 4>(W, V, F0, Fout, snaps, salpha, p, c, grid, cpb, Lptr, max_iter, grad_tol, recs, results, st, tracebuf, wtab, s);
NENMF_NNLS_MMA_IMPL(float)
}  // namespace nenmf
