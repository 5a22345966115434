// Instantiation of the cyclic tridiagonal column solve (sr_tri.cuh).
#include "sr_tri.cuh"
namespace srsb {
ColTriKernel pick_col_tri() { return k_cols_tri<kTriLogL>; }
ColTriRmKernel pick_col_tri_rm() { return k_cols_tri_rm<kTriLogL>; }
}  // namespace srsb
