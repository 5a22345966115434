// Instantiations of the one-kernel cluster solve for small images (sr_solve_cl.cuh).
#include "sr_solve_cl.cuh"
namespace srsb {
SolveClKernel pick_solve_cluster(int lg, int lg_rpc) {
#define SRSB_SHAPE(LH, LR) if (lg == LH && lg_rpc == LR) return k_solve_cluster<LH, LR>;
    SRSB_SHAPE(6, 4) SRSB_SHAPE(6, 5) SRSB_SHAPE(7, 4) SRSB_SHAPE(7, 5) SRSB_SHAPE(8, 4) SRSB_SHAPE(8, 5)
#undef SRSB_SHAPE
    return nullptr;
}
}  // namespace srsb
