// Instantiates the stencil kernels for one window radius SRSB_R (both window shapes).
#include "sr_kernels.h"
namespace srsb {
#define SRSB_CAT2(a, b) a##b
#define SRSB_CAT(a, b) SRSB_CAT2(a, b)
template <int SH>
static void set_r(RhsKernel& rhs, WbKernel (&wb)[2][2]) {
    rhs = k_rhs<SRSB_R, SH>;
    wb[0][0] = k_wb<SRSB_R, SH, 0, false>;
    wb[0][1] = k_wb<SRSB_R, SH, 0, true>;
    wb[1][0] = k_wb<SRSB_R, SH, 1, false>;
    wb[1][1] = k_wb<SRSB_R, SH, 1, true>;
}
bool SRSB_CAT(pick_stencil_r, SRSB_R)(int shape, RhsKernel& rhs, WbKernel (&wb)[2][2], int& smem) {
    if (shape == 0) set_r<0>(rhs, wb);
    else if (shape == 1) set_r<1>(rhs, wb);
    else return false;
    smem = TileGeom<SRSB_R>::BYTES;
    return true;
}
}  // namespace srsb
