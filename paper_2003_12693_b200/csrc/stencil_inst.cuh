// Instantiates the stencil kernels for one window radius SRSB_R (both window shapes).
#include "sr_kernels.h"
namespace srsb {
#define SRSB_CAT2(a, b) a##b
#define SRSB_CAT(a, b) SRSB_CAT2(a, b)
template <int SH, bool LEQ>
static void set_r(RhsKernel& rhs, WbKernel (&wb)[2][2], WbKernel& wb_mon) {
    rhs = k_rhs<SRSB_R, SH, LEQ>;
    wb_mon = k_wb<SRSB_R, SH, 0, true, LEQ, true>;
    wb[0][0] = k_wb<SRSB_R, SH, 0, false, LEQ>;
    wb[0][1] = k_wb<SRSB_R, SH, 0, true, LEQ>;
    wb[1][0] = k_wb<SRSB_R, SH, 1, false, LEQ>;
    wb[1][1] = k_wb<SRSB_R, SH, 1, true, LEQ>;
}
bool SRSB_CAT(pick_stencil_r, SRSB_R)(int shape, bool leq, RhsKernel& rhs, WbKernel (&wb)[2][2], WbKernel& wb_mon,
                                       int& smem) {
    if (shape == 0 && leq) set_r<0, true>(rhs, wb, wb_mon);
    else if (shape == 0) set_r<0, false>(rhs, wb, wb_mon);
    else if (shape == 1 && leq) set_r<1, true>(rhs, wb, wb_mon);
    else if (shape == 1) set_r<1, false>(rhs, wb, wb_mon);
    else return false;
    smem = TileGeom<SRSB_R>::BYTES;
    return true;
}
bool SRSB_CAT(pick_rhs_tma_r, SRSB_R)(int shape, bool leq, RhsTmaKernel& k, int& smem) {
    if (shape == 0 && leq) k = k_rhs_tma<SRSB_R, 0, true>;
    else if (shape == 0) k = k_rhs_tma<SRSB_R, 0, false>;
    else if (shape == 1 && leq) k = k_rhs_tma<SRSB_R, 1, true>;
    else if (shape == 1) k = k_rhs_tma<SRSB_R, 1, false>;
    else return false;
    smem = TmaGeom<SRSB_R>::BYTES;
    return true;
}
}  // namespace srsb
