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
template <int SH, bool LEQ>
static void set_tma(RhsTmaKernel& k, WbTmaKernel (&wb)[2][2], WbTmaKernel& wb_mon) {
    k = k_rhs_tma<SRSB_R, SH, LEQ>;
    wb_mon = k_wb_tma<SRSB_R, SH, 0, true, LEQ, true>;
    wb[0][0] = k_wb_tma<SRSB_R, SH, 0, false, LEQ>;
    wb[0][1] = k_wb_tma<SRSB_R, SH, 0, true, LEQ>;
    wb[1][0] = k_wb_tma<SRSB_R, SH, 1, false, LEQ>;
    wb[1][1] = k_wb_tma<SRSB_R, SH, 1, true, LEQ>;
}
bool SRSB_CAT(pick_tma_r, SRSB_R)(int shape, bool leq, RhsTmaKernel& k, WbTmaKernel (&wb)[2][2], WbTmaKernel& wb_mon,
                                  int& smem_rhs, int& smem_wb) {
    if (shape == 0 && leq) set_tma<0, true>(k, wb, wb_mon);
    else if (shape == 0) set_tma<0, false>(k, wb, wb_mon);
    else if (shape == 1 && leq) set_tma<1, true>(k, wb, wb_mon);
    else if (shape == 1) set_tma<1, false>(k, wb, wb_mon);
    else return false;
    smem_rhs = TmaGeom<SRSB_R>::BYTES;
    smem_wb = WbGeom<SRSB_R>::BYTES;
    return true;
}
}  // namespace srsb
