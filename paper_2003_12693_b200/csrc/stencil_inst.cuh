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
template <int SH, bool LEQ>
static RhsR2cKernel fused_h(int log2_h) {
    switch (log2_h) {
        case 6: return k_rhs_r2c<SRSB_R, SH, LEQ, 6>;
        case 7: return k_rhs_r2c<SRSB_R, SH, LEQ, 7>;
        case 8: return k_rhs_r2c<SRSB_R, SH, LEQ, 8>;
        case 9: return k_rhs_r2c<SRSB_R, SH, LEQ, 9>;
    }
    return nullptr;
}
RhsR2cKernel SRSB_CAT(pick_fused_r, SRSB_R)(int shape, bool leq, int log2_h, int& smem) {
    smem = TmaGeom<SRSB_R>::BYTES;
    if (shape == 0) return leq ? fused_h<0, true>(log2_h) : fused_h<0, false>(log2_h);
    if (shape == 1) return leq ? fused_h<1, true>(log2_h) : fused_h<1, false>(log2_h);
    return nullptr;
}
}  // namespace srsb
