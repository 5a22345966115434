// Instantiates the 3-D stencil kernels for one window radius SRSB_R (sr_vol.cuh, NEXT-3).
#include "sr_vol3.h"
namespace srsb {
#define SRSB_VCAT2(a, b) a##b
#define SRSB_VCAT(a, b) SRSB_VCAT2(a, b)
template <int SH, bool LEQ>
static void set_v(VolRhsKernel& rhs, VolWbKernel (&wb)[2][2]) {
    rhs = k3_rhs<SRSB_R, SH, LEQ>;
    wb[0][0] = k3_wb<SRSB_R, SH, 0, false, LEQ>;
    wb[0][1] = k3_wb<SRSB_R, SH, 0, true, LEQ>;
    wb[1][0] = k3_wb<SRSB_R, SH, 1, false, LEQ>;
    wb[1][1] = k3_wb<SRSB_R, SH, 1, true, LEQ>;
}
bool SRSB_VCAT(pick_vol_r, SRSB_R)(int shape, bool leq, VolRhsKernel& rhs, VolWbKernel (&wb)[2][2], int& smem) {
    if (shape == 0 && leq) set_v<0, true>(rhs, wb);
    else if (shape == 0) set_v<0, false>(rhs, wb);
    else if (shape == 1 && leq) set_v<1, true>(rhs, wb);
    else if (shape == 1) set_v<1, false>(rhs, wb);
    else return false;
    smem = VolGeom<SRSB_R>::BYTES;
    return true;
}
}  // namespace srsb
