// Instantiates the 3-D stencil kernels (sr_vol.cuh, NEXT-3) for one (window radius SRSB_R, window
// shape SRSB_VSHAPE, l == eps SRSB_VLEQ) triple: one translation unit each, so the fully unrolled
// ball sums compile in parallel.
#include "sr_vol3.h"
namespace srsb {
#define SRSB_VCAT2(a, b, c, d) a##b##_s##c##_l##d
#define SRSB_VCAT(a, b, c, d) SRSB_VCAT2(a, b, c, d)
void SRSB_VCAT(set_vol_r, SRSB_R, SRSB_VSHAPE, SRSB_VLEQ)(VolRhsKernel& rhs, VolWbKernel (&wb)[2][2], int& smem) {
    constexpr bool LEQ = SRSB_VLEQ != 0;
    rhs = k3_rhs<SRSB_R, SRSB_VSHAPE, LEQ>;
    wb[0][0] = k3_wb<SRSB_R, SRSB_VSHAPE, 0, false, LEQ>;
    wb[0][1] = k3_wb<SRSB_R, SRSB_VSHAPE, 0, true, LEQ>;
    wb[1][0] = k3_wb<SRSB_R, SRSB_VSHAPE, 1, false, LEQ>;
    wb[1][1] = k3_wb<SRSB_R, SRSB_VSHAPE, 1, true, LEQ>;
    smem = VolGeom<SRSB_R>::BYTES;
}
}  // namespace srsb
