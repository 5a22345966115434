// Instantiations of the row C2R pass (sr_fft.cuh) for N/2 = 4 .. 4096.
#include "sr_kernels.h"
namespace srsb {
template <int LG> static RowInvKernel ri() { return k_rows_c2r<LG, (LG < 4 ? LG : 4)>; }
RowInvKernel pick_row_inv(int lg) {
    switch (lg) {
        case 2: return ri<2>();   case 3: return ri<3>();   case 4: return ri<4>();   case 5: return ri<5>();
        case 6: return ri<6>();   case 7: return ri<7>();   case 8: return ri<8>();   case 9: return ri<9>();
        case 10: return ri<10>(); case 11: return ri<11>(); case 12: return ri<12>();
    }
    return nullptr;
}
// Launch-shape instances (log2 H, log2 rows per CTA, log2 G) of the measured configs: C1 128^2, C2 512^2,
// C3 64 x 1024^2, C4 4096^2, C5 8192^2 (whole-image contexts; srsb.cu configure() picks these shapes).
RowInvKernel pick_row_inv_shape(int lg, int lg_rpc, int lg_G) {
#define SRSB_SHAPE(LH, LR, LG_) if (lg == LH && lg_rpc == LR && lg_G == LG_) return k_rows_c2r<LH, 4, LR, LG_>;
    SRSB_SHAPE(6, 4, 0) SRSB_SHAPE(8, 3, 0) SRSB_SHAPE(9, 1, 0) SRSB_SHAPE(9, 2, 0) SRSB_SHAPE(9, 3, 0) SRSB_SHAPE(9, 4, 0) SRSB_SHAPE(11, 2, 0) SRSB_SHAPE(11, 2, 1) SRSB_SHAPE(12, 1, 0)
    // row-major spectrum (G = H; k_cols_tri_rm): one row per CTA
    SRSB_SHAPE(9, 0, 9) SRSB_SHAPE(9, 1, 9) SRSB_SHAPE(10, 0, 10) SRSB_SHAPE(11, 0, 11) SRSB_SHAPE(12, 0, 12)
#undef SRSB_SHAPE
    return pick_row_inv(lg);
}
}  // namespace srsb
