// Instantiations of the row R2C pass (sr_fft.cuh) for N/2 = 4 .. 4096.
#include "sr_kernels.h"
namespace srsb {
template <int LG> static RowKernel rf() { return k_rows_r2c<LG, (LG < 4 ? LG : 4)>; }
RowKernel pick_row_fwd(int lg) {
    switch (lg) {
        case 2: return rf<2>();   case 3: return rf<3>();   case 4: return rf<4>();   case 5: return rf<5>();
        case 6: return rf<6>();   case 7: return rf<7>();   case 8: return rf<8>();   case 9: return rf<9>();
        case 10: return rf<10>(); case 11: return rf<11>(); case 12: return rf<12>();
    }
    return nullptr;
}
// Launch-shape instances (log2 H, log2 rows per CTA, log2 G) of the measured configs: C1 128^2, C2 512^2,
// C3 64 x 1024^2, C4 4096^2, C5 8192^2 (whole-image contexts; srsb.cu configure() picks these shapes).
RowKernel pick_row_fwd_shape(int lg, int lg_rpc, int lg_G) {
#define SRSB_SHAPE(LH, LR, LG_) if (lg == LH && lg_rpc == LR && lg_G == LG_) return k_rows_r2c<LH, 4, LR, LG_>;
    SRSB_SHAPE(6, 4, 0) SRSB_SHAPE(8, 3, 0) SRSB_SHAPE(9, 3, 0) SRSB_SHAPE(11, 2, 0) SRSB_SHAPE(11, 2, 1) SRSB_SHAPE(12, 1, 0)
    SRSB_SHAPE(12, 2, 0)   // C5 wide: 4 rows x 256 threads, 32-byte transposed chunks (configure(): SRSB_R2C_WIDE)
    // row-major spectrum (G = H; k_cols_tri_rm): C3 (2 rows per CTA), C4, C5 (1 row), 512-wide rows
    SRSB_SHAPE(9, 1, 9) SRSB_SHAPE(9, 2, 9) SRSB_SHAPE(10, 0, 10) SRSB_SHAPE(10, 1, 10) SRSB_SHAPE(11, 0, 11) SRSB_SHAPE(12, 0, 12)
#undef SRSB_SHAPE
    return pick_row_fwd(lg);
}
}  // namespace srsb
