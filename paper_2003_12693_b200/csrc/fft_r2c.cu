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
}  // namespace srsb
