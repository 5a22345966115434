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
}  // namespace srsb
