// Instantiations of the column solve pass (sr_fft.cuh) for M = 8 .. 8192.
#include "sr_kernels.h"
namespace srsb {
template <int LG> static ColKernel cs(bool contig) {
    return contig ? k_cols_solve<LG, (LG < 4 ? LG : 4), true> : k_cols_solve<LG, (LG < 4 ? LG : 4), false>;
}
ColKernel pick_col(int lg, bool contig) {
    switch (lg) {
        case 3: return cs<3>(contig);   case 4: return cs<4>(contig);   case 5: return cs<5>(contig);   case 6: return cs<6>(contig);
        case 7: return cs<7>(contig);   case 8: return cs<8>(contig);   case 9: return cs<9>(contig);   case 10: return cs<10>(contig);
        case 11: return cs<11>(contig); case 12: return cs<12>(contig); case 13: return cs<13>(contig);
    }
    return nullptr;
}
ColPKernel pick_col_p(int lg) {   // long columns only
    switch (lg) {
        case 12: return k_cols_solve_p<12, 4>;
        case 13: return k_cols_solve_p<13, 4>;
    }
    return nullptr;
}
}  // namespace srsb
