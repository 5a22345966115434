// Instantiations of the column solve pass (sr_fft.cuh) for M = 8 .. 8192.
#include "sr_kernels.h"
namespace srsb {
template <int LG, bool SYMT> static ColKernel cs(bool contig) {
    return contig ? k_cols_solve<LG, (LG < 4 ? LG : 4), true, SYMT> : k_cols_solve<LG, (LG < 4 ? LG : 4), false, SYMT>;
}
template <bool SYMT> static ColKernel pick(int lg, bool contig) {
    switch (lg) {
        case 3: return cs<3, SYMT>(contig);   case 4: return cs<4, SYMT>(contig);   case 5: return cs<5, SYMT>(contig);
        case 6: return cs<6, SYMT>(contig);   case 7: return cs<7, SYMT>(contig);   case 8: return cs<8, SYMT>(contig);
        case 9: return cs<9, SYMT>(contig);   case 10: return cs<10, SYMT>(contig); case 11: return cs<11, SYMT>(contig);
        case 12: return cs<12, SYMT>(contig); case 13: return cs<13, SYMT>(contig);
    }
    return nullptr;
}
ColKernel pick_col(int lg, bool contig, bool symt) { return symt ? pick<true>(lg, contig) : pick<false>(lg, contig); }
ColPKernel pick_col_p(int lg, bool symt) {   // long columns only
    switch (lg) {
        case 12: return symt ? k_cols_solve_p<12, 4, true> : k_cols_solve_p<12, 4, false>;
        case 13: return symt ? k_cols_solve_p<13, 4, true> : k_cols_solve_p<13, 4, false>;
    }
    return nullptr;
}
}  // namespace srsb
