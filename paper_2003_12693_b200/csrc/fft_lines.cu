// Instantiations of the batched complex line FFT (sr_fft.cuh, k_lines_fft) for M = 8 .. 8192.
#include "sr_kernels.h"
namespace srsb {
template <int LG> static LinesFftKernel lf(bool inv) {
    return inv ? k_lines_fft<LG, (LG < 4 ? LG : 4), true> : k_lines_fft<LG, (LG < 4 ? LG : 4), false>;
}
LinesFftKernel pick_lines_fft(int lg, bool inv) {
    switch (lg) {
        case 3: return lf<3>(inv);   case 4: return lf<4>(inv);   case 5: return lf<5>(inv);   case 6: return lf<6>(inv);
        case 7: return lf<7>(inv);   case 8: return lf<8>(inv);   case 9: return lf<9>(inv);   case 10: return lf<10>(inv);
        case 11: return lf<11>(inv); case 12: return lf<12>(inv); case 13: return lf<13>(inv);
    }
    return nullptr;
}
}  // namespace srsb
