// sr_vol3.h -- 3-D kernel pointer types and the per-radius pickers (vol_r<R>.cu), NEXT-3.
#pragma once
#include "sr_vol.cuh"

namespace srsb {

typedef void (*VolRhsKernel)(const float*, const float*, const float*, const float*, float*, VolArgs);
typedef void (*VolWbKernel)(const float*, const float*, float*, float*, const float*, int*, VolArgs);
constexpr int kMaxWindow3 = 4;   // ball radius supported in 3-D
bool pick_vol(int R, int shape, bool leq, VolRhsKernel& rhs, VolWbKernel (&wb)[2][2], int& smem);
#define SRSB_DECLARE_VOL(R, S, L) void set_vol_r##R##_s##S##_l##L(VolRhsKernel& rhs, VolWbKernel (&wb)[2][2], int& smem);
#define SRSB_DECLARE_VOL_R(R) SRSB_DECLARE_VOL(R, 0, 0) SRSB_DECLARE_VOL(R, 0, 1) SRSB_DECLARE_VOL(R, 1, 0) SRSB_DECLARE_VOL(R, 1, 1)
SRSB_DECLARE_VOL_R(0) SRSB_DECLARE_VOL_R(1) SRSB_DECLARE_VOL_R(2) SRSB_DECLARE_VOL_R(3) SRSB_DECLARE_VOL_R(4)
#undef SRSB_DECLARE_VOL_R
#undef SRSB_DECLARE_VOL

}  // namespace srsb
