// 3-D stencils, window radius 3
#define SRSB_R 3
#include "vol_inst.cuh"
