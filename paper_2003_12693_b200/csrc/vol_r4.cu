// 3-D stencils, window radius 4
#define SRSB_R 4
#include "vol_inst.cuh"
