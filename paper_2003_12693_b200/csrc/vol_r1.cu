// 3-D stencils, window radius 1
#define SRSB_R 1
#include "vol_inst.cuh"
