// 3-D stencils, window radius 2
#define SRSB_R 2
#include "vol_inst.cuh"
