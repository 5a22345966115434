// 3-D stencils, window radius 0
#define SRSB_R 0
#include "vol_inst.cuh"
