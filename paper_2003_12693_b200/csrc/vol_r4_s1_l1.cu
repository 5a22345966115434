// 3-D stencils: window radius 4, shape 1, l == eps 1
#define SRSB_R 4
#define SRSB_VSHAPE 1
#define SRSB_VLEQ 1
#include "vol_inst.cuh"
