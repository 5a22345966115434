// 3-D stencils: window radius 0, shape 1, l == eps 1
#define SRSB_R 0
#define SRSB_VSHAPE 1
#define SRSB_VLEQ 1
#include "vol_inst.cuh"
