// 3-D stencils: window radius 2, shape 1, l == eps 1
#define SRSB_R 2
#define SRSB_VSHAPE 1
#define SRSB_VLEQ 1
#include "vol_inst.cuh"
