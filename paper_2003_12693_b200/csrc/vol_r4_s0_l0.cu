// 3-D stencils: window radius 4, shape 0, l == eps 0
#define SRSB_R 4
#define SRSB_VSHAPE 0
#define SRSB_VLEQ 0
#include "vol_inst.cuh"
