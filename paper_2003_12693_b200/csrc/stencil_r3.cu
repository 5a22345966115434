// window radius 3
#define SRSB_R 3
#include "stencil_inst.cuh"
