// window radius 6
#define SRSB_R 6
#include "stencil_inst.cuh"
