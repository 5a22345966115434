// window radius 4
#define SRSB_R 4
#include "stencil_inst.cuh"
