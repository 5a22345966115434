// window radius 2
#define SRSB_R 2
#include "stencil_inst.cuh"
