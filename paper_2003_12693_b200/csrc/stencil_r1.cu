// window radius 1
#define SRSB_R 1
#include "stencil_inst.cuh"
