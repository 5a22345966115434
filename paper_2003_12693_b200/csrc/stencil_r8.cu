// window radius 8
#define SRSB_R 8
#include "stencil_inst.cuh"
