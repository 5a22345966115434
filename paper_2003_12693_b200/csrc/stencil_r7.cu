// window radius 7
#define SRSB_R 7
#include "stencil_inst.cuh"
