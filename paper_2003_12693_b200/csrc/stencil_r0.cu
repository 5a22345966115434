// window radius 0
#define SRSB_R 0
#include "stencil_inst.cuh"
