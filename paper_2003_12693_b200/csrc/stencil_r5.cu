// window radius 5
#define SRSB_R 5
#include "stencil_inst.cuh"
