#define TFFFT_REAL float
#include "kernels_inst.cuh"
