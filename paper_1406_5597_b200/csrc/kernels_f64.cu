#define TFFFT_REAL double
#include "kernels_inst.cuh"
