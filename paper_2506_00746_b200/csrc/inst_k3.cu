// Fused operator kernels for Q3 (ND = NQ = 4).
#define FEOD_ND 4
#include "inst.cuh"
