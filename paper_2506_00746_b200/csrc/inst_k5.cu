// Fused operator kernels for Q5 (ND = NQ = 6).
#define FEOD_ND 6
#include "inst.cuh"
