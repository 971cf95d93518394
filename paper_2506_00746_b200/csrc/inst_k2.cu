// Fused operator kernels for Q2 (ND = NQ = 3).
#define FEOD_ND 3
#include "inst.cuh"
