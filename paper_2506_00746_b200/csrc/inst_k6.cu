// Fused operator kernels for Q6 (ND = NQ = 7).
#define FEOD_ND 7
#include "inst.cuh"
