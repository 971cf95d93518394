// Fused operator kernels for Q4 (ND = NQ = 5).
#define FEOD_ND 5
#include "inst.cuh"
