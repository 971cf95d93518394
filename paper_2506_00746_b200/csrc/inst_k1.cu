// Fused operator kernels for Q1 (ND = NQ = 2).
#define FEOD_ND 2
#include "inst.cuh"
