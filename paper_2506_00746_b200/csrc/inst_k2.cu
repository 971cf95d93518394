// Fused operator kernels for Q2 (ND = NQ = 3): the column kernel.
#define FEOD_ND 3
#include "inst_col.cuh"
