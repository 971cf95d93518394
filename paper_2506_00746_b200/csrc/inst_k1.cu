// Fused operator kernels for Q1 (ND = NQ = 2): the column kernel.
#define FEOD_ND 2
#include "inst_col.cuh"
