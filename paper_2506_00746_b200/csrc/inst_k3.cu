// Fused operator kernels for Q3 (ND = NQ = 4): the plane kernel.
#define FEOD_ND 4
#include "inst_plane.cuh"
