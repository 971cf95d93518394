// Fused operator kernels for Q4 (ND = NQ = 5): the plane kernel.
#define FEOD_ND 5
#include "inst_plane.cuh"
