// Fused operator kernels for Q5 (ND = NQ = 6): the plane kernel.
#define FEOD_ND 6
#include "inst_plane.cuh"
