// Fused operator kernels for Q6 (ND = NQ = 7): the plane kernel.
#define FEOD_ND 7
#include "inst_plane.cuh"
