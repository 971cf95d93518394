// Instantiation of the plane kernel (Q3..Q6) for one order (ND = k+1 nodes,
// NQ = k+1 points per axis): 7 modes x 3 models x {affine, stored metric}.
#pragma once
#include "kernels.h"
#include "fixup.cuh"
#include "plane_kernel.cuh"

namespace feod {

// Persistent grid: as many CTAs as fit on the device at once (occupancy x SMs),
// never more than there are bricks; each CTA walks bricks blockIdx.x + k gridDim.x.
template <int ND, int NQ, int MODE, int MODEL, bool AFF>
static cudaError_t launch_one(int nbricks, const OpParams& P, const Tables& T, const OpPtrs& p, cudaStream_t st,
                              int* grid_out) {
  using S = PShape<ND, MODE>;
  const size_t smem = S::SMEM_BYTES;
  int slots = 0;
  cudaError_t e = persistent_slots((const void*)plane_kernel<ND, MODE, MODEL, AFF>, S::NT, smem, &slots);
  if (e != cudaSuccess) return e;
  const int grid = nbricks < slots ? nbricks : slots;
  *grid_out = grid;
#if FEOD_PDL_OPERATOR
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)S::NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, plane_kernel<ND, MODE, MODEL, AFF>, P, T, p.in0, p.in1, p.out0, p.out1, p.shell0,
                            p.shell1, p.gout);
#else
  plane_kernel<ND, MODE, MODEL, AFF><<<grid, S::NT, smem, st>>>(P, T, p.in0, p.in1, p.out0, p.out1, p.shell0,
                                                                p.shell1, p.gout);
  return cudaGetLastError();
#endif
}

template <int ND, int NQ, int MODE, int MODEL, bool AFF>
static cudaError_t prep_one() {
  using S = PShape<ND, MODE>;
  return cudaFuncSetAttribute(plane_kernel<ND, MODE, MODEL, AFF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)S::SMEM_BYTES);
}

template <int ND, int NQ, int MODE>
static cudaError_t launch_mode(int model, bool aff, int grid, const OpParams& P, const Tables& T, const OpPtrs& p,
                               cudaStream_t st, int* grid_out) {
  switch (model) {
    case PLAPLACE: return aff ? launch_one<ND, NQ, MODE, PLAPLACE, true>(grid, P, T, p, st, grid_out)
                              : launch_one<ND, NQ, MODE, PLAPLACE, false>(grid, P, T, p, st, grid_out);
    case NLDIFF: return aff ? launch_one<ND, NQ, MODE, NLDIFF, true>(grid, P, T, p, st, grid_out)
                            : launch_one<ND, NQ, MODE, NLDIFF, false>(grid, P, T, p, st, grid_out);
    case HEAT: return aff ? launch_one<ND, NQ, MODE, HEAT, true>(grid, P, T, p, st, grid_out)
                          : launch_one<ND, NQ, MODE, HEAT, false>(grid, P, T, p, st, grid_out);
  }
  return cudaErrorInvalidValue;
}

template <int ND, int NQ, int MODE>
static cudaError_t prep_mode() {
  cudaError_t e;
  if ((e = prep_one<ND, NQ, MODE, PLAPLACE, true>()) != cudaSuccess) return e;
  if ((e = prep_one<ND, NQ, MODE, PLAPLACE, false>()) != cudaSuccess) return e;
  if ((e = prep_one<ND, NQ, MODE, NLDIFF, true>()) != cudaSuccess) return e;
  if ((e = prep_one<ND, NQ, MODE, NLDIFF, false>()) != cudaSuccess) return e;
  if ((e = prep_one<ND, NQ, MODE, HEAT, true>()) != cudaSuccess) return e;
  return prep_one<ND, NQ, MODE, HEAT, false>();
}

template <>
bool brick_info<FEOD_ND>(BrickInfo* bi) {
  using S = PShape<FEOD_ND, MODE_RES>;
  bi->BX = S::BX; bi->BY = S::BY; bi->BZ = S::BZ; bi->threads = S::NT; bi->ptx = 1; bi->minb = S::MINB;
  bi->smem[MODE_RES] = PShape<FEOD_ND, MODE_RES>::SMEM_BYTES;
  bi->smem[MODE_JVP] = PShape<FEOD_ND, MODE_JVP>::SMEM_BYTES;
  bi->smem[MODE_JVPRES] = PShape<FEOD_ND, MODE_JVPRES>::SMEM_BYTES;
  bi->smem[MODE_DESIGN] = PShape<FEOD_ND, MODE_DESIGN>::SMEM_BYTES;
  bi->smem[MODE_VJP] = PShape<FEOD_ND, MODE_VJP>::SMEM_BYTES;
  bi->smem[MODE_LIN] = PShape<FEOD_ND, MODE_LIN>::SMEM_BYTES;
  bi->smem[MODE_PAJVP] = PShape<FEOD_ND, MODE_PAJVP>::SMEM_BYTES;
  return true;
}

template <>
cudaError_t prepare_order<FEOD_ND>() {
  cudaError_t e;
  if ((e = prep_mode<FEOD_ND, FEOD_ND, MODE_RES>()) != cudaSuccess) return e;
  if ((e = prep_mode<FEOD_ND, FEOD_ND, MODE_JVP>()) != cudaSuccess) return e;
  if ((e = prep_mode<FEOD_ND, FEOD_ND, MODE_JVPRES>()) != cudaSuccess) return e;
  if ((e = prep_mode<FEOD_ND, FEOD_ND, MODE_DESIGN>()) != cudaSuccess) return e;
  if ((e = prep_mode<FEOD_ND, FEOD_ND, MODE_VJP>()) != cudaSuccess) return e;
  if ((e = prep_mode<FEOD_ND, FEOD_ND, MODE_LIN>()) != cudaSuccess) return e;
  return prep_mode<FEOD_ND, FEOD_ND, MODE_PAJVP>();
}

template <>
cudaError_t launch_order<FEOD_ND>(int mode, int model, bool aff, int grid, const OpParams& P, const Tables& T,
                                  const OpPtrs& p, cudaStream_t st, int* grid_out) {
  switch (mode) {
    case MODE_RES: return launch_mode<FEOD_ND, FEOD_ND, MODE_RES>(model, aff, grid, P, T, p, st, grid_out);
    case MODE_JVP: return launch_mode<FEOD_ND, FEOD_ND, MODE_JVP>(model, aff, grid, P, T, p, st, grid_out);
    case MODE_JVPRES: return launch_mode<FEOD_ND, FEOD_ND, MODE_JVPRES>(model, aff, grid, P, T, p, st, grid_out);
    case MODE_DESIGN: return launch_mode<FEOD_ND, FEOD_ND, MODE_DESIGN>(model, aff, grid, P, T, p, st, grid_out);
    case MODE_VJP: return launch_mode<FEOD_ND, FEOD_ND, MODE_VJP>(model, aff, grid, P, T, p, st, grid_out);
    case MODE_LIN: return launch_mode<FEOD_ND, FEOD_ND, MODE_LIN>(model, aff, grid, P, T, p, st, grid_out);
    case MODE_PAJVP: return launch_mode<FEOD_ND, FEOD_ND, MODE_PAJVP>(model, aff, grid, P, T, p, st, grid_out);
  }
  return cudaErrorInvalidValue;
}

template <>
cudaError_t fixup_order<FEOD_ND>(const OpParams& P, const double* shell0, double* out0, const double* shell1,
                                 double* out1, cudaStream_t st) {
  return launch_fixup_t<FEOD_ND - 1, PShape<FEOD_ND, MODE_RES>::BX, PShape<FEOD_ND, MODE_RES>::BY>(P, shell0, out0, shell1, out1, st);
}

template <>
int fixup_rows_order<FEOD_ND>(const OpParams& P, int2* rows, unsigned long long* keys) {
  return fixup_rows<FEOD_ND - 1>(P, rows, keys);
}

}  // namespace feod
