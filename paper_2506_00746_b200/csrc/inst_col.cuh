// Instantiation of the column kernel (Q1, Q2; col_kernel.cuh) for one order
// (ND = k+1 nodes, NQ = k+1 points per axis): 7 modes x 3 models x {affine, stored metric}.
#pragma once
#include "kernels.h"
#include "fixup.cuh"
#include "col_kernel.cuh"

namespace feod {

template <int ND, int MODE, int MODEL, bool AFF>
static cudaError_t launch_col(int nbricks, const OpParams& P, const Tables& T, const OpPtrs& p, cudaStream_t st,
                              int* grid_out) {
  using S = CShape<ND, MODE>;
  const size_t smem = S::SMEM_BYTES;
  int slots = 0;
  cudaError_t e = persistent_slots((const void*)col_kernel<ND, MODE, MODEL, AFF>, S::NT, smem, &slots);
  if (e != cudaSuccess) return e;
  const int grid = nbricks < slots ? nbricks : slots;
  *grid_out = grid;
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
  return cudaLaunchKernelEx(&cfg, col_kernel<ND, MODE, MODEL, AFF>, P, T, p.in0, p.in1, p.out0, p.out1, p.shell0,
                            p.shell1, p.gout);
}

template <int ND, int MODE, int MODEL, bool AFF>
static cudaError_t prep_col() {
  return cudaFuncSetAttribute(col_kernel<ND, MODE, MODEL, AFF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)CShape<ND, MODE>::SMEM_BYTES);
}

template <int ND, int MODE>
static cudaError_t launch_col_mode(int model, bool aff, int nbricks, const OpParams& P, const Tables& T,
                                   const OpPtrs& p, cudaStream_t st, int* grid_out) {
  switch (model) {
    case PLAPLACE: return aff ? launch_col<ND, MODE, PLAPLACE, true>(nbricks, P, T, p, st, grid_out)
                              : launch_col<ND, MODE, PLAPLACE, false>(nbricks, P, T, p, st, grid_out);
    case NLDIFF: return aff ? launch_col<ND, MODE, NLDIFF, true>(nbricks, P, T, p, st, grid_out)
                            : launch_col<ND, MODE, NLDIFF, false>(nbricks, P, T, p, st, grid_out);
    case HEAT: return aff ? launch_col<ND, MODE, HEAT, true>(nbricks, P, T, p, st, grid_out)
                          : launch_col<ND, MODE, HEAT, false>(nbricks, P, T, p, st, grid_out);
  }
  return cudaErrorInvalidValue;
}

template <int ND, int MODE>
static cudaError_t prep_col_mode() {
  cudaError_t e;
  if ((e = prep_col<ND, MODE, PLAPLACE, true>()) != cudaSuccess) return e;
  if ((e = prep_col<ND, MODE, PLAPLACE, false>()) != cudaSuccess) return e;
  if ((e = prep_col<ND, MODE, NLDIFF, true>()) != cudaSuccess) return e;
  if ((e = prep_col<ND, MODE, NLDIFF, false>()) != cudaSuccess) return e;
  if ((e = prep_col<ND, MODE, HEAT, true>()) != cudaSuccess) return e;
  return prep_col<ND, MODE, HEAT, false>();
}

template <>
bool brick_info<FEOD_ND>(BrickInfo* bi) {
  using S = CShape<FEOD_ND, MODE_RES>;
  bi->BX = S::TX; bi->BY = S::TY; bi->BZ = 16; bi->threads = S::NT; bi->ptx = S::TX; bi->minb = CShape<FEOD_ND, MODE_JVP>::MINB;   // brick-depth choice: the JVP's residency
  bi->smem[MODE_RES] = CShape<FEOD_ND, MODE_RES>::SMEM_BYTES;
  bi->smem[MODE_JVP] = CShape<FEOD_ND, MODE_JVP>::SMEM_BYTES;
  bi->smem[MODE_JVPRES] = CShape<FEOD_ND, MODE_JVPRES>::SMEM_BYTES;
  bi->smem[MODE_DESIGN] = CShape<FEOD_ND, MODE_DESIGN>::SMEM_BYTES;
  bi->smem[MODE_VJP] = CShape<FEOD_ND, MODE_VJP>::SMEM_BYTES;
  bi->smem[MODE_LIN] = CShape<FEOD_ND, MODE_LIN>::SMEM_BYTES;
  bi->smem[MODE_PAJVP] = CShape<FEOD_ND, MODE_PAJVP>::SMEM_BYTES;
  bi->smem[MODE_RESDES] = CShape<FEOD_ND, MODE_RESDES>::SMEM_BYTES;
  return true;
}

template <>
cudaError_t prepare_order<FEOD_ND>() {
  cudaError_t e;
  if ((e = prep_col_mode<FEOD_ND, MODE_RES>()) != cudaSuccess) return e;
  if ((e = prep_col_mode<FEOD_ND, MODE_JVP>()) != cudaSuccess) return e;
  if ((e = prep_col_mode<FEOD_ND, MODE_JVPRES>()) != cudaSuccess) return e;
  if ((e = prep_col_mode<FEOD_ND, MODE_DESIGN>()) != cudaSuccess) return e;
  if ((e = prep_col_mode<FEOD_ND, MODE_VJP>()) != cudaSuccess) return e;
  if ((e = prep_col_mode<FEOD_ND, MODE_LIN>()) != cudaSuccess) return e;
  if ((e = prep_col<FEOD_ND, MODE_RESDES, HEAT, true>()) != cudaSuccess) return e;
  if ((e = prep_col<FEOD_ND, MODE_RESDES, HEAT, false>()) != cudaSuccess) return e;
  return prep_col_mode<FEOD_ND, MODE_PAJVP>();
}

template <>
cudaError_t launch_order<FEOD_ND>(int mode, int model, bool aff, int nbricks, const OpParams& P, const Tables& T,
                                  const OpPtrs& p, cudaStream_t st, int* grid_out) {
  switch (mode) {
    case MODE_RES: return launch_col_mode<FEOD_ND, MODE_RES>(model, aff, nbricks, P, T, p, st, grid_out);
    case MODE_JVP: return launch_col_mode<FEOD_ND, MODE_JVP>(model, aff, nbricks, P, T, p, st, grid_out);
    case MODE_JVPRES: return launch_col_mode<FEOD_ND, MODE_JVPRES>(model, aff, nbricks, P, T, p, st, grid_out);
    case MODE_DESIGN: return launch_col_mode<FEOD_ND, MODE_DESIGN>(model, aff, nbricks, P, T, p, st, grid_out);
    case MODE_VJP: return launch_col_mode<FEOD_ND, MODE_VJP>(model, aff, nbricks, P, T, p, st, grid_out);
    case MODE_LIN: return launch_col_mode<FEOD_ND, MODE_LIN>(model, aff, nbricks, P, T, p, st, grid_out);
    case MODE_PAJVP: return launch_col_mode<FEOD_ND, MODE_PAJVP>(model, aff, nbricks, P, T, p, st, grid_out);
    case MODE_RESDES:   // HEAT only (the only model with a design variable)
      if (model != HEAT) return cudaErrorInvalidValue;
      return aff ? launch_col<FEOD_ND, MODE_RESDES, HEAT, true>(nbricks, P, T, p, st, grid_out)
                 : launch_col<FEOD_ND, MODE_RESDES, HEAT, false>(nbricks, P, T, p, st, grid_out);
  }
  return cudaErrorInvalidValue;
}

template <>
cudaError_t fixup_order<FEOD_ND>(const OpParams& P, const double* shell0, double* out0, const double* shell1,
                                 double* out1, cudaStream_t st) {
  return launch_fixup_t<FEOD_ND - 1, CShape<FEOD_ND, MODE_RES>::TX, CShape<FEOD_ND, MODE_RES>::TY>(P, shell0, out0, shell1, out1, st);
}

template <>
int fixup_rows_order<FEOD_ND>(const OpParams& P, int2* rows, unsigned long long* keys) {
  return fixup_rows<FEOD_ND - 1>(P, rows, keys);
}

}  // namespace feod
