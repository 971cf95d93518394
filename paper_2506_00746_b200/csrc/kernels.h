// Internal launch interface of libfeod (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>
#include "common.cuh"

namespace feod {

struct OpPtrs {
  const double* in0;
  const double* in1;
  double* out0;
  double* out1;
  double* shell0;
  double* shell1;
  double* gout;
};

// Brick shape (elements) and kernel family of one order: ptx = per-point stream
// interleave (OpParams::ptx: the column kernel's tile width, 1 for the plane kernel),
// minb = resident CTAs per SM the kernel is built for.
struct BrickInfo { int BX, BY, BZ, threads, ptx, minb; size_t smem[kModes]; };

// Resident CTAs of a persistent kernel on the current device (SMs x occupancy),
// cached per (kernel, device) (dispatch.cu).
cudaError_t persistent_slots(const void* kernel, int threads, size_t smem, int* slots);

cudaError_t launch_geometry(const double* verts, const OpParams& P, int nq, const Tables& T, double* geom, int* bad,
                            cudaStream_t st);

// Per-order entry points (inst_kN.cu), ND = k+1, NQ = k+1.
template <int ND> bool brick_info(BrickInfo* bi);
template <int ND> cudaError_t prepare_order();
template <int ND> cudaError_t launch_order(int mode, int model, bool affine, int grid, const OpParams& P,
                                           const Tables& T, const OpPtrs& p, cudaStream_t st, int* grid_out);
template <int ND> cudaError_t fixup_order(const OpParams& P, const double* shell0, double* out0,
                                          const double* shell1, double* out1, cudaStream_t st);
template <int ND> int fixup_rows_order(const OpParams& P, int2* rows, unsigned long long* keys);

#define FEOD_DECLARE_ORDER(ND)                                                                    \
  template <> bool brick_info<ND>(BrickInfo * bi);                                                \
  template <> cudaError_t prepare_order<ND>();                                                    \
  template <> cudaError_t launch_order<ND>(int mode, int model, bool affine, int grid, const OpParams& P, \
                                           const Tables& T, const OpPtrs& p, cudaStream_t st, int* grid_out); \
  template <> cudaError_t fixup_order<ND>(const OpParams& P, const double* shell0, double* out0, \
                                          const double* shell1, double* out1, cudaStream_t st); \
  template <> int fixup_rows_order<ND>(const OpParams& P, int2* rows, unsigned long long* keys);
FEOD_DECLARE_ORDER(2)
FEOD_DECLARE_ORDER(3)
FEOD_DECLARE_ORDER(4)
FEOD_DECLARE_ORDER(5)
FEOD_DECLARE_ORDER(6)
FEOD_DECLARE_ORDER(7)

bool brick_info_nd(int nd, BrickInfo* bi);
cudaError_t prepare_nd(int nd);
cudaError_t launch_nd(int nd, int mode, int model, bool affine, int grid, const OpParams& P, const Tables& T,
                      const OpPtrs& p, cudaStream_t st, int* grid_out);
cudaError_t fixup_nd(int nd, const OpParams& P, const double* shell0, double* out0, const double* shell1,
                     double* out1, cudaStream_t st);
int fixup_rows_nd(int nd, const OpParams& P, int2* rows, unsigned long long* keys);

// BLAS-1 (blas1.cu): deterministic fixed-grid two-stage reductions.
constexpr int kRedBlocks = 148 * 8;   // fixed reduction grid: full occupancy on 148 SMs
cudaError_t dot_partial(const double* x, const double* y, int64_t n, double* partials, cudaStream_t st);
cudaError_t reduce_final(const double* partials, double* out, cudaStream_t st);

}  // namespace feod

namespace feod {
cudaError_t cg_init(const double* F, double* r, double* p, double* d, int64_t n, cudaStream_t st,
                    const double* diag = nullptr);
cudaError_t cg_update(const double* rr, const double* pAp_partials, double* pAp, const double* Ap, double* r, int64_t n,
                      double* partials, int* bad, cudaStream_t st, const double* diag = nullptr);
cudaError_t cg_dir(const double* rr_partials, double* rr_new, const double* rr_old, const double* pAp, const double* r,
                   double* p, double* d, int64_t n, cudaStream_t st, const double* diag = nullptr);
// element tangent matrices on the FP64 tensor cores (elemat.cu, K9): nd = 2..4
cudaError_t element_matrices_nd(int nd, int model, bool affine, bool elm, const OpParams& P, const Tables& T,
                                const double* u, int e0, int ne, double* Ke, cudaStream_t st);
// Q6 residual / JVP on the FP64 tensor cores, one warp per element, through an element
// vector (q6tc.cu, K11); out gets the assembled L-vector
// Jacobi diagonal of the stored linearisation at Q6 on affine meshes (q6tc.cu, K12)
cudaError_t q6tc_diag(int model, const OpParams& P, const Tables& T, double* ev, double* diag, cudaStream_t st);
bool q6tc_supports(int mode);
// The CG update fused behind the Q6 operator (Newton-CG, NEXT-3): the operator kernel forms
// the partials of p.Ap element by element (p's Dirichlet entries are 0 in the CG), and the
// assembly, instead of writing Ap, applies r -= alpha Ap row by row (alpha = *rr / p.Ap) and
// forms the partials of r.z -- the Ap vector is never written or re-read, cg_update is not
// launched. Fixed grids and summation orders throughout.
struct CgFuse {
  const double* rr;     // r.z of the current iterate (device scalar)
  double* pAp_part;     // kRedBlocks partials of p.Ap (written by the operator kernel)
  double* pAp;          // p.Ap (device scalar, written by the assembly's CTA 0; cg_dir reads it)
  double* r;            // residual vector, updated in place
  double* rz_part;      // kRedBlocks partials of r.z (z = r / diag, or r)
  int* bad;             // set when p.Ap <= 0
  const double* diag;   // Jacobi diagonal or null
};
cudaError_t q6tc_run(int mode, int model, const OpParams& P, const Tables& T, const double* in0, const double* in1,
                     double* ev, double* out, const double* dotx, double* dpart, cudaStream_t st,
                     const CgFuse* fuse = nullptr);
// element tangents by element-level forward AD through B, D and B^T (elm.cu, K10; Table 1's ELM);
// nd >= 5 keeps the per-seed tangent arrays in scr (elm_scratch_per_cta(nd) doubles per CTA; the
// grid is bounded by scr_doubles)
size_t elm_scratch_per_cta(int nd);
cudaError_t element_matrices_elm_nd(int nd, int model, bool affine, const OpParams& P, const Tables& T,
                                    const double* u, int e0, int ne, double* Ke, double* scr, size_t scr_doubles,
                                    cudaStream_t st);
// element tangents at nd = 5..7 (Q4..Q6): tiled M^T N with on-chip operand generation (elemat_hi.cu, K9b)
cudaError_t element_matrices_hi_nd(int nd, int model, bool affine, const OpParams& P, const Tables& T,
                                   const double* u, int e0, int ne, double* Ke, cudaStream_t st);
// Jacobi diagonal of the stored linearisation (diag.cu, K8)
// ev: scratch for the discontinuous L-vector (nd^3 x E doubles) of the Q3..Q5 path, or null
cudaError_t jacobi_diag_nd(int nd, int model, const OpParams& P, const Tables& T, double* ev, double* diag,
                           cudaStream_t st);
cudaError_t axpy1(double* u, const double* d, int64_t n, cudaStream_t st);
// BiCGStab for the adjoint solve (krylov.cu)
cudaError_t mask_dirichlet(double* x, const OpParams& P, cudaStream_t st);
cudaError_t bicg_init(const double* b, double* x, double* r, double* rhat, double* p, double* v, int64_t n,
                      cudaStream_t st);
cudaError_t bicg_p(const double* sc, int it, const double* r, const double* v, double* p, int64_t n, cudaStream_t st);
cudaError_t bicg_s(double* sc, int it, const double* r, const double* v, double* s, int64_t n, int* bad,
                   cudaStream_t st);
cudaError_t bicg_x(double* sc, const double* p, const double* s, const double* t, const double* rhat, double* x,
                   double* r, int64_t n, double* part_rr, double* part_r2, int* bad, cudaStream_t st);
}  // namespace feod
