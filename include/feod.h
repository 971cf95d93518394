/*
 * feod.h — C-ABI of libfeod: the matrix-free FEOD hot path of
 * "Scalable Analysis and Design Using Automatic Differentiation"
 * (Andrej, Kolev, Lazarov; arXiv 2506.00746), built B200-native (sm_100a, fp64).
 *
 * Citations: "PAPER.md:nnn" is a line of the paper's LaTeX source
 * (§2 "Automatic differentiation in finite element analysis"); readings A1..A19
 * are listed in DESIGN.md §Readings.
 *
 * The operator (Eq. 1 at PAPER.md:155):
 *     F(u) = P^T G^T B^T D(B G P u)
 *   P    T-vector -> L-vector; on one GPU the identity plus Dirichlet-row
 *        handling (reading A2): F_i = 0 on Dirichlet rows, u carries its own
 *        Dirichlet data.
 *   G    element restriction (gather) L -> E, G^T the atomic-free scatter-add.
 *   B    sum-factorised interpolation of values and reference gradients at the
 *        q^3 Gauss points of each hex Q_k element.
 *   D    pointwise flux, the only differentiated operator.
 * Its Jacobian action (Eq. 2): J(u) v = d/dt F(u + t v)|_{t=0}
 *   = P^T G^T B^T J_D(u_q) B G P v, with J_D applied in forward mode by a
 *   device dual-number type ("native ... dual number type").
 * Design sensitivity with AD at integration points (reading A14):
 *   g_e = - sum_{i free} lambda_i dF_i/drho_e.
 *
 * Conventions (readings A1-A17):
 *   - mesh: structured nx x ny x nz hexahedra on the unit cube, trilinear
 *     geometry from the vertex array (or uniform); Q_k with GLL nodes (A3);
 *     qorder = Gauss points per axis (A5); reference cube [0,1]^3 (A4).
 *   - vectors u, v, lambda, r, Jv: length N = (k nx+1)(k ny+1)(k nz+1), fp64,
 *     x-fastest lexicographic DOF order, Dirichlet entries included (A16).
 *   - g, rho: length E = nx ny nz, x-fastest lexicographic element order.
 *   - residual sign: r_i = sum_e int D(grad u).grad phi_i - f phi_i (A1).
 *
 * Memory and ownership: every double* argument of the compute calls is a CUDA
 * DEVICE pointer to caller-owned memory (e.g. a torch.float64 CUDA tensor),
 * 8-byte aligned, not aliased with any other argument of the same call
 * (FEOD_EINVAL otherwise). The library owns its tables, geometry and scratch;
 * feod_destroy frees them. coeffs->rho is borrowed (device, length E) and must
 * stay valid while calls that read it are in flight.
 *
 * Streams: every compute call is asynchronous on the handle's stream (set at
 * create or with feod_set_stream). One stream per handle at a time: the
 * handle's scratch (scatter fix-up buffer) is per handle.
 *
 * Errors: 0 on success, a negative FEOD_E* code otherwise; feod_last_error()
 * returns a thread-local message. No C++ exception crosses the ABI. Kernel
 * execution faults are asynchronous and surface as FEOD_ECUDA at a later call
 * or synchronisation.
 */
#ifndef FEOD_H
#define FEOD_H

#include <stdint.h>

#if defined(__GNUC__)
#define FEOD_API __attribute__((visibility("default")))
#else
#define FEOD_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define FEOD_OK 0
#define FEOD_EINVAL (-1)        /* bad argument (null, aliasing, out of range) */
#define FEOD_EUNSUPPORTED (-2)  /* valid but not built (order/qorder combination) */
#define FEOD_ENOMEM (-3)        /* device or host allocation failed */
#define FEOD_ECUDA (-4)         /* CUDA runtime error */

/* Dirichlet face bits (feod_mesh.dirichlet_faces) */
#define FEOD_FACE_X0 1u
#define FEOD_FACE_X1 2u
#define FEOD_FACE_Y0 4u
#define FEOD_FACE_Y1 8u
#define FEOD_FACE_Z0 16u
#define FEOD_FACE_Z1 32u

typedef struct feod_mesh {
  int32_t nx, ny, nz;        /* hexahedra per axis, >= 1 */
  const double* vertices;    /* HOST pointer, (nx+1)(ny+1)(nz+1) x 3 doubles, x-fastest,
                                copied at create; NULL = uniform grid of the unit cube
                                (constant-metric fast path, no stored geometry) */
  uint32_t dirichlet_faces;  /* OR of FEOD_FACE_* */
} feod_mesh;

typedef enum feod_model {
  FEOD_PLAPLACE = 0,    /* D = (eps^2 + |grad u|^2)^((p-2)/2) grad u */
  FEOD_NLDIFF = 1,      /* D = (1 + u^2) grad u                         (BASELINE configs[2]) */
  FEOD_HEAT_DESIGN = 2  /* D = rho_e^3 (1 + u^2) grad u                 (BASELINE configs[4]) */
} feod_model;

typedef struct feod_coeffs {
  feod_model model;
  double p;             /* PLAPLACE: p >= 2 */
  double eps;           /* PLAPLACE: eps >= 0 */
  double f;             /* constant source term */
  const double* rho;    /* DEVICE pointer, length E; required for HEAT_DESIGN, else ignored */
} feod_coeffs;

typedef struct feod_op* feod_handle;

/* Create an operator. order k in [1, 6], qorder = k+1 (reading A5; other
 * combinations return FEOD_EUNSUPPORTED). Builds the 1D tables on the host,
 * copies the vertices and computes the per-point metric
 * M_q = w_q detJ_q J_q^{-1} J_q^{-T} (6 doubles per point)
 * on `cuda_stream` (a cudaStream_t, NULL = legacy default stream). Rejects
 * meshes with detJ <= 0 at any point and meshes of 2^31 or more elements
 * (FEOD_EINVAL). Synchronises the stream. */
FEOD_API int feod_create(const feod_mesh* mesh, int order, int qorder, const feod_coeffs* coeffs,
                void* cuda_stream, feod_handle* out);
FEOD_API int feod_destroy(feod_handle h);
FEOD_API int feod_set_stream(feod_handle h, void* cuda_stream);
/* Replace rho (HEAT_DESIGN); device pointer, length E. */
FEOD_API int feod_set_rho(feod_handle h, const double* rho);
FEOD_API int64_t feod_num_dofs(feod_handle h);
FEOD_API int64_t feod_num_elems(feod_handle h);
/* Diagnostic: the brick shape (elements per brick along x, y, z) the operator kernels
 * tile the mesh with (their scatter seams: brick faces go through the fix-up kernel).
 * Q1/Q2 use the column kernel (the depth bz is chosen per mesh), Q3..Q6 the plane
 * kernel. Any of the pointers may be NULL. FEOD_EINVAL on a null handle. */
FEOD_API int feod_brick_shape(feod_handle h, int* bx, int* by, int* bz);

/* r = F(u)                               (Eq. 1)          */
FEOD_API int feod_residual(feod_handle h, const double* u, double* r);
/* Jv = J(u) v, one pass with dual<double> (Eq. 2)        */
FEOD_API int feod_jvp(feod_handle h, const double* u, const double* v, double* Jv);
/* r = F(u) and Jv = J(u) v from the same dual pass (value and tangent)  */
FEOD_API int feod_jvp_res(feod_handle h, const double* u, const double* v, double* r, double* Jv);
/* JTw = J(u)^T w, the transpose of Eq. 2 — the adjoint   *
 * action behind PAPER.md:199's adjoint analysis.   *
 * J has zero Dirichlet rows (A2), so w's Dirichlet entries are ignored   *
 * and every row of JTw is kept (reading A17). One pass: J_D^T at each    *
 * point from two dual evaluations (DESIGN.md §2 A17).                    */
FEOD_API int feod_vjp(feod_handle h, const double* u, const double* w, double* JTw);
/* Element tangent matrices K_e = B^T J_D(u_q) B (Eq. 3;    *
 * the hex analogue of Table 1) for elements             *
 * e0 .. e0+ne-1 (lexicographic). Ke (device) gets ne x nd^3 x nd^3 doubles,  *
 * Ke[e][i][j] = d r_e,i / d u_e,j, local nodes a + nd (b + nd c).            *
 * elm = 0: RES (integration-point AD, the paper's approach): J_D from 4 dual *
 *   evaluations per point, then K_e = M^T N on the FP64 tensor cores (DMMA). *
 * elm = 1: ELM (element-level forward AD, Table 1's other column): column j  *
 *   is the tangent of the element residual B^T D(B u_e) along e_j, the dual  *
 *   pushed through the sum-factorised B, D and B^T -- nd^3 dual evaluations  *
 *   of D per point.                                       *
 * No Dirichlet handling (element level). All orders 1..6: from order 4 on    *
 * RES runs as a tiled product with on-chip operand generation, and ELM keeps *
 * its per-seed tangent arrays in a handle-owned device scratch (allocated on *
 * first use, up to 296 CTAs' worth: Q6 ~1.1 GB; FEOD_ENOMEM if it cannot be  *
 * allocated). Q6 K_e is 941 KB per element: the caller sizes ne to Ke.      */
FEOD_API int feod_element_matrices(feod_handle h, const double* u, int64_t e0, int64_t ne, int elm, double* Ke);
/* Adjoint solve (the adjoint analysis of PAPER.md:199): *
 * lambda (device, length N) <- `iters` BiCGStab iterations from lambda = 0 on  *
 *   P^T J(u)^T lambda = P^T rhs   over the free DOFs (lambda_Dir = 0),         *
 * the operator applied by the fused J^T kernel (feod_vjp with P^T). Fixed      *
 * iteration count, device-resident scalars, deterministic reductions.          *
 * res_norms_host (HOST, length iters+1, or NULL) gets ||P^T(rhs - J^T lambda)||*
 * as BiCGStab's recursive residual before the first and after each iteration.  *
 * A converged solve (r = 0) stays frozen; FEOD_EINVAL on a true breakdown     *
 * ((rhat, v) = 0 while (rhat, r) != 0). Synchronises.                          */
FEOD_API int feod_adjoint_solve(feod_handle h, const double* u, const double* rhs, double* lambda, int iters,
                                double* res_norms_host);
/* Stored linearisation (Fig. 1 caption:  *
 * "store only the innermost, pointwise operator component"):               *
 * feod_linearize computes r = F(u) and, in the same pass, stores per        *
 * quadrature point dFh/dgh (symmetric 3x3, 6 values, reading A17) and,      *
 * for NLDIFF / HEAT_DESIGN, dFh/du (3 values) in a handle-owned buffer      *
 * (allocated at the first call: 8 x {6|9} x E x qorder^3 bytes).            *
 * feod_jvp_lin then applies J(u) v from that buffer alone (one field        *
 * forward, no metric, no u): same conventions as feod_jvp. FEOD_EINVAL if   *
 * no linearisation is stored. A later feod_linearize replaces it.          */
FEOD_API int feod_linearize(feod_handle h, const double* u, double* r);
/* diag (device, length N) <- the diagonal of J at the stored linearisation  *
 * on free rows, 1 on Dirichlet rows (J's rows there are zero). Sum-         *
 * factorised per element with squared 1D tables, assembled by 8 element     *
 * colours (no atomics, deterministic). FEOD_EINVAL without feod_linearize.  */
FEOD_API int feod_jacobi_diag(feod_handle h, double* diag);
FEOD_API int feod_jvp_lin(feod_handle h, const double* v, double* Jv);
/* g_e = -lambda^T dF/drho_e, lambda's Dirichlet entries ignored          *
 * (A14); HEAT_DESIGN only (others: FEOD_EINVAL)           */
FEOD_API int feod_design_grad(feod_handle h, const double* u, const double* lambda, double* g);
/* r = F(u) and g_e = -sum_{i free} lambda_i dF_i/drho_e together (SURVEY §8(b) optional
 * fused entry point; the adjoint-load use of PAPER.md:199): one dual evaluation of D per
 * point seeded along rho gives the residual flux (value part) and dF/drho (tangent part).
 * Same conventions as feod_residual and feod_design_grad (HEAT_DESIGN only; r length N,
 * g length E, no output may alias an input or the other output). Q1/Q2: one fused
 * kernel; Q3..Q6: the two calls. */
FEOD_API int feod_res_design_grad(feod_handle h, const double* u, const double* lambda, double* r, double* g);

/* Same operations on HOST buffers: copies host->device, computes, copies
 * device->host and synchronises the stream before returning (the e2e path).
 * op: 0 residual(in0=u, out=r), 1 jvp(in0=u, in1=v, out=Jv),
 *     2 design_grad(in0=u, in1=lambda, out=g), 3 vjp(in0=u, in1=w, out=JTw),
 *     4 residual + jvp (in0=u, in1=v, out = [r | Jv], 2N doubles): the upload
 *       of v overlaps the residual and the download of r overlaps the JVP
 *       (a second, library-owned copy stream).
 * Host memory should be pinned. */
FEOD_API int feod_apply_host(feod_handle h, int op, const double* in0, const double* in1, double* out);

/* A stream of nbatch independent problems on HOST buffers, op as in         *
 * feod_apply_host: step b reads in0[b] (and in1[b] for op != 0) and writes  *
 * out[b] (N doubles; E for op 2; 2N = [r | Jv] for op 4). Arrays of nbatch  *
 * host pointers; buffers should be pinned; out[b] must not alias any input. *
 * Two library-owned device staging sets (8 max(N, E) doubles, allocated on  *
 * first use): step b+1's uploads overlap step b's operator and downloads    *
 * (the host link is full duplex), so a step costs max(H2D, D2H, operator)   *
 * in steady state. Synchronises before returning; on error the steps        *
 * already queued may have completed. Results are bitwise those of nbatch    *
 * feod_apply_host calls (the same kernels on the same stream).              */
FEOD_API int feod_apply_host_batch(feod_handle h, int op, int64_t nbatch, const double* const* in0,
                                   const double* const* in1, double* const* out);

/* Jacobian-free Newton with unpreconditioned CG (reading A15, BASELINE
 * configs[3]): u (device, length N) is updated in place; for each of
 * newton_steps steps: F = F(u), CG on J(u) d = -F from d = 0 for exactly
 * cg_iters iterations, u += d. norms_host (length newton_steps+1, HOST) gets
 * ||F|| before each step and after the last. Returns FEOD_EINVAL if
 * p^T J p <= 0 occurs (CG breakdown). Synchronises the stream. */
FEOD_API int feod_newton_cg(feod_handle h, double* u, int newton_steps, int cg_iters, double* norms_host);
/* Newton-CG option: capture each Newton step's CG iterations as a
 * CUDA graph on an internal stream and replay it (default on; the captured kernels take
 * the same arguments every step, the per-call scheduling state lives on the device).
 * enable: 0 or 1. A capture that fails falls back to direct launches. */
FEOD_API int feod_set_cg_graphs(feod_handle h, int enable);
/* Newton-CG option: on the Q6 tensor-core path (k = 6,
 * affine mesh) fuse the CG update into the operator call -- p^T J p is formed element by
 * element in the operator kernel and r -= alpha J p (with the r.z partials) in the assembly
 * of its element vector, so J p is never written to or re-read from HBM and the separate
 * update launch disappears (default on; other paths ignore it). Fixed summation orders:
 * results are reproducible run to run, and agree with the unfused loop up to rounding
 * order. enable: 0 or 1; FEOD_EINVAL otherwise. */
FEOD_API int feod_set_cg_fusion(feod_handle h, int enable);
/* Number of CG graph replays so far (diagnostic; -1 on a null handle). */
FEOD_API int64_t feod_cg_graph_launches(feod_handle h);
/* Newton-CG Jacobian: 0 (default) matrix-free feod_jvp at the current u;   *
 * 1 feod_linearize once per Newton step (it also yields F) and            *
 * feod_jvp_lin in every CG iteration; 2 as 1 plus Jacobi preconditioning   *
 * (feod_jacobi_diag once per Newton step, CG becomes PCG).  */
FEOD_API int feod_set_newton_linearization(feod_handle h, int stored);

/* BLAS-1 used by the Newton-CG driver (deterministic two-stage reductions).  *
 * result: DEVICE pointer to one double.                                      */
FEOD_API int feod_dot(feod_handle h, const double* x, const double* y, int64_t n, double* result);

/* Profiling hook (bench.py roofline): the NEXT operator call on this handle
 * records cudaEvent_t ev_begin on the handle's stream right before its fused
 * operator kernel and ev_end right after it (before the scatter fix-up), so
 * that kernel's duration can be timed live. One-shot; NULLs clear it. */
FEOD_API int feod_profile_next(feod_handle h, void* ev_begin, void* ev_end);

FEOD_API const char* feod_last_error(void);
FEOD_API const char* feod_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FEOD_H */
