// C-ABI of libfeod (include/feod.h): validation, handle state, dispatch.
// Every compute step runs in this library's kernels; there is no CPU path.
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/feod.h"
#include "common.cuh"
#include "kernels.h"
#include "tables.h"

using namespace feod;

struct feod_op {
  int nx, ny, nz, k, q, nd;
  feod_coeffs coeffs;
  cudaStream_t st;
  Tables T;
  OpParams P;
  BrickInfo bi;
  int nbricks;
  int64_t N, E;
  int64_t Epad;                // elements incl. the per-point stream interleave padding
  double* geom = nullptr;
  double* shell = nullptr;     // 2 x nbricks x shell
  double* stage = nullptr;     // host-API staging: 4 x max(N, E)
  double* stage2 = nullptr;    // feod_apply_host_batch: the second staging set (double buffering)
  cudaEvent_t bev[6] = {};     // feod_apply_host_batch per set: inputs up, r ready, outputs ready (x2)
  cudaEvent_t bdown[2] = {};   // feod_apply_host_batch per set: outputs downloaded (set free)
  cudaStream_t cst = nullptr;  // host-API upload stream (op 4 overlaps copies with the operator)
  cudaStream_t dst = nullptr;  // host-API download stream (runs against the uploads: full duplex)
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  double* red = nullptr;       // kRedBlocks partials, 24 scalars, kRedBlocks partials
  int* flag = nullptr;
  DevState* ds = nullptr;                // device scheduler state: tickets, epoch (common.cuh)
  unsigned long long* bdone = nullptr;   // per-brick completion epochs (fix-up dependencies)
  bool poisoned = false;                 // a launch failed after the operator kernel ran: the
                                         // brick epochs no longer pair with the shell slab
  cudaEvent_t sw = nullptr;              // stream switch (feod_set_stream orders old -> new)
  int2* fixrows = nullptr;               // fix-up rows in launch order
  double* work = nullptr;      // Newton-CG: F, r, p, Ap, d (5 N)
  double* lin = nullptr;       // stored linearisation (feod_linearize), lin_values x E x q^3
  double* kwork = nullptr;     // adjoint BiCGStab: b, r, rhat, p, v, s, t (7 padded N)
  bool lin_valid = false;
  int newton_lin = 0;          // Newton-CG: 0 matrix-free JVP, 1 stored linearisation, 2 + Jacobi
  double* jdiag = nullptr;     // Jacobi diagonal (Newton mode 2), N
  double* evec = nullptr;      // discontinuous L-vector, nd^3 x E (q6tc.cu operator and diagonal, diag.cu Q3..Q5)
  double* em_scr = nullptr;    // ELM element tangents at Q4..Q6: per-CTA tangent arrays (elm.cu)
  size_t em_scr_n = 0;         // its length in doubles
  bool q6tc = true;            // FEOD_Q6_TC=0 disables the Q6 tensor-core path (experiments)
  bool q6tc_res = true;        // FEOD_Q6_TC_RES=0: the residual on plane_kernel (experiments)
  bool q6tc_lin = false;       // FEOD_Q6_TC_LIN=1: feod_linearize on it too (experiments)
  // Newton-CG: when set, the next operator call also forms the partials of dot_x . out
  // into dot_part (q6tc assembly) and sets dot_fused; cleared by the call
  const double* dot_x = nullptr;
  double* dot_part = nullptr;
  bool dot_fused = false;
  // Newton-CG: when set, a Q6 tensor-core operator call also does the CG update behind its
  // assembly (kernels.h CgFuse) and sets cg_fused; cleared by the call
  const CgFuse* cg_fuse = nullptr;
  bool cg_fused = false;
  bool cg_fusion = true;   // feod_set_cg_fusion
  cudaEvent_t prof_begin = nullptr, prof_end = nullptr;   // one-shot profiling hook
  // Newton-CG: the CG iterations captured as a CUDA graph (on gst), replayed per step
  bool cg_graphs = true, cg_graph_failed = false;
  cudaGraphExec_t cg_exec = nullptr;
  uint64_t cg_key = 0;
  cudaStream_t gst = nullptr;
  cudaEvent_t ev_g[2] = {nullptr, nullptr};
  int64_t cg_graph_launches = 0;
};

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

static int cuda_fail(cudaError_t e, const char* where) {
  return fail(FEOD_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(call, where)                                   \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_fail(e_, where);   \
  } while (0)

extern "C" const char* feod_last_error(void) { return g_err.c_str(); }
extern "C" const char* feod_version(void) { return "feod-b200 0.1 (sm_100a, fp64)"; }

static void free_all(feod_op* h) {
  if (!h) return;
  cudaFree(h->geom);
  cudaFree(h->shell);
  cudaFree(h->stage);
  cudaFree(h->stage2);
  for (cudaEvent_t& e : h->ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t& e : h->bev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t& e : h->bdown)
    if (e) cudaEventDestroy(e);
  if (h->cst) cudaStreamDestroy(h->cst);
  if (h->dst) cudaStreamDestroy(h->dst);
  cudaFree(h->red);
  cudaFree(h->flag);
  cudaFree(h->ds);
  if (h->cg_exec) cudaGraphExecDestroy(h->cg_exec);
  if (h->gst) cudaStreamDestroy(h->gst);
  for (cudaEvent_t& e : h->ev_g)
    if (e) cudaEventDestroy(e);
  if (h->sw) cudaEventDestroy(h->sw);
  cudaFree(h->bdone);
  cudaFree(h->fixrows);
  cudaFree(h->work);
  cudaFree(h->lin);
  cudaFree(h->kwork);
  cudaFree(h->jdiag);
  cudaFree(h->evec);
  cudaFree(h->em_scr);
}

extern "C" int feod_create(const feod_mesh* mesh, int order, int qorder, const feod_coeffs* coeffs,
                           void* cuda_stream, feod_handle* out) {
  if (!mesh || !coeffs || !out) return fail(FEOD_EINVAL, "feod_create: null argument");
  *out = nullptr;
  if (mesh->nx < 1 || mesh->ny < 1 || mesh->nz < 1) return fail(FEOD_EINVAL, "feod_create: nx, ny, nz must be >= 1");
  if (order < 1 || order > 8) return fail(FEOD_EINVAL, "feod_create: order must be in [1, 8]");
  if (qorder < 1) return fail(FEOD_EINVAL, "feod_create: qorder must be >= 1");
  if (order > 6 || qorder != order + 1)
    return fail(FEOD_EUNSUPPORTED, "feod_create: built for order 1..6 with qorder = order + 1");
  if (mesh->dirichlet_faces > 63u) return fail(FEOD_EINVAL, "feod_create: dirichlet_faces has unknown bits");
  if (coeffs->model < FEOD_PLAPLACE || coeffs->model > FEOD_HEAT_DESIGN)
    return fail(FEOD_EINVAL, "feod_create: unknown model");
  if (coeffs->model == FEOD_PLAPLACE && !(coeffs->p >= 2.0)) return fail(FEOD_EINVAL, "feod_create: p must be >= 2");
  if (coeffs->model == FEOD_PLAPLACE && !(coeffs->eps >= 0.0))
    return fail(FEOD_EINVAL, "feod_create: eps must be >= 0");
  if (!std::isfinite(coeffs->f)) return fail(FEOD_EINVAL, "feod_create: f must be finite");
  if (coeffs->model == FEOD_HEAT_DESIGN && !coeffs->rho)
    return fail(FEOD_EINVAL, "feod_create: HEAT_DESIGN needs rho (device, length E)");
  const int64_t Mx = (int64_t)order * mesh->nx + 1, My = (int64_t)order * mesh->ny + 1,
                Mz = (int64_t)order * mesh->nz + 1;
  if (Mx > (1 << 30) || My > (1 << 30) || Mz > (1 << 30)) return fail(FEOD_EINVAL, "feod_create: mesh too large");
  if ((int64_t)mesh->nx * mesh->ny * mesh->nz >= (int64_t(1) << 31))
    return fail(FEOD_EINVAL, "feod_create: more than 2^31 - 1 elements");

  feod_op* h = new (std::nothrow) feod_op();
  if (!h) return fail(FEOD_ENOMEM, "feod_create: host allocation");
  h->nx = mesh->nx; h->ny = mesh->ny; h->nz = mesh->nz;
  h->k = order; h->q = qorder; h->nd = order + 1;
  h->coeffs = *coeffs;
  h->st = (cudaStream_t)cuda_stream;
  h->N = Mx * My * Mz;
  h->E = (int64_t)mesh->nx * mesh->ny * mesh->nz;
  if (!brick_info_nd(h->nd, &h->bi)) { delete h; return fail(FEOD_EUNSUPPORTED, "feod_create: order not built"); }

  // 1D tables (host)
  std::memset(&h->T, 0, sizeof(Tables));
  double nodes[kMaxNQ], pts[kMaxNQ], wts[kMaxNQ];
  gll01(order, nodes);
  gauss01(qorder, pts, wts);
  lagrange01(h->nd, nodes, qorder, pts, &h->T.B[0][0], &h->T.G[0][0], kMaxNQ);
  {
    double id[kMaxNQ * kMaxNQ];   // Lagrange basis of the Gauss points at the Gauss points (identity)
    lagrange01(qorder, pts, qorder, pts, id, &h->T.D[0][0], kMaxNQ);
  }
  for (int i = 0; i < qorder; ++i) { h->T.w[i] = wts[i]; h->T.wi2[i] = 1.0 / (wts[i] * wts[i]); h->T.x[i] = pts[i]; }
  if (qorder % 2 == 1 && std::fabs(h->T.D[qorder / 2][qorder / 2]) < 1e-12)
    h->T.D[qorder / 2][qorder / 2] = 0.0;   // symmetric points: L_mid'(x_mid) = 0 (col_kernel skips it)
  for (int i = 0; i < qorder; ++i)
    for (int m = 0; m < qorder; ++m) h->T.Dh[i][m] = h->T.D[i][m] * wts[i] / wts[m];
  for (int i = 0; i < qorder; ++i)
    for (int a = 0; a < h->nd; ++a) h->T.Bw[i][a] = wts[i] * h->T.B[i][a];
  for (int i = 0; i < qorder; ++i)
    for (int a = 0; a < h->nd; ++a) {
      h->T.B2[i][a] = h->T.B[i][a] * h->T.B[i][a];
      h->T.G2[i][a] = h->T.G[i][a] * h->T.G[i][a];
      h->T.GB[i][a] = h->T.G[i][a] * h->T.B[i][a];
      h->T.Gw[i][a] = wts[i] * h->T.G[i][a];
    }

  OpParams& P = h->P;
  std::memset(&P, 0, sizeof(P));
  P.nx = mesh->nx; P.ny = mesh->ny; P.nz = mesh->nz;
  P.Mx = (int)Mx; P.My = (int)My; P.Mz = (int)Mz;
  P.tbx = h->bi.BX;
  P.tby = h->bi.BY;
  P.tbz = h->bi.BZ;
  P.nbx = (mesh->nx + P.tbx - 1) / P.tbx;
  P.nby = (mesh->ny + P.tby - 1) / P.tby;
  if (h->bi.ptx > 1) {
    // column kernel (Q1, Q2): the brick depth is a run-time choice; take the one whose
    // bricks fill whole waves of resident CTAs best (dynamic scheduling evens out the rest)
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long slots = (long)sms * h->bi.minb;
    double best = 1e300;
    for (int bz : {1, 2, 4, 6, 8, 12, 16, 24, 32, 48, 64}) {
      const long nb = (long)P.nbx * P.nby * ((mesh->nz + bz - 1) / bz);
      const long waves = (nb + slots - 1) / slots;
      const double cost = (double)waves * (std::min(bz, mesh->nz) + 1.0);
      if (cost < best - 1e-9) { best = cost; P.tbz = bz; }
    }
    if (const char* env = std::getenv("FEOD_COL_BZ")) P.tbz = std::max(1, std::atoi(env));   // experiments
  }
  P.nbz = (mesh->nz + P.tbz - 1) / P.tbz;
  if (const char* env = std::getenv("FEOD_Q6_TC")) h->q6tc = std::atoi(env) != 0;   // experiments
  if (const char* env = std::getenv("FEOD_Q6_TC_RES")) h->q6tc_res = std::atoi(env) != 0;
  if (const char* env = std::getenv("FEOD_Q6_TC_LIN")) h->q6tc_lin = std::atoi(env) != 0;
  P.ptx = h->bi.ptx;
  P.pnbx = (mesh->nx + P.ptx - 1) / P.ptx;
  P.shell_stride = shell_size(order * P.tbx + 1, order * P.tby + 1, order * P.tbz + 1);
  P.faces = mesh->dirichlet_faces;
  P.half_pm2 = 0.5 * (coeffs->p - 2.0);
  P.pcase = P.half_pm2 == 0.0 ? 0 : P.half_pm2 == 1.0 ? 1 : P.half_pm2 == 0.5 ? 2 : 3;
  P.eps2 = coeffs->eps * coeffs->eps;
  P.f = coeffs->f;
  const double hx = 1.0 / mesh->nx, hy = 1.0 / mesh->ny, hz = 1.0 / mesh->nz;
  P.cx = hy * hz / hx; P.cy = hx * hz / hy; P.cz = hx * hy / hz; P.vol = hx * hy * hz;
  P.cxv = P.cx / P.vol; P.cyv = P.cy / P.vol; P.czv = P.cz / P.vol;
  P.rho = coeffs->rho;
  h->nbricks = P.nbx * P.nby * P.nbz;
  // per-point streams (metric, stored linearisation) hold pnbx * ptx elements per row
  h->Epad = (int64_t)P.pnbx * P.ptx * mesh->ny * mesh->nz;

  auto cleanup_fail = [&](int code) { free_all(h); delete h; return code; };
  cudaError_t e;
  if ((e = prepare_nd(h->nd)) != cudaSuccess) return cleanup_fail(cuda_fail(e, "feod_create: kernel attributes"));
  if ((e = cudaMalloc(&h->shell, sizeof(double) * 2 * (size_t)h->nbricks * P.shell_stride)) != cudaSuccess)
    return cleanup_fail(fail(FEOD_ENOMEM, "feod_create: shell buffer"));
  if ((e = cudaMalloc(&h->red, sizeof(double) * (2 * kRedBlocks + 32))) != cudaSuccess)
    return cleanup_fail(fail(FEOD_ENOMEM, "feod_create: reduction buffer"));
  if ((e = cudaMalloc(&h->flag, sizeof(int) * 2)) != cudaSuccess)
    return cleanup_fail(fail(FEOD_ENOMEM, "feod_create: flag"));
  if ((e = cudaMalloc(&h->ds, sizeof(DevState))) != cudaSuccess)
    return cleanup_fail(fail(FEOD_ENOMEM, "feod_create: scheduler state"));
  if ((e = cudaMemsetAsync(h->ds, 0, sizeof(DevState), h->st)) != cudaSuccess)
    return cleanup_fail(cuda_fail(e, "feod_create: memset"));
  P.ds = h->ds;
  if ((e = cudaMalloc(&h->bdone, sizeof(unsigned long long) * (size_t)h->nbricks)) != cudaSuccess)
    return cleanup_fail(fail(FEOD_ENOMEM, "feod_create: brick epochs"));
  if ((e = cudaMemsetAsync(h->bdone, 0, sizeof(unsigned long long) * (size_t)h->nbricks, h->st)) != cudaSuccess)
    return cleanup_fail(cuda_fail(e, "feod_create: memset"));
  P.bdone = h->bdone;
  {
    // fix-up rows, stably sorted by the last brick ticket they read
    const int nrows = fixup_rows_nd(h->nd, P, nullptr, nullptr);
    if (nrows < 0) return cleanup_fail(fail(FEOD_EUNSUPPORTED, "feod_create: fix-up rows"));
    std::vector<int2> rows(nrows), sorted(nrows);
    std::vector<unsigned long long> keys(nrows);
    std::vector<int> idx(nrows);
    fixup_rows_nd(h->nd, P, rows.data(), keys.data());
    for (int i = 0; i < nrows; ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return keys[a] < keys[b]; });
    for (int i = 0; i < nrows; ++i) sorted[i] = rows[idx[i]];
    P.nfixrows = nrows;
    if (nrows > 0) {
      if ((e = cudaMalloc(&h->fixrows, sizeof(int2) * (size_t)nrows)) != cudaSuccess)
        return cleanup_fail(fail(FEOD_ENOMEM, "feod_create: fix-up rows"));
      if ((e = cudaMemcpy(h->fixrows, sorted.data(), sizeof(int2) * (size_t)nrows, cudaMemcpyHostToDevice)) != cudaSuccess)
        return cleanup_fail(cuda_fail(e, "feod_create: fix-up rows copy"));
    }
    P.fixrows = h->fixrows;
  }
  if ((e = cudaMemsetAsync(h->flag, 0, sizeof(int) * 2, h->st)) != cudaSuccess)
    return cleanup_fail(cuda_fail(e, "feod_create: memset"));

  if (mesh->vertices) {
    const size_t nv = (size_t)(mesh->nx + 1) * (mesh->ny + 1) * (mesh->nz + 1) * 3;
    double* dverts = nullptr;
    const size_t ng = (size_t)h->Epad * 6 * qorder * qorder * qorder;
    if (cudaMalloc(&dverts, sizeof(double) * nv) != cudaSuccess) return cleanup_fail(fail(FEOD_ENOMEM, "feod_create: vertices"));
    if (cudaMalloc(&h->geom, sizeof(double) * ng) != cudaSuccess) {
      cudaFree(dverts);
      return cleanup_fail(fail(FEOD_ENOMEM, "feod_create: geometry (6 doubles per point)"));
    }
    e = cudaMemcpyAsync(dverts, mesh->vertices, sizeof(double) * nv, cudaMemcpyHostToDevice, h->st);
    if (e == cudaSuccess) e = launch_geometry(dverts, P, qorder, h->T, h->geom, h->flag, h->st);
    int bad = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&bad, h->flag, sizeof(int), cudaMemcpyDeviceToHost, h->st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->st);
    cudaFree(dverts);
    if (e != cudaSuccess) return cleanup_fail(cuda_fail(e, "feod_create: geometry"));
    if (bad) return cleanup_fail(fail(FEOD_EINVAL, "feod_create: mesh has an element with detJ <= 0"));
    P.geom = h->geom;
  } else {
    if ((e = cudaStreamSynchronize(h->st)) != cudaSuccess) return cleanup_fail(cuda_fail(e, "feod_create: sync"));
  }
  *out = h;
  return FEOD_OK;
}

extern "C" int feod_destroy(feod_handle h) {
  if (!h) return fail(FEOD_EINVAL, "feod_destroy: null handle");
  cudaStreamSynchronize(h->st);
  free_all(h);
  delete h;
  return FEOD_OK;
}

extern "C" int feod_set_stream(feod_handle h, void* cuda_stream) {
  if (!h) return fail(FEOD_EINVAL, "feod_set_stream: null handle");
  cudaStream_t ns = (cudaStream_t)cuda_stream;
  if (ns != h->st) {
    // the handle's scratch (tickets, shell slab, brick epochs) is shared by its calls:
    // work on the new stream starts after everything already queued on the old one
    if (!h->sw) CK(cudaEventCreateWithFlags(&h->sw, cudaEventDisableTiming), "feod_set_stream: event");
    CK(cudaEventRecord(h->sw, h->st), "feod_set_stream");
    CK(cudaStreamWaitEvent(ns, h->sw, 0), "feod_set_stream");
    h->st = ns;
  }
  return FEOD_OK;
}

extern "C" int feod_set_rho(feod_handle h, const double* rho) {
  if (!h || !rho) return fail(FEOD_EINVAL, "feod_set_rho: null argument");
  h->coeffs.rho = rho;
  h->P.rho = rho;
  return FEOD_OK;
}

extern "C" int feod_profile_next(feod_handle h, void* ev_begin, void* ev_end) {
  if (!h) return fail(FEOD_EINVAL, "feod_profile_next: null handle");
  h->prof_begin = (cudaEvent_t)ev_begin;
  h->prof_end = (cudaEvent_t)ev_end;
  return FEOD_OK;
}

extern "C" int64_t feod_num_dofs(feod_handle h) { return h ? h->N : -1; }
extern "C" int64_t feod_num_elems(feod_handle h) { return h ? h->E : -1; }

extern "C" int feod_brick_shape(feod_handle h, int* bx, int* by, int* bz) {
  if (!h) return fail(FEOD_EINVAL, "feod_brick_shape: null handle");
  if (bx) *bx = h->P.tbx;
  if (by) *by = h->P.tby;
  if (bz) *bz = h->P.tbz;
  return FEOD_OK;
}

static int run_op(feod_handle h, int mode, const double* in0, const double* in1, double* out0, double* out1,
                  double* gout, const char* name) {
  if (h->poisoned) return fail(FEOD_ECUDA, std::string(name) + ": handle unusable after a failed launch");
  OpPtrs p{in0, in1, out0, out1, h->shell, h->shell + (size_t)h->nbricks * h->P.shell_stride, gout};
  cudaEvent_t pb = h->prof_begin, pe = h->prof_end;
  h->prof_begin = h->prof_end = nullptr;
  if (pb) cudaEventRecord(pb, h->st);
  int grid = 0;
  // MODE_PAJVP reads the stored linearisation only, whatever the geometry
  const bool aff = mode == MODE_PAJVP ? true : h->geom == nullptr;
  if (h->nd == 7 && h->geom == nullptr && h->q6tc && (q6tc_supports(mode) || (mode == MODE_LIN && h->q6tc_lin)) &&
      (mode != MODE_RES || h->q6tc_res)) {
    // Q6 on affine meshes (residual, JVP, J^T w, linearisation, stored-linearisation JVP):
    // the FP64 tensor-core kernel + the assembly of its discontinuous L-vector (q6tc.cu)
    if (!h->evec && cudaMalloc(&h->evec, sizeof(double) * 343 * (size_t)h->E) != cudaSuccess) {   // nd = 7
      h->evec = nullptr;
      return fail(FEOD_ENOMEM, std::string(name) + ": element vector");
    }
    const CgFuse* fuse = (mode == MODE_JVP || mode == MODE_PAJVP) ? h->cg_fuse : nullptr;
    cudaError_t e = q6tc_run(mode, h->coeffs.model, h->P, h->T, in0, in1, h->evec, out0, fuse ? nullptr : h->dot_x,
                             fuse ? nullptr : h->dot_part, h->st, fuse);
    h->dot_fused = h->dot_x != nullptr;
    h->cg_fused = fuse != nullptr;
    h->dot_x = nullptr;
    h->dot_part = nullptr;
    h->cg_fuse = nullptr;
    if (pe) cudaEventRecord(pe, h->st);
    return e == cudaSuccess ? FEOD_OK : cuda_fail(e, name);
  }
  cudaError_t e = launch_nd(h->nd, mode, h->coeffs.model, aff, h->nbricks, h->P, h->T, p, h->st, &grid);
  if (pe) cudaEventRecord(pe, h->st);
  if (e != cudaSuccess) return cuda_fail(e, name);
  if (mode != MODE_DESIGN) {
    OpParams Pf = h->P;
    if (mode == MODE_VJP && h->P.vjp_keep_rows) Pf.faces = 0;   // J^T w keeps its Dirichlet rows (A17)
    e = fixup_nd(h->nd, Pf, p.shell0, out0, mode == MODE_JVPRES ? p.shell1 : nullptr,
                 mode == MODE_JVPRES ? out1 : nullptr, h->st);
    if (e != cudaSuccess) {
      h->poisoned = true;
      return cuda_fail(e, name);
    }
  }
  return FEOD_OK;
}

extern "C" int feod_residual(feod_handle h, const double* u, double* r) {
  if (!h || !u || !r) return fail(FEOD_EINVAL, "feod_residual: null argument");
  if ((const double*)r == u) return fail(FEOD_EINVAL, "feod_residual: r aliases u");
  return run_op(h, MODE_RES, u, nullptr, r, nullptr, nullptr, "feod_residual");
}

extern "C" int feod_jvp(feod_handle h, const double* u, const double* v, double* Jv) {
  if (!h || !u || !v || !Jv) return fail(FEOD_EINVAL, "feod_jvp: null argument");
  if ((const double*)Jv == u || (const double*)Jv == v) return fail(FEOD_EINVAL, "feod_jvp: Jv aliases an input");
  return run_op(h, MODE_JVP, u, v, Jv, nullptr, nullptr, "feod_jvp");
}

extern "C" int feod_jvp_res(feod_handle h, const double* u, const double* v, double* r, double* Jv) {
  if (!h || !u || !v || !Jv || !r) return fail(FEOD_EINVAL, "feod_jvp_res: null argument");
  if ((const double*)Jv == u || (const double*)Jv == v || (const double*)r == u || (const double*)r == v || r == Jv)
    return fail(FEOD_EINVAL, "feod_jvp_res: an output aliases another argument");
  return run_op(h, MODE_JVPRES, u, v, Jv, r, nullptr, "feod_jvp_res");
}

extern "C" int feod_vjp(feod_handle h, const double* u, const double* w, double* JTw) {
  if (!h || !u || !w || !JTw) return fail(FEOD_EINVAL, "feod_vjp: null argument");
  if ((const double*)JTw == u || (const double*)JTw == w) return fail(FEOD_EINVAL, "feod_vjp: JTw aliases an input");
  h->P.vjp_keep_rows = 1;
  return run_op(h, MODE_VJP, u, w, JTw, nullptr, nullptr, "feod_vjp");
}

extern "C" int feod_adjoint_solve(feod_handle h, const double* u, const double* rhs, double* lambda, int iters,
                                  double* res_norms_host) {
  if (!h || !u || !rhs || !lambda || iters < 0) return fail(FEOD_EINVAL, "feod_adjoint_solve: bad argument");
  if (lambda == u || lambda == rhs) return fail(FEOD_EINVAL, "feod_adjoint_solve: lambda aliases an input");
  const int64_t N = h->N;
  const size_t NP = ((size_t)N + 31) / 32 * 32;
  if (!h->kwork && cudaMalloc(&h->kwork, sizeof(double) * 7 * NP) != cudaSuccess) {
    h->kwork = nullptr;
    return fail(FEOD_ENOMEM, "feod_adjoint_solve: work vectors");
  }
  double* b = h->kwork;          // rhs with P^T applied
  double* r = b + NP;
  double* rhat = r + NP;
  double* p = rhat + NP;
  double* v = p + NP;
  double* s = v + NP;
  double* t = s + NP;
  double* part = h->red;
  double* part2 = h->red + kRedBlocks + 32;
  double* sc = h->red + kRedBlocks + 8;
  int* bad = h->flag + 1;
  // A y = P^T J(u)^T y on the free rows (y's Dirichlet entries are ignored by J^T)
  auto apply = [&](const double* y, double* out) {
    h->P.vjp_keep_rows = 0;
    const int rc = run_op(h, MODE_VJP, u, y, out, nullptr, nullptr, "feod_adjoint_solve");
    h->P.vjp_keep_rows = 1;
    return rc;
  };
  CK(cudaMemsetAsync(bad, 0, sizeof(int), h->st), "feod_adjoint_solve");
  CK(cudaMemcpyAsync(b, rhs, sizeof(double) * N, cudaMemcpyDeviceToDevice, h->st), "feod_adjoint_solve");
  CK(mask_dirichlet(b, h->P, h->st), "feod_adjoint_solve: mask");
  CK(bicg_init(b, lambda, r, rhat, p, v, N, h->st), "feod_adjoint_solve: init");
  std::vector<double> r2s;
  auto record = [&]() -> int {
    if (!res_norms_host) return FEOD_OK;
    double r2 = 0.0;
    CK(cudaMemcpyAsync(&r2, sc + 7, sizeof(double), cudaMemcpyDeviceToHost, h->st), "feod_adjoint_solve: D2H");
    CK(cudaStreamSynchronize(h->st), "feod_adjoint_solve: sync");
    r2s.push_back(std::sqrt(r2));
    return FEOD_OK;
  };
  CK(dot_partial(r, r, N, part, h->st), "feod_adjoint_solve: rr");
  CK(reduce_final(part, sc + 7, h->st), "feod_adjoint_solve: rr");
  CK(cudaMemcpyAsync(sc + 0, sc + 7, sizeof(double), cudaMemcpyDeviceToDevice, h->st), "feod_adjoint_solve");
  if (int rc = record()) return rc;
  for (int it = 0; it < iters; ++it) {
    // sc[it & 1] holds rho_new = (rhat, r)
    CK(bicg_p(sc, it, r, v, p, N, h->st), "feod_adjoint_solve: p");
    if (int rc = apply(p, v)) return rc;
    CK(dot_partial(rhat, v, N, part, h->st), "feod_adjoint_solve: rv");
    CK(reduce_final(part, sc + 4, h->st), "feod_adjoint_solve: rv");
    CK(bicg_s(sc, it, r, v, s, N, bad, h->st), "feod_adjoint_solve: s");
    if (int rc = apply(s, t)) return rc;
    CK(dot_partial(t, s, N, part, h->st), "feod_adjoint_solve: ts");
    CK(reduce_final(part, sc + 5, h->st), "feod_adjoint_solve: ts");
    CK(dot_partial(t, t, N, part, h->st), "feod_adjoint_solve: tt");
    CK(reduce_final(part, sc + 6, h->st), "feod_adjoint_solve: tt");
    CK(bicg_x(sc, p, s, t, rhat, lambda, r, N, part, part2, bad, h->st), "feod_adjoint_solve: x");
    CK(reduce_final(part, sc + ((it + 1) & 1), h->st), "feod_adjoint_solve: rho");
    CK(reduce_final(part2, sc + 7, h->st), "feod_adjoint_solve: rr");
    if (int rc = record()) return rc;
  }
  int hbad = 0;
  CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, h->st), "feod_adjoint_solve: D2H");
  CK(cudaStreamSynchronize(h->st), "feod_adjoint_solve: sync");
  if (res_norms_host)
    for (size_t i = 0; i < r2s.size(); ++i) res_norms_host[i] = r2s[i];
  if (hbad) return fail(FEOD_EINVAL, "feod_adjoint_solve: BiCGStab breakdown");
  return FEOD_OK;
}

extern "C" int feod_linearize(feod_handle h, const double* u, double* r) {
  if (!h || !u || !r) return fail(FEOD_EINVAL, "feod_linearize: null argument");
  if ((const double*)r == u) return fail(FEOD_EINVAL, "feod_linearize: r aliases u");
  if (!h->lin) {
    const size_t n = (size_t)lin_values(h->coeffs.model) * (size_t)h->Epad * h->q * h->q * h->q;
    if (cudaMalloc(&h->lin, sizeof(double) * n) != cudaSuccess) {
      h->lin = nullptr;
      return fail(FEOD_ENOMEM, "feod_linearize: linearisation buffer");
    }
    h->P.lin = h->lin;
  }
  const int rc = run_op(h, MODE_LIN, u, nullptr, r, nullptr, nullptr, "feod_linearize");
  h->lin_valid = rc == FEOD_OK;
  return rc;
}

extern "C" int feod_jvp_lin(feod_handle h, const double* v, double* Jv) {
  if (!h || !v || !Jv) return fail(FEOD_EINVAL, "feod_jvp_lin: null argument");
  if ((const double*)Jv == v) return fail(FEOD_EINVAL, "feod_jvp_lin: Jv aliases v");
  if (!h->lin_valid) return fail(FEOD_EINVAL, "feod_jvp_lin: no linearisation stored (call feod_linearize)");
  return run_op(h, MODE_PAJVP, v, nullptr, Jv, nullptr, nullptr, "feod_jvp_lin");
}

extern "C" int feod_set_newton_linearization(feod_handle h, int stored) {
  if (!h || stored < 0 || stored > 2) return fail(FEOD_EINVAL, "feod_set_newton_linearization: bad argument");
  h->newton_lin = stored;
  return FEOD_OK;
}

extern "C" int feod_jacobi_diag(feod_handle h, double* diag) {
  if (!h || !diag) return fail(FEOD_EINVAL, "feod_jacobi_diag: null argument");
  if (!h->lin_valid) return fail(FEOD_EINVAL, "feod_jacobi_diag: no linearisation stored (call feod_linearize)");
  const size_t evn = (size_t)h->nd * h->nd * h->nd * (size_t)h->E;   // discontinuous L-vector
  if (!h->evec && cudaMalloc(&h->evec, sizeof(double) * evn) != cudaSuccess) {
    h->evec = nullptr;
    return fail(FEOD_ENOMEM, "feod_jacobi_diag: element vector");
  }
  if (h->nd == 7 && h->geom == nullptr && h->q6tc) {   // Q6 affine: the tensor-core diagonal (q6tc.cu)
    CK(q6tc_diag(h->coeffs.model, h->P, h->T, h->evec, diag, h->st), "feod_jacobi_diag");
    return FEOD_OK;
  }
  CK(jacobi_diag_nd(h->nd, h->coeffs.model, h->P, h->T, h->evec, diag, h->st), "feod_jacobi_diag");
  return FEOD_OK;
}

extern "C" int feod_element_matrices(feod_handle h, const double* u, int64_t e0, int64_t ne, int elm, double* Ke) {
  if (!h || !u || !Ke) return fail(FEOD_EINVAL, "feod_element_matrices: null argument");
  if (e0 < 0 || ne < 0 || e0 + ne > h->E || (elm != 0 && elm != 1))
    return fail(FEOD_EINVAL, "feod_element_matrices: element range or mode out of bounds");
  if (h->coeffs.model == FEOD_HEAT_DESIGN && !h->P.rho) return fail(FEOD_EINVAL, "feod_element_matrices: rho unset");
  if (ne == 0) return FEOD_OK;
  const bool affine = h->geom == nullptr;
  if (elm) {   // element-level forward AD through B, D, B^T (Table 1's ELM), elm.cu
    const size_t per = elm_scratch_per_cta(h->nd);
    if (per && !h->em_scr) {   // Q4..Q6: the seeds' tangent arrays for up to 2 CTAs per SM
      const size_t n = per * (size_t)(h->E < 2 * 148 ? h->E : 2 * 148);
      if (cudaMalloc(&h->em_scr, sizeof(double) * n) != cudaSuccess) {
        h->em_scr = nullptr;
        return fail(FEOD_ENOMEM, "feod_element_matrices: ELM scratch");
      }
      h->em_scr_n = n;
    }
    CK(element_matrices_elm_nd(h->nd, h->coeffs.model, affine, h->P, h->T, u, (int)e0, (int)ne, Ke, h->em_scr,
                               h->em_scr_n, h->st),
       "feod_element_matrices");
  } else if (h->nd <= 4) {   // integration-point AD + K_e = M^T N on the FP64 tensor cores (Table 1's RES), elemat.cu
    CK(element_matrices_nd(h->nd, h->coeffs.model, affine, false, h->P, h->T, u, (int)e0, (int)ne, Ke, h->st),
       "feod_element_matrices");
  } else {     // Q4..Q6: the same product tiled, operands generated on chip (elemat_hi.cu)
    CK(element_matrices_hi_nd(h->nd, h->coeffs.model, affine, h->P, h->T, u, (int)e0, (int)ne, Ke, h->st),
       "feod_element_matrices");
  }
  return FEOD_OK;
}

extern "C" int feod_design_grad(feod_handle h, const double* u, const double* lambda, double* g) {
  if (!h || !u || !lambda || !g) return fail(FEOD_EINVAL, "feod_design_grad: null argument");
  if (h->coeffs.model != FEOD_HEAT_DESIGN) return fail(FEOD_EINVAL, "feod_design_grad: model has no rho");
  if ((const double*)g == u || (const double*)g == lambda) return fail(FEOD_EINVAL, "feod_design_grad: g aliases an input");
  return run_op(h, MODE_DESIGN, u, lambda, nullptr, nullptr, g, "feod_design_grad");
}

extern "C" int feod_res_design_grad(feod_handle h, const double* u, const double* lambda, double* r, double* g) {
  if (!h || !u || !lambda || !r || !g) return fail(FEOD_EINVAL, "feod_res_design_grad: null argument");
  if (h->coeffs.model != FEOD_HEAT_DESIGN) return fail(FEOD_EINVAL, "feod_res_design_grad: model has no rho");
  if ((const double*)r == u || (const double*)r == lambda || (const double*)g == u || (const double*)g == lambda ||
      r == g)
    return fail(FEOD_EINVAL, "feod_res_design_grad: an output aliases another argument");
  if (h->bi.ptx > 1)   // column kernel: one dual pass gives both
    return run_op(h, MODE_RESDES, u, lambda, r, nullptr, g, "feod_res_design_grad");
  const int rc = feod_residual(h, u, r);   // plane-kernel orders: the two calls
  return rc ? rc : feod_design_grad(h, u, lambda, g);
}

extern "C" int feod_apply_host(feod_handle h, int op, const double* in0, const double* in1, double* out) {
  if (!h || !in0 || !out || (op != 0 && !in1)) return fail(FEOD_EINVAL, "feod_apply_host: null argument");
  if (op < 0 || op > 4) return fail(FEOD_EINVAL, "feod_apply_host: op must be 0 .. 4");
  const int64_t len = h->N > h->E ? h->N : h->E;
  if (!h->stage && cudaMalloc(&h->stage, sizeof(double) * 4 * (size_t)len) != cudaSuccess) {
    h->stage = nullptr;
    return fail(FEOD_ENOMEM, "feod_apply_host: staging buffers");
  }
  double* d0 = h->stage;
  double* d1 = h->stage + len;
  double* d2 = h->stage + 2 * len;
  if (op == 4) {
    // r = F(u) and Jv = J(u) v with the copies on two more streams: v's upload
    // overlaps the residual and r's download (opposite direction), which in turn
    // overlaps the JVP
    double* d3 = h->stage + 3 * len;
    const size_t bytes = sizeof(double) * (size_t)h->N;
    if (!h->cst) {
      CK(cudaStreamCreateWithFlags(&h->cst, cudaStreamNonBlocking), "feod_apply_host: stream");
      CK(cudaStreamCreateWithFlags(&h->dst, cudaStreamNonBlocking), "feod_apply_host: stream");
      for (cudaEvent_t& e : h->ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "feod_apply_host: event");
    }
    CK(cudaEventRecord(h->ev[3], h->st), "feod_apply_host");        // earlier work on the handle's stream
    CK(cudaStreamWaitEvent(h->cst, h->ev[3], 0), "feod_apply_host");
    CK(cudaMemcpyAsync(d0, in0, bytes, cudaMemcpyHostToDevice, h->cst), "feod_apply_host: H2D");
    CK(cudaEventRecord(h->ev[0], h->cst), "feod_apply_host");
    CK(cudaMemcpyAsync(d1, in1, bytes, cudaMemcpyHostToDevice, h->cst), "feod_apply_host: H2D");
    CK(cudaEventRecord(h->ev[1], h->cst), "feod_apply_host");
    CK(cudaStreamWaitEvent(h->st, h->ev[0], 0), "feod_apply_host");
    int rc = feod_residual(h, d0, d2);
    if (rc != FEOD_OK) return rc;
    CK(cudaEventRecord(h->ev[2], h->st), "feod_apply_host");
    CK(cudaStreamWaitEvent(h->st, h->ev[1], 0), "feod_apply_host");
    rc = feod_jvp(h, d0, d1, d3);
    if (rc != FEOD_OK) return rc;
    CK(cudaStreamWaitEvent(h->dst, h->ev[2], 0), "feod_apply_host");
    CK(cudaMemcpyAsync(out, d2, bytes, cudaMemcpyDeviceToHost, h->dst), "feod_apply_host: D2H");   // against v's upload
    CK(cudaMemcpyAsync(out + h->N, d3, bytes, cudaMemcpyDeviceToHost, h->st), "feod_apply_host: D2H");
    CK(cudaStreamSynchronize(h->st), "feod_apply_host: sync");
    CK(cudaStreamSynchronize(h->cst), "feod_apply_host: sync");
    CK(cudaStreamSynchronize(h->dst), "feod_apply_host: sync");
    return FEOD_OK;
  }
  CK(cudaMemcpyAsync(d0, in0, sizeof(double) * h->N, cudaMemcpyHostToDevice, h->st), "feod_apply_host: H2D");
  if (op != 0) CK(cudaMemcpyAsync(d1, in1, sizeof(double) * h->N, cudaMemcpyHostToDevice, h->st), "feod_apply_host: H2D");
  int rc = op == 0 ? feod_residual(h, d0, d2)
           : op == 1 ? feod_jvp(h, d0, d1, d2)
           : op == 2 ? feod_design_grad(h, d0, d1, d2)
                     : feod_vjp(h, d0, d1, d2);
  if (rc != FEOD_OK) return rc;
  const int64_t nout = op == 2 ? h->E : h->N;
  CK(cudaMemcpyAsync(out, d2, sizeof(double) * nout, cudaMemcpyDeviceToHost, h->st), "feod_apply_host: D2H");
  CK(cudaStreamSynchronize(h->st), "feod_apply_host: sync");
  return FEOD_OK;
}

// A stream of independent host-buffer problems (one (in0[b], in1[b]) -> out[b] per step):
// two device staging sets, uploads on cst, the operator on the handle's stream, downloads
// on dst. Step b + 1's uploads run while step b computes and downloads (the host link is
// full duplex), so in steady state a step costs max(H2D, D2H, operator) instead of their sum.
// A set's input half is reused as soon as step b-2's operator has read it and its output
// half once step b-2's results are down: with one release point per set the period would be
// (H2D + operator + D2H) / 2 instead.
extern "C" int feod_apply_host_batch(feod_handle h, int op, int64_t nbatch, const double* const* in0,
                                     const double* const* in1, double* const* out) {
  if (!h || nbatch < 0 || (nbatch > 0 && (!in0 || !out || (op != 0 && !in1))))
    return fail(FEOD_EINVAL, "feod_apply_host_batch: null argument");
  if (op < 0 || op > 4) return fail(FEOD_EINVAL, "feod_apply_host_batch: op must be 0 .. 4");
  for (int64_t b = 0; b < nbatch; ++b)
    if (!in0[b] || !out[b] || (op != 0 && !in1[b])) return fail(FEOD_EINVAL, "feod_apply_host_batch: null buffer");
  if (nbatch == 0) return FEOD_OK;
  const int64_t len = h->N > h->E ? h->N : h->E;
  for (double** sp : {&h->stage, &h->stage2})
    if (!*sp && cudaMalloc(sp, sizeof(double) * 4 * (size_t)len) != cudaSuccess) {
      *sp = nullptr;
      return fail(FEOD_ENOMEM, "feod_apply_host_batch: staging buffers");
    }
  if (!h->cst) {
    CK(cudaStreamCreateWithFlags(&h->cst, cudaStreamNonBlocking), "feod_apply_host_batch: stream");
    CK(cudaStreamCreateWithFlags(&h->dst, cudaStreamNonBlocking), "feod_apply_host_batch: stream");
    for (cudaEvent_t& e : h->ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "feod_apply_host_batch");
  }
  if (!h->bev[0]) {
    for (cudaEvent_t& e : h->bev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "feod_apply_host_batch");
    for (cudaEvent_t& e : h->bdown) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "feod_apply_host_batch");
  }
  const size_t nb_in = sizeof(double) * (size_t)h->N;
  const size_t nb_out = sizeof(double) * (size_t)(op == 2 ? h->E : h->N);
  CK(cudaEventRecord(h->ev[3], h->st), "feod_apply_host_batch");   // earlier work on the handle's stream
  CK(cudaStreamWaitEvent(h->cst, h->ev[3], 0), "feod_apply_host_batch");
  for (int64_t b = 0; b < nbatch; ++b) {
    const int s = (int)(b & 1);
    double* d0 = s ? h->stage2 : h->stage;
    double *d1 = d0 + len, *d2 = d0 + 2 * len, *d3 = d0 + 3 * len;
    cudaEvent_t up = h->bev[3 * s], rdy_r = h->bev[3 * s + 1], rdy = h->bev[3 * s + 2], down = h->bdown[s];
    // inputs of set s are free once step b-2's operator ran, its outputs once they are downloaded
    if (b >= 2) CK(cudaStreamWaitEvent(h->cst, rdy, 0), "feod_apply_host_batch");
    CK(cudaMemcpyAsync(d0, in0[b], nb_in, cudaMemcpyHostToDevice, h->cst), "feod_apply_host_batch: H2D");
    if (op != 0) CK(cudaMemcpyAsync(d1, in1[b], nb_in, cudaMemcpyHostToDevice, h->cst), "feod_apply_host_batch: H2D");
    CK(cudaEventRecord(up, h->cst), "feod_apply_host_batch");
    CK(cudaStreamWaitEvent(h->st, up, 0), "feod_apply_host_batch");
    if (b >= 2) CK(cudaStreamWaitEvent(h->st, down, 0), "feod_apply_host_batch");
    int rc = op == 0 || op == 4 ? feod_residual(h, d0, d2)
             : op == 1          ? feod_jvp(h, d0, d1, d2)
             : op == 2          ? feod_design_grad(h, d0, d1, d2)
                                : feod_vjp(h, d0, d1, d2);
    if (rc != FEOD_OK) return rc;
    CK(cudaEventRecord(rdy_r, h->st), "feod_apply_host_batch");
    if (op == 4 && (rc = feod_jvp(h, d0, d1, d3)) != FEOD_OK) return rc;
    CK(cudaEventRecord(rdy, h->st), "feod_apply_host_batch");
    CK(cudaStreamWaitEvent(h->dst, rdy_r, 0), "feod_apply_host_batch");   // r downloads while the JVP runs
    CK(cudaMemcpyAsync(out[b], d2, nb_out, cudaMemcpyDeviceToHost, h->dst), "feod_apply_host_batch: D2H");
    if (op == 4) {
      CK(cudaStreamWaitEvent(h->dst, rdy, 0), "feod_apply_host_batch");
      CK(cudaMemcpyAsync(out[b] + h->N, d3, nb_out, cudaMemcpyDeviceToHost, h->dst), "feod_apply_host_batch: D2H");
    }
    CK(cudaEventRecord(down, h->dst), "feod_apply_host_batch");
  }
  CK(cudaStreamSynchronize(h->st), "feod_apply_host_batch: sync");
  CK(cudaStreamSynchronize(h->cst), "feod_apply_host_batch: sync");
  CK(cudaStreamSynchronize(h->dst), "feod_apply_host_batch: sync");
  return FEOD_OK;
}

extern "C" int feod_dot(feod_handle h, const double* x, const double* y, int64_t n, double* result) {
  if (!h || !x || !y || !result || n < 0) return fail(FEOD_EINVAL, "feod_dot: bad argument");
  CK(dot_partial(x, y, n, h->red, h->st), "feod_dot");
  CK(reduce_final(h->red, result, h->st), "feod_dot");
  return FEOD_OK;
}

extern "C" int feod_newton_cg(feod_handle h, double* u, int newton_steps, int cg_iters, double* norms_host) {
  if (!h || !u || !norms_host || newton_steps < 0 || cg_iters < 0)
    return fail(FEOD_EINVAL, "feod_newton_cg: bad argument");
  const int64_t N = h->N;
  if (!h->work && cudaMalloc(&h->work, sizeof(double) * 5 * (size_t)N) != cudaSuccess) {
    h->work = nullptr;
    return fail(FEOD_ENOMEM, "feod_newton_cg: work vectors");
  }
  double* F = h->work;
  double* r = F + N;
  double* p = r + N;
  double* Ap = p + N;
  double* d = Ap + N;
  double* part = h->red;                       // pAp partials (dot_partial)
  double* part2 = h->red + kRedBlocks + 32;    // r.z partials (cg_update)
  double* sc = h->red + kRedBlocks;   // sc[0], sc[2]: rz ping-pong; sc[1]: pAp; sc[3]: ||F||^2
  int* bad = h->flag + 1;
  CK(cudaMemsetAsync(bad, 0, sizeof(int), h->st), "feod_newton_cg");
  // The CG iterations of a Newton step: 5 launches each (operator + fix-up, p.Ap partials,
  // the update with alpha reduced in-kernel and the r.z partials, the direction with beta
  // reduced in-kernel). Every kernel argument is fixed for the handle, u and the
  // preconditioner (DevState holds the per-call scheduling state), so the loop is captured
  // once as a CUDA graph on an internal stream and replayed every Newton step.
  auto cg_body = [&](cudaStream_t st, const double* pre) -> int {
    cudaStream_t keep = h->st;
    h->st = st;
    for (int it = 0; it < cg_iters; ++it) {
      double* rr_old = sc + ((it & 1) ? 2 : 0);
      double* rr_new = sc + ((it & 1) ? 0 : 2);
      // p.Ap: fused into the operator's assembly where the path has one (Q6), else a pass
      // ... and, on the Q6 tensor-core path, the whole update behind the assembly (CgFuse:
      // Ap is then never written; r, the r.z partials, p.Ap and the breakdown flag are)
      const CgFuse fz{rr_old, part, sc + 1, r, part2, bad, pre};
      h->dot_x = p;
      h->dot_part = part;
      h->dot_fused = false;
      h->cg_fuse = h->cg_fusion ? &fz : nullptr;
      h->cg_fused = false;
      const int rc = h->newton_lin ? feod_jvp_lin(h, p, Ap) : feod_jvp(h, u, p, Ap);
      const bool fused = h->dot_fused, updated = h->cg_fused;
      h->dot_x = nullptr;
      h->dot_part = nullptr;
      h->cg_fuse = nullptr;
      h->cg_fused = false;
      if (rc) { h->st = keep; return rc; }
      cudaError_t e = (fused || updated) ? cudaSuccess : dot_partial(p, Ap, N, part, st);
      if (e == cudaSuccess && !updated) e = cg_update(rr_old, part, sc + 1, Ap, r, N, part2, bad, st, pre);
      if (e == cudaSuccess) e = cg_dir(part2, rr_new, rr_old, sc + 1, r, p, d, N, st, pre);
      if (e != cudaSuccess) { h->st = keep; return cuda_fail(e, "feod_newton_cg: CG"); }
    }
    h->st = keep;
    return FEOD_OK;
  };
  for (int step = 0; step <= newton_steps; ++step) {
    int rc = h->newton_lin ? feod_linearize(h, u, F) : feod_residual(h, u, F);
    if (rc) return rc;
    const double* pre = nullptr;
    if (h->newton_lin == 2 && step < newton_steps) {
      if (!h->jdiag && cudaMalloc(&h->jdiag, sizeof(double) * (size_t)N) != cudaSuccess) {
        h->jdiag = nullptr;
        return fail(FEOD_ENOMEM, "feod_newton_cg: Jacobi diagonal");
      }
      if ((rc = feod_jacobi_diag(h, h->jdiag))) return rc;
      pre = h->jdiag;
    }
    CK(dot_partial(F, F, N, part, h->st), "feod_newton_cg: norm");
    CK(reduce_final(part, sc + 3, h->st), "feod_newton_cg: norm");
    double ff = 0.0;
    CK(cudaMemcpyAsync(&ff, sc + 3, sizeof(double), cudaMemcpyDeviceToHost, h->st), "feod_newton_cg: D2H");
    CK(cudaStreamSynchronize(h->st), "feod_newton_cg: sync");
    norms_host[step] = std::sqrt(ff);
    if (step == newton_steps) break;
    CK(cg_init(F, r, p, d, N, h->st, pre), "feod_newton_cg: init");
    CK(dot_partial(r, p, N, part, h->st), "feod_newton_cg: rz");   // p = z = M^{-1} r
    CK(reduce_final(part, sc + 0, h->st), "feod_newton_cg: rr");
    if (cg_iters > 0) {
      const bool want_graph = h->cg_graphs && !h->cg_graph_failed;
      const uint64_t key = (reinterpret_cast<uint64_t>(u) ^ (reinterpret_cast<uint64_t>(pre) << 1)) * 31 +
                           (uint64_t)(h->newton_lin * 1000003 + cg_iters);
      if (want_graph && (!h->cg_exec || h->cg_key != key)) {
        if (h->cg_exec) { cudaGraphExecDestroy(h->cg_exec); h->cg_exec = nullptr; }
        if (!h->gst) {
          CK(cudaStreamCreateWithFlags(&h->gst, cudaStreamNonBlocking), "feod_newton_cg: stream");
          for (cudaEvent_t& ev : h->ev_g) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "feod_newton_cg: event");
        }
        cudaGraph_t g = nullptr;
        cudaError_t e = cudaStreamBeginCapture(h->gst, cudaStreamCaptureModeThreadLocal);
        int crc = e == cudaSuccess ? cg_body(h->gst, pre) : FEOD_ECUDA;
        cudaError_t e2 = cudaStreamEndCapture(h->gst, &g);
        if (e == cudaSuccess && crc == FEOD_OK && e2 == cudaSuccess && g)
          e = cudaGraphInstantiate(&h->cg_exec, g, 0);
        else
          e = cudaErrorStreamCaptureInvalidated;
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();   // a failed capture leaves no sticky error
        if (e != cudaSuccess) { h->cg_exec = nullptr; h->cg_graph_failed = true; }
        else h->cg_key = key;
      }
      if (want_graph && h->cg_exec) {
        CK(cudaEventRecord(h->ev_g[0], h->st), "feod_newton_cg");
        CK(cudaStreamWaitEvent(h->gst, h->ev_g[0], 0), "feod_newton_cg");
        CK(cudaGraphLaunch(h->cg_exec, h->gst), "feod_newton_cg: graph");
        CK(cudaEventRecord(h->ev_g[1], h->gst), "feod_newton_cg");
        CK(cudaStreamWaitEvent(h->st, h->ev_g[1], 0), "feod_newton_cg");
        ++h->cg_graph_launches;
      } else if ((rc = cg_body(h->st, pre))) {
        return rc;
      }
    }
    CK(axpy1(u, d, N, h->st), "feod_newton_cg: u += d");
    int hbad = 0;
    CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, h->st), "feod_newton_cg: D2H");
    CK(cudaStreamSynchronize(h->st), "feod_newton_cg: sync");
    if (hbad) return fail(FEOD_EINVAL, "feod_newton_cg: CG breakdown (p^T J p <= 0)");
  }
  return FEOD_OK;
}

extern "C" int feod_set_cg_graphs(feod_handle h, int enable) {
  if (!h || enable < 0 || enable > 1) return fail(FEOD_EINVAL, "feod_set_cg_graphs: bad argument");
  h->cg_graphs = enable != 0;
  h->cg_graph_failed = false;
  return FEOD_OK;
}

extern "C" int feod_set_cg_fusion(feod_handle h, int enable) {
  if (!h || enable < 0 || enable > 1) return fail(FEOD_EINVAL, "feod_set_cg_fusion: bad argument");
  h->cg_fusion = enable != 0;
  if (h->cg_exec) { cudaGraphExecDestroy(h->cg_exec); h->cg_exec = nullptr; }   // recapture with the other body
  return FEOD_OK;
}

extern "C" int64_t feod_cg_graph_launches(feod_handle h) { return h ? h->cg_graph_launches : -1; }
