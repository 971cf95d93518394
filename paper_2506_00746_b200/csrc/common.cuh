// Shared device-side definitions of libfeod (product path; independent of oracle/).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define FEOD_DEV __device__ __forceinline__
#define FEOD_HD __host__ __device__ __forceinline__

namespace feod {

// MODE_RESDES: r = F(u) and g_e = -lambda^T dF/drho_e from one dual pass (feod_res_design_grad;
// column kernel only -- the plane-kernel orders compose it from MODE_RES and MODE_DESIGN)
enum Mode { MODE_RES = 0, MODE_JVP = 1, MODE_JVPRES = 2, MODE_DESIGN = 3, MODE_VJP = 4, MODE_LIN = 5, MODE_PAJVP = 6,
            MODE_RESDES = 7 };
constexpr int kModes = 8;
enum Model { PLAPLACE = 0, NLDIFF = 1, HEAT = 2 };
constexpr int kMaxNQ = 8;

// 1D tables, passed by value as a kernel parameter: the entries sit in the
// constant bank and feed DFMA directly (uniform across the warp).
//   B[i][a] = l_a(x_i), G[i][a] = l_a'(x_i)  (GLL Lagrange basis at Gauss points)
//   w[i]    = 1D Gauss weight on [0,1]; wi2[i] = 1 / w[i]^2
//   x[i]    = 1D Gauss point on [0,1] (geometry setup only)
//   D[i][m] = L_m'(x_i), L_m the Lagrange polynomial of the Gauss points
//             (collocated derivative: sum_m D[i][m] B[m][a] = G[i][a] exactly,
//             since l_a has degree k <= q-1)
// Values per quadrature point of the stored linearisation (MODE_LIN -> MODE_PAJVP,
// SURVEY §8(f) NEXT-2): dFh/dgh (symmetric, 6) and, when kappa depends on u, dFh/du (3).
FEOD_HD constexpr int lin_values(int model) { return model == 0 ? 6 : 9; }

struct Tables {
  double B[kMaxNQ][kMaxNQ];
  double G[kMaxNQ][kMaxNQ];
  double D[kMaxNQ][kMaxNQ];
  double w[kMaxNQ];
  double wi2[kMaxNQ];   // 1 / w[i]^2
  double x[kMaxNQ];
  // weight-folded tables of the affine column kernel (col_kernel.cuh FOLD): with
  // M = w_q diag(c) and F = w_q Ft, the quadrature weight w_q = w_i w_j w_l moves out of
  // the per-point work into the transposed 1D operators:
  //   Dh[i][m] = D[i][m] w_i / w_m  (R = w_q Rt at the points),  Bw[i][a] = w_i B[i][a]
  double Dh[kMaxNQ][kMaxNQ];
  double Bw[kMaxNQ][kMaxNQ];
  // products for the Jacobi diagonal (diag.cu): B2 = B^2, G2 = G^2, GB = G B (entrywise)
  double B2[kMaxNQ][kMaxNQ];
  double G2[kMaxNQ][kMaxNQ];
  double GB[kMaxNQ][kMaxNQ];
  double Gw[kMaxNQ][kMaxNQ];   // w_i G[i][a] (weight-folded z-transpose of the Q6 tensor-core kernel)
};

// Device-resident scheduler state of one handle.
//   sched  ticket counter: the CTA that draws the last ticket of a launch (#bricks + grid
//          tickets in all) resets it to 0, so every launch starts from 0
//   epoch  operator calls completed; a call's bricks publish bdone[b] = epoch + 1, and the
//          same last-ticket CTA advances it (pointwise.cuh claim_brick)
//   cur    epoch + 1 of the running call, for its scatter fix-up (pointwise.cuh call_begin)
struct DevState {
  unsigned long long sched;
  unsigned long long epoch;
  unsigned long long cur;
  unsigned long long pad;
};

// Everything a fused operator kernel needs besides the vectors.
struct OpParams {
  int nx, ny, nz;        // elements per axis
  int Mx, My, Mz;        // DOFs per axis (k n + 1)
  int nbx, nby, nbz;     // bricks per axis
  int shell_stride;      // doubles per brick in the shell buffer
  uint32_t faces;        // Dirichlet face bits
  // physics
  double half_pm2;       // (p-2)/2 (PLAPLACE)
  int pcase;             // half_pm2 == 0 / 1 / 0.5 / other: 0 / 1 / 2 / 3 (dual.cuh pow_case)
  double eps2;           // eps^2
  double f;              // source
  // geometry: uniform grid (geom == nullptr): M = w_q diag(cx, cy, cz), W = w_q * vol
  double cx, cy, cz, vol;
  double cxv, cyv, czv;  // cx / vol, cy / vol, cz / vol: |grad u|^2 = sum_d c_d gh_d^2 / vol on such grids
  const double* geom;    // [E][NQ][6][NQ][NQ] metric, components xx yy zz xy xz yz
  double* lin;           // [E][NQ][lin_values][NQ][NQ] stored linearisation (MODE_LIN writes, MODE_PAJVP reads)
  int vjp_keep_rows;     // MODE_VJP: 1 keeps every row of J^T w (feod_vjp), 0 applies P^T (adjoint solve)
  const double* rho;     // [E] (HEAT)
  // dynamic brick scheduling and the scatter fix-up's dependencies, all on the device
  // (DevState): the kernel arguments do not change from call to call, so a sequence of
  // calls can be captured in a CUDA graph
  DevState* ds;
  // bdone[b] = epoch + 1 of the last call whose operator kernel finished brick b's
  // stores (release); fixrows = the fix-up rows in launch order
  unsigned long long* bdone;
  const int2* fixrows;
  int nfixrows;
  // brick shape in elements (the fix-up reads it at run time; both kernel families)
  int tbx, tby, tbz;
  // per-point streams (metric, stored linearisation): element (ex, ey, ez) lives in
  // chunk ((ez ny + ey) pnbx + ex / ptx), its values interleaved with the ptx - 1 other
  // elements of the chunk: value w of the element at chunk * (nv q^3 ptx) + w ptx + ex % ptx.
  // ptx = 1 (pnbx = nx) is plain element-major; the column kernel (Q1, Q2) uses ptx = its
  // tile width, so that a warp's threads (consecutive elements) read consecutive doubles
  int ptx, pnbx;
};

// Base index and stride of an element's per-point values (OpParams::ptx).
FEOD_HD int64_t pt_base(const OpParams& P, int ex, int ey, int ez, int nvq3) {
  const int64_t chunk = ((int64_t)ez * P.ny + ey) * P.pnbx + ex / P.ptx;
  return chunk * (int64_t)nvq3 * P.ptx + ex % P.ptx;
}

#ifdef __CUDACC__
FEOD_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Streaming load that the compiler may not sink toward its use (per-point streams).
FEOD_DEV double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// mbarriers (shared memory, CTA scope)
FEOD_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
FEOD_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
FEOD_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
FEOD_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// 1D bulk copy global -> shared by the TMA engine, completion counted on bar
// (16-byte aligned source, destination and size)
FEOD_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// L2 prefetch of a contiguous byte range by the bulk-copy engine (no completion
// tracking); start and size must be 16-byte multiples.
FEOD_DEV void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
#endif

FEOD_HD bool is_dirichlet(int X, int Y, int Z, int Mx, int My, int Mz, uint32_t faces) {
  return ((faces & 1u) && X == 0) || ((faces & 2u) && X == Mx - 1) ||
         ((faces & 4u) && Y == 0) || ((faces & 8u) && Y == My - 1) ||
         ((faces & 16u) && Z == 0) || ((faces & 32u) && Z == Mz - 1);
}

// Rank of a point on the surface of an LX x LY x LZ box (any coordinate at 0
// or L-1): z=0 plane, then for each middle z a ring, then the z=L-1 plane.
FEOD_HD int shell_rank(int X, int Y, int Z, int LX, int LY, int LZ) {
  if (Z == 0) return X + LX * Y;
  const int base = LX * LY;
  const int ring = 2 * LX + 2 * (LY - 2);
  if (Z == LZ - 1) return base + (LZ - 2) * ring + X + LX * Y;
  const int r = base + (Z - 1) * ring;
  if (Y == 0) return r + X;
  if (Y == LY - 1) return r + LX + X;
  return r + 2 * LX + 2 * (Y - 1) + (X == 0 ? 0 : 1);
}

FEOD_HD int shell_size(int LX, int LY, int LZ) {
  return LX * LY * LZ - (LX - 2) * (LY - 2) * (LZ - 2);
}

}  // namespace feod
