// Shared device-side definitions of libfeod (product path; independent of oracle/).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define FEOD_DEV __device__ __forceinline__
#define FEOD_HD __host__ __device__ __forceinline__

namespace feod {

enum Mode { MODE_RES = 0, MODE_JVP = 1, MODE_JVPRES = 2, MODE_DESIGN = 3, MODE_VJP = 4, MODE_LIN = 5, MODE_PAJVP = 6 };
constexpr int kModes = 7;
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
  double eps2;           // eps^2
  double f;              // source
  // geometry: uniform grid (geom == nullptr): M = w_q diag(cx, cy, cz), W = w_q * vol
  double cx, cy, cz, vol;
  const double* geom;    // [E][NQ][6][NQ][NQ] metric, components xx yy zz xy xz yz
  double* lin;           // [E][NQ][lin_values][NQ][NQ] stored linearisation (MODE_LIN writes, MODE_PAJVP reads)
  int vjp_keep_rows;     // MODE_VJP: 1 keeps every row of J^T w (feod_vjp), 0 applies P^T (adjoint solve)
  const double* rho;     // [E] (HEAT)
  // dynamic brick scheduling: tickets atomicAdd(sched, 1) - sched_base < #bricks
  // are bricks, the rest end a CTA; the host advances sched_base by #bricks + grid
  unsigned long long* sched;
  unsigned long long sched_base;
  // fix-up dependencies: bdone[b] = sched_base + 1 of the last call whose IO warp
  // finished brick b's stores (release); fixrows = the fix-up rows in launch order
  unsigned long long* bdone;
  const int2* fixrows;
  int nfixrows;
};

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

// Brick shape for order k = ND-1: a CTA owns a BX x BY tile of elements and
// sweeps BZ element layers along z; one layer of BX*BY
// elements is processed concurrently, NQ*NQ threads per element.
// SB = sub-batches per layer: with SB = 2 the layer's even and odd element rows
// (y) are processed one after the other by the same threads (half the threads
// for twice the tile).
template <int ND> struct BrickShape;
template <> struct BrickShape<2> { static constexpr int BX = 8, BY = 8, BZ = 16, SB = 1; };
template <> struct BrickShape<3> { static constexpr int BX = 4, BY = 4, BZ = 16, SB = 1; };
template <> struct BrickShape<4> { static constexpr int BX = 4, BY = 4, BZ = 8, SB = 2; };
template <> struct BrickShape<5> { static constexpr int BX = 4, BY = 2, BZ = 8, SB = 1; };
template <> struct BrickShape<6> { static constexpr int BX = 2, BY = 2, BZ = 8, SB = 1; };
template <> struct BrickShape<7> { static constexpr int BX = 2, BY = 2, BZ = 8, SB = 1; };

}  // namespace feod
