// K5 — deterministic scatter fix-up: the G^T step for the DOFs on faces shared
// by neighbouring bricks. Each shared DOF sums the shell values
// its 2, 4 or 8 bricks wrote, in a fixed order (z, y, x ascending: low brick
// first), and applies P^T (0 on Dirichlet rows). No atomics: the result is
// bitwise reproducible run to run.
//
// The tile shape (K, BX, BY, BZ) is a template parameter, so every brick index
// is a division by a constant. Work is laid out as rows so that one CTA row has
// uniform y/z bookkeeping and consecutive threads touch consecutive X (or Y):
//   set Y: DOF planes Y = m PY (m = 1..nby-1), rows along X (X on an x-plane skipped), per (m, Z)
//   set X: planes X = m PX, rows along Y, per (m, Z) (x-y / x-z edges and corners too)
//   set Z: planes Z = m PZ, rows along X (X on an x-plane or Y on a y-plane skipped), per (m, Y)
// Shell slab of a brick with box LX x LY x LZ (common.cuh shell_rank): the z = 0
// plane, one ring per middle z, the z = LZ-1 plane.
#pragma once
#include "common.cuh"

namespace feod {

constexpr int kFixThreads = 128;

// box extent of brick b along an axis (the last brick may be ragged)
template <int K, int B>
FEOD_DEV int box_len(int b, int ne) { return K * min(B, ne - b * B) + 1; }

// rank of (lx, ly, lz) on the surface of an LX x LY x LZ box
FEOD_DEV int srank(int lx, int ly, int lz, int LX, int LY, int LZ) {
  const int base = LX * LY, ring = 2 * LX + 2 * (LY - 2);
  if (lz == 0) return lx + LX * ly;
  if (lz == LZ - 1) return base + (LZ - 2) * ring + lx + LX * ly;
  const int r = base + (lz - 1) * ring;
  if (ly == 0) return r + lx;
  if (ly == LY - 1) return r + LX + lx;
  return r + 2 * LX + 2 * (ly - 1) + (lx == 0 ? 0 : 1);
}

// offset of brick-local (lx, ly, lz) in the shell buffer
template <int K, int BX, int BY, int BZ>
FEOD_DEV int64_t shell_off(const OpParams& P, int bx, int by, int bz, int lx, int ly, int lz) {
  const int LX = box_len<K, BX>(bx, P.nx), LY = box_len<K, BY>(by, P.ny), LZ = box_len<K, BZ>(bz, P.nz);
  return (bx + (int64_t)P.nbx * (by + (int64_t)P.nby * bz)) * P.shell_stride + srank(lx, ly, lz, LX, LY, LZ);
}

template <int K, int BX, int BY, int BZ, bool TWO>
__global__ void __launch_bounds__(kFixThreads) fixup_kernel(const OpParams P, int bxX, int bxY, int nX, int nY,
                                                            const double* __restrict__ shell0, double* __restrict__ out0,
                                                            const double* __restrict__ shell1, double* __restrict__ out1) {
  constexpr int PX = K * BX, PY = K * BY, PZ = K * BZ;
  int blk = blockIdx.x;
  int X, Y, Z;
  // contributors along the three axes: brick index and local index of each (up to 2);
  // the shared axis of the set and the row's fixed coordinate are CTA-uniform
  int bxa[2], lxa[2], bya[2], lya[2], bza[2], lza[2], nx, ny, nz;
  auto single = [](int g, int PS, int nb, int* b, int* l, int& n) {
    int bb = g / PS;
    if (bb >= nb) bb = nb - 1;
    b[0] = bb; l[0] = g - bb * PS; n = 1;
    if (l[0] == 0 && bb > 0) { b[1] = bb; l[1] = 0; b[0] = bb - 1; l[0] = PS; n = 2; }
  };
  if (blk < nY) {                            // set Y: row along X (X on an x-plane skipped)
    const int xb = blk % bxY, rest = blk / bxY;
    const int m = rest % (P.nby - 1) + 1;
    Z = rest / (P.nby - 1);
    Y = m * PY;
    X = xb * kFixThreads + threadIdx.x;
    if (X >= P.Mx || (X % PX == 0 && X > 0 && X < P.Mx - 1)) return;
    bya[0] = m - 1; lya[0] = PY; bya[1] = m; lya[1] = 0; ny = 2;
    single(Z, PZ, P.nbz, bza, lza, nz);
    bxa[0] = min(X / PX, P.nbx - 1); lxa[0] = X - bxa[0] * PX; nx = 1;
  } else if (blk < nY + nX) {                // set X: row along Y (edges and corners too)
    blk -= nY;
    const int xb = blk % bxX, rest = blk / bxX;
    const int m = rest % (P.nbx - 1) + 1;
    Z = rest / (P.nbx - 1);
    X = m * PX;
    Y = xb * kFixThreads + threadIdx.x;
    if (Y >= P.My) return;
    bxa[0] = m - 1; lxa[0] = PX; bxa[1] = m; lxa[1] = 0; nx = 2;
    single(Z, PZ, P.nbz, bza, lza, nz);
    single(Y, PY, P.nby, bya, lya, ny);
  } else {                                   // set Z: row along X (X / Y on a plane skipped)
    blk -= nY + nX;
    const int xb = blk % bxY, rest = blk / bxY;
    const int m = rest % (P.nbz - 1) + 1;
    Y = rest / (P.nbz - 1);
    if (Y % PY == 0 && Y > 0 && Y < P.My - 1) return;
    X = xb * kFixThreads + threadIdx.x;
    if (X >= P.Mx || (X % PX == 0 && X > 0 && X < P.Mx - 1)) return;
    Z = m * PZ;
    bza[0] = m - 1; lza[0] = PZ; bza[1] = m; lza[1] = 0; nz = 2;
    bya[0] = min(Y / PY, P.nby - 1); lya[0] = Y - bya[0] * PY; ny = 1;
    bxa[0] = min(X / PX, P.nbx - 1); lxa[0] = X - bxa[0] * PX; nx = 1;
  }
  // gather the (2, 4 or 8) contributions first, then sum in fixed order (z, y, x ascending)
  double v0[8], v1[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int cx = q & 1, cy = (q >> 1) & 1, cz = q >> 2;
    if (cx < nx && cy < ny && cz < nz) {
      const int64_t o = shell_off<K, BX, BY, BZ>(P, bxa[cx], bya[cy], bza[cz], lxa[cx], lya[cy], lza[cz]);
      v0[q] = __ldcs(shell0 + o);
      if constexpr (TWO) v1[q] = __ldcs(shell1 + o);
    }
  }
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int cx = q & 1, cy = (q >> 1) & 1, cz = q >> 2;
    if (cx < nx && cy < ny && cz < nz) {
      s0 += v0[q];
      if constexpr (TWO) s1 += v1[q];
    }
  }
  const bool dir = is_dirichlet(X, Y, Z, P.Mx, P.My, P.Mz, P.faces);
  const int64_t g = (int64_t)X + (int64_t)P.Mx * (Y + (int64_t)P.My * Z);
  out0[g] = dir ? 0.0 : s0;
  if constexpr (TWO) out1[g] = dir ? 0.0 : s1;
}

template <int K, int BX, int BY, int BZ>
cudaError_t launch_fixup_t(const OpParams& P, const double* shell0, double* out0, const double* shell1, double* out1,
                           cudaStream_t st) {
  const int bxY = (P.Mx + kFixThreads - 1) / kFixThreads;   // row blocks along X (sets Y, Z)
  const int bxX = (P.My + kFixThreads - 1) / kFixThreads;   // row blocks along Y (set X)
  const int64_t nY = (int64_t)bxY * (P.nby - 1) * P.Mz;
  const int64_t nX = (int64_t)bxX * (P.nbx - 1) * P.Mz;
  const int64_t nZ = (int64_t)bxY * (P.nbz - 1) * P.My;
  const int64_t blocks = nX + nY + nZ;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffff) return cudaErrorInvalidConfiguration;
  if (shell1)
    fixup_kernel<K, BX, BY, BZ, true><<<(unsigned)blocks, kFixThreads, 0, st>>>(P, bxX, bxY, (int)nX, (int)nY, shell0,
                                                                               out0, shell1, out1);
  else
    fixup_kernel<K, BX, BY, BZ, false><<<(unsigned)blocks, kFixThreads, 0, st>>>(P, bxX, bxY, (int)nX, (int)nY, shell0,
                                                                                out0, nullptr, nullptr);
  return cudaGetLastError();
}

}  // namespace feod
