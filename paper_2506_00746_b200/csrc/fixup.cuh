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

// brick index along one axis of global DOF coordinate g, and whether g sits on
// an interior brick face (then the lower brick, local index P, contributes too)
struct Axis { int b, loc, n; };

template <int PS>
FEOD_DEV Axis axis_of(int g, int nb) {
  int b = g / PS;
  if (b >= nb) b = nb - 1;
  const int loc = g - b * PS;
  Axis a;
  a.b = b;
  a.loc = loc;
  a.n = (loc == 0 && b > 0) ? 2 : 1;
  return a;
}

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

template <int K, int BX, int BY, int BZ, bool TWO>
__global__ void __launch_bounds__(kFixThreads) fixup_kernel(const OpParams P, int bxX, int bxY, int nX, int nY,
                                                            const double* __restrict__ shell0, double* __restrict__ out0,
                                                            const double* __restrict__ shell1, double* __restrict__ out1) {
  constexpr int PX = K * BX, PY = K * BY, PZ = K * BZ;
  int blk = blockIdx.x;
  int X, Y, Z;
  if (blk < nY) {                            // set Y: row along X
    const int xb = blk % bxY, rest = blk / bxY;
    Y = (rest % (P.nby - 1) + 1) * PY;
    Z = rest / (P.nby - 1);
    X = xb * kFixThreads + threadIdx.x;
    if (X >= P.Mx || (X % PX == 0 && X > 0 && X < P.Mx - 1)) return;
  } else if (blk < nY + nX) {                // set X: row along Y
    blk -= nY;
    const int xb = blk % bxX, rest = blk / bxX;
    X = (rest % (P.nbx - 1) + 1) * PX;
    Z = rest / (P.nbx - 1);
    Y = xb * kFixThreads + threadIdx.x;
    if (Y >= P.My) return;
  } else {                                   // set Z: row along X
    blk -= nY + nX;
    const int xb = blk % bxY, rest = blk / bxY;
    Z = (rest % (P.nbz - 1) + 1) * PZ;
    Y = rest / (P.nbz - 1);
    if (Y % PY == 0 && Y > 0 && Y < P.My - 1) return;
    X = xb * kFixThreads + threadIdx.x;
    if (X >= P.Mx || (X % PX == 0 && X > 0 && X < P.Mx - 1)) return;
  }
  const Axis ax = axis_of<PX>(X, P.nbx), ay = axis_of<PY>(Y, P.nby), az = axis_of<PZ>(Z, P.nbz);
  // gather all contributions first (independent loads), then sum in fixed order
  double v0[8], v1[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int cx = q & 1, cy = (q >> 1) & 1, cz = q >> 2;
    v0[q] = 0.0;
    v1[q] = 0.0;
    if (cx < ax.n && cy < ay.n && cz < az.n) {
      // c = 0 is the lower brick when the axis is shared
      const int bxx = ax.b - (ax.n - 1 - cx), byy = ay.b - (ay.n - 1 - cy), bzz = az.b - (az.n - 1 - cz);
      const int LX = box_len<K, BX>(bxx, P.nx), LY = box_len<K, BY>(byy, P.ny), LZ = box_len<K, BZ>(bzz, P.nz);
      const int lx = (bxx < ax.b) ? LX - 1 : ax.loc, ly = (byy < ay.b) ? LY - 1 : ay.loc, lz = (bzz < az.b) ? LZ - 1 : az.loc;
      const int64_t o = (bxx + (int64_t)P.nbx * (byy + (int64_t)P.nby * bzz)) * P.shell_stride + srank(lx, ly, lz, LX, LY, LZ);
      v0[q] = __ldcs(shell0 + o);
      if constexpr (TWO) v1[q] = __ldcs(shell1 + o);
    }
  }
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int cx = q & 1, cy = (q >> 1) & 1, cz = q >> 2;
    if (cx < ax.n && cy < ay.n && cz < az.n) {
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
