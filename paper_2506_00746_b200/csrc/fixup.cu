// K5 — deterministic scatter fix-up (the G^T step for DOFs on faces shared by
// neighbouring bricks). Each shared DOF sums the shell
// values its 2, 4 or 8 bricks wrote, in a fixed order (z, y, x ascending), and
// applies P^T (0 on Dirichlet rows). No atomics: the result is bitwise
// reproducible run to run.
//
// Work is laid out as rows along one axis so that consecutive threads touch
// consecutive shell entries and no per-thread integer division is needed:
//   set X: planes X = m PX (m = 1..nbx-1), rows along Y, one block row per (m, Z)
//   set Y: planes Y = m PY, rows along X (X on an x-plane skipped), per (m, Z)
//   set Z: planes Z = m PZ, rows along X (X or Y on a plane skipped), per (m, Y)
#include "common.cuh"
#include "kernels.h"

namespace feod {

constexpr int kFixThreads = 128;

struct AxisEntry { int b[2]; int loc[2]; int n; };

FEOD_DEV AxisEntry axis_entries(int Xg, int span, int nb) {
  AxisEntry r;
  int b = Xg / span;
  if (b >= nb) b = nb - 1;
  const int loc = Xg - b * span;
  if (loc == 0 && b > 0) {
    r.b[0] = b - 1; r.loc[0] = span; r.b[1] = b; r.loc[1] = 0; r.n = 2;
  } else {
    r.b[0] = b; r.loc[0] = loc; r.b[1] = b; r.loc[1] = loc; r.n = 1;
  }
  return r;
}

FEOD_DEV bool on_plane(int X, int span, int M) { return X > 0 && X < M - 1 && X % span == 0; }

__global__ void __launch_bounds__(kFixThreads) fixup_kernel(const OpParams P, int K, int BX, int BY, int BZ,
                                                            int bxX, int bxY, int nX, int nY,
                                                            const double* __restrict__ shell0, double* __restrict__ out0,
                                                            const double* __restrict__ shell1, double* __restrict__ out1) {
  const int PX = K * BX, PY = K * BY, PZ = K * BZ;
  int b = blockIdx.x;
  int X, Y, Z;
  if (b < nX) {                        // set X: row along Y
    const int xb = b % bxX, rest = b / bxX;
    const int m = rest % (P.nbx - 1) + 1, zz = rest / (P.nbx - 1);
    Y = xb * kFixThreads + threadIdx.x;
    if (Y >= P.My) return;
    X = m * PX; Z = zz;
  } else if (b < nX + nY) {            // set Y: row along X
    b -= nX;
    const int xb = b % bxY, rest = b / bxY;
    const int m = rest % (P.nby - 1) + 1, zz = rest / (P.nby - 1);
    X = xb * kFixThreads + threadIdx.x;
    if (X >= P.Mx || on_plane(X, PX, P.Mx)) return;
    Y = m * PY; Z = zz;
  } else {                             // set Z: row along X
    b -= nX + nY;
    const int xb = b % bxY, rest = b / bxY;
    const int m = rest % (P.nbz - 1) + 1, yy = rest / (P.nbz - 1);
    X = xb * kFixThreads + threadIdx.x;
    if (X >= P.Mx || on_plane(X, PX, P.Mx) || on_plane(yy, PY, P.My)) return;
    Y = yy; Z = m * PZ;
  }
  const AxisEntry ax = axis_entries(X, PX, P.nbx), ay = axis_entries(Y, PY, P.nby), az = axis_entries(Z, PZ, P.nbz);
  // gather all (<= 8) contributions first, then sum in fixed order
  double v0[8], v1[8];
#pragma unroll
  for (int cz = 0; cz < 2; ++cz)
#pragma unroll
    for (int cy = 0; cy < 2; ++cy)
#pragma unroll
      for (int cx = 0; cx < 2; ++cx) {
        const int q = cx + 2 * (cy + 2 * cz);
        v0[q] = 0.0;
        v1[q] = 0.0;
        if (cz < az.n && cy < ay.n && cx < ax.n) {
          const int bz = az.b[cz], by = ay.b[cy], bx = ax.b[cx];
          const int LZ = K * min(BZ, P.nz - bz * BZ) + 1;
          const int LY = K * min(BY, P.ny - by * BY) + 1;
          const int LX = K * min(BX, P.nx - bx * BX) + 1;
          const int64_t brick = bx + (int64_t)P.nbx * (by + (int64_t)P.nby * bz);
          const int64_t o = brick * P.shell_stride + shell_rank(ax.loc[cx], ay.loc[cy], az.loc[cz], LX, LY, LZ);
          v0[q] = shell0[o];
          if (shell1) v1[q] = shell1[o];
        }
      }
  double s0 = 0.0, s1 = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int cx = q & 1, cy = (q >> 1) & 1, cz = q >> 2;
    if (cz < az.n && cy < ay.n && cx < ax.n) {
      s0 += v0[q];
      s1 += v1[q];
    }
  }
  const bool dir = is_dirichlet(X, Y, Z, P.Mx, P.My, P.Mz, P.faces);
  const int64_t g = (int64_t)X + (int64_t)P.Mx * (Y + (int64_t)P.My * Z);
  out0[g] = dir ? 0.0 : s0;
  if (out1) out1[g] = dir ? 0.0 : s1;
}

cudaError_t launch_fixup(const OpParams& P, int K, int BX, int BY, int BZ, const double* shell0, double* out0,
                         const double* shell1, double* out1, cudaStream_t st) {
  const int bxX = (P.My + kFixThreads - 1) / kFixThreads;   // row blocks along Y (set X)
  const int bxY = (P.Mx + kFixThreads - 1) / kFixThreads;   // row blocks along X (sets Y, Z)
  const int64_t nX = (int64_t)bxX * (P.nbx - 1) * P.Mz;
  const int64_t nY = (int64_t)bxY * (P.nby - 1) * P.Mz;
  const int64_t nZ = (int64_t)bxY * (P.nbz - 1) * P.My;
  const int64_t blocks = nX + nY + nZ;
  if (blocks == 0) return cudaSuccess;
  if (blocks > 0x7fffffff) return cudaErrorInvalidConfiguration;
  fixup_kernel<<<(unsigned)blocks, kFixThreads, 0, st>>>(P, K, BX, BY, BZ, bxX, bxY, (int)nX, (int)nY, shell0, out0,
                                                         shell1, out1);
  return cudaGetLastError();
}

}  // namespace feod
