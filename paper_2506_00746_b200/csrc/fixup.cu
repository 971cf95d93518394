// K5 — deterministic scatter fix-up (the G^T step for DOFs on faces shared by
// neighbouring bricks). Each shared DOF sums the shell
// values its 2, 4 or 8 bricks wrote, in a fixed order (z, y, x ascending), and
// applies P^T (0 on Dirichlet rows). No atomics: the result is bitwise
// reproducible run to run.
#include "common.cuh"
#include "kernels.h"

namespace feod {

struct AxisEntry { int b[2]; int loc[2]; int n; };

FEOD_DEV AxisEntry axis_entries(int Xg, int span, int nb) {
  AxisEntry r;
  int b = Xg / span;
  if (b >= nb) b = nb - 1;
  const int loc = Xg - b * span;
  if (loc == 0 && b > 0) {
    r.b[0] = b - 1; r.loc[0] = span; r.b[1] = b; r.loc[1] = 0; r.n = 2;
  } else {
    r.b[0] = b; r.loc[0] = loc; r.n = 1;
  }
  return r;
}

__global__ void fixup_kernel(const OpParams P, int K, int BX, int BY, int BZ, int64_t nX, int64_t nY,
                             int64_t nZ, const double* __restrict__ shell0, double* __restrict__ out0,
                             const double* __restrict__ shell1, double* __restrict__ out1) {
  const int PX = K * BX, PY = K * BY, PZ = K * BZ;
  const int64_t total = nX + nY + nZ;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int X, Y, Z;
    if (t < nX) {                       // x-planes: X = m PX, all Y, Z
      const int64_t s = t;
      const int m = (int)(s / ((int64_t)P.My * P.Mz)) + 1;
      const int64_t r = s % ((int64_t)P.My * P.Mz);
      X = m * PX; Y = (int)(r % P.My); Z = (int)(r / P.My);
    } else if (t < nX + nY) {           // y-planes, X not on an x-plane
      const int64_t s = t - nX;
      const int m = (int)(s / ((int64_t)P.Mx * P.Mz)) + 1;
      const int64_t r = s % ((int64_t)P.Mx * P.Mz);
      Y = m * PY; X = (int)(r % P.Mx); Z = (int)(r / P.Mx);
      if (X % PX == 0 && X > 0 && X < P.Mx - 1) continue;
    } else {                            // z-planes, X and Y on neither
      const int64_t s = t - nX - nY;
      const int m = (int)(s / ((int64_t)P.Mx * P.My)) + 1;
      const int64_t r = s % ((int64_t)P.Mx * P.My);
      Z = m * PZ; X = (int)(r % P.Mx); Y = (int)(r / P.Mx);
      if (X % PX == 0 && X > 0 && X < P.Mx - 1) continue;
      if (Y % PY == 0 && Y > 0 && Y < P.My - 1) continue;
    }
    const AxisEntry ax = axis_entries(X, PX, P.nbx), ay = axis_entries(Y, PY, P.nby), az = axis_entries(Z, PZ, P.nbz);
    double s0 = 0.0, s1 = 0.0;
    for (int cz = 0; cz < az.n; ++cz) {
      const int bz = az.b[cz];
      const int LZ = K * min(BZ, P.nz - bz * BZ) + 1;
      for (int cy = 0; cy < ay.n; ++cy) {
        const int by = ay.b[cy];
        const int LY = K * min(BY, P.ny - by * BY) + 1;
        for (int cx = 0; cx < ax.n; ++cx) {
          const int bx = ax.b[cx];
          const int LX = K * min(BX, P.nx - bx * BX) + 1;
          const int64_t brick = bx + (int64_t)P.nbx * (by + (int64_t)P.nby * bz);
          const int64_t o = brick * P.shell_stride + shell_rank(ax.loc[cx], ay.loc[cy], az.loc[cz], LX, LY, LZ);
          s0 += shell0[o];
          if (shell1) s1 += shell1[o];
        }
      }
    }
    const bool dir = is_dirichlet(X, Y, Z, P.Mx, P.My, P.Mz, P.faces);
    const int64_t g = (int64_t)X + (int64_t)P.Mx * (Y + (int64_t)P.My * Z);
    out0[g] = dir ? 0.0 : s0;
    if (out1) out1[g] = dir ? 0.0 : s1;
  }
}

cudaError_t launch_fixup(const OpParams& P, int K, int BX, int BY, int BZ, const double* shell0, double* out0,
                         const double* shell1, double* out1, cudaStream_t st) {
  const int64_t nX = (int64_t)(P.nbx - 1) * P.My * P.Mz;
  const int64_t nY = (int64_t)(P.nby - 1) * P.Mx * P.Mz;
  const int64_t nZ = (int64_t)(P.nbz - 1) * P.Mx * P.My;
  const int64_t total = nX + nY + nZ;
  if (total == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t want = (total + threads - 1) / threads;
  const int blocks = (int)(want < 148 * 32 ? want : 148 * 32);
  fixup_kernel<<<blocks, threads, 0, st>>>(P, K, BX, BY, BZ, nX, nY, nZ, shell0, out0, shell1, out1);
  return cudaGetLastError();
}

}  // namespace feod
