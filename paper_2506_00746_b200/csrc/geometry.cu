// K1 — geometry setup (feod_create, untimed): the per-point symmetric metric
//   M_q = w_q detJ_q J_q^{-1} J_q^{-T} = w_q adj(J_q) adj(J_q)^T / detJ_q
// of the trilinear map of each hexahedron (the linear,
// solution-independent part of B that PAPER.md:25 keeps "excluded from the
// differentiation loop"). One thread per (element, point); components xx yy zz
// xy xz yz; per element [l][6][j][i] (component-major within each z-row l of points,
// x fastest), elements interleaved by OpParams::ptx (pt_base, common.cuh): with
// ptx = 1 (plane kernel) the ND*ND threads that own an element's points read one
// contiguous run per (row, component); with ptx = TX (column kernel) the threads of
// a tile row, one element each, read consecutive doubles.
#include "common.cuh"
#include "kernels.h"

namespace feod {

__global__ void geometry_kernel(const double* __restrict__ verts, const OpParams P, int nq, Tables T,
                                double* __restrict__ geom, int* __restrict__ bad) {
  const int nx = P.nx, ny = P.ny, nz = P.nz;
  const int nq3 = nq * nq * nq;
  const int64_t total = (int64_t)nx * ny * nz * nq3;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = idx / nq3;
    const int p = (int)(idx % nq3);
    const int i = p % nq, j = (p / nq) % nq, l = p / (nq * nq);
    const int ex = (int)(e % nx), ey = (int)((e / nx) % ny), ez = (int)(e / ((int64_t)nx * ny));
    const double xi = T.x[i], eta = T.x[j], zeta = T.x[l];
    double X[2][2][2][3];
    for (int dz = 0; dz < 2; ++dz)
      for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
          const int64_t v = (ex + dx) + (int64_t)(nx + 1) * ((ey + dy) + (int64_t)(ny + 1) * (ez + dz));
          for (int c = 0; c < 3; ++c) X[dz][dy][dx][c] = verts[3 * v + c];
        }
    const double Nx[2] = {1.0 - xi, xi}, Ny[2] = {1.0 - eta, eta}, Nz[2] = {1.0 - zeta, zeta};
    double J[3][3];   // J[c][d] = dx_c / dxi_d
    for (int c = 0; c < 3; ++c) {
      double d0 = 0.0, d1 = 0.0, d2 = 0.0;
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
          d0 += (X[b][a][1][c] - X[b][a][0][c]) * Ny[a] * Nz[b];
          d1 += (X[b][1][a][c] - X[b][0][a][c]) * Nx[a] * Nz[b];
          d2 += (X[1][b][a][c] - X[0][b][a][c]) * Nx[a] * Ny[b];
        }
      J[c][0] = d0;
      J[c][1] = d1;
      J[c][2] = d2;
    }
    // adjugate A = adj(J) = detJ J^{-1}:  A[d][c] = cofactor(J)[c][d]
    double A[3][3];
    A[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    A[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
    A[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
    A[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    A[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
    A[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
    A[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    A[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
    A[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    const double det = J[0][0] * A[0][0] + J[0][1] * A[1][0] + J[0][2] * A[2][0];
    if (!(det > 0.0)) atomicExch(bad, 1);
    const double s = T.w[i] * T.w[j] * T.w[l] / det;
    const int nq2 = nq * nq;
    const int64_t px = P.ptx;
    double* g = geom + pt_base(P, ex, ey, ez, 6 * nq3) + (l * 6 * nq2 + j * nq + i) * px;
    auto dot = [&](int r, int c) { return A[r][0] * A[c][0] + A[r][1] * A[c][1] + A[r][2] * A[c][2]; };
    g[0 * nq2 * px] = s * dot(0, 0);
    g[1 * nq2 * px] = s * dot(1, 1);
    g[2 * nq2 * px] = s * dot(2, 2);
    g[3 * nq2 * px] = s * dot(0, 1);
    g[4 * nq2 * px] = s * dot(0, 2);
    g[5 * nq2 * px] = s * dot(1, 2);
  }
}

cudaError_t launch_geometry(const double* verts, const OpParams& P, int nq, const Tables& T, double* geom, int* bad,
                            cudaStream_t st) {
  const int64_t total = (int64_t)P.nx * P.ny * P.nz * nq * nq * nq;
  const int threads = 256;
  const int64_t want = (total + threads - 1) / threads;
  const int blocks = (int)(want < 148 * 64 ? (want > 0 ? want : 1) : 148 * 64);
  geometry_kernel<<<blocks, threads, 0, st>>>(verts, P, nq, T, geom, bad);
  return cudaGetLastError();
}

}  // namespace feod
