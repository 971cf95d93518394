// K11 — Q6 operator kernel on the FP64 tensor cores (C4):
// F(u) and J(u)v (Eq. 1 / Eq. 2) for k = 6, q = 7 on affine meshes.
//
// One WARP per element, no shared memory, no block barriers. Each z-plane c (or point
// plane l) of a 7x7x7 element array is one 8x8 DMMA fragment (padding row/column 7 = 0):
// lane L holds entries (r = L/4, c = 2 (L%4) + t), t = 0, 1 ("D layout" of
// mma.sync.m8n8k4.f64). Then
//   - a contraction over the fragment's COLUMN index is two DMMAs with no data movement:
//     with the k-order permuted to (k-step s, k-lane q) <-> column 2q + s, the A operand of
//     k-step s is the lane's own register t = s (the 1D table is arranged to match);
//   - a contraction over the ROW index first transposes the fragment inside the warp
//     (8 64-bit shuffles per fragment);
//   - the z-contraction (across the 7 fragments) is plain register DFMA.
// B: x (columns, DMMA), y (transpose + DMMA), z (DFMA) to the points; gradients by
// collocation (D on the Gauss points): Uy (columns), Ux (transpose, DMMA, transpose back),
// Uz (DFMA). D: point_op (pointwise.cuh) on the 14 slots a lane holds per plane.
// B^T: Dz^T (DFMA), Dy^T (DMMA accumulating), Dx^T (transpose, DMMA, transpose back,
// add), then B^T z (DFMA), y (DMMA), x (transpose + DMMA) to the nodes.
// DMMA runs at 37.2 TF/s (profiles/r02_peaks_fp64.json); the 7 -> 8 padding leaves 77 %
// of its FMAs useful. The element's node results go to an element vector (E x 343); the
// assembly kernel sums each DOF's <= 8 contributions in a fixed order and applies P^T
// -- deterministic, no atomics.
#include "common.cuh"
#include "dual.cuh"
#include "kernels.h"
#include "physics.cuh"
#include "pointwise.cuh"

namespace feod {

namespace q6 {
constexpr int ND = 7, NQ = 7, K = 6, NN = 343;
constexpr int WARPS = 4;

struct Frag { double v[2]; };   // lane's two entries of an 8x8 fragment (D layout)

FEOD_DEV void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// out[r][n] (+)= sum_c M[r][c] W[c][n]: the lane's table operand w[s] = W[2q + s][L/4]
FEOD_DEV Frag contract_cols(const Frag& m, const double w[2], Frag acc) {
  dmma(acc.v[0], acc.v[1], m.v[0], w[0]);
  dmma(acc.v[0], acc.v[1], m.v[1], w[1]);
  return acc;
}

// M^T in D layout: entry (r', c') = M[c'][r'] lives in lane 4 c' + r'/2, register r' % 2
FEOD_DEV Frag transpose(const Frag& m, int lane) {
  Frag o;
  const int r = lane >> 2, q = lane & 3;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int src = 4 * (2 * q + t) + (r >> 1);
    const double a = __shfl_sync(0xffffffffu, m.v[0], src);
    const double b = __shfl_sync(0xffffffffu, m.v[1], src);
    o.v[t] = (r & 1) ? b : a;
  }
  return o;
}
}  // namespace q6

#ifndef FEOD_Q6_MINB_JVP
#define FEOD_Q6_MINB_JVP 3
#endif
#ifndef FEOD_Q6_MINB_RES
#define FEOD_Q6_MINB_RES 3
#endif
template <int MODE, int MODEL>
__global__ void __launch_bounds__(32 * q6::WARPS, MODE == MODE_RES ? FEOD_Q6_MINB_RES : FEOD_Q6_MINB_JVP)
q6tc_kernel(const OpParams P, const Tables T, const double* __restrict__ in0, const double* __restrict__ in1,
            double* __restrict__ ev) {
  using namespace q6;
  constexpr int NIN = MODE == MODE_RES ? 1 : 2;
  // two-field modes: the first field's four point channels are parked in shared memory
  // (lane-interleaved, conflict-free), so only one field's 56 doubles are live in registers
  extern __shared__ double q6sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* park = q6sm + (size_t)wid * (4 * 7 * 2 * 32);   // [channel][plane][t][lane]
  auto pk = [&](int ch, int l, int t) -> double& { return park[((ch * 7 + l) * 2 + t) * 32 + lane]; };
  const int r = lane >> 2, q = lane & 3;                  // fragment row, column pair (2q, 2q+1)
  const int64_t E = (int64_t)P.nx * P.ny * P.nz;
  // table operands (k-order permuted: k-step s <-> column 2q + s), zero outside 7x7
  auto tab = [&](int kind, int s) {   // 0: B[n][c] 1: D[n][c] 2: B[c][n] 3: D[c][n]
    const int c = 2 * q + s, n = r;
    if (c >= 7 || n >= 7) return 0.0;
    return kind == 0 ? T.B[n][c] : kind == 1 ? T.D[n][c] : kind == 2 ? T.B[c][n] : T.D[c][n];
  };
  const double WB[2] = {tab(0, 0), tab(0, 1)}, WD[2] = {tab(1, 0), tab(1, 1)};
  const double WBt[2] = {tab(2, 0), tab(2, 1)}, WDt[2] = {tab(3, 0), tab(3, 1)};
  const bool rowv = r < 7;
  const bool colv[2] = {2 * q < 7, 2 * q + 1 < 7};
  const Frag zero = {{0.0, 0.0}};

  // B and the collocated gradients of one field: nodes z = c in fragment c (rows y,
  // columns x) -> U, Ux, Uy, Uz at the points, plane l, fragment [i][j]
  auto forward = [&](const double* __restrict__ src, int ex, int ey, int ez, Frag* U, Frag* Ux, Frag* Uy, Frag* Uz) {
    Frag X[7];
#pragma unroll
    for (int c = 0; c < 7; ++c) {
      const int64_t row = (int64_t)(K * ex) + (int64_t)P.Mx * ((K * ey + r) + (int64_t)P.My * (K * ez + c));
#pragma unroll
      for (int t = 0; t < 2; ++t) X[c].v[t] = (rowv && colv[t]) ? __ldg(src + row + 2 * q + t) : 0.0;
    }
    Frag Ep[7];   // after x and y: [i][j] per node plane c
#pragma unroll
    for (int c = 0; c < 7; ++c) {
      const Frag t1 = contract_cols(X[c], WB, zero);          // [y][i]
      Ep[c] = contract_cols(transpose(t1, lane), WB, zero);   // [i][j]
    }
#pragma unroll
    for (int l = 0; l < 7; ++l)   // z: points plane l, [i][j]
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        double s = T.B[l][0] * Ep[0].v[t];
#pragma unroll
        for (int c = 1; c < 7; ++c) s = fma(T.B[l][c], Ep[c].v[t], s);
        U[l].v[t] = s;
      }
#pragma unroll
    for (int l = 0; l < 7; ++l) {
      Uy[l] = contract_cols(U[l], WD, zero);                                  // d/dy: [i][j']
      Ux[l] = transpose(contract_cols(transpose(U[l], lane), WD, zero), lane);   // d/dx: [i'][j]
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        double s = T.D[l][0] * U[0].v[t];
#pragma unroll
        for (int m = 1; m < 7; ++m) s = fma(T.D[l][m], U[m].v[t], s);
        Uz[l].v[t] = s;
      }
    }
  };

  for (int64_t e = (int64_t)blockIdx.x * WARPS + wid; e < E; e += (int64_t)gridDim.x * WARPS) {
    const int ex = (int)(e % P.nx), ey = (int)((e / P.nx) % P.ny), ez = (int)(e / ((int64_t)P.nx * P.ny));
    Frag U[7], Ux[7], Uy[7], Uz[7];   // the last field's channels (the fluxes overwrite Ux, Uy, Uz)
    if constexpr (NIN == 2) {
      forward(in0, ex, ey, ez, U, Ux, Uy, Uz);
#pragma unroll
      for (int l = 0; l < 7; ++l)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          pk(0, l, t) = U[l].v[t];
          pk(1, l, t) = Ux[l].v[t];
          pk(2, l, t) = Uy[l].v[t];
          pk(3, l, t) = Uz[l].v[t];
        }
      __syncwarp();
      forward(in1, ex, ey, ez, U, Ux, Uy, Uz);
    } else {
      forward(in0, ex, ey, ez, U, Ux, Uy, Uz);
    }
    // ---- D at the points (slot (i = r, j = 2q + t) of plane l); fluxes over Ux / Uy / Uz
    const double rho_e = (MODEL == HEAT) ? __ldg(P.rho + e) : 1.0;
    Frag V[7];   // value channel (residual: the load term)
#pragma unroll
    for (int l = 0; l < 7; ++l)
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int j = 2 * q + t;
        double F0[4] = {0.0, 0.0, 0.0, 0.0}, F1[4];
        if (rowv && colv[t]) {
          const double wq = T.w[r] * T.w[j] * T.w[l];
          const Metric M = {wq * P.cx, wq * P.cy, wq * P.cz, 0.0, 0.0, 0.0};
          const double W = wq * P.vol;
          double Ul[NIN], Uxl[NIN], Uyl[NIN], Uzl[NIN];
          if constexpr (NIN == 2) {
            Ul[0] = pk(0, l, t); Uxl[0] = pk(1, l, t); Uyl[0] = pk(2, l, t); Uzl[0] = pk(3, l, t);
          }
          Ul[NIN - 1] = U[l].v[t];
          Uxl[NIN - 1] = Ux[l].v[t];
          Uyl[NIN - 1] = Uy[l].v[t];
          Uzl[NIN - 1] = Uz[l].v[t];
          double gpart = 0.0, lv[9];
          point_op<MODE, MODEL, true>(Ul, Uxl, Uyl, Uzl, M, W, rho_e, P, nullptr, F0, F1, gpart, lv);
        }
        Ux[l].v[t] = F0[0];
        Uy[l].v[t] = F0[1];
        Uz[l].v[t] = F0[2];
        V[l].v[t] = value_channel(MODE, 0) ? F0[3] : 0.0;
      }
    if constexpr (NIN == 2) __syncwarp();   // park reads done before the next element's writes
    // ---- B^T: R = Dx^T Fx + Dy^T Fy + Dz^T Fz + V at the points, then z, y, x to the nodes
    Frag R[7];
#pragma unroll
    for (int m = 0; m < 7; ++m)
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        double s = V[m].v[t];
#pragma unroll
        for (int l = 0; l < 7; ++l) s = fma(T.D[l][m], Uz[l].v[t], s);
        R[m].v[t] = s;
      }
#pragma unroll
    for (int l = 0; l < 7; ++l) {
      const Frag rx = transpose(contract_cols(transpose(Ux[l], lane), WDt, zero), lane);   // Dx^T Fx
      Frag acc = R[l];
      acc.v[0] += rx.v[0];
      acc.v[1] += rx.v[1];
      R[l] = contract_cols(Uy[l], WDt, acc);   // + Dy^T Fy
    }
    double* out = ev + e * NN;
#pragma unroll
    for (int c = 0; c < 7; ++c) {
      Frag S;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        double s = T.B[0][c] * R[0].v[t];
#pragma unroll
        for (int l = 1; l < 7; ++l) s = fma(T.B[l][c], R[l].v[t], s);
        S.v[t] = s;
      }
      const Frag ty = contract_cols(S, WBt, zero);                      // [i][b]
      const Frag nd = contract_cols(transpose(ty, lane), WBt, zero);    // [b][a]
      if (rowv) {
#pragma unroll
        for (int t = 0; t < 2; ++t)
          if (colv[t]) out[c * 49 + r * 7 + 2 * q + t] = nd.v[t];
      }
    }
  }
}

// G^T + P^T from the element vector: each DOF sums its <= 8 element contributions in
// ascending element order (z, y, x), Dirichlet rows 0 -- deterministic. One CTA row per
// DOF row (Y, Z): the y / z contributors are row-uniform, the x ones come from K = 6
// (compile-time division); consecutive threads read consecutive element-vector entries.
__global__ void __launch_bounds__(256) evec_assemble_kernel(const OpParams P, const double* __restrict__ ev,
                                                             double* __restrict__ out) {
  constexpr int K = q6::K, ND = q6::ND;
  auto axis = [&](int G, int ne, int* c, int* a) {
    int nc = 0;
    const int hi = min(G / K, ne - 1);
    if (G - K * hi == 0 && hi > 0) { c[nc] = hi - 1; a[nc] = K; ++nc; }
    c[nc] = hi; a[nc] = G - K * hi; ++nc;
    return nc;
  };
  const int rows = P.My * P.Mz;
  // a warp per DOF row (Y, Z): its y / z contributors are row-uniform, the x ones come
  // from K = 6 (compile-time division); the lanes read consecutive element-vector entries
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int YZ = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); YZ < rows; YZ += warps) {
    const int Y = YZ % P.My, Z = YZ / P.My;
    int cy[2], ay[2], cz[2], az[2];
    const int nyc = axis(Y, P.ny, cy, ay), nzc = axis(Z, P.nz, cz, az);
    const bool dyz = ((P.faces & 4u) && Y == 0) || ((P.faces & 8u) && Y == P.My - 1) ||
                     ((P.faces & 16u) && Z == 0) || ((P.faces & 32u) && Z == P.Mz - 1);
    const int64_t row = (int64_t)P.Mx * (Y + (int64_t)P.My * Z);
    for (int X = threadIdx.x & 31; X < P.Mx; X += 32) {
      int cx[2], ax[2];
      const int nxc = axis(X, P.nx, cx, ax);
      double s = 0.0;
      for (int kz = 0; kz < nzc; ++kz)
        for (int ky = 0; ky < nyc; ++ky) {
          const int64_t e0 = (int64_t)P.nx * (cy[ky] + (int64_t)P.ny * cz[kz]);
          const int off = az[kz] * ND * ND + ay[ky] * ND;
          for (int kx = 0; kx < nxc; ++kx) s += __ldcs(ev + (e0 + cx[kx]) * q6::NN + off + ax[kx]);
        }
      const bool dir = dyz || ((P.faces & 1u) && X == 0) || ((P.faces & 2u) && X == P.Mx - 1);
      out[row + X] = dir ? 0.0 : s;
    }
  }
}

template <int MODE, int MODEL>
static cudaError_t q6tc_launch(const OpParams& P, const Tables& T, const double* in0, const double* in1, double* ev,
                               double* out, cudaStream_t st) {
  constexpr size_t smem = MODE == MODE_RES ? 0 : sizeof(double) * q6::WARPS * 4 * 7 * 2 * 32;
  cudaError_t e = cudaFuncSetAttribute(q6tc_kernel<MODE, MODEL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int slots = 0;
  if ((e = persistent_slots((const void*)q6tc_kernel<MODE, MODEL>, 32 * q6::WARPS, smem, &slots)) != cudaSuccess) return e;
  const int64_t E = (int64_t)P.nx * P.ny * P.nz;
  const int64_t want = (E + q6::WARPS - 1) / q6::WARPS;
  q6tc_kernel<MODE, MODEL><<<(unsigned)(want < slots ? want : slots), 32 * q6::WARPS, smem, st>>>(P, T, in0, in1, ev);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int rows = P.My * P.Mz, wpb = 8;
  const int blocks = (rows + wpb - 1) / wpb;
  evec_assemble_kernel<<<blocks < 148 * 8 ? blocks : 148 * 8, 32 * wpb, 0, st>>>(P, ev, out);
  return cudaGetLastError();
}

// C4's path: Q6, affine, residual or JVP (other modes / perturbed meshes use plane_kernel)
cudaError_t q6tc_run(int mode, int model, const OpParams& P, const Tables& T, const double* in0, const double* in1,
                     double* ev, double* out, cudaStream_t st) {
  if (mode == MODE_RES) {
    switch (model) {
      case PLAPLACE: return q6tc_launch<MODE_RES, PLAPLACE>(P, T, in0, in1, ev, out, st);
      case NLDIFF: return q6tc_launch<MODE_RES, NLDIFF>(P, T, in0, in1, ev, out, st);
      case HEAT: return q6tc_launch<MODE_RES, HEAT>(P, T, in0, in1, ev, out, st);
    }
  } else if (mode == MODE_JVP) {
    switch (model) {
      case PLAPLACE: return q6tc_launch<MODE_JVP, PLAPLACE>(P, T, in0, in1, ev, out, st);
      case NLDIFF: return q6tc_launch<MODE_JVP, NLDIFF>(P, T, in0, in1, ev, out, st);
      case HEAT: return q6tc_launch<MODE_JVP, HEAT>(P, T, in0, in1, ev, out, st);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace feod
