// K8 — diagonal of the stored linearisation's Jacobian (SURVEY §8(f) NEXT-3,
// Jacobi preconditioning "from the PA diagonal"). With the stored per-point
// linearisation A = dFh/dgh (symmetric) and b = dFh/du (feod_linearize), the
// element Jacobian is K_e[i][j] = sum_q grad phi_i . (A grad phi_j + b phi_j)
// (Eq. 2 / Eq. 3), so its diagonal at the tensor-product node (a, b, c) is
//   sum_q [ A_xx G_a^2 B_b^2 B_c^2 + A_yy B_a^2 G_b^2 B_c^2 + A_zz B_a^2 B_b^2 G_c^2
//         + 2 A_xy (GB)_a (BG)_b B_c^2 + 2 A_xz (GB)_a B_b^2 (BG)_c + 2 A_yz B_a^2 (GB)_b (GB)_c
//         + b_x (GB)_a B_b^2 B_c^2 + b_y B_a^2 (GB)_b B_c^2 + b_z B_a^2 B_b^2 (GB)_c ]
// with the 1D tables evaluated at the Gauss points (B = l_a(x_i), G = l_a'(x_i)):
// every term is a sum-factorised contraction with squared / mixed 1D tables.
// Persistent CTAs per colour (the next element's values prefetched in registers);
// G^T without atomics by 8 element colours (parity of
// ex, ey, ez): elements of one colour share no DOF, the colours run in a fixed
// order, so the assembled diagonal is bitwise reproducible. Dirichlet rows get
// 1 (J's Dirichlet rows are zero; the preconditioner is the identity there).
#include "common.cuh"
#include "kernels.h"
#include "evec.cuh"

#ifndef FEOD_DIAG_Q3_WARP
#define FEOD_DIAG_Q3_WARP 1   // Q3: the half-warp-per-element diagonal (0: thread per node plane)
#endif

namespace feod {

constexpr int kDiagThreads = 128;

template <int ND, int NT>
__global__ void __launch_bounds__(kDiagThreads) diag_color_kernel(const OpParams P, const Tables T, int color,
                                                                  double* __restrict__ diag) {
  constexpr int NQ = ND, NQ2 = NQ * NQ, NQ3 = NQ2 * NQ, NL = NT;
  // per-term tables along x, y, z: 0 = B^2, 1 = G^2, 2 = G B
  constexpr int TX[9] = {1, 0, 0, 2, 2, 0, 2, 0, 0};
  constexpr int TY[9] = {0, 1, 0, 2, 0, 2, 0, 2, 0};
  constexpr int TZ[9] = {0, 0, 1, 0, 2, 2, 0, 0, 2};
  constexpr double WT[9] = {1, 1, 1, 2, 2, 2, 1, 1, 1};
  extern __shared__ double dsm[];
  double(*tab)[NQ][ND] = reinterpret_cast<double(*)[NQ][ND]>(dsm);                       // [3][NQ][ND]
  double(*S0)[NQ3] = reinterpret_cast<double(*)[NQ3]>(dsm + 3 * NQ * ND);                 // A terms [l][j][i]
  double(*S1)[NQ2 * ND] = reinterpret_cast<double(*)[NQ2 * ND]>(dsm + 3 * NQ * ND + NT * NQ3);   // [j][i][c]
  double(*S2)[NQ * ND * ND] = reinterpret_cast<double(*)[NQ * ND * ND]>(dsm + 3 * NQ * ND);  // [i][b][c], over S0
  const int tid = threadIdx.x;
  const int hx = (P.nx + 1 - (color & 1)) / 2, hy = (P.ny + 1 - ((color >> 1) & 1)) / 2;
  const int hz = (P.nz + 1 - ((color >> 2) & 1)) / 2;
  const int ne = hx * hy * hz;
  auto elem = [&](int e, int& ex, int& ey, int& ez) {
    ex = 2 * (e % hx) + (color & 1);
    ey = 2 * ((e / hx) % hy) + ((color >> 1) & 1);
    ez = 2 * (e / (hx * hy)) + ((color >> 2) & 1);
    return (int64_t)ex + (int64_t)P.nx * (ey + (int64_t)P.ny * ez);
  };
  for (int t = tid; t < NQ * ND; t += kDiagThreads) {
    const int i = t / ND, a = t % ND;
    const double b = T.B[i][a], g = T.G[i][a];
    tab[0][i][a] = b * b;
    tab[1][i][a] = g * g;
    tab[2][i][a] = g * b;
  }
  // persistent over the colour's elements; the next element's linearisation is loaded
  // into registers while the current one is contracted
  constexpr int PF = (NT * NQ3 + kDiagThreads - 1) / kDiagThreads;
  double pf[PF];
  auto load = [&](int e) {
    int ex, ey, ez;
    elem(e, ex, ey, ez);
    const int64_t px = P.ptx;   // interleaved per-point layout (pt_base, common.cuh)
    const double* lin = P.lin + pt_base(P, ex, ey, ez, NL * NQ3);
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      const int t = tid + k * kDiagThreads;
      if (t < NT * NQ3) {
        const int term = t / NQ3, r = t % NQ3, l = r / NQ2, ji = r % NQ2;   // r = (l, j, i), i fastest
        pf[k] = __ldcs(lin + (l * NL * NQ2 + term * NQ2 + ji) * px);
      }
    }
  };
  int e = blockIdx.x;
  if (e < ne) load(e);
  for (; e < ne; e += gridDim.x) {
  int ex, ey, ez;
  elem(e, ex, ey, ez);
#pragma unroll
  for (int k = 0; k < PF; ++k) {
    const int t = tid + k * kDiagThreads;
    if (t < NT * NQ3) S0[t / NQ3][t % NQ3] = pf[k];
  }
  if (e + (int)gridDim.x < ne) load(e + gridDim.x);
  __syncthreads();
  // contract l: S1[t][j][i][c] = sum_l S0[t][l][j][i] Z_t[l][c]
  for (int t = tid; t < NT * NQ2 * ND; t += kDiagThreads) {
    const int term = t / (NQ2 * ND), r = t % (NQ2 * ND), ji = r / ND, c = r % ND;
    const int tz = TZ[term];
    double s = 0.0;
#pragma unroll
    for (int l = 0; l < NQ; ++l) s = fma(S0[term][l * NQ2 + ji], tab[tz][l][c], s);
    S1[term][r] = s;
  }
  __syncthreads();
  // contract j: S2[t][i][b][c] = sum_j S1[t][j][i][c] Y_t[j][b]
  for (int t = tid; t < NT * NQ * ND * ND; t += kDiagThreads) {
    const int term = t / (NQ * ND * ND), r = t % (NQ * ND * ND);
    const int i = r / (ND * ND), b = (r / ND) % ND, c = r % ND;
    const int ty = TY[term];
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < NQ; ++j) s = fma(S1[term][(j * NQ + i) * ND + c], tab[ty][j][b], s);
    S2[term][r] = s;
  }
  __syncthreads();
  // contract i and sum the terms in a fixed order; add into the diagonal (colour-exclusive)
  const int Mx = P.Mx, My = P.My;
  for (int t = tid; t < ND * ND * ND; t += kDiagThreads) {
    const int a = t % ND, b = (t / ND) % ND, c = t / (ND * ND);
    double s = 0.0;
#pragma unroll
    for (int term = 0; term < NT; ++term) {
      const int tx = TX[term];
      double st = 0.0;
#pragma unroll
      for (int i = 0; i < NQ; ++i) st = fma(S2[term][(i * ND + b) * ND + c], tab[tx][i][a], st);
      s = fma(WT[term], st, s);
    }
    const int64_t g = (int64_t)((ND - 1) * ex + a) + (int64_t)Mx * (((ND - 1) * ey + b) + (int64_t)My * ((ND - 1) * ez + c));
    diag[g] += s;
  }
  __syncthreads();   // S0 / S1 / S2 reused by the next element
  }   // elements
}

// Q1 / Q2: one thread per element of the colour, the element's diagonal sum-factorised in
// registers (the same 9 terms), then added into the colour-exclusive DOFs -- no shared
// memory and no block barriers (the per-element CTA version above is latency-bound at
// low order: C5 2.3 ms).
template <int ND, int NT>
__global__ void __launch_bounds__(128) diag_elem_kernel(const OpParams P, const Tables T, int color,
                                                        double* __restrict__ diag, double* __restrict__ ev) {
  constexpr int NQ = ND, NQ2 = NQ * NQ, NQ3 = NQ2 * NQ, NL = NT;
  constexpr int TX[9] = {1, 0, 0, 2, 2, 0, 2, 0, 0};
  constexpr int TY[9] = {0, 1, 0, 2, 0, 2, 0, 2, 0};
  constexpr int TZ[9] = {0, 0, 1, 0, 2, 2, 0, 0, 2};
  constexpr double WT[9] = {1, 1, 1, 2, 2, 2, 1, 1, 1};
  // ev != nullptr: every element in natural order (consecutive threads = consecutive x
  // elements: the interleaved per-point stream is read coalesced), the element diagonal
  // written to the discontinuous L-vector for evec.cuh's assembly; else colour `color`
  // (stride-2 elements) with read-modify-write into diag
  const bool all = ev != nullptr;
  const int hx = all ? P.nx : (P.nx + 1 - (color & 1)) / 2, hy = all ? P.ny : (P.ny + 1 - ((color >> 1) & 1)) / 2;
  const int hz = all ? P.nz : (P.nz + 1 - ((color >> 2) & 1)) / 2;
  const int64_t ne = (int64_t)hx * hy * hz;
  const int sx = all ? 1 : 2, ox = all ? 0 : (color & 1), oy = all ? 0 : ((color >> 1) & 1), oz = all ? 0 : ((color >> 2) & 1);
  // 1D factor tables: 0 = B^2, 1 = G^2, 2 = G B
  auto tab = [&](int k, int i, int a) {
    const double b = T.B[i][a], g = T.G[i][a];
    return k == 0 ? b * b : k == 1 ? g * g : g * b;
  };
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    const int ex = sx * (int)(e % hx) + ox;
    const int ey = sx * (int)((e / hx) % hy) + oy;
    const int ez = sx * (int)(e / ((int64_t)hx * hy)) + oz;
    const int64_t px = P.ptx;
    const double* lin = P.lin + pt_base(P, ex, ey, ez, NL * NQ3);
    double dg[ND * ND * ND];
#pragma unroll
    for (int n = 0; n < ND * ND * ND; ++n) dg[n] = 0.0;
#pragma unroll
    for (int term = 0; term < NT; ++term) {
      double S0[NQ3];
#pragma unroll
      for (int q = 0; q < NQ3; ++q) S0[q] = __ldcs(lin + ((q / NQ2) * NL * NQ2 + term * NQ2 + q % NQ2) * px);
      double S1[ND][NQ2];   // [c][j i]
#pragma unroll
      for (int c = 0; c < ND; ++c)
#pragma unroll
        for (int ji = 0; ji < NQ2; ++ji) {
          double s = 0.0;
#pragma unroll
          for (int l = 0; l < NQ; ++l) s = fma(S0[l * NQ2 + ji], tab(TZ[term], l, c), s);
          S1[c][ji] = s;
        }
      double S2[ND][ND][NQ];   // [c][b][i]
#pragma unroll
      for (int c = 0; c < ND; ++c)
#pragma unroll
        for (int b = 0; b < ND; ++b)
#pragma unroll
          for (int i = 0; i < NQ; ++i) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < NQ; ++j) s = fma(S1[c][j * NQ + i], tab(TY[term], j, b), s);
            S2[c][b][i] = s;
          }
#pragma unroll
      for (int c = 0; c < ND; ++c)
#pragma unroll
        for (int b = 0; b < ND; ++b)
#pragma unroll
          for (int a = 0; a < ND; ++a) {
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < NQ; ++i) s = fma(S2[c][b][i], tab(TX[term], i, a), s);
            dg[a + ND * (b + ND * c)] = fma(WT[term], s, dg[a + ND * (b + ND * c)]);
          }
    }
    const int K = ND - 1;
    if (all) {
      const int64_t LXd = ND * (int64_t)P.nx, LYd = ND * (int64_t)P.ny;
      double* out = ev + ((int64_t)(ND * ez) * LYd + ND * ey) * LXd + ND * ex;
#pragma unroll
      for (int c = 0; c < ND; ++c)
#pragma unroll
        for (int b = 0; b < ND; ++b)
#pragma unroll
          for (int a = 0; a < ND; ++a) out[((int64_t)c * LYd + b) * LXd + a] = dg[a + ND * (b + ND * c)];
    } else {
#pragma unroll
      for (int c = 0; c < ND; ++c)
#pragma unroll
        for (int b = 0; b < ND; ++b)
#pragma unroll
          for (int a = 0; a < ND; ++a) {
            const int64_t g = (int64_t)(K * ex + a) + (int64_t)P.Mx * ((K * ey + b) + (int64_t)P.My * (K * ez + c));
            diag[g] += dg[a + ND * (b + ND * c)];
          }
    }
  }
}

template <int ND, int NT>
static cudaError_t diag_elem_t(const OpParams& P, const Tables& T, double* ev, double* diag, cudaStream_t st) {
  if (ev) {   // one launch over all elements + the deterministic assembly (Dirichlet rows 1)
    const int64_t ne = (int64_t)P.nx * P.ny * P.nz;
    const int64_t b = (ne + 127) / 128;
    diag_elem_kernel<ND, NT><<<(unsigned)(b < 148 * 32 ? b : 148 * 32), 128, 0, st>>>(P, T, 0, diag, ev);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return evec_assemble<ND - 1>(P, ev, diag, nullptr, nullptr, 1.0, st);
  }
  for (int color = 0; color < 8; ++color) {
    const int hx = (P.nx + 1 - (color & 1)) / 2, hy = (P.ny + 1 - ((color >> 1) & 1)) / 2,
              hz = (P.nz + 1 - ((color >> 2) & 1)) / 2;
    const int64_t ne = (int64_t)hx * hy * hz;
    if (ne == 0) continue;
    const int64_t b = (ne + 127) / 128;
    diag_elem_kernel<ND, NT><<<(unsigned)(b < 148 * 32 ? b : 148 * 32), 128, 0, st>>>(P, T, color, diag, nullptr);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

__global__ void diag_dirichlet_kernel(const OpParams P, double* __restrict__ diag) {
  const int64_t n = (int64_t)P.Mx * P.My * P.Mz;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int X = (int)(i % P.Mx);
    const int64_t yz = i / P.Mx;
    const int Y = (int)(yz % P.My), Z = (int)(yz / P.My);
    if (is_dirichlet(X, Y, Z, P.Mx, P.My, P.Mz, P.faces)) diag[i] = 1.0;
  }
}

template <int ND, int NT>
static cudaError_t diag_nd_t(const OpParams& P, const Tables& T, double* diag, cudaStream_t st) {
  constexpr size_t smem = sizeof(double) * (3 * ND * ND + NT * ND * ND * ND + NT * ND * ND * ND);
  cudaError_t e0 = cudaFuncSetAttribute(diag_color_kernel<ND, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem);
  if (e0 != cudaSuccess) return e0;
  int slots = 0;
  if ((e0 = persistent_slots((const void*)diag_color_kernel<ND, NT>, kDiagThreads, smem, &slots)) != cudaSuccess)
    return e0;
  for (int color = 0; color < 8; ++color) {
    const int hx = (P.nx + 1 - (color & 1)) / 2, hy = (P.ny + 1 - ((color >> 1) & 1)) / 2,
              hz = (P.nz + 1 - ((color >> 2) & 1)) / 2;
    const int64_t ne = (int64_t)hx * hy * hz;
    if (ne == 0) continue;
    const int64_t grid = ne < slots ? ne : slots;
    diag_color_kernel<ND, NT><<<(unsigned)grid, kDiagThreads, smem, st>>>(P, T, color, diag);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  const int64_t n = (int64_t)P.Mx * P.My * P.Mz;
  const int64_t b = (n + 255) / 256;
  diag_dirichlet_kernel<<<(unsigned)(b < kRedBlocks ? b : kRedBlocks), 256, 0, st>>>(P, diag);
  return cudaGetLastError();
}


// Q3, Q4 (plane-kernel orders): one thread per (element, node plane c). Its element's
// stored linearisation is read straight from HBM (the ND threads of an element are
// adjacent lanes: one broadcast load), 16-byte loads along i where ND is even:
//   Z[j][i] = sum_l w_t TZ_t[l][c] A_t(i, j, l)          (z first, TZ from shared memory)
//   dg[b][a] += sum_i TX_t[i][a] sum_j TY_t[j][b] Z[j][i]   (the products in Tables)
// The element diagonals go to the discontinuous L-vector and through evec.cuh's
// deterministic assembly (Dirichlet rows 1) -- one launch per call pair instead of the
// colour sweep's eight.
template <int ND, int NL>
__global__ void __launch_bounds__(128) diag_pt_kernel(const OpParams P, const Tables T, double* __restrict__ ev) {
  constexpr int NQ = ND, NQ2 = NQ * NQ, NQ3 = NQ2 * NQ;
  constexpr int TX[9] = {1, 0, 0, 2, 2, 0, 2, 0, 0};
  constexpr int TY[9] = {0, 1, 0, 2, 0, 2, 0, 2, 0};
  constexpr int TZ[9] = {0, 0, 1, 0, 2, 2, 0, 0, 2};
  constexpr double WT[9] = {1, 1, 1, 2, 2, 2, 1, 1, 1};
  __shared__ double zt[3][NQ][ND];
  for (int k = threadIdx.x; k < 3 * NQ * ND; k += blockDim.x) {
    const int kind = k / (NQ * ND), l = (k / ND) % NQ, c = k % ND;
    zt[kind][l][c] = kind == 0 ? T.B2[l][c] : kind == 1 ? T.G2[l][c] : T.GB[l][c];
  }
  __syncthreads();
  auto tab = [&](int kind, int i, int a) { return kind == 0 ? T.B2[i][a] : kind == 1 ? T.G2[i][a] : T.GB[i][a]; };
  const int64_t E = (int64_t)P.nx * P.ny * P.nz;
  const int64_t LXd = ND * (int64_t)P.nx, LYd = ND * (int64_t)P.ny;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < E * ND; it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = it / ND;
    const int c = (int)(it - e * ND);
    const double* lin = P.lin + e * (NL * NQ3);   // ptx = 1 at these orders
    double dg[ND][ND];
#pragma unroll
    for (int b = 0; b < ND; ++b)
#pragma unroll
      for (int a = 0; a < ND; ++a) dg[b][a] = 0.0;
#pragma unroll
    for (int t = 0; t < NL; ++t) {
      double Z[NQ][NQ];
#pragma unroll
      for (int j = 0; j < NQ; ++j)
#pragma unroll
        for (int i = 0; i < NQ; ++i) Z[j][i] = 0.0;
#pragma unroll
      for (int l = 0; l < NQ; ++l) {
        const double tz = WT[t] * zt[TZ[t]][l][c];
        const double* row = lin + (l * NL + t) * NQ2;
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
          if constexpr (NQ % 2 == 0) {
#pragma unroll
            for (int i = 0; i < NQ; i += 2) {
              const double2 v = __ldg(reinterpret_cast<const double2*>(row + j * NQ + i));
              Z[j][i] = fma(tz, v.x, Z[j][i]);
              Z[j][i + 1] = fma(tz, v.y, Z[j][i + 1]);
            }
          } else {
#pragma unroll
            for (int i = 0; i < NQ; ++i) Z[j][i] = fma(tz, __ldg(row + j * NQ + i), Z[j][i]);
          }
        }
      }
#pragma unroll
      for (int b = 0; b < ND; ++b) {
        double y[NQ];
#pragma unroll
        for (int i = 0; i < NQ; ++i) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < NQ; ++j) s = fma(tab(TY[t], j, b), Z[j][i], s);
          y[i] = s;
        }
#pragma unroll
        for (int a = 0; a < ND; ++a) {
          double s = dg[b][a];
#pragma unroll
          for (int i = 0; i < NQ; ++i) s = fma(tab(TX[t], i, a), y[i], s);
          dg[b][a] = s;
        }
      }
    }
    const int ex = (int)(e % P.nx), ey = (int)((e / P.nx) % P.ny), ez = (int)(e / ((int64_t)P.nx * P.ny));
    double* out = ev + ((int64_t)(ND * ez + c) * LYd + ND * ey) * LXd + ND * ex;
#pragma unroll
    for (int b = 0; b < ND; ++b)
#pragma unroll
      for (int a = 0; a < ND; ++a) out[(int64_t)b * LXd + a] = dg[b][a];
  }
}

template <int ND, int NL>
static cudaError_t diag_pt_t(const OpParams& P, const Tables& T, double* ev, double* diag, cudaStream_t st) {
  int slots = 0;
  cudaError_t e = persistent_slots((const void*)diag_pt_kernel<ND, NL>, 128, 0, &slots);
  if (e != cudaSuccess) return e;
  const int64_t items = (int64_t)P.nx * P.ny * P.nz * ND;
  const int64_t b = (items + 127) / 128;
  diag_pt_kernel<ND, NL><<<(unsigned)(b < slots ? b : slots), 128, 0, st>>>(P, T, ev);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return evec_assemble<ND - 1>(P, ev, diag, nullptr, nullptr, 1.0, st);   // Dirichlet rows: 1
}


// Q3 (the C3 order): a half-warp per element, lane = point column (j, i). The element's
// stored linearisation plane (l, term) is one coalesced 128-byte row per half-warp; each
// lane contracts its column along z in registers, the terms sharing (x, y) tables are
// summed (6 groups), then the y and the x contractions are two rotated 4-lane
// reduce-scatters (3 64-bit shuffles each, the tables rotated per lane as in the plane
// kernel's B^T): lane (j, i) ends with diag(a = i, b = j, c) for c = 0..3.
template <int NL>
__global__ void __launch_bounds__(128, 4) diag_q3_kernel(const OpParams P, const Tables T, double* __restrict__ ev) {
  constexpr int TZ[9] = {0, 0, 1, 0, 2, 2, 0, 0, 2};
  constexpr int GT[9] = {0, 1, 2, 3, 4, 5, 4, 5, 2};   // term -> group of equal (x, y) tables
  constexpr int GX[6] = {1, 0, 0, 2, 2, 0};            // group x table kind (0 B^2, 1 G^2, 2 GB)
  constexpr int GY[6] = {0, 1, 0, 2, 0, 2};            // group y table kind
  const int lane = threadIdx.x & 31, half = lane >> 4, pl = lane & 15, j = pl >> 2, i = pl & 3;
  auto tab = [&](int kind, int p, int n) { return kind == 0 ? T.B2[p][n] : kind == 1 ? T.G2[p][n] : T.GB[p][n]; };
  // receive-side tables: lane (j, i) takes Z(i, j') from lane j' = (j + k) & 3 and weights it
  // with TY[j'][j] (ty[kind][k]); likewise TX[i'][i] for i' = (i + k) & 3
  double ty[3][4], tx[3][4];
  int sy[4], sx[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    sy[k] = half * 16 + ((j + k) & 3) * 4 + i;
    sx[k] = half * 16 + j * 4 + ((i + k) & 3);
#pragma unroll
    for (int kd = 0; kd < 3; ++kd) {
      ty[kd][k] = tab(kd, (j + k) & 3, j);
      tx[kd][k] = tab(kd, (i + k) & 3, i);
    }
  }
  const int64_t E = (int64_t)P.nx * P.ny * P.nz;
  const int64_t LXd = 4 * (int64_t)P.nx, LYd = 4 * (int64_t)P.ny;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); 2 * w < E; w += nw) {
    const int64_t e = 2 * w + half;
    const bool ev_ok = e < E;
    const double* lin = P.lin + (ev_ok ? e : 0) * (NL * 64) + pl;
    double Z[6][4];
#pragma unroll
    for (int g = 0; g < 6; ++g)
#pragma unroll
      for (int c = 0; c < 4; ++c) Z[g][c] = 0.0;
#pragma unroll
    for (int t = 0; t < NL; ++t) {
      double A[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) A[l] = __ldcs(lin + (l * NL + t) * 16);
      if (t >= 3 && t < 6) {   // the off-diagonal A terms count twice
#pragma unroll
        for (int l = 0; l < 4; ++l) A[l] += A[l];
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double s = Z[GT[t]][c];
#pragma unroll
        for (int l = 0; l < 4; ++l) s = fma(tab(TZ[t], l, c), A[l], s);
        Z[GT[t]][c] = s;
      }
    }
    double dg[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      // y per group: Y(i, b = j) = sum_j' TY[j'][j] Z(i, j'), summed over the groups that share
      // an x table (3 x-contractions instead of 6: the shuffles bound this kernel); then
      // x: D(a = i, b = j) = sum_i' TX[i'][i] Y(i', j)
      double Yx[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int g = 0; g < 6; ++g) {
        double y = ty[GY[g]][0] * Z[g][c];
#pragma unroll
        for (int k = 1; k < 4; ++k) y = fma(ty[GY[g]][k], __shfl_sync(0xffffffffu, Z[g][c], sy[k]), y);
        Yx[GX[g]] += y;
      }
#pragma unroll
      for (int kd = 0; kd < 3; ++kd) {
        double x = tx[kd][0] * Yx[kd];
#pragma unroll
        for (int k = 1; k < 4; ++k) x = fma(tx[kd][k], __shfl_sync(0xffffffffu, Yx[kd], sx[k]), x);
        dg[c] += x;
      }
    }
    if (ev_ok) {
      int ex, ey, ez;
      {
        const unsigned u = (unsigned)e, q = u / (unsigned)P.nx;
        ex = (int)(u - q * (unsigned)P.nx);
        ey = (int)(q % (unsigned)P.ny);
        ez = (int)(q / (unsigned)P.ny);
      }
      double* out = ev + ((int64_t)(4 * ez) * LYd + 4 * ey + j) * LXd + 4 * ex + i;
#pragma unroll
      for (int c = 0; c < 4; ++c) out[(int64_t)c * LYd * LXd] = dg[c];
    }
  }
}

template <int NL>
static cudaError_t diag_q3_t(const OpParams& P, const Tables& T, double* ev, double* diag, cudaStream_t st) {
  int slots = 0;
  cudaError_t e = persistent_slots((const void*)diag_q3_kernel<NL>, 128, 0, &slots);
  if (e != cudaSuccess) return e;
  const int64_t warps = ((int64_t)P.nx * P.ny * P.nz + 1) / 2;
  const int64_t b = (warps + 3) / 4;
  diag_q3_kernel<NL><<<(unsigned)(b < slots ? b : slots), 128, 0, st>>>(P, T, ev);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return evec_assemble<3>(P, ev, diag, nullptr, nullptr, 1.0, st);   // Dirichlet rows: 1
}

cudaError_t jacobi_diag_nd(int nd, int model, const OpParams& P, const Tables& T, double* ev, double* diag,
                           cudaStream_t st) {
  const bool nine = lin_values(model) == 9;
  // Q1, Q2: every element in one launch into the discontinuous L-vector + assembly (the
  // Dirichlet rows set there); C5 2293 (8 colours, r01) -> 714 (colours, thread per element)
  if (ev && nd <= 3 && (size_t)nd * P.nx * sizeof(double) * (kAsmThreads / 32) <= 227 * 1024)
    return nd == 2 ? (nine ? diag_elem_t<2, 9>(P, T, ev, diag, st) : diag_elem_t<2, 6>(P, T, ev, diag, st))
                   : (nine ? diag_elem_t<3, 9>(P, T, ev, diag, st) : diag_elem_t<3, 6>(P, T, ev, diag, st));
  if (ev && nd >= 4 && nd <= 5 && P.ptx == 1 && (size_t)nd * P.nx * sizeof(double) * (kAsmThreads / 32) <= 227 * 1024) {
    switch (nd) {
      case 4:
        if (FEOD_DIAG_Q3_WARP) return nine ? diag_q3_t<9>(P, T, ev, diag, st) : diag_q3_t<6>(P, T, ev, diag, st);
        return nine ? diag_pt_t<4, 9>(P, T, ev, diag, st) : diag_pt_t<4, 6>(P, T, ev, diag, st);
      case 5: return nine ? diag_pt_t<5, 9>(P, T, ev, diag, st) : diag_pt_t<5, 6>(P, T, ev, diag, st);
    }   // (Q5: 36 + 36 accumulators per thread spill; the colour sweep stays)
  }
  const cudaError_t e = cudaMemsetAsync(diag, 0, sizeof(double) * (size_t)P.Mx * P.My * P.Mz, st);
  if (e != cudaSuccess) return e;
  switch (nd) {
    case 2:
    case 3: {
      cudaError_t e2 = nd == 2 ? (nine ? diag_elem_t<2, 9>(P, T, nullptr, diag, st) : diag_elem_t<2, 6>(P, T, nullptr, diag, st))
                               : (nine ? diag_elem_t<3, 9>(P, T, nullptr, diag, st) : diag_elem_t<3, 6>(P, T, nullptr, diag, st));
      if (e2 != cudaSuccess) return e2;
      const int64_t n = (int64_t)P.Mx * P.My * P.Mz;
      const int64_t b = (n + 255) / 256;
      diag_dirichlet_kernel<<<(unsigned)(b < kRedBlocks ? b : kRedBlocks), 256, 0, st>>>(P, diag);
      return cudaGetLastError();
    }
    case 4: return nine ? diag_nd_t<4, 9>(P, T, diag, st) : diag_nd_t<4, 6>(P, T, diag, st);
    case 5: return nine ? diag_nd_t<5, 9>(P, T, diag, st) : diag_nd_t<5, 6>(P, T, diag, st);
    case 6: return nine ? diag_nd_t<6, 9>(P, T, diag, st) : diag_nd_t<6, 6>(P, T, diag, st);
    case 7: return nine ? diag_nd_t<7, 9>(P, T, diag, st) : diag_nd_t<7, 6>(P, T, diag, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace feod
