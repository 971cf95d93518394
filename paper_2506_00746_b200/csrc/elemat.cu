// K9 — element tangent matrices K_e = B^T J_D(u_q) B (Eq. 3) on
// the FP64 tensor cores: the hex analogue of Table 1 (SURVEY
// §8(f) NEXT-4). With the per-point linearisation of D (A = dFh/dgh, b = dFh/du)
//   K_e = M^T N,  M[(d,q)][i] = d_d phi_i(x_q),  N[(d,q)][j] = sum_d' A_dd'(q) d_d' phi_j(x_q) + b_d(q) phi_j(x_q),
// a (nd^3 x 3Q) x (3Q x nd^3) product per element, run as 8x8x4 DMMA tiles
// (mma.sync m8n8k4 f64: sm_100a executes it on the same FP64 pipe as DFMA, at
// 37 TF/s measured vs 32 TF/s for DFMA — tools/dmma_probe.cu).
//   RES (integration-point AD, the paper's approach): A and b from 4 dual
//       evaluations of D per point, then N from the tables.
//   ELM (element-level forward AD, B inside the differentiation loop): elm.cu (K10).
// One CTA (8 warps) per element, persistent over a range of elements. M^T and the
// 1D tables are element-independent and built once per CTA in shared memory.
#include "common.cuh"
#include "dual.cuh"
#include "kernels.h"
#include "physics.cuh"

namespace feod {

constexpr int kEmThreads = 256;
// M^T as a shared-memory table (Q1, Q2: measured faster) or rebuilt from the 1D tables
// where used (Q3: the 96 KB table would leave one CTA per SM; without it, two —
// RES 169 -> 123 ns/element); FEOD_EM_MT = 0 / 1 forces either for experiments
#ifndef FEOD_EM_MT
#define FEOD_EM_MT -1
#endif
template <int ND>
constexpr bool em_table() { return FEOD_EM_MT >= 0 ? FEOD_EM_MT == 1 : ND <= 3; }

FEOD_DEV void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int ND>
struct EmShape {
  static constexpr int NQ = ND, Q = ND * ND * ND, NN = ND * ND * ND;
  static constexpr int NP = (NN + 7) / 8 * 8;          // padded node count (DMMA m, n)
  static constexpr int KD = (3 * Q + 3) / 4 * 4;       // padded inner dimension (DMMA k)
  static constexpr int MT = em_table<ND>() ? NP * KD : 0;   // M^T [i][k]
  // N's row stride: = 4 (mod 16) doubles, so the B fragment's 4 k-rows x 4 columns of a
  // half-warp hit 16 different bank pairs (a stride of NP = 64 put all 4 rows on one bank)
  static constexpr int NPS = NP + ((4 - NP % 16) + 16) % 16;
  static constexpr int NM = KD * NPS;                  // N [k][j]
  static constexpr size_t SMEM = sizeof(double) * (MT + NM + 9 * Q + 4 * Q + NN + 2 * NQ * ND + 3 * NQ);
};

template <int ND, int MODEL, bool AFFINE, bool ELM>
__global__ void __launch_bounds__(kEmThreads, 1) elemat_kernel(const OpParams P, const Tables T,
                                                               const double* __restrict__ u, int e0, int ne,
                                                               double* __restrict__ Ke) {
  using S = EmShape<ND>;
  constexpr int NQ = S::NQ, Q = S::Q, NN = S::NN, NP = S::NP, KD = S::KD, NPS = S::NPS;
  constexpr int K = ND - 1;
  extern __shared__ double sm[];
  double* MTs = sm;                      // [NP][KD]
  double* Ns = MTs + S::MT;              // [KD][NPS]
  double* PW = Ns + S::NM;               // [9][Q]: A (xx yy zz xy xz yz), b
  double* UQ = PW + 9 * Q;               // [4][Q]: u, gh_x, gh_y, gh_z at the points
  double* UE = UQ + 4 * Q;               // [NN] element DOFs
  double* Bt = UE + NN;                  // [NQ][ND]
  double* Gt = Bt + NQ * ND;             // [NQ][ND]
  double* Wt = Gt + NQ * ND;             // [NQ]
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);

  for (int t = tid; t < NQ * ND; t += kEmThreads) {
    Bt[t] = T.B[t / ND][t % ND];
    Gt[t] = T.G[t / ND][t % ND];
  }
  for (int t = tid; t < NQ; t += kEmThreads) Wt[t] = T.w[t];
  __syncthreads();
  // shape-function tables: phi_d(q, i) from the 1D tables (d = 0 value, 1..3 x y z derivative)
  auto phi = [&](int d, int q, int i) {
    const int qx = q % NQ, qy = (q / NQ) % NQ, qz = q / (NQ * NQ);
    const int ia = i % ND, ib = (i / ND) % ND, ic = i / (ND * ND);
    const double fx = d == 1 ? Gt[qx * ND + ia] : Bt[qx * ND + ia];
    const double fy = d == 2 ? Gt[qy * ND + ib] : Bt[qy * ND + ib];
    const double fz = d == 3 ? Gt[qz * ND + ic] : Bt[qz * ND + ic];
    return fx * fy * fz;
  };
  // M^T[i][k] = d_{k / Q} phi_i(x_{k % Q}), zero padded
  auto mt = [&](int i, int k) {
    if constexpr (em_table<ND>()) return MTs[i * KD + k];
    else return (i < NN && k < 3 * Q) ? phi(1 + k / Q, k % Q, i) : 0.0;
  };
  for (int t = tid; t < S::MT; t += kEmThreads) {
    const int i = t / KD, k = t % KD;
    MTs[t] = (i < NN && k < 3 * Q) ? phi(1 + k / Q, k % Q, i) : 0.0;
  }
  __syncthreads();

  for (int e = e0 + blockIdx.x; e < e0 + ne; e += gridDim.x) {
    const int ex = e % P.nx, ey = (e / P.nx) % P.ny, ez = e / (P.nx * P.ny);
    // G: element DOFs
    for (int t = tid; t < NN; t += kEmThreads) {
      const int ia = t % ND, ib = (t / ND) % ND, ic = t / (ND * ND);
      UE[t] = u[(int64_t)(K * ex + ia) + (int64_t)P.Mx * ((K * ey + ib) + (int64_t)P.My * (K * ez + ic))];
    }
    __syncthreads();
    // B: value and reference gradient of u at the points, sum-factorised x, y, z in shared
    // memory (PW is free scratch until the linearisation below): V = B_x u, Vx = G_x u;
    // W = B_y V, Wy = G_y V, Wx = B_y Vx; U = B_z W, Uz = G_z W, Uy = B_z Wy, Ux = B_z Wx
    {
      constexpr int S1 = NQ * ND * ND, S2 = NQ * NQ * ND;
      double* V = PW;             // [2][c][b][i]
      double* Wc = PW + 2 * S1;   // [3][c][j][i]
      for (int t = tid; t < 2 * S1; t += kEmThreads) {
        const int ch = t / S1, r = t % S1, i = r % NQ, cb = r / NQ;
        const double* tb = (ch == 0 ? Bt : Gt) + i * ND;
        const double* ue = UE + cb * ND;
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < ND; ++a) s = fma(tb[a], ue[a], s);
        V[t] = s;
      }
      __syncthreads();
      for (int t = tid; t < 3 * S2; t += kEmThreads) {
        const int ch = t / S2, r = t % S2, i = r % NQ, j = (r / NQ) % NQ, c = r / (NQ * NQ);
        const double* tb = (ch == 1 ? Gt : Bt) + j * ND;
        const double* vs = V + (ch == 2 ? S1 : 0) + c * ND * NQ + i;
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < ND; ++b) s = fma(tb[b], vs[b * NQ], s);
        Wc[t] = s;
      }
      __syncthreads();
      for (int t = tid; t < 4 * Q; t += kEmThreads) {
        const int d = t / Q, q = t % Q, ij = q % (NQ * NQ), l = q / (NQ * NQ);
        // d = 0: U from W (B), 1: Ux from Wx (B), 2: Uy from Wy (B), 3: Uz from W (G)
        const double* tb = (d == 3 ? Gt : Bt) + l * ND;
        const double* ws = Wc + (d == 1 ? 2 * S2 : d == 2 ? S2 : 0) + ij;
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < ND; ++c) s = fma(tb[c], ws[c * NQ * NQ], s);
        UQ[t] = s;
      }
      __syncthreads();
    }
    const double rho = (MODEL == HEAT) ? P.rho[e] : 1.0;
    auto metric = [&](int q, Metric& M, double& W) {
      const int qx = q % NQ, qy = (q / NQ) % NQ, qz = q / (NQ * NQ);
      const double wq = Wt[qx] * Wt[qy] * Wt[qz];
      if constexpr (AFFINE) {
        M = {wq * P.cx, wq * P.cy, wq * P.cz, 0.0, 0.0, 0.0};
        W = wq * P.vol;
      } else {
        const int64_t px = P.ptx;   // interleaved per-point layout (pt_base, common.cuh)
        const double* g = P.geom + pt_base(P, ex, ey, ez, 6 * Q) + (qz * 6 * NQ * NQ + qy * NQ + qx) * px;
        M = {g[0], g[NQ * NQ * px], g[2 * NQ * NQ * px], g[3 * NQ * NQ * px], g[4 * NQ * NQ * px], g[5 * NQ * NQ * px]};
        const double det = M.xx * (M.yy * M.zz - M.yz * M.yz) - M.xy * (M.xy * M.zz - M.yz * M.xz) +
                           M.xz * (M.xy * M.yz - M.yy * M.xz);
        W = det / (wq * wq);
      }
    };
    using D = dual<double>;
    if constexpr (!ELM) {
      // RES: D's linearisation at each point, one dual evaluation per thread: seed s = 0..2
      // along e_s gives column s of A (the upper triangle is kept), s = 3 along u gives b
      for (int t = tid; t < 4 * Q; t += kEmThreads) {
        const int q = t >> 2, sd = t & 3;
        Metric M;
        double W;
        metric(q, M, W);
        const D ud(UQ[q], sd == 3 ? 1.0 : 0.0);
        const D gh[3] = {D(UQ[Q + q], sd == 0 ? 1.0 : 0.0), D(UQ[2 * Q + q], sd == 1 ? 1.0 : 0.0),
                         D(UQ[3 * Q + q], sd == 2 ? 1.0 : 0.0)};
        D Fh[3];
        flux_hat<MODEL>(ud, gh, M, W, rho, P, Fh);
        if (sd == 0) {
          PW[0 * Q + q] = Fh[0].d;                                   // xx
        } else if (sd == 1) {
          PW[1 * Q + q] = Fh[1].d; PW[3 * Q + q] = Fh[0].d;          // yy, xy
        } else if (sd == 2) {
          PW[2 * Q + q] = Fh[2].d; PW[4 * Q + q] = Fh[0].d; PW[5 * Q + q] = Fh[1].d;   // zz, xz, yz
        } else {
          PW[6 * Q + q] = Fh[0].d; PW[7 * Q + q] = Fh[1].d; PW[8 * Q + q] = Fh[2].d;   // b
        }
      }
      __syncthreads();
      for (int t = tid; t < Q * NP; t += kEmThreads) {   // N[(d, q)][j], the three d rows per thread
        const int q = t / NP, j = t % NP;
        double n0 = 0.0, n1 = 0.0, n2 = 0.0;
        if (j < NN) {
          const double g0 = mt(j, q), g1 = mt(j, Q + q), g2 = mt(j, 2 * Q + q), p0 = phi(0, q, j);
          const double axx = PW[q], ayy = PW[Q + q], azz = PW[2 * Q + q], axy = PW[3 * Q + q], axz = PW[4 * Q + q],
                       ayz = PW[5 * Q + q];
          n0 = axx * g0 + axy * g1 + axz * g2 + PW[6 * Q + q] * p0;
          n1 = axy * g0 + ayy * g1 + ayz * g2 + PW[7 * Q + q] * p0;
          n2 = axz * g0 + ayz * g1 + azz * g2 + PW[8 * Q + q] * p0;
        }
        Ns[(0 * Q + q) * NPS + j] = n0;
        Ns[(1 * Q + q) * NPS + j] = n1;
        Ns[(2 * Q + q) * NPS + j] = n2;
      }
      for (int t = tid; t < (KD - 3 * Q) * NPS; t += kEmThreads) Ns[3 * Q * NPS + t] = 0.0;
    } else {
      // ELM: column j of N from a dual evaluation of D seeded with (phi_j, grad phi_j)
      for (int t = tid; t < Q * NP; t += kEmThreads) {
        const int q = t / NP, j = t % NP;
        double c0 = 0.0, c1 = 0.0, c2 = 0.0;
        if (j < NN) {
          Metric M;
          double W;
          metric(q, M, W);
          const D ud(UQ[q], phi(0, q, j));
          const D gh[3] = {D(UQ[Q + q], mt(j, q)), D(UQ[2 * Q + q], mt(j, Q + q)), D(UQ[3 * Q + q], mt(j, 2 * Q + q))};
          D Fh[3];
          flux_hat<MODEL>(ud, gh, M, W, rho, P, Fh);
          c0 = Fh[0].d; c1 = Fh[1].d; c2 = Fh[2].d;
        }
        Ns[(0 * Q + q) * NPS + j] = c0;
        Ns[(1 * Q + q) * NPS + j] = c1;
        Ns[(2 * Q + q) * NPS + j] = c2;
      }
      for (int t = tid; t < (KD - 3 * Q) * NPS; t += kEmThreads) Ns[3 * Q * NPS + t] = 0.0;
    }
    __syncthreads();
    // K = M^T N on the tensor cores: a warp owns one 8-row strip and all TR column
    // tiles (TR independent accumulator chains; one A fragment per k-step reused TR times)
    constexpr int TR = NP / 8;
    double* Ko = Ke + (int64_t)(e - e0) * NN * NN;
    for (int rt = warp; rt < TR; rt += kEmThreads / 32) {
      const int r8 = rt * 8;
      double acc[TR][2];
#pragma unroll
      for (int c = 0; c < TR; ++c) acc[c][0] = acc[c][1] = 0.0;
      const int ai = r8 + (lane >> 2);
      const double* bp = Ns + (lane & 3) * NPS + (lane >> 2);
#pragma unroll 2
      for (int k0 = 0; k0 < KD; k0 += 4) {
        const double a = mt(ai, k0 + (lane & 3));
#pragma unroll
        for (int c = 0; c < TR; ++c) dmma884(acc[c][0], acc[c][1], a, bp[k0 * NPS + 8 * c]);
      }
      const int i = r8 + (lane >> 2);
#pragma unroll
      for (int c = 0; c < TR; ++c) {
        const int j = 8 * c + 2 * (lane & 3);
        if (i < NN && j < NN) Ko[(int64_t)i * NN + j] = acc[c][0];
        if (i < NN && j + 1 < NN) Ko[(int64_t)i * NN + j + 1] = acc[c][1];
      }
    }
    __syncthreads();   // Ns / UQ / PW reused by the next element
  }
}

template <int ND, int MODEL, bool AFFINE, bool ELM>
static cudaError_t elemat_launch(const OpParams& P, const Tables& T, const double* u, int e0, int ne, double* Ke,
                                 cudaStream_t st) {
  constexpr size_t smem = EmShape<ND>::SMEM;
  // per call (a handle may live on any device): the attribute, then the cached occupancy
  cudaError_t e = cudaFuncSetAttribute(elemat_kernel<ND, MODEL, AFFINE, ELM>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int grid = 0;
  if ((e = persistent_slots((const void*)elemat_kernel<ND, MODEL, AFFINE, ELM>, kEmThreads, smem, &grid)) !=
      cudaSuccess)
    return e;
  const int g = ne < grid ? ne : grid;
  if (g <= 0) return cudaSuccess;
  elemat_kernel<ND, MODEL, AFFINE, ELM><<<g, kEmThreads, smem, st>>>(P, T, u, e0, ne, Ke);
  return cudaGetLastError();
}

template <int ND, int MODEL>
static cudaError_t elemat_model(bool affine, bool elm, const OpParams& P, const Tables& T, const double* u, int e0,
                                int ne, double* Ke, cudaStream_t st) {
  // RES only: the element-level AD variant (Table 1's ELM) is elm.cu (K10)
  if (elm) return cudaErrorInvalidValue;
  return affine ? elemat_launch<ND, MODEL, true, false>(P, T, u, e0, ne, Ke, st)
                : elemat_launch<ND, MODEL, false, false>(P, T, u, e0, ne, Ke, st);
}

template <int ND>
static cudaError_t elemat_nd_t(int model, bool affine, bool elm, const OpParams& P, const Tables& T, const double* u,
                               int e0, int ne, double* Ke, cudaStream_t st) {
  switch (model) {
    case PLAPLACE: return elemat_model<ND, PLAPLACE>(affine, elm, P, T, u, e0, ne, Ke, st);
    case NLDIFF: return elemat_model<ND, NLDIFF>(affine, elm, P, T, u, e0, ne, Ke, st);
    case HEAT: return elemat_model<ND, HEAT>(affine, elm, P, T, u, e0, ne, Ke, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t element_matrices_nd(int nd, int model, bool affine, bool elm, const OpParams& P, const Tables& T,
                                const double* u, int e0, int ne, double* Ke, cudaStream_t st) {
  switch (nd) {
    case 2: return elemat_nd_t<2>(model, affine, elm, P, T, u, e0, ne, Ke, st);
    case 3: return elemat_nd_t<3>(model, affine, elm, P, T, u, e0, ne, Ke, st);
    case 4: return elemat_nd_t<4>(model, affine, elm, P, T, u, e0, ne, Ke, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace feod
