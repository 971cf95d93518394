// K10 — element tangent matrices by element-level forward AD ("ELM", Table 1 of the
// paper): K_e[:, j] = d r_e / d u_j is obtained
// by pushing the dual (u_e, e_j) through the WHOLE element residual
//   r_e(u_e) = B^T D(B u_e)        (Eq. 1 restricted to one element)
// -- the sum-factorised interpolation B (values + collocated gradients), the dual-number
// flux D (physics.cuh) and the transposed contraction B^T -- one forward-mode pass per
// seed j. B is inside the differentiation loop, as Table 1's ELM column defines it
// ("including the operator B in the differentiation loop"); the
// number of dual flux evaluations per point grows with the element's DOFs (nd^3 of them
// against RES's 4), which is the growth Table 1 reports.
//
// One CTA per element (persistent over the range), one thread per seed j; the seed's
// tangent arrays are thread-interleaved ([slot][thread]: conflict-free / coalesced) in
// shared memory up to Q3, and from Q4 on (Q4: 512 KB per CTA, Q6: 3.9 MB) in a global
// scratch slice per CTA (L2 / HBM traffic: ELM is the slow column of Table 1).
// The value part of the dual (u_e, B u_e at the points) is the same for every seed and
// is computed once per element.
#include "common.cuh"
#include "dual.cuh"
#include "kernels.h"
#include "physics.cuh"

namespace feod {

template <int ND>
struct ElmShape {
  static constexpr int NQ = ND, Q = ND * ND * ND, NN = ND * ND * ND;
  static constexpr int NT = (NN + 31) / 32 * 32;        // one thread per seed column
  static constexpr int SLOTS = 4 * Q;                    // per-thread tangent arrays (values + 3 gradients)
  static constexpr bool GLOBAL = ND >= 5;                // tangent arrays in the global scratch
  static constexpr size_t SCRATCH = GLOBAL ? (size_t)SLOTS * NT : 0;   // doubles per CTA
  static constexpr size_t SMEM = sizeof(double) * ((GLOBAL ? 0 : (size_t)SLOTS * NT) + 4 * Q + NN);
};

template <int ND, int MODEL, bool AFFINE>
__global__ void __launch_bounds__(ElmShape<ND>::NT) elm_kernel(const OpParams P, const Tables T,
                                                               const double* __restrict__ u, int e0, int ne,
                                                               double* __restrict__ Ke, double* __restrict__ scr) {
  using S = ElmShape<ND>;
  constexpr int NQ = S::NQ, Q = S::Q, NN = S::NN, NT = S::NT, K = ND - 1;
  constexpr int NQ2 = NQ * NQ;
  extern __shared__ double sm[];
  double* W = S::GLOBAL ? scr + blockIdx.x * S::SCRATCH : sm;   // [SLOTS][NT] this thread's tangent arrays
  double* UQ = S::GLOBAL ? sm : W + (size_t)S::SLOTS * NT;        // [4][Q] value part: u, gh_x, gh_y, gh_z
  double* UE = UQ + 4 * Q;                // [NN] element DOFs
  const int tid = threadIdx.x;
  const bool seed = tid < NN;             // thread tid differentiates along e_tid
  auto w = [&](int slot) -> double& { return W[(size_t)slot * NT + tid]; };

  for (int e = e0 + blockIdx.x; e < e0 + ne; e += gridDim.x) {
    const int ex = e % P.nx, ey = (e / P.nx) % P.ny, ez = e / (P.nx * P.ny);
    for (int t = tid; t < NN; t += NT) {
      const int ia = t % ND, ib = (t / ND) % ND, ic = t / (ND * ND);
      UE[t] = u[(int64_t)(K * ex + ia) + (int64_t)P.Mx * ((K * ey + ib) + (int64_t)P.My * (K * ez + ic))];
    }
    __syncthreads();
    // value part at the points (shared by all seeds): B then the collocated gradient
    for (int q = tid; q < Q; q += NT) {
      const int i = q % NQ, j = (q / NQ) % NQ, l = q / NQ2;
      double s = 0.0;
      for (int c = 0; c < ND; ++c)
        for (int b = 0; b < ND; ++b)
          for (int a = 0; a < ND; ++a) s = fma(T.B[i][a] * T.B[j][b] * T.B[l][c], UE[a + ND * (b + ND * c)], s);
      UQ[q] = s;
    }
    __syncthreads();
    for (int q = tid; q < Q; q += NT) {
      const int i = q % NQ, j = (q / NQ) % NQ, l = q / NQ2;
      double gx = 0.0, gy = 0.0, gz = 0.0;
      for (int m = 0; m < NQ; ++m) {
        gx = fma(T.D[i][m], UQ[m + NQ * (j + NQ * l)], gx);
        gy = fma(T.D[j][m], UQ[i + NQ * (m + NQ * l)], gy);
        gz = fma(T.D[l][m], UQ[i + NQ * (j + NQ * m)], gz);
      }
      UQ[Q + q] = gx;
      UQ[2 * Q + q] = gy;
      UQ[3 * Q + q] = gz;
    }
    __syncthreads();

    if (seed) {
      // ---- tangent through B: the seed e_tid as a nodal vector, sum-factorised like the operator
      // slots [0, NN): x0[c][b][a]; x-pass -> slots [Q, ..) t1[c][b][i]; y -> t2[c][j][i]; z -> U_t[l][j][i]
      for (int n = 0; n < NN; ++n) w(n) = (n == tid) ? 1.0 : 0.0;
      for (int c = 0; c < ND; ++c)
        for (int b = 0; b < ND; ++b)
          for (int i = 0; i < NQ; ++i) {
            double s = 0.0;
            for (int a = 0; a < ND; ++a) s = fma(T.B[i][a], w(a + ND * (b + ND * c)), s);
            w(Q + i + NQ * (b + ND * c)) = s;
          }
      for (int c = 0; c < ND; ++c)
        for (int j = 0; j < NQ; ++j)
          for (int i = 0; i < NQ; ++i) {
            double s = 0.0;
            for (int b = 0; b < ND; ++b) s = fma(T.B[j][b], w(Q + i + NQ * (b + ND * c)), s);
            w(2 * Q + i + NQ * (j + NQ * c)) = s;
          }
      for (int l = 0; l < NQ; ++l)
        for (int ji = 0; ji < NQ2; ++ji) {
          double s = 0.0;
          for (int c = 0; c < ND; ++c) s = fma(T.B[l][c], w(2 * Q + ji + NQ2 * c), s);
          w(ji + NQ2 * l) = s;   // U_t in slots [0, Q)
        }
      // collocated gradients of the tangent -> slots [Q, 4Q)
      for (int q = 0; q < Q; ++q) {
        const int i = q % NQ, j = (q / NQ) % NQ, l = q / NQ2;
        double gx = 0.0, gy = 0.0, gz = 0.0;
        for (int m = 0; m < NQ; ++m) {
          gx = fma(T.D[i][m], w(m + NQ * (j + NQ * l)), gx);
          gy = fma(T.D[j][m], w(i + NQ * (m + NQ * l)), gy);
          gz = fma(T.D[l][m], w(i + NQ * (j + NQ * m)), gz);
        }
        w(Q + q) = gx;
        w(2 * Q + q) = gy;
        w(3 * Q + q) = gz;
      }
      // ---- D in dual numbers at every point: (value, this seed's tangent) -> tangent flux
      const double rho = (MODEL == HEAT) ? P.rho[e] : 1.0;
      for (int q = 0; q < Q; ++q) {
        const int i = q % NQ, j = (q / NQ) % NQ, l = q / NQ2;
        const double wq = T.w[i] * T.w[j] * T.w[l];
        Metric M;
        double Wq;
        if constexpr (AFFINE) {
          M = {wq * P.cx, wq * P.cy, wq * P.cz, 0.0, 0.0, 0.0};
          Wq = wq * P.vol;
        } else {
          const int64_t px = P.ptx;
          const double* g = P.geom + pt_base(P, ex, ey, ez, 6 * Q) + (l * 6 * NQ2 + j * NQ + i) * px;
          M = {g[0], g[NQ2 * px], g[2 * NQ2 * px], g[3 * NQ2 * px], g[4 * NQ2 * px], g[5 * NQ2 * px]};
          const double det = M.xx * (M.yy * M.zz - M.yz * M.yz) - M.xy * (M.xy * M.zz - M.yz * M.xz) +
                             M.xz * (M.xy * M.yz - M.yy * M.xz);
          Wq = det / (wq * wq);
        }
        using Dd = dual<double>;
        const Dd ud(UQ[q], w(q));
        const Dd gh[3] = {Dd(UQ[Q + q], w(Q + q)), Dd(UQ[2 * Q + q], w(2 * Q + q)), Dd(UQ[3 * Q + q], w(3 * Q + q))};
        Dd Fh[3];
        flux_hat<MODEL>(ud, gh, M, Wq, rho, P, Fh);
        w(Q + q) = Fh[0].d;
        w(2 * Q + q) = Fh[1].d;
        w(3 * Q + q) = Fh[2].d;
      }
      // ---- B^T: R = sum_d D_d^T F_d at the points (slots [0, Q)), then z, y, x transposes
      for (int q = 0; q < Q; ++q) w(q) = 0.0;
      for (int q = 0; q < Q; ++q) {
        const int i = q % NQ, j = (q / NQ) % NQ, l = q / NQ2;
        const double fx = w(Q + q), fy = w(2 * Q + q), fz = w(3 * Q + q);
        for (int m = 0; m < NQ; ++m) {
          w(m + NQ * (j + NQ * l)) = fma(T.D[i][m], fx, w(m + NQ * (j + NQ * l)));
          w(i + NQ * (m + NQ * l)) = fma(T.D[j][m], fy, w(i + NQ * (m + NQ * l)));
          w(i + NQ * (j + NQ * m)) = fma(T.D[l][m], fz, w(i + NQ * (j + NQ * m)));
        }
      }
      for (int c = 0; c < ND; ++c)   // z: slots [Q, ..) s1[c][j][i]
        for (int ji = 0; ji < NQ2; ++ji) {
          double s = 0.0;
          for (int l = 0; l < NQ; ++l) s = fma(T.B[l][c], w(ji + NQ2 * l), s);
          w(Q + ji + NQ2 * c) = s;
        }
      for (int c = 0; c < ND; ++c)   // y: slots [2Q, ..) s2[c][b][i]
        for (int b = 0; b < ND; ++b)
          for (int i = 0; i < NQ; ++i) {
            double s = 0.0;
            for (int j = 0; j < NQ; ++j) s = fma(T.B[j][b], w(Q + i + NQ * (j + NQ * c)), s);
            w(2 * Q + i + NQ * (b + ND * c)) = s;
          }
      double* col = Ke + (int64_t)(e - e0) * NN * NN + tid;   // K_e[n][tid]
      for (int c = 0; c < ND; ++c)   // x: the column's node values
        for (int b = 0; b < ND; ++b)
          for (int a = 0; a < ND; ++a) {
            double s = 0.0;
            for (int i = 0; i < NQ; ++i) s = fma(T.B[i][a], w(2 * Q + i + NQ * (b + ND * c)), s);
            col[(int64_t)(a + ND * (b + ND * c)) * NN] = s;
          }
    }
    __syncthreads();   // UE / UQ reused by the next element
  }
}

template <int ND, int MODEL, bool AFFINE>
static cudaError_t elm_launch(const OpParams& P, const Tables& T, const double* u, int e0, int ne, double* Ke,
                              double* scr, size_t scr_doubles, cudaStream_t st) {
  using S = ElmShape<ND>;
  cudaError_t e = cudaFuncSetAttribute(elm_kernel<ND, MODEL, AFFINE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)S::SMEM);
  if (e != cudaSuccess) return e;
  int slots = 0;
  if ((e = persistent_slots((const void*)elm_kernel<ND, MODEL, AFFINE>, S::NT, S::SMEM, &slots)) != cudaSuccess)
    return e;
  if (S::GLOBAL) {   // the grid is bounded by the scratch the caller provides
    if (!scr) return cudaErrorInvalidValue;
    const size_t cap = scr_doubles / S::SCRATCH;
    if ((size_t)slots > cap) slots = (int)cap;
  }
  const int g = ne < slots ? ne : slots;
  if (g <= 0) return ne > 0 ? cudaErrorInvalidValue : cudaSuccess;
  elm_kernel<ND, MODEL, AFFINE><<<g, S::NT, S::SMEM, st>>>(P, T, u, e0, ne, Ke, scr);
  return cudaGetLastError();
}

template <int ND>
static cudaError_t elm_nd_t(int model, bool affine, const OpParams& P, const Tables& T, const double* u, int e0,
                            int ne, double* Ke, double* scr, size_t scr_doubles, cudaStream_t st) {
  switch (model) {
    case PLAPLACE: return affine ? elm_launch<ND, PLAPLACE, true>(P, T, u, e0, ne, Ke, scr, scr_doubles, st)
                                 : elm_launch<ND, PLAPLACE, false>(P, T, u, e0, ne, Ke, scr, scr_doubles, st);
    case NLDIFF: return affine ? elm_launch<ND, NLDIFF, true>(P, T, u, e0, ne, Ke, scr, scr_doubles, st)
                               : elm_launch<ND, NLDIFF, false>(P, T, u, e0, ne, Ke, scr, scr_doubles, st);
    case HEAT: return affine ? elm_launch<ND, HEAT, true>(P, T, u, e0, ne, Ke, scr, scr_doubles, st)
                             : elm_launch<ND, HEAT, false>(P, T, u, e0, ne, Ke, scr, scr_doubles, st);
  }
  return cudaErrorInvalidValue;
}

size_t elm_scratch_per_cta(int nd) {
  switch (nd) {
    case 5: return ElmShape<5>::SCRATCH;
    case 6: return ElmShape<6>::SCRATCH;
    case 7: return ElmShape<7>::SCRATCH;
  }
  return 0;
}

cudaError_t element_matrices_elm_nd(int nd, int model, bool affine, const OpParams& P, const Tables& T,
                                    const double* u, int e0, int ne, double* Ke, double* scr, size_t scr_doubles,
                                    cudaStream_t st) {
  switch (nd) {
    case 2: return elm_nd_t<2>(model, affine, P, T, u, e0, ne, Ke, scr, scr_doubles, st);
    case 3: return elm_nd_t<3>(model, affine, P, T, u, e0, ne, Ke, scr, scr_doubles, st);
    case 4: return elm_nd_t<4>(model, affine, P, T, u, e0, ne, Ke, scr, scr_doubles, st);
    case 5: return elm_nd_t<5>(model, affine, P, T, u, e0, ne, Ke, scr, scr_doubles, st);
    case 6: return elm_nd_t<6>(model, affine, P, T, u, e0, ne, Ke, scr, scr_doubles, st);
    case 7: return elm_nd_t<7>(model, affine, P, T, u, e0, ne, Ke, scr, scr_doubles, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace feod
