// K9b — element tangent matrices K_e = B^T J_D(u_q) B (Eq. 3) at
// Q4..Q6 (nd = 5..7) on the FP64 tensor cores; the Q1..Q3 kernel is elemat.cu (K9).
// Same factorisation as K9 (Table 1's RES: D linearised at the points by 4 dual
// evaluations):
//   K_e = M^T N,  M[(q,d)][i] = d_d phi_i(x_q),  N[(q,d)][j] = sum_d' A_dd'(q) d_d' phi_j(x_q) + b_d(q) phi_j(x_q)
// but M and N no longer fit in shared memory (Q6: 1029 x 343 doubles each, 2.8 MB), so
// the product runs as a tiled GEMM whose operands are generated on chip: K_e is cut into
// 128 x 128 output tiles, and for each tile the k = (point, direction) dimension is
// streamed in chunks of KC points -- the chunk's M rows (the i-tile's reference
// gradients) and N rows (the j-tile's gradients mixed by the point's 3x3 A and b) are
// evaluated from the 1D tables into a double-buffered shared-memory stage while the
// warps run the previous chunk's 8x8x4 DMMA steps. 16 warps as 4 x 4, each a 32 x 32
// sub-tile (16 accumulator chains; 4 A + 4 B fragments per 16 DMMA): ptxas issues a warp's
// DMMAs ~16 cycles apart, so the FP64 pipe needs several warps per scheduler in their DMMA
// phase while others stage. Measured (C4, Q6, us/element): 8 warps with 128 x 64 tiles
// 14.1, 128 x 128 12.6, + hoisted index math 11.2, 16 warps 10.2; 4-point chunks at two
// CTAs per SM 14.2.
// One CTA per element (persistent over the range); the element's u at the points and
// its linearisation (9 values per point) are computed once per element.
#include "common.cuh"
#include "dual.cuh"
#include "kernels.h"
#include "physics.cuh"

namespace feod {

#ifndef FEOD_EH_WARPS
#define FEOD_EH_WARPS 16
#endif
constexpr int kEhThreads = 32 * FEOD_EH_WARPS;   // warps as 4 x (WARPS / 4) over the output tile
// experiment knobs: points per k-chunk, output-tile width (128: 32x64 warp tiles, 64: 32x32),
// CTAs per SM the register budget is sized for
#ifndef FEOD_EH_KC
#define FEOD_EH_KC 8
#endif
#ifndef FEOD_EH_CB
#define FEOD_EH_CB 128
#endif
#ifndef FEOD_EH_MINB
#define FEOD_EH_MINB 1
#endif

FEOD_DEV void dmma884_hi(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int ND>
struct EhShape {
  static constexpr int NQ = ND, Q = ND * ND * ND, NN = ND * ND * ND;
  static constexpr int KC = FEOD_EH_KC, KR = 3 * KC;     // points per k-chunk, k-rows per chunk (4 | KR)
  static_assert(KR % 4 == 0, "k-chunk of whole DMMA k-steps");
  static constexpr int NCH = (Q + KC - 1) / KC;
  static constexpr int RB = 128, CB = FEOD_EH_CB;        // output tile
  static constexpr int WCT = CB / (2 * FEOD_EH_WARPS);  // 8-column tiles per warp (warps as 4 x WARPS/4)
  static constexpr int RT = (NN + RB - 1) / RB, CT = (NN + CB - 1) / CB;
  static constexpr int MS = RB + 4, NS = CB + 4;         // row strides = 4 (mod 16) doubles: conflict-free fragments
  static constexpr int STAGE = KR * (MS + NS);
  static constexpr int QP = NCH * KC;                    // points padded to whole chunks
  static constexpr size_t SMEM = sizeof(double) * (2 * STAGE + 9 * Q + 4 * Q + NN + 2 * NQ * ND + NQ) + sizeof(int) * QP;
  static_assert(kEhThreads % RB == 0 && kEhThreads % CB == 0, "a thread's tile column is loop-invariant");
  static_assert(2 * NQ * ND * ND + 3 * NQ * NQ * ND <= 9 * Q, "interpolation scratch fits in PW");
};

template <int ND, int MODEL, bool AFFINE>
__global__ void __launch_bounds__(kEhThreads, FEOD_EH_MINB) elemat_hi_kernel(const OpParams P, const Tables T,
                                                                  const double* __restrict__ u, int e0, int ne,
                                                                  double* __restrict__ Ke) {
  using S = EhShape<ND>;
  constexpr int NQ = S::NQ, Q = S::Q, NN = S::NN, KC = S::KC, KR = S::KR, MS = S::MS, NS = S::NS;
  constexpr int RB = S::RB, CB = S::CB, WCT = S::WCT;
  constexpr int K = ND - 1;
  extern __shared__ double sm[];
  double* STG = sm;                       // [2][KR][MS] M^T chunk, then [2][KR][NS] N chunk
  double* PW = STG + 2 * S::STAGE;        // [9][Q]: A (xx yy zz xy xz yz), b
  double* UQ = PW + 9 * Q;                // [4][Q]: u, gh_x, gh_y, gh_z at the points
  double* UE = UQ + 4 * Q;                // [NN] element DOFs
  double* Bt = UE + NN;                   // [NQ][ND]
  double* Gt = Bt + NQ * ND;              // [NQ][ND]
  double* Wt = Gt + NQ * ND;              // [NQ]
  int* PQ = reinterpret_cast<int*>(Wt + NQ);   // [QP] point q's table row offsets (x | y << 8 | z << 16), -1 past Q
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int wr = warp & 3, wc = warp >> 2;   // the warp's 32 x (8 WCT) sub-tile of the RB x CB output tile

  for (int t = tid; t < NQ * ND; t += kEhThreads) {
    Bt[t] = T.B[t / ND][t % ND];
    Gt[t] = T.G[t / ND][t % ND];
  }
  for (int t = tid; t < NQ; t += kEhThreads) Wt[t] = T.w[t];
  for (int q = tid; q < S::QP; q += kEhThreads)
    PQ[q] = q < Q ? (q % NQ) * ND | ((q / NQ) % NQ) * ND << 8 | (q / (NQ * NQ)) * ND << 16 : -1;
  __syncthreads();

  for (int e = e0 + blockIdx.x; e < e0 + ne; e += gridDim.x) {
    const int ex = e % P.nx, ey = (e / P.nx) % P.ny, ez = e / (P.nx * P.ny);
    for (int t = tid; t < NN; t += kEhThreads) {   // G: element DOFs
      const int ia = t % ND, ib = (t / ND) % ND, ic = t / (ND * ND);
      UE[t] = u[(int64_t)(K * ex + ia) + (int64_t)P.Mx * ((K * ey + ib) + (int64_t)P.My * (K * ez + ic))];
    }
    __syncthreads();
    // B: u and its reference gradient at the points, sum-factorised x, y, z (PW as scratch):
    // V = B_x u, Vx = G_x u; W = B_y V, Wy = G_y V, Wx = B_y Vx; U = B_z W, Uz = G_z W, Uy = B_z Wy, Ux = B_z Wx
    {
      constexpr int S1 = NQ * ND * ND, S2 = NQ * NQ * ND;
      double* V = PW;             // [2][c][b][i]
      double* Wc = PW + 2 * S1;   // [3][c][j][i]
      for (int t = tid; t < 2 * S1; t += kEhThreads) {
        const int ch = t / S1, r = t % S1, i = r % NQ, cb = r / NQ;
        const double* tb = (ch == 0 ? Bt : Gt) + i * ND;
        const double* ue = UE + cb * ND;
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < ND; ++a) s = fma(tb[a], ue[a], s);
        V[t] = s;
      }
      __syncthreads();
      for (int t = tid; t < 3 * S2; t += kEhThreads) {
        const int ch = t / S2, r = t % S2, i = r % NQ, j = (r / NQ) % NQ, c = r / (NQ * NQ);
        const double* tb = (ch == 1 ? Gt : Bt) + j * ND;
        const double* vs = V + (ch == 2 ? S1 : 0) + c * ND * NQ + i;
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < ND; ++b) s = fma(tb[b], vs[b * NQ], s);
        Wc[t] = s;
      }
      __syncthreads();
      for (int t = tid; t < 4 * Q; t += kEhThreads) {
        const int d = t / Q, q = t % Q, ij = q % (NQ * NQ), l = q / (NQ * NQ);
        const double* tb = (d == 3 ? Gt : Bt) + l * ND;
        const double* ws = Wc + (d == 1 ? 2 * S2 : d == 2 ? S2 : 0) + ij;
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < ND; ++c) s = fma(tb[c], ws[c * NQ * NQ], s);
        UQ[t] = s;
      }
      __syncthreads();
    }
    // D's linearisation at each point (RES): seed s = 0..2 along e_s gives column s of
    // A = dFh/dgh (upper triangle kept), s = 3 along u gives b = dFh/du
    {
      const double rho = (MODEL == HEAT) ? P.rho[e] : 1.0;
      using D = dual<double>;
      for (int t = tid; t < 4 * Q; t += kEhThreads) {
        const int q = t >> 2, sd = t & 3;
        const int qx = q % NQ, qy = (q / NQ) % NQ, qz = q / (NQ * NQ);
        const double wq = Wt[qx] * Wt[qy] * Wt[qz];
        Metric M;
        double W;
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
        const D ud(UQ[q], sd == 3 ? 1.0 : 0.0);
        const D gh[3] = {D(UQ[Q + q], sd == 0 ? 1.0 : 0.0), D(UQ[2 * Q + q], sd == 1 ? 1.0 : 0.0),
                         D(UQ[3 * Q + q], sd == 2 ? 1.0 : 0.0)};
        D Fh[3];
        flux_hat<MODEL>(ud, gh, M, W, rho, P, Fh);
        if (sd == 0) {
          PW[0 * Q + q] = Fh[0].d;
        } else if (sd == 1) {
          PW[1 * Q + q] = Fh[1].d; PW[3 * Q + q] = Fh[0].d;
        } else if (sd == 2) {
          PW[2 * Q + q] = Fh[2].d; PW[4 * Q + q] = Fh[0].d; PW[5 * Q + q] = Fh[1].d;
        } else {
          PW[6 * Q + q] = Fh[0].d; PW[7 * Q + q] = Fh[1].d; PW[8 * Q + q] = Fh[2].d;
        }
      }
      __syncthreads();
    }

    // shape functions of node (ia, ib, ic) at the point with table offsets pk (PQ) from the
    // 1D tables: value and reference gradient
    auto shape = [&](int pk, int ia, int ib, int ic, double& v, double& gx, double& gy, double& gz) {
      const int ox = (pk & 255) + ia, oy = ((pk >> 8) & 255) + ib, oz = (pk >> 16) + ic;
      const double bx = Bt[ox], by = Bt[oy], bz = Bt[oz];
      const double dx = Gt[ox], dy = Gt[oy], dz = Gt[oz];
      const double byz = by * bz;
      v = bx * byz;
      gx = dx * byz;
      gy = bx * dy * bz;
      gz = bx * by * dz;
    };
    // stage chunk ch into buffer b: k-row 3 qq + d of point q = KC ch + qq. A thread's tile
    // column (il = tid % RB of the M rows, tid % CB of the N rows) is fixed, so its node
    // indices (mi, mj: a | b << 8 | c << 16, -1 outside the element) are computed per tile
    auto stage = [&](int ch, int mi, int mj, int b) {
      double* Ms = STG + b * KR * MS;
      double* Ns = STG + 2 * KR * MS + b * KR * NS;
      const int il = tid % RB, jl = tid % CB;
#pragma unroll
      for (int m = 0; m < KC * RB / kEhThreads; ++m) {   // M^T rows: reference gradients of the i-tile
        const int qq = tid / RB + m * (kEhThreads / RB), pk = PQ[KC * ch + qq];
        double v = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
        if (pk >= 0 && mi >= 0) shape(pk, mi & 255, (mi >> 8) & 255, mi >> 16, v, gx, gy, gz);
        Ms[(3 * qq + 0) * MS + il] = gx;
        Ms[(3 * qq + 1) * MS + il] = gy;
        Ms[(3 * qq + 2) * MS + il] = gz;
      }
#pragma unroll
      for (int m = 0; m < KC * CB / kEhThreads; ++m) {   // N rows: A grad phi_j + b phi_j
        const int qq = tid / CB + m * (kEhThreads / CB), q = KC * ch + qq, pk = PQ[q];
        double n0 = 0.0, n1 = 0.0, n2 = 0.0;
        if (pk >= 0 && mj >= 0) {
          double v, gx, gy, gz;
          shape(pk, mj & 255, (mj >> 8) & 255, mj >> 16, v, gx, gy, gz);
          const double axx = PW[q], ayy = PW[Q + q], azz = PW[2 * Q + q], axy = PW[3 * Q + q],
                       axz = PW[4 * Q + q], ayz = PW[5 * Q + q];
          n0 = axx * gx + axy * gy + axz * gz + PW[6 * Q + q] * v;
          n1 = axy * gx + ayy * gy + ayz * gz + PW[7 * Q + q] * v;
          n2 = axz * gx + ayz * gy + azz * gz + PW[8 * Q + q] * v;
        }
        Ns[(3 * qq + 0) * NS + jl] = n0;
        Ns[(3 * qq + 1) * NS + jl] = n1;
        Ns[(3 * qq + 2) * NS + jl] = n2;
      }
    };
    auto node = [](int n) { return n < NN ? n % ND | (n / ND) % ND << 8 | n / (ND * ND) << 16 : -1; };

    double* Ko = Ke + (int64_t)(e - e0) * NN * NN;
    for (int tile = 0; tile < S::RT * S::CT; ++tile) {
      const int r0 = (tile / S::CT) * RB, c0 = (tile % S::CT) * CB;
      const int mi = node(r0 + tid % RB), mj = node(c0 + tid % CB);
      const int wr0 = r0 + 32 * wr, wc0 = c0 + 8 * WCT * wc;   // the warp's sub-tile origin
      const bool live = wr0 < NN && wc0 < NN;
      double acc[4][WCT][2];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < WCT; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
      stage(0, mi, mj, 0);
      __syncthreads();
      for (int ch = 0; ch < S::NCH; ++ch) {
        if (ch + 1 < S::NCH) stage(ch + 1, mi, mj, (ch + 1) & 1);   // overlaps this chunk's product
        if (live) {
          const double* Ms = STG + (ch & 1) * KR * MS + (lane & 3) * MS + 32 * wr + (lane >> 2);
          const double* Ns = STG + 2 * KR * MS + (ch & 1) * KR * NS + (lane & 3) * NS + 8 * WCT * wc + (lane >> 2);
#pragma unroll
          for (int k0 = 0; k0 < KR; k0 += 4) {
            double fa[4], fb[WCT];
#pragma unroll
            for (int a = 0; a < 4; ++a) fa[a] = Ms[k0 * MS + 8 * a];
#pragma unroll
            for (int c = 0; c < WCT; ++c) fb[c] = Ns[k0 * NS + 8 * c];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int c = 0; c < WCT; ++c) dmma884_hi(acc[a][c][0], acc[a][c][1], fa[a], fb[c]);
          }
        }
        __syncthreads();   // buffer ch & 1 is restaged at ch + 2
      }
      if (live) {
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int i = wr0 + 8 * a + (lane >> 2);
#pragma unroll
          for (int c = 0; c < WCT; ++c) {
            const int j = wc0 + 8 * c + 2 * (lane & 3);
            if (i < NN && j < NN) Ko[(int64_t)i * NN + j] = acc[a][c][0];
            if (i < NN && j + 1 < NN) Ko[(int64_t)i * NN + j + 1] = acc[a][c][1];
          }
        }
      }
    }
    __syncthreads();   // UE / UQ / PW reused by the next element
  }
}

template <int ND, int MODEL, bool AFFINE>
static cudaError_t elemat_hi_launch(const OpParams& P, const Tables& T, const double* u, int e0, int ne, double* Ke,
                                    cudaStream_t st) {
  constexpr size_t smem = EhShape<ND>::SMEM;
  cudaError_t e = cudaFuncSetAttribute(elemat_hi_kernel<ND, MODEL, AFFINE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int grid = 0;
  if ((e = persistent_slots((const void*)elemat_hi_kernel<ND, MODEL, AFFINE>, kEhThreads, smem, &grid)) !=
      cudaSuccess)
    return e;
  const int g = ne < grid ? ne : grid;
  if (g <= 0) return cudaSuccess;
  elemat_hi_kernel<ND, MODEL, AFFINE><<<g, kEhThreads, smem, st>>>(P, T, u, e0, ne, Ke);
  return cudaGetLastError();
}

template <int ND>
static cudaError_t elemat_hi_nd_t(int model, bool affine, const OpParams& P, const Tables& T, const double* u,
                                  int e0, int ne, double* Ke, cudaStream_t st) {
  switch (model) {
    case PLAPLACE: return affine ? elemat_hi_launch<ND, PLAPLACE, true>(P, T, u, e0, ne, Ke, st)
                                 : elemat_hi_launch<ND, PLAPLACE, false>(P, T, u, e0, ne, Ke, st);
    case NLDIFF: return affine ? elemat_hi_launch<ND, NLDIFF, true>(P, T, u, e0, ne, Ke, st)
                               : elemat_hi_launch<ND, NLDIFF, false>(P, T, u, e0, ne, Ke, st);
    case HEAT: return affine ? elemat_hi_launch<ND, HEAT, true>(P, T, u, e0, ne, Ke, st)
                             : elemat_hi_launch<ND, HEAT, false>(P, T, u, e0, ne, Ke, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t element_matrices_hi_nd(int nd, int model, bool affine, const OpParams& P, const Tables& T,
                                   const double* u, int e0, int ne, double* Ke, cudaStream_t st) {
  switch (nd) {
    case 5: return elemat_hi_nd_t<5>(model, affine, P, T, u, e0, ne, Ke, st);
    case 6: return elemat_hi_nd_t<6>(model, affine, P, T, u, e0, ne, Ke, st);
    case 7: return elemat_hi_nd_t<7>(model, affine, P, T, u, e0, ne, Ke, st);
  }
  return cudaErrorNotSupported;
}

}  // namespace feod
