// K11 / K12 -- Q6 on affine meshes on the FP64 tensor cores (C4):
// F(u), J(u)v, J(u)^T w and the stored-linearisation J v (Eq. 1 / Eq. 2, PAPER.md:155,
// :160) for k = 6, q = 7, and the Jacobi diagonal of the stored linearisation.
//
// One WARP per element, no block barriers. Each z-plane c (or point plane l) of a 7x7x7
// element array is one 8x8 DMMA fragment (padding row/column 7 = 0): lane L holds entries
// (r = L/4, c = 2 (L%4) + t), t = 0, 1 ("D layout" of mma.sync.m8n8k4.f64). Then
//   - a contraction over the fragment's COLUMN index is two DMMAs with no data movement:
//     with the k-order permuted to (k-step s, k-lane q) <-> column 2q + s, the A operand of
//     k-step s is the lane's own register t = s (the 1D table is arranged to match);
//   - a contraction over the ROW index first transposes the fragment inside the warp
//     (through a per-warp shared-memory scratch, FEOD_Q6_SMT; or 64-bit shuffles);
//   - the z-contraction (across the 7 fragments) is plain register DFMA.
// DMMA runs at 37.2 TF/s (profiles/r02_peaks_fp64.json) on the same FP64 pipe as DFMA;
// the 7 -> 8 padding leaves 67 % of its FMAs useful. The element's node results go to the
// discontinuous L-vector and evec.cuh's assembly sums each DOF's <= 8 contributions in a
// fixed order and applies P^T -- deterministic, no atomics. DESIGN.md §6.0b.
#include <algorithm>

#include "common.cuh"
#include "dual.cuh"
#include "kernels.h"
#include "physics.cuh"
#include "pointwise.cuh"
#include "evec.cuh"

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

// (M W)^T without data movement: the A and B operand layouts of m8n8k4 are each other's
// transposes, so the same lane registers with the operands swapped give
// out[m][n] = sum_c W[c][m] M[n][c] -- the column contraction landing transposed
FEOD_DEV Frag contract_cols_t(const Frag& m, const double w[2], Frag acc) {
  dmma(acc.v[0], acc.v[1], w[0], m.v[0]);
  dmma(acc.v[0], acc.v[1], w[1], m.v[1]);
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
// The same through a per-warp shared-memory scratch (two 8 x 18 buffers used in turn: one
// __syncwarp per transpose; the pitch 18 = 2 mod 16 doubles keeps each half-warp's column
// reads on 16 different bank pairs): one 16-byte store + two 8-byte loads instead of
// eight 32-bit shuffles and four selects
template <int NBUF>
FEOD_DEV Frag transpose_sm(const Frag& m, int lane, double* scr, int& tb) {
  const int r = lane >> 2, q = lane & 3;
  double* b = scr + tb * (8 * 18);
  if (NBUF == 2) tb ^= 1;
  *reinterpret_cast<double2*>(b + r * 18 + 2 * q) = make_double2(m.v[0], m.v[1]);
  __syncwarp();
  Frag o;
  o.v[0] = b[(2 * q) * 18 + r];
  o.v[1] = b[(2 * q + 1) * 18 + r];
  if (NBUF == 1) __syncwarp();   // one buffer: reads done before its next write
  return o;
}
// element coordinates by 32-bit unsigned division (E < 2^31, checked at feod_create; the
// 64-bit divisions were ~10 % of the kernel's instructions)
FEOD_DEV void q6_coords(const OpParams& P, int64_t e, int& ex, int& ey, int& ez) {
  const unsigned u = (unsigned)e, t = u / (unsigned)P.nx;
  ex = (int)(u - t * (unsigned)P.nx);
  ey = (int)(t % (unsigned)P.ny);
  ez = (int)(t / (unsigned)P.ny);
}
}  // namespace q6

#ifndef FEOD_Q6_SMT   // shared-memory transposes in q6tc_perl_kernel
#define FEOD_Q6_SMT 1
#endif
#ifndef FEOD_Q6_SMT_PA   // ... also in PAJVP, with ONE scratch buffer per warp (its shared memory also
#define FEOD_Q6_SMT_PA 0 // holds the stored linearisation; measured C4 jvp_lin 235 -> 240 us: off)
#endif
// modes: RES (F(u)), JVP (J(u) v), VJP (J(u)^T w, w's Dirichlet entries masked, reading
// A17), LIN (F(u) and the point linearisation written to P.lin), PAJVP (J(u0) v from P.lin)
template <int MODE> constexpr int q6_nin() { return (MODE == MODE_JVP || MODE == MODE_VJP) ? 2 : 1; }

// Per point plane: after x and y, each field keeps only its 7 node-plane fragments Ep[c]
// ([i][j]); point plane l is then formed, differentiated, passed through D and transposed
// back in one step -- U_l = sum_c B[l][c] Ep[c] and Uz_l = sum_c G[l][c] Ep[c] (DFMA),
// Uy_l / Ux_l by DMMA with the collocated derivative D (G = D B exactly, k <= q - 1); after
// D, R_l = V_l + Dy^T Fy_l + Dx^T Fx_l (DMMA) and the z-transpose accumulates
// S[c] += B[l][c] R_l + G[l][c] Fz_l (DFMA); finally y and x of each S[c] (DMMA). 7 fragments
// per field and 7 accumulators live (the first version held all 4 x 7 point channels and
// parked a field in shared memory: more registers, slower -- DESIGN.md §11).
#ifndef FEOD_Q6_FSTAGE   // shared-memory staging of the input fields (measured C4: JVP 304 -> 336 us
#define FEOD_Q6_FSTAGE 0   // with it, residual 225 -> 255; the L2 prefetch alone is kept)
#endif
#ifndef FEOD_Q6P_MINB1   // residual (measured C4: 4 CTAs of 4 warps per SM, 128 registers)
#define FEOD_Q6P_MINB1 4
#endif
#ifndef FEOD_Q6P_MINB2   // two-field modes and PAJVP (3 CTAs, 168 registers; PAJVP spills at 128)
#define FEOD_Q6P_MINB2 3
#endif
// DOT (CgFuse, JVP / PAJVP): also the partials of v . (J v) per CTA into dpart, formed at the
// points: v_e . (B^T F) = (B v_e) . F = sum_q w_q (grad v . F~ + v V~), F~ the tangent flux the
// point already holds -- no extra loads, 4 FMAs per point (v's Dirichlet entries are 0 in the
// CG, so the row mask P^T changes nothing). A fixed order: per lane over l and the elements,
// lanes by a butterfly, warps in order.
template <int MODE, int MODEL, bool DOT = false>
__global__ void __launch_bounds__(32 * q6::WARPS,
                                  (q6_nin<MODE>() == 2 || MODE == MODE_PAJVP) ? FEOD_Q6P_MINB2 : FEOD_Q6P_MINB1)
q6tc_perl_kernel(const OpParams P, const Tables T, const double* __restrict__ in0, const double* __restrict__ in1,
                 double* __restrict__ ev, double* __restrict__ dpart) {
  static_assert(!DOT || MODE == MODE_JVP || MODE == MODE_PAJVP, "v . (J v) needs a tangent mode");
  using namespace q6;
  constexpr int NIN = q6_nin<MODE>();
  constexpr int NL = lin_values(MODEL);
  extern __shared__ __align__(16) double q6sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int r = lane >> 2, q = lane & 3;
  const int64_t E = (int64_t)P.nx * P.ny * P.nz;
  auto tab = [&](int kind, int s) {   // 0: B[n][c] 1: D[n][c] 2: B[c][n] 3: D[c][n]
    const int c = 2 * q + s, n = r;
    if (c >= 7 || n >= 7) return 0.0;
    return kind == 0 ? T.B[n][c] : kind == 1 ? T.D[n][c] : kind == 2 ? T.B[c][n] : T.D[c][n];
  };
  // FOLD: the quadrature weight w_i w_j w_l moves out of the points into the transposed
  // tables (F = w_q F~ with M = diag(c), W = vol at the points; R = w_i w_j w_l R~ with
  // Dh[i][m] = D[i][m] w_i / w_m, then w_l into the z-transpose (Bw, Gw) and w_j, w_i into
  // the y / x transposes (Bw)). Not for PAJVP, whose stored values carry the weight.
  constexpr bool FOLD = MODE != MODE_PAJVP && MODE != MODE_LIN;
  auto tabf = [&](int kind, int s) {   // 2: Bw[c][n] 3: Dh[c][n]
    const int c = 2 * q + s, n = r;
    if (c >= 7 || n >= 7) return 0.0;
    return kind == 2 ? T.Bw[c][n] : T.Dh[c][n];
  };
  const double WB[2] = {tab(0, 0), tab(0, 1)}, WD[2] = {tab(1, 0), tab(1, 1)};
  const double WBt[2] = {FOLD ? tabf(2, 0) : tab(2, 0), FOLD ? tabf(2, 1) : tab(2, 1)};
  const double WDt[2] = {FOLD ? tabf(3, 0) : tab(3, 0), FOLD ? tabf(3, 1) : tab(3, 1)};
  const bool rowv = r < 7;
  const bool colv[2] = {2 * q < 7, 2 * q + 1 < 7};
  const Frag zero = {{0.0, 0.0}};
  constexpr bool SMT = FEOD_Q6_SMT && (MODE != MODE_PAJVP || FEOD_Q6_SMT_PA);
  // shared memory: [stored linearisation per warp + mbarriers (PAJVP) | staged fields] [transpose scratch]
  constexpr size_t LEAD_DOUBLES = (MODE == MODE_PAJVP && (NL * 49 * sizeof(double)) % 16 == 0)
                                      ? (size_t)WARPS * NL * 343 + WARPS * 8
                                  : FEOD_Q6_FSTAGE ? (size_t)WARPS * NIN * 344 : 0;
  constexpr int TBUF = MODE == MODE_PAJVP ? 1 : 2;   // transpose scratch buffers per warp
  double* const tscr = q6sm + LEAD_DOUBLES + (size_t)wid * (TBUF * 8 * 18);
  int tbuf = 0;
  auto tr = [&](const Frag& m) -> Frag {
    if constexpr (SMT) return transpose_sm<TBUF>(m, lane, tscr, tbuf);
    else return transpose(m, lane);
  };

  // x and y of one field: node plane c (rows y, columns x) -> Ep[c] = [i][j]; the nodes come
  // from the warp's shared-memory copy of the element (fb, staged one element ahead) or,
  // when that space holds the stored linearisation (PAJVP), from global memory
  auto nodes_xy = [&](const double* __restrict__ src, const double* fb, int ex, int ey, int ez, bool mask, Frag* Ep) {
    Frag X[7];
#pragma unroll
    for (int c = 0; c < 7; ++c) {
      const int64_t row = (int64_t)(K * ex) + (int64_t)P.Mx * ((K * ey + r) + (int64_t)P.My * (K * ez + c));
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        double x = !(rowv && colv[t]) ? 0.0 : fb ? fb[c * 49 + r * 7 + 2 * q + t] : __ldg(src + row + 2 * q + t);
        if (mask && is_dirichlet(K * ex + 2 * q + t, K * ey + r, K * ez + c, P.Mx, P.My, P.Mz, P.faces)) x = 0.0;
        X[c].v[t] = x;
      }
    }
#pragma unroll
    for (int c = 0; c < 7; ++c) Ep[c] = contract_cols(contract_cols_t(X[c], WB, zero), WB, zero);
  };

  constexpr bool TMA_LIN = MODE == MODE_PAJVP && (NL * 49 * sizeof(double)) % 16 == 0;
  double* const lbuf = q6sm + (size_t)wid * (NL * 343);
  // PAJVP: the element's stored linearisation arrives plane by plane ([l][NL][j][i], 2352 B
  // per point plane at NL = 6) through a ring of 7 plane slots per warp, one mbarrier each:
  // as soon as plane l of this element is consumed, the NEXT element's plane l is issued into
  // the same slot, so every copy has a whole element's time to land (one copy of the whole
  // element after the last plane left the load exposed: C4 jvp_lin kernel ~195 us against
  // ~85 us of HBM and ~82 us of FP64 pipe time)
  constexpr uint32_t PLANE_BYTES = NL * 49 * sizeof(double);
  uint64_t* const lbar = reinterpret_cast<uint64_t*>(q6sm + (size_t)WARPS * (NL * 343)) + 8 * wid;
  uint32_t lphase = 0;
  auto issue_plane = [&](int64_t en, int l) {
    if constexpr (TMA_LIN) {
      if (lane == 0 && en < E) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(lbar + l, PLANE_BYTES);
        mbar_arrive(lbar + l);
        bulk_g2s(lbuf + l * (NL * 49), P.lin + en * (NL * 343) + l * (NL * 49), PLANE_BYTES, lbar + l);
      }
    }
  };
  if constexpr (TMA_LIN) {
    if (lane == 0) {
      for (int l = 0; l < 7; ++l) mbar_init(lbar + l, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    for (int l = 0; l < 7; ++l) issue_plane((int64_t)blockIdx.x * WARPS + wid, l);
  }
  // the next element's input fields: prefetched into L2 right after this element's x-y
  // phase (49 node rows per field); FEOD_Q6_FSTAGE=1 stages them in shared memory by
  // 8-byte cp.async instead (measured slower)
  constexpr bool FSTAGE = FEOD_Q6_FSTAGE && !TMA_LIN;
  constexpr int FB = 344;
  double* const fbuf = q6sm + (size_t)wid * (NIN * FB);
  auto stage_fields = [&](int64_t en) {
    if (en >= E) return;
    int ex, ey, ez;
    q6_coords(P, en, ex, ey, ez);
    const int64_t base = (int64_t)(K * ex) + (int64_t)P.Mx * ((K * ey) + (int64_t)P.My * (K * ez));
    if constexpr (FSTAGE) {
      for (int idx = lane; idx < 343; idx += 32) {
        const int c = idx / 49, rem = idx - 49 * c, y = rem / 7, x = rem - 7 * y;
        const int64_t g = base + x + (int64_t)P.Mx * (y + (int64_t)P.My * c);
#pragma unroll
        for (int f = 0; f < NIN; ++f)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(fbuf + f * FB + idx)),
                       "l"((f == 0 ? in0 : in1) + g)
                       : "memory");
      }
    } else if (lane < 49) {
      const int c = lane / 7, y = lane - 7 * c;
      const int64_t o = base + (int64_t)P.Mx * (y + (int64_t)P.My * c);
      asm volatile("prefetch.global.L2 [%0];" ::"l"(in0 + o));   // (field 1 too: measured no better)
    }
  };
  if constexpr (FSTAGE) {
    stage_fields((int64_t)blockIdx.x * WARPS + wid);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }

  double dacc = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * WARPS + wid; e < E; e += (int64_t)gridDim.x * WARPS) {
    int ex, ey, ez;
    q6_coords(P, e, ex, ey, ez);
    Frag Ep[NIN][7];
    if constexpr (FSTAGE) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncwarp();
    }
    nodes_xy(in0, FSTAGE ? fbuf : nullptr, ex, ey, ez, false, Ep[0]);
    if constexpr (NIN == 2) nodes_xy(in1, FSTAGE ? fbuf + FB : nullptr, ex, ey, ez, MODE == MODE_VJP, Ep[NIN - 1]);
    if constexpr (FSTAGE) __syncwarp();   // buffer consumed
    stage_fields(e + (int64_t)gridDim.x * WARPS);
    if constexpr (FSTAGE) asm volatile("cp.async.commit_group;" ::: "memory");
    const double rho_e = (MODEL == HEAT && MODE != MODE_PAJVP) ? __ldg(P.rho + e) : 1.0;
    double* const linp = (MODE == MODE_LIN || MODE == MODE_PAJVP) ? P.lin + e * (NL * 343) : nullptr;
    if constexpr (MODE == MODE_PAJVP && !TMA_LIN) {
      const int64_t en = e + (int64_t)gridDim.x * WARPS;
      if (lane == 0 && en < E) prefetch_l2_bulk(P.lin + en * (NL * 343), NL * 343 * sizeof(double));
    }
    Frag S[7];
#pragma unroll
    for (int c = 0; c < 7; ++c) S[c] = zero;
    double dz[2] = {0.0, 0.0};   // DOT: sum_l w_l (grad v . F~ + v V~) at the lane's two (i, j)
#pragma unroll
    for (int l = 0; l < 7; ++l) {
      // point plane l of each field: value, collocated x / y derivatives, z derivative
      Frag Ul[NIN], Uxl[NIN], Uyl[NIN], Uzl[NIN];
#pragma unroll
      for (int f = 0; f < NIN; ++f) {
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          double a = T.B[l][0] * Ep[f][0].v[t], b = T.G[l][0] * Ep[f][0].v[t];
#pragma unroll
          for (int c = 1; c < 7; ++c) {
            a = fma(T.B[l][c], Ep[f][c].v[t], a);
            b = fma(T.G[l][c], Ep[f][c].v[t], b);
          }
          Ul[f].v[t] = a;
          Uzl[f].v[t] = b;
        }
        Uyl[f] = contract_cols(Ul[f], WD, zero);                                   // d/dy: [i][j']
        Uxl[f] = contract_cols_t(tr(Ul[f]), WD, zero);     // d/dx: [i'][j]
      }
      Frag Fx, Fy, Fz, V;
      if constexpr (TMA_LIN) mbar_wait(lbar + l, lphase);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int j = 2 * q + t;
        double F0[4] = {0.0, 0.0, 0.0, 0.0}, F1[4];
        if (rowv && colv[t]) {
          const double wq = FOLD ? 1.0 : T.w[r] * T.w[j] * T.w[l];
          const Metric M = {wq * P.cx, wq * P.cy, wq * P.cz, 0.0, 0.0, 0.0};
          const double W = wq * P.vol;
          double u0[NIN], gx[NIN], gy[NIN], gz[NIN];
#pragma unroll
          for (int f = 0; f < NIN; ++f) {
            u0[f] = Ul[f].v[t]; gx[f] = Uxl[f].v[t]; gy[f] = Uyl[f].v[t]; gz[f] = Uzl[f].v[t];
          }
          double sv[MODE == MODE_PAJVP ? NL : 1];
          if constexpr (MODE == MODE_PAJVP) {
#pragma unroll
            for (int c = 0; c < NL; ++c) {
              const int o = (l * NL + c) * 49 + j * 7 + r;
              sv[c] = TMA_LIN ? lbuf[o] : ld_stream(linp + o);
            }
          }
          double gpart = 0.0, lv[NL];
          point_op<MODE, MODEL, true>(u0, gx, gy, gz, M, W, rho_e, P, sv, F0, F1, gpart, lv);
          if constexpr (MODE == MODE_LIN) {
#pragma unroll
            for (int c = 0; c < NL; ++c) linp[(l * NL + c) * 49 + j * 7 + r] = lv[c];
          }
          if constexpr (DOT) {
            constexpr int fv = NIN - 1;   // the direction v: field 1 of the JVP, field 0 of PAJVP
            double dq = fma(F0[0], gx[fv], fma(F0[1], gy[fv], F0[2] * gz[fv]));
            if (value_channel(MODE, 0)) dq = fma(F0[3], u0[fv], dq);
            dz[t] = FOLD ? fma(T.w[l], dq, dz[t]) : dz[t] + dq;   // PAJVP's stored values carry w_q
          }
        }
        Fx.v[t] = F0[0];
        Fy.v[t] = F0[1];
        Fz.v[t] = F0[2];
        V.v[t] = value_channel(MODE, 0) ? F0[3] : 0.0;
      }
      if constexpr (TMA_LIN) {   // plane l's slot is read: refill it with the next element's plane l
        __syncwarp();
        issue_plane(e + (int64_t)gridDim.x * WARPS, l);
      }
      // B^T at plane l: R_l = V + Dx^T Fx + Dy^T Fy, then z into the node-plane accumulators
      Frag R = contract_cols_t(tr(Fx), WDt, V);
      R = contract_cols(Fy, WDt, R);
#pragma unroll
      for (int c = 0; c < 7; ++c)
#pragma unroll
        for (int t = 0; t < 2; ++t)
          S[c].v[t] = FOLD ? fma(T.Bw[l][c], R.v[t], fma(T.Gw[l][c], Fz.v[t], S[c].v[t]))
                           : fma(T.B[l][c], R.v[t], fma(T.G[l][c], Fz.v[t], S[c].v[t]));
    }
    if constexpr (TMA_LIN) lphase ^= 1u;
    const int64_t LXd = 7 * (int64_t)P.nx, LYd = 7 * (int64_t)P.ny;
    double* out = ev + ((int64_t)(7 * ez) * LYd + 7 * ey) * LXd + 7 * ex;
#pragma unroll
    for (int c = 0; c < 7; ++c) {
      const Frag ty = contract_cols_t(S[c], WBt, zero);                    // [b][i]
      const Frag nd = contract_cols(ty, WBt, zero);                        // [b][a]
      if (rowv) {
        double* o = out + ((int64_t)c * LYd + r) * LXd;
#pragma unroll
        for (int t = 0; t < 2; ++t)
          if (colv[t]) o[2 * q + t] = nd.v[t];
      }
    }
    if constexpr (DOT) {
      if (rowv) {
        const double wr = FOLD ? T.w[r] : 1.0;
        if (colv[0]) dacc = fma(FOLD ? wr * T.w[2 * q] : 1.0, dz[0], dacc);
        if (colv[1]) dacc = fma(FOLD ? wr * T.w[2 * q + 1] : 1.0, dz[1], dacc);
      }
    }
  }
  if constexpr (DOT) {   // per-CTA partial in a fixed order (lanes by a butterfly, warps in order); CTA 0 zeroes the tail
    __shared__ double wsum[WARPS];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dacc += __shfl_xor_sync(0xffffffffu, dacc, o);
    if (lane == 0) wsum[wid] = dacc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double sum = 0.0;
      for (int w = 0; w < WARPS; ++w) sum += wsum[w];
      dpart[blockIdx.x] = sum;
    }
    if (blockIdx.x == 0)
      for (int i = gridDim.x + threadIdx.x; i < kRedBlocks; i += blockDim.x) dpart[i] = 0.0;
  }
}

template <int MODE, int MODEL>
static cudaError_t q6tc_launch(const OpParams& P, const Tables& T, const double* in0, const double* in1, double* ev,
                               double* out, const double* dotx, double* dpart, cudaStream_t st, const CgFuse* fuse) {
  constexpr int NL = lin_values(MODEL);
  constexpr bool TMA_LIN = MODE == MODE_PAJVP && (NL * 49 * sizeof(double)) % 16 == 0;
  constexpr size_t smem = TMA_LIN ? (sizeof(double) * NL * 343 + 8 * sizeof(uint64_t)) * q6::WARPS +
                                        (FEOD_Q6_SMT && FEOD_Q6_SMT_PA ? sizeof(double) * q6::WARPS * 1 * 8 * 18 : 0)
                                  : sizeof(double) * q6::WARPS *
                                        ((FEOD_Q6_FSTAGE ? q6_nin<MODE>() * 344 : 0) + (FEOD_Q6_SMT ? 2 * 8 * 18 : 0));
  const void* kfn = (const void*)q6tc_perl_kernel<MODE, MODEL>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int slots = 0;
  if ((e = persistent_slots(kfn, 32 * q6::WARPS, smem, &slots)) != cudaSuccess) return e;
  const int64_t E = (int64_t)P.nx * P.ny * P.nz;
  const int64_t want = (E + q6::WARPS - 1) / q6::WARPS;
  unsigned grid = (unsigned)(want < slots ? want : slots);
  // CgFuse (JVP / stored-linearisation JVP only): the direction p is the v field
  const bool fused = fuse && (MODE == MODE_JVP || MODE == MODE_PAJVP);
  if (fused && grid > (unsigned)kRedBlocks) grid = (unsigned)kRedBlocks;
  if constexpr (MODE == MODE_JVP || MODE == MODE_PAJVP) {
    if (fused) {
      const void* kd = (const void*)q6tc_perl_kernel<MODE, MODEL, true>;
      if ((e = cudaFuncSetAttribute(kd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess) return e;
      q6tc_perl_kernel<MODE, MODEL, true><<<grid, 32 * q6::WARPS, smem, st>>>(P, T, in0, in1, ev, fuse->pAp_part);
    }
  }
  if (!fused) q6tc_perl_kernel<MODE, MODEL><<<grid, 32 * q6::WARPS, smem, st>>>(P, T, in0, in1, ev, nullptr);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  OpParams Pa = P;
  if (MODE == MODE_VJP && P.vjp_keep_rows) Pa.faces = 0;   // J^T w keeps its Dirichlet rows (A17)
  return evec_assemble<q6::K>(Pa, ev, out, dotx, dpart, 0.0, st, fused ? fuse : nullptr);
}

// C4's path: Q6 on affine meshes, the modes above (other modes / perturbed meshes use plane_kernel)
template <int MODE>
static cudaError_t q6tc_mode(int model, const OpParams& P, const Tables& T, const double* in0, const double* in1,
                             double* ev, double* out, const double* dotx, double* dpart, cudaStream_t st,
                             const CgFuse* fuse) {
  switch (model) {
    case PLAPLACE: return q6tc_launch<MODE, PLAPLACE>(P, T, in0, in1, ev, out, dotx, dpart, st, fuse);
    case NLDIFF: return q6tc_launch<MODE, NLDIFF>(P, T, in0, in1, ev, out, dotx, dpart, st, fuse);
    case HEAT: return q6tc_launch<MODE, HEAT>(P, T, in0, in1, ev, out, dotx, dpart, st, fuse);
  }
  return cudaErrorInvalidValue;
}

// MODE_LIN stays on plane_kernel (measured C4: 343 us there, 415 us here -- three dual
// evaluations per point spill at this kernel's 168 registers); both write the same layout
bool q6tc_supports(int mode) {
  return mode == MODE_RES || mode == MODE_JVP || mode == MODE_VJP || mode == MODE_PAJVP;
}

cudaError_t q6tc_run(int mode, int model, const OpParams& P, const Tables& T, const double* in0, const double* in1,
                     double* ev, double* out, const double* dotx, double* dpart, cudaStream_t st, const CgFuse* fuse) {
  switch (mode) {
    case MODE_RES: return q6tc_mode<MODE_RES>(model, P, T, in0, in1, ev, out, dotx, dpart, st, fuse);
    case MODE_JVP: return q6tc_mode<MODE_JVP>(model, P, T, in0, in1, ev, out, dotx, dpart, st, fuse);
    case MODE_VJP: return q6tc_mode<MODE_VJP>(model, P, T, in0, in1, ev, out, dotx, dpart, st, fuse);
    case MODE_LIN: return q6tc_mode<MODE_LIN>(model, P, T, in0, in1, ev, out, dotx, dpart, st, fuse);
    case MODE_PAJVP: return q6tc_mode<MODE_PAJVP>(model, P, T, in0, in1, ev, out, dotx, dpart, st, fuse);
  }
  return cudaErrorInvalidValue;
}


// K12 -- Jacobi diagonal of the stored linearisation at Q6 on the
// FP64 tensor cores: the diagonal of K_e = B^T J_D B at node (a, b, c) is
//   sum_terms w_t sum_{i,j,l} TX_t[i][a] TY_t[j][b] TZ_t[l][c] A_t(i, j, l)
// (the nine terms of diag.cu's header: A_xx G^2 B^2 B^2, ..., 2 A_xy (GB)(GB) B^2, ...,
// b_x (GB) B^2 B^2, ...). One warp per element as in q6tc_perl_kernel: per term and point
// plane l, the y and x contractions of A_t(l) ([i][j] fragment) with the squared / mixed
// tables are two DMMA pairs and a transpose, the z contraction a DFMA accumulation into
// the 7 node-plane fragments. The element diagonals go through the same discontinuous
// L-vector and assembly as the operator (fixed order, no atomics); Dirichlet rows get 1.
template <int NL>
__global__ void __launch_bounds__(32 * q6::WARPS, 3)
q6tc_diag_kernel(const OpParams P, const Tables T, double* __restrict__ ev) {
  using namespace q6;
  constexpr bool TMA = (NL * 49 * sizeof(double)) % 16 == 0;
  constexpr uint32_t PLANE_BYTES = NL * 49 * sizeof(double);
  extern __shared__ __align__(16) double q6sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int r = lane >> 2, q = lane & 3;
  const int64_t E = (int64_t)P.nx * P.ny * P.nz;
  const bool rowv = r < 7;
  const bool colv[2] = {2 * q < 7, 2 * q + 1 < 7};
  const Frag zero = {{0.0, 0.0}};
  // W operands: W[c = point 2q + s][n = node r] of the kind 0: B^2, 1: G^2, 2: G B
  auto tk = [&](int kind, int s) {
    const int c = 2 * q + s, n = r;
    if (c >= 7 || n >= 7) return 0.0;
    const double b = T.B[c][n], g = T.G[c][n];
    return kind == 0 ? b * b : kind == 1 ? g * g : g * b;
  };
  const double W0[2] = {tk(0, 0), tk(0, 1)}, W1[2] = {tk(1, 0), tk(1, 1)}, W2[2] = {tk(2, 0), tk(2, 1)};
  // per term: x table, y table, z table, weight (diag.cu's TX / TY / TZ / WT)
  constexpr int TX[9] = {1, 0, 0, 2, 2, 0, 2, 0, 0};
  constexpr int TY[9] = {0, 1, 0, 2, 0, 2, 0, 2, 0};
  constexpr int TZ[9] = {0, 0, 1, 0, 2, 2, 0, 0, 2};
  // z tables in shared memory (broadcast reads; kept out of registers): zt[kind][l][c]
  double* const zt = q6sm + (TMA ? (size_t)WARPS * (NL * 343) + WARPS * 8 : 0);
  for (int k = threadIdx.x; k < 3 * 49; k += blockDim.x) {
    const int kind = k / 49, l = (k % 49) / 7, c = k % 7;
    const double b = T.B[l][c], g = T.G[l][c];
    zt[k] = kind == 0 ? b * b : kind == 1 ? g * g : g * b;
  }
  __syncthreads();
  // the stored linearisation through the same ring of 7 point-plane slots per warp as
  // q6tc_perl_kernel<MODE_PAJVP>: plane l of the next element is issued as soon as plane l
  // of this one is consumed (the loops run plane-outer, term-inner for that)
  double* const lbuf = q6sm + (size_t)wid * (NL * 343);
  uint64_t* const lbar = reinterpret_cast<uint64_t*>(q6sm + (size_t)WARPS * (NL * 343)) + 8 * wid;
  uint32_t lphase = 0;
  auto issue_plane = [&](int64_t en, int l) {
    if constexpr (TMA) {
      if (lane == 0 && en < E) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(lbar + l, PLANE_BYTES);
        mbar_arrive(lbar + l);
        bulk_g2s(lbuf + l * (NL * 49), P.lin + en * (NL * 343) + l * (NL * 49), PLANE_BYTES, lbar + l);
      }
    }
  };
  if constexpr (TMA) {
    if (lane == 0) {
      for (int l = 0; l < 7; ++l) mbar_init(lbar + l, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    for (int l = 0; l < 7; ++l) issue_plane((int64_t)blockIdx.x * WARPS + wid, l);
  }
  for (int64_t e = (int64_t)blockIdx.x * WARPS + wid; e < E; e += (int64_t)gridDim.x * WARPS) {
    int ex, ey, ez;
    q6_coords(P, e, ex, ey, ez);
    const double* linp = P.lin + e * (NL * 343);
    Frag Dg[7];
#pragma unroll
    for (int c = 0; c < 7; ++c) Dg[c] = zero;
#pragma unroll 1
    for (int l = 0; l < 7; ++l) {
      if constexpr (TMA) mbar_wait(lbar + l, lphase);
      Frag A[NL];
#pragma unroll
      for (int t = 0; t < NL; ++t)
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
          const int o = (l * NL + t) * 49 + (2 * q + s2) * 7 + r;
          A[t].v[s2] = !(rowv && colv[s2]) ? 0.0 : TMA ? lbuf[o] : __ldcs(linp + o);
        }
      if constexpr (TMA) {   // plane l's slot is in registers: refill it with the next element's plane l
        __syncwarp();
        issue_plane(e + (int64_t)gridDim.x * WARPS, l);
      }
#pragma unroll
      for (int t = 0; t < NL; ++t) {
        const int ky = TY[t], kx = TX[t];
        const double* wy = ky == 0 ? W0 : ky == 1 ? W1 : W2;
        const double* wx = kx == 0 ? W0 : kx == 1 ? W1 : W2;
        const double wt = t >= 3 && t < 6 ? 2.0 : 1.0;   // off-diagonal A terms count twice
        const double* ztt = zt + 49 * TZ[t] + l * 7;
        const Frag yb = contract_cols_t(A[t], wy, zero);                     // [b][i]
        Frag ba = contract_cols(yb, wx, zero);                               // [b][a]
        ba.v[0] *= wt;
        ba.v[1] *= wt;
#pragma unroll
        for (int c = 0; c < 7; ++c) {
          const double tz = ztt[c];
#pragma unroll
          for (int s2 = 0; s2 < 2; ++s2) Dg[c].v[s2] = fma(tz, ba.v[s2], Dg[c].v[s2]);
        }
      }
    }
    if constexpr (TMA) lphase ^= 1u;
    const int64_t LXd = 7 * (int64_t)P.nx, LYd = 7 * (int64_t)P.ny;
    double* out = ev + ((int64_t)(7 * ez) * LYd + 7 * ey) * LXd + 7 * ex;
#pragma unroll
    for (int c = 0; c < 7; ++c) {
      if (rowv) {
        double* o = out + ((int64_t)c * LYd + r) * LXd;
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2)
          if (colv[s2]) o[2 * q + s2] = Dg[c].v[s2];
      }
    }
  }
}

template <int NL>
static cudaError_t q6tc_diag_t(const OpParams& P, const Tables& T, double* ev, double* diag, cudaStream_t st) {
  constexpr bool TMA = (NL * 49 * sizeof(double)) % 16 == 0;
  constexpr size_t smem = (TMA ? (sizeof(double) * NL * 343 + 8 * sizeof(uint64_t)) * q6::WARPS : 0) + sizeof(double) * 3 * 49;
  const void* kfn = (const void*)q6tc_diag_kernel<NL>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int slots = 0;
  if ((e = persistent_slots(kfn, 32 * q6::WARPS, smem, &slots)) != cudaSuccess) return e;
  const int64_t E = (int64_t)P.nx * P.ny * P.nz;
  const int64_t want = (E + q6::WARPS - 1) / q6::WARPS;
  q6tc_diag_kernel<NL><<<(unsigned)(want < slots ? want : slots), 32 * q6::WARPS, smem, st>>>(P, T, ev);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return evec_assemble<q6::K>(P, ev, diag, nullptr, nullptr, 1.0, st);   // Dirichlet rows: 1 (the identity there)
}

cudaError_t q6tc_diag(int model, const OpParams& P, const Tables& T, double* ev, double* diag, cudaStream_t st) {
  return lin_values(model) == 9 ? q6tc_diag_t<9>(P, T, ev, diag, st) : q6tc_diag_t<6>(P, T, ev, diag, st);
}

}  // namespace feod
