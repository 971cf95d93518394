// Fused FEOD operator kernel for low orders (Q1, Q2): one thread per element
// column, the whole sum factorisation of an element in registers.
//
// The chain is the paper's F(u) = P^T G^T B^T D(B G P u) (Eq. 1) and
// its Jacobian action (Eq. 2), with AD confined to the pointwise D
// (pointwise.cuh). At Q1/Q2 an element is small enough (8 / 27 nodes
// and points) that one thread can hold its nodal values, its point values and its
// transposed accumulators in registers, so B and B^T need no shuffles, no shared-
// memory exchange and no barriers: every contraction is a chain of DFMAs with
// compile-time table operands (constant bank). plane_kernel.cuh (Q3..Q6) splits an
// element over ND^2 threads instead; for Q2 that left the FP64 pipe at ~25 %.
//
// CTA = a TX x TY tile of element columns, one thread each, sweeping the brick's
// element layers along z (persistent CTAs, dynamic brick scheduling, DevState).
//   G     the tile's DOF planes (u, and v / lambda / w) stream into a shared ring of
//         RS planes, DPF layers ahead: one TMA bulk copy per tile row, issued by the
//         lanes of warp 0, completion counted on the layer's mbarrier. The L-vector
//         rows are 8 mod 16 bytes apart, so a row is copied from its 16-byte aligned
//         start and stored at an odd virtual pitch VP (Mx odd): element (X, Y) of a
//         plane sits at Y VP + X + s0, s0 the parity of the plane's first row
//         (DESIGN.md §5). One __syncthreads per layer (element buffer, ring reuse).
//   B     per field: x, y, z interpolation to the q^3 Gauss points (B (x) B (x) B),
//         then the reference gradient by collocation, Ux = D_x U etc. (D = L'_m(x_i)
//         on the Gauss points: exact for the degree-k interpolant, q = k+1)
//   D     point_op<MODE, MODEL> at every point (double / dual<double>)
//   B^T   R = D_x^T Fx + D_y^T Fy + D_z^T Fz + V at the points, then z first:
//         S[c] = sum_l B[l][c] R[l]; the element's top plane S[K] is carried in
//         registers to the next layer's element (z-sharing of G^T summed before the
//         x-y transposed contraction, which runs once per shared DOF plane), and
//         the finished planes go through B_y^T B_x^T to the nodes
//   G^T   node values of the finished DOF planes -> shared buffer; after the layer's
//         barrier every thread sums the <= 4 contributions of the nodes it owns in a
//         fixed order (ascending element index) and stores them: interior DOFs to
//         the output (P^T: Dirichlet rows 0), brick-face DOFs to the shell slab that
//         fixup_kernel sums across bricks -> deterministic, no atomics
//   a8    MODE_DESIGN: the element's g_e is one thread's sum, stored directly
// Per-point streams (perturbed-mesh metric, stored linearisation) use the
// interleaved layout OpParams::ptx = TX, so a warp reads 128-byte runs.
#pragma once
#include "common.cuh"
#include "dual.cuh"
#include "physics.cuh"
#include "pointwise.cuh"

namespace feod {

#ifndef FEOD_COL_MINB_Q1
#define FEOD_COL_MINB_Q1 0   // 0: per mode (residual 4 CTAs per SM, the two-field / linearising modes 3)
#endif
#ifndef FEOD_COL_MINB_Q2
#define FEOD_COL_MINB_Q2 2
#endif
#ifndef FEOD_COL_MPD_Q1
#define FEOD_COL_MPD_Q1 0   // Q1: per-point stream loads in flight (points ahead); 0: 3 at 4 CTAs, 4 at 3 CTAs
#endif
#ifndef FEOD_COL_TY_Q2
#define FEOD_COL_TY_Q2 8
#endif
// Tile (TX x TY element columns, one thread each) and resident CTAs per SM by order and
// mode. Q1 (measured on C2): the residual at 4 CTAs per SM (128 registers), the heavier
// modes at 3 (168 registers, no spills; JVP -3 %, J^T w -12 %, linearise -10 %).
template <int ND, int MODE> struct ColTile;
template <int MODE> struct ColTile<2, MODE> {
  static constexpr int TX = 32, TY = 4;
  static constexpr int MINB = FEOD_COL_MINB_Q1 > 0 ? FEOD_COL_MINB_Q1 : (MODE == MODE_RES ? 4 : 3);
  static constexpr int MPD = FEOD_COL_MPD_Q1 > 0 ? FEOD_COL_MPD_Q1 : (MINB >= 4 ? 3 : 4);
};
template <int MODE> struct ColTile<3, MODE> {
  static constexpr int TX = 16, TY = FEOD_COL_TY_Q2, MINB = FEOD_COL_MINB_Q2, MPD = 1;
};

template <int ND, int MODE>
struct CShape {
  static constexpr int K = ND - 1;
  static constexpr int TX = ColTile<ND, MODE>::TX, TY = ColTile<ND, MODE>::TY, NT = TX * TY, NW = NT / 32;
  static constexpr int NIN = (MODE == MODE_RES || MODE == MODE_LIN || MODE == MODE_PAJVP) ? 1 : 2;
  static constexpr int NOUT = (MODE == MODE_DESIGN) ? 0 : (MODE == MODE_JVPRES ? 2 : 1);
  static constexpr int PITCH = (K * TX + 2) / 2 * 2;         // even row pitch (doubles); VP = PITCH + (Mx & 1)
  static constexpr int ROWS = K * TY + 1;
  static constexpr int PLANE = (ROWS * (PITCH + 1) + 2 + 1) / 2 * 2;   // one ring slot (16-byte multiple)
  static constexpr int DPF = 2;                              // layers prefetched ahead
  static constexpr int RS = K * DPF + 2;                     // ring planes (one extra across a brick boundary)
  static constexpr int ESTR = (ND * ND) | 1;                 // odd stride: conflict-free 8-byte accesses
  static constexpr int EBP = NOUT == 2 ? 1 : 2;              // element-buffer parities
  static constexpr int EB = (NOUT > 0 ? NOUT : 0) * (K + 1) * NT * ESTR;   // one parity
  static constexpr int RING = NIN * RS * PLANE;
  // + 2 mbarriers, the brick queue (8 x int4), the plane shifts (NIN x RS ints, padded to 16 B)
  // and the affine metric table (q^3 x 4 doubles)
  static constexpr int PSH = (NIN * RS + 3) / 4 * 4;
  static constexpr size_t SMEM_BYTES =
      sizeof(double) * (RING + EBP * EB) + 16 + 8 * 16 + PSH * 4 + sizeof(double) * 4 * ND * ND * ND;
  static constexpr int MINB = ColTile<ND, MODE>::MINB, MPD = ColTile<ND, MODE>::MPD;
  static_assert(NT % 32 == 0, "whole warps");
};

template <int ND, int MODE, int MODEL, bool AFFINE>
__global__ void __launch_bounds__(CShape<ND, MODE>::NT, CShape<ND, MODE>::MINB)
col_kernel(const OpParams P, const Tables T, const double* __restrict__ in0, const double* __restrict__ in1,
           double* __restrict__ out0, double* __restrict__ out1, double* __restrict__ shell0,
           double* __restrict__ shell1, double* __restrict__ gout) {
  using S = CShape<ND, MODE>;
  constexpr int K = S::K, NQ = ND, NQ2 = NQ * NQ, NQ3 = NQ2 * NQ;
  constexpr int TX = S::TX, TY = S::TY, NT = S::NT, NIN = S::NIN, NOUT = S::NOUT, RS = S::RS;
  constexpr int NO1 = NOUT > 0 ? NOUT : 1;
  constexpr bool STREAM = (MODE == MODE_PAJVP) || !AFFINE;
  constexpr int NSV = (MODE == MODE_PAJVP) ? lin_values(MODEL) : 6;
  constexpr int MID = (NQ % 2 == 1) ? NQ / 2 : -1;   // middle Gauss point (odd q)
  // FOLD (affine meshes, the modes whose outputs are plain B^T of the point fluxes): the
  // weight w_q of M = w_q diag(c) and W = w_q vol is folded into the transposed tables
  // (Tables::Dh, Bw), so the points work with M = diag(c), W = vol -- the p-Laplacian's
  // s = gh.M gh / W is unchanged (w_q cancels), every flux is F = w_q Ft
  constexpr bool FOLD = AFFINE && (MODE == MODE_RES || MODE == MODE_JVP || MODE == MODE_JVPRES || MODE == MODE_VJP);
  constexpr bool MASK1 = MODE == MODE_DESIGN || MODE == MODE_VJP || MODE == MODE_RESDES;   // field 1 (lambda / w) masked
  extern __shared__ __align__(16) double smem[];
  double* ring = smem;                                          // [NIN][RS][PLANE]
  double* ebuf = smem + S::RING;                                // [EBP][NOUT][K+1][NT][ESTR]
  uint64_t* mb = reinterpret_cast<uint64_t*>(ebuf + S::EBP * S::EB);   // [2] layer-slot mbarriers
  int4* bq = reinterpret_cast<int4*>(mb + 2);                   // [8] (id, ex0, ey0, ez0) of the n-th brick
  int* psh = reinterpret_cast<int*>(bq + 8);                    // [NIN][RS] s0 of the plane in each ring slot
  double* wc = reinterpret_cast<double*>(psh + S::PSH);         // [q^3][4] affine metric: w_q (cx, cy, cz, vol)

  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  const int tx = tid % TX, ty = tid / TX;
  const int nbricks = P.nbx * P.nby * P.nbz;
  const int BZ = P.tbz;
  const int64_t MxMy = (int64_t)P.Mx * P.My;
  const int VP = S::PITCH + (P.Mx & 1);   // virtual row pitch of the ring planes
  asm volatile("griddepcontrol.wait;" ::: "memory");   // previous call's results are visible
  // this call's epoch; the fix-up kernel may launch from here on (it waits per brick on P.bdone)
  const unsigned long long epoch = call_begin(P.ds);
  auto claim = [&](int slot) {            // thread 0: claim a brick, publish (id, origin)
    const int id = claim_brick(P.ds, nbricks, epoch);
    int4 q = make_int4(-1, 0, 0, 0);
    if (id >= 0) q = make_int4(id, (id % P.nbx) * TX, ((id / P.nbx) % P.nby) * TY, (id / (P.nbx * P.nby)) * BZ);
    bq[slot & 7] = q;
  };
  if constexpr (AFFINE || MODE == MODE_PAJVP) {
    for (int t = tid; t < NQ3; t += NT) {
      const double wq = T.w[t % NQ] * T.w[(t / NQ) % NQ] * T.w[t / NQ2];
      wc[4 * t + 0] = wq * P.cx;
      wc[4 * t + 1] = wq * P.cy;
      wc[4 * t + 2] = wq * P.cz;
      wc[4 * t + 3] = wq * P.vol;
    }
  }
  if (tid == 0) {
    mbar_init(&mb[0], S::NW);   // one arrival per warp (each issues its share of the row copies)
    mbar_init(&mb[1], S::NW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid == 0) claim(0);
  __syncthreads();

  // ---- prefetch cursor: brick ordinal pn, its queue entry pq, layer pz, CTA-global plane
  // base pbase, layer counter pL. The next brick is claimed only when the cursor has issued
  // the current brick's last layer (late claiming: a CTA never holds a brick it is not about
  // to stream), and read at the next step, after a layer barrier has published it.
  int pn = 0, pz = 0, pbase = 0, pL = 0;
  int4 pq = bq[0];
  bool pend = false;
  auto prefetch = [&]() {
    if (pend) {
      pq = bq[pn & 7];
      pend = false;
    }
    if (pq.x >= 0) {
      const int ex0 = pq.y, ey0 = pq.z, ez0 = pq.w;
      const int LX = K * min(TX, P.nx - ex0) + 1, LY = K * min(TY, P.ny - ey0) + 1;
      const int bzr = min(BZ, P.nz - ez0);
      {
        // one bulk copy per (field, plane, row) of the layer's new planes: warp w takes the
        // (field, plane) pairs w, w + NW, ..., lane = row; every warp's lane 0 arrives
        uint64_t* bar = &mb[pL & 1];
        const int p0 = pz == 0 ? 0 : K * pz + 1, npl = K * pz + K - p0 + 1;
        for (int fp = warp; fp < NIN * npl; fp += S::NW) {
          const int f = fp / npl, p = p0 + fp - f * npl;
          const int slot = (pbase + p) % RS;
          for (int Y = lane; Y < LY; Y += 32) {
            const double* src = (f == 0 ? in0 : in1) + (int64_t)(K * ez0 + p) * MxMy + (int64_t)(K * ey0 + Y) * P.Mx + K * ex0;
            const uint64_t ga = reinterpret_cast<uint64_t>(src);
            const int sh = (int)((ga >> 3) & 1);                            // this row's 8-byte phase
            const int s0 = (int)(((ga >> 3) - (uint64_t)Y * P.Mx) & 1);     // the plane's first row's phase
            if (Y == 0) psh[f * RS + slot] = s0;
            const uint32_t bytes = (uint32_t)(((LX + sh) * 8 + 15) & ~15);
            double* dst = ring + (f * RS + slot) * S::PLANE + (Y * VP + s0 - sh);
            mbar_expect_tx(bar, bytes);
            bulk_g2s(dst, reinterpret_cast<const void*>(ga & ~uint64_t(15)), bytes, bar);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar);
      }
      if constexpr (STREAM) {
        // the layer's per-point stream into L2 (bulk engine), one contiguous chunk per tile row
        const int byr = min(TY, P.ny - ey0);
        if (tid < byr) {
          const double* sb = (MODE == MODE_PAJVP) ? P.lin : P.geom;
          prefetch_l2_bulk(sb + pt_base(P, ex0, ey0 + tid, ez0 + pz, NSV * NQ3),
                           (uint32_t)(sizeof(double) * NSV * NQ3 * TX));
        }
      }
      ++pL;
      if (++pz == bzr) {   // brick issued: claim the next one
        pz = 0;
        pbase += K * bzr + 1;
        ++pn;
        pend = true;
        if (tid == 0) claim(pn);
      }
    }
  };
  static_assert(S::DPF == 2, "two layers in flight: mbarrier slot = layer & 1");
  prefetch();
  __syncthreads();   // a one-layer brick: the next brick written by thread 0 above
  prefetch();

  // ---- compute cursor
  int cn = 0, cz = 0, cbase = 0;
  double rho_nx = 1.0;   // HEAT: rho of this thread's element one layer ahead
  if constexpr (MODEL == HEAT && MODE != MODE_PAJVP) {
    const int4 q0 = bq[0];   // the first layer's element
    if (q0.x >= 0 && q0.y + tx < P.nx && q0.z + ty < P.ny)
      rho_nx = ld_stream(P.rho + (q0.y + tx) + (int64_t)P.nx * ((q0.z + ty) + (int64_t)P.ny * q0.w));
  }

#pragma unroll 1
  for (int L = 0;; ++L) {
    const int4 cq = bq[cn & 7];
    const int cid = cq.x;
    if (cid < 0) break;
    const int ex0 = cq.y, ey0 = cq.z, ez0 = cq.w;
    const int bxr = min(TX, P.nx - ex0), byr = min(TY, P.ny - ey0), bzr = min(BZ, P.nz - ez0);
    const bool ev = tx < bxr && ty < byr;
    const bool last = cz == bzr - 1;
    const int ex = ex0 + tx, ey = ey0 + ty, ez = ez0 + cz;
    double rho_e = 1.0;
    if constexpr (MODEL == HEAT && MODE != MODE_PAJVP) {
      // rho one layer ahead: this layer's value came with the previous layer; request the next
      // layer's (the next brick's first layer is claimed by now: the prefetch cursor is ahead)
      rho_e = rho_nx;   // (no predicated load into rho_e: its scoreboard would stall the first use)
      int4 nq = cq;
      int nz_ = cz + 1;
      if (nz_ == bzr) { nq = bq[(cn + 1) & 7]; nz_ = 0; }
      if (nq.x >= 0 && nq.y + tx < P.nx && nq.z + ty < P.ny && nq.w + nz_ < P.nz)
        rho_nx = ld_stream(P.rho + (nq.y + tx) + (int64_t)P.nx * ((nq.z + ty) + (int64_t)P.ny * (nq.w + nz_)));
    }
    double* eb = ebuf + (S::EBP == 2 ? (L & 1) : 0) * S::EB;
    if (S::EBP == 1 && NOUT > 0) __syncthreads();   // single element buffer: previous scatter done
    mbar_wait(&mb[L & 1], (L >> 1) & 1);             // this layer's DOF planes landed

    if (ev) {
      // ---- gather the element's nodes from the ring; B: values at the q^3 points
      double U[NIN][NQ3];
#pragma unroll
      for (int f = 0; f < NIN; ++f) {
        double x[ND][ND][ND];   // [c][b][a]
#pragma unroll
        for (int c = 0; c < ND; ++c) {
          const int slot = (cbase + K * cz + c) % RS;
          const double* pl = ring + (f * RS + slot) * S::PLANE + psh[f * RS + slot] + K * ty * VP + K * tx;
#pragma unroll
          for (int b = 0; b < ND; ++b)
#pragma unroll
            for (int a = 0; a < ND; ++a) x[c][b][a] = pl[b * VP + a];
        }
        if (MASK1 && f == 1) {
          // lambda's / w's Dirichlet entries are masked (readings A14, A17): only elements
          // touching a Dirichlet face look at their nodes
          const bool touch = ((P.faces & 1u) && ex == 0) || ((P.faces & 2u) && ex == P.nx - 1) ||
                             ((P.faces & 4u) && ey == 0) || ((P.faces & 8u) && ey == P.ny - 1) ||
                             ((P.faces & 16u) && ez == 0) || ((P.faces & 32u) && ez == P.nz - 1);
          if (touch) {
#pragma unroll
            for (int c = 0; c < ND; ++c)
#pragma unroll
              for (int b = 0; b < ND; ++b)
#pragma unroll
                for (int a = 0; a < ND; ++a)
                  if (is_dirichlet(K * ex + a, K * ey + b, K * ez + c, P.Mx, P.My, P.Mz, P.faces)) x[c][b][a] = 0.0;
          }
        }
        double t1[ND][ND][NQ];   // x: [c][b][i]
#pragma unroll
        for (int c = 0; c < ND; ++c)
#pragma unroll
          for (int b = 0; b < ND; ++b)
#pragma unroll
            for (int i = 0; i < NQ; ++i) {
              double s = T.B[i][0] * x[c][b][0];
#pragma unroll
              for (int a = 1; a < ND; ++a) s = fma(T.B[i][a], x[c][b][a], s);
              t1[c][b][i] = s;
            }
        double t2[ND][NQ][NQ];   // y: [c][j][i]
#pragma unroll
        for (int c = 0; c < ND; ++c)
#pragma unroll
          for (int j = 0; j < NQ; ++j)
#pragma unroll
            for (int i = 0; i < NQ; ++i) {
              double s = T.B[j][0] * t1[c][0][i];
#pragma unroll
              for (int b = 1; b < ND; ++b) s = fma(T.B[j][b], t1[c][b][i], s);
              t2[c][j][i] = s;
            }
#pragma unroll
        for (int l = 0; l < NQ; ++l)   // z: [l][j][i]
#pragma unroll
          for (int ji = 0; ji < NQ2; ++ji) {
            double s = T.B[l][0] * t2[0][ji / NQ][ji % NQ];
#pragma unroll
            for (int c = 1; c < ND; ++c) s = fma(T.B[l][c], t2[c][ji / NQ][ji % NQ], s);
            U[f][l * NQ2 + ji] = s;
          }
      }

      // ---- D at every point, B^T's collocated part accumulated in R
      double R[NO1][NQ3];
#pragma unroll
      for (int o = 0; o < NO1; ++o)
#pragma unroll
        for (int t = 0; t < NQ3; ++t) R[o][t] = 0.0;
      double gpart = 0.0;
      const double* gp = nullptr;   // this element's per-point stream (stride TX = ptx)
      if constexpr (STREAM) {
        const double* sb = (MODE == MODE_PAJVP) ? P.lin : P.geom;
        gp = sb + pt_base(P, ex, ey, ez, NSV * NQ3);
      }
      double* lp = nullptr;
      if constexpr (MODE == MODE_LIN) lp = P.lin + pt_base(P, ex, ey, ez, lin_values(MODEL) * NQ3);
      // the point stream, MPD points ahead in registers (streaming loads, L2-prefetched a
      // brick step earlier)
      constexpr int MPD = S::MPD;
      double snext[STREAM ? MPD : 1][STREAM ? NSV : 1];
      if constexpr (STREAM) {
#pragma unroll
        for (int r = 0; r < MPD; ++r)
#pragma unroll
          for (int c = 0; c < NSV; ++c)
            snext[r][c] = ld_stream(gp + (((r / NQ2) * NSV + c) * NQ2 + r % NQ2) * TX);
      }
#pragma unroll
      for (int l = 0; l < NQ; ++l)
#pragma unroll
        for (int j = 0; j < NQ; ++j)
#pragma unroll
          for (int i = 0; i < NQ; ++i) {
            const int q = (l * NQ + j) * NQ + i;
            double sv[STREAM ? NSV : 1];
            if constexpr (STREAM) {
              // layout [l][c][j][i] per element (as the geometry kernel writes it)
#pragma unroll
              for (int c = 0; c < NSV; ++c) sv[c] = snext[q % MPD][c];
              if (q + MPD < NQ3) {
                const int l1 = (q + MPD) / NQ2, ji1 = (q + MPD) % NQ2;
#pragma unroll
                for (int c = 0; c < NSV; ++c) snext[q % MPD][c] = ld_stream(gp + ((l1 * NSV + c) * NQ2 + ji1) * TX);
              }
            }
            Metric M;
            double W;
            if constexpr (FOLD) {
              M = {P.cx, P.cy, P.cz, 0.0, 0.0, 0.0};
              W = P.vol;
            } else if constexpr (AFFINE || MODE == MODE_PAJVP) {
              const double2 m01 = *reinterpret_cast<const double2*>(wc + 4 * q);
              const double2 m23 = *reinterpret_cast<const double2*>(wc + 4 * q + 2);
              M = {m01.x, m01.y, m23.x, 0.0, 0.0, 0.0};
              W = m23.y;
            } else {
              M = {sv[0], sv[1], sv[2], sv[3], sv[4], sv[5]};
              const double det = M.xx * (M.yy * M.zz - M.yz * M.yz) - M.xy * (M.xy * M.zz - M.yz * M.xz) +
                                 M.xz * (M.xy * M.yz - M.yy * M.xz);
              W = det * (T.wi2[i] * T.wi2[j] * T.wi2[l]);   // W = w detJ = det(M) / w^2
            }
            double Ul[NIN], Uxl[NIN], Uyl[NIN], Uzl[NIN];
#pragma unroll
            for (int f = 0; f < NIN; ++f) {
              Ul[f] = U[f][q];
              double gx = T.D[i][0] * U[f][(l * NQ + j) * NQ];
              double gy = T.D[j][0] * U[f][l * NQ2 + i];
              double gz = T.D[l][0] * U[f][j * NQ + i];
#pragma unroll
              for (int m = 1; m < NQ; ++m) {
                // D[mid][mid] = 0 on the symmetric Gauss points (odd q; set exactly at create)
                if (!(i == MID && m == MID)) gx = fma(T.D[i][m], U[f][(l * NQ + j) * NQ + m], gx);
                if (!(j == MID && m == MID)) gy = fma(T.D[j][m], U[f][(l * NQ + m) * NQ + i], gy);
                if (!(l == MID && m == MID)) gz = fma(T.D[l][m], U[f][(m * NQ + j) * NQ + i], gz);
              }
              Uxl[f] = gx;
              Uyl[f] = gy;
              Uzl[f] = gz;
            }
            double F0[4], F1[4];
            double lv[lin_values(MODEL)];
            point_op<MODE, MODEL, AFFINE || MODE == MODE_PAJVP>(Ul, Uxl, Uyl, Uzl, M, W, rho_e, P, sv, F0, F1, gpart, lv);
            if constexpr (MODE == MODE_LIN) {
#pragma unroll
              for (int c = 0; c < lin_values(MODEL); ++c) lp[((l * lin_values(MODEL) + c) * NQ2 + j * NQ + i) * TX] = lv[c];
            }
#pragma unroll
            for (int o = 0; o < NOUT; ++o) {
              const double* Fo = o == 0 ? F0 : F1;
              if (value_channel(MODE, o)) R[o][q] += Fo[3];
#pragma unroll
              for (int m = 0; m < NQ; ++m) {
                const auto& DT = FOLD ? T.Dh : T.D;
                if (!(i == MID && m == MID)) R[o][(l * NQ + j) * NQ + m] = fma(DT[i][m], Fo[0], R[o][(l * NQ + j) * NQ + m]);
                if (!(j == MID && m == MID)) R[o][(l * NQ + m) * NQ + i] = fma(DT[j][m], Fo[1], R[o][(l * NQ + m) * NQ + i]);
                if (!(l == MID && m == MID)) R[o][(m * NQ + j) * NQ + i] = fma(DT[l][m], Fo[2], R[o][(m * NQ + j) * NQ + i]);
              }
            }
          }
      if constexpr (MODE == MODE_DESIGN || MODE == MODE_RESDES) gout[ex + (int64_t)P.nx * (ey + (int64_t)P.ny * ez)] = gpart;

      // ---- B^T: z first, z-carry of the top plane, then y and x per finished DOF plane
#pragma unroll
      for (int o = 0; o < NOUT; ++o) {
        double Sz[ND][NQ2];
#pragma unroll
        for (int c = 0; c < ND; ++c)
#pragma unroll
          for (int ji = 0; ji < NQ2; ++ji) {
            const auto& BT = FOLD ? T.Bw : T.B;
            double s = BT[0][c] * R[o][ji];
#pragma unroll
            for (int l = 1; l < NQ; ++l) s = fma(BT[l][c], R[o][l * NQ2 + ji], s);
            Sz[c][ji] = s;
          }
        // z-carry of the column's top plane (after B_z^T, before B_y^T B_x^T), parked in the
        // element buffer's plane-K slot of the layer's parity, which only the brick's last
        // layer uses for nodes: read from the previous layer's slot, written to this one's
        if (cz > 0) {
          const double* cp = ebuf + (S::EBP == 2 ? ((L - 1) & 1) : 0) * S::EB + ((o * (K + 1) + K) * NT + tid) * S::ESTR;
#pragma unroll
          for (int ji = 0; ji < NQ2; ++ji) Sz[0][ji] = cp[ji] + Sz[0][ji];
        }
        if (!last) {
          double* cp = eb + ((o * (K + 1) + K) * NT + tid) * S::ESTR;
#pragma unroll
          for (int ji = 0; ji < NQ2; ++ji) cp[ji] = Sz[K][ji];
        }
#pragma unroll
        for (int c = 0; c < ND; ++c) {
          if (c == K && !last) break;
          double sy[ND][NQ];   // [b][i]
#pragma unroll
          for (int b = 0; b < ND; ++b)
#pragma unroll
            for (int i = 0; i < NQ; ++i) {
              const auto& BT = FOLD ? T.Bw : T.B;
              double s = BT[0][b] * Sz[c][i];
#pragma unroll
              for (int j = 1; j < NQ; ++j) s = fma(BT[j][b], Sz[c][j * NQ + i], s);
              sy[b][i] = s;
            }
          double* e = eb + ((o * (K + 1) + c) * NT + tid) * S::ESTR;
#pragma unroll
          for (int b = 0; b < ND; ++b)
#pragma unroll
            for (int a = 0; a < ND; ++a) {
              const auto& BT = FOLD ? T.Bw : T.B;
              double s = BT[0][a] * sy[b][0];
#pragma unroll
              for (int i = 1; i < NQ; ++i) s = fma(BT[i][a], sy[b][i], s);
              e[b * ND + a] = s;
            }
        }
      }
    }
    __syncthreads();

    // ---- G^T + P^T: the finished DOF planes of the layer, each node's <= 4 contributions
    // summed in ascending element order (ty-1, tx-1), (ty-1, tx), (ty, tx-1), (ty, tx).
    //  main pass      thread (tx, ty) owns its element's nodes a, b < K that are not on the
    //                 tile plane's perimeter: never on an x / y brick face or Dirichlet face,
    //                 so only the plane decides the destination (output row, the shell's
    //                 z-face plane at rank X + LX Y, or a Dirichlet zero)
    //  perimeter      thread p < 2(LX + LY) - 4 owns perimeter node p in the shell's ring
    //  pass           order (row Y = 0, row Y = LY-1, then (X = 0, X = LX-1) per middle row)
    if constexpr (NOUT > 0) {
      const int LX = K * bxr + 1, LY = K * byr + 1, LZ = K * bzr + 1;
      const bool lowZ = ez0 > 0, highZ = ez0 + bzr < P.nz;
      const bool keep = MODE == MODE_VJP && P.vjp_keep_rows;   // J^T w keeps every row (reading A17)
      const int nfp = last ? K + 1 : K;
      const int ring_len = 2 * LX + 2 * (LY - 2);
      const int np = 2 * (LX + LY) - 4;   // perimeter nodes
#pragma unroll
      for (int c = 0; c < K + 1; ++c) {
        if (c >= nfp) break;
        const int lz = K * cz + c;
        const int gz = K * ez0 + lz;
        const bool zlo = lz == 0 && lowZ, zhi = lz == LZ - 1 && highZ;
        const bool zdir = !keep && (((P.faces & 16u) && gz == 0) || ((P.faces & 32u) && gz == P.Mz - 1));
        // z-face planes go to the shell whole: rank X + LX Y (+ the top plane's offset)
        const int64_t zsh_off = (int64_t)cid * P.shell_stride + (zhi ? LX * LY + (LZ - 2) * ring_len : 0);
#pragma unroll
        for (int o = 0; o < NOUT; ++o) {
          const double* e = eb + (o * (K + 1) + c) * NT * S::ESTR;
          double* outo = o == 0 ? out0 : out1;
          double* sho = o == 0 ? shell0 : shell1;
          if (ev) {
#pragma unroll
            for (int b = 0; b < K; ++b)
#pragma unroll
              for (int a = 0; a < K; ++a) {
                if ((a == 0 && tx == 0) || (b == 0 && ty == 0)) continue;   // perimeter node
                double v = 0.0;
                if (b == 0) {
                  if (a == 0) v += e[(tid - TX - 1) * S::ESTR + K * ND + K];
                  v += e[(tid - TX) * S::ESTR + K * ND + a];
                }
                if (a == 0) v += e[(tid - 1) * S::ESTR + b * ND + K];
                v += e[tid * S::ESTR + b * ND + a];
                const int X = K * tx + a, Y = K * ty + b;
                if (zlo || zhi) sho[zsh_off + X + LX * Y] = v;
                else outo[(int64_t)gz * MxMy + (int64_t)(K * ey0 + Y) * P.Mx + K * ex0 + X] = zdir ? 0.0 : v;
              }
          }
          // perimeter pass: threads rotated by a warp per plane, so that every warp gets a share
          for (int pp = (tid + NT - 32 * ((c + o) % S::NW)) % NT; pp < np; pp += NT) {
            int X, Y;
            if (pp < LX) { X = pp; Y = 0; }
            else if (pp < 2 * LX) { X = pp - LX; Y = LY - 1; }
            else { const int r = pp - 2 * LX; Y = 1 + (r >> 1); X = (r & 1) ? LX - 1 : 0; }
            // contributing elements along x and y (the low one first), and local node indices
            const int cx1 = min(X / K, bxr - 1), cy1 = min(Y / K, byr - 1);
            const int ax1 = X - K * cx1, ay1 = Y - K * cy1;
            const bool two_x = ax1 == 0 && cx1 > 0, two_y = ay1 == 0 && cy1 > 0;
            double v = 0.0;
            if (two_y) {
              if (two_x) v += e[((cy1 - 1) * TX + cx1 - 1) * S::ESTR + K * ND + K];
              v += e[((cy1 - 1) * TX + cx1) * S::ESTR + K * ND + ax1];
            }
            if (two_x) v += e[(cy1 * TX + cx1 - 1) * S::ESTR + ay1 * ND + K];
            v += e[(cy1 * TX + cx1) * S::ESTR + ay1 * ND + ax1];
            const bool xyface = (X == 0 && ex0 > 0) || (X == LX - 1 && ex0 + bxr < P.nx) || (Y == 0 && ey0 > 0) ||
                                (Y == LY - 1 && ey0 + byr < P.ny);
            if (zlo || zhi) {
              sho[zsh_off + X + LX * Y] = v;
            } else if (xyface) {   // common.cuh shell_rank: the ring (rank pp) on middle planes
              const int rk = lz == 0 ? X + LX * Y
                             : lz == LZ - 1 ? LX * LY + (LZ - 2) * ring_len + X + LX * Y
                                            : LX * LY + (lz - 1) * ring_len + pp;
              sho[(int64_t)cid * P.shell_stride + rk] = v;
            } else {
              const int gx = K * ex0 + X, gy = K * ey0 + Y;
              const bool dir = zdir || (!keep && (((P.faces & 1u) && gx == 0) || ((P.faces & 2u) && gx == P.Mx - 1) ||
                                                  ((P.faces & 4u) && gy == 0) || ((P.faces & 8u) && gy == P.My - 1)));
              outo[(int64_t)gz * MxMy + (int64_t)gy * P.Mx + gx] = dir ? 0.0 : v;
            }
          }
        }
      }
      if (last) {   // brick done: publish its epoch to the fix-up rows that read it
        __syncthreads();
        if (tid == 0) publish_brick(P.bdone, cid, epoch + 1);
      }
    }

    prefetch();
    if (++cz == bzr) {
      cz = 0;
      cbase += K * bzr + 1;
      ++cn;
    }
  }
}

}  // namespace feod
