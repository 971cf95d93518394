// Fused FEOD operator kernel: P -> G -> B -> D -> B^T -> G^T -> P^T for one
// brick of hexahedra per CTA (Eq. 1 at :155, Eq. 2 at :160, the
// adjoint load of :199). DESIGN.md §6 is the prose version of this file.
//
// Warp-specialised z-sweep. A CTA owns a BX x BY tile of elements and sweeps BZ
// element layers along z. It runs NWC compute warps and one IO warp that talk
// only through shared memory and mbarriers (no block-wide barrier in the loop):
//
//   IO warp      streams the DOF planes of u (and v / lambda) into a ring with
//                cp.async, two layers ahead (ring_full / ring_empty); gathers
//                the element results of the previous layer (e_full / e_empty),
//                sums every tile DOF's <= 4 x-y contributions in a fixed order,
//                carries the layer's top DOF plane in registers, applies P^T and
//                stores (owned DOFs to the output, brick-face DOFs to the shell
//                slab summed later by fixup_kernel) -> deterministic, no atomics.
//   compute      each element of the layer is worked on by ND*ND threads, ND
//   warps        lane-groups of ND lanes (a group never straddles a warp); the
//                group's role changes with the phase:
//     node phase (B, x-y)     group = DOF plane c, lane = x-point i:
//        V[b] = sum_a B[i][a] u[a][b][c],  Vx[b] = sum_a G[i][a] u[a][b][c]
//        W[j] = sum_b B[j][b] V[b],  Wy[j] = sum_b G[j][b] V[b],  Wx[j] = sum_b B[j][b] Vx[b]
//        -> the element's exchange slot (3 channels)
//     point phase (B z, D, B^T z)  group = y-point j, lane = x-point i, loop over l:
//        U = sum_c B[l][c] W[c], Uz = sum_c G[l][c] W[c], Ux = .. Wx, Uy = .. Wy
//        D at the point (double or dual<double>), then
//        PX[c] += B[l][c] Fx,  PY[c] += B[l][c] Fy,  PZ[c] += G[l][c] Fz + B[l][c] V
//        -> back into the thread's own slot (3 channels)
//     node phase (B^T, x-y)   group = DOF plane c, lane = x-point i:
//        QX[b] = sum_j B[j][b] PX[j],  QW[b] = sum_j G[j][b] PY[j] + B[j][b] PZ[j]
//        r[a][b] = sum_i G[i][a] QX_i[b] + B[i][a] QW_i[b]  (shuffle reduce-scatter
//        over the group; lane a keeps r[a][.])  -> element buffer for the IO warp
// The per-point metric (perturbed meshes) is read from HBM straight into
// registers one point-row ahead, with an L2 bulk prefetch of the next layer.
#pragma once
#include "common.cuh"
#include "dual.cuh"
#include "physics.cuh"
#include "pointwise.cuh"
#if defined(FEOD_PROFILE_IO) || defined(FEOD_PROFILE_TAIL)
#include <cstdio>
#endif

#ifndef FEOD_J_UNROLL3
#define FEOD_J_UNROLL3 7
#endif
#ifndef FEOD_L_UNROLL3
#define FEOD_L_UNROLL3 1   // point-row loop unroll with 3 exchange channels (Q5/Q6)
#endif
#ifndef FEOD_Q2_LEAN_MORE
#define FEOD_Q2_LEAN_MORE 0
#endif
#ifndef FEOD_PREFETCH
#define FEOD_PREFETCH 1
#endif
#ifndef FEOD_Q3_RES_NCH3
#define FEOD_Q3_RES_NCH3 1   // the Q3 residual with 3 exchange channels (measured 1-2 % faster at full clock)
#endif
#ifndef FEOD_NCH3_MIN
#define FEOD_NCH3_MIN 6   // orders (ND) from which the exchange carries 3 channels
#endif
#ifndef FEOD_PDL_OPERATOR
#define FEOD_PDL_OPERATOR 1
#endif
#ifndef FEOD_MPD
#define FEOD_MPD 0
#endif
#ifndef FEOD_PLANE_VALUE_ALWAYS
#define FEOD_PLANE_VALUE_ALWAYS 1   // the tangent modes' zero value channel kept: dropping it measured
                                    // slower (C3 JVP 247 -> 257 us; schedule, not FLOPs)
#endif
#ifndef FEOD_MINB_OVERRIDE
#define FEOD_MINB_OVERRIDE 0
#endif
namespace feod {

template <int ND> struct PlaneTile;
#ifndef FEOD_Q1_BX
#define FEOD_Q1_BX 8
#endif
#ifndef FEOD_Q1_BY
#define FEOD_Q1_BY 4
#endif
template <> struct PlaneTile<2> { static constexpr int BX = FEOD_Q1_BX, BY = FEOD_Q1_BY, BZ = 16; };
template <> struct PlaneTile<3> { static constexpr int BX = 4, BY = 3, BZ = 16; };
#ifndef FEOD_Q3_BY
#define FEOD_Q3_BY 2
#endif
template <> struct PlaneTile<4> { static constexpr int BX = 4, BY = FEOD_Q3_BY, BZ = 16; };
template <> struct PlaneTile<5> { static constexpr int BX = 4, BY = 2, BZ = 8; };
template <> struct PlaneTile<6> { static constexpr int BX = 2, BY = 2, BZ = 8; };
template <> struct PlaneTile<7> { static constexpr int BX = 2, BY = 2, BZ = 8; };

// ---- compile-time bank-conflict model of the exchange slot ----
// Lane L of warp 0: group g = L / ND, lane-in-group i = L % ND, element e = g / ND,
// role r = g % ND. Element slot stride SE, x-point stride SI, role stride SJ.
//  node-phase 8-byte accesses   addr = e SE + i SI + r          (per half-warp)
//  point-phase 16-byte accesses addr = e SE + i SI + r SJ + 2m  (per quarter-warp)
constexpr int xb_cost(int nd, int SI, int SJ, int SE) {
  const int gpw = (nd * nd <= 32) ? (32 / (nd * nd)) * nd : 32 / nd;   // as PShape::GPW
  int cost = 0;
  for (int half = 0; half < 2; ++half) {
    int cnt[16] = {};
    int seen[16] = {};
    int ns = 0;
    for (int L = 16 * half; L < 16 * half + 16; ++L) {
      const int g = L / nd;
      if (g >= gpw) continue;
      const int i = L % nd, e = g / nd, r = g % nd;
      const int a = e * SE + i * SI + r;
      bool dup = false;
      for (int s = 0; s < ns; ++s) dup = dup || seen[s] == a;
      if (dup) continue;
      seen[ns++] = a;
      cnt[a % 16]++;
    }
    int mx = 0;
    for (int b = 0; b < 16; ++b) mx = cnt[b] > mx ? cnt[b] : mx;
    cost += mx;
  }
  for (int q = 0; q < 4; ++q) {
    int cnt[8] = {};
    for (int L = 8 * q; L < 8 * q + 8; ++L) {
      const int g = L / nd;
      if (g >= gpw) continue;
      const int i = L % nd, e = g / nd, r = g % nd;
      const int a = e * SE + i * SI + r * SJ;
      cnt[(a / 2) % 8]++;
    }
    int mx = 0;
    for (int b = 0; b < 8; ++b) mx = cnt[b] > mx ? cnt[b] : mx;
    cost += mx;
  }
  return cost;
}

struct XbPad { int SI, SJ, SE; };

constexpr XbPad xb_pad(int nd, int nin, int nch) {
  const int s0 = (nch * nd + 1) / 2 * 2;
  XbPad best{s0, s0 * nd, s0 * nd * nd * nin};
  int bc = 1 << 30;
  for (int si = s0; si <= s0 + 14; si += 2)
    for (int sj = nd * si; sj <= nd * si + 14; sj += 2)
      for (int pe = 0; pe <= 14; pe += 2) {
        const int se = nin * nd * sj + pe;
        const int c = xb_cost(nd, si, sj, se) * 4096 + se;   // conflicts first, then size
        if (c < bc) { bc = c; best = XbPad{si, sj, se}; }
      }
  return best;
}

// DOF-plane stride of the input ring: ring slots land on different bank pairs.
constexpr int plane_pad(int n) { return n + ((2 - n % 16) + 16) % 16; }

template <int ND, int MODE>
struct PShape {
  static constexpr int K = ND - 1;
  static constexpr int BX = PlaneTile<ND>::BX, BY = PlaneTile<ND>::BY, BZ = PlaneTile<ND>::BZ;
  static constexpr int EL = BX * BY;                         // elements per layer
  // lane groups per warp: whole elements per warp when an element fits (ND^2 <= 32),
  // so that element-level syncs are warp barriers (Q2: 3 elements on 27 lanes)
  static constexpr int GPW = (ND * ND <= 32) ? (32 / (ND * ND)) * ND : 32 / ND;
  static constexpr int NG = EL * ND;                         // groups in use
  static constexpr int NWC = (NG + GPW - 1) / GPW;           // compute warps
  static constexpr int NTC = 32 * NWC;
  static constexpr int NT = NTC + 32;                        // + the IO warp
  static constexpr bool WARP_ELEM = (GPW % ND) == 0;         // an element never straddles a warp
  // register budget: 128 per thread (occupancy first), except the two-field
  // (tangent) modes of Q5/Q6, whose per-thread state stays in registers (one CTA per SM)
  // Q1 / Q2: 4 CTAs per SM (<= 96 registers, measured: C2 residual -8 %, JVP -4.5 %,
  // C5 JVP -2 %) for the modes that fit without spills
  static constexpr bool LEAN = (ND == 2 && (MODE == MODE_RES || MODE == MODE_JVP || MODE == MODE_JVPRES ||
                                            MODE == MODE_PAJVP)) ||
                               (ND == 3 && (MODE == MODE_JVP || MODE == MODE_JVPRES || MODE == MODE_PAJVP ||
                                            (FEOD_Q2_LEAN_MORE && (MODE == MODE_DESIGN || MODE == MODE_VJP))));
  static constexpr int MINB = FEOD_MINB_OVERRIDE > 0 ? FEOD_MINB_OVERRIDE
                              : (ND >= 6 && (MODE == MODE_JVP || MODE == MODE_JVPRES || MODE == MODE_VJP ||
                                             MODE == MODE_PAJVP))   // PAJVP: C4 jvp_lin 413 -> 358 us
                                    ? 1
                              : LEAN ? 4
                                     : ((65536 / (NT * 128)) < 1 ? 1 : (65536 / (NT * 128)));
  static constexpr int LXF = K * BX + 1, LYF = K * BY + 1;
  static constexpr int NPOS = LXF * LYF;
  static constexpr int PLANE = plane_pad(NPOS);
  static constexpr int RIN = 2 * ND;                         // current layer + next layer (a brick's first layer: ND planes)
  static constexpr int NIN = (MODE == MODE_RES || MODE == MODE_LIN || MODE == MODE_PAJVP) ? 1 : 2;
  static constexpr int NOUT = (MODE == MODE_DESIGN) ? 0 : (MODE == MODE_JVPRES ? 2 : 1);
  // exchange channels: 2 ([W | Wy], x-derivative collocated over the lane group,
  // fewer FLOPs) up to Q4; 3 ([W | Wx | Wy], no cross-lane traffic) for Q5/Q6
  // (Q3 residual: 3 channels measured 1-2 % faster, the Q3 two-field modes 2 channels)
  static constexpr int NCH = (ND >= FEOD_NCH3_MIN || (ND == 4 && MODE == MODE_RES && FEOD_Q3_RES_NCH3)) ? 3 : 2;
  static constexpr XbPad XP = xb_pad(ND, NIN, NCH);
  static constexpr int SI = XP.SI, SJ = XP.SJ, SE = XP.SE, SF = ND * SJ;
  // element buffer (compute -> IO), per layer parity and output: [EL][b][a][c]
  // with the DOF planes c fastest (the IO warp reads a node's ND planes with
  // 16-byte loads); NDP = ND rounded up to even keeps them 16-byte aligned
  static constexpr int NDP = (ND + 1) / 2 * 2;
  static constexpr int EBE = ND * ND * NDP;                  // per element
  static constexpr int EBUF = (NOUT > 0 ? NOUT : 0) * EL * EBE;
  static constexpr int NPIO = (NPOS + 31) / 32;              // tile positions per IO lane
  static constexpr int INSZ = (NIN * RIN * PLANE + 1) / 2 * 2;
  static constexpr int TAB = (4 * ND * ND + 1) / 2 * 2;      // per-lane 1D tables
  static constexpr int SMEM_DOUBLES = INSZ + TAB + EL * SE + 2 * EBUF + 8 + 4;   // + 8 mbarriers + brick queue
  static constexpr size_t SMEM_BYTES = sizeof(double) * SMEM_DOUBLES;
  static constexpr int LZF = K * BZ + 1;
  static constexpr int SHELL = LXF * LYF * LZF - (LXF - 2) * (LYF - 2) * (LZF - 2);
  static_assert(EL * EBE < 65536, "packed 16-bit element-buffer offsets");
};

// ---- async copies and mbarriers (PTX) -----------------------------------------
// 8-byte asynchronous global -> shared copy (LDGSTS). The L-vector row pitch
// 8(kn+1) B is not 16-byte aligned, so TMA tensor maps cannot describe it.
FEOD_DEV void cp_async8(double* smem_dst, const double* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
// arrive on the mbarrier when all prior cp.async of this thread have landed
FEOD_DEV void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// L2 prefetch of a contiguous byte range (bulk-copy engine; no completion tracking).
// The bulk engine needs a 16-byte aligned start and a multiple of 16 bytes: the
// range is widened to that (odd per-element strides, e.g. 9 x 27 doubles, exist).
FEOD_DEV void prefetch_l2(const void* p, uint32_t bytes) {
  const uint64_t a = reinterpret_cast<uint64_t>(p);
  const uint64_t a0 = a & ~uint64_t(15), a1 = (a + bytes + 15) & ~uint64_t(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
}

// Barrier among the compute threads of one element: a warp barrier when an
// element never straddles a warp, else named barrier 1 over all compute warps.
template <bool WARP_ELEM, int NTC>
FEOD_DEV void elem_sync() {
  if constexpr (WARP_ELEM) __syncwarp();
  else asm volatile("bar.sync 1, %0;" ::"n"(NTC) : "memory");
}

FEOD_DEV double grp_shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

// Geometry of brick b: tile origin, ragged extents, DOF box, neighbour flags.
struct Brick {
  int b, ex0, ey0, ez0, bxr, byr, bzr, LX, LY, LZ, gX0, gY0, gZ0;
  bool lowX, highX, lowY, highY, lowZ, highZ;
};
template <int K, int BX, int BY, int BZ>
FEOD_DEV Brick brick_geo(const OpParams& P, int b) {
  Brick g;
  g.b = b;
  const int bx = b % P.nbx, by = (b / P.nbx) % P.nby, bz = b / (P.nbx * P.nby);
  g.ex0 = bx * BX; g.ey0 = by * BY; g.ez0 = bz * BZ;
  g.bxr = min(BX, P.nx - g.ex0); g.byr = min(BY, P.ny - g.ey0); g.bzr = min(BZ, P.nz - g.ez0);
  g.LX = K * g.bxr + 1; g.LY = K * g.byr + 1; g.LZ = K * g.bzr + 1;
  g.gX0 = K * g.ex0; g.gY0 = K * g.ey0; g.gZ0 = K * g.ez0;
  g.lowX = g.ex0 > 0; g.highX = g.ex0 + g.bxr < P.nx;
  g.lowY = g.ey0 > 0; g.highY = g.ey0 + g.byr < P.ny;
  g.lowZ = g.ez0 > 0; g.highZ = g.ez0 + g.bzr < P.nz;
  return g;
}

// Persistent CTAs with dynamic brick scheduling: the IO warp claims bricks from
// a global ticket counter (P.sched) and publishes them in a small shared queue;
// a CTA-global layer counter L drives the mbarrier phases and a CTA-global plane
// counter the input-ring slots, so the IO warp streams the next brick's first
// layers while the compute warps finish the current one. CTAs that run faster
// (the schedulers favour older warps) simply take more bricks.
template <int ND, int MODE, int MODEL, bool AFFINE>
__global__ void __launch_bounds__(PShape<ND, MODE>::NT, PShape<ND, MODE>::MINB)
plane_kernel(const OpParams P, const Tables T, const double* __restrict__ in0, const double* __restrict__ in1,
             double* __restrict__ out0, double* __restrict__ out1, double* __restrict__ shell0,
             double* __restrict__ shell1, double* __restrict__ gout) {
  using S = PShape<ND, MODE>;
  constexpr int K = S::K;
  constexpr int NQ = ND;
  constexpr int NQ2 = NQ * NQ, NQ3 = NQ2 * NQ;
  extern __shared__ __align__(16) double smem[];
  double* ring_in = smem;                   // [NIN][RIN][PLANE]
  double* tab = smem + S::INSZ;             // [4][ND lanes][ND]: Brow, Grow, Bt, Gt
  double* xb = tab + S::TAB;                // [EL][SE] exchange slots (compute warps)
  double* ebuf = xb + S::EL * S::SE;        // [2 parity][NOUT][EL][EBE] element results
  uint64_t* bars = reinterpret_cast<uint64_t*>(ebuf + 2 * S::EBUF);
  uint64_t* ring_full = bars;               // [2] layer z's DOF planes landed      (IO -> compute)
  uint64_t* ring_empty = bars + 2;          // [2] layer z's node phase done         (compute -> IO)
  uint64_t* e_full = bars + 4;              // [2] layer z's element results written (compute -> IO)
  uint64_t* e_empty = bars + 6;             // [2] layer z's element results consumed (IO -> compute)
  int* bq = reinterpret_cast<int*>(bars + 8);   // [8] claimed brick of the CTA's n-th brick (-1: done)

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);   // warp-uniform: lets the compiler keep table constants in uniform registers
  const int nbricks = P.nbx * P.nby * P.nbz;
  const int G = gridDim.x;

  // per-lane rows of the 1D tables (lane i), rotated for the group shuffles:
  //   2 channels: Brow[a] = B[i][a]; Dx[k] = Dh[i][(i+k)%ND] (Ux = sum_k Dx[k] U_{(i+k)%ND});
  //               DxT[k] = Dh[(i+k)%ND][i] (Ax = sum_k DxT[k] Fx_{(i+k)%ND});
  //               Bt[k] = B[i][(i-k)%ND] (reduce-scatter: lane (i-k)%ND receives B[i][i-k] Q_i)
  //   3 channels: Brow[a] = B[i][a]; Grow[a] = G[i][a]; Bt[k] = B[i][(i-k)%ND]; Gt[k] = G[i][(i-k)%ND]
  for (int t = tid; t < ND * ND; t += S::NT) {
    const int i = t / ND, k = t % ND, up = (i + k) % ND, dn = (i - k + ND) % ND;
    tab[t] = T.B[i][k];
    if constexpr (S::NCH == 2) {
      tab[ND * ND + t] = T.D[i][up];
      tab[2 * ND * ND + t] = T.D[up][i];
      tab[3 * ND * ND + t] = T.B[i][dn];
    } else {
      tab[ND * ND + t] = T.G[i][k];
      tab[2 * ND * ND + t] = T.B[i][dn];
      tab[3 * ND * ND + t] = T.G[i][dn];
    }
  }
  if (tid == 0) {
    // ring_full: one cp.async-arrival per IO lane (+ one plain arrival per lane for
    // the synchronously masked lambda of the design mode) + one plain arrival of
    // IO lane 0 that publishes the brick queue
    const uint32_t nfull = (MODE == MODE_DESIGN || MODE == MODE_VJP) ? 65u : 33u;
    mbar_init(&ring_full[0], nfull);
    mbar_init(&ring_full[1], nfull);
    mbar_init(&ring_empty[0], S::NWC);
    mbar_init(&ring_empty[1], S::NWC);
    mbar_init(&e_full[0], S::NWC);
    mbar_init(&e_full[1], S::NWC);
    mbar_init(&e_empty[0], 1);
    mbar_init(&e_empty[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
#if FEOD_PDL_OPERATOR
  // launched as a programmatic dependent of the previous call's fix-up: the table and
  // barrier set-up above overlapped it; nothing global is read before this point
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  // this call's epoch; the fix-up kernel may launch from here on (it waits per brick on P.bdone)
  const unsigned long long epoch = call_begin(P.ds);

  if (warp == S::NWC) {
    // =========================== IO warp ===================================
    // loader cursor (brick lb, layer lz, ring base of the brick) and storer cursor
    // (brick sb, layer sz); tile-plane positions of this lane: idx = lane + 32 m
    Brick gl, gs;
    int lz = 0, sz = 0, lbase = 0, ln = 0, sn = 0;   // loader / storer brick ordinals
    bool ldone = false;
    //   loader:  lpg   in-plane global offset (gX0 + X) + Mx (gY0 + Y); lpinfo bit0 valid, bit2 Dirichlet in x/y
    int lpg[S::NPIO], lpinfo[S::NPIO];
    auto loader_positions = [&]() {
#pragma unroll
      for (int m = 0; m < S::NPIO; ++m) {
        const int idx = lane + 32 * m;
        const int X = idx % S::LXF, Y = idx / S::LXF;
        const bool v = idx < S::NPOS && X < gl.LX && Y < gl.LY;
        const int gx = gl.gX0 + X, gy = gl.gY0 + Y;
        lpg[m] = v ? gx + P.Mx * gy : 0;
        const bool dxy = ((P.faces & 1u) && gx == 0) || ((P.faces & 2u) && gx == P.Mx - 1) ||
                         ((P.faces & 4u) && gy == 0) || ((P.faces & 8u) && gy == P.My - 1);
        lpinfo[m] = (v ? 1 : 0) | (dxy ? 4 : 0);
      }
    };
    //   storer:  pg, pinfo (bit1 on a shared x/y brick face, bits 3.. ring index),
    //            pxy = X + LX Y, pcnt / pofs = element-buffer contributions in a
    //            fixed order, fptr / fstr = affine destination of middle layers
    int pg[S::NPIO], pinfo[S::NPIO], pxy[S::NPIO], pcnt[S::NPIO];
    uint32_t pofs[S::NPIO][2];
    int64_t fptr[S::NOUT > 0 ? S::NOUT : 1][S::NPIO];
    int fstr[S::NPIO];
    double carry[S::NOUT > 0 ? S::NOUT : 1][S::NPIO];
    auto storer_positions = [&]() {
#pragma unroll
      for (int m = 0; m < S::NPIO; ++m) {
        const int idx = lane + 32 * m;
        const int X = idx % S::LXF, Y = idx / S::LXF;
        const bool v = idx < S::NPOS && X < gs.LX && Y < gs.LY;
        const int gx = gs.gX0 + X, gy = gs.gY0 + Y;
        pg[m] = v ? gx + P.Mx * gy : 0;
        const bool shxy = (X == 0 && gs.lowX) || (X == gs.LX - 1 && gs.highX) || (Y == 0 && gs.lowY) ||
                          (Y == gs.LY - 1 && gs.highY);
        const bool dxy = ((P.faces & 1u) && gx == 0) || ((P.faces & 2u) && gx == P.Mx - 1) ||
                         ((P.faces & 4u) && gy == 0) || ((P.faces & 8u) && gy == P.My - 1);
        const int ringpos = (Y == 0) ? X : (Y == gs.LY - 1) ? gs.LX + X : 2 * gs.LX + 2 * (Y - 1) + (X == 0 ? 0 : 1);
        pinfo[m] = (v ? 1 : 0) | (shxy ? 2 : 0) | (dxy ? 4 : 0) | (ringpos << 3);
        pxy[m] = X + gs.LX * Y;
        int cx[2] = {0, 0}, ax[2] = {0, 0}, cy[2] = {0, 0}, ay[2] = {0, 0}, nxc = 1, nyc = 1;
        cx[0] = min(X / K, max(gs.bxr - 1, 0));
        ax[0] = X - K * cx[0];
        if (ax[0] == 0 && cx[0] > 0) { cx[1] = cx[0]; ax[1] = 0; cx[0] -= 1; ax[0] = K; nxc = 2; }
        cy[0] = min(Y / K, max(gs.byr - 1, 0));
        ay[0] = Y - K * cy[0];
        if (ay[0] == 0 && cy[0] > 0) { cy[1] = cy[0]; ay[1] = 0; cy[0] -= 1; ay[0] = K; nyc = 2; }
        uint32_t o4[4] = {0, 0, 0, 0};
        int n = 0;
        for (int t = 0; t < nyc; ++t)
          for (int q = 0; q < nxc; ++q)
            o4[n++] = (uint32_t)((cx[q] + S::BX * cy[t]) * S::EBE + (ay[t] * ND + ax[q]) * S::NDP);
        pofs[m][0] = o4[0] | (o4[1] << 16);
        pofs[m][1] = o4[2] | (o4[3] << 16);
        pcnt[m] = v ? n : 0;
        // middle layers (brick planes 1 .. LZ-2: no bottom/top face, no z-Dirichlet
        // plane) have an affine destination in the plane index p:
        //   shell: brick*stride + base + (p-1)*ring + ringpos      out: Mx*My*(gZ0 + p) + pg
        const int base = gs.LX * gs.LY, ring = 2 * gs.LX + 2 * (gs.LY - 2);
        fstr[m] = shxy ? ring : P.Mx * P.My;
#pragma unroll
        for (int o = 0; o < (S::NOUT > 0 ? S::NOUT : 1); ++o) {
          const double* b0 = shxy ? (o == 0 ? shell0 : shell1) : (o == 0 ? out0 : out1);
          const int64_t off = shxy ? (int64_t)gs.b * P.shell_stride + base - ring + ringpos
                                   : (int64_t)P.Mx * P.My * gs.gZ0 + pg[m];
          fptr[o][m] = reinterpret_cast<int64_t>(b0) + off * (int64_t)sizeof(double);
          carry[o][m] = 0.0;
        }
      }
    };

    // G: stream DOF plane p of the loader brick into its ring slot
    auto load_plane = [&](int p) {
      const int slot = (lbase + p) % S::RIN;
      const int64_t zoff = (int64_t)P.Mx * P.My * (gl.gZ0 + p);
      const bool dz = ((P.faces & 16u) && gl.gZ0 + p == 0) || ((P.faces & 32u) && gl.gZ0 + p == P.Mz - 1);
#pragma unroll
      for (int m = 0; m < S::NPIO; ++m) {
        if (!(lpinfo[m] & 1)) continue;
        const int idx = lane + 32 * m;
        const int64_t g = zoff + lpg[m];
        cp_async8(ring_in + slot * S::PLANE + idx, in0 + g);
        if constexpr (S::NIN == 2) {
          double* dst = ring_in + (S::RIN + slot) * S::PLANE + idx;
          if constexpr (MODE == MODE_DESIGN || MODE == MODE_VJP) {
            // lambda's / w's Dirichlet entries are masked (readings A14, A17): those
            // slots get a plain zero store (published by the lane's plain arrival),
            // the rest stream in with cp.async like every other field
            if ((lpinfo[m] & 4) || dz) *dst = 0.0;
            else cp_async8(dst, in1 + g);
          } else {
            cp_async8(dst, in1 + g);
          }
        }
      }
    };
    // load global layer LL (the loader cursor's next layer) and advance the cursor
    auto load_layer = [&](int LL) {
      uint64_t* bar = &ring_full[LL & 1];
      if (lz == 0) {   // claim the next brick and publish it
        int id = -1;
        if (lane == 0) {
          id = claim_brick(P.ds, nbricks, epoch);
          bq[ln & 7] = id;
        }
        id = __shfl_sync(0xffffffffu, id, 0);
        ++ln;
        if (id < 0) {   // phantom layer: lets the compute warps read the end marker
          ldone = true;
          mbar_arrive(bar);
          if constexpr (MODE == MODE_DESIGN || MODE == MODE_VJP) mbar_arrive(bar);
          if (lane == 0) mbar_arrive(bar);
          return;
        }
        gl = brick_geo<K, S::BX, S::BY, S::BZ>(P, id);
        loader_positions();
      }
      const int p0 = (lz == 0) ? 0 : K * lz + 1;
      for (int p = p0; p <= K * lz + K; ++p) load_plane(p);
      cp_async_arrive(bar);
      if constexpr (MODE == MODE_DESIGN || MODE == MODE_VJP) mbar_arrive(bar);
      if (lane == 0) mbar_arrive(bar);
      if (++lz == gl.bzr) {
        lbase += gl.LZ;
        lz = 0;
      }
    };

    // P^T + store of the finished value v of output o at position m, DOF plane p (general path)
    auto store_dof = [&](int o, int m, int p, double v) {
      const int info = pinfo[m];
      const bool shared = (info & 2) || (p == 0 && gs.lowZ) || (p == gs.LZ - 1 && gs.highZ);
      if (shared) {
        const int base = gs.LX * gs.LY, ring = 2 * gs.LX + 2 * (gs.LY - 2);
        const int rank = (p == 0) ? pxy[m] : (p == gs.LZ - 1) ? base + (gs.LZ - 2) * ring + pxy[m]
                                                               : base + (p - 1) * ring + (info >> 3);
        (o == 0 ? shell0 : shell1)[(int64_t)gs.b * P.shell_stride + rank] = v;
      } else {
        const int gz = gs.gZ0 + p;
        // P^T: Dirichlet rows are zero, except for J^T w, which keeps every row (reading A17)
        const bool dir = !(MODE == MODE_VJP && P.vjp_keep_rows) &&
                         ((info & 4) || ((P.faces & 16u) && gz == 0) || ((P.faces & 32u) && gz == P.Mz - 1));
        (o == 0 ? out0 : out1)[(int64_t)P.Mx * P.My * gz + pg[m]] = dir ? 0.0 : v;
      }
    };

#ifdef FEOD_PROFILE_IO
    long long t_wre = 0, t_load = 0, t_wef = 0, t_gt = 0, t0 = clock64(), t1;
    int nl = 0;
#define FEOD_TICK(acc) do { t1 = clock64(); acc += t1 - t0; t0 = t1; } while (0)
#else
#define FEOD_TICK(acc) do { } while (0)
#endif
    load_layer(0);
    if (!ldone) load_layer(1);
    FEOD_TICK(t_load);
    for (int L = 0;; ++L) {
      if (sz == 0) {   // storer moves to its next brick (claimed by the loader already)
        __syncwarp();
        const int id = __shfl_sync(0xffffffffu, bq[sn & 7], 0);
        ++sn;
        if (id < 0) break;
        gs = brick_geo<K, S::BX, S::BY, S::BZ>(P, id);
        storer_positions();
      }
      if (!ldone) {
        mbar_wait(&ring_empty[L & 1], (L >> 1) & 1);   // compute is done reading layer L's planes
        FEOD_TICK(t_wre);
        load_layer(L + 2);
        FEOD_TICK(t_load);
      }
      if constexpr (S::NOUT > 0) {
        const int z = sz;
        const int bzr = gs.bzr;
        mbar_wait(&e_full[L & 1], (L >> 1) & 1);
        FEOD_TICK(t_wef);
        const double* eb = ebuf + (L & 1) * S::EBUF;
        // G^T: every tile DOF sums its (<= 4) x-y contributions in a fixed order
        // (all ND planes of a contributing node come in 16-byte loads);
        // z-sharing through the carried top plane
#pragma unroll
        for (int m = 0; m < S::NPIO; ++m) {
          const int n = pcnt[m];
          if (n == 0) continue;
          const int off[4] = {(int)(pofs[m][0] & 0xffff), (int)(pofs[m][0] >> 16), (int)(pofs[m][1] & 0xffff),
                              (int)(pofs[m][1] >> 16)};
#pragma unroll
          for (int o = 0; o < S::NOUT; ++o) {
            const double* e = eb + o * S::EL * S::EBE;
            double v[S::NDP];
#pragma unroll
            for (int c = 0; c < S::NDP; c += 2) {
              const double2 t0 = *reinterpret_cast<const double2*>(e + off[0] + c);
              v[c] = t0.x;
              v[c + 1] = t0.y;
            }
#pragma unroll
            for (int t = 1; t < 4; ++t) {
              if (t < n) {
#pragma unroll
                for (int c = 0; c < S::NDP; c += 2) {
                  const double2 t1 = *reinterpret_cast<const double2*>(e + off[t] + c);
                  v[c] += t1.x;
                  v[c + 1] += t1.y;
                }
              }
            }
            v[0] = carry[o][m] + v[0];
            if (z > 0 && z < bzr - 1) {   // middle layer: affine destination, one add per store
              const bool zero = !(MODE == MODE_VJP && P.vjp_keep_rows) && (pinfo[m] & 6) == 4;
              double* d = reinterpret_cast<double*>(fptr[o][m]) + (int64_t)(K * z) * fstr[m];
#pragma unroll
#pragma unroll
              for (int c = 0; c < K; ++c) d[(int64_t)c * fstr[m]] = zero ? 0.0 : v[c];
              carry[o][m] = v[K];
            } else {
#pragma unroll
              for (int c = 0; c < K; ++c) store_dof(o, m, K * z + c, v[c]);
              if (z == bzr - 1) store_dof(o, m, K * z + K, v[K]);
              else carry[o][m] = v[K];
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&e_empty[L & 1]);
        FEOD_TICK(t_gt);
      }
#ifdef FEOD_PROFILE_IO
      ++nl;
#endif
      if (++sz == gs.bzr) {
        sz = 0;
        if constexpr (S::NOUT > 0) {   // brick done: publish its epoch to the fix-up rows that read it
          __syncwarp();
          if (lane == 0) publish_brick(P.bdone, gs.b, epoch + 1);
        }
      }
    }
#ifdef FEOD_PROFILE_IO
    if (lane == 0 && blockIdx.x % 97 == 0 && nl > 0)
      printf("IO blk %d layers %d: wait_ring_empty %lld load %lld wait_e_full %lld gather_store %lld cycles/layer\n", blockIdx.x,
             nl, t_wre / nl, t_load / nl, t_wef / nl, t_gt / nl);
#endif
  } else {

  // ============================== compute warps ==============================
  const int gw = lane / ND;                          // group within the warp
  const int li = lane - gw * ND;                     // lane within the group: x-point i (or node a)
  const int grp = warp * S::GPW + gw;
  const bool lvalid = gw < S::GPW && grp < S::NG;    // lane carries real work
  const int Gc = lvalid ? grp : 0;
  const int el = Gc / ND;                            // element slot in the layer
  const int gr = Gc - el * ND;                       // group role: plane c / point row j
  const int gbase = lvalid ? lane - li : 0;
  const int lic = lvalid ? li : 0;
  const int exl = el % S::BX, eyl = el / S::BX;

  const double* Brow = tab + lic * ND;
  const double* Dx = tab + ND * ND + lic * ND;                                      // 2 channels
  const double* DxT = tab + 2 * ND * ND + lic * ND;                                // 2 channels
  const double* Grow = tab + ND * ND + lic * ND;                                    // 3 channels
  const double* Gt = tab + 3 * ND * ND + lic * ND;                                  // 3 channels
  const double* Bt = tab + (S::NCH == 2 ? 3 : 2) * ND * ND + lic * ND;
  int src[ND];
#pragma unroll
  for (int k = 0; k < ND; ++k) src[k] = gbase + (lic + k) % ND;

  // per-point global stream: the metric (stored-metric meshes) or the stored linearisation (MODE_PAJVP)
  constexpr int NSV = (MODE == MODE_PAJVP) ? lin_values(MODEL) : 6;
  constexpr bool STREAM = (MODE == MODE_PAJVP) || !AFFINE;
  constexpr int MPD = FEOD_MPD > 0 ? FEOD_MPD : (ND == 2 ? 2 : 1);   // point rows of the stream in flight (Q1: 2, measured)
  double* const xe = xb + el * S::SE;   // this element's exchange slot
  // node-phase y loops: rolled with 3 channels when FEOD_J_UNROLL3 says so (code size)
  constexpr int JUNR = S::NCH == 3 ? FEOD_J_UNROLL3 : ND;
  const double wij = T.w[lic] * T.w[gr];
  const double iwij2 = T.wi2[lic] * T.wi2[gr];

#ifdef FEOD_PROFILE_IO
  long long c_wrf = 0, c_wee = 0, c_start = clock64();
  unsigned long long ns_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns_start));
#endif
#ifdef FEOD_PROFILE_TAIL
  unsigned long long tail_t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tail_t0));
#endif
  int L = 0;       // CTA-global layer counter (mbarrier phases, element-buffer parity)
  int rbase = 0;   // CTA-global index of the brick's first DOF plane (input-ring slots)
  for (int n = 0;; ++n) {
  // the first layer of the CTA's n-th brick: its planes (or the end marker) are published
  mbar_wait(&ring_full[L & 1], (L >> 1) & 1);
  const int bid = __shfl_sync(0xffffffffu, bq[n & 7], 0);   // warp-uniform brick id
  if (bid < 0) break;
  const Brick gb = brick_geo<K, S::BX, S::BY, S::BZ>(P, bid);
  const int ex0 = gb.ex0, ey0 = gb.ey0, ez0 = gb.ez0, bxr = gb.bxr, byr = gb.byr, bzr = gb.bzr;
  const bool evalid = lvalid && exl < bxr && eyl < byr;
  const int X0 = evalid ? K * exl : 0, Y0 = evalid ? K * eyl : 0;
  for (int z = 0; z < bzr; ++z, ++L) {
    const int64_t eg = (int64_t)(ex0 + exl) + (int64_t)P.nx * ((ey0 + eyl) + (int64_t)P.ny * (ez0 + z));
    // per-point stream of this thread's points (i = li, j = gr, l), layout [E][l][NSV][j][i]:
    // the metric (NSV = 6) on stored-metric meshes, or the stored linearisation (MODE_PAJVP)
    const double* gm = nullptr;
    double mnext[STREAM ? MPD : 1][STREAM ? NSV : 1];   // rows l .. l+MPD-1 in flight
    if constexpr (STREAM) {
      const double* sb = (MODE == MODE_PAJVP) ? P.lin : P.geom;
      gm = sb + (evalid ? eg : 0) * (NSV * NQ3) + gr * NQ + lic;
#pragma unroll
      for (int r = 0; r < MPD; ++r)
#pragma unroll
        for (int c = 0; c < NSV; ++c) mnext[r][c] = r < NQ ? ld_stream(gm + r * NSV * NQ2 + c * NQ2) : 0.0;
      // L2 prefetch of the stream FEOD_PREFETCH layers ahead (the first layer of a brick
      // also requests the layers in between), one x-row of elements per y
      if (FEOD_PREFETCH > 0 && tid < byr) {
#pragma unroll
        for (int a = (z == 0 ? 1 : FEOD_PREFETCH); a <= FEOD_PREFETCH; ++a) {
          if (z + a < bzr) {
            const int64_t e1 = (int64_t)ex0 + (int64_t)P.nx * ((ey0 + tid) + (int64_t)P.ny * (ez0 + z + a));
            prefetch_l2(sb + e1 * (NSV * NQ3), (uint32_t)(bxr * NSV * NQ3 * sizeof(double)));
          }
        }
      }
    }
    double rho_e = 0.0;
    if constexpr (MODEL == HEAT && MODE != MODE_PAJVP) rho_e = evalid ? __ldg(P.rho + eg) : 1.0;

#ifdef FEOD_PROFILE_IO
    long long c0 = clock64();
#endif
    if (z > 0) mbar_wait(&ring_full[L & 1], (L >> 1) & 1);
#ifdef FEOD_PROFILE_IO
    c_wrf += clock64() - c0;
#endif

    // ---- node phase (B, x and y): group = plane c = gr, lane = x-point i
#pragma unroll
    for (int f = 0; f < S::NIN; ++f) {
      const double* pl = ring_in + (f * S::RIN + (rbase + K * z + gr) % S::RIN) * S::PLANE + X0 + S::LXF * Y0;
      double V[ND], Vx[ND];
#pragma unroll
      for (int b = 0; b < ND; ++b) {
        double acc = 0.0, accx = 0.0;
#pragma unroll
        for (int a = 0; a < ND; ++a) {
          const double ua = pl[a + S::LXF * b];
          acc = fma(Brow[a], ua, acc);
          if constexpr (S::NCH == 3) accx = fma(Grow[a], ua, accx);
        }
        V[b] = acc;
        Vx[b] = accx;
      }
      double* xo = xe + f * S::SF + lic * S::SI + gr;
#pragma unroll(JUNR)
      for (int j = 0; j < ND; ++j) {
        double w = 0.0, wy = 0.0, wx = 0.0;
#pragma unroll
        for (int b = 0; b < ND; ++b) {
          w = fma(T.B[j][b], V[b], w);
          wy = fma(T.G[j][b], V[b], wy);
          if constexpr (S::NCH == 3) wx = fma(T.B[j][b], Vx[b], wx);
        }
        if (lvalid) {   // [W | Wy] or [W | Wy | Wx]
          xo[j * S::SJ] = w;
          xo[j * S::SJ + ND] = wy;
          if constexpr (S::NCH == 3) xo[j * S::SJ + 2 * ND] = wx;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring_empty[L & 1]);   // this warp no longer reads layer L's planes
    elem_sync<S::WARP_ELEM, S::NTC>();

    // ---- point phase: group = y-point j = gr, lane = x-point i; inputs stay in registers
    double w[S::NIN][S::NCH * ND];   // [W | Wy (| Wx)] over c
#pragma unroll
    for (int f = 0; f < S::NIN; ++f) {
      const double* xi = xe + f * S::SF + gr * S::SJ + lic * S::SI;
#pragma unroll
      for (int c = 0; c + 1 < S::NCH * ND; c += 2) {
        const double2 t0 = *reinterpret_cast<const double2*>(xi + c);
        w[f][c] = t0.x;
        w[f][c + 1] = t0.y;
      }
      if constexpr ((S::NCH * ND) % 2) w[f][S::NCH * ND - 1] = xi[S::NCH * ND - 1];
    }
    // values at all z-points of the column, then the collocated x-derivative
    // with one batched all-gather over the group's x-line
    constexpr int NB = S::NCH == 2 ? NQ : 1;   // batched column arrays (2 channels only)
    double U[S::NIN][NB], Ux[S::NIN][NB];
    if constexpr (S::NCH == 2) {
#pragma unroll
      for (int f = 0; f < S::NIN; ++f)
#pragma unroll
        for (int l = 0; l < NQ; ++l) {
          double a0 = 0.0;
#pragma unroll
          for (int c = 0; c < ND; ++c) a0 = fma(T.B[l][c], w[f][c], a0);
          U[f][l] = a0;
        }
#pragma unroll
      for (int f = 0; f < S::NIN; ++f)
#pragma unroll
        for (int l = 0; l < NQ; ++l) {
          double ux = Dx[0] * U[f][l];
#pragma unroll
          for (int k = 1; k < ND; ++k) ux = fma(Dx[k], grp_shfl(U[f][l], src[k]), ux);
          Ux[f][l] = ux;
        }
    }

    constexpr int NO1 = S::NOUT > 0 ? S::NOUT : 1;
    // unroll of the point-row loop: full with 2 channels (l-indexed register arrays);
    // with 3 channels (Q5/Q6) nothing is indexed by l, so it may stay rolled (code size)
    // (measured on C4: rolled, residual -15 %, JVP -8.5 %, linearize -30 %, J^T w -16 %;
    // jvp_lin is faster unrolled)
    constexpr int LUNR = (ND >= 6 && MODE != MODE_PAJVP) ? FEOD_L_UNROLL3 : NQ;   // (not the Q3 residual's 3 channels)
    double PZ[NO1][ND], PY[NO1][ND], FX[NO1][NB], PX[NO1][S::NCH == 3 ? ND : 1];
#pragma unroll
    for (int o = 0; o < NO1; ++o)
#pragma unroll
      for (int c = 0; c < ND; ++c) {
        PZ[o][c] = PY[o][c] = 0.0;
        if constexpr (S::NCH == 3) PX[o][c] = 0.0;
      }
    double gpart = 0.0;

#pragma unroll(LUNR)
    for (int l = 0; l < NQ; ++l) {
      // metric of point (i, j, l); request the next row's
      Metric M;
      double W;
      const double wq = wij * T.w[l];
      double sv[STREAM ? NSV : 1];   // this point's stream values
      if constexpr (STREAM) {
#pragma unroll
        for (int c = 0; c < NSV; ++c) sv[c] = mnext[l % MPD][c];
        if (l + MPD < NQ) {
#pragma unroll
          for (int c = 0; c < NSV; ++c) mnext[l % MPD][c] = ld_stream(gm + (l + MPD) * NSV * NQ2 + c * NQ2);
        }
      }
      if constexpr (AFFINE || MODE == MODE_PAJVP) {
        M = {wq * P.cx, wq * P.cy, wq * P.cz, 0.0, 0.0, 0.0};
        W = wq * P.vol;
      } else {
        M = {sv[0], sv[1], sv[2], sv[3], sv[4], sv[5]};
        const double det = M.xx * (M.yy * M.zz - M.yz * M.yz) - M.xy * (M.xy * M.zz - M.yz * M.xz) +
                           M.xz * (M.xy * M.yz - M.yy * M.xz);
        W = det * (iwij2 * T.wi2[l]);   // W = w detJ = det(M) / w^2
      }
      // z- and y-derivative of row l (3 channels: value and x-derivative too)
      double Ul[S::NIN], Uxl[S::NIN], Uzl[S::NIN], Uyl[S::NIN];
#pragma unroll
      for (int f = 0; f < S::NIN; ++f) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int c = 0; c < ND; ++c) {
          a1 = fma(T.G[l][c], w[f][c], a1);
          a2 = fma(T.B[l][c], w[f][ND + c], a2);
          if constexpr (S::NCH == 3) {
            a0 = fma(T.B[l][c], w[f][c], a0);
            a3 = fma(T.B[l][c], w[f][2 * ND + c], a3);
          }
        }
        Uzl[f] = a1;
        Uyl[f] = a2;
        if constexpr (S::NCH == 3) {
          Ul[f] = a0;
          Uxl[f] = a3;
        } else {
          Ul[f] = U[f][l];
          Uxl[f] = Ux[f][l];
        }
      }
      double F0[4], F1[4];   // Fx, Fy, Fz, V of output 0 (and 1)
      double lv[lin_values(MODEL)];
      point_op<MODE, MODEL, AFFINE || MODE == MODE_PAJVP>(Ul, Uxl, Uyl, Uzl, M, W, rho_e, P, sv, F0, F1, gpart, lv);
      if constexpr (MODE == MODE_LIN) {
        constexpr int NL = lin_values(MODEL);
        if (evalid) {
          double* lp = P.lin + eg * (NL * NQ3) + l * NL * NQ2 + gr * NQ + lic;   // ptx = 1 (plane kernel)
#pragma unroll
          for (int c = 0; c < NL; ++c) lp[c * NQ2] = lv[c];
        }
      }
      // transposed z-contraction of the y, z and value channels at the point;
      // the x channel is kept for the batched transposed x-derivative below
#pragma unroll
      for (int o = 0; o < S::NOUT; ++o) {
        const double* Fo = (o == 0) ? F0 : F1;
        if constexpr (S::NCH == 2) FX[o][l] = Fo[0];
#pragma unroll
        for (int c = 0; c < ND; ++c) {
          if constexpr (S::NCH == 3) PX[o][c] = fma(T.B[l][c], Fo[0], PX[o][c]);
          PY[o][c] = fma(T.B[l][c], Fo[1], PY[o][c]);
          if (FEOD_PLANE_VALUE_ALWAYS || value_channel(MODE, o)) PZ[o][c] = fma(T.G[l][c], Fo[2], fma(T.B[l][c], Fo[3], PZ[o][c]));
          else PZ[o][c] = fma(T.G[l][c], Fo[2], PZ[o][c]);
        }
      }
    }
    // 2 channels: transposed collocated x-derivative (one batched all-gather), then its z-contraction
    if constexpr (S::NCH == 2) {
#pragma unroll
      for (int o = 0; o < S::NOUT; ++o)
#pragma unroll
        for (int l = 0; l < NQ; ++l) {
          double ax = DxT[0] * FX[o][l];
#pragma unroll
          for (int k = 1; k < ND; ++k) ax = fma(DxT[k], grp_shfl(FX[o][l], src[k]), ax);
#pragma unroll
          for (int c = 0; c < ND; ++c) PZ[o][c] = fma(T.B[l][c], ax, PZ[o][c]);
        }
    }

    if constexpr (MODE == MODE_DESIGN) {
      elem_sync<S::WARP_ELEM, S::NTC>();             // all forward inputs of the element consumed
      if (lvalid) xe[gr * ND + lic] = gpart;
      elem_sync<S::WARP_ELEM, S::NTC>();
      if (evalid && gr == 0 && lic == 0) {
        double s = 0.0;
        for (int t = 0; t < ND * ND; ++t) s += xe[t];
        gout[eg] = s;
      }
      elem_sync<S::WARP_ELEM, S::NTC>();             // sums read before the next layer's writes
    } else {
      // write PZ, PY in place of this thread's (consumed) forward inputs
#pragma unroll
      for (int o = 0; o < S::NOUT; ++o) {
        double* xo = xe + o * S::SF + gr * S::SJ + lic * S::SI;
        if (lvalid) {   // [PZ | PY (| PX)]
#pragma unroll
          for (int c = 0; c + 1 < ND; c += 2) {
            *reinterpret_cast<double2*>(xo + c) = make_double2(PZ[o][c], PZ[o][c + 1]);
            *reinterpret_cast<double2*>(xo + ND + c) = make_double2(PY[o][c], PY[o][c + 1]);
            if constexpr (S::NCH == 3)
              *reinterpret_cast<double2*>(xo + 2 * ND + c) = make_double2(PX[o][c], PX[o][c + 1]);
          }
          if constexpr (ND % 2) {
            xo[ND - 1] = PZ[o][ND - 1];
            xo[2 * ND - 1] = PY[o][ND - 1];
            if constexpr (S::NCH == 3) xo[3 * ND - 1] = PX[o][ND - 1];
          }
        }
      }
      elem_sync<S::WARP_ELEM, S::NTC>();

      // ---- node phase (B^T, y and x): group = plane c = gr, lane = x-point i
      double R[S::NOUT][ND];
#pragma unroll
      for (int o = 0; o < S::NOUT; ++o) {
        const double* xi = xe + o * S::SF + lic * S::SI + gr;
        // Q[b] = sum_j B[j][b] PZ[j] + G[j][b] PY[j]  (3 channels: QX[b] = sum_j B[j][b] PX[j] apart)
        double Q[ND], QX[ND];
#pragma unroll
        for (int b = 0; b < ND; ++b) Q[b] = QX[b] = 0.0;
#pragma unroll(JUNR)
        for (int j = 0; j < ND; ++j) {
          const double pz = xi[j * S::SJ], py = xi[j * S::SJ + ND];
#pragma unroll
          for (int b = 0; b < ND; ++b) Q[b] = fma(T.B[j][b], pz, fma(T.G[j][b], py, Q[b]));
          if constexpr (S::NCH == 3) {
            const double px = xi[j * S::SJ + 2 * ND];
#pragma unroll
            for (int b = 0; b < ND; ++b) QX[b] = fma(T.B[j][b], px, QX[b]);
          }
        }
        // r[a][b] = sum_i B[i][a] Q_i[b] (+ G[i][a] QX_i[b]): lane a keeps its row
#pragma unroll
        for (int b = 0; b < ND; ++b) {
          if constexpr (S::NCH == 2) {
            double r = Bt[0] * Q[b];
#pragma unroll
            for (int k = 1; k < ND; ++k) r += grp_shfl(Bt[k] * Q[b], src[k]);
            R[o][b] = r;
          } else {
            double r = fma(Gt[0], QX[b], Bt[0] * Q[b]);
#pragma unroll
            for (int k = 1; k < ND; ++k) r += grp_shfl(fma(Gt[k], QX[b], Bt[k] * Q[b]), src[k]);
            R[o][b] = r;
          }
        }
      }
      // element results -> the IO warp (double-buffered by layer parity)
#ifdef FEOD_PROFILE_IO
      long long c1 = clock64();
#endif
      if (L >= 2) mbar_wait(&e_empty[L & 1], ((L >> 1) - 1) & 1);
#ifdef FEOD_PROFILE_IO
      c_wee += clock64() - c1;
#endif
      double* eb = ebuf + (L & 1) * S::EBUF + el * S::EBE + lic * S::NDP + gr;
      if (lvalid) {
#pragma unroll
        for (int o = 0; o < S::NOUT; ++o)
#pragma unroll
          for (int b = 0; b < ND; ++b) eb[o * S::EL * S::EBE + b * ND * S::NDP] = R[o][b];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&e_full[L & 1]);
      elem_sync<S::WARP_ELEM, S::NTC>();             // P reads done before the next layer's writes
    }
  }
  rbase += gb.LZ;
  }   // bricks
#ifdef FEOD_PROFILE_TAIL
  {
    unsigned long long tail_t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tail_t1));
    if (tid == 0) printf("TAIL %d %llu %d %d %llu %llu\n", MODE, 0ull, blockIdx.x, L, tail_t0, tail_t1);
  }
#endif
#ifdef FEOD_PROFILE_IO
  unsigned long long ns_end;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns_end));
  if (tid == 0 && (blockIdx.x % 97 == 0 || blockIdx.x == gridDim.x - 1) && L > 0)
    printf("CW mode %d blk %d: total %lld wait_ring_full %lld wait_e_empty %lld cycles/layer (%d layers), start %llu end %llu ns, %.1f us, %.0f MHz\n", MODE, blockIdx.x,
           (clock64() - c_start) / L, c_wrf / L, c_wee / L, L, ns_start % 100000000ull, ns_end % 100000000ull, (ns_end - ns_start) * 1e-3,
           (double)(clock64() - c_start) / (double)(ns_end - ns_start) * 1e3);
#endif
  }   // compute warps

}

}  // namespace feod
