// Fused FEOD operator kernel: P -> G -> B -> D -> B^T -> G^T -> P^T for one
// brick of hexahedra per CTA (Eq. 1 at :155, Eq. 2 at :160, the
// adjoint load of :199). DESIGN.md §6 is the prose version of this file.
//
// Work decomposition. A CTA owns a BX x BY tile of elements and sweeps BZ
// element layers along z. Each element of the current layer is worked on by
// ND*ND threads arranged as ND lane-groups of ND lanes (a group never straddles
// a warp). A group's role changes with the phase:
//   node phase (B, x-y part)   group = DOF plane c of the element, lane = x-point i:
//       V[b]  = sum_a B[i][a] u[a][b][c]              (x contraction)
//       W[j]  = sum_b B[j][b] V[b],  Wy[j] = sum_b G[j][b] V[b]   (y contraction)
//       -> written once to the element's exchange buffer (2 channels)
//   point phase (B z-part, D, B^T z-part)   group = y-point j, lane = x-point i:
//       U[l] = sum_c B[l][c] W[c],  Uz[l] = sum_c G[l][c] W[c],  Uy[l] = sum_c B[l][c] Wy[c]
//       Ux    = sum_m Dh[i][m] U[m]   (collocated x-derivative: the ND lanes of
//                                      the group hold the x-line; shuffles)
//       D at the point (double or dual<double>), then the transposed chain:
//       Ax = V + sum_m Dh[m][i] Fx[m]  (shuffles), PA[c] += B[l][c] Ax + G[l][c] Fz,
//       PY[c] += B[l][c] Fy           -> written back in place (2 channels)
//   node phase (B^T, x-y part)  group = DOF plane c, lane = x-point i:
//       Q[b] = sum_j B[j][b] PA[j] + G[j][b] PY[j];  r[a][b] = sum_i B[i][a] Q[i][b]
//       (the sum over i is a shuffle reduce-scatter; lane a keeps r[a][.])
//   G^T: every element adds its ND x ND plane results into a shared output ring
//       of DOF planes, four x-y colour classes one after the other (elements of
//       one class share no DOF) -> a fixed summation order, no atomics. Points
//       on a face shared with a neighbouring brick go to this brick's shell
//       slab and are summed by fixup_kernel in a fixed order.
// The DOF planes of u (and v / lambda) stream into a shared ring with cp.async
// one layer ahead; the per-point metric (perturbed meshes) is read from HBM
// straight into registers one point-row ahead, with an L2 bulk prefetch of the
// next layer.
#pragma once
#include "common.cuh"
#include "dual.cuh"
#include "physics.cuh"

namespace feod {

template <int ND> struct PlaneTile;
template <> struct PlaneTile<2> { static constexpr int BX = 8, BY = 8, BZ = 16; };
template <> struct PlaneTile<3> { static constexpr int BX = 4, BY = 4, BZ = 16; };
template <> struct PlaneTile<4> { static constexpr int BX = 4, BY = 4, BZ = 16; };
template <> struct PlaneTile<5> { static constexpr int BX = 4, BY = 2, BZ = 8; };
template <> struct PlaneTile<6> { static constexpr int BX = 2, BY = 2, BZ = 8; };
template <> struct PlaneTile<7> { static constexpr int BX = 2, BY = 2, BZ = 8; };

// ---- compile-time bank-conflict model of the exchange buffer --
// Lane L of warp 0: group g = L / ND, lane-in-group i = L % ND, element e = g / ND,
// role r = g % ND. Element slot stride SE, x-point stride SI, role stride SJ.
//  node-phase 8-byte accesses  addr = e SE + i SI + r          (per half-warp)
//  point-phase 16-byte accesses addr = e SE + i SI + r SJ + 2m (per quarter-warp)
constexpr int xb_cost(int nd, int SI, int SJ, int SE) {
  const int gpw = 32 / nd;
  int cost = 0;
  for (int half = 0; half < 2; ++half) {          // 8-byte: 16 lanes, 16 double-banks
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
  for (int q = 0; q < 4; ++q) {                   // 16-byte: 8 lanes, 8 bank quads
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

constexpr XbPad xb_pad(int nd, int nin) {
  XbPad best{2 * nd, 2 * nd * nd, 2 * nd * nd * nd * nin};
  int bc = 1 << 30;
  for (int si = 2 * nd; si <= 2 * nd + 14; si += 2)
    for (int sj = nd * si; sj <= nd * si + 14; sj += 2)
      for (int pe = 0; pe <= 14; pe += 2) {
        const int se = nin * nd * sj + pe;
        const int c = xb_cost(nd, si, sj, se) * 4096 + se;   // conflicts first, then size
        if (c < bc) { bc = c; best = XbPad{si, sj, se}; }
      }
  return best;
}

// DOF-plane stride of the shared rings: make the ring slots land on different
// bank pairs (stride = 2 mod 16 doubles).
constexpr int plane_pad(int n) { return n + ((2 - n % 16) + 16) % 16; }

template <int ND, int MODE>
struct PShape {
  static constexpr int K = ND - 1;
  static constexpr int BX = PlaneTile<ND>::BX, BY = PlaneTile<ND>::BY, BZ = PlaneTile<ND>::BZ;
  static constexpr int EL = BX * BY;                         // elements per layer
  static constexpr int GPW = 32 / ND;                        // lane groups per warp
  static constexpr int NG = EL * ND;                         // groups in use
  static constexpr int NW = (NG + GPW - 1) / GPW;
  static constexpr int NT = 32 * NW;
  static constexpr bool WARP_ELEM = (32 % (ND * ND)) == 0;   // an element never straddles a warp
  static constexpr int MINB = (512 / NT) < 1 ? 1 : ((512 / NT) > 4 ? 4 : (512 / NT));
  static constexpr int LXF = K * BX + 1, LYF = K * BY + 1;
  static constexpr int PLANE = plane_pad(LXF * LYF);
  static constexpr int RIN = 2 * K + 1;                      // current layer (ND planes) + next layer (K planes)
  static constexpr int ROUT = K + 1;
  static constexpr int NIN = (MODE == MODE_RES) ? 1 : 2;
  static constexpr int NOUT = (MODE == MODE_DESIGN) ? 0 : (MODE == MODE_JVPRES ? 2 : 1);
  static constexpr XbPad XP = xb_pad(ND, NIN);
  static constexpr int SI = XP.SI, SJ = XP.SJ, SE = XP.SE, SF = ND * SJ;
  static constexpr int OUTSZ = (NOUT * ROUT * PLANE + 1) / 2 * 2;
  static constexpr int INSZ = (NIN * RIN * PLANE + 1) / 2 * 2;
  static constexpr int SMEM_DOUBLES = INSZ + OUTSZ + EL * SE;
  static constexpr size_t SMEM_BYTES = sizeof(double) * SMEM_DOUBLES;
  static constexpr int LZF = K * BZ + 1;
  static constexpr int SHELL = LXF * LYF * LZF - (LXF - 2) * (LYF - 2) * (LZF - 2);
  static_assert(SE >= NIN * SF, "exchange slot too small");
};

// 8-byte asynchronous global -> shared copy (LDGSTS). The L-vector row pitch
// 8(kn+1) B is not 16-byte aligned, so TMA tensor maps cannot describe it.
FEOD_DEV void cp_async8(double* smem_dst, const double* gsrc) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gsrc) : "memory");
}
FEOD_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
FEOD_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Streaming metric load that the compiler may not sink toward its use.
FEOD_DEV double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// L2 prefetch of a contiguous byte range (bulk-copy engine; no completion tracking).
FEOD_DEV void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <bool WARP_ELEM>
FEOD_DEV void elem_sync() {
  if constexpr (WARP_ELEM) __syncwarp();
  else __syncthreads();
}

template <int ND>
FEOD_DEV double grp_shfl(double v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

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
  double* ring_out = smem + S::INSZ;        // [NOUT][ROUT][PLANE]
  double* xb = ring_out + S::OUTSZ;         // [EL][SE] exchange slots

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int gw = lane / ND;                          // group within the warp
  const int li = lane - gw * ND;                     // lane within the group: x-point i (or node a)
  const int G = warp * S::GPW + gw;
  const bool lvalid = gw < S::GPW && G < S::NG;      // lane carries real work
  const int Gc = lvalid ? G : 0;
  const int el = Gc / ND;                            // element slot in the layer
  const int gr = Gc - el * ND;                       // group role: plane c / point row j
  const int gbase = lvalid ? lane - li : 0;
  const int lic = lvalid ? li : 0;

  const int brick = blockIdx.x;
  const int bx = brick % P.nbx, by = (brick / P.nbx) % P.nby, bz = brick / (P.nbx * P.nby);
  const int ex0 = bx * S::BX, ey0 = by * S::BY, ez0 = bz * S::BZ;
  const int bxr = min(S::BX, P.nx - ex0), byr = min(S::BY, P.ny - ey0), bzr = min(S::BZ, P.nz - ez0);
  const int LX = K * bxr + 1, LY = K * byr + 1, LZ = K * bzr + 1;
  const int gX0 = K * ex0, gY0 = K * ey0, gZ0 = K * ez0;

  const int exl = el % S::BX, eyl = el / S::BX;
  const bool evalid = lvalid && exl < bxr && eyl < byr;
  const int X0 = evalid ? K * exl : 0, Y0 = evalid ? K * eyl : 0;
  const int colour = (exl & 1) + 2 * (eyl & 1);

  // per-lane rows of the 1D tables (lane i; indices rotated for the shuffles)
  double Brow[ND], Dx[ND], Dt[ND], Bt[ND];
#pragma unroll
  for (int a = 0; a < ND; ++a) Brow[a] = T.B[lic][a];
#pragma unroll
  for (int k = 0; k < ND; ++k) {
    const int up = (lic + k) % ND, dn = (lic - k + ND) % ND;
    Dx[k] = T.D[lic][up];   // all-gather: Ux = sum_k Dx[k] U[(i+k)%ND]
    Dt[k] = T.D[lic][dn];   // reduce-scatter: lane (i-k) receives D[i][i-k] Fx[i]
    Bt[k] = T.B[lic][dn];   // reduce-scatter: lane (i-k) receives B[i][i-k] Q[i][.]
  }
  int src[ND];
#pragma unroll
  for (int k = 0; k < ND; ++k) src[k] = gbase + (lic + k) % ND;

  // ---- G (gather): stream DOF plane p (brick-local z index) into its ring slot
  auto load_plane = [&](int p) {
    const int slot = p % S::RIN;
    const int64_t zoff = (int64_t)P.Mx * P.My * (gZ0 + p);
    for (int idx = tid; idx < S::LXF * S::LYF; idx += S::NT) {
      const int X = idx % S::LXF, Y = idx / S::LXF;
      if (X >= LX || Y >= LY) continue;
      const int64_t g = zoff + (int64_t)(gX0 + X) + (int64_t)P.Mx * (gY0 + Y);
      cp_async8(ring_in + slot * S::PLANE + idx, in0 + g);
      if constexpr (S::NIN == 2) {
        double* dst = ring_in + (S::RIN + slot) * S::PLANE + idx;
        if constexpr (MODE == MODE_DESIGN) {
          // lambda's Dirichlet entries are masked (reading A14)
          *dst = is_dirichlet(gX0 + X, gY0 + Y, gZ0 + p, P.Mx, P.My, P.Mz, P.faces) ? 0.0 : __ldg(in1 + g);
        } else {
          cp_async8(dst, in1 + g);
        }
      }
    }
  };
  for (int p = 0; p <= K; ++p) load_plane(p);
  cp_async_commit();
  if constexpr (S::NOUT > 0)
    for (int i = tid; i < S::NOUT * S::ROUT * S::PLANE; i += S::NT) ring_out[i] = 0.0;

  const bool lowX = ex0 > 0, highX = ex0 + bxr < P.nx;
  const bool lowY = ey0 > 0, highY = ey0 + byr < P.ny;
  const bool lowZ = ez0 > 0, highZ = ez0 + bzr < P.nz;

  // ---- P^T + store of a finished output plane p (brick-local), then clear its slot
  auto flush_plane = [&](int p) {
    const int slot = p % S::ROUT;
    const int64_t zoff = (int64_t)P.Mx * P.My * (gZ0 + p);
    for (int idx = tid; idx < S::LXF * S::LYF; idx += S::NT) {
      const int X = idx % S::LXF, Y = idx / S::LXF;
      if (X >= LX || Y >= LY) continue;
      const bool shared = (X == 0 && lowX) || (X == LX - 1 && highX) || (Y == 0 && lowY) || (Y == LY - 1 && highY) ||
                          (p == 0 && lowZ) || (p == LZ - 1 && highZ);
      const int gx = gX0 + X, gy = gY0 + Y, gz = gZ0 + p;
      const bool dir = is_dirichlet(gx, gy, gz, P.Mx, P.My, P.Mz, P.faces);
      const int64_t g = zoff + (int64_t)gx + (int64_t)P.Mx * gy;
#pragma unroll
      for (int o = 0; o < S::NOUT; ++o) {
        double* cell = ring_out + (o * S::ROUT + slot) * S::PLANE + idx;
        const double v = *cell;
        *cell = 0.0;
        if (shared) {
          (o == 0 ? shell0 : shell1)[(int64_t)brick * P.shell_stride + shell_rank(X, Y, p, LX, LY, LZ)] = v;
        } else {
          (o == 0 ? out0 : out1)[g] = dir ? 0.0 : v;
        }
      }
    }
  };

  double* const xe = xb + el * S::SE;   // this element's exchange slot

  for (int z = 0; z < bzr; ++z) {
    cp_async_wait_all();
    __syncthreads();                                 // planes K z .. K z + K resident; previous layer done
    if (z + 1 < bzr) {
      for (int p = K * (z + 1) + 1; p <= K * (z + 1) + K; ++p) load_plane(p);
      cp_async_commit();
    }
    const int64_t eg = (int64_t)(ex0 + exl) + (int64_t)P.nx * ((ey0 + eyl) + (int64_t)P.ny * (ez0 + z));
    // metric of this thread's points (i = li, j = gr, l): layout [E][l][6][j][i]
    const double* gm = nullptr;
    double mnext[AFFINE ? 1 : 6];
    if constexpr (!AFFINE) {
      gm = P.geom + (evalid ? eg : 0) * (6 * NQ3) + gr * NQ + lic;
#pragma unroll
      for (int c = 0; c < 6; ++c) mnext[c] = ld_stream(gm + c * NQ2);
      if (tid < byr && z + 1 < bzr) {   // L2 prefetch of the next layer's metric, one x-row of elements per y
        const int64_t e1 = (int64_t)ex0 + (int64_t)P.nx * ((ey0 + tid) + (int64_t)P.ny * (ez0 + z + 1));
        prefetch_l2(P.geom + e1 * (6 * NQ3), (uint32_t)(bxr * 6 * NQ3 * sizeof(double)));
      }
    }
    double rho_e = 0.0;
    if constexpr (MODEL == HEAT) rho_e = evalid ? __ldg(P.rho + eg) : 1.0;

    // ---- node phase (B, x and y): group = plane c = gr, lane = x-point i
#pragma unroll
    for (int f = 0; f < S::NIN; ++f) {
      const double* pl = ring_in + (f * S::RIN + (K * z + gr) % S::RIN) * S::PLANE + X0 + S::LXF * Y0;
      double V[ND];
#pragma unroll
      for (int b = 0; b < ND; ++b) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < ND; ++a) acc = fma(Brow[a], pl[a + S::LXF * b], acc);
        V[b] = acc;
      }
      double* xo = xe + f * S::SF + lic * S::SI + gr;
#pragma unroll
      for (int j = 0; j < ND; ++j) {
        double w = 0.0, wy = 0.0;
#pragma unroll
        for (int b = 0; b < ND; ++b) {
          w = fma(T.B[j][b], V[b], w);
          wy = fma(T.G[j][b], V[b], wy);
        }
        if (lvalid) {
          xo[j * S::SJ] = w;
          xo[j * S::SJ + ND] = wy;
        }
      }
    }
    elem_sync<S::WARP_ELEM>();

    // ---- point phase: group = y-point j = gr, lane = x-point i
    double U[S::NIN][NQ], Uz[S::NIN][NQ], Uy[S::NIN][NQ];
#pragma unroll
    for (int f = 0; f < S::NIN; ++f) {
      const double* xi = xe + f * S::SF + gr * S::SJ + lic * S::SI;
      double w[ND], wy[ND];
#pragma unroll
      for (int c = 0; c < ND; c += 2) {
        if (c + 1 < ND) {
          const double2 t0 = *reinterpret_cast<const double2*>(xi + c);
          w[c] = t0.x;
          w[c + 1] = t0.y;
        } else {
          w[c] = xi[c];
        }
      }
#pragma unroll
      for (int c = 0; c < ND; ++c) wy[c] = xi[ND + c];
#pragma unroll
      for (int l = 0; l < NQ; ++l) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
        for (int c = 0; c < ND; ++c) {
          a0 = fma(T.B[l][c], w[c], a0);
          a1 = fma(T.G[l][c], w[c], a1);
          a2 = fma(T.B[l][c], wy[c], a2);
        }
        U[f][l] = a0;
        Uz[f][l] = a1;
        Uy[f][l] = a2;
      }
    }

    double PA[S::NOUT > 0 ? S::NOUT : 1][ND], PY[S::NOUT > 0 ? S::NOUT : 1][ND];
#pragma unroll
    for (int o = 0; o < (S::NOUT > 0 ? S::NOUT : 1); ++o)
#pragma unroll
      for (int c = 0; c < ND; ++c) PA[o][c] = PY[o][c] = 0.0;
    double gpart = 0.0;
    const double wij = T.w[lic] * T.w[gr];
    const double iwij2 = T.wi2[lic] * T.wi2[gr];

#pragma unroll
    for (int l = 0; l < NQ; ++l) {
      // metric of point (i, j, l); request the next row's
      Metric M;
      double W;
      const double wq = wij * T.w[l];
      if constexpr (AFFINE) {
        M = {wq * P.cx, wq * P.cy, wq * P.cz, 0.0, 0.0, 0.0};
        W = wq * P.vol;
      } else {
        M = {mnext[0], mnext[1], mnext[2], mnext[3], mnext[4], mnext[5]};
        if (l + 1 < NQ) {
#pragma unroll
          for (int c = 0; c < 6; ++c) mnext[c] = ld_stream(gm + (l + 1) * 6 * NQ2 + c * NQ2);
        }
        const double det = M.xx * (M.yy * M.zz - M.yz * M.yz) - M.xy * (M.xy * M.zz - M.yz * M.xz) +
                           M.xz * (M.xy * M.yz - M.yy * M.xz);
        W = det * (iwij2 * T.wi2[l]);   // W = w detJ = det(M) / w^2
      }
      // collocated x-derivative over the group's x-line
      double Ux[S::NIN];
#pragma unroll
      for (int f = 0; f < S::NIN; ++f) {
        double ux = Dx[0] * U[f][l];
#pragma unroll
        for (int k = 1; k < ND; ++k) ux = fma(Dx[k], grp_shfl<ND>(U[f][l], src[k]), ux);
        Ux[f] = ux;
      }
      double F0[4], F1[4];   // Fx, Fy, Fz, V of output 0 (and 1)
      if constexpr (MODE == MODE_RES) {
        const double gh[3] = {Ux[0], Uy[0][l], Uz[0][l]};
        double Fh[3];
        flux_hat<MODEL>(U[0][l], gh, M, W, rho_e, P, Fh);
        F0[0] = Fh[0]; F0[1] = Fh[1]; F0[2] = Fh[2];
        F0[3] = -P.f * W;
      } else if constexpr (MODE == MODE_JVP || MODE == MODE_JVPRES) {
        using D = dual<double>;
        const D ud(U[0][l], U[1][l]);
        const D gh[3] = {D(Ux[0], Ux[1]), D(Uy[0][l], Uy[1][l]), D(Uz[0][l], Uz[1][l])};
        D Fh[3];
        flux_hat<MODEL>(ud, gh, M, W, rho_e, P, Fh);
        F0[0] = Fh[0].d; F0[1] = Fh[1].d; F0[2] = Fh[2].d;
        F0[3] = 0.0;
        if constexpr (MODE == MODE_JVPRES) {
          F1[0] = Fh[0].v; F1[1] = Fh[1].v; F1[2] = Fh[2].v;
          F1[3] = -P.f * W;
        }
      } else {   // MODE_DESIGN: seed d/drho; field 1 is lambda
        using D = dual<double>;
        const D ud(U[0][l]);
        const D gh[3] = {D(Ux[0]), D(Uy[0][l]), D(Uz[0][l])};
        const D rd(rho_e, 1.0);
        D Fh[3];
        flux_hat<MODEL>(ud, gh, M, W, rd, P, Fh);
        gpart -= Ux[1] * Fh[0].d + Uy[1][l] * Fh[1].d + Uz[1][l] * Fh[2].d;
      }
      // transposed chain at the point: x (collocated, shuffles) then z
#pragma unroll
      for (int o = 0; o < S::NOUT; ++o) {
        const double* Fo = (o == 0) ? F0 : F1;
        double ax = fma(Dt[0], Fo[0], Fo[3]);
#pragma unroll
        for (int k = 1; k < ND; ++k) ax += grp_shfl<ND>(Dt[k] * Fo[0], src[k]);
#pragma unroll
        for (int c = 0; c < ND; ++c) {
          PA[o][c] = fma(T.B[l][c], ax, fma(T.G[l][c], Fo[2], PA[o][c]));
          PY[o][c] = fma(T.B[l][c], Fo[1], PY[o][c]);
        }
      }
    }

    if constexpr (MODE == MODE_DESIGN) {
      elem_sync<S::WARP_ELEM>();                     // all forward inputs of the element consumed
      if (lvalid) xe[gr * ND + lic] = gpart;
      elem_sync<S::WARP_ELEM>();
      if (evalid && gr == 0 && lic == 0) {
        double s = 0.0;
        for (int t = 0; t < ND * ND; ++t) s += xe[t];
        gout[eg] = s;
      }
    } else {
      // write PA, PY in place of this thread's (consumed) forward inputs
#pragma unroll
      for (int o = 0; o < S::NOUT; ++o) {
        double* xo = xe + o * S::SF + gr * S::SJ + lic * S::SI;
        if (lvalid) {
#pragma unroll
          for (int c = 0; c < ND; c += 2) {
            if (c + 1 < ND) *reinterpret_cast<double2*>(xo + c) = make_double2(PA[o][c], PA[o][c + 1]);
            else xo[c] = PA[o][c];
          }
#pragma unroll
          for (int c = 0; c < ND; ++c) xo[ND + c] = PY[o][c];
        }
      }
      elem_sync<S::WARP_ELEM>();

      // ---- node phase (B^T, y and x): group = plane c = gr, lane = x-point i
      double R[S::NOUT][ND];
#pragma unroll
      for (int o = 0; o < S::NOUT; ++o) {
        const double* xi = xe + o * S::SF + lic * S::SI + gr;
        double Q[ND];
#pragma unroll
        for (int b = 0; b < ND; ++b) Q[b] = 0.0;
#pragma unroll
        for (int j = 0; j < ND; ++j) {
          const double pa = xi[j * S::SJ], py = xi[j * S::SJ + ND];
#pragma unroll
          for (int b = 0; b < ND; ++b) Q[b] = fma(T.B[j][b], pa, fma(T.G[j][b], py, Q[b]));
        }
        // r[a][b] = sum_i B[i][a] Q_i[b]: lane a keeps its row
#pragma unroll
        for (int b = 0; b < ND; ++b) {
          double r = Bt[0] * Q[b];
#pragma unroll
          for (int k = 1; k < ND; ++k) r += grp_shfl<ND>(Bt[k] * Q[b], src[k]);
          R[o][b] = r;
        }
      }
      // ---- G^T into the output ring: four x-y colour classes in turn
      const int slot = (K * z + gr) % S::ROUT;
#pragma unroll
      for (int cls = 0; cls < 4; ++cls) {
        if (cls > 0) __syncthreads();
        if (evalid && colour == cls) {
#pragma unroll
          for (int o = 0; o < S::NOUT; ++o) {
            double* cell = ring_out + (o * S::ROUT + slot) * S::PLANE + (X0 + lic) + S::LXF * Y0;
#pragma unroll
            for (int b = 0; b < ND; ++b) cell[S::LXF * b] += R[o][b];
          }
        }
      }
      __syncthreads();
      // planes K z .. K z + K-1 are complete (the top plane carries into the next layer)
      for (int c = 0; c < K; ++c) flush_plane(K * z + c);
      if (z == bzr - 1) flush_plane(K * z + K);
    }
  }
}

}  // namespace feod
