// Fused FEOD operator kernel: G -> B -> D -> B^T -> G^T (-> P^T) for one brick
// of hexahedra per CTA (PAPER.md:25, Eq. 1 :155, Eq. 2 :160, :199).
//
// Structure:
//  1. the brick's DOF box of each input vector is staged in shared memory
//     (row-contiguous loads; lambda's Dirichlet entries masked for DESIGN);
//  2. elements are processed EB at a time, NQ*NQ threads per element, each
//     thread owning one 1D line of the element; sum factorisation (operator B)
//     runs as three 1D contractions z -> y -> x in registers, with the line
//     ownership rotated through a per-element scratch in shared memory;
//     1D tables B, G come from the kernel-parameter (constant) bank;
//  3. the pointwise flux D runs on the x-line of points each thread owns, as
//     double (residual) or dual<double> (JVP / design derivative);
//  4. B^T runs the same contractions transposed (x -> y -> z) and each element
//     writes its element vector to a shared-memory E-buffer;
//  5. G^T: every box point sums its (<= 8) element contributions in a fixed
//     order; points owned by this brick alone go straight to the output
//     (P^T: 0 on Dirichlet rows), points on a face shared with a neighbouring
//     brick go to this brick's slab of the shell buffer, summed later in a
//     fixed order by fixup_kernel — deterministic, no atomics.
#pragma once
#include "common.cuh"
#include "dual.cuh"
#include "physics.cuh"

namespace feod {

// Shared-memory scratch layouts of the line-ownership transposes, padded so
// that both the producing and the consuming half-warp hit 16 distinct 8-byte
// bank pairs (for NQ = 4 the outer stride is 20 = 4 mod 16).
constexpr int pad_stride(int x, int nq) {
  if (nq == 4) return x + ((4 - x % 16) + 16) % 16;
  return (x % 2 == 0) ? x + 1 : x;
}

template <int ND, int NQ>
struct Lay {
  // S: Z-step output, written by (a,b) for each l, read by (a,l) for each b
  static constexpr int SL = pad_stride(ND * ND, NQ);
  static constexpr int SN = SL * NQ;
  FEOD_HD static constexpr int S(int a, int b, int l) { return a + ND * b + SL * l; }
  // T: Y-step output, written by (a,l) for each j, read by (j,l) for each a
  static constexpr int TJ = pad_stride(NQ * ND, NQ);
  static constexpr int TN = TJ * NQ;
  FEOD_HD static constexpr int T(int a, int j, int l) { return l + NQ * a + TJ * j; }
  // P: X^T output, written by (j,l) for each a, read by (a,l) for each j
  static constexpr int PA = pad_stride(NQ * NQ, NQ);
  static constexpr int PN = PA * ND;
  FEOD_HD static constexpr int Pi(int a, int j, int l) { return l + NQ * j + PA * a; }
  // Q: Y^T output, written by (a,l) for each b, read by (a,b) for each l
  static constexpr int QB = pad_stride(ND * NQ, NQ);
  static constexpr int QN = QB * ND;
  FEOD_HD static constexpr int Qi(int a, int b, int l) { return a + ND * l + QB * b; }
  static constexpr int mx(int x, int y) { return x > y ? x : y; }
  static constexpr int SCR1 = mx(mx(2 * SN, 3 * TN), mx(mx(3 * PN, 2 * QN), NQ * NQ));
};

template <int ND, int NQ, int MODE>
struct OpShape {
  using S = BrickShape<ND>;
  static constexpr int K = ND - 1;
  static constexpr int BX = S::BX, BY = S::BY, BZ = S::BZ;
  static constexpr int EL = BX * BY;                        // elements per layer
  static constexpr int SB = S::SB;                          // sub-batches per layer
  static constexpr int EB = EL / SB;                        // elements per sub-batch
  static constexpr int NCLS = SB == 1 ? 4 : 2;              // colour classes per sub-batch
  static constexpr int LXF = K * BX + 1, LYF = K * BY + 1;  // DOF plane of the tile
  static constexpr int PLANE = LXF * LYF;
  static constexpr int RIN = 2 * K + 1;                     // input plane ring (layer + prefetch)
  static constexpr int ROUT = K + 1;                        // output plane ring
  static constexpr int LINES = NQ * NQ;
  static constexpr int NT = LINES * EB;
  static constexpr int MINB = (512 / NT) < 1 ? 1 : ((512 / NT) > 4 ? 4 : 512 / NT);   // CTAs/SM the register budget is sized for
  static constexpr int NIN = (MODE == MODE_RES) ? 1 : 2;
  static constexpr int NOUT = (MODE == MODE_DESIGN) ? 0 : (MODE == MODE_JVPRES ? 2 : 1);
  static constexpr int SCR = Lay<ND, NQ>::SCR1;   // doubles per element
  static constexpr int OUTSZ = (NOUT * ROUT * PLANE + 1) / 2 * 2;   // keeps the scratch 16-byte aligned
  static constexpr int SMEM_DOUBLES = NIN * RIN * PLANE + OUTSZ + EB * SCR;
  static constexpr size_t SMEM_BYTES = sizeof(double) * SMEM_DOUBLES;
  static constexpr int LZF = K * BZ + 1;
  static constexpr int SHELL = LXF * LYF * LZF - (LXF - 2) * (LYF - 2) * (LZF - 2);
};

// 8-byte asynchronous global -> shared copy (LDGSTS): the next layer's DOF
// planes stream in while the current layer computes. (The L-vector row pitch
// 8(kn+1) B is not 16-byte aligned, so TMA tensor maps cannot describe it.)
FEOD_DEV void cp_async8(double* smem_dst, const double* gsrc) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gsrc) : "memory");
}
FEOD_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
FEOD_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Non-coherent global load that the compiler may not sink toward its use: the
// metric stream is requested before the forward contractions so its HBM
// latency overlaps them.
FEOD_DEV double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// Hint the L2 to start fetching a contiguous byte range (TMA prefetch; no
// completion tracking, no shared memory).
FEOD_DEV void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Barrier among the threads of one element: the element's scratch is private
// to its NQ*NQ threads, so when they sit inside one warp a warp barrier is
// enough and warps run the contraction phases independently of each other.
template <int LINES>
FEOD_DEV void elem_sync() {
  if constexpr (32 % LINES == 0) __syncwarp();
  else __syncthreads();
}

// Forward interpolation of one field from the element's ND DOF planes in the
// shared ring (planes[c] = node level c): returns, for the
// x-line (j, l) this thread owns, U[i], dU/dxi1[i], dU/dxi2[i], dU/dxi3[i].
template <int ND, int NQ, int LXF>
FEOD_DEV void forward_field(const Tables& T, const double* const (&planes)[ND], double* scr, int line,
                            int X0, int Y0, double (&out)[4][NQ]) {
  using L = Lay<ND, NQ>;
  constexpr int SA = L::SN;   // S0 | S1
  constexpr int SB = L::TN;   // T0 | T1 | T2
  // ---- z: nodes c -> points l, values (t0) and z-derivative (t1)
  {
    const int a = line % NQ, b = line / NQ;
    if ((ND == NQ) || (a < ND && b < ND)) {
      double x[ND];
#pragma unroll
      for (int c = 0; c < ND; ++c) x[c] = planes[c][(X0 + a) + LXF * (Y0 + b)];
#pragma unroll
      for (int l = 0; l < NQ; ++l) {
        double t0 = 0.0, t1 = 0.0;
#pragma unroll
        for (int c = 0; c < ND; ++c) {
          t0 = fma(T.B[l][c], x[c], t0);
          t1 = fma(T.G[l][c], x[c], t1);
        }
        scr[L::S(a, b, l)] = t0;
        scr[SA + L::S(a, b, l)] = t1;
      }
    }
  }
  elem_sync<NQ * NQ>();
  // ---- y: nodes b -> points j
  {
    const int a = line % NQ, l = line / NQ;
    double s0[ND], s1[ND];
    if ((ND == NQ) || a < ND) {
#pragma unroll
      for (int b = 0; b < ND; ++b) {
        s0[b] = scr[L::S(a, b, l)];
        s1[b] = scr[SA + L::S(a, b, l)];
      }
    }
    elem_sync<NQ * NQ>();
    if ((ND == NQ) || a < ND) {
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        double y0 = 0.0, y1 = 0.0, y2 = 0.0;
#pragma unroll
        for (int b = 0; b < ND; ++b) {
          y0 = fma(T.B[j][b], s0[b], y0);
          y1 = fma(T.G[j][b], s0[b], y1);
          y2 = fma(T.B[j][b], s1[b], y2);
        }
        scr[L::T(a, j, l)] = y0;
        scr[SB + L::T(a, j, l)] = y1;
        scr[2 * SB + L::T(a, j, l)] = y2;
      }
    }
  }
  elem_sync<NQ * NQ>();
  // ---- x: nodes a -> points i
  {
    const int j = line % NQ, l = line / NQ;
    double r0[ND], r1[ND], r2[ND];
#pragma unroll
    for (int a = 0; a < ND; ++a) {
      r0[a] = scr[L::T(a, j, l)];
      r1[a] = scr[SB + L::T(a, j, l)];
      r2[a] = scr[2 * SB + L::T(a, j, l)];
    }
#pragma unroll
    for (int i = 0; i < NQ; ++i) {
      double U = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
#pragma unroll
      for (int a = 0; a < ND; ++a) {
        U = fma(T.B[i][a], r0[a], U);
        gx = fma(T.G[i][a], r0[a], gx);
        gy = fma(T.B[i][a], r1[a], gy);
        gz = fma(T.B[i][a], r2[a], gz);
      }
      out[0][i] = U;
      out[1][i] = gx;
      out[2][i] = gy;
      out[3][i] = gz;
    }
  }
  elem_sync<NQ * NQ>();
}

// Transposed interpolation: from the x-line of point values (Fx, Fy, Fz and
// optionally the value channel V) back to the element's nodal vector; the
// thread owning node column (a, b) returns r[c] = r_e[a, b, c] for all c.
template <int ND, int NQ, bool HASV>
FEOD_DEV void backward_field(const Tables& T, double* scr, int line, const double (&F)[4][NQ],
                             double (&rout)[ND]) {
  using L = Lay<ND, NQ>;
  constexpr int SA = L::QN;   // Q0 | Q1
  constexpr int SB = L::PN;   // P0 | P1 | P2
  // ---- x^T: points i -> nodes a
  {
    const int j = line % NQ, l = line / NQ;
#pragma unroll
    for (int a = 0; a < ND; ++a) {
      double p0 = 0.0, p1 = 0.0, p2 = 0.0;
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        p0 = fma(T.G[i][a], F[0][i], p0);
        if constexpr (HASV) p0 = fma(T.B[i][a], F[3][i], p0);
        p1 = fma(T.B[i][a], F[1][i], p1);
        p2 = fma(T.B[i][a], F[2][i], p2);
      }
      scr[L::Pi(a, j, l)] = p0;
      scr[SB + L::Pi(a, j, l)] = p1;
      scr[2 * SB + L::Pi(a, j, l)] = p2;
    }
  }
  elem_sync<NQ * NQ>();
  // ---- y^T: points j -> nodes b
  {
    const int a = line % NQ, l = line / NQ;
    double p0[NQ], p1[NQ], p2[NQ];
    if ((ND == NQ) || a < ND) {
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        p0[j] = scr[L::Pi(a, j, l)];
        p1[j] = scr[SB + L::Pi(a, j, l)];
        p2[j] = scr[2 * SB + L::Pi(a, j, l)];
      }
    }
    elem_sync<NQ * NQ>();
    if ((ND == NQ) || a < ND) {
#pragma unroll
      for (int b = 0; b < ND; ++b) {
        double q0 = 0.0, q1 = 0.0;
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
          q0 = fma(T.B[j][b], p0[j], q0);
          q0 = fma(T.G[j][b], p1[j], q0);
          q1 = fma(T.B[j][b], p2[j], q1);
        }
        scr[L::Qi(a, b, l)] = q0;
        scr[SA + L::Qi(a, b, l)] = q1;
      }
    }
  }
  elem_sync<NQ * NQ>();
  // ---- z^T: points l -> nodes c
  {
    const int a = line % NQ, b = line / NQ;
    if ((ND == NQ) || (a < ND && b < ND)) {
      double q0[NQ], q1[NQ];
#pragma unroll
      for (int l = 0; l < NQ; ++l) {
        q0[l] = scr[L::Qi(a, b, l)];
        q1[l] = scr[SA + L::Qi(a, b, l)];
      }
#pragma unroll
      for (int c = 0; c < ND; ++c) {
        double r = 0.0;
#pragma unroll
        for (int l = 0; l < NQ; ++l) {
          r = fma(T.B[l][c], q0[l], r);
          r = fma(T.G[l][c], q1[l], r);
        }
        rout[c] = r;
      }
    }
  }
  elem_sync<NQ * NQ>();
}

template <int ND, int NQ, int MODE, int MODEL, bool AFFINE>
__global__ void __launch_bounds__(OpShape<ND, NQ, MODE>::NT, OpShape<ND, NQ, MODE>::MINB)
op_kernel(const OpParams P, const Tables T, const double* __restrict__ in0, const double* __restrict__ in1,
          double* __restrict__ out0, double* __restrict__ out1, double* __restrict__ shell0,
          double* __restrict__ shell1, double* __restrict__ gout) {
  using S = OpShape<ND, NQ, MODE>;
  constexpr int K = S::K;
  constexpr int NQ3 = NQ * NQ * NQ;
  extern __shared__ __align__(16) double smem[];
  double* ring_in = smem;                                   // [NIN][RIN][PLANE]
  double* ring_out = smem + S::NIN * S::RIN * S::PLANE;     // [NOUT][ROUT][PLANE]
  double* scratch = ring_out + S::OUTSZ;

  const int tid = threadIdx.x;
  const int brick = blockIdx.x;
  const int bx = brick % P.nbx, by = (brick / P.nbx) % P.nby, bz = brick / (P.nbx * P.nby);
  const int ex0 = bx * S::BX, ey0 = by * S::BY, ez0 = bz * S::BZ;
  const int bxr = min(S::BX, P.nx - ex0), byr = min(S::BY, P.ny - ey0), bzr = min(S::BZ, P.nz - ez0);
  const int LX = K * bxr + 1, LY = K * byr + 1, LZ = K * bzr + 1;
  const int gX0 = K * ex0, gY0 = K * ey0, gZ0 = K * ez0;

  // ---- G (gather): stream DOF plane p (brick-local z index) into its ring slot
  auto load_plane = [&](int p) {
    const int slot = p % S::RIN;
    const int64_t zoff = (int64_t)P.Mx * P.My * (gZ0 + p);
    for (int idx = tid; idx < S::PLANE; idx += S::NT) {
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

  const int line = tid % S::LINES;
  const int eslot = tid / S::LINES;                // element slot of the sub-batch this thread works on
  double* scr = scratch + eslot * S::SCR;
  const int jl = line % NQ, ll = line / NQ;        // x-line owned in the point phase
  const int ra = line % NQ, rb = line / NQ;        // node column owned after B^T
  const double wjl = T.w[jl] * T.w[ll];

  // shell classification of the tile's sides
  const bool lowX = ex0 > 0, highX = ex0 + bxr < P.nx;
  const bool lowY = ey0 > 0, highY = ey0 + byr < P.ny;
  const bool lowZ = ez0 > 0, highZ = ez0 + bzr < P.nz;

  // ---- write finished output plane p (brick-local), then clear its slot
  auto flush_plane = [&](int p) {
    const int slot = p % S::ROUT;
    const int64_t zoff = (int64_t)P.Mx * P.My * (gZ0 + p);
    for (int idx = tid; idx < S::PLANE; idx += S::NT) {
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

  for (int z = 0; z < bzr; ++z) {
    cp_async_wait_all();
    __syncthreads();                                 // planes K z .. K z + K resident; previous layer flushed
    if (z + 1 < bzr) {
      for (int p = K * (z + 1) + 1; p <= K * (z + 1) + K; ++p) load_plane(p);
      cp_async_commit();
    }
   for (int sb = 0; sb < S::SB; ++sb) {
    // element of this sub-batch: SB = 1 -> the whole layer; SB = 2 -> rows of y-parity sb
    const int exl = eslot % S::BX, eyl = S::SB * (eslot / S::BX) + sb;
    const bool valid = exl < bxr && eyl < byr;
    const int X0 = valid ? K * exl : 0, Y0 = valid ? K * eyl : 0;
    const int colour = S::SB == 1 ? (exl & 1) + 2 * (eyl & 1) : (exl & 1);
    const int64_t eg = (int64_t)(ex0 + exl) + (int64_t)P.nx * ((ey0 + eyl) + (int64_t)P.ny * (ez0 + z));

    // metric of this element's x-lines: requested before the contractions
    double gmr[AFFINE ? 1 : 6][NQ];
    if constexpr (!AFFINE) {
      const double* gm = P.geom + (valid ? eg : 0) * (6 * NQ3) + line;
#pragma unroll
      for (int c = 0; c < 6; ++c)
#pragma unroll
        for (int i = 0; i < NQ; ++i) gmr[c][i] = ld_stream(gm + c * NQ3 + NQ * NQ * i);
      // L2 prefetch of the next layer's metric (one contiguous x-row of elements per y)
      if (sb == 0 && tid < S::BY && z + 1 < bzr && tid < byr) {
        const int64_t e1 = (int64_t)ex0 + (int64_t)P.nx * ((ey0 + tid) + (int64_t)P.ny * (ez0 + z + 1));
        prefetch_l2(P.geom + e1 * (6 * NQ3), (uint32_t)(bxr * 6 * NQ3 * sizeof(double)));
      }
    }
    double rho_e = 0.0;
    if constexpr (MODEL == HEAT) rho_e = valid ? __ldg(P.rho + eg) : 1.0;

    const double* pl0[ND];
    const double* pl1[ND];
#pragma unroll
    for (int c = 0; c < ND; ++c) {
      const int slot = (K * z + c) % S::RIN;
      pl0[c] = ring_in + slot * S::PLANE;
      pl1[c] = ring_in + (S::RIN + slot) * S::PLANE;
    }
    double fu[4][NQ];
    forward_field<ND, NQ, S::LXF>(T, pl0, scr, line, X0, Y0, fu);
    double fv[4][NQ];
    if constexpr (S::NIN == 2) forward_field<ND, NQ, S::LXF>(T, pl1, scr, line, X0, Y0, fv);

    // ---- D: pointwise on the x-line (i, jl, ll)
    double F0[4][NQ];   // first output channel set (r for RES, Jv for JVP/JVPRES)
    double F1[4][NQ];   // second (r for JVPRES)
    double gpart = 0.0;
#pragma unroll
    for (int i = 0; i < NQ; ++i) {
      const double wq = T.w[i] * wjl;
      Metric M;
      double W;
      if constexpr (AFFINE) {
        M = {wq * P.cx, wq * P.cy, wq * P.cz, 0.0, 0.0, 0.0};
        W = wq * P.vol;
      } else {
        M = {gmr[0][i], gmr[1][i], gmr[2][i], gmr[3][i], gmr[4][i], gmr[5][i]};
        const double det = M.xx * (M.yy * M.zz - M.yz * M.yz) - M.xy * (M.xy * M.zz - M.yz * M.xz) +
                           M.xz * (M.xy * M.yz - M.yy * M.xz);
        W = det / (wq * wq);
      }
      if constexpr (MODE == MODE_RES) {
        const double gh[3] = {fu[1][i], fu[2][i], fu[3][i]};
        double Fh[3];
        flux_hat<MODEL>(fu[0][i], gh, M, W, rho_e, P, Fh);
        F0[0][i] = Fh[0];
        F0[1][i] = Fh[1];
        F0[2][i] = Fh[2];
        F0[3][i] = -P.f * W;
      } else if constexpr (MODE == MODE_JVP || MODE == MODE_JVPRES) {
        using D = dual<double>;
        const D ud(fu[0][i], fv[0][i]);
        const D gh[3] = {D(fu[1][i], fv[1][i]), D(fu[2][i], fv[2][i]), D(fu[3][i], fv[3][i])};
        D Fh[3];
        flux_hat<MODEL>(ud, gh, M, W, rho_e, P, Fh);
        F0[0][i] = Fh[0].d;
        F0[1][i] = Fh[1].d;
        F0[2][i] = Fh[2].d;
        F0[3][i] = 0.0;
        if constexpr (MODE == MODE_JVPRES) {
          F1[0][i] = Fh[0].v;
          F1[1][i] = Fh[1].v;
          F1[2][i] = Fh[2].v;
          F1[3][i] = -P.f * W;
        }
      } else {   // MODE_DESIGN: seed d/drho
        using D = dual<double>;
        const D ud(fu[0][i]);
        const D gh[3] = {D(fu[1][i]), D(fu[2][i]), D(fu[3][i])};
        const D rd(rho_e, 1.0);
        D Fh[3];
        flux_hat<MODEL>(ud, gh, M, W, rd, P, Fh);
        gpart -= fv[1][i] * Fh[0].d + fv[2][i] * Fh[1].d + fv[3][i] * Fh[2].d;
      }
    }

    if constexpr (MODE == MODE_DESIGN) {
      scr[line] = gpart;
      elem_sync<S::LINES>();
      if (line == 0 && valid) {
        double s = 0.0;
        for (int t = 0; t < S::LINES; ++t) s += scr[t];
        gout[eg] = s;
      }
      elem_sync<S::LINES>();
    } else {
      // ---- B^T, then G^T into the output ring: the four x-y colour classes of
      // the layer add their element vectors one class at a time (elements of one
      // class share no DOF), so every DOF sums its contributions in a fixed order
      double r0[ND], r1[ND];
      backward_field<ND, NQ, MODE == MODE_RES>(T, scr, line, F0, r0);
      if constexpr (MODE == MODE_JVPRES) backward_field<ND, NQ, true>(T, scr, line, F1, r1);
      const bool owner = valid && ((ND == NQ) || (ra < ND && rb < ND));
      const int node = (X0 + ra) + S::LXF * (Y0 + rb);
#pragma unroll
      for (int cls = 0; cls < S::NCLS; ++cls) {
        if (cls > 0 || sb > 0) __syncthreads();
        if (owner && colour == cls) {
#pragma unroll
          for (int c = 0; c < ND; ++c) {
            double* cell = ring_out + ((K * z + c) % S::ROUT) * S::PLANE + node;
            *cell += r0[c];
            if constexpr (MODE == MODE_JVPRES) cell[S::ROUT * S::PLANE] += r1[c];
          }
        }
      }
    }
   }  // sub-batches
    if constexpr (S::NOUT > 0) {
      __syncthreads();
      // planes K z .. K z + K-1 are complete (the top plane carries into the next layer)
      for (int c = 0; c < K; ++c) flush_plane(K * z + c);
      if (z == bzr - 1) flush_plane(K * z + K);
    }
  }
}

}  // namespace feod
