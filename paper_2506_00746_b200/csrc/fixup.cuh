// K5 — deterministic scatter fix-up: the G^T step for the DOFs on faces shared
// by neighbouring bricks. Each shared DOF sums the shell values
// its 2, 4 or 8 bricks wrote, in a fixed order (z, y, x ascending: low brick
// first), and applies P^T (0 on Dirichlet rows). No atomics: the result is
// bitwise reproducible run to run.
//
// One CTA per DOF row; threads stride along the row (consecutive threads touch
// consecutive X, or Y on set X):
//   set 0 (Y): DOF planes Y = m PY (m = 1..nby-1), rows along X at Z (X on an interior x-plane skipped)
//   set 1 (Z): planes Z = m PZ, rows along X at Y (X on an x-plane or Y on a y-plane skipped)
//   set 2 (X): planes X = m PX, rows along Y at Z (x-y / x-z edges and corners too)
// Shell slab of a brick with box LX x LY x LZ (common.cuh shell_rank): the z = 0
// plane, one ring per middle z, the z = LZ-1 plane.
//
// Overlap with the operator kernel: the fix-up is launched as a programmatic
// dependent of plane_kernel (which triggers its dependents at entry), so its CTAs
// start as soon as an SM has room (64-thread CTAs fit beside the operator CTAs, so
// rows are summed while the operator kernel still runs). A row does not wait for the whole grid:
// it waits only for the bricks it reads, whose IO warps publish a per-brick epoch
// (P.bdone, release) after their last store. The host orders the rows by the last
// brick ticket they depend on (P.fixrows), so rows become ready in launch order.
// The last CTA ends with griddepcontrol.wait, so the fix-up never completes before
// the operator kernel.
#pragma once
#include "common.cuh"
#include "pointwise.cuh"

namespace feod {

constexpr int kFixMaxThreads = 256;

#ifndef FEOD_FIX_SLEEP_NS
#define FEOD_FIX_SLEEP_NS 200   // back-off of a row waiting for its bricks
#endif

// box extent of brick b along an axis (the last brick may be ragged)
FEOD_HD int box_len(int K, int B, int b, int ne) { return K * min(B, ne - b * B) + 1; }

// contributors of global DOF index g along one axis: brick b[.] and local index l[.]
// (two when g lies on an interior brick plane: the low brick first)
FEOD_HD void axis_contrib(int g, int PS, int nb, int* b, int* l, int& n) {
  int bb = g / PS;
  if (bb >= nb) bb = nb - 1;
  b[0] = bb; l[0] = g - bb * PS; n = 1;
  if (l[0] == 0 && bb > 0) { b[1] = bb; l[1] = 0; b[0] = bb - 1; l[0] = PS; n = 2; }
}

FEOD_DEV unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// On an X-row (sets Y and Z) ly and lz of every contributor are CTA-uniform and
// the contributor sits on a y- or z-face of its box, so its shell rank is linear
// in the box extent LX and the local lx (common.cuh shell_rank):
//   lz = 0:                    lx + LX ly
//   lz = LZ-1:                 lx + LX (LY + 2(LZ-2) + ly) + 2(LZ-2)(LY-2)
//   0 < lz < LZ-1, ly = 0:     lx + LX (LY + 2(lz-1))      + 2(lz-1)(LY-2)
//   0 < lz < LZ-1, ly = LY-1:  lx + LX (LY + 2(lz-1) + 1)  + 2(lz-1)(LY-2)
// so each contributor costs one IMAD per DOF: offset = U + C LX + (bx stride + lx).
// The brick shape: BX, BY are compile-time (the inner loops divide by them), the depth
// BZ is read from P.tbz (the column kernel chooses it per mesh). Both kernel families
// (plane_kernel, col_kernel) write the same shell layout for their own bricks.
template <int K, int BX, int BY, bool TWO>
__global__ void __launch_bounds__(kFixMaxThreads) fixup_kernel(const OpParams P,
                                                               const double* __restrict__ shell0, double* __restrict__ out0,
                                                               const double* __restrict__ shell1, double* __restrict__ out1) {
  const int BZ = P.tbz;
  constexpr int PX = K * BX, PY = K * BY;
  const int PZ = K * BZ;
  // the value this call's bricks publish (set by the operator kernel before it let this grid launch)
  const unsigned long long epoch = ld_acquire_u64(&P.ds->cur);
  const int2 rw = P.fixrows[blockIdx.x];
  const int set = rw.x >> 24, m = rw.x & 0xffffff, coord = rw.y;
  const int64_t bstride = P.shell_stride;

  // contributors along the three axes (brick, local index; the summation order is z, y, x ascending)
  int bxa[2] = {0, 0}, lxa[2] = {0, 0}, bya[2] = {0, 0}, lya[2] = {0, 0}, bza[2] = {0, 0}, lza[2] = {0, 0};
  int ny = 2, nz = 2;
  int X = 0, Y = 0, Z = 0;
  if (set == 0) {
    Y = m * PY; Z = coord;
    bya[0] = m - 1; lya[0] = PY; bya[1] = m; lya[1] = 0;
    axis_contrib(Z, PZ, P.nbz, bza, lza, nz);
  } else if (set == 1) {
    Z = m * PZ; Y = coord;
    bza[0] = m - 1; lza[0] = PZ; bza[1] = m; lza[1] = 0;
    axis_contrib(Y, PY, P.nby, bya, lya, ny);
  } else {
    X = m * PX; Z = coord;
    bxa[0] = m - 1; lxa[0] = PX; bxa[1] = m; lxa[1] = 0;
    axis_contrib(Z, PZ, P.nbz, bza, lza, nz);
  }

  // wait for the bricks this row reads: a box of brick indices, the full range along the row's axis
  {
    const int x0 = set == 2 ? m - 1 : 0, cx = set == 2 ? 2 : P.nbx;
    const int y0 = set == 2 ? 0 : bya[0], cy = set == 2 ? P.nby : ny;
    const int z0 = bza[0], cz = nz;
    const int cnt = cx * cy * cz;
    for (int d = threadIdx.x; d < cnt; d += blockDim.x) {
      const int ix = d % cx, iy = (d / cx) % cy, iz = d / (cx * cy);
      const unsigned long long* f = P.bdone + ((x0 + ix) + (int64_t)P.nbx * ((y0 + iy) + (int64_t)P.nby * (z0 + iz)));
      // bounded wait: a brick that never publishes (a fault upstream) ends in a trap
      // (a reported launch error) instead of a hung GPU
      const long long t0 = clock64();
      while (ld_acquire_u64(f) < epoch) {
        __nanosleep(FEOD_FIX_SLEEP_NS);
        if (clock64() - t0 > (1ll << 35)) __trap();   // ~17 s at 2 GHz
      }
    }
    __syncthreads();
  }

  if (set != 2) {
    // uniform linear forms, slot q = 2 cz + cy
    int64_t U[4];
    int C[4];
#pragma unroll
    for (int cz = 0; cz < 2; ++cz)
#pragma unroll
      for (int cy = 0; cy < 2; ++cy) {
        const int q = 2 * cz + cy;
        U[q] = 0; C[q] = 0;
        if (cz < nz && cy < ny) {
          const int LY = box_len(K, BY, bya[cy], P.ny), LZ = box_len(K, BZ, bza[cz], P.nz);
          const int ly = lya[cy], lz = lza[cz];
          int A, Cc;
          if (lz == 0) { A = 0; Cc = ly; }
          else if (lz == LZ - 1) { A = 2 * (LZ - 2) * (LY - 2); Cc = LY + 2 * (LZ - 2) + ly; }
          else { A = 2 * (lz - 1) * (LY - 2); Cc = LY + 2 * (lz - 1) + (ly == 0 ? 0 : 1); }
          U[q] = ((int64_t)bya[cy] + (int64_t)P.nby * bza[cz]) * P.nbx * bstride + A;
          C[q] = Cc;
        }
      }
    const bool dyz = ((P.faces & 4u) && Y == 0) || ((P.faces & 8u) && Y == P.My - 1) ||
                     ((P.faces & 16u) && Z == 0) || ((P.faces & 32u) && Z == P.Mz - 1);
    const int64_t g0 = (int64_t)P.Mx * (Y + (int64_t)P.My * Z);
    for (int x = threadIdx.x; x < P.Mx; x += blockDim.x) {
      if (x % PX == 0 && x > 0 && x < P.Mx - 1) continue;
      const int bx = min(x / PX, P.nbx - 1);
      const int lx = x - bx * PX;
      const int LX = K * min(BX, P.nx - bx * BX) + 1;
      const int64_t base = bx * bstride + lx;
      double v0[4], v1[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if ((q >> 1) < nz && (q & 1) < ny) {
          const int64_t o = U[q] + (int64_t)C[q] * LX + base;
          v0[q] = __ldcg(shell0 + o);   // L2 only: written by other SMs during this kernel's lifetime
          if constexpr (TWO) v1[q] = __ldcg(shell1 + o);
        }
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if ((q >> 1) < nz && (q & 1) < ny) {
          s0 += v0[q];
          if constexpr (TWO) s1 += v1[q];
        }
      const bool dir = dyz || ((P.faces & 1u) && x == 0) || ((P.faces & 2u) && x == P.Mx - 1);
      out0[g0 + x] = dir ? 0.0 : s0;
      if constexpr (TWO) out1[g0 + x] = dir ? 0.0 : s1;
    }
  } else {
    const int LXa[2] = {PX + 1, box_len(K, BX, m, P.nx)};
    const int LZa[2] = {box_len(K, BZ, bza[0], P.nz), box_len(K, BZ, nz == 2 ? bza[1] : bza[0], P.nz)};
    const bool dxz = ((P.faces & 1u) && X == 0) || ((P.faces & 2u) && X == P.Mx - 1) ||
                     ((P.faces & 16u) && Z == 0) || ((P.faces & 32u) && Z == P.Mz - 1);
    for (int y = threadIdx.x; y < P.My; y += blockDim.x) {
      int byt[2], lyt[2], nyt;
      axis_contrib(y, PY, P.nby, byt, lyt, nyt);
      const int LYa[2] = {box_len(K, BY, byt[0], P.ny), box_len(K, BY, nyt == 2 ? byt[1] : byt[0], P.ny)};
      double v0[8], v1[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int cx = q & 1, cy = (q >> 1) & 1, cz = q >> 2;
        if (cy < nyt && cz < nz) {
          const int64_t o = (bxa[cx] + (int64_t)P.nbx * (byt[cy] + (int64_t)P.nby * bza[cz])) * bstride +
                            shell_rank(lxa[cx], lyt[cy], lza[cz], LXa[cx], LYa[cy], LZa[cz]);
          v0[q] = __ldcg(shell0 + o);
          if constexpr (TWO) v1[q] = __ldcg(shell1 + o);
        }
      }
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int cy = (q >> 1) & 1, cz = q >> 2;
        if (cy < nyt && cz < nz) {
          s0 += v0[q];
          if constexpr (TWO) s1 += v1[q];
        }
      }
      const bool dir = dxz || ((P.faces & 4u) && y == 0) || ((P.faces & 8u) && y == P.My - 1);
      const int64_t g = (int64_t)X + (int64_t)P.Mx * (y + (int64_t)P.My * Z);
      out0[g] = dir ? 0.0 : s0;
      if constexpr (TWO) out1[g] = dir ? 0.0 : s1;
    }
  }
  // the fix-up grid must not complete before its primary (the operator kernel)
  if (blockIdx.x == gridDim.x - 1) asm volatile("griddepcontrol.wait;" ::: "memory");
}


// Host: the fix-up rows, keyed by the largest brick index (= ticket) they read.
// Entry: x = set << 24 | m, y = the row's fixed coordinate.
template <int K>
int fixup_rows(const OpParams& P, int2* rows, unsigned long long* keys) {
  const int PY = K * P.tby, PZ = K * P.tbz;
  int c = 0;
  auto bmax = [](int g, int PS, int nb) { int b[2], l[2], k; axis_contrib(g, PS, nb, b, l, k); return b[k - 1]; };
  for (int m = 1; m < P.nby; ++m)
    for (int Z = 0; Z < P.Mz; ++Z) {
      if (rows) {
        rows[c] = make_int2(0 << 24 | m, Z);
        keys[c] = (unsigned long long)((P.nbx - 1) + (int64_t)P.nbx * (m + (int64_t)P.nby * bmax(Z, PZ, P.nbz)));
      }
      ++c;
    }
  for (int m = 1; m < P.nbz; ++m)
    for (int Y = 0; Y < P.My; ++Y) {
      if (Y % PY == 0 && Y > 0 && Y < P.My - 1) continue;
      if (rows) {
        rows[c] = make_int2(1 << 24 | m, Y);
        keys[c] = (unsigned long long)((P.nbx - 1) + (int64_t)P.nbx * (bmax(Y, PY, P.nby) + (int64_t)P.nby * m));
      }
      ++c;
    }
  for (int m = 1; m < P.nbx; ++m)
    for (int Z = 0; Z < P.Mz; ++Z) {
      if (rows) {
        rows[c] = make_int2(2 << 24 | m, Z);
        keys[c] = (unsigned long long)(m + (int64_t)P.nbx * ((P.nby - 1) + (int64_t)P.nby * bmax(Z, PZ, P.nbz)));
      }
      ++c;
    }
  return c;
}

template <int K, int BX, int BY>
cudaError_t launch_fixup_t(const OpParams& P, const double* shell0, double* out0, const double* shell1, double* out1,
                           cudaStream_t st) {
  if (P.nfixrows == 0) return cudaSuccess;
  const int len = max(P.Mx, P.My);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)P.nfixrows);
  // two warps per row: small enough that fix-up CTAs become resident beside the
  // persistent operator CTAs (registers left over per SM sub-partition) and run
  // while it still works, instead of only in its tail (measured: 32 / 64 / 96 /
  // 128 / 224 threads -> C3 JVP call 245.9 / 242.6 / 244.3 / 246.5 / 255.1 us)
#ifdef FEOD_FIX_THREADS
  cfg.blockDim = dim3((unsigned)FEOD_FIX_THREADS);
#else
  cfg.blockDim = dim3((unsigned)min(64, (len + 31) / 32 * 32));
#endif
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (shell1)
    e = cudaLaunchKernelEx(&cfg, fixup_kernel<K, BX, BY, true>, P, shell0, out0, shell1, out1);
  else
    e = cudaLaunchKernelEx(&cfg, fixup_kernel<K, BX, BY, false>, P, shell0, out0, (const double*)nullptr,
                           (double*)nullptr);
  return e;
}

}  // namespace feod
