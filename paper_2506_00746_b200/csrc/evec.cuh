// G^T + P^T from a discontinuous L-vector (the per-element results of the warp-per-element
// kernels: q6tc.cu's operator and diagonal at Q6, diag.cu's diagonal at Q3..Q5).
//
// Layout: element e's node (a, b, c) of an order-K element (ND = K + 1 nodes per axis) at
// X' = ND ex + a, Y' = ND ey + b, Z' = ND ez + c of an (ND nx) x (ND ny) x (ND nz) array,
// x fastest: neighbouring elements' node rows are adjacent, so the assembly reads it row
// by row, coalesced. DOF X of an axis is node a = X - K e of element e (X' = X + e); an
// element-boundary DOF (X = K e, 0 < e < n) has the two candidates X' = ND e - 1 and ND e
// (ascending element order), any other DOF the one X' = ND min(X / K, n - 1) + a.
//
// A warp per DOF row (Y, Z) with a shared-memory row buffer of its own: stage 1 sums each
// X' of the row over the row's <= 4 source rows (the row-uniform y / z candidates, z then
// y ascending; lanes over X', coalesced, kAsmUnroll X' in flight per lane), stage 2 gives
// each DOF X its one or two X' sums (left element first) and applies P^T (Dirichlet rows
// get dirval). A fixed summation order everywhere: deterministic, no atomics.
// With dotx != nullptr (Newton-CG) the kernel also forms the partial sums of dotx . out per
// CTA (rows in the warp's order, lanes by a butterfly, warps in order) into dpart[blockIdx.x]
// over a fixed grid of kRedBlocks CTAs: the CG's p.Ap needs no pass of its own and stays
// bitwise reproducible (reduce_partials in blas1.cu finishes it).
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace feod {

template <int K>
FEOD_DEV int evec_cands(int G, int ne, int* c) {
  constexpr int ND = K + 1;
  if (G % K == 0 && G > 0 && G < K * ne) {
    c[0] = ND * (G / K) - 1;
    c[1] = ND * (G / K);
    return 2;
  }
  const int e = min(G / K, ne - 1);
  c[0] = ND * e + (G - K * e);
  return 1;
}

#ifndef FEOD_ASM_PREFETCH   // L2 prefetch of the warp's next row (measured slower: C4 JVP 248 -> 259 us,
#define FEOD_ASM_PREFETCH 0   // residual 194 -> 204)
#endif
// FEOD_ASM_MINB (experiment knob): resident CTAs per SM the assembly is compiled for. Unset
// (default): no min-blocks hint -- 64 registers, no spills, 4 CTAs per SM. Set to 4 it spills
// ~170 B after the FUSE refactoring (measured C4 JVP 249 -> 259 us, C3 diagonal 280 -> 307);
// 5 / 6 are worse still.
#ifdef FEOD_ASM_MINB
#define FEOD_ASM_BOUNDS __launch_bounds__(kAsmThreads, FEOD_ASM_MINB)
#elif defined(FEOD_ASM_FUSE_MINB)   // the FUSE variant alone (110 registers without a hint)
#define FEOD_ASM_BOUNDS __launch_bounds__(kAsmThreads, FUSE ? FEOD_ASM_FUSE_MINB : 1)
#else
#define FEOD_ASM_BOUNDS __launch_bounds__(kAsmThreads)
#endif
constexpr int kAsmThreads = 256;
constexpr int kAsmUnroll = 8;
constexpr int kFuseUnroll = 4;

// FUSE (Newton-CG, kernels.h CgFuse): the row's assembled values update r instead of going
// to out, and the partials are those of r.z; alpha from the operator kernel's p.Ap partials
// (the same thread mapping and tree as blas1.cu's reduce_partials, in every CTA)
template <int K, bool FUSE>
__global__ void FEOD_ASM_BOUNDS evec_assemble_kernel(const OpParams P, const double* __restrict__ ev,
                                                                     double* __restrict__ out,
                                                                     const double* __restrict__ dotx,
                                                                     double* __restrict__ dpart, double dirval,
                                                                     const CgFuse F) {
  constexpr int ND = K + 1;
  extern __shared__ __align__(16) double asm_sm[];
  double acc = 0.0;
  double alpha = 0.0;
  if constexpr (FUSE) {
    static_assert(kAsmThreads == 256, "the reduction tree below is blas1.cu's (256 threads)");
    __shared__ double sh[kAsmThreads];
    double a = 0.0;
    for (int i = threadIdx.x; i < kRedBlocks; i += kAsmThreads) a += F.pAp_part[i];
    sh[threadIdx.x] = a;
    __syncthreads();
    for (int s = kAsmThreads / 2; s > 0; s >>= 1) {
      if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
      __syncthreads();
    }
    const double den = sh[0];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *F.pAp = den;
      if (!(den > 0.0)) *F.bad = 1;
    }
    alpha = *F.rr / den;
  }
  const int LX = ND * P.nx;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* const t = asm_sm + (size_t)wid * LX;
  const int64_t LYd = ND * (int64_t)P.ny;
  const int rows = P.My * P.Mz;
  const int warps = gridDim.x * (kAsmThreads / 32);
  for (int YZ = blockIdx.x * (kAsmThreads / 32) + wid; YZ < rows; YZ += warps) {
    const int Y = YZ % P.My, Z = YZ / P.My;
    int cy[2], cz[2];
    const int nyc = evec_cands<K>(Y, P.ny, cy), nzc = evec_cands<K>(Z, P.nz, cz);
    const double* src[4] = {ev, ev, ev, ev};
    int ns = 0;
    for (int kz = 0; kz < nzc; ++kz)
      for (int ky = 0; ky < nyc; ++ky) src[ns++] = ev + ((int64_t)cz[kz] * LYd + cy[ky]) * LX;
#if FEOD_ASM_PREFETCH
    {   // the warp's NEXT row: its source rows on their way to L2 while this row is summed
      const int YZn = YZ + warps;
      if (YZn < rows) {
        const int Yn = YZn % P.My, Zn = YZn / P.My;
        int cyn[2], czn[2];
        const int nyn = evec_cands<K>(Yn, P.ny, cyn), nzn = evec_cands<K>(Zn, P.nz, czn);
        for (int kz = 0; kz < nzn; ++kz)
          for (int ky = 0; ky < nyn; ++ky) {
            const double* sp = ev + ((int64_t)czn[kz] * LYd + cyn[ky]) * LX;
            for (int X = 16 * lane; X < LX; X += 16 * 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(sp + X));
          }
      }
    }
#endif
    if constexpr (FUSE) {   // the row of r (and of the diagonal) on its way to L2 while stage 1 runs
      for (int X = 16 * lane; X < P.Mx; X += 16 * 32) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(F.r + (int64_t)P.Mx * YZ + X));
        if (F.diag) asm volatile("prefetch.global.L2 [%0];" ::"l"(F.diag + (int64_t)P.Mx * YZ + X));
      }
    }
    for (int X0 = 0; X0 < LX; X0 += 32 * kAsmUnroll) {
      double v[kAsmUnroll][4];
#pragma unroll
      for (int m = 0; m < kAsmUnroll; ++m) {
        const int Xp = X0 + 32 * m + lane;
#pragma unroll
        for (int k = 0; k < 4; ++k) v[m][k] = (k < ns && Xp < LX) ? __ldcs(src[k] + Xp) : 0.0;
      }
#pragma unroll
      for (int m = 0; m < kAsmUnroll; ++m) {
        const int Xp = X0 + 32 * m + lane;
        if (Xp < LX) t[Xp] = ((v[m][0] + v[m][1]) + v[m][2]) + v[m][3];   // absent sources add +0.0 (exact)
      }
    }
    __syncwarp();
    const bool dyz = ((P.faces & 4u) && Y == 0) || ((P.faces & 8u) && Y == P.My - 1) ||
                     ((P.faces & 16u) && Z == 0) || ((P.faces & 32u) && Z == P.Mz - 1);
    double* orow = out + (int64_t)P.Mx * YZ;
    auto row_sum = [&](int X) {
      const int e = X / K, a = X - K * e;
      double s;
      if (a == 0 && e > 0 && e < P.nx) s = t[ND * e - 1] + t[ND * e];   // left element first
      else s = t[X + min(e, P.nx - 1)];   // X = K nx: the last element's node K, X' = ND nx - 1
      const bool dir = dyz || ((P.faces & 1u) && X == 0) || ((P.faces & 2u) && X == P.Mx - 1);
      return dir ? dirval : s;
    };
    if constexpr (FUSE) {
      // r (and the Jacobi diagonal) kFuseUnroll entries per lane in flight: r is read and
      // written through one pointer, so a plain per-X loop serialises on every load
      const int64_t g0 = (int64_t)P.Mx * YZ;
      for (int X0 = 0; X0 < P.Mx; X0 += 32 * kFuseUnroll) {
        double rv[kFuseUnroll], dv[kFuseUnroll];
#pragma unroll
        for (int m = 0; m < kFuseUnroll; ++m) {
          const int X = X0 + 32 * m + lane;
          rv[m] = X < P.Mx ? __ldcs(F.r + g0 + X) : 0.0;
          dv[m] = (F.diag && X < P.Mx) ? __ldcs(F.diag + g0 + X) : 1.0;
        }
#pragma unroll
        for (int m = 0; m < kFuseUnroll; ++m) {
          const int X = X0 + 32 * m + lane;
          if (X < P.Mx) {
            const double ri = fma(-alpha, row_sum(X), rv[m]);
            F.r[g0 + X] = ri;
            acc = fma(ri, F.diag ? ri / dv[m] : ri, acc);
          }
        }
      }
    } else {
      for (int X = lane; X < P.Mx; X += 32) {
        const double o = row_sum(X);
        orow[X] = o;
        if (dotx) acc = fma(__ldcs(dotx + (int64_t)P.Mx * YZ + X), o, acc);
      }
    }
    __syncwarp();
  }
  if (FUSE || dotx) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __syncthreads();   // the row buffers are free: reuse for the warp sums
    if (lane == 0) asm_sm[wid] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double sum = 0.0;
      for (int w = 0; w < kAsmThreads / 32; ++w) sum += asm_sm[w];
      (FUSE ? F.rz_part : dpart)[blockIdx.x] = sum;
    }
  }
}

template <int K>
inline cudaError_t evec_assemble(const OpParams& P, const double* ev, double* out, const double* dotx, double* dpart,
                                 double dirval, cudaStream_t st, const CgFuse* fuse = nullptr) {
  const int rows = P.My * P.Mz;
  const size_t smem = sizeof(double) * (K + 1) * (size_t)P.nx * (kAsmThreads / 32);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;   // (K + 1) nx <= 3632 (8 row buffers)
  if (smem > 48 * 1024) {   // beyond the default: opt in (per call: a handle may live on any device)
    const cudaError_t e = fuse ? cudaFuncSetAttribute(evec_assemble_kernel<K, true>,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                               : cudaFuncSetAttribute(evec_assemble_kernel<K, false>,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const int ctas = (rows + kAsmThreads / 32 - 1) / (kAsmThreads / 32);
  const unsigned grid = (dotx || fuse) ? (unsigned)kRedBlocks : (unsigned)(ctas < kRedBlocks ? ctas : kRedBlocks);
  if (fuse) evec_assemble_kernel<K, true><<<grid, kAsmThreads, smem, st>>>(P, ev, out, nullptr, nullptr, dirval, *fuse);
  else evec_assemble_kernel<K, false><<<grid, kAsmThreads, smem, st>>>(P, ev, out, dotx, dpart, dirval, CgFuse{});
  return cudaGetLastError();
}

}  // namespace feod
