// K6 — BLAS-1 for the Jacobian-free Newton-CG driver (reading A15): dot
// products as deterministic two-stage reductions over a FIXED grid (the same
// partial-sum tree every call), and the fused CG vector updates with the
// scalars kept on the device (no host round trip inside the CG loop).
// HBM-bound: a full-occupancy fixed grid (8 CTAs x 256 threads per SM) and
// kUnroll independent element streams per thread keep enough loads in flight.
#include "common.cuh"
#include "kernels.h"

namespace feod {

constexpr int kRedThreads = 256;
constexpr int kUnroll = 4;
constexpr int64_t kRedStride = (int64_t)kRedBlocks * kRedThreads;

FEOD_DEV double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = kRedThreads / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  return sh[0];
}

__global__ void __launch_bounds__(kRedThreads) dot_partial_kernel(const double* __restrict__ x,
                                                                  const double* __restrict__ y, int64_t n,
                                                                  double* __restrict__ partials) {
  __shared__ double sh[kRedThreads];
  double acc[kUnroll] = {};
  int64_t i = (int64_t)blockIdx.x * kRedThreads + threadIdx.x;
  for (; i + (kUnroll - 1) * kRedStride < n; i += kUnroll * kRedStride) {
    double xv[kUnroll], yv[kUnroll];
#pragma unroll
    for (int t = 0; t < kUnroll; ++t) { xv[t] = __ldcs(x + i + t * kRedStride); yv[t] = __ldcs(y + i + t * kRedStride); }
#pragma unroll
    for (int t = 0; t < kUnroll; ++t) acc[t] = fma(xv[t], yv[t], acc[t]);
  }
#pragma unroll
  for (int t = 0; t < kUnroll - 1; ++t)
    if (i < n) { acc[t] = fma(x[i], y[i], acc[t]); i += kRedStride; }
  const double s = block_sum((acc[0] + acc[1]) + (acc[2] + acc[3]), sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kRedThreads) reduce_final_kernel(const double* __restrict__ partials,
                                                                   double* __restrict__ out) {
  __shared__ double sh[kRedThreads];
  double acc = 0.0;
  for (int i = threadIdx.x; i < kRedBlocks; i += kRedThreads) acc += partials[i];
  const double s = block_sum(acc, sh);
  if (threadIdx.x == 0) *out = s;
}

cudaError_t dot_partial(const double* x, const double* y, int64_t n, double* partials, cudaStream_t st) {
  dot_partial_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(x, y, n, partials);
  return cudaGetLastError();
}

cudaError_t reduce_final(const double* partials, double* out, cudaStream_t st) {
  reduce_final_kernel<<<1, kRedThreads, 0, st>>>(partials, out);
  return cudaGetLastError();
}

// r = -F, p = z = M^{-1} r (M = diag, or the identity when diag == nullptr), d = 0
__global__ void cg_init_kernel(const double* __restrict__ F, double* __restrict__ r, double* __restrict__ p,
                               double* __restrict__ d, const double* __restrict__ diag, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = -F[i];
    r[i] = v;
    p[i] = diag ? v / diag[i] : v;
    d[i] = 0.0;
  }
}

// The final stage of a dot product, done redundantly by every CTA of the kernel that
// needs the scalar: the same thread mapping and tree as reduce_final_kernel, so every
// CTA (and reduce_final) gets the same bits -- one launch less per scalar.
FEOD_DEV double reduce_partials(const double* __restrict__ partials, double* sh) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < kRedBlocks; i += kRedThreads) acc += partials[i];
  const double s = block_sum(acc, sh);
  __syncthreads();   // sh reused by the caller
  return s;
}

// alpha = rr / pAp (pAp reduced here from dot_partial's partials; CTA 0 keeps it in
// *pAp);  r -= alpha Ap;  partials of r.r (same fixed grid as dot_partial)
// (with diag: the partials are of r . M^{-1} r, the preconditioned CG's rz). The update
// d += alpha p is deferred to cg_dir, which reads p anyway (one vector pass less, the same
// alpha and p: bitwise the same d).
__global__ void __launch_bounds__(kRedThreads) cg_update_kernel(const double* __restrict__ rr,
                                                                const double* __restrict__ pAp_partials,
                                                                double* __restrict__ pAp,
                                                                const double* __restrict__ Ap,
                                                                double* __restrict__ r, int64_t n,
                                                                double* __restrict__ partials, int* __restrict__ bad,
                                                                const double* __restrict__ diag) {
  __shared__ double sh[kRedThreads];
  const double den = reduce_partials(pAp_partials, sh);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *pAp = den;
    if (!(den > 0.0)) *bad = 1;
  }
  const double alpha = *rr / den;
  double acc[kUnroll] = {};
  int64_t i = (int64_t)blockIdx.x * kRedThreads + threadIdx.x;
  for (; i + (kUnroll - 1) * kRedStride < n; i += kUnroll * kRedStride) {
    double av[kUnroll], rv[kUnroll];
#pragma unroll
    for (int t = 0; t < kUnroll; ++t) {
      const int64_t j = i + t * kRedStride;
      av[t] = __ldcs(Ap + j); rv[t] = r[j];
    }
#pragma unroll
    for (int t = 0; t < kUnroll; ++t) {
      const int64_t j = i + t * kRedStride;
      const double ri = fma(-alpha, av[t], rv[t]);
      r[j] = ri;
      acc[t] = fma(ri, diag ? ri / diag[j] : ri, acc[t]);
    }
  }
#pragma unroll
  for (int t = 0; t < kUnroll - 1; ++t)
    if (i < n) {
      const double ri = fma(-alpha, Ap[i], r[i]);
      r[i] = ri;
      acc[t] = fma(ri, diag ? ri / diag[i] : ri, acc[t]);
      i += kRedStride;
    }
  const double s = block_sum((acc[0] + acc[1]) + (acc[2] + acc[3]), sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// d += (rz_old / pAp) p  (the update deferred from cg_update: the same alpha bits), then
// p = z + (rz_new / rz_old) p,  z = M^{-1} r (z = r without preconditioner); rz_new is
// reduced here from cg_update's partials (CTA 0 stores it for the next iteration, the
// other slot of the ping-pong than the rz_old read here)
__global__ void __launch_bounds__(kRedThreads) cg_dir_kernel(const double* __restrict__ rr_partials,
                                                             double* __restrict__ rr_new,
                                                             const double* __restrict__ rr_old,
                                                             const double* __restrict__ pAp,
                                                             const double* __restrict__ r, double* __restrict__ p,
                                                             double* __restrict__ d, int64_t n,
                                                             const double* __restrict__ diag) {
  __shared__ double sh[kRedThreads];
  const double rn = reduce_partials(rr_partials, sh);
  if (blockIdx.x == 0 && threadIdx.x == 0) *rr_new = rn;
  const double beta = rn / *rr_old;
  const double alpha = *rr_old / *pAp;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (kUnroll - 1) * stride < n; i += kUnroll * stride) {
    double pv[kUnroll], rv[kUnroll], dv[kUnroll];
#pragma unroll
    for (int t = 0; t < kUnroll; ++t) {
      pv[t] = p[i + t * stride];
      dv[t] = d[i + t * stride];
      rv[t] = diag ? __ldcs(r + i + t * stride) / diag[i + t * stride] : __ldcs(r + i + t * stride);
    }
#pragma unroll
    for (int t = 0; t < kUnroll; ++t) {
      d[i + t * stride] = fma(alpha, pv[t], dv[t]);
      p[i + t * stride] = fma(beta, pv[t], rv[t]);
    }
  }
  for (; i < n; i += stride) {
    const double pv = p[i];
    d[i] = fma(alpha, pv, d[i]);
    p[i] = fma(beta, pv, diag ? r[i] / diag[i] : r[i]);
  }
}

// u += d
__global__ void axpy1_kernel(double* __restrict__ u, const double* __restrict__ d, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    u[i] += d[i];
}

static int grid_for(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return (int)(b < kRedBlocks ? (b > 0 ? b : 1) : kRedBlocks);
}

cudaError_t cg_init(const double* F, double* r, double* p, double* d, int64_t n, cudaStream_t st, const double* diag) {
  cg_init_kernel<<<grid_for(n), 256, 0, st>>>(F, r, p, d, diag, n);
  return cudaGetLastError();
}
cudaError_t cg_update(const double* rr, const double* pAp_partials, double* pAp, const double* Ap, double* r, int64_t n,
                      double* partials, int* bad, cudaStream_t st, const double* diag) {
  cg_update_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(rr, pAp_partials, pAp, Ap, r, n, partials, bad, diag);
  return cudaGetLastError();
}
cudaError_t cg_dir(const double* rr_partials, double* rr_new, const double* rr_old, const double* pAp, const double* r,
                   double* p, double* d, int64_t n, cudaStream_t st, const double* diag) {
  cg_dir_kernel<<<grid_for(n), kRedThreads, 0, st>>>(rr_partials, rr_new, rr_old, pAp, r, p, d, n, diag);
  return cudaGetLastError();
}
cudaError_t axpy1(double* u, const double* d, int64_t n, cudaStream_t st) {
  axpy1_kernel<<<grid_for(n), 256, 0, st>>>(u, d, n);
  return cudaGetLastError();
}

}  // namespace feod
