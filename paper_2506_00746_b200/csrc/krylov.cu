// K7 — BiCGStab vector kernels for the adjoint solve J(u)^T lambda = rhs
// (feod_adjoint_solve). Fixed iteration count, every scalar
// stays on the device (sc[]), and every dot product is the deterministic
// fixed-grid two-stage reduction of blas1.cu, so a solve is bitwise
// reproducible. Scalars: sc[0..1] rho ping-pong, sc[2] alpha, sc[3] omega,
// sc[4] (rhat, v), sc[5] (t, s), sc[6] (t, t), sc[7] (r, r).
#include "common.cuh"
#include "kernels.h"

namespace feod {

constexpr int kKThreads = 256;

static int kgrid(int64_t n) {
  const int64_t b = (n + kKThreads - 1) / kKThreads;
  return (int)(b < kRedBlocks ? (b > 0 ? b : 1) : kRedBlocks);
}

// p = r + beta (p - omega v),  beta = (rho_new / rho_old) (alpha / omega)
__global__ void bicg_p_kernel(const double* __restrict__ sc, int it, const double* __restrict__ r,
                              const double* __restrict__ v, double* __restrict__ p, int64_t n) {
  const double rho_new = sc[it & 1], rho_old = sc[(it + 1) & 1];
  const double alpha = sc[2], omega = sc[3];
  // a converged solve (r = 0) freezes: alpha = omega = beta = 0 keep x as it is
  const double beta = (it == 0 || rho_old == 0.0 || omega == 0.0) ? 0.0 : (rho_new / rho_old) * (alpha / omega);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    p[i] = it == 0 ? r[i] : fma(beta, fma(-omega, v[i], p[i]), r[i]);
}

// alpha = rho_new / (rhat, v);  s = r - alpha v
__global__ void bicg_s_kernel(double* __restrict__ sc, int it, const double* __restrict__ r,
                              const double* __restrict__ v, double* __restrict__ s, int64_t n, int* bad) {
  const double rv = sc[4], rho = sc[it & 1];
  const double alpha = rv != 0.0 ? rho / rv : 0.0;
  if (blockIdx.x == 0 && threadIdx.x == 0 && rv == 0.0 && rho != 0.0) *bad = 1;   // breakdown, not convergence
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) s[i] = fma(-alpha, v[i], r[i]);
}

__global__ void bicg_alpha_kernel(double* __restrict__ sc, int it) {
  if (threadIdx.x == 0) sc[2] = sc[4] != 0.0 ? sc[it & 1] / sc[4] : 0.0;
}

// omega = (t, s) / (t, t);  x += alpha p + omega s;  r = s - omega t;
// block partials of (rhat, r) and (r, r) (fixed grid)
__global__ void __launch_bounds__(kKThreads) bicg_x_kernel(double* __restrict__ sc, const double* __restrict__ p,
                                                           const double* __restrict__ s, const double* __restrict__ t,
                                                           const double* __restrict__ rhat, double* __restrict__ x,
                                                           double* __restrict__ r, int64_t n,
                                                           double* __restrict__ part_rr, double* __restrict__ part_r2,
                                                           int* bad) {
  __shared__ double sh[2][kKThreads];
  const double tt = sc[6];
  const double omega = tt > 0.0 ? sc[5] / tt : 0.0, alpha = sc[2];   // t = 0 only when s = 0 (J nonsingular)
  (void)bad;
  double a0 = 0.0, a1 = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kKThreads + threadIdx.x; i < n; i += (int64_t)kRedBlocks * kKThreads) {
    x[i] = fma(omega, s[i], fma(alpha, p[i], x[i]));
    const double ri = fma(-omega, t[i], s[i]);
    r[i] = ri;
    a0 = fma(rhat[i], ri, a0);
    a1 = fma(ri, ri, a1);
  }
  sh[0][threadIdx.x] = a0;
  sh[1][threadIdx.x] = a1;
  __syncthreads();
  for (int k = kKThreads / 2; k > 0; k >>= 1) {
    if ((int)threadIdx.x < k) {
      sh[0][threadIdx.x] += sh[0][threadIdx.x + k];
      sh[1][threadIdx.x] += sh[1][threadIdx.x + k];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part_rr[blockIdx.x] = sh[0][0];
    part_r2[blockIdx.x] = sh[1][0];
  }
}

__global__ void bicg_omega_kernel(double* __restrict__ sc) {
  if (threadIdx.x == 0) sc[3] = sc[6] > 0.0 ? sc[5] / sc[6] : 0.0;
}

// x = 0, r = rhat = b (b's Dirichlet entries already zero), p = v = 0
__global__ void bicg_init_kernel(const double* __restrict__ b, double* __restrict__ x, double* __restrict__ r,
                                 double* __restrict__ rhat, double* __restrict__ p, double* __restrict__ v, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double bi = b[i];
    x[i] = 0.0; r[i] = bi; rhat[i] = bi; p[i] = 0.0; v[i] = 0.0;
  }
}

// P^T on a vector: zero its Dirichlet rows
__global__ void mask_dir_kernel(double* __restrict__ x, const OpParams P) {
  const int64_t n = (int64_t)P.Mx * P.My * P.Mz;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int X = (int)(i % P.Mx);
    const int64_t yz = i / P.Mx;
    const int Y = (int)(yz % P.My), Z = (int)(yz / P.My);
    if (is_dirichlet(X, Y, Z, P.Mx, P.My, P.Mz, P.faces)) x[i] = 0.0;
  }
}

cudaError_t mask_dirichlet(double* x, const OpParams& P, cudaStream_t st) {
  mask_dir_kernel<<<kgrid((int64_t)P.Mx * P.My * P.Mz), kKThreads, 0, st>>>(x, P);
  return cudaGetLastError();
}

cudaError_t bicg_init(const double* b, double* x, double* r, double* rhat, double* p, double* v, int64_t n,
                      cudaStream_t st) {
  bicg_init_kernel<<<kgrid(n), kKThreads, 0, st>>>(b, x, r, rhat, p, v, n);
  return cudaGetLastError();
}
cudaError_t bicg_p(const double* sc, int it, const double* r, const double* v, double* p, int64_t n, cudaStream_t st) {
  bicg_p_kernel<<<kgrid(n), kKThreads, 0, st>>>(sc, it, r, v, p, n);
  return cudaGetLastError();
}
cudaError_t bicg_s(double* sc, int it, const double* r, const double* v, double* s, int64_t n, int* bad,
                   cudaStream_t st) {
  bicg_alpha_kernel<<<1, 32, 0, st>>>(sc, it);
  bicg_s_kernel<<<kgrid(n), kKThreads, 0, st>>>(sc, it, r, v, s, n, bad);
  return cudaGetLastError();
}
cudaError_t bicg_x(double* sc, const double* p, const double* s, const double* t, const double* rhat, double* x,
                   double* r, int64_t n, double* part_rr, double* part_r2, int* bad, cudaStream_t st) {
  bicg_omega_kernel<<<1, 32, 0, st>>>(sc);
  bicg_x_kernel<<<kRedBlocks, kKThreads, 0, st>>>(sc, p, s, t, rhat, x, r, n, part_rr, part_r2, bad);
  return cudaGetLastError();
}

}  // namespace feod
