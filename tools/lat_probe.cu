// Latency / throughput probe for the FP64 design (one warp, clock64 timing):
// dependent DFMA chain, dependent SHFL chain (64-bit), dependent LDS.64 chain,
// and DFMA throughput with 1..8 independent chains per warp, 1..16 warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_dfma(double* out, long long* cyc, double a, double b, int n) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = fma(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lat_shfl(double* out, long long* cyc, int n) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lat_lds(double* out, long long* cyc, int n) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (double)((i * 7 + 1) & 1023);
  __syncthreads();
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x = s[(int)x];
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int C>
__global__ void thr_dfma(double* out, long long* cyc, double a, double b, int n) {
  double x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) x[c] = threadIdx.x * 1e-3 + c;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int c = 0; c < C; ++c) x[c] = fma(x[c], a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 1 << 16);
  long long h;
  const int n = 4096;
  lat_dfma<<<1, 32>>>(out, cyc, 0.999, 1e-3, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"dfma_dep_latency_cyc\": %.2f,", (double)h / (16.0 * n));
  lat_shfl<<<1, 32>>>(out, cyc, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf(" \"shfl64_dep_latency_cyc\": %.2f,", (double)h / (16.0 * n));
  lat_lds<<<1, 32>>>(out, cyc, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf(" \"lds64_dep_latency_cyc\": %.2f,", (double)h / (16.0 * n));
  // throughput: per-SM DFMA/clk with W warps and C chains
  printf(" \"dfma_per_clk_per_sm\": {");
  int first = 1;
  for (int w : {1, 2, 4, 8, 16}) {
    for (int c : {1, 2, 4, 8}) {
      auto k = c == 1 ? thr_dfma<1> : c == 2 ? thr_dfma<2> : c == 4 ? thr_dfma<4> : thr_dfma<8>;
      k<<<148, 32 * w>>>(out, cyc, 0.999, 1e-3, 512);
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      const double fl = 32.0 * w * c * 8 * 512;
      printf("%s\"w%d_c%d\": %.1f", first ? "" : ", ", w, c, fl / (double)h);
      first = 0;
    }
  }
  printf("}}\n");
  return 0;
}
