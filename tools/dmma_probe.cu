// Probe: FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput on B200, alone
// and concurrently with vector DFMA, to decide whether the sum-factorised
// contractions should move to DMMA. Output: one JSON line.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// mode 0: DMMA only; 1: DFMA only; 2: both in every warp (independent chains)
template <int MODE>
__global__ void probe(double* out, int iters, double a, double b) {
  double acc[8][2];
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) { acc[c][0] = acc[c][1] = threadIdx.x * 1e-9 + c; x[c] = c + 0.5; }
  for (int it = 0; it < iters; ++it) {
    if (MODE != 1) {
#pragma unroll
      for (int c = 0; c < 8; ++c) dmma(acc[c][0], acc[c][1], a, b);
    }
    if (MODE != 0) {
#pragma unroll
      for (int c = 0; c < 8; ++c) x[c] = fma(x[c], a, b);
#pragma unroll
      for (int c = 0; c < 8; ++c) x[c] = fma(x[c], b, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1] + x[c];
  if (s == 123.456) out[0] = s;
}

template <int MODE>
double run(int blocks, int threads, int iters, double* d) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  probe<MODE><<<blocks, threads>>>(d, iters, 1.0000001, 1e-12);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  probe<MODE><<<blocks, threads>>>(d, iters, 1.0000001, 1e-12);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms * 1e-3;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* d; CK(cudaMalloc(&d, 8));
  const int threads = 256, blocks = sms * 4, iters = 20000;
  const double warps = (double)blocks * threads / 32;
  const double t0 = run<0>(blocks, threads, iters, d);
  const double t1 = run<1>(blocks, threads, iters, d);
  const double t2 = run<2>(blocks, threads, iters, d);
  const double dmma_flops = warps * iters * 8 * 512.0;          // 8 DMMA x (8x8x4 FMA x 2)
  const double dfma_flops = warps * 32 * iters * 16 * 2.0;      // 16 DFMA per thread
  printf("{\"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f, \"both_s\": %.6f, \"dmma_s\": %.6f, \"dfma_s\": %.6f, "
         "\"both_tflops\": %.2f}\n", dmma_flops / t0 * 1e-12, dfma_flops / t1 * 1e-12, t2, t0, t1,
         (dmma_flops + dfma_flops) / t2 * 1e-12);
  return 0;
}
