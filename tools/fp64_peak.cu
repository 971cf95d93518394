// K0: sustained FP64 DFMA throughput and a read-dominated HBM probe on one B200.
// Used once to fill the FP64 roofline denominator that MEASURED_PEAKS.json lacks
// (SURVEY.md §0.1 fact 6, §7.1 step 0). Output: one JSON line on stdout.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

// 8 independent FMA chains per thread hide the DFMA latency.
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], a, b);
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], b, a);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == 123.456) out[0] = s;
}

// DMMA (mma.sync m8n8k4 f64): 4 independent accumulator chains per warp
__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  double c[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 123.456) out[0] = s;
}

__global__ void read_kernel(const double2* __restrict__ p, size_t n, double* out) {
  double2 acc = make_double2(0, 0);
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double2 v = __ldcs(p + i);
    acc.x += v.x; acc.y += v.y;
  }
  if (acc.x == 123.456) out[0] = acc.y;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) b[i] = __ldcs(a + i);
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  // ---- DFMA ----
  int threads = 256, blocks = sms * 8, iters = 20000;
  dfma_kernel<<<blocks, threads>>>(out, 100, 0.999, 1e-7);
  CK(cudaDeviceSynchronize());
  float best = 1e30f, total = 0; int reps = 0;
  for (int r = 0; r < 40; ++r) {   // ~seconds of sustained load
    CK(cudaEventRecord(e0));
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-7);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms; total += ms; ++reps;
  }
  double flops = 2.0 * 16.0 * iters * (double)blocks * threads;
  double tf_burst = flops / (best * 1e-3) / 1e12;
  double tf_sust = flops / (total / reps * 1e-3) / 1e12;
  // ---- DMMA ----
  float dbest = 1e30f;
  for (int r = 0; r < 20; ++r) {
    CK(cudaEventRecord(e0));
    dmma_kernel<<<sms * 8, 256>>>(out, 20000);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < dbest) dbest = ms;
  }
  const double dmma_flops = 2.0 * 8 * 8 * 4 * 4 * 20000.0 * (sms * 8.0 * 256 / 32);
  const double dmma_tf = dmma_flops / (dbest * 1e-3) / 1e12;
  // ---- HBM read / copy ----
  size_t bytes = (size_t)4 << 30; size_t n2 = bytes / 16;
  double2 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
  CK(cudaMemset(a, 0, bytes)); CK(cudaMemset(b, 0, bytes));
  float rbest = 1e30f, cbest = 1e30f;
  for (int r = 0; r < 10; ++r) {
    CK(cudaEventRecord(e0)); read_kernel<<<sms * 16, 512>>>(a, n2, out); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1)); float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < rbest) rbest = ms;
    CK(cudaEventRecord(e0)); copy_kernel<<<sms * 16, 512>>>(a, b, n2 / 2); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < cbest) cbest = ms;
  }
  double read_gbs = bytes / (rbest * 1e-3) / 1e9;
  double copy_gbs = 2.0 * (bytes / 2) / (cbest * 1e-3) / 1e9;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"fp64_tflops_burst\": %.3f, \"fp64_tflops_sustained\": %.3f, "
         "\"hbm_read_gbs\": %.1f, \"hbm_copy_gbs\": %.1f, \"dfma_kernel_ms_best\": %.4f, \"dmma_tflops_burst\": %.3f}\n",
         prop.name, sms, tf_burst, tf_sust, read_gbs, copy_gbs, best, dmma_tf);
  return 0;
}
