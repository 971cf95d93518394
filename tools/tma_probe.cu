// TMA bulk-copy probe: CTAs stream a 805 MB buffer into shared memory with
// cp.async.bulk + mbarrier complete_tx, D copies of S bytes in flight per CTA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void tma_stream(const double* src, size_t nchunks, int chunk_bytes, int depth, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  unsigned char* buf = sm + 128;
  if (threadIdx.x == 0) {
    for (int d = 0; d < depth; ++d) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar + d)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double acc = 0;
  size_t it = 0;
  // chunk c handled by CTA c % gridDim.x
  auto issue = [&](size_t c, int d) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar + d)), "r"(chunk_bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su(buf + (size_t)d * chunk_bytes)), "l"((const char*)src + c * chunk_bytes), "r"(chunk_bytes),
                   "r"(su(bar + d)) : "memory");
    }
  };
  size_t c0 = blockIdx.x;
  for (int d = 0; d < depth && c0 + (size_t)d * gridDim.x < nchunks; ++d) issue(c0 + (size_t)d * gridDim.x, d);
  for (size_t c = c0; c < nchunks; c += gridDim.x, ++it) {
    const int d = it % depth;
    const uint32_t par = (it / depth) & 1;
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(su(bar + d)), "r"(par) : "memory");
    acc += reinterpret_cast<const double*>(buf + (size_t)d * chunk_bytes)[threadIdx.x];
    __syncthreads();
    const size_t cn = c + (size_t)depth * gridDim.x;
    if (cn < nchunks) issue(cn, d);
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  const size_t bytes = 805306368;
  double* src;
  double* out;
  cudaMalloc(&src, bytes);
  cudaMalloc(&out, 64);
  cudaMemset(src, 0, bytes);
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  printf("{");
  int first = 1;
  for (int cb : {768, 6144, 24576}) {
    for (int depth : {1, 2, 4}) {
      for (int cps : {1, 3}) {
        const size_t n = bytes / cb;
        const int smem = 128 + depth * cb;
        if (smem * cps > 220 * 1024) continue;
        tma_stream<<<148 * cps, 32, smem>>>(src, n, cb, depth, out);
        cudaEventRecord(a);
        tma_stream<<<148 * cps, 32, smem>>>(src, n, cb, depth, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%s\"c%d_d%d_cta%d\": {\"GBps\": %.0f, \"us_per_copy_per_cta\": %.2f}", first ? "" : ", ", cb, depth, cps,
               bytes / (ms * 1e-3) / 1e9, ms * 1e3 / ((double)n / (148 * cps)));
        first = 0;
      }
    }
  }
  printf("}\n");
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
