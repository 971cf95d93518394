// Order dispatch of the fused operator kernels.
#include <map>
#include <mutex>
#include <utility>

#include "kernels.h"

namespace feod {

cudaError_t persistent_slots(const void* kernel, int threads, size_t smem, int* slots) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;   // (kernel, device) -> SMs x occupancy
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({kernel, dev});
    if (it != cache.end()) { *slots = it->second; return cudaSuccess; }
  }
  int sms = 0, occ = 0;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem)) != cudaSuccess) return e;
  const int s = sms * (occ > 0 ? occ : 1);
  std::lock_guard<std::mutex> lk(mu);
  cache[{kernel, dev}] = s;
  *slots = s;
  return cudaSuccess;
}

bool brick_info_nd(int nd, BrickInfo* bi) {
  switch (nd) {
    case 2: return brick_info<2>(bi);
    case 3: return brick_info<3>(bi);
    case 4: return brick_info<4>(bi);
    case 5: return brick_info<5>(bi);
    case 6: return brick_info<6>(bi);
    case 7: return brick_info<7>(bi);
  }
  return false;
}

cudaError_t prepare_nd(int nd) {
  switch (nd) {
    case 2: return prepare_order<2>();
    case 3: return prepare_order<3>();
    case 4: return prepare_order<4>();
    case 5: return prepare_order<5>();
    case 6: return prepare_order<6>();
    case 7: return prepare_order<7>();
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_nd(int nd, int mode, int model, bool affine, int grid, const OpParams& P, const Tables& T,
                      const OpPtrs& p, cudaStream_t st, int* grid_out) {
  switch (nd) {
    case 2: return launch_order<2>(mode, model, affine, grid, P, T, p, st, grid_out);
    case 3: return launch_order<3>(mode, model, affine, grid, P, T, p, st, grid_out);
    case 4: return launch_order<4>(mode, model, affine, grid, P, T, p, st, grid_out);
    case 5: return launch_order<5>(mode, model, affine, grid, P, T, p, st, grid_out);
    case 6: return launch_order<6>(mode, model, affine, grid, P, T, p, st, grid_out);
    case 7: return launch_order<7>(mode, model, affine, grid, P, T, p, st, grid_out);
  }
  return cudaErrorInvalidValue;
}

cudaError_t fixup_nd(int nd, const OpParams& P, const double* shell0, double* out0, const double* shell1,
                     double* out1, cudaStream_t st) {
  switch (nd) {
    case 2: return fixup_order<2>(P, shell0, out0, shell1, out1, st);
    case 3: return fixup_order<3>(P, shell0, out0, shell1, out1, st);
    case 4: return fixup_order<4>(P, shell0, out0, shell1, out1, st);
    case 5: return fixup_order<5>(P, shell0, out0, shell1, out1, st);
    case 6: return fixup_order<6>(P, shell0, out0, shell1, out1, st);
    case 7: return fixup_order<7>(P, shell0, out0, shell1, out1, st);
  }
  return cudaErrorInvalidValue;
}

int fixup_rows_nd(int nd, const OpParams& P, int2* rows, unsigned long long* keys) {
  switch (nd) {
    case 2: return fixup_rows_order<2>(P, rows, keys);
    case 3: return fixup_rows_order<3>(P, rows, keys);
    case 4: return fixup_rows_order<4>(P, rows, keys);
    case 5: return fixup_rows_order<5>(P, rows, keys);
    case 6: return fixup_rows_order<6>(P, rows, keys);
    case 7: return fixup_rows_order<7>(P, rows, keys);
  }
  return -1;
}

}  // namespace feod
