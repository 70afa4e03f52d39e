// Device-side entry helpers: sm_100a check and CUDA error mapping.
#pragma once
#include <cuda_runtime.h>

#include "../common.h"

namespace skr {

// SKR_OK iff the current device is compute capability 10.0 (B200, sm_100a).
inline skr_status check_sm100() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(SKR_E_UNSUPPORTED, "no CUDA device");
  int maj = 0, min = 0;
  cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&min, cudaDevAttrComputeCapabilityMinor, dev);
  if (maj != 10 || min != 0) return fail(SKR_E_UNSUPPORTED, "needs an sm_100a device, found sm_%d%d", maj, min);
  return SKR_OK;
}

// SM count of the CURRENT device (cached per device ordinal: a process may drive several GPUs).
inline int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

inline skr_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return SKR_OK;
  return fail(SKR_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

inline skr_status launch_status(const char* what) { return cuda_status(cudaGetLastError(), what); }

}  // namespace skr
