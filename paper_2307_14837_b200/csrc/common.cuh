// Shared helpers for the sm_100a kernels of the DNN-MG correction step.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "dnnmg_b200.h"

namespace dnnmg {

// Records a detail message for dnnmg_last_error() and returns the status.
int32_t set_error(int32_t status, const char* fmt, ...);

inline cudaStream_t as_stream(dnnmg_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

#define DNNMG_CHECK_LAUNCH(name)                                                   \
  do {                                                                             \
    cudaError_t _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess)                                                         \
      return ::dnnmg::set_error(DNNMG_ERR_CUDA, "%s: %s", name, cudaGetErrorString(_e)); \
  } while (0)

#define DNNMG_REQUIRE(cond, code, ...)                                             \
  do {                                                                             \
    if (!(cond)) return ::dnnmg::set_error(code, __VA_ARGS__);                     \
  } while (0)

constexpr int kSMs = 148;  // B200

// true the first time it is called on the current device for this `seen` mask: kernel
// attributes (dynamic shared memory limits) are per device, so one process driving several
// GPUs must set them on each
inline bool first_use_on_device(uint64_t& seen) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (seen & bit) return false;
  seen |= bit;
  return true;
}

inline int grid_for(int64_t n, int block, int max_waves = 64) {
  int64_t g = (n + block - 1) / block;
  int64_t cap = (int64_t)kSMs * max_waves;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// 1-D Q2 basis on {0, 1/2, 1} (elements.py:34-46)
__host__ __device__ inline void q2_1d(double x, double* v, double* d) {
  v[0] = 2.0 * (x - 0.5) * (x - 1.0);
  v[1] = 4.0 * x * (1.0 - x);
  v[2] = 2.0 * x * (x - 0.5);
  d[0] = 4.0 * x - 3.0;
  d[1] = 4.0 - 8.0 * x;
  d[2] = 4.0 * x - 1.0;
}

}  // namespace dnnmg
