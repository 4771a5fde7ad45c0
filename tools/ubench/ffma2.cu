// Throughput of FFMA (3-register form) vs FFMA2 (paired fp32) on one SM pipe.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k1(float* out, float a, float b, int n) {
  float c[8];
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x + i;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fmaf(c[i], a, b + c[(i + 1) & 7] * 0.f);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k1r(float* out, float a, float b, int n) {  // pure register FFMA chains
  float c[8], x[8];
  for (int i = 0; i < 8; ++i) { c[i] = threadIdx.x + i; x[i] = a + i * 1e-3f; }
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fmaf(c[i], x[i], x[(i + 3) & 7]);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k2(float* out, float a, float b, int n) {
  float2 c[8], x[8];
  for (int i = 0; i < 8; ++i) { c[i] = make_float2(threadIdx.x + i, i); x[i] = make_float2(a + i * 1e-3f, a); }
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = __ffma2_rn(c[i], x[i], x[(i + 3) & 7]);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += c[i].x + c[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int n = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0);
    k1r<<<148 * 8, 256>>>(out, 1.0001f, 1e-3f, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * n * 148.0 * 8 * 256;
    printf("FFMA  (reg): %.1f TFLOP/s\n", fl / ms / 1e9);
    cudaEventRecord(e0);
    k2<<<148 * 8, 256>>>(out, 1.0001f, 1e-3f, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA2 (reg): %.1f TFLOP/s\n", 2 * fl / ms / 1e9);
  }
  return 0;
}
