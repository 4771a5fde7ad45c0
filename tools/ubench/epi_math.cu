// Throughput of the MLP epilogue's per-value math on one SM sub-partition mix (B200):
// z = fma(acc, s, t); a = tanh via 1 - 2 / (1 + 2^z); h += a — for 16 independent values
// per thread, as in mlp_tc.cu's hidden-layer epilogue, repeated R times.
//  variant 0: ex2.approx + rcp.approx (two MUFU ops per value, the kernel's form)
//  variant 1: ex2.approx + bit-trick seed and three Newton steps (one MUFU op)
//  variant 2: tanh.approx (one MUFU op; not fp32-accurate, for reference)
//  variant 3: FMA-only work of the same instruction count as variant 0 (no MUFU)
// Reports cycles per 16 values per warp for W warps per SM (1 CTA per SM, 148 CTAs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o epi_math epi_math.cu && ./epi_math
#include <cstdio>
#include <cstdint>

template <int VAR>
__device__ __forceinline__ float act(float z) {
  float a;
  if (VAR == 0) {
    float ez, r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ez) : "f"(z));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + ez));
    a = fmaf(-2.0f, r, 1.0f);
  } else if (VAR == 1) {
    float ez;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ez) : "f"(fminf(z, 64.0f)));
    const float d = 1.0f + ez;
    float r = __int_as_float(0x7EF311C7 - __float_as_int(d));
    r = fmaf(r, fmaf(-d, r, 1.0f), r);
    r = fmaf(r, fmaf(-d, r, 1.0f), r);
    r = fmaf(r, fmaf(-d, r, 1.0f), r);
    a = fmaf(-2.0f, r, 1.0f);
  } else if (VAR == 2) {
    asm("tanh.approx.f32 %0, %1;" : "=f"(a) : "f"(z));
  } else {
    const float e = fmaf(z, 0.5f, 1.0f);
    a = fmaf(-2.0f, fmaf(e, 0.25f, 0.5f), 1.0f);
  }
  return a;
}

template <int VAR>
__global__ void bench(const float* __restrict__ st, float* out, long long* cyc, int reps) {
  float h[16], v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { h[i] = 0.f; v[i] = 0.01f * (threadIdx.x + i); }
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float z = fmaf(v[i], st[i], st[16 + i]);
      h[i] += act<VAR>(z);
      v[i] = h[i] * 0.5f;
    }
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += h[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int VAR>
void run(int warps, float* st, float* out, long long* cyc) {
  const int reps = 256;
  bench<VAR><<<148, 32 * warps>>>(st, out, cyc, reps);
  bench<VAR><<<148, 32 * warps>>>(st, out, cyc, reps);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 148; ++i) m += h[i];
  m /= 148;
  printf("variant %d warps/SM %2d (%d per SMSP): %7.1f cycles per 16 values per warp, "
         "%6.1f cycles per 16 values x all warps of one SMSP\n",
         VAR, warps, warps / 4, m / reps, m / reps);
}

int main() {
  float *st, *out;
  long long* cyc;
  cudaMalloc(&st, 32 * sizeof(float));
  float hs[32];
  for (int i = 0; i < 32; ++i) hs[i] = i < 16 ? 0.5f : 0.1f;
  cudaMemcpy(st, hs, sizeof(hs), cudaMemcpyHostToDevice);
  cudaMalloc(&out, 148 * 1024 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  for (int w : {4, 8, 12, 16}) {
    run<0>(w, st, out, cyc);
    run<1>(w, st, out, cyc);
    run<2>(w, st, out, cyc);
    run<3>(w, st, out, cyc);
  }
  return 0;
}
