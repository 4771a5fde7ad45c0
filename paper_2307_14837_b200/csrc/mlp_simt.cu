// K4 (generic path): eval-mode patch MLP in fp32 FFMA for any widths.
//
// Reference: net._forward eval branch (net.py:124-159):
//   h = (X - input_mean) / input_std
//   layer i < depth: z = h W_i; a = act((z - rm_i)/sqrt(rv_i + eps) * gamma_i + beta_i);
//                    h = a (+ h for i >= 1)
//   head: Y = h W_depth
// BN is folded on the host into bn_scale/bn_shift.  This kernel serves every
// width (J=2's 1024 -> 512 and config 4's H = 1024) and the fp32 reference mode;
// the tcgen05 kernels (mlp_tc.cu) are the fast paths for H = 256.
#include "common.cuh"

namespace dnnmg {

constexpr int kRT = 16;       // rows per tile
constexpr int kThreads = 256;

__device__ __forceinline__ float activate(float x, int act) {
  return act == DNNMG_ACT_TANH ? tanhf(x) : fmaxf(x, 0.f);
}

struct MlpArgs {
  int n_in, H, depth, n_out, act, width;  // width = max(n_in, H), padded to 4
  const float* W[DNNMG_MAX_LAYERS];
  const float* scale;
  const float* shift;
  const float* in_mean;
  const float* in_std;
  const float* X;
  float* Y;
  int64_t n_rows;
};

// acc[r] += h[r][k] * W[k][n] over k, h in smem (row stride `ld`)
__device__ __forceinline__ void dot_rows(const float* __restrict__ h, int ld, int K,
                                         const float* __restrict__ W, int ncols, int n,
                                         float acc[kRT]) {
  int k = 0;
  for (; k + 4 <= K; k += 4) {
    const float w0 = __ldg(W + (int64_t)k * ncols + n);
    const float w1 = __ldg(W + (int64_t)(k + 1) * ncols + n);
    const float w2 = __ldg(W + (int64_t)(k + 2) * ncols + n);
    const float w3 = __ldg(W + (int64_t)(k + 3) * ncols + n);
#pragma unroll
    for (int r = 0; r < kRT; ++r) {
      const float4 hv = *reinterpret_cast<const float4*>(h + r * ld + k);
      acc[r] = fmaf(hv.x, w0, acc[r]);
      acc[r] = fmaf(hv.y, w1, acc[r]);
      acc[r] = fmaf(hv.z, w2, acc[r]);
      acc[r] = fmaf(hv.w, w3, acc[r]);
    }
  }
  for (; k < K; ++k) {
    const float w = __ldg(W + (int64_t)k * ncols + n);
#pragma unroll
    for (int r = 0; r < kRT; ++r) acc[r] = fmaf(h[r * ld + k], w, acc[r]);
  }
}

__global__ void __launch_bounds__(kThreads) mlp_simt_kernel(MlpArgs A) {
  extern __shared__ float sm[];
  const int ld = A.width;
  float* hA = sm;
  float* hB = sm + kRT * ld;
  const int64_t n_tiles = (A.n_rows + kRT - 1) / kRT;
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int64_t row0 = tile * kRT;
    // input normalisation (net.py:131)
    for (int i = threadIdx.x; i < kRT * A.n_in; i += kThreads) {
      const int r = i / A.n_in, c = i - r * A.n_in;
      const int64_t row = row0 + r;
      float v = 0.f;
      if (row < A.n_rows) v = (A.X[row * A.n_in + c] - A.in_mean[c]) / A.in_std[c];
      hA[r * ld + c] = v;
    }
    __syncthreads();
    int K = A.n_in;
    for (int layer = 0; layer < A.depth; ++layer) {
      const float* W = A.W[layer];
      const float* sc = A.scale + layer * A.H;
      const float* sh = A.shift + layer * A.H;
      for (int n = threadIdx.x; n < A.H; n += kThreads) {
        float acc[kRT];
#pragma unroll
        for (int r = 0; r < kRT; ++r) acc[r] = 0.f;
        dot_rows(hA, ld, K, W, A.H, n, acc);
        const float s = sc[n], b = sh[n];
#pragma unroll
        for (int r = 0; r < kRT; ++r) {
          float a = activate(fmaf(acc[r], s, b), A.act);
          if (layer >= 1) a += hA[r * ld + n];  // skip (net.py:151)
          hB[r * ld + n] = a;
        }
      }
      __syncthreads();
      float* tmp = hA; hA = hB; hB = tmp;
      K = A.H;
    }
    const float* W = A.W[A.depth];
    for (int n = threadIdx.x; n < A.n_out; n += kThreads) {
      float acc[kRT];
#pragma unroll
      for (int r = 0; r < kRT; ++r) acc[r] = 0.f;
      dot_rows(hA, ld, K, W, A.n_out, n, acc);
#pragma unroll
      for (int r = 0; r < kRT; ++r) {
        const int64_t row = row0 + r;
        if (row < A.n_rows) A.Y[row * A.n_out + n] = acc[r];
      }
    }
    __syncthreads();
    if (hA != sm) {  // keep the buffer roles stable across tiles
      float* tmp = hA; hA = hB; hB = tmp;
    }
  }
}

int32_t launch_mlp_simt(const dnnmg_mlp_t* m, const float* X, int64_t n_rows, float* Y,
                        cudaStream_t s) {
  MlpArgs A;
  A.n_in = m->n_in;
  A.H = m->n_hidden;
  A.depth = m->depth;
  A.n_out = m->n_out;
  A.act = m->activation;
  A.width = ((m->n_in > m->n_hidden ? m->n_in : m->n_hidden) + 3) / 4 * 4;
  for (int i = 0; i <= m->depth; ++i) A.W[i] = m->W[i];
  A.scale = m->bn_scale;
  A.shift = m->bn_shift;
  A.in_mean = m->in_mean;
  A.in_std = m->in_std;
  A.X = X;
  A.Y = Y;
  A.n_rows = n_rows;
  const size_t smem = sizeof(float) * 2 * kRT * A.width;
  DNNMG_REQUIRE(smem <= 200 * 1024, DNNMG_ERR_UNSUPPORTED, "mlp: layer width %d too large", A.width);
  cudaFuncSetAttribute(mlp_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t tiles = (n_rows + kRT - 1) / kRT;
  int blocks = (int)(tiles < kSMs * 8 ? tiles : kSMs * 8);
  if (blocks < 1) return DNNMG_OK;
  mlp_simt_kernel<<<blocks, kThreads, smem, s>>>(A);
  DNNMG_CHECK_LAUNCH("mlp_simt_kernel");
  return DNNMG_OK;
}

}  // namespace dnnmg
