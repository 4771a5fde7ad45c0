// Probe of two tcgen05 features the K2 v2 design relies on (run on the B200):
//  (1) kind::f16 MMA with the A operand in TMEM (row r = lane r, two fp16 per 32-bit column)
//  (2) a shared-memory B descriptor with LBO = 0 (both K core-matrix groups read the same bytes)
// A[128][16] written by tcgen05.st, B[32][16] canonical K-major in smem, D[128][32] fp32.
// mode 0: B desc LBO = 128 (distinct K groups); mode 1: LBO = 0.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tc_probe tc_probe.cu && ./tc_probe
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_fp16.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__global__ void probe(const __half* A, const __half* B, float* D, int mode, int acol) {
  __shared__ __align__(1024) uint8_t sB[2048];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5;
  // B: rows n (0..31) x K 16; K group kg at kg*128 (mode 0) ; row groups at SBO 256 (mode 0)
  // mode 1: only K group 0 stored, row groups at SBO 128, LBO 0
  for (int i = t; i < 32 * 16; i += blockDim.x) {
    const int n = i / 16, k = i % 16;
    uint32_t off;
    if (mode == 0) off = (n >> 3) * 256 + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2;
    else { if (k >= 8) continue; off = (n >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2; }
    *reinterpret_cast<__half*>(sB + off) = B[i];
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  // A row t -> TMEM lane t, columns acol..acol+7 (k pairs)
  {
    uint32_t r[8];
    for (int j = 0; j < 8; ++j) {
      __half2 h = __halves2half2(A[t * 16 + 2 * j], A[t * 16 + 2 * j + 1]);
      r[j] = *reinterpret_cast<uint32_t*>(&h);
    }
    const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + acol;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (t == 0) {
    const uint64_t bd = mode == 0 ? sdesc(smem_u32(sB), 128, 256) : sdesc(smem_u32(sB), 0, 128);
    const uint32_t id = (1u << 4) | (0u << 7) | (0u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t d = tmem + 64, a = tmem + acol;
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a),
                 "l"(bd), "r"(id), "r"(0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c = 0; c < 32; c += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + 64 + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) D[t * 32 + c + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
  __half *A, *B;
  float* D;
  cudaMallocManaged(&A, 128 * 16 * 2);
  cudaMallocManaged(&B, 32 * 16 * 2);
  cudaMallocManaged(&D, 128 * 32 * 4);
  int fails = 0;
  for (int mode = 0; mode < 2; ++mode)
    for (int acol = 0; acol < 16; acol += 4) {
      srand(1 + mode + acol);
      for (int i = 0; i < 128 * 16; ++i) A[i] = __float2half((float)(rand() % 17 - 8));
      for (int i = 0; i < 32 * 16; ++i) {
        const int k = i % 16;
        B[i] = __float2half((float)(rand() % 13 - 6));
        if (mode == 1 && k >= 8) B[i] = B[i - 8];   // both K groups equal (LBO 0)
      }
      probe<<<1, 128>>>(A, B, D, mode, acol);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("mode %d acol %d: %s\n", mode, acol, cudaGetErrorString(e)); return 1; }
      double maxerr = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 32; ++n) {
          double s = 0;
          for (int k = 0; k < 16; ++k) s += (double)__half2float(A[m * 16 + k]) * __half2float(B[n * 16 + k]);
          maxerr = fmax(maxerr, fabs(s - D[m * 32 + n]));
        }
      printf("mode %d (LBO %s) A at TMEM col %2d: max |err| %g %s\n", mode, mode ? "0" : "128", acol, maxerr,
             maxerr == 0 ? "OK" : "MISMATCH");
      fails += maxerr != 0;
    }
  return fails ? 2 : 0;
}
