// Issue rate of back-to-back kind::f16 tcgen05.mma (M = 128, K = 16) by one thread, per code
// pattern and N (B200): cycles per MMA from the first issue to the commit's mbarrier phase.
//  pattern 0: lane 0 only (divergent branch), one asm statement per MMA
//  pattern 1: whole warp, elect.sync inside each MMA's asm statement
//  pattern 2: whole warp, one asm statement issuing 8 MMAs under one elect.sync
//  pattern 3: as 1 with the A operand in TMEM (columns 256..263)
//   nvcc -gencode arch=compute_100a,code=sm_100a -o mma_issue mma_issue.cu && ./mma_issue
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}

template <int PAT, int N>
__global__ void bench(long long* out, int reps) {
  __shared__ __align__(1024) uint8_t s[40960];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 40960 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(s)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t id = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  const uint64_t da = sdesc(smem_u32(s), 128, 256), db = sdesc(smem_u32(s + 32768), 128, 256);
  long long t0 = clock64();
  if (PAT == 0) {
    if (lane == 0) {
      for (int r = 0; r < reps; ++r)
#pragma unroll
        for (int k = 0; k < 8; ++k)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(N == 256 ? 256u * (k & 1) : 0u + 32 * (k & 3)),
                       "l"(da + 2 * k), "l"(db + 2 * k), "r"(id), "r"(1u));
    }
  } else if (PAT == 1) {
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k)
        asm volatile("{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(N == 256 ? 256u * (k & 1) : 0u + 32 * (k & 3)),
                     "l"(da + 2 * k), "l"(db + 2 * k), "r"(id), "r"(1u));
  } else if (PAT == 3) {
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k)
        asm volatile("{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(0u + 32 * (k & 3)),
                     "r"(256u + 8 * (k & 1)), "l"(db + 2 * k), "r"(id), "r"(1u));
  } else {
    for (int r = 0; r < reps; ++r)
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %3, %4, 1;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %3, %4, 1;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %3, %4, 1;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %3, %4, 1;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %3, %4, 1;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %3, %4, 1;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %3, %4, 1;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %3, %4, 1;\n\t}" ::"r"(0u),
          "r"(N == 256 ? 256u : 64u), "l"(da), "l"(db), "r"(id));
  }
  long long t1 = clock64();
  if (lane == 0)
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(&bar)));
  long long t2 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  asm volatile("tcgen05.fence::after_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int PAT, int N>
void run(long long* d) {
  const int reps = 64;
  bench<PAT, N><<<1, 32>>>(d, reps);
  cudaDeviceSynchronize();
  bench<PAT, N><<<1, 32>>>(d, reps);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return; }
  printf("pattern %d N %3d: issue %6.1f cyc/MMA, complete %6.1f cyc/MMA\n", PAT, N,
         (double)d[0] / (8 * reps), (double)d[1] / (8 * reps));
}

int main() {
  long long* d;
  cudaMallocManaged(&d, 16);
  run<0, 16>(d); run<0, 32>(d); run<0, 64>(d);
  run<1, 16>(d); run<1, 32>(d); run<1, 64>(d);
  run<2, 16>(d); run<2, 32>(d); run<2, 64>(d); run<2, 128>(d);
  run<3, 16>(d); run<3, 32>(d); run<3, 64>(d); run<3, 128>(d);
  return 0;
}
