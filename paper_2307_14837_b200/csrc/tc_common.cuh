// Shared tcgen05 / TMA / mbarrier helpers and the canonical operand layout of the
// tensor-core MLP kernels (mlp_tc.cu: fused per-tile MLP, mlp_layer.cu: layer GEMMs).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include "common.cuh"

namespace dnnmg {

constexpr int kTcM = 128;  // rows per tile (TMEM lanes)

// packed weight image: header (per-GEMM output unscale 2^-s and shift s), then the chunks
constexpr int kPackHdr = 1024;
struct PackHdr {
  float unscale[DNNMG_MAX_LAYERS];
  int32_t shift[DNNMG_MAX_LAYERS];
};
int32_t launch_pack_scales(const dnnmg_mlp_t* m, PackHdr* hdr, cudaStream_t s,
                           bool fold_bn = false);
// fp32-accurate tanh evaluates 1 - 2 / (1 + 2^z) with z = 2 log2(e) x: the factor is folded
// into the epilogue affine (and, in the fused kernel, into the packed hidden weights)
constexpr float kTanhK2 = 2.8853900817779268f;
__host__ __device__ constexpr bool tanh_folded(int precision, int act) {
  return precision != DNNMG_PREC_BF16 && act == DNNMG_ACT_TANH;
}

template <int MODE> struct TcCfg;
// KC: K elements per pipeline chunk (one TMA weight copy, one A-ring stage);
// both modes give 64-byte K rows per part, i.e. an SBO of 512 B between 8-row groups
template <> struct TcCfg<DNNMG_PREC_BF16> {
  static constexpr int ESZ = 2, PARTS = 1, NW = 6, NA = 4, KSTEP = 16, KC = 32;
};
template <> struct TcCfg<DNNMG_PREC_TF32X3> {
  static constexpr int ESZ = 4, PARTS = 2, NW = 3, NA = 4, KSTEP = 8, KC = 16;
};
template <> struct TcCfg<DNNMG_PREC_FP8> {
  static constexpr int ESZ = 1, PARTS = 1, NW = 6, NA = 4, KSTEP = 32, KC = 64;
};
#ifndef DNNMG_F16X3_NA
#define DNNMG_F16X3_NA 5
#endif
template <> struct TcCfg<DNNMG_PREC_F16X3> {
  static constexpr int ESZ = 2, PARTS = 2, NW = 2, NA = DNNMG_F16X3_NA, KSTEP = 16, KC = 32;
};
static int kc_of(int precision) {
  return precision == DNNMG_PREC_TF32X3 ? 16 : precision == DNNMG_PREC_FP8 ? 64 : 32;
}

// ---- PTX helpers ------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// as mbar_try, but the waiting warp is suspended (up to `ns`) until the phase completes
// instead of returning at once: a polling warp steals issue slots from the warps that
// share its SM sub-partition
#ifndef DNNMG_MBAR_SLEEP_NS
#define DNNMG_MBAR_SLEEP_NS 1000
#endif
__device__ __forceinline__ bool mbar_try_sleep(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity), "n"(DNNMG_MBAR_SLEEP_NS)
      : "memory");
  return ok != 0;
}
// bounded wait: a protocol bug traps (kernel error) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  uint32_t n = 0;
#if DNNMG_MBAR_SLEEP_NS > 0
  while (!mbar_try_sleep(bar, parity)) {
    if (++n > (1u << 24)) __trap();
  }
#else
  while (!mbar_try(bar, parity)) {
    if (++n > (1u << 26)) __trap();
  }
#endif
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_add_tx(uint32_t bar, uint32_t bytes) {  // no arrival
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
// shared -> global bulk copy (TMA), tracked by the issuing thread's bulk group
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}
template <int MODE>
__device__ __forceinline__ void tc_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  if constexpr (MODE == DNNMG_PREC_FP8) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  } else if constexpr (MODE != DNNMG_PREC_TF32X3) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  }
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float* v) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}
template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float* v) {
  static_assert(N == 16 || N == 8 || N == 4, "tmem_ld width");
  if constexpr (N == 16) tmem_ld16(taddr, v);
  else if constexpr (N == 8) tmem_ld8(taddr, v);
  else tmem_ld4(taddr, v);
}
__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
// x = hi + lo for a pair of values: hi = fp16(x), lo = fp16(x - hi) (x - hi is exact)
// hi = x with its fp32 mantissa truncated to the 10 bits fp16 keeps (exact in fp16 for
// |x| >= 2^-14), lo = x - hi (exact) rounded to fp16: |x - hi - lo| <= 2^-21 |x|.
// (Rounding hi to nearest instead, which makes lo symmetric, measured no accuracy change
// — tests/prec_cmp.py — and costs one more integer op per value.)
__device__ __forceinline__ void split_f16x2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const float ha = __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
  const float hb = __uint_as_float(__float_as_uint(b) & 0xFFFFE000u);
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(hb), "f"(ha));
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(b - hb), "f"(a - ha));
}

// canonical K-major no-swizzle shared-memory matrix descriptor
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((128u >> 4) & 0x3FFFu) << 16;  // LBO: K-adjacent core matrices
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;   // SBO: 8-row groups
  d |= (uint64_t)1 << 46;                        // descriptor version (sm_100)
  return d;
}
template <int MODE>
__host__ __device__ constexpr uint32_t ab_format() {  // F16 = 0, BF16 = 1, TF32 = 2
  // kind::f16: F16 = 0, BF16 = 1; kind::tf32: TF32 = 2; kind::f8f6f4: E4M3 = 0
  return MODE == DNNMG_PREC_BF16 ? 1u : MODE == DNNMG_PREC_TF32X3 ? 2u : 0u;
}
template <int MODE>
__host__ __device__ constexpr uint32_t idesc_for(int N) {
  return (1u << 4)                                              // D = F32
         | (ab_format<MODE>() << 7)                             // A format
         | (ab_format<MODE>() << 10)                            // B format
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kTcM >> 4) << 24);
}

// tanh: bf16 mode uses the MUFU tanh.approx (rel. err ~2^-11, below bf16 resolution);
// the fp32-accuracy mode uses 1 - 2/(1 + e^{2x}) with MUFU ex2/rcp: absolute error
// ~2e-7 on [-1, 1], saturating correctly for |x| -> inf.
__device__ __forceinline__ float act_fast(float x, int act, bool accurate) {
  if (act != DNNMG_ACT_TANH) return fmaxf(x, 0.f);
  if (accurate) {
    // e = 2^(2x log2 e); 1 - 2/(1+e) with MUFU ex2 / rcp (no range branches)
    float e, r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(2.8853900817779268f * x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
    return fmaf(-2.0f, r, 1.0f);
  }
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// byte offset of element (row, kk) in a canonical chunk part (kk < KC)
template <int ESZ, int KC>
__host__ __device__ constexpr uint32_t canon_off(int row, int kk) {
  return (uint32_t)((row >> 3) * (KC * ESZ * 8) + (kk / (16 / ESZ)) * 128 + (row & 7) * 16 +
                    (kk % (16 / ESZ)) * ESZ);
}

// write NV (default KC/2) consecutive K values (kk0.., kk0 % NV == 0) of one row into an A stage
template <int MODE, int NV = TcCfg<MODE>::KC / 2>
__device__ __forceinline__ void put_row(uint8_t* stage, int row, int kk0, const float* v) {
  using C = TcCfg<MODE>;
  constexpr int HC = NV;
  static_assert(MODE == DNNMG_PREC_FP8 ? NV % 16 == 0
                : MODE == DNNMG_PREC_TF32X3 ? NV % 4 == 0 : NV % 8 == 0, "put_row width");
  if constexpr (MODE == DNNMG_PREC_FP8) {
#pragma unroll
    for (int j = 0; j < HC / 16; ++j) {
      uint32_t q[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        uint16_t lo2, hi2;
        asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(lo2) : "f"(v[16 * j + 4 * w + 1]), "f"(v[16 * j + 4 * w]));
        asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(hi2) : "f"(v[16 * j + 4 * w + 3]), "f"(v[16 * j + 4 * w + 2]));
        q[w] = (uint32_t)lo2 | ((uint32_t)hi2 << 16);
      }
      *reinterpret_cast<uint4*>(stage + canon_off<1, C::KC>(row, kk0 + 16 * j)) =
          make_uint4(q[0], q[1], q[2], q[3]);
    }
  } else if constexpr (MODE == DNNMG_PREC_BF16) {
#pragma unroll
    for (int j = 0; j < HC / 8; ++j) {
      uint4 q;
      q.x = pack_bf16(v[8 * j + 0], v[8 * j + 1]);
      q.y = pack_bf16(v[8 * j + 2], v[8 * j + 3]);
      q.z = pack_bf16(v[8 * j + 4], v[8 * j + 5]);
      q.w = pack_bf16(v[8 * j + 6], v[8 * j + 7]);
      *reinterpret_cast<uint4*>(stage + canon_off<2, C::KC>(row, kk0 + 8 * j)) = q;
    }
  } else if constexpr (MODE == DNNMG_PREC_F16X3) {
    constexpr int part = kTcM * C::KC * C::ESZ;
#pragma unroll
    for (int j = 0; j < HC / 8; ++j) {
      uint4 hi, lo;
      split_f16x2(v[8 * j + 0], v[8 * j + 1], hi.x, lo.x);
      split_f16x2(v[8 * j + 2], v[8 * j + 3], hi.y, lo.y);
      split_f16x2(v[8 * j + 4], v[8 * j + 5], hi.z, lo.z);
      split_f16x2(v[8 * j + 6], v[8 * j + 7], hi.w, lo.w);
      const uint32_t off = canon_off<2, C::KC>(row, kk0 + 8 * j);
      *reinterpret_cast<uint4*>(stage + off) = hi;
      *reinterpret_cast<uint4*>(stage + part + off) = lo;
    }
  } else {
    constexpr int part = kTcM * C::KC * C::ESZ;
#pragma unroll
    for (int j = 0; j < HC / 4; ++j) {
      uint4 hi, lo;
      uint32_t* h = &hi.x;
      uint32_t* l = &lo.x;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        // exact split x = hi + lo: hi = x truncated to tf32 (10 mantissa bits), lo = x - hi
        // (exact), lo rounded to nearest tf32 (|err| <= 2^-11 |lo| <= 2^-21 |x|)
        const uint32_t xb = __float_as_uint(v[4 * j + e]);
        const uint32_t t = xb & 0xFFFFE000u;
        const uint32_t lb = __float_as_uint(v[4 * j + e] - __uint_as_float(t));
        h[e] = t;
        l[e] = (lb + 0x1000u) & 0xFFFFE000u;
      }
      const uint32_t off = canon_off<4, C::KC>(row, kk0 + 4 * j);
      *reinterpret_cast<uint4*>(stage + off) = hi;
      *reinterpret_cast<uint4*>(stage + part + off) = lo;
    }
  }
}

}  // namespace dnnmg
