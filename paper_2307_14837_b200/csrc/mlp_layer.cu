// Layer-major tensor-core MLP for the widths the fused per-tile kernel (mlp_tc.cu) cannot
// hold on chip: n_hidden != 256, n_in > 256 or n_out > 256 (BASELINE config 2:
// 1024 -> 512x3 -> 375, config 4: 174 -> {128..1024}x3 -> 81).
//
// Reference: net._forward eval branch (net.py:124-159):
//   h0 = (X - mean)/std; layer i: z = h W_i, a = act(z*scale_i + shift_i) (BN folded),
//   h_{i+1} = a (+ h_i for i >= 1); head Y = h_depth W_depth.
//
// Every layer is one persistent tcgen05 GEMM over all rows of a row chunk, tiled as
// 128-row x 256-column work items (a TMEM accumulator each, double buffered so the
// epilogue of item i overlaps the MMAs of item i+1).  Operands stream through a
// shared-memory ring by bulk (TMA) copies: the activation operand is kept in HBM already
// split (hi/lo) in the UMMA canonical K-major layout, chunk by chunk, exactly as the MMA
// consumes it, so the producer is one bulk copy per K chunk; weights are pre-packed per
// (K chunk, N block) the same way.  The fused epilogue applies BN + activation + the
// fp32 skip sum and writes both the fp32 skip state and the next layer's split operand
// (or, for the head, Y).  Warp roles (576 threads): warps 0-15 epilogue (TMEM lane quadrant
// x every fourth column step), warp 16 TMA producer, warp 17 MMA issuer.
#include <cstdlib>

#include "tc_common.cuh"

namespace dnnmg {

constexpr int kLN = 256;          // accumulator columns per work item
#ifndef DNNMG_LAYER_EPI_WARPS
#define DNNMG_LAYER_EPI_WARPS 16
#endif
constexpr int kLEpi = DNNMG_LAYER_EPI_WARPS;   // epilogue warps: 4 per TMEM lane quadrant (the
                                               // hidden layers are epilogue-latency-bound: with 2
                                               // per quadrant the tensor pipe idled half the time)
constexpr int kLThreads = 32 * (kLEpi + 2);
constexpr int kLProd = kLEpi, kLMma = kLEpi + 1;
constexpr int64_t kLChunkRows = 1 << 19;   // rows per pass (bounds the workspace)

template <int MODE> struct LCfg { static constexpr int NS = 4; };
template <> struct LCfg<DNNMG_PREC_BF16> { static constexpr int NS = 6; };
template <> struct LCfg<DNNMG_PREC_FP8> { static constexpr int NS = 6; };

struct LayerArgs {
  const uint8_t* A;        // operand [tiles][n_kc][PARTS][kTcM*KC*ESZ]
  const uint8_t* W;        // packed weights of the layer: per K chunk, the N blocks in order
  int64_t w_kc_bytes;      // bytes of one K chunk (all N blocks)
  int n_tiles, n_kc, n_nb, N, Nlast;
  int64_t n_rows;          // valid rows of this pass
  const float* scale;      // [N] folded epilogue affine (hidden layers)
  const float* shift;
  int act, fold, head;
  const float* h_in;       // skip input  [tiles][N/16][kTcM][16] or NULL
  float* h_out;            // layer output, same layout, or NULL
  uint8_t* A_out;          // next operand [tiles][N/KC][PARTS][...] or NULL
  int n_kc_out;
  float* Y;                // head: [rows][n_out]
  int n_out;
  const float* y_unscale;  // head: 2^-s of the packed head weights (device, pack header)
};

template <int MODE>
__global__ void __launch_bounds__(kLThreads, 1) mlp_layer_kernel(LayerArgs A) {
  using C = TcCfg<MODE>;
  constexpr int KC = C::KC;
  constexpr int HC = KC / 2;
  constexpr int NS = LCfg<MODE>::NS;
  constexpr uint32_t APART = kTcM * KC * C::ESZ;
  constexpr uint32_t AST = APART * C::PARTS;
  constexpr uint32_t WST = kLN * KC * C::ESZ * C::PARTS;
  constexpr uint32_t STG = AST + WST;
  constexpr uint32_t SBO = KC * C::ESZ * 8;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NS * STG);
  uint64_t* full = bars;
  uint64_t* empty = bars + NS;
  uint64_t* acc_full = bars + 2 * NS;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  // head epilogue: a padded 32 x GS staging tile per epilogue warp (after the barriers)
  float* ystage = reinterpret_cast<float*>(smem + NS * STG + 8 * (2 * NS + 4) + 16);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_items = (int64_t)A.n_tiles * A.n_nb;
  const bool seg2 = MODE == DNNMG_PREC_TF32X3 && A.n_kc * KC > 512;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(smem_u32(&full[i]), 1);
      mbar_init(smem_u32(&empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&acc_full[i]), 1);
      mbar_init(smem_u32(&acc_empty[i]), kLEpi);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kLProd) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kLProd) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int t = (int)(item / A.n_nb), b = (int)(item % A.n_nb);
        const int nbw = b == A.n_nb - 1 ? A.Nlast : kLN;
        const uint32_t wbytes = (uint32_t)nbw * KC * C::ESZ * C::PARTS;
        for (int kc = 0; kc < A.n_kc; ++kc, ++it) {
          const int s = it % NS;
          mbar_wait(smem_u32(&empty[s]), ((it / NS) & 1) ^ 1);
          mbar_expect_tx(smem_u32(&full[s]), AST + wbytes);
          bulk_g2s(smem_u32(smem + s * STG), A.A + ((int64_t)t * A.n_kc + kc) * AST, AST,
                   smem_u32(&full[s]));
          bulk_g2s(smem_u32(smem + s * STG + AST),
                   A.W + kc * A.w_kc_bytes + (int64_t)b * kLN * KC * C::ESZ * C::PARTS, wbytes,
                   smem_u32(&full[s]));
        }
      }
    }
  } else if (warp == kLMma) {
    if (lane == 0) {
      uint32_t it = 0, j = 0;
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x, ++j) {
        const int b = (int)(item % A.n_nb);
        const int nbw = b == A.n_nb - 1 ? A.Nlast : kLN;
        const uint32_t idesc = idesc_for<MODE>(nbw);
        // seg2: the K loop in two halves accumulated in the two buffers (both per item), so
        // that no tensor-core accumulation runs over more than K/2 (its fp32 accumulation
        // rounds per step: tf32x3 measured 1.2e-5 at K = 1024 in one accumulator)
        const int buf = seg2 ? 0 : (j & 1);
        const int khalf = seg2 ? (A.n_kc + 1) / 2 : A.n_kc;
        if (seg2) {
          mbar_wait(smem_u32(&acc_empty[0]), (j & 1) ^ 1);
          mbar_wait(smem_u32(&acc_empty[1]), (j & 1) ^ 1);
        } else {
          mbar_wait(smem_u32(&acc_empty[buf]), ((j >> 1) & 1) ^ 1);
        }
        tc_fence_after();
        for (int kc = 0; kc < A.n_kc; ++kc, ++it) {
          const int s = it % NS;
          const bool second = kc >= khalf;
          const uint32_t d = tmem + (second ? 1 : buf) * kLN;
          mbar_wait(smem_u32(&full[s]), (it / NS) & 1);
          tc_fence_after();
          const uint32_t ab = smem_u32(smem + s * STG);
          const uint32_t wb = ab + AST;
#pragma unroll
          for (int ks = 0; ks < KC / C::KSTEP; ++ks) {
            const uint32_t koff = ks * 256;
            const uint32_t acc = ((kc > 0 && kc != khalf) || ks > 0) ? 1u : 0u;
            const uint64_t ahi = sdesc(ab + koff, SBO), bhi = sdesc(wb + koff, SBO);
            tc_mma<MODE>(d, ahi, bhi, idesc, acc);
            if constexpr (C::PARTS == 2) {
              const uint64_t alo = sdesc(ab + APART + koff, SBO);
              const uint64_t blo = sdesc(wb + (uint32_t)nbw * KC * C::ESZ + koff, SBO);
              tc_mma<MODE>(d, ahi, blo, idesc, 1u);
              tc_mma<MODE>(d, alo, bhi, idesc, 1u);
            }
          }
          tc_commit(smem_u32(&empty[s]));
          if (seg2 && kc == khalf - 1) tc_commit(smem_u32(&acc_full[0]));
        }
        tc_commit(smem_u32(&acc_full[seg2 ? 1 : buf]));
      }
    }
  } else {
    // ---------------- epilogue warps ----------------
    const int quad = warp & 3, part = warp >> 2;   // part: which GS-column steps of an item
    const int row = quad * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    constexpr bool accurate = MODE == DNNMG_PREC_F16X3 || MODE == DNNMG_PREC_TF32X3;
    constexpr int GS = HC > 16 ? HC : 16;   // columns per epilogue step (FP8: one 64-K half chunk)
    const int g16 = A.N / 16;   // 16-column groups of the layer output
    const float yu = A.head ? __ldg(A.y_unscale) : 1.f;
    uint32_t j = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x, ++j) {
      const int t = (int)(item / A.n_nb), b = (int)(item % A.n_nb);
      const int nbw = b == A.n_nb - 1 ? A.Nlast : kLN;
      const int buf = seg2 ? 0 : (j & 1);
      const int64_t grow = (int64_t)t * kTcM + row;
      const bool live = grow < A.n_rows;
      if (seg2) {
        mbar_wait(smem_u32(&acc_full[0]), j & 1);
        mbar_wait(smem_u32(&acc_full[1]), j & 1);
      } else {
        mbar_wait(smem_u32(&acc_full[buf]), (j >> 1) & 1);
      }
      tc_fence_after();
      for (int cc = part * GS; cc < nbw; cc += (kLEpi / 4) * GS) {
        float v[GS];
#pragma unroll
        for (int p = 0; p < GS / 16; ++p) tmem_ld16(tmem + lane_addr + buf * kLN + cc + 16 * p, v + 16 * p);
        if (seg2) {   // the second K half, added in fp32
          float v2[GS];
#pragma unroll
          for (int p = 0; p < GS / 16; ++p) tmem_ld16(tmem + lane_addr + kLN + cc + 16 * p, v2 + 16 * p);
#pragma unroll
          for (int e = 0; e < GS; ++e) v[e] += v2[e];
        }
        const int col0 = b * kLN + cc;          // layer column of v[0]
        if (A.head) {
          // Y rows are n_out floats apart (375 or 81: not 16-byte aligned), and a lane holds one
          // row: stored from the registers, every store instruction hit 32 sectors with 4 bytes
          // each (the head took longer than a hidden layer).  The 32 x GS block goes through a
          // padded shared-memory tile and leaves as 64- or 128-byte row segments.
          float* st = ystage + (warp * 32) * (GS + 1);
#pragma unroll
          for (int e = 0; e < GS; ++e) st[lane * (GS + 1) + e] = v[e] * yu;
          __syncwarp();
          constexpr int RPI = 32 / GS;   // rows per store instruction
          const int e = lane % GS;
#pragma unroll 4
          for (int rr = 0; rr < 32; rr += RPI) {
            const int rl = rr + lane / GS;
            const int64_t gr = (int64_t)t * kTcM + quad * 32 + rl;
            if (gr < A.n_rows && col0 + e < A.n_out)
              A.Y[gr * A.n_out + col0 + e] = st[rl * (GS + 1) + e];
          }
          __syncwarp();
          continue;
        }
        float hv[GS];
        if (A.h_in) {
#pragma unroll
          for (int p = 0; p < GS / 16; ++p) {
            const int64_t hoff = (((int64_t)t * g16 + col0 / 16 + p) * kTcM + row) * 16;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 x = __ldg(reinterpret_cast<const float4*>(A.h_in + hoff) + q);
              hv[16 * p + 4 * q] = x.x;
              hv[16 * p + 4 * q + 1] = x.y;
              hv[16 * p + 4 * q + 2] = x.z;
              hv[16 * p + 4 * q + 3] = x.w;
            }
          }
        } else {
#pragma unroll
          for (int e = 0; e < GS; ++e) hv[e] = 0.f;
        }
#pragma unroll
        for (int q = 0; q < GS / 4; ++q) {
          const float4 s4 = __ldg(reinterpret_cast<const float4*>(A.scale + col0) + q);
          const float4 t4 = __ldg(reinterpret_cast<const float4*>(A.shift + col0) + q);
          const float sv[4] = {s4.x, s4.y, s4.z, s4.w}, tv[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float z = fmaf(v[4 * q + u], sv[u], tv[u]);
            float a;
            if (A.fold) {   // z = 2 log2(e) BN(acc): tanh = 1 - 2 / (1 + 2^z)
              float ez, r;
              asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ez) : "f"(z));
              asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + ez));
              a = fmaf(-2.0f, r, 1.0f);
            } else {
              a = act_fast(z, A.act, accurate);
            }
            v[4 * q + u] = a + hv[4 * q + u];
          }
        }
        if (A.h_out) {
#pragma unroll
          for (int p = 0; p < GS / 16; ++p) {
            const int64_t hoff = (((int64_t)t * g16 + col0 / 16 + p) * kTcM + row) * 16;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              reinterpret_cast<float4*>(A.h_out + hoff)[q] =
                  make_float4(v[16 * p + 4 * q], v[16 * p + 4 * q + 1], v[16 * p + 4 * q + 2],
                              v[16 * p + 4 * q + 3]);
          }
        }
        if (A.A_out) {
#pragma unroll
          for (int g = 0; g < GS; g += HC) {
            const int col = col0 + g;
            uint8_t* chunk = A.A_out + ((int64_t)t * A.n_kc_out + col / KC) * AST;
            put_row<MODE>(chunk, row, col % KC, v + g);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(smem_u32(&acc_empty[buf]));
        if (seg2) mbar_arrive(smem_u32(&acc_empty[1]));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kLProd) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// layer-0 operand: (X - mean) / std of rows [r0, r0 + n) split into the canonical chunks;
// one thread per (row, HC-column group); rows and columns past the data are zero
// patch source of the layer-0 rows (K3 fused into the layered MLP): row p =
// [x~ of node_table[p][s] | r of node_table[p][s] | geom[p]] (patch_ops.py:49-53)
struct PatchRows {
  const int32_t* table;
  const float* x;
  const float* r;
  const float* geom;
  int npp, n_geo;
};

__device__ __forceinline__ float patch_value(const PatchRows& P, int64_t p, int col) {
  const int nb = 4 * P.npp;
  if (col < nb) return __ldg(P.x + 4 * (int64_t)__ldg(P.table + p * P.npp + (col >> 2)) + (col & 3));
  if (col < 2 * nb) {
    const int c = col - nb;
    return __ldg(P.r + 4 * (int64_t)__ldg(P.table + p * P.npp + (c >> 2)) + (c & 3));
  }
  return __ldg(P.geom + p * P.n_geo + (col - 2 * nb));
}

template <int MODE, bool PATCH>
__global__ void __launch_bounds__(256) layer_input_kernel(const float* __restrict__ X, PatchRows P,
                                                          int64_t r0, int64_t n, int64_t n_rows_pad,
                                                          int n_in, int n_kc,
                                                          const float* __restrict__ mean,
                                                          const float* __restrict__ std_,
                                                          uint8_t* __restrict__ out) {
  using C = TcCfg<MODE>;
  constexpr int KC = C::KC, HC = KC / 2;
  constexpr uint32_t AST = kTcM * KC * C::ESZ * C::PARTS;
  const int groups = n_kc * 2;
  const int64_t total = n_rows_pad * groups;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / groups;
    const int g = (int)(i - r * groups);
    const int col0 = g * HC;
    float v[HC];
#pragma unroll
    for (int e = 0; e < HC; ++e) {
      const int col = col0 + e;
      float x = 0.f;
      if (r < n && col < n_in) {
        if constexpr (PATCH) x = patch_value(P, r0 + r, col);
        else x = __ldg(X + (r0 + r) * n_in + col);
      }
      v[e] = (r < n && col < n_in) ? (x - __ldg(mean + col)) / __ldg(std_ + col) : 0.f;
    }
    const int64_t t = r / kTcM;
    uint8_t* chunk = out + (t * n_kc + col0 / KC) * AST;
    put_row<MODE>(chunk, (int)(r % kTcM), col0 % KC, v);
  }
}

// per-layer epilogue affine: scale' = bn_scale * unscale * k2, shift' = bn_shift * k2
// (k2 = 2 log2 e when the accurate tanh takes 2^z), zero-padded to the padded width
__global__ void layer_affine_kernel(const float* __restrict__ scale, const float* __restrict__ shift,
                                    const PackHdr* __restrict__ hdr, int depth, int H, int Hp,
                                    float k2, float* __restrict__ out) {
  const int total = depth * Hp;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int g = i / Hp, c = i % Hp;
    const float us = hdr->unscale[g];
    out[i] = c < H ? scale[g * H + c] * us * k2 : 0.f;
    out[total + i] = c < H ? shift[g * H + c] * k2 : 0.f;
  }
}

}  // namespace dnnmg

namespace dnnmg {

// weights of layer g in the layered image: per K chunk of KC rows, the N blocks of up to
// kLN columns in order, each [hi | lo] canonical (nbw rows x KC)
template <int MODE>
__global__ void pack_layered_kernel(const float* __restrict__ W, int K, int N, int Kp, int Np,
                                    const PackHdr* __restrict__ hdr, int g, uint8_t* __restrict__ out) {
  using C = TcCfg<MODE>;
  constexpr int KC = C::KC;
  const int shift = hdr->shift[g];
  const int64_t total = (int64_t)Kp * Np;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(i % Np), k = (int)(i / Np);
    const float w = (k < K && n < N) ? W[(int64_t)k * N + n] : 0.f;
    const int kc = k / KC, kk = k % KC, b = n / kLN, nr = n % kLN;
    const int nbw = Np - b * kLN < kLN ? Np - b * kLN : kLN;
    uint8_t* chunk = out + (int64_t)kc * Np * KC * C::ESZ * C::PARTS +
                     (int64_t)b * kLN * KC * C::ESZ * C::PARTS;
    const uint32_t off = canon_off<C::ESZ, KC>(nr, kk);
    const uint32_t part = (uint32_t)nbw * KC * C::ESZ;
    if constexpr (MODE == DNNMG_PREC_FP8) {
      uint16_t q;
      asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(q) : "f"(0.f), "f"(ldexpf(w, shift)));
      *(chunk + off) = (uint8_t)(q & 0xFF);
    } else if constexpr (MODE == DNNMG_PREC_BF16) {
      *reinterpret_cast<__nv_bfloat16_raw*>(chunk + off) =
          static_cast<__nv_bfloat16_raw>(__float2bfloat16_rn(w));
    } else if constexpr (MODE == DNNMG_PREC_F16X3) {
      const float ws = ldexpf(w, shift);
      const __half hi = __float2half_rn(ws);
      *reinterpret_cast<__half*>(chunk + off) = hi;
      *reinterpret_cast<__half*>(chunk + part + off) = __float2half_rn(ws - __half2float(hi));
    } else {
      const uint32_t hi = to_tf32(w);
      *reinterpret_cast<uint32_t*>(chunk + off) = hi;
      *reinterpret_cast<uint32_t*>(chunk + part + off) = to_tf32(w - __uint_as_float(hi));
    }
  }
}

static int rup(int x, int m) { return (x + m - 1) / m * m; }
static int64_t rup64(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

struct LayeredGeom {
  int KC, esz, parts;
  int K[DNNMG_MAX_LAYERS], N[DNNMG_MAX_LAYERS];
  int64_t goff[DNNMG_MAX_LAYERS];
  int64_t packed;
  int64_t chunk_rows, tiles;
  int64_t a_bytes, h_bytes, ws;   // per operand buffer, per skip buffer, total workspace
};

static LayeredGeom layered_geom(const dnnmg_mlp_t* m, int64_t n_rows) {
  LayeredGeom L{};
  L.KC = kc_of(m->precision);
  L.esz = m->precision == DNNMG_PREC_TF32X3 ? 4 : m->precision == DNNMG_PREC_FP8 ? 1 : 2;
  L.parts = (m->precision == DNNMG_PREC_BF16 || m->precision == DNNMG_PREC_FP8) ? 1 : 2;
  int64_t off = kPackHdr;
  for (int g = 0; g <= m->depth; ++g) {
    L.K[g] = rup(g == 0 ? m->n_in : m->n_hidden, L.KC);
    // N blocks split into two column halves of whole epilogue steps (FP8: 32 columns)
    L.N[g] = rup(g < m->depth ? m->n_hidden : m->n_out, m->precision == DNNMG_PREC_FP8 ? 64 : 32);
    L.goff[g] = off;
    off += (int64_t)L.K[g] * L.N[g] * L.esz * L.parts;
  }
  L.packed = off;
  L.chunk_rows = n_rows < kLChunkRows ? n_rows : kLChunkRows;
  L.tiles = (L.chunk_rows + kTcM - 1) / kTcM;
  const int kmax = L.K[0] > m->n_hidden ? L.K[0] : m->n_hidden;
  L.a_bytes = rup64(L.tiles * kTcM * kmax * L.esz * L.parts, 1024);
  L.h_bytes = rup64(L.tiles * kTcM * (int64_t)m->n_hidden * 4, 1024);
  L.ws = 2 * L.a_bytes + 2 * L.h_bytes + rup64(2LL * m->depth * m->n_hidden * 4, 1024);
  return L;
}

int32_t mlp_layered_supported(const dnnmg_mlp_t* m) {
  return (m->precision == DNNMG_PREC_BF16 || m->precision == DNNMG_PREC_TF32X3 ||
          m->precision == DNNMG_PREC_F16X3 || m->precision == DNNMG_PREC_FP8) &&
         m->n_hidden % (m->precision == DNNMG_PREC_FP8 ? 64 : 32) == 0 && m->n_hidden <= 4096 && m->n_in <= 8192 && m->n_out <= 4096 &&
         m->depth >= 1 && m->depth < DNNMG_MAX_LAYERS;
}

int32_t mlp_layered_packed_bytes(const dnnmg_mlp_t* m, int64_t* bytes) {
  *bytes = layered_geom(m, 1).packed;
  return DNNMG_OK;
}

int32_t mlp_layered_workspace_bytes(const dnnmg_mlp_t* m, int64_t n_rows, int64_t* bytes) {
  *bytes = n_rows > 0 ? layered_geom(m, n_rows).ws : 0;
  return DNNMG_OK;
}

// The patch form with whole nodes per load: 4 consecutive operand columns are the 4 components
// of one node (x~ or r, a float4 gather through the patch's node table) or 4 geometry values, so
// a thread's HC columns take HC/4 table loads and HC/4 float4 loads instead of 2 HC dependent
// scalar loads; mean / std are read as float4.  (Needs n_geo % 4 == 0 and 16-byte aligned x, r,
// geom, mean, std.)  LANES_ROWS: consecutive lanes take consecutive rows of one column group
// (their 16-byte operand stores form 128-byte runs of the canonical layout) instead of
// consecutive column groups of one row.
template <int MODE, bool LANES_ROWS>
__global__ void __launch_bounds__(256) layer_input_patch4_kernel(PatchRows P, int64_t r0, int64_t n,
                                                                 int64_t n_rows_pad, int n_in,
                                                                 int n_kc,
                                                                 const float* __restrict__ mean,
                                                                 const float* __restrict__ std_,
                                                                 uint8_t* __restrict__ out) {
  using C = TcCfg<MODE>;
  constexpr int KC = C::KC, HC = KC / 2;
  constexpr uint32_t AST = kTcM * KC * C::ESZ * C::PARTS;
  const int groups = n_kc * 2;
  const int64_t total = n_rows_pad * groups;
  const int nb = 4 * P.npp;
  const float4* x4 = reinterpret_cast<const float4*>(P.x);
  const float4* r4 = reinterpret_cast<const float4*>(P.r);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = LANES_ROWS ? i % n_rows_pad : i / groups;
    const int g = (int)(LANES_ROWS ? i / n_rows_pad : i - r * groups);
    const int col0 = g * HC;
    const int64_t p = r0 + r;
    float v[HC];
#pragma unroll
    for (int q = 0; q < HC / 4; ++q) {
      const int col = col0 + 4 * q;
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < n && col < n_in) {
        if (col < nb) x = __ldg(x4 + __ldg(P.table + p * P.npp + (col >> 2)));
        else if (col < 2 * nb) x = __ldg(r4 + __ldg(P.table + p * P.npp + ((col - nb) >> 2)));
        else x = __ldg(reinterpret_cast<const float4*>(P.geom + p * P.n_geo + (col - 2 * nb)));
        const float4 m = __ldg(reinterpret_cast<const float4*>(mean + col));
        const float4 sd = __ldg(reinterpret_cast<const float4*>(std_ + col));
        x = make_float4((x.x - m.x) / sd.x, (x.y - m.y) / sd.y, (x.z - m.z) / sd.z,
                        (x.w - m.w) / sd.w);
      }
      v[4 * q] = x.x;
      v[4 * q + 1] = x.y;
      v[4 * q + 2] = x.z;
      v[4 * q + 3] = x.w;
    }
    const int64_t t = r / kTcM;
    uint8_t* chunk = out + (t * n_kc + col0 / KC) * AST;
    put_row<MODE>(chunk, (int)(r % kTcM), col0 % KC, v);
  }
}

int32_t launch_mlp_layered_pack(const dnnmg_mlp_t* m, void* packed, cudaStream_t s) {
  DNNMG_REQUIRE(mlp_layered_supported(m), DNNMG_ERR_UNSUPPORTED,
                "mlp: layered tensor-core mode needs n_hidden %% 32 == 0");
  const LayeredGeom L = layered_geom(m, 1);
  PackHdr* hdr = static_cast<PackHdr*>(packed);
  int32_t rc = launch_pack_scales(m, hdr, s);
  if (rc) return rc;
  for (int g = 0; g <= m->depth; ++g) {
    const int K = g == 0 ? m->n_in : m->n_hidden;
    const int N = g < m->depth ? m->n_hidden : m->n_out;
    uint8_t* out = static_cast<uint8_t*>(packed) + L.goff[g];
    const int64_t n = (int64_t)L.K[g] * L.N[g];
    if (m->precision == DNNMG_PREC_FP8)
      pack_layered_kernel<DNNMG_PREC_FP8><<<grid_for(n, 256), 256, 0, s>>>(m->W[g], K, N, L.K[g], L.N[g], hdr, g, out);
    else if (m->precision == DNNMG_PREC_BF16)
      pack_layered_kernel<DNNMG_PREC_BF16><<<grid_for(n, 256), 256, 0, s>>>(m->W[g], K, N, L.K[g], L.N[g], hdr, g, out);
    else if (m->precision == DNNMG_PREC_F16X3)
      pack_layered_kernel<DNNMG_PREC_F16X3><<<grid_for(n, 256), 256, 0, s>>>(m->W[g], K, N, L.K[g], L.N[g], hdr, g, out);
    else
      pack_layered_kernel<DNNMG_PREC_TF32X3><<<grid_for(n, 256), 256, 0, s>>>(m->W[g], K, N, L.K[g], L.N[g], hdr, g, out);
    DNNMG_CHECK_LAUNCH("pack_layered_kernel");
  }
  return DNNMG_OK;
}

template <int MODE>
static int32_t layered_mode(const dnnmg_mlp_t* m, const float* X, const PatchRows* P,
                            int64_t n_rows, float* Y, void* ws, cudaStream_t s) {
  using C = TcCfg<MODE>;
  constexpr int NS = LCfg<MODE>::NS;
  constexpr size_t STG = (size_t)kTcM * C::KC * C::ESZ * C::PARTS +
                         (size_t)kLN * C::KC * C::ESZ * C::PARTS;
  constexpr int GS = C::KC / 2 > 16 ? C::KC / 2 : 16;   // (as in the kernel's epilogue)
  const size_t smem = NS * STG + 8 * (2 * NS + 4) + 16 + kLEpi * 32 * (GS + 1) * sizeof(float);
  const LayeredGeom L = layered_geom(m, n_rows);
  uint8_t* base = static_cast<uint8_t*>(ws);
  uint8_t* abuf[2] = {base, base + L.a_bytes};
  float* hbuf[2] = {reinterpret_cast<float*>(base + 2 * L.a_bytes),
                    reinterpret_cast<float*>(base + 2 * L.a_bytes + L.h_bytes)};
  float* affine = reinterpret_cast<float*>(base + 2 * L.a_bytes + 2 * L.h_bytes);
  const PackHdr* hdr = static_cast<const PackHdr*>(m->packed);
  const bool fold = (MODE == DNNMG_PREC_F16X3 || MODE == DNNMG_PREC_TF32X3) &&
                    m->activation == DNNMG_ACT_TANH;
  const int H = m->n_hidden;
  layer_affine_kernel<<<grid_for((int64_t)m->depth * H, 256), 256, 0, s>>>(
      m->bn_scale, m->bn_shift, hdr, m->depth, H, H, fold ? 2.8853900817779268f : 1.0f, affine);
  DNNMG_CHECK_LAUNCH("layer_affine_kernel");
  static uint64_t configured = 0;
  if (first_use_on_device(configured)) {
    cudaFuncSetAttribute(mlp_layer_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  for (int64_t r0 = 0; r0 < n_rows; r0 += L.chunk_rows) {
    const int64_t n = n_rows - r0 < L.chunk_rows ? n_rows - r0 : L.chunk_rows;
    const int tiles = (int)((n + kTcM - 1) / kTcM);
    const int kc0 = L.K[0] / C::KC;
    const int in_grid = grid_for((int64_t)tiles * kTcM * kc0 * 2, 256);
    const bool vec4 = P && P->n_geo % 4 == 0 && m->n_in % 4 == 0 &&
                      (((uintptr_t)P->x | (uintptr_t)P->r | (uintptr_t)P->geom |
                        (uintptr_t)m->in_mean | (uintptr_t)m->in_std) & 15) == 0;
    static const int in_mode = getenv("DNNMG_LAYER_INPUT") ? atoi(getenv("DNNMG_LAYER_INPUT")) : 2;
    if (vec4 && in_mode == 2)
      layer_input_patch4_kernel<MODE, true><<<in_grid, 256, 0, s>>>(
          *P, r0, n, (int64_t)tiles * kTcM, m->n_in, kc0, m->in_mean, m->in_std, abuf[0]);
    else if (vec4 && in_mode == 1)
      layer_input_patch4_kernel<MODE, false><<<in_grid, 256, 0, s>>>(
          *P, r0, n, (int64_t)tiles * kTcM, m->n_in, kc0, m->in_mean, m->in_std, abuf[0]);
    else if (P)
      layer_input_kernel<MODE, true><<<in_grid, 256, 0, s>>>(
          nullptr, *P, r0, n, (int64_t)tiles * kTcM, m->n_in, kc0, m->in_mean, m->in_std, abuf[0]);
    else
      layer_input_kernel<MODE, false><<<in_grid, 256, 0, s>>>(
          X, PatchRows{}, r0, n, (int64_t)tiles * kTcM, m->n_in, kc0, m->in_mean, m->in_std, abuf[0]);
    DNNMG_CHECK_LAUNCH("layer_input_kernel");
    for (int g = 0; g <= m->depth; ++g) {
      LayerArgs A{};
      const bool head = g == m->depth;
      A.A = abuf[g % 2];
      A.W = static_cast<const uint8_t*>(m->packed) + L.goff[g];
      A.w_kc_bytes = (int64_t)L.N[g] * C::KC * C::ESZ * C::PARTS;
      A.n_tiles = tiles;
      A.n_kc = L.K[g] / C::KC;
      A.N = L.N[g];
      A.n_nb = (L.N[g] + kLN - 1) / kLN;
      A.Nlast = L.N[g] - (A.n_nb - 1) * kLN;
      A.n_rows = n;
      A.scale = affine + (int64_t)g * H;
      A.shift = affine + (int64_t)m->depth * H + (int64_t)g * H;
      A.act = m->activation;
      A.fold = fold;
      A.head = head;
      A.h_in = (!head && g >= 1) ? hbuf[g % 2] : nullptr;
      A.h_out = (!head && g + 1 < m->depth) ? hbuf[(g + 1) % 2] : nullptr;
      A.A_out = head ? nullptr : abuf[(g + 1) % 2];
      A.n_kc_out = H / C::KC;
      A.Y = Y + r0 * m->n_out;
      A.n_out = m->n_out;
      A.y_unscale = &hdr->unscale[m->depth];
      const int64_t items = (int64_t)tiles * A.n_nb;
      const int grid = (int)(items < kSMs ? items : kSMs);
      mlp_layer_kernel<MODE><<<grid, kLThreads, smem, s>>>(A);
      DNNMG_CHECK_LAUNCH("mlp_layer_kernel");
    }
  }
  return DNNMG_OK;
}

int32_t launch_mlp_layered_rows(const dnnmg_mlp_t* m, const float* X, const PatchRows* P,
                                int64_t n_rows, float* Y, void* ws, int64_t ws_bytes,
                                cudaStream_t s) {
  DNNMG_REQUIRE(mlp_layered_supported(m) && m->packed, DNNMG_ERR_UNSUPPORTED,
                "mlp: layered tensor-core mode needs packed weights and n_hidden %% 32 == 0");
  if (n_rows == 0) return DNNMG_OK;
  DNNMG_REQUIRE(ws, DNNMG_ERR_ARG, "mlp: the layered tensor-core MLP needs a workspace "
                "(dnnmg_mlp_workspace_bytes)");
  // the workspace layout depends on n_rows (up to the pass size): a buffer sized for fewer
  // rows would be overrun
  const int64_t need = layered_geom(m, n_rows).ws;
  DNNMG_REQUIRE(ws_bytes >= need, DNNMG_ERR_ARG,
                "mlp: workspace of %lld bytes is smaller than the %lld bytes %lld rows need "
                "(dnnmg_mlp_workspace_bytes)", (long long)ws_bytes, (long long)need,
                (long long)n_rows);
  if (m->precision == DNNMG_PREC_FP8) return layered_mode<DNNMG_PREC_FP8>(m, X, P, n_rows, Y, ws, s);
  if (m->precision == DNNMG_PREC_BF16) return layered_mode<DNNMG_PREC_BF16>(m, X, P, n_rows, Y, ws, s);
  if (m->precision == DNNMG_PREC_F16X3) return layered_mode<DNNMG_PREC_F16X3>(m, X, P, n_rows, Y, ws, s);
  return layered_mode<DNNMG_PREC_TF32X3>(m, X, P, n_rows, Y, ws, s);
}

int32_t launch_mlp_layered(const dnnmg_mlp_t* m, const float* X, int64_t n_rows, float* Y, void* ws,
                           int64_t ws_bytes, cudaStream_t s) {
  return launch_mlp_layered_rows(m, X, nullptr, n_rows, Y, ws, ws_bytes, s);
}

// K3 fused into the layered MLP: the layer-0 operand is gathered straight from x~, r and the
// patch geometry (no X in HBM)
int32_t launch_mlp_layered_patches(const dnnmg_mlp_t* m, const dnnmg_patchset_t* ps, const float* x,
                                   const float* r, float* Y, void* ws, int64_t ws_bytes,
                                   cudaStream_t s) {
  DNNMG_REQUIRE(8 * ps->nodes_per_patch + ps->n_geo == m->n_in, DNNMG_ERR_ARCH,
                "model architecture (%d inputs) does not match the patch layout (%d)", m->n_in,
                8 * ps->nodes_per_patch + ps->n_geo);
  PatchRows P{ps->node_table, x, r, ps->geom, ps->nodes_per_patch, ps->n_geo};
  return launch_mlp_layered_rows(m, nullptr, &P, ps->n_patches, Y, ws, ws_bytes, s);
}

}  // namespace dnnmg
