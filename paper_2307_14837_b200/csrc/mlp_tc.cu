// K4 fast path: the patch MLP on 5th-generation tensor cores (tcgen05 + TMEM).
//
// Reference: net._forward eval branch (net.py:124-159):
//   h0 = (X - mean)/std; layer i: z = h W_i, a = act(z*scale_i + shift_i) (BN folded),
//   h_{i+1} = a (+ h_i for i >= 1); head Y = h_depth W_depth.
//
// One persistent CTA per SM processes 128-row tiles of a network with hidden width
// H = 128 or 256 (template).  Warp roles (352 threads):
//   warps 0..7  compute: stage the layer-0 A operand (input normalisation) from X, from
//               a direct per-(patch, slot) gather or from the staged tile nodes,
//               run every epilogue (TMEM -> registers -> BN/activation/skip) and
//               write the next GEMM's A operand into the SMEM ring chunk by chunk;
//               the fp32 skip state h lives in their registers (H/2 values/thread)
//   warp 8      weight producer: cp.async.bulk (TMA) of pre-packed weight chunks
//               (already in the UMMA canonical layout) into the SMEM ring
//   warp 9      MMA issuer: one thread issues tcgen05.mma into TMEM, commits to
//               mbarriers that release SMEM stages and signal the epilogue
//   warp 10     staged gather (GM_STAGED): cp.async of the next tile's distinct nodes,
//               bulk copies of its slot block and geometry; bulk store of Y (y_mode 3)
// TMEM holds two 128 x H fp32 accumulators, so the epilogue of GEMM j overlaps
// the MMAs of GEMM j+1 (which consume the A chunks the epilogue produces).
//
// Precision modes:
//   BF16    kind::f16, bf16 A/B, fp32 accumulate in TMEM
//   TF32X3  kind::tf32, x = hi + lo (both tf32), D += Ahi*Bhi + Ahi*Blo + Alo*Bhi:
//           fp32-level accuracy
//   F16X3   kind::f16 with fp16 operands, the same 3-pass split at twice the tf32 rate:
//           fp16 carries 11 significant bits like tf32, so hi + lo holds 22 bits.  Each
//           weight matrix is pre-scaled by 2^s (max|W| 2^s < 2^14, exact) to keep hi and
//           lo in the fp16 normal range; 2^-s is folded into the BN scale (or applied to
//           the head output), which is exact.  Activations enter unscaled (|h| < 65504:
//           normalised inputs and tanh skip sums; relu models use TF32X3).
// Operands use the K-major, no-swizzle canonical layout: 8x16-byte core matrices,
// LBO = 128 B between K-adjacent core matrices, SBO between 8-row groups.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdlib>
#include <type_traits>
#include "common.cuh"
#include "tc_common.cuh"

namespace dnnmg {

constexpr int kTcH = 256;   // hidden width of the largest instantiation
constexpr int kTcIn = 256;  // network inputs the fused kernel stages (n_in <= kTcIn)
// warp roles for NQ compute warps per TMEM lane quadrant (each takes KC / NQ columns of every
// K chunk): 4 NQ compute warps, then the weight producer, the MMA issuer and the staged-gather
// warp.  The staged fused gather runs NQ = 4 (16 compute warps at the 96-register budget: four
// warps per sub-partition hide the epilogue's TMEM-load / MUFU / shared-store latencies; 0.68
// -> 0.63 ms at config 3); the other layer-0 sources keep NQ = 2, whose 168-register budget
// holds their prefetched input rows without spilling.
template <int GM> struct TcRoles {
  static constexpr int NQ = GM == 2 ? 4 : 2;
  static constexpr int kComputeWarps = 4 * NQ;
  static constexpr int kComputeThreads = 32 * kComputeWarps;
  static constexpr int kProducerWarp = kComputeWarps;
  static constexpr int kMmaWarp = kComputeWarps + 1;
  static constexpr int kGatherWarp = kComputeWarps + 2;  // GM_STAGED: cp.async of a tile's nodes
  static constexpr int kThreads = 32 * (kComputeWarps + 3);
};
// sources of the layer-0 operand
enum { GM_X = 0,        // rows of a stored X
       GM_DIRECT = 1,   // fused gather: per-(patch, slot) global loads at the tile boundary
       GM_STAGED = 2 }; // fused gather: the tile's distinct nodes staged in SMEM one tile ahead


struct TcArgs {
  const float* X;
  float* Y;
  int64_t n_rows;
  int n_in, n_out, depth, act;
  int K0p, Nhead;
  int y_mode;  // 0: direct stores, 2: staged in a dedicated shared-memory buffer,
               // 3 (GM_STAGED): the whole 128-row tile staged in the gather staging area and
               //   written by one bulk (TMA) store from the gather warp
  const uint8_t* packed;
  int64_t goff[DNNMG_MAX_LAYERS];
  const float* scale;
  const float* shift;
  const float* in_mean;
  const float* in_std;
  // fused patch gather (K3 into K4): row p = [x~ rows | r rows | geometry] of patch p
  const int32_t* node_table;  // [n_rows][npp] or NULL (then X is read)
  const float4* xg;           // x~ (float4 per node)
  const float4* rg;           // r
  const float* geom;          // [n_rows][n_geo]
  int npp, n_geo;
  // GM_STAGED: distinct nodes per tile (dnnmg_patchset_t.tile_*)
  int tile_cap;
  const int32_t* tile_nodes;
  const int32_t* tile_count;
  const uint16_t* tile_slot;
  long long* trace;  // debug timeline of CTA 0 (env DNNMG_MLP_TRACE=file), else NULL
};
constexpr int kTraceSlots = 12288;
// timeline probe (tools/mlp_trace.py): one clock64() sample per slot, CTA 0 only.  Compiled
// in only with -DDNNMG_MLP_TRACE_BUILD (tools/gpu/trace_mlp.sh): even when disabled at run
// time, a probe's divergent branch in the chunk loop costs ~10 % of the kernel.
#ifdef DNNMG_MLP_TRACE_BUILD
#define TC_TRACE(slot)                                                              \
  do {                                                                              \
    if (A.trace && blockIdx.x == 0 && (slot) < kTraceSlots) A.trace[(slot)] = clock64();   \
  } while (0)
#else
#define TC_TRACE(slot) \
  do {                 \
  } while (0)
#endif

// shared-memory bytes of the GM_STAGED staging area: slot block, geometry rows, x~/r rows
__host__ __device__ inline uint32_t staged_slot_bytes(int npp) { return (kTcM * npp * 2 + 15) / 16 * 16; }
__host__ __device__ inline uint32_t staged_bytes(int npp, int n_geo, int cap) {
  return staged_slot_bytes(npp) + kTcM * n_geo * 4 + 2u * 16u * cap;
}

template <int MODE, int GM, int H>
__global__ void __launch_bounds__(TcRoles<GM>::kThreads, 1) mlp_tc_kernel(TcArgs A) {
  using R = TcRoles<GM>;
  constexpr int kNQ = R::NQ, kComputeWarps = R::kComputeWarps, kComputeThreads = R::kComputeThreads;
  constexpr int kProducerWarp = R::kProducerWarp, kMmaWarp = R::kMmaWarp, kGatherWarp = R::kGatherWarp;
  constexpr bool GATHER = GM != GM_X;
  using C = TcCfg<MODE>;
  constexpr int KC = C::KC;
  constexpr int HC = KC / kNQ;                     // K columns per thread per chunk
  constexpr int NCH = H / KC;                      // chunks of a hidden layer
  constexpr int NCH0 = kTcIn / KC;                 // chunks of the (at most kTcIn) inputs
  constexpr int WST = H * KC * C::ESZ * C::PARTS;  // bytes per weight stage
  constexpr int AST = kTcM * KC * C::ESZ * C::PARTS;  // bytes per A stage
  constexpr uint32_t SBO = KC * C::ESZ * 8;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* wring = smem;
  uint8_t* aring = smem + C::NW * WST;
  uint64_t* bars = reinterpret_cast<uint64_t*>(aring + C::NA * AST);
  uint64_t* w_full = bars;
  uint64_t* w_empty = bars + C::NW;
  uint64_t* a_full = bars + 2 * C::NW;
  uint64_t* a_empty = bars + 2 * C::NW + C::NA;
  uint64_t* acc_full = bars + 2 * C::NW + 2 * C::NA;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* idx_full = acc_empty + 2;   // fused gather: next tile's node indices staged by TMA
  uint64_t* idx_empty = idx_full + 1;
  uint64_t* stage_full = idx_empty + 1;   // GM_STAGED: the tile's nodes are in SMEM
  uint64_t* stage_empty = stage_full + 1; // GM_STAGED: staging area free (layer 0 consumed it,
                                          // or, y_mode 3, the previous tile's Y written to it)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(stage_empty + 1);
  // BN shift per hidden layer and the input normalisation, staged once per CTA.  The BN scale
  // (times k2 below) is folded into the packed weight columns (pack_kernel), so a hidden
  // epilogue computes z = acc * 2^-s_g + shift' with one warp-uniform factor per layer and
  // reads only the shift from shared memory.
  float* p_shift = reinterpret_cast<float*>(tmem_slot + 4);
  float* p_mean = p_shift + A.depth * H;
  float* p_rstd = p_mean + kTcIn;
  const PackHdr* hdr = reinterpret_cast<const PackHdr*>(A.packed);
  // fp32-accuracy tanh takes 2^(2 log2(e) z): fold 2 log2(e) into the BN scale and shift so
  // that the epilogue needs one FFMA before ex2 (the activation never needs z itself)
  const bool fold = tanh_folded(MODE, A.act);
  const float k2 = fold ? kTanhK2 : 1.0f;
  for (int i = threadIdx.x; i < A.depth * H; i += blockDim.x) p_shift[i] = A.shift[i] * k2;
  const float y_unscale = hdr->unscale[A.depth];
  int32_t* idx_s = reinterpret_cast<int32_t*>(p_rstd + kTcIn);  // [kTcM][npp] (GM_DIRECT only)
  // GM_STAGED: slot block [kTcM][npp] u16 | geometry rows [kTcM][n_geo] | x~ [cap] | r [cap]
  uint8_t* st_base = reinterpret_cast<uint8_t*>(p_rstd + kTcIn);
  const uint16_t* slot_s = reinterpret_cast<const uint16_t*>(st_base);
  float4* geo_s = reinterpret_cast<float4*>(st_base + staged_slot_bytes(A.npp));
  float4* stx = geo_s + kTcM * A.n_geo / 4;
  float4* str = stx + A.tile_cap;
  float* y_stage = reinterpret_cast<float*>(
      st_base + (GM == GM_DIRECT ? kTcM * A.npp * 4
                                 : GM == GM_STAGED ? staged_bytes(A.npp, A.n_geo, A.tile_cap) : 0));
  for (int i = threadIdx.x; i < kTcIn; i += blockDim.x) {
    p_mean[i] = i < A.n_in ? A.in_mean[i] : 0.f;
    p_rstd[i] = i < A.n_in ? 1.0f / A.in_std[i] : 0.f;
  }

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t n_tiles = (A.n_rows + kTcM - 1) / kTcM;
  const int G = A.depth + 1;  // GEMMs per tile

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NW; ++i) {
      mbar_init(smem_u32(&w_full[i]), 1);
      mbar_init(smem_u32(&w_empty[i]), 1);
    }
    for (int i = 0; i < C::NA; ++i) {
      mbar_init(smem_u32(&a_full[i]), kComputeWarps);
      mbar_init(smem_u32(&a_empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&acc_full[i]), 1);
      mbar_init(smem_u32(&acc_empty[i]), kComputeWarps);
    }
    mbar_init(smem_u32(idx_full), 1);
    mbar_init(smem_u32(idx_empty), kComputeWarps);
    mbar_init(smem_u32(stage_full), 1);
    mbar_init(smem_u32(stage_empty), kComputeWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kProducerWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kProducerWarp) {
    // ---------------- weight producer ----------------
    if (lane == 0) {
      uint32_t item = 0;
      // fused gather: each full tile's node-index block (kTcM x npp int32, contiguous) is
      // copied into shared memory one tile ahead (partial tiles read the indices directly)
      const uint32_t idx_bytes = (uint32_t)kTcM * A.npp * 4;
      auto full_tile = [&](int64_t t) { return t < n_tiles && (t + 1) * kTcM <= A.n_rows; };
      uint32_t icopy = 0;
      auto stage_idx = [&](int64_t t) {
        if (GM != GM_DIRECT || !full_tile(t) || (idx_bytes & 15)) return;
        if (icopy > 0) mbar_wait(smem_u32(idx_empty), (icopy - 1) & 1);
        mbar_expect_tx(smem_u32(idx_full), idx_bytes);
        bulk_g2s(smem_u32(idx_s), A.node_table + t * kTcM * A.npp, idx_bytes, smem_u32(idx_full));
        ++icopy;
      };
      stage_idx(blockIdx.x);
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        stage_idx(tile + gridDim.x);
        for (int g = 0; g < G; ++g) {
          const int N = g < A.depth ? H : A.Nhead;
          const int nk = (g == 0 ? A.K0p : H) / KC;
          const uint32_t bytes = (uint32_t)N * KC * C::ESZ * C::PARTS;
          for (int c = 0; c < nk; ++c, ++item) {
            const int s = item % C::NW;
            const uint32_t round = item / C::NW;
            mbar_wait(smem_u32(&w_empty[s]), (round & 1) ^ 1);
            mbar_expect_tx(smem_u32(&w_full[s]), bytes);
            bulk_g2s(smem_u32(wring + s * WST), A.packed + A.goff[g] + (int64_t)c * bytes, bytes,
                     smem_u32(&w_full[s]));
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      uint32_t witem = 0, aitem = 0, j = 0;
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        for (int g = 0; g < G; ++g, ++j) {
          const int N = g < A.depth ? H : A.Nhead;
          const int nk = (g == 0 ? A.K0p : H) / KC;
          const uint32_t idesc = idesc_for<MODE>(N);
          const int buf = j & 1;
          mbar_wait(smem_u32(&acc_empty[buf]), ((j >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d = tmem + buf * H;
          // layer 0: k-steps wholly inside the zero padding of K0p (n_in = 240 -> 256 at
          // KC = 32) are skipped; their products are exact zeros
          const int nks_last = g == 0 ? (A.n_in - (nk - 1) * KC + C::KSTEP - 1) / C::KSTEP : KC / C::KSTEP;
          for (int c = 0; c < nk; ++c, ++witem, ++aitem) {
            const int sw = witem % C::NW, sa = aitem % C::NA;
            const int nks = c == nk - 1 ? nks_last : KC / C::KSTEP;
            mbar_wait(smem_u32(&w_full[sw]), (witem / C::NW) & 1);
            TC_TRACE(4 * aitem);
            mbar_wait(smem_u32(&a_full[sa]), (aitem / C::NA) & 1);
            TC_TRACE(4 * aitem + 1);
            tc_fence_after();
            const uint32_t wb = smem_u32(wring + sw * WST);
            const uint32_t ab = smem_u32(aring + sa * AST);
#pragma unroll
            for (int ks = 0; ks < KC / C::KSTEP; ++ks) {
              if (ks >= nks) break;
              const uint32_t koff = ks * 256;
              const uint32_t acc = (c > 0 || ks > 0) ? 1u : 0u;
              const uint64_t ahi = sdesc(ab + koff, SBO), bhi = sdesc(wb + koff, SBO);
              tc_mma<MODE>(d, ahi, bhi, idesc, acc);
              if constexpr (C::PARTS == 2) {
                const uint64_t alo = sdesc(ab + kTcM * KC * C::ESZ + koff, SBO);
                const uint64_t blo = sdesc(wb + (uint32_t)N * KC * C::ESZ + koff, SBO);
                tc_mma<MODE>(d, ahi, blo, idesc, 1u);
                tc_mma<MODE>(d, alo, bhi, idesc, 1u);
              }
            }
            tc_commit(smem_u32(&w_empty[sw]));
            tc_commit(smem_u32(&a_empty[sa]));
            TC_TRACE(4 * aitem + 2);
          }
          tc_commit(smem_u32(&acc_full[buf]));
          TC_TRACE(6400 + j);
        }
      }
    }
  } else if (warp == kGatherWarp) {
    // ---------------- staged gather (GM_STAGED) ----------------
    // Tile t's distinct x~ and r rows (cp.async, 16 B each), its slot block and its geometry
    // rows (bulk copies) land in SMEM while the compute warps run tile t - grid; the
    // layer-0 operand of tile t is then built from SMEM (patch_ops.py:49-53).
    if constexpr (GM == GM_STAGED) {
      // y_mode 3: the staging area alternates between staged nodes and the previous tile's
      // Y; phase it-1 of stage_empty = area free (it = 1: tile 0 consumed; it >= 2: Y of the
      // tile it-2 written), so store that Y, then stage tile it
      const bool ystore = A.y_mode == 3;
      const int64_t n_mine = (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
      auto store_y = [&](int64_t yt) {
        const int64_t r0 = yt * kTcM;
        const int nv = (int)((A.n_rows - r0) < kTcM ? (A.n_rows - r0) : kTcM);
        const uint32_t bytes = (uint32_t)nv * A.n_out * 4;
        float* dst = A.Y + r0 * A.n_out;
        const float* ys = reinterpret_cast<const float*>(st_base);
        if ((bytes & 15) == 0) {
          if (lane == 0) {
            bulk_s2g(dst, smem_u32(ys), bytes);
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
        } else {
          for (uint32_t i = lane; i < bytes / 4; i += 32) dst[i] = ys[i];
        }
        __syncwarp();
      };
      uint32_t it = 0;
      for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
        if (it > 0) mbar_wait(smem_u32(stage_empty), (it - 1) & 1);
        if (ystore && it >= 2) store_y(tile - 2 * gridDim.x);
        const int64_t r0 = tile * kTcM;
        const int nvalid = (int)((A.n_rows - r0) < kTcM ? (A.n_rows - r0) : kTcM);
        if (lane == 0) {
          const uint32_t sb = (uint32_t)kTcM * A.npp * 2, gb = (uint32_t)nvalid * A.n_geo * 4;
          mbar_add_tx(smem_u32(stage_full), sb + gb);
          bulk_g2s(smem_u32(slot_s), A.tile_slot + r0 * A.npp, sb, smem_u32(stage_full));
          bulk_g2s(smem_u32(geo_s), A.geom + r0 * A.n_geo, gb, smem_u32(stage_full));
        }
        const int cnt = __ldg(A.tile_count + tile);
        const int32_t* un = A.tile_nodes + tile * A.tile_cap;
        constexpr int kIdxPerLane = 64;   // up to 2048 distinct nodes: all index loads in flight
        if (cnt <= 32 * kIdxPerLane) {
          int u[kIdxPerLane];
#pragma unroll
          for (int k = 0; k < kIdxPerLane; ++k) {
            const int i = 32 * k + lane;
            u[k] = i < cnt ? __ldg(un + i) : -1;
          }
#pragma unroll
          for (int k = 0; k < kIdxPerLane; ++k) {
            if (u[k] >= 0) {
              cp_async16(stx + 32 * k + lane, A.xg + u[k]);
              cp_async16(str + 32 * k + lane, A.rg + u[k]);
            }
          }
        } else
        for (int i0 = 0; i0 < cnt; i0 += 32 * 8) {
          int u[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int i = i0 + 32 * k + lane;
            u[k] = i < cnt ? __ldg(un + i) : -1;
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int i = i0 + 32 * k + lane;
            if (u[k] >= 0) {
              cp_async16(stx + i, A.xg + u[k]);
              cp_async16(str + i, A.rg + u[k]);
            }
          }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(stage_full));
      }
      if (ystore) {
        // remaining phases: n_mine - 1 (Y of tile n_mine - 2; for n_mine = 1 phase 0, tile 0
        // consumed) and n_mine (Y of the last tile).  The last tile has no next tile to stage,
        // so the area being free again is signalled on stage_full explicitly.
        for (int64_t ph = (n_mine >= 2 ? n_mine - 1 : 0); ph <= n_mine; ++ph) {
          mbar_wait(smem_u32(stage_empty), (uint32_t)ph & 1);
          if (ph >= 1) store_y(blockIdx.x + (ph - 1) * gridDim.x);
          if (ph == n_mine - 1 && n_mine >= 2 && lane == 0) mbar_arrive(smem_u32(stage_full));
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      }
    }
  } else {
    // ---------------- compute warps ----------------
    const int quad = warp & 3;          // TMEM lane quadrant
    const int hh = warp >> 2;           // which KC / kNQ column slice of every K chunk
    const int row_in_tile = quad * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    constexpr bool accurate = MODE != DNNMG_PREC_BF16;
    float h[NCH][HC];                   // fp32 skip state of this thread's row, 128 columns
    uint32_t aitem = 0, j = 0;

    auto produce_chunk = [&](int c, const float* v) {
      const int s = aitem % C::NA;
      mbar_wait(smem_u32(&a_empty[s]), ((aitem / C::NA) & 1) ^ 1);
      if (warp == 0 && lane == 0) TC_TRACE(8192 + aitem);
      put_row<MODE, HC>(aring + s * AST, row_in_tile, HC * hh, v);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&a_full[s]));
      if (warp == 0 && lane == 0) TC_TRACE(4 * aitem + 3);
      ++aitem;
      (void)c;
    };

    const int nck0 = A.K0p / KC;
    const bool vec_x = (A.n_in & 3) == 0;
    float xin[NCH0][HC];                 // raw input row slice of the next tile (prefetched)
    uint32_t iload = 0;                 // staged index blocks consumed
    const bool idx_staged = GATHER && ((kTcM * A.npp * 4) & 15) == 0;
    auto load_x = [&](int64_t tile) {
      const int64_t row = tile * kTcM + row_in_tile;
      const bool from_smem = idx_staged && tile < n_tiles && (tile + 1) * kTcM <= A.n_rows;
      if (from_smem) mbar_wait(smem_u32(idx_full), iload & 1);
      const bool ok = tile < n_tiles && row < A.n_rows;
      if constexpr (GM == GM_DIRECT) {
        // fused gather (patch_ops.py:49-53): float4 slot s of the row is x~ of node s,
        // r of node s - npp, or geometry; indices first, then all value loads in flight
        const int32_t* nt = A.node_table + row * A.npp;
        const int geo4 = A.n_geo / 4;
        int nidx[NCH0][HC / 4];
#pragma unroll
        for (int c = 0; c < NCH0; ++c)
#pragma unroll
          for (int j = 0; j < HC / 4; ++j) {
            const int f4 = (KC / 4) * c + (HC / 4) * hh + j;
            const int s = f4 < A.npp ? f4 : f4 - A.npp;
            nidx[c][j] = (ok && c < nck0 && f4 < 2 * A.npp)
                             ? (from_smem ? idx_s[row_in_tile * A.npp + s] : __ldg(nt + s))
                             : 0;
          }
        if (from_smem) {  // the index block may be overwritten with the next tile's
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(idx_empty));
          ++iload;
        }
#pragma unroll
        for (int c = 0; c < NCH0; ++c)
#pragma unroll
          for (int j = 0; j < HC / 4; ++j) {
            const int f4 = (KC / 4) * c + (HC / 4) * hh + j;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (ok && c < nck0) {
              if (f4 < A.npp) v = __ldg(A.xg + nidx[c][j]);
              else if (f4 < 2 * A.npp) v = __ldg(A.rg + nidx[c][j]);
              else if (f4 < 2 * A.npp + geo4)
                v = __ldg(reinterpret_cast<const float4*>(A.geom + row * A.n_geo) + (f4 - 2 * A.npp));
            }
            xin[c][4 * j] = v.x;
            xin[c][4 * j + 1] = v.y;
            xin[c][4 * j + 2] = v.z;
            xin[c][4 * j + 3] = v.w;
          }
        return;
      } else {
      const float* xr = A.X + row * A.n_in;
#pragma unroll
      for (int c = 0; c < NCH0; ++c) {
#pragma unroll
        for (int j = 0; j < HC / 4; ++j) {
          const int col = c * KC + HC * hh + 4 * j;
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (ok && c < nck0) {
            if (vec_x) {
              if (col < A.n_in) v = __ldg(reinterpret_cast<const float4*>(xr + col));
            } else {
              if (col < A.n_in) v.x = __ldg(xr + col);
              if (col + 1 < A.n_in) v.y = __ldg(xr + col + 1);
              if (col + 2 < A.n_in) v.z = __ldg(xr + col + 2);
              if (col + 3 < A.n_in) v.w = __ldg(xr + col + 3);
            }
          }
          xin[c][4 * j] = v.x;
          xin[c][4 * j + 1] = v.y;
          xin[c][4 * j + 2] = v.z;
          xin[c][4 * j + 3] = v.w;
        }
      }
      }
    };
    // layer-0 operand: normalised input rows (net.py:131), from the prefetched registers
    auto produce_layer0 = [&]() {
#pragma unroll
      for (int c = 0; c < NCH0; ++c) {
        if (c < nck0) {
          float v[HC];
#pragma unroll
          for (int e = 0; e < HC; e += 4) {
            const int col = c * KC + HC * hh + e;
            const float4 mu = *reinterpret_cast<const float4*>(p_mean + col);
            const float4 rs = *reinterpret_cast<const float4*>(p_rstd + col);
            v[e + 0] = (xin[c][e + 0] - mu.x) * rs.x;
            v[e + 1] = (xin[c][e + 1] - mu.y) * rs.y;
            v[e + 2] = (xin[c][e + 2] - mu.z) * rs.z;
            v[e + 3] = (xin[c][e + 3] - mu.w) * rs.w;
          }
          produce_chunk(c, v);
        }
      }
    };
    // GM_STAGED: layer-0 operand of `tile` from the staged nodes (gather warp)
    uint32_t sit = 0;
    auto produce_layer0_staged = [&](int64_t tile) {
      mbar_wait(smem_u32(stage_full), sit & 1);
      if (warp == 0 && lane == 0) TC_TRACE(6915 + 4 * (int)sit);
      const bool ok = tile * kTcM + row_in_tile < A.n_rows;
      const uint16_t* sl = slot_s + row_in_tile * A.npp;
      const float4* gr = geo_s + row_in_tile * (A.n_geo / 4);
      const int geo4 = A.n_geo / 4;
#pragma unroll
      for (int c = 0; c < NCH0; ++c) {
        if (c < nck0) {
          float v[HC];
#pragma unroll
          for (int j = 0; j < HC / 4; ++j) {
            const int f4 = (KC / 4) * c + (HC / 4) * hh + j;
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
            if (ok) {
              if (f4 < A.npp) x = stx[sl[f4]];
              else if (f4 < 2 * A.npp) x = str[sl[f4 - A.npp]];
              else if (f4 < 2 * A.npp + geo4) x = gr[f4 - 2 * A.npp];
            }
            const int col = c * KC + HC * hh + 4 * j;
            const float4 mu = *reinterpret_cast<const float4*>(p_mean + col);
            const float4 rs = *reinterpret_cast<const float4*>(p_rstd + col);
            v[4 * j + 0] = (x.x - mu.x) * rs.x;
            v[4 * j + 1] = (x.y - mu.y) * rs.y;
            v[4 * j + 2] = (x.z - mu.z) * rs.z;
            v[4 * j + 3] = (x.w - mu.w) * rs.w;
          }
          produce_chunk(c, v);
        }
      }
      // y_mode 3: after the first tile the area is released by the head epilogue instead
      if (A.y_mode != 3 || sit == 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(stage_empty));
      }
      ++sit;
    };
    if constexpr (GM == GM_STAGED) {
      produce_layer0_staged(blockIdx.x);
    } else {
      load_x(blockIdx.x);
      produce_layer0();
    }

    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const int64_t row = tile * kTcM + row_in_tile;
      const bool live = row < A.n_rows;
      // hidden layers: h = act(BN(z)) + h with h = 0 entering layer 0 (net.py:151: no skip
      // for layer 0); one epilogue body keeps the unrolled code (and I-cache footprint) small
#pragma unroll
      for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int e = 0; e < HC; ++e) h[c][e] = 0.f;
      for (int g = 0; g < A.depth; ++g) {
        const int buf = j & 1;
        if (warp == 0 && lane == 0) TC_TRACE(6656 + j);
        mbar_wait(smem_u32(&acc_full[buf]), (j >> 1) & 1);
        if (warp == 0 && lane == 0) TC_TRACE(6144 + j);
        tc_fence_after();
        const float us = hdr->unscale[g];  // 2^-s_g: exact
        const float* sh = p_shift + g * H;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          float v[HC];
          if (warp == 0 && lane == 0) TC_TRACE(9216 + aitem);
          tmem_ld<HC>(tmem + lane_addr + buf * H + c * KC + HC * hh, v);
          if (warp == 0 && lane == 0) TC_TRACE(10240 + aitem);
#pragma unroll
          for (int e = 0; e < HC; e += 4) {
            const int col = c * KC + HC * hh + e;
            const float4 t4 = *reinterpret_cast<const float4*>(sh + col);
            const float tv[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float z = fmaf(v[e + u], us, tv[u]);
              float a;
              if (fold) {  // z = 2 log2(e) * BN(acc): tanh = 1 - 2 / (1 + 2^z)
                float ez, r;
                asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(ez) : "f"(z));
                asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + ez));
                a = fmaf(-2.0f, r, 1.0f);
              } else {
                a = act_fast(z, A.act, accurate);
              }
              h[c][e + u] = a + h[c][e + u];
              v[e + u] = h[c][e + u];
            }
          }
          if (warp == 0 && lane == 0) TC_TRACE(11264 + aitem);
          produce_chunk(c, v);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&acc_empty[buf]));
        ++j;
      }
      // the skip state is dead now: prefetch the next tile's input under the head GEMM
      if (warp == 0 && lane == 0) TC_TRACE(6912 + (int)((tile - blockIdx.x) / gridDim.x) * 4);
      if constexpr (GM != GM_STAGED) load_x(tile + gridDim.x);
      if (warp == 0 && lane == 0) TC_TRACE(6913 + (int)((tile - blockIdx.x) / gridDim.x) * 4);
      // the next tile's layer-0 operand goes into the ring right behind this tile's head
      // chunks: the MMA warp runs it while this tile's head epilogue is in progress
      if (tile + gridDim.x < n_tiles) {
        if constexpr (GM == GM_STAGED) produce_layer0_staged(tile + gridDim.x);
        else produce_layer0();
      }
      // head: Y = h W_depth
      {
        const int buf = j & 1;
        if (warp == 0 && lane == 0) TC_TRACE(6656 + j);
        mbar_wait(smem_u32(&acc_full[buf]), (j >> 1) & 1);
        if (warp == 0 && lane == 0) TC_TRACE(6144 + j);
        tc_fence_after();
        if (A.y_mode == 3) {
          // the whole tile into the staging area (its nodes were consumed above: wait for all
          // compute warps), then one bulk store from the gather warp (stage_empty)
          asm volatile("bar.sync 1, %0;" ::"n"(kComputeThreads) : "memory");
          if (tile + gridDim.x >= n_tiles && tile >= (int64_t)gridDim.x) {
            // last tile of several: wait until the previous tile's Y has left the area
            mbar_wait(smem_u32(stage_full), sit & 1);
            ++sit;
          }
          float* ys = reinterpret_cast<float*>(st_base);
          for (int sl = hh; sl < A.Nhead / 16; sl += kNQ) {
            float v[16];
            tmem_ld16(tmem + lane_addr + buf * H + sl * 16, v);
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int col = sl * 16 + e;
              if (col < A.n_out) ys[row_in_tile * A.n_out + col] = v[e] * y_unscale;
            }
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(stage_empty));
        } else if (A.y_mode == 0) {
          for (int sl = hh; sl < A.Nhead / 16; sl += kNQ) {
            float v[16];
            tmem_ld16(tmem + lane_addr + buf * H + sl * 16, v);
            if (live) {
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                const int col = sl * 16 + e;
                if (col < A.n_out) A.Y[row * A.n_out + col] = v[e] * y_unscale;
              }
            }
          }
        } else {
        // stage the 128 x n_out tile through a 64-row SMEM buffer in two halves (the A ring
        // already carries the next tile's layer-0 chunks; a small buffer leaves more L1 for
        // the fused gather), each followed by one coalesced block copy
        float* ys = y_stage;
        const int64_t r0 = tile * kTcM;
        const int nvalid = (int)((A.n_rows - r0) < kTcM ? (A.n_rows - r0) : kTcM);
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          if ((quad >> 1) == half) {
            for (int sl = hh; sl < A.Nhead / 16; sl += kNQ) {
              float v[16];
              tmem_ld16(tmem + lane_addr + buf * H + sl * 16, v);
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                const int col = sl * 16 + e;
                if (col < A.n_out) ys[(row_in_tile - 64 * half) * A.n_out + col] = v[e] * y_unscale;
              }
            }
          }
          tc_fence_before();
          asm volatile("bar.sync 1, %0;" ::"n"(kComputeThreads) : "memory");
          {  // coalesced copy of this half's contiguous Y block
            const int nh = nvalid - 64 * half;
            const int nf = (nh < 0 ? 0 : nh > 64 ? 64 : nh) * A.n_out;
            float* dst = A.Y + (r0 + 64 * half) * A.n_out;
            const int tid = threadIdx.x;
            const int n4 = nf >> 2;
            for (int i = tid; i < n4; i += kComputeThreads)
              reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(ys)[i];
            for (int i = 4 * n4 + tid; i < nf; i += kComputeThreads) dst[i] = ys[i];
          }
          asm volatile("bar.sync 1, %0;" ::"n"(kComputeThreads) : "memory");
        }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&acc_empty[buf]));
        if (warp == 0 && lane == 0) TC_TRACE(6914 + (int)((tile - blockIdx.x) / gridDim.x) * 4);
        ++j;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kProducerWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// ---- weight packing: W[g] (K x N row-major fp32) -> canonical chunk images -----
// per-GEMM exponent s with max|W'| 2^s < 2^14 (F16X3), else s = 0; one block.  W' = W, or
// for the fused kernel's hidden GEMMs W with column n scaled by colf[n] * k2 (BN scale fold)
__global__ void pack_scale_kernel(const float* __restrict__ W, int size, int N,
                                  const float* __restrict__ colf, float k2, int mode, int g,
                                  PackHdr* __restrict__ hdr) {
  float m = 0.f;
  for (int i = threadIdx.x; i < size; i += blockDim.x)
    m = fmaxf(m, fabsf(colf ? W[i] * (colf[i % N] * k2) : W[i]));
  __shared__ float red[32];
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) m = fmaxf(m, red[i]);
    m = fmaxf(m, red[0]);
    int s = 0;
    if ((mode == DNNMG_PREC_F16X3 || mode == DNNMG_PREC_FP8) && m > 0.f && isfinite(m)) {
      int e;
      frexpf(m, &e);  // m < 2^e
      s = (mode == DNNMG_PREC_FP8 ? 8 : 14) - e;   // e4m3 max 448, fp16 max 65504
    }
    hdr->shift[g] = s;
    hdr->unscale[g] = ldexpf(1.0f, -s);
  }
}

template <int MODE>
__global__ void pack_kernel(const float* __restrict__ W, int K, int N, int Kp, int Np,
                            const float* __restrict__ colf, float k2,
                            const PackHdr* __restrict__ hdr, int g, uint8_t* __restrict__ out) {
  const int shift = hdr->shift[g];
  using C = TcCfg<MODE>;
  constexpr int KC = C::KC;
  const int64_t total = (int64_t)Kp * Np;
  const uint32_t part = (uint32_t)Np * KC * C::ESZ;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(i % Np);
    const int k = (int)(i / Np);
    float w = (k < K && n < N) ? W[(int64_t)k * N + n] : 0.f;
    if (colf && n < N) w *= colf[n] * k2;
    const int c = k / KC, kk = k % KC;
    uint8_t* chunk = out + (int64_t)c * part * C::PARTS;
    const uint32_t off = canon_off<C::ESZ, KC>(n, kk);
    if constexpr (MODE == DNNMG_PREC_BF16) {
      *reinterpret_cast<__nv_bfloat16_raw*>(chunk + off) =
          static_cast<__nv_bfloat16_raw>(__float2bfloat16_rn(w));
    } else if constexpr (MODE == DNNMG_PREC_F16X3) {
      const float ws = ldexpf(w, shift);  // exact power-of-two scaling
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

// per-GEMM weight exponents into the header of a packed image (shared with mlp_layer.cu;
// fold_bn: exponents of the BN-scale-folded hidden weights of the fused kernel)
int32_t launch_pack_scales(const dnnmg_mlp_t* m, PackHdr* hdr, cudaStream_t s, bool fold_bn) {
  const float k2 = tanh_folded(m->precision, m->activation) ? kTanhK2 : 1.0f;
  for (int g = 0; g <= m->depth; ++g) {
    const int N = g < m->depth ? m->n_hidden : m->n_out;
    const int size = (g == 0 ? m->n_in : m->n_hidden) * N;
    const float* colf = fold_bn && g < m->depth ? m->bn_scale + (int64_t)g * m->n_hidden : nullptr;
    pack_scale_kernel<<<1, 256, 0, s>>>(m->W[g], size, N, colf, k2, m->precision, g, hdr);
    DNNMG_CHECK_LAUNCH("pack_scale_kernel");
  }
  return DNNMG_OK;
}

static int round_up(int x, int m) { return (x + m - 1) / m * m; }

int32_t mlp_tc_supported(const dnnmg_mlp_t* m) {
  return (m->precision == DNNMG_PREC_BF16 || m->precision == DNNMG_PREC_TF32X3 ||
          m->precision == DNNMG_PREC_F16X3) &&
         (m->n_hidden == 256 || m->n_hidden == 128) && m->n_in <= kTcIn &&
         m->n_out <= m->n_hidden && m->depth >= 1 &&
         m->depth < DNNMG_MAX_LAYERS;
}

static void layout(const dnnmg_mlp_t* m, int64_t* goff, int64_t* total) {
  const int esz = m->precision == DNNMG_PREC_TF32X3 ? 4 : 2;
  const int parts = m->precision == DNNMG_PREC_BF16 ? 1 : 2;
  int64_t off = kPackHdr;
  for (int g = 0; g <= m->depth; ++g) {
    const int K = g == 0 ? round_up(m->n_in, kc_of(m->precision)) : m->n_hidden;
    const int N = g < m->depth ? m->n_hidden : round_up(m->n_out, 16);
    goff[g] = off;
    off += (int64_t)K * N * esz * parts;
  }
  *total = off;
}

int32_t mlp_tc_packed_bytes(const dnnmg_mlp_t* m, int64_t* bytes) {
  DNNMG_REQUIRE(mlp_tc_supported(m), DNNMG_ERR_UNSUPPORTED,
                "mlp: fused tensor-core mode needs n_hidden 128 or 256, n_in <= 256, "
                "n_out <= n_hidden");
  int64_t goff[DNNMG_MAX_LAYERS];
  layout(m, goff, bytes);
  return DNNMG_OK;
}

int32_t launch_mlp_tc_pack(const dnnmg_mlp_t* m, void* packed, cudaStream_t s) {
  DNNMG_REQUIRE(mlp_tc_supported(m), DNNMG_ERR_UNSUPPORTED,
                "mlp: fused tensor-core mode needs n_hidden 128 or 256, n_in <= 256, "
                "n_out <= n_hidden");
  int64_t goff[DNNMG_MAX_LAYERS], total;
  layout(m, goff, &total);
  PackHdr* hdr = static_cast<PackHdr*>(packed);
  static_assert(sizeof(PackHdr) <= kPackHdr, "pack header");
  int32_t rc = launch_pack_scales(m, hdr, s, true);
  if (rc) return rc;
  const float k2 = tanh_folded(m->precision, m->activation) ? kTanhK2 : 1.0f;
  for (int g = 0; g <= m->depth; ++g) {
    const int H = m->n_hidden;
    const float* colf = g < m->depth ? m->bn_scale + (int64_t)g * H : nullptr;
    const int K = g == 0 ? m->n_in : H;
    const int N = g < m->depth ? H : m->n_out;
    const int Kp = g == 0 ? round_up(m->n_in, kc_of(m->precision)) : H;
    const int Np = g < m->depth ? H : round_up(m->n_out, 16);
    uint8_t* out = static_cast<uint8_t*>(packed) + goff[g];
    const int64_t n = (int64_t)Kp * Np;
    if (m->precision == DNNMG_PREC_BF16)
      pack_kernel<DNNMG_PREC_BF16><<<grid_for(n, 256), 256, 0, s>>>(m->W[g], K, N, Kp, Np, colf, k2, hdr, g, out);
    else if (m->precision == DNNMG_PREC_F16X3)
      pack_kernel<DNNMG_PREC_F16X3><<<grid_for(n, 256), 256, 0, s>>>(m->W[g], K, N, Kp, Np, colf, k2, hdr, g, out);
    else
      pack_kernel<DNNMG_PREC_TF32X3><<<grid_for(n, 256), 256, 0, s>>>(m->W[g], K, N, Kp, Np, colf, k2, hdr, g, out);
    DNNMG_CHECK_LAUNCH("pack_kernel");
  }
  return DNNMG_OK;
}

struct GatherSrc {
  const int32_t* node_table;
  const float* x;
  const float* r;
  const float* geom;
  int npp, n_geo;
  int tile_cap;
  const int32_t* tile_nodes;
  const int32_t* tile_count;
  const uint16_t* tile_slot;
};
constexpr size_t kSmemMax = 227 * 1024;

template <int MODE>
static size_t smem_base(const dnnmg_mlp_t* m) {
  using C = TcCfg<MODE>;
  const size_t WST = (size_t)m->n_hidden * C::KC * C::ESZ * C::PARTS;
  constexpr int AST = kTcM * C::KC * C::ESZ * C::PARTS;
  return (size_t)C::NW * WST + (size_t)C::NA * AST + 8 * (2 * C::NW + 2 * C::NA + 8) + 16 +
         sizeof(float) * ((size_t)m->depth * m->n_hidden + 2 * kTcIn);
}
static size_t smem_base_of(const dnnmg_mlp_t* m) {
  return m->precision == DNNMG_PREC_BF16 ? smem_base<DNNMG_PREC_BF16>(m)
         : m->precision == DNNMG_PREC_F16X3 ? smem_base<DNNMG_PREC_F16X3>(m)
                                            : smem_base<DNNMG_PREC_TF32X3>(m);
}
// layer-0 source: staged gather when the tile tables exist and the staging area fits next
// to the rings (env DNNMG_NO_STAGED forces the direct gather, for A/B measurements)
static int choose_gm(const dnnmg_mlp_t* m, const GatherSrc* g) {
  if (!g) return GM_X;
  if (g->tile_nodes && g->tile_count && g->tile_slot && g->tile_cap > 0 &&
      smem_base_of(m) + staged_bytes(g->npp, g->n_geo, g->tile_cap) <= kSmemMax &&
      !getenv("DNNMG_NO_STAGED"))
    return GM_STAGED;
  return GM_DIRECT;
}

template <int MODE>
static int32_t launch_mode(const dnnmg_mlp_t* m, const float* X, int64_t n_rows, float* Y,
                           cudaStream_t s, const GatherSrc* g) {
  using C = TcCfg<MODE>;
  TcArgs A;
  A.X = X;
  A.node_table = g ? g->node_table : nullptr;
  A.xg = g ? reinterpret_cast<const float4*>(g->x) : nullptr;
  A.rg = g ? reinterpret_cast<const float4*>(g->r) : nullptr;
  A.geom = g ? g->geom : nullptr;
  A.npp = g ? g->npp : 0;
  A.n_geo = g ? g->n_geo : 0;
  A.tile_cap = g ? g->tile_cap : 0;
  A.tile_nodes = g ? g->tile_nodes : nullptr;
  A.tile_count = g ? g->tile_count : nullptr;
  A.tile_slot = g ? g->tile_slot : nullptr;
  A.Y = Y;
  A.trace = nullptr;
  static const char* trace_file = getenv("DNNMG_MLP_TRACE");
  if (trace_file) {
    cudaMalloc(&A.trace, kTraceSlots * sizeof(long long));
    cudaMemsetAsync(A.trace, 0, kTraceSlots * sizeof(long long), s);
  }
  A.n_rows = n_rows;
  A.n_in = m->n_in;
  A.n_out = m->n_out;
  A.depth = m->depth;
  A.act = m->activation;
  A.K0p = round_up(m->n_in, C::KC);
  A.Nhead = round_up(m->n_out, 16);
  A.packed = static_cast<const uint8_t*>(m->packed);
  int64_t total;
  layout(m, A.goff, &total);
  A.scale = m->bn_scale;
  A.shift = m->bn_shift;
  A.in_mean = m->in_mean;
  A.in_std = m->in_std;
  const size_t base = smem_base<MODE>(m);
  const int gm = choose_gm(m, g);
  size_t smem = base + (gm == GM_DIRECT ? (size_t)kTcM * g->npp * 4
                        : gm == GM_STAGED ? staged_bytes(g->npp, g->n_geo, g->tile_cap) : 0);
  const size_t ybytes = (size_t)(kTcM / 2) * m->n_out * 4;  // staged in two 64-row halves
  if (gm == GM_STAGED && (size_t)kTcM * m->n_out * 4 <= staged_bytes(g->npp, g->n_geo, g->tile_cap) &&
      !getenv("DNNMG_Y_HALVES")) {
    A.y_mode = 3;
  } else if (smem + ybytes <= kSmemMax && !getenv("DNNMG_Y_DIRECT")) {
    A.y_mode = 2;
    smem += ybytes;
  } else {
    A.y_mode = 0;
  }
  if (smem < 120 * 1024) smem = 120 * 1024;  // one CTA per SM: TMEM (512 columns) is per SM
  const int64_t tiles = (n_rows + kTcM - 1) / kTcM;
  const int grid = (int)(tiles < kSMs ? tiles : kSMs);
  if (m->n_hidden == 128) {   // width 128: stored-X rows only (the patch paths use 256)
    DNNMG_REQUIRE(gm == GM_X, DNNMG_ERR_UNSUPPORTED,
                  "mlp: the fused patch gather needs n_hidden == 256");
    cudaFuncSetAttribute(mlp_tc_kernel<MODE, GM_X, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    mlp_tc_kernel<MODE, GM_X, 128><<<grid, TcRoles<GM_X>::kThreads, smem, s>>>(A);
  } else if (gm == GM_STAGED) {
    cudaFuncSetAttribute(mlp_tc_kernel<MODE, GM_STAGED, kTcH>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    mlp_tc_kernel<MODE, GM_STAGED, kTcH><<<grid, TcRoles<GM_STAGED>::kThreads, smem, s>>>(A);
  } else if (gm == GM_DIRECT) {
    cudaFuncSetAttribute(mlp_tc_kernel<MODE, GM_DIRECT, kTcH>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    mlp_tc_kernel<MODE, GM_DIRECT, kTcH><<<grid, TcRoles<GM_DIRECT>::kThreads, smem, s>>>(A);
  } else {
    cudaFuncSetAttribute(mlp_tc_kernel<MODE, GM_X, kTcH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    mlp_tc_kernel<MODE, GM_X, kTcH><<<grid, TcRoles<GM_X>::kThreads, smem, s>>>(A);
  }
  DNNMG_CHECK_LAUNCH("mlp_tc_kernel");
  if (A.trace) {  // debug only: synchronous copy-out of CTA 0's timeline
    static long long host[kTraceSlots];
    cudaMemcpyAsync(host, A.trace, sizeof(host), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaFree(A.trace);
    if (FILE* f = fopen(trace_file, "wb")) {
      fwrite(host, sizeof(host), 1, f);
      fclose(f);
    }
  }
  return DNNMG_OK;
}

int32_t launch_mlp_tc(const dnnmg_mlp_t* m, const float* X, int64_t n_rows, float* Y,
                      cudaStream_t s) {
  if (m->precision == DNNMG_PREC_BF16) return launch_mode<DNNMG_PREC_BF16>(m, X, n_rows, Y, s, nullptr);
  if (m->precision == DNNMG_PREC_F16X3) return launch_mode<DNNMG_PREC_F16X3>(m, X, n_rows, Y, s, nullptr);
  return launch_mode<DNNMG_PREC_TF32X3>(m, X, n_rows, Y, s, nullptr);
}

// K3 fused into K4: the network input rows are gathered from x~, r and the patch
// geometry while staging the layer-0 operand; X never touches HBM
int32_t mlp_tc_gather_mode(const dnnmg_mlp_t* m, const dnnmg_patchset_t* ps) {
  GatherSrc g{ps->node_table, nullptr,      nullptr,        ps->geom,      ps->nodes_per_patch,
              ps->n_geo,      ps->tile_cap, ps->tile_nodes, ps->tile_count, ps->tile_slot};
  return choose_gm(m, &g);
}

int32_t launch_mlp_tc_gather(const dnnmg_mlp_t* m, const dnnmg_patchset_t* ps, const float* x,
                             const float* r, float* Y, cudaStream_t s) {
  DNNMG_REQUIRE(ps->n_geo % 4 == 0 && 8 * ps->nodes_per_patch + ps->n_geo == m->n_in &&
                    m->n_in <= kTcH,
                DNNMG_ERR_UNSUPPORTED, "mlp_gather: needs 8*npp + n_geo == n_in <= 256");
  GatherSrc g{ps->node_table, x,         r,        ps->geom,      ps->nodes_per_patch, ps->n_geo,
              ps->tile_cap,   ps->tile_nodes, ps->tile_count, ps->tile_slot};
  if (m->precision == DNNMG_PREC_BF16)
    return launch_mode<DNNMG_PREC_BF16>(m, nullptr, ps->n_patches, Y, s, &g);
  if (m->precision == DNNMG_PREC_F16X3)
    return launch_mode<DNNMG_PREC_F16X3>(m, nullptr, ps->n_patches, Y, s, &g);
  return launch_mode<DNNMG_PREC_TF32X3>(m, nullptr, ps->n_patches, Y, s, &g);
}

}  // namespace dnnmg
