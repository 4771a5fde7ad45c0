// Training-data rows on the GPU: the feature/target rows of
// driver.export_training_data / oracle_loop_features (driver.py:317-431) in the byte
// layout of the reference's dataset shards (io.write_dataset, io.py:219-287).
//
//   row p = [ x~[node_table[p]] (4 npp) | r[...] (4 npp) | geom[p] (n_geo) | T (3 npp) ]
//   T     = (v_ref - x~) at the velocity slots  (patch_ops.patch_targets, patch_ops.py:79-82)
//
// Features come from the fp32 device vectors (the correction path's own x~ and r), the
// targets are formed in float64 from the fine reference run.  One warp per patch row: the
// lanes walk the row's float64 columns in order, so every row is written as one
// contiguous, coalesced stream (the row block is the D2H / disk payload).
//
// Column statistics (sum, centred sum of squares M2, min, max per column) for the dataset
// sidecar are reduced in a fixed order — per-block partials over fixed row ranges (one
// pass, sums shifted by the block's first row, M2 = q - s^2/n), then an in-order pairwise
// (Chan) combination over the blocks — so they are deterministic and free of the
// E[x^2] - mean^2 cancellation.
#include <cfloat>
#include "common.cuh"

namespace dnnmg {

__global__ void __launch_bounds__(256) dataset_rows_kernel(
    int n_patches, int npp, int n_geo, const int32_t* __restrict__ table,
    const float* __restrict__ x, const float* __restrict__ r, const float* __restrict__ geom,
    const double* __restrict__ v_ref, const double* __restrict__ x_ref, double* __restrict__ rows) {
  const int nf = 8 * npp + n_geo;
  const int w = nf + 3 * npp;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n_patches; p += warps) {
    const int32_t* tp = table + (int64_t)p * npp;
    double* out = rows + (int64_t)p * w;
    for (int j = lane; j < w; j += 32) {
      double v;
      if (j < 4 * npp) {                       // state block, node-major (p, vx, vy, vz)
        v = (double)__ldg(x + 4 * (int64_t)__ldg(tp + (j >> 2)) + (j & 3));
      } else if (j < 8 * npp) {                // residual block
        const int jj = j - 4 * npp;
        v = r ? (double)__ldg(r + 4 * (int64_t)__ldg(tp + (jj >> 2)) + (jj & 3)) : 0.0;
      } else if (j < nf) {                     // geometry
        v = (double)__ldg(geom + (int64_t)p * n_geo + (j - 8 * npp));
      } else {                                 // targets: velocity comps of node jj/3
        const int jj = j - nf;
        const int64_t dof = 4 * (int64_t)__ldg(tp + jj / 3) + 1 + jj % 3;
        if (v_ref) {
          const double xr = x_ref ? __ldg(x_ref + dof) : (double)__ldg(x + dof);
          v = __ldg(v_ref + dof) - xr;
        } else {
          v = 0.0;
        }
      }
      out[j] = v;
    }
  }
}

constexpr int kStatBlocks = 2048;  // fixed row partition of the column statistics

// partial[b][4][w]: block b reduces rows [b*chunk, (b+1)*chunk) column by column
__global__ void __launch_bounds__(256) column_stats_partial_kernel(const double* __restrict__ rows,
                                                                    int64_t n, int w,
                                                                    double* __restrict__ partial) {
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * chunk;
  const int64_t r1 = r0 + chunk < n ? r0 + chunk : n;
  double* pb = partial + (int64_t)blockIdx.x * 4 * w;
  for (int c = threadIdx.x; c < w; c += blockDim.x) {
    double s = 0.0, q = 0.0, mn = DBL_MAX, mx = -DBL_MAX;
    const double shift = r1 > r0 ? __ldg(rows + r0 * w + c) : 0.0;
    for (int64_t i = r0; i < r1; ++i) {
      const double v = __ldg(rows + i * w + c);
      const double d = v - shift;
      s += d;
      q = fma(d, d, q);
      mn = fmin(mn, v);
      mx = fmax(mx, v);
    }
    const int64_t n_b = r1 - r0;
    if (n_b > 0) {
      q = fmax(q - s * s / (double)n_b, 0.0);   // centred M2 of the block
      s += shift * (double)n_b;
    }
    pb[c] = s;
    pb[w + c] = q;
    pb[2 * w + c] = mn;
    pb[3 * w + c] = mx;
  }
}

// (n, sum, M2) pairwise combination (Chan et al.)
struct ColAcc {
  double n, s, q, mn, mx;
};
__device__ __forceinline__ ColAcc col_merge(const ColAcc& a, const ColAcc& b) {
  if (a.n == 0.0) return b;
  if (b.n == 0.0) return a;
  const double n = a.n + b.n;
  const double delta = b.s / b.n - a.s / a.n;
  return {n, a.s + b.s, a.q + b.q + delta * delta * (a.n * b.n / n), fmin(a.mn, b.mn),
          fmax(a.mx, b.mx)};
}

// one warp per column: lane l merges the partials of a fixed contiguous block range in
// order, then a fixed butterfly merges the lanes (a fixed tree: deterministic)
__global__ void __launch_bounds__(256) column_stats_final_kernel(const double* __restrict__ partial,
                                                                  int64_t n, int nb, int w,
                                                                  double* __restrict__ stats) {
  const int64_t chunk = (n + nb - 1) / nb;
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int per = (nb + 31) / 32;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < w; c += warps) {
    ColAcc acc{0.0, 0.0, 0.0, DBL_MAX, -DBL_MAX};
    for (int b = lane * per; b < nb && b < (lane + 1) * per; ++b) {
      const int64_t r0 = b * chunk, r1 = r0 + chunk < n ? r0 + chunk : n;
      if (r1 <= r0) continue;
      const double* pb = partial + (int64_t)b * 4 * w;
      acc = col_merge(acc, ColAcc{(double)(r1 - r0), pb[c], pb[w + c], pb[2 * w + c], pb[3 * w + c]});
    }
    for (int o = 1; o < 32; o <<= 1) {   // partner lane ^ o; the lower lane is "a"
      ColAcc other;
      other.n = __shfl_xor_sync(0xffffffffu, acc.n, o);
      other.s = __shfl_xor_sync(0xffffffffu, acc.s, o);
      other.q = __shfl_xor_sync(0xffffffffu, acc.q, o);
      other.mn = __shfl_xor_sync(0xffffffffu, acc.mn, o);
      other.mx = __shfl_xor_sync(0xffffffffu, acc.mx, o);
      acc = (lane & o) ? col_merge(other, acc) : col_merge(acc, other);
    }
    if (lane == 0) {
      stats[c] = acc.s;
      stats[w + c] = acc.q;
      stats[2 * w + c] = acc.mn;
      stats[3 * w + c] = acc.mx;
    }
  }
}

}  // namespace dnnmg

extern "C" int32_t dnnmg_dataset_rows(const dnnmg_patchset_t* ps, const float* x_tilde,
                                      const float* r, const double* v_ref, const double* x_ref,
                                      double* rows, dnnmg_stream_t s) {
  using namespace dnnmg;
  DNNMG_REQUIRE(ps && ps->node_table && ps->geom && x_tilde && rows, DNNMG_ERR_ARG,
                "dataset_rows: null argument");
  if (ps->n_patches == 0) return DNNMG_OK;
  const int64_t threads = (int64_t)ps->n_patches * 32;
  dataset_rows_kernel<<<grid_for(threads, 256, 16), 256, 0, as_stream(s)>>>(
      ps->n_patches, ps->nodes_per_patch, ps->n_geo, ps->node_table, x_tilde, r, ps->geom, v_ref,
      x_ref, rows);
  DNNMG_CHECK_LAUNCH("dataset_rows_kernel");
  return DNNMG_OK;
}

extern "C" int32_t dnnmg_column_stats_scratch(int32_t w) {
  return dnnmg::kStatBlocks * 4 * w;
}

extern "C" int32_t dnnmg_column_stats(const double* rows, int64_t n, int32_t w, double* scratch,
                                      double* stats, dnnmg_stream_t s) {
  using namespace dnnmg;
  DNNMG_REQUIRE(n >= 0 && w > 0 && stats && scratch && (n == 0 || rows), DNNMG_ERR_ARG,
                "column_stats: null argument or bad shape");
  column_stats_partial_kernel<<<kStatBlocks, 256, 0, as_stream(s)>>>(rows, n, w, scratch);
  DNNMG_CHECK_LAUNCH("column_stats_partial_kernel");
  column_stats_final_kernel<<<(w + 7) / 8, 256, 0, as_stream(s)>>>(scratch, n, kStatBlocks, w,
                                                                  stats);
  DNNMG_CHECK_LAUNCH("column_stats_final_kernel");
  return DNNMG_OK;
}

namespace dnnmg {
__global__ void __launch_bounds__(256) ideal_update_kernel(int n_nodes, const float4* __restrict__ xt,
                                                           const double* __restrict__ v_ref,
                                                           const uint8_t* __restrict__ mask,
                                                           float4* __restrict__ xc) {
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < n_nodes; n += gridDim.x * blockDim.x) {
    const float4 x = xt[n];
    const uint8_t m = mask ? mask[n] : 0;
    float o[4] = {x.x, x.y, x.z, x.w};
    const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int c = 1; c < 4; ++c) {   // pressure (c = 0) and constrained dofs keep x~
      if (!(m & (1 << c))) {
        const double d = v_ref[4 * (int64_t)n + c] - (double)xv[c];
        o[c] = (float)((double)xv[c] + d);
      }
    }
    xc[n] = make_float4(o[0], o[1], o[2], o[3]);
  }
}
}  // namespace dnnmg

extern "C" int32_t dnnmg_ideal_update(int32_t n_nodes, const float* x_tilde, const double* v_ref,
                                      const uint8_t* dof_mask, float* x_corr, dnnmg_stream_t s) {
  using namespace dnnmg;
  DNNMG_REQUIRE(n_nodes >= 0 && (n_nodes == 0 || (x_tilde && v_ref && x_corr)), DNNMG_ERR_ARG,
                "ideal_update: null argument");
  if (n_nodes == 0) return DNNMG_OK;
  ideal_update_kernel<<<grid_for(n_nodes, 256), 256, 0, as_stream(s)>>>(
      n_nodes, reinterpret_cast<const float4*>(x_tilde), v_ref, dof_mask,
      reinterpret_cast<float4*>(x_corr));
  DNNMG_CHECK_LAUNCH("ideal_update_kernel");
  return DNNMG_OK;
}
