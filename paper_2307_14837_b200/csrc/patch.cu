// K3 (patch gather) and K5 (owner-computes valence-averaging scatter + update).
//
// Reference: patch_ops.local_restrict / assemble_network_input (patch_ops.py:23-29,
// 49-53) — a pure index gather x[dof_table] — and global_extend / predict_correction
// (patch_ops.py:32-38, 56-76): np.bincount(dof_table, rows) * mu, pressure slots zero,
// masked dofs zero, then x_corr = x~ + scale*d (driver.py:268).
//
// The scatter is owner-computes: one thread per fine node walks its incident
// (patch, slot) list in ascending patch id — the summation order of bincount —
// and multiplies by mu = 1/valence, the reference's stored reciprocal.  No float
// atomics, so results are bitwise reproducible.
#include "common.cuh"

namespace dnnmg {

// X row: [x(4*npp) | r(4*npp) | geom(n_geo)], one float4 per thread-chunk.
__global__ void __launch_bounds__(256) gather_kernel(int n_patches, int npp, int n_geo,
                                                     const int32_t* __restrict__ table,
                                                     const float4* __restrict__ x,
                                                     const float4* __restrict__ r,
                                                     const float* __restrict__ geom,
                                                     float* __restrict__ X) {
  const int geo4 = n_geo / 4;
  const int chunks = 2 * npp + geo4;
  const int row = 8 * npp + n_geo;
  const int64_t total = (int64_t)n_patches * chunks;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(i / chunks);
    const int ch = (int)(i - (int64_t)p * chunks);
    float4 v;
    if (ch < npp) {
      v = __ldg(x + __ldg(table + (int64_t)p * npp + ch));
    } else if (ch < 2 * npp) {
      v = __ldg(r + __ldg(table + (int64_t)p * npp + ch - npp));
    } else {
      v = __ldg(reinterpret_cast<const float4*>(geom + (int64_t)p * n_geo) + (ch - 2 * npp));
    }
    reinterpret_cast<float4*>(X + (int64_t)p * row)[ch] = v;
  }
}

__global__ void __launch_bounds__(256) restrict_kernel(int n_patches, int npp,
                                                       const int32_t* __restrict__ table,
                                                       const float4* __restrict__ x,
                                                       float4* __restrict__ rows) {
  const int64_t total = (int64_t)n_patches * npp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    rows[i] = __ldg(x + __ldg(table + i));
}

// out = mu * bincount(dof_table, rows) for all 4 components
__global__ void __launch_bounds__(256) extend_kernel(int n_nodes, const int32_t* __restrict__ ptr,
                                                     const int32_t* __restrict__ idx,
                                                     const float4* __restrict__ rows,
                                                     float4* __restrict__ out) {
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < n_nodes; n += gridDim.x * blockDim.x) {
    const int s = __ldg(ptr + n), e = __ldg(ptr + n + 1);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = s; i < e; ++i) {
      const float4 v = __ldg(rows + __ldg(idx + i));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    const float mu = e > s ? 1.0f / (float)(e - s) : 0.f;
    out[n] = make_float4(mu * acc.x, mu * acc.y, mu * acc.z, mu * acc.w);
  }
}

// d = mu * sum over incident (patch, slot) of Y[patch][3*slot .. 3*slot+2]; pressure 0;
// d[mask] = 0; x_corr = x~ + scale*d
// Up to kBatch incident entries of a node are loaded before any is summed (all Y loads of a
// node in flight at once); the sum stays in ascending entry order.  NPP > 0 makes the
// (patch, slot) split a constant division.
constexpr int kBatch = 8;

template <int NPP>
__global__ void __launch_bounds__(256) scatter_update_kernel(
    int n_nodes, int npp_rt, const int32_t* __restrict__ ptr,
    const int32_t* __restrict__ idx, const float* __restrict__ Y, const uint8_t* __restrict__ mask,
    const float4* __restrict__ xt, float scale, float4* __restrict__ d, float4* __restrict__ xc,
    const int32_t* __restrict__ order, const int32_t* __restrict__ vptr,
    const int32_t* __restrict__ vidx) {
  const int npp = NPP > 0 ? NPP : npp_rt;
  const int n_out = 3 * npp;
  if (vptr) idx = vidx;   // rows in visiting order: the bounds load next to the node id
  for (int pos = blockIdx.x * blockDim.x + threadIdx.x; pos < n_nodes;
       pos += gridDim.x * blockDim.x) {
    const int n = order ? __ldg(order + pos) : pos;
    const int s = vptr ? __ldg(vptr + pos) : __ldg(ptr + n);
    const int e = vptr ? __ldg(vptr + pos + 1) : __ldg(ptr + n + 1);
    // the node's own loads first: in flight with the entry loads
    const float4 x = xc ? __ldg(xt + n) : make_float4(0.f, 0.f, 0.f, 0.f);
    const uint8_t m = mask ? __ldg(mask + n) : 0;
    int ent[kBatch];
#pragma unroll
    for (int k = 0; k < kBatch; ++k) ent[k] = s + k < e ? __ldg(idx + s + k) : -1;
    float y0[kBatch], y1[kBatch], y2[kBatch];
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
      y0[k] = y1[k] = y2[k] = 0.f;
      if (ent[k] >= 0) {
        const int p = ent[k] / npp;
        const float* y = Y + (int64_t)p * n_out + 3 * (ent[k] - p * npp);
        y0[k] = __ldg(y);
        y1[k] = __ldg(y + 1);
        y2[k] = __ldg(y + 2);
      }
    }
    float a0 = 0.f, a1 = 0.f, a2 = 0.f;
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
      if (ent[k] >= 0) {
        a0 += y0[k];
        a1 += y1[k];
        a2 += y2[k];
      }
    }
    for (int i = s + kBatch; i < e; ++i) {
      const int ps = __ldg(idx + i);
      const int p = ps / npp;
      const float* y = Y + (int64_t)p * n_out + 3 * (ps - p * npp);
      a0 += __ldg(y);
      a1 += __ldg(y + 1);
      a2 += __ldg(y + 2);
    }
    const float mu = e > s ? 1.0f / (float)(e - s) : 0.f;
    float4 dv = make_float4(0.f, mu * a0, mu * a1, mu * a2);
    if (m & 2) dv.y = 0.f;
    if (m & 4) dv.z = 0.f;
    if (m & 8) dv.w = 0.f;
    if (d) d[n] = dv;
    if (xc) {
      xc[n] = make_float4(x.x, fmaf(scale, dv.y, x.y), fmaf(scale, dv.z, x.z), fmaf(scale, dv.w, x.w));
    }
  }
}

static int32_t check_ps(const dnnmg_patchset_t* ps, const char* who) {
  DNNMG_REQUIRE(ps && ps->node_table && ps->node_patch_ptr && ps->node_patch_idx, DNNMG_ERR_ARG,
                "%s: incomplete patch tables", who);
  DNNMG_REQUIRE(ps->nodes_per_patch > 0, DNNMG_ERR_ARG, "%s: nodes_per_patch must be > 0", who);
  return DNNMG_OK;
}

int32_t launch_gather(const dnnmg_patchset_t* ps, const float* x, const float* r, float* X,
                      cudaStream_t s) {
  int32_t st = check_ps(ps, "gather");
  if (st) return st;
  DNNMG_REQUIRE(x && r && X && ps->geom, DNNMG_ERR_ARG, "gather: null argument");
  DNNMG_REQUIRE(ps->n_geo % 4 == 0, DNNMG_ERR_UNSUPPORTED, "gather: n_geo must be a multiple of 4");
  DNNMG_REQUIRE(((uintptr_t)X & 15) == 0 && ((uintptr_t)ps->geom & 15) == 0, DNNMG_ERR_ARG,
                "gather: X and geom must be 16-byte aligned");
  const int64_t total = (int64_t)ps->n_patches * (2 * ps->nodes_per_patch + ps->n_geo / 4);
  if (total == 0) return DNNMG_OK;
  gather_kernel<<<grid_for(total, 256), 256, 0, s>>>(
      ps->n_patches, ps->nodes_per_patch, ps->n_geo, ps->node_table,
      reinterpret_cast<const float4*>(x), reinterpret_cast<const float4*>(r), ps->geom, X);
  DNNMG_CHECK_LAUNCH("gather_kernel");
  return DNNMG_OK;
}

int32_t launch_restrict(const dnnmg_patchset_t* ps, const float* x, float* rows, cudaStream_t s) {
  int32_t st = check_ps(ps, "local_restrict");
  if (st) return st;
  DNNMG_REQUIRE(x && rows, DNNMG_ERR_ARG, "local_restrict: null argument");
  const int64_t total = (int64_t)ps->n_patches * ps->nodes_per_patch;
  if (total == 0) return DNNMG_OK;
  restrict_kernel<<<grid_for(total, 256), 256, 0, s>>>(ps->n_patches, ps->nodes_per_patch,
                                                      ps->node_table,
                                                      reinterpret_cast<const float4*>(x),
                                                      reinterpret_cast<float4*>(rows));
  DNNMG_CHECK_LAUNCH("restrict_kernel");
  return DNNMG_OK;
}

int32_t launch_extend(const dnnmg_patchset_t* ps, const float* rows, float* out, cudaStream_t s) {
  int32_t st = check_ps(ps, "global_extend");
  if (st) return st;
  DNNMG_REQUIRE(rows && out, DNNMG_ERR_ARG, "global_extend: null argument");
  if (ps->n_nodes == 0) return DNNMG_OK;
  extend_kernel<<<grid_for(ps->n_nodes, 256), 256, 0, s>>>(
      ps->n_nodes, ps->node_patch_ptr, ps->node_patch_idx, reinterpret_cast<const float4*>(rows),
      reinterpret_cast<float4*>(out));
  DNNMG_CHECK_LAUNCH("extend_kernel");
  return DNNMG_OK;
}

int32_t launch_scatter_update(const dnnmg_patchset_t* ps, const float* Y, const uint8_t* mask,
                              const float* xt, float scale, float* d, float* xc, cudaStream_t s) {
  int32_t st = check_ps(ps, "scatter_update");
  if (st) return st;
  DNNMG_REQUIRE(Y && (d || xc), DNNMG_ERR_ARG, "scatter_update: null argument");
  DNNMG_REQUIRE(!xc || xt, DNNMG_ERR_ARG, "scatter_update: x_corr requested without x_tilde");
  if (ps->n_nodes == 0) return DNNMG_OK;
  auto kern = ps->nodes_per_patch == 27    ? scatter_update_kernel<27>
              : ps->nodes_per_patch == 125 ? scatter_update_kernel<125>
                                           : scatter_update_kernel<0>;
  // one node per thread (no grid cap): 0.098 -> 0.097 ms at config 3
  kern<<<grid_for(ps->n_nodes, 256, 1 << 20), 256, 0, s>>>(
      ps->n_nodes, ps->nodes_per_patch, ps->node_patch_ptr, ps->node_patch_idx, Y, mask,
      reinterpret_cast<const float4*>(xt), scale, reinterpret_cast<float4*>(d),
      reinterpret_cast<float4*>(xc), ps->node_order, ps->node_order ? ps->visit_ptr : nullptr,
      ps->visit_idx);
  DNNMG_CHECK_LAUNCH("scatter_update_kernel");
  return DNNMG_OK;
}

}  // namespace dnnmg
