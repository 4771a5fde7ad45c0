// Slab-interface (halo) kernels of the x-slab domain decomposition.
//
// Each rank owns a contiguous x-range of coarse cells.  Fine nodes on an interface
// plane belong to both neighbouring slabs; two quantities are exchanged per step:
//   (a) the partial operator A_h(x~) at interface nodes, so both sides form the
//       same r = b - (A_left + A_right)  (assembly.py:261-267 summed over all cells)
//   (b) the raw patch sums and patch counts at interface nodes, so both sides form
//       d = (S_left + S_right) / (count_left + count_right)  (patch_ops.py:32-38)
// Sums are always taken left partial first, so both ranks hold bitwise identical
// interface values.
#include "common.cuh"

namespace dnnmg {

// out[i] = a[idx[i]] - (b ? b[idx[i]] : 0)         (float4 rows)
__global__ void halo_gather_kernel(int n, const int32_t* __restrict__ idx,
                                   const float4* __restrict__ a, const float4* __restrict__ b,
                                   float4* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int k = idx[i];
    float4 v = a[k];
    if (b) {
      const float4 w = b[k];
      v.x -= w.x; v.y -= w.y; v.z -= w.z; v.w -= w.w;
    }
    out[i] = v;
  }
}

// r[idx[i]] = b[idx[i]] - (A_left + A_right), then constrained rows -> 0
__global__ void halo_residual_kernel(int n, const int32_t* __restrict__ idx,
                                     const float4* __restrict__ b, const float4* __restrict__ own,
                                     const float4* __restrict__ nb, int own_is_left,
                                     const uint8_t* __restrict__ mask, float4* __restrict__ r) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int k = idx[i];
    const float4 L = own_is_left ? own[i] : nb[i];
    const float4 R = own_is_left ? nb[i] : own[i];
    const float4 bb = b[k];
    float4 v = make_float4(bb.x - (L.x + R.x), bb.y - (L.y + R.y), bb.z - (L.z + R.z),
                           bb.w - (L.w + R.w));
    if (mask) {
      const uint8_t m = mask[k];
      if (m & 1) v.x = 0.f;
      if (m & 2) v.y = 0.f;
      if (m & 4) v.z = 0.f;
      if (m & 8) v.w = 0.f;
    }
    r[k] = v;
  }
}

// out[i] = (count, S_x, S_y, S_z): raw patch sums of the velocity predictions at idx[i]
__global__ void halo_scatter_sums_kernel(int n, const int32_t* __restrict__ idx, int npp, int n_out,
                                         const int32_t* __restrict__ ptr,
                                         const int32_t* __restrict__ pidx,
                                         const float* __restrict__ Y, float4* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int node = idx[i];
    const int s = ptr[node], e = ptr[node + 1];
    float a0 = 0.f, a1 = 0.f, a2 = 0.f;
    for (int j = s; j < e; ++j) {
      const int ps = pidx[j];
      const int p = ps / npp, slot = ps - p * npp;
      const float* y = Y + (int64_t)p * n_out + 3 * slot;
      a0 += y[0];
      a1 += y[1];
      a2 += y[2];
    }
    out[i] = make_float4((float)(e - s), a0, a1, a2);
  }
}

// d = (S_left + S_right) / (count_left + count_right) at interface nodes; mask;
// x_corr = x~ + scale*d
__global__ void halo_scatter_apply_kernel(int n, const int32_t* __restrict__ idx,
                                          const float4* __restrict__ own,
                                          const float4* __restrict__ nb, int own_is_left,
                                          const uint8_t* __restrict__ mask,
                                          const float4* __restrict__ xt, float scale,
                                          float4* __restrict__ d, float4* __restrict__ xc) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int k = idx[i];
    const float4 L = own_is_left ? own[i] : nb[i];
    const float4 R = own_is_left ? nb[i] : own[i];
    const float mu = 1.0f / (L.x + R.x);
    float4 dv = make_float4(0.f, mu * (L.y + R.y), mu * (L.z + R.z), mu * (L.w + R.w));
    if (mask) {
      const uint8_t m = mask[k];
      if (m & 2) dv.y = 0.f;
      if (m & 4) dv.z = 0.f;
      if (m & 8) dv.w = 0.f;
    }
    if (d) d[k] = dv;
    if (xc) {
      const float4 x = xt[k];
      xc[k] = make_float4(x.x, fmaf(scale, dv.y, x.y), fmaf(scale, dv.z, x.z), fmaf(scale, dv.w, x.w));
    }
  }
}

}  // namespace dnnmg

using namespace dnnmg;

extern "C" {

int32_t dnnmg_halo_gather(const int32_t* idx, int32_t n, const float* a, const float* b, float* out,
                          dnnmg_stream_t s) {
  DNNMG_REQUIRE(n >= 0 && (n == 0 || (idx && a && out)), DNNMG_ERR_ARG, "halo_gather: null argument");
  if (n == 0) return DNNMG_OK;
  halo_gather_kernel<<<grid_for(n, 256), 256, 0, as_stream(s)>>>(
      n, idx, reinterpret_cast<const float4*>(a), reinterpret_cast<const float4*>(b),
      reinterpret_cast<float4*>(out));
  DNNMG_CHECK_LAUNCH("halo_gather_kernel");
  return DNNMG_OK;
}

int32_t dnnmg_halo_residual(const int32_t* idx, int32_t n, const float* b, const float* own,
                            const float* nb, int32_t own_is_left, const uint8_t* mask, float* r,
                            dnnmg_stream_t s) {
  DNNMG_REQUIRE(n >= 0 && (n == 0 || (idx && b && own && nb && r)), DNNMG_ERR_ARG,
                "halo_residual: null argument");
  if (n == 0) return DNNMG_OK;
  halo_residual_kernel<<<grid_for(n, 256), 256, 0, as_stream(s)>>>(
      n, idx, reinterpret_cast<const float4*>(b), reinterpret_cast<const float4*>(own),
      reinterpret_cast<const float4*>(nb), own_is_left, mask, reinterpret_cast<float4*>(r));
  DNNMG_CHECK_LAUNCH("halo_residual_kernel");
  return DNNMG_OK;
}

int32_t dnnmg_halo_scatter_sums(const dnnmg_patchset_t* ps, const float* Y, const int32_t* idx,
                                int32_t n, float* out, dnnmg_stream_t s) {
  DNNMG_REQUIRE(ps && ps->node_patch_ptr && ps->node_patch_idx, DNNMG_ERR_ARG,
                "halo_scatter_sums: incomplete patch tables");
  DNNMG_REQUIRE(n >= 0 && (n == 0 || (idx && Y && out)), DNNMG_ERR_ARG,
                "halo_scatter_sums: null argument");
  if (n == 0) return DNNMG_OK;
  halo_scatter_sums_kernel<<<grid_for(n, 256), 256, 0, as_stream(s)>>>(
      n, idx, ps->nodes_per_patch, 3 * ps->nodes_per_patch, ps->node_patch_ptr, ps->node_patch_idx,
      Y, reinterpret_cast<float4*>(out));
  DNNMG_CHECK_LAUNCH("halo_scatter_sums_kernel");
  return DNNMG_OK;
}

int32_t dnnmg_halo_scatter_apply(const int32_t* idx, int32_t n, const float* own, const float* nb,
                                 int32_t own_is_left, const uint8_t* mask, const float* x_tilde,
                                 float scale, float* d, float* x_corr, dnnmg_stream_t s) {
  DNNMG_REQUIRE(n >= 0 && (n == 0 || (idx && own && nb)), DNNMG_ERR_ARG,
                "halo_scatter_apply: null argument");
  DNNMG_REQUIRE(!x_corr || x_tilde, DNNMG_ERR_ARG, "halo_scatter_apply: x_corr needs x_tilde");
  if (n == 0) return DNNMG_OK;
  halo_scatter_apply_kernel<<<grid_for(n, 256), 256, 0, as_stream(s)>>>(
      n, idx, reinterpret_cast<const float4*>(own), reinterpret_cast<const float4*>(nb), own_is_left,
      mask, reinterpret_cast<const float4*>(x_tilde), scale, reinterpret_cast<float4*>(d),
      reinterpret_cast<float4*>(x_corr));
  DNNMG_CHECK_LAUNCH("halo_scatter_apply_kernel");
  return DNNMG_OK;
}

}  // extern "C"

namespace dnnmg {
// out[i] = sum over the incident (cell, local node) of node idx[i], ascending cell id,
// of the element vectors: this rank's partial operator A_h(x~) at interface nodes
__global__ void halo_operator_kernel(int n, const int32_t* __restrict__ idx,
                                     const int32_t* __restrict__ ptr,
                                     const int32_t* __restrict__ cidx,
                                     const float4* __restrict__ elem, float4* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int node = idx[i];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = ptr[node]; j < ptr[node + 1]; ++j) {
      const float4 v = elem[cidx[j]];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    out[i] = acc;
  }
}
}  // namespace dnnmg

extern "C" int32_t dnnmg_halo_operator(const dnnmg_level_t* lv, const float* elem,
                                       const int32_t* idx, int32_t n, float* out,
                                       dnnmg_stream_t s) {
  using namespace dnnmg;
  DNNMG_REQUIRE(lv && lv->node_cell_ptr && lv->node_cell_idx, DNNMG_ERR_ARG,
                "halo_operator: incomplete level tables");
  DNNMG_REQUIRE(n >= 0 && (n == 0 || (idx && elem && out)), DNNMG_ERR_ARG,
                "halo_operator: null argument");
  if (n == 0) return DNNMG_OK;
  halo_operator_kernel<<<grid_for(n, 256), 256, 0, as_stream(s)>>>(
      n, idx, lv->node_cell_ptr, lv->node_cell_idx, reinterpret_cast<const float4*>(elem),
      reinterpret_cast<float4*>(out));
  DNNMG_CHECK_LAUNCH("halo_operator_kernel");
  return DNNMG_OK;
}

namespace dnnmg {
// out[idx[i]] = A_left[i] + A_right[i]   (complete interface rows of an assembled dual vector)
__global__ void halo_sum_kernel(int n, const int32_t* __restrict__ idx, const float4* __restrict__ own,
                                const float4* __restrict__ nb, int own_is_left,
                                float4* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float4 L = own_is_left ? own[i] : nb[i];
    const float4 R = own_is_left ? nb[i] : own[i];
    out[idx[i]] = make_float4(L.x + R.x, L.y + R.y, L.z + R.z, L.w + R.w);
  }
}
}  // namespace dnnmg

extern "C" int32_t dnnmg_halo_sum(const int32_t* idx, int32_t n, const float* own, const float* nb,
                                  int32_t own_is_left, float* out, dnnmg_stream_t s) {
  using namespace dnnmg;
  DNNMG_REQUIRE(n >= 0 && (n == 0 || (idx && own && nb && out)), DNNMG_ERR_ARG,
                "halo_sum: null argument");
  if (n == 0) return DNNMG_OK;
  halo_sum_kernel<<<grid_for(n, 256), 256, 0, as_stream(s)>>>(
      n, idx, reinterpret_cast<const float4*>(own), reinterpret_cast<const float4*>(nb), own_is_left,
      reinterpret_cast<float4*>(out));
  DNNMG_CHECK_LAUNCH("halo_sum_kernel");
  return DNNMG_OK;
}
