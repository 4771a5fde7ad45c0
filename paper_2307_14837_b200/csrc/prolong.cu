// K1: exact Q2 embedding level l -> l+1 with fused Dirichlet re-imposition.
//
// Reference: space.prolongation_matrix / full_prolongation / prolongate
// (space.py:117-185) and apply_dirichlet (space.py:245-255).  The reference
// builds a scipy CSR P (<= 27 nnz per row) and applies kron(P, I4).  Here the
// row of fine node n is never materialised: it is the tensor product of three
// 1-D Q2 stencils at quarter positions of the parent cell, decoded from
// fine_src[n] = C*216 + o*27 + a.  Per axis the child-local lattice position
// p = 2*o_k + a_k in {0..4} hits a coarse node (p even, weight 1) or a quarter
// point (p odd, weights phi(p/4) = {3/8, 3/4, -1/8} or mirrored).  All weights
// are dyadic, so they are exact in fp32.  Each node is one float4 (p, vx, vy, vz).
#include "common.cuh"

namespace dnnmg {

__device__ __forceinline__ int stencil_1d(int p, int* idx, float* w) {
  if ((p & 1) == 0) {
    idx[0] = p >> 1;
    w[0] = 1.0f;
    return 1;
  }
  idx[0] = 0; idx[1] = 1; idx[2] = 2;
  if (p == 1) { w[0] = 0.375f; w[1] = 0.75f; w[2] = -0.125f; }
  else        { w[0] = -0.125f; w[1] = 0.75f; w[2] = 0.375f; }
  return 3;
}

__global__ void __launch_bounds__(256) prolongate_kernel(
    int n_fine, const int32_t* __restrict__ ctab, const int32_t* __restrict__ src,
    const float4* __restrict__ xc, float4* __restrict__ xf,
    const uint8_t* __restrict__ bc_code, const float* __restrict__ bc_values) {
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < n_fine; n += gridDim.x * blockDim.x) {
    const int s = __ldg(src + n);
    const int C = s / 216;
    const int oa = s - C * 216;
    const int o = oa / 27;
    const int a = oa - o * 27;
    const int px = 2 * (o & 1) + a % 3;
    const int py = 2 * ((o >> 1) & 1) + (a / 3) % 3;
    const int pz = 2 * (o >> 2) + a / 9;
    int ix[3], iy[3], iz[3];
    float wx[3], wy[3], wz[3];
    const int nx = stencil_1d(px, ix, wx);
    const int ny = stencil_1d(py, iy, wy);
    const int nz = stencil_1d(pz, iz, wz);
    const int32_t* row = ctab + (int64_t)C * 27;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int kz = 0; kz < nz; ++kz) {
      for (int ky = 0; ky < ny; ++ky) {
        const float wyz = wy[ky] * wz[kz];
        for (int kx = 0; kx < nx; ++kx) {
          const float w = wx[kx] * wyz;  // exact: product of dyadic weights
          const float4 v = __ldg(xc + __ldg(row + ix[kx] + 3 * iy[ky] + 9 * iz[kz]));
          acc.x = fmaf(w, v.x, acc.x);
          acc.y = fmaf(w, v.y, acc.y);
          acc.z = fmaf(w, v.z, acc.z);
          acc.w = fmaf(w, v.w, acc.w);
        }
      }
    }
    if (bc_code) {
      const uint8_t code = bc_code[n];
      if (code == 1) {
        acc.y = acc.z = acc.w = 0.f;
      } else if (code == 2) {
        acc.y = bc_values[3 * (int64_t)n];
        acc.z = bc_values[3 * (int64_t)n + 1];
        acc.w = bc_values[3 * (int64_t)n + 2];
      }
    }
    xf[n] = acc;
  }
}

__global__ void __launch_bounds__(256) dirichlet_kernel(int n, const uint8_t* __restrict__ code,
                                                        const float* __restrict__ vals,
                                                        float4* __restrict__ x) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint8_t c = code[i];
    if (c == 0) continue;
    float4 v = x[i];
    if (c == 1) {
      v.y = v.z = v.w = 0.f;
    } else {
      v.y = vals[3 * (int64_t)i];
      v.z = vals[3 * (int64_t)i + 1];
      v.w = vals[3 * (int64_t)i + 2];
    }
    x[i] = v;
  }
}

// v2: one warp per parent cell C.  The fine nodes whose first-appearance parent is C
// (owner list, CSR by C) are computed from C's 27 coarse values staged in shared
// memory once, instead of every fine node re-gathering its coarse row.
constexpr int kProlongWarps = 8;

__global__ void __launch_bounds__(32 * kProlongWarps) prolongate_owner_kernel(
    int n_coarse_cells, const int32_t* __restrict__ ctab, const int32_t* __restrict__ owner_ptr,
    const int32_t* __restrict__ owner_node, const uint8_t* __restrict__ owner_code,
    const float4* __restrict__ xc, float4* __restrict__ xf, const uint8_t* __restrict__ bc_code,
    const float* __restrict__ bc_values) {
  __shared__ float4 cv[kProlongWarps][27];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int C = blockIdx.x * kProlongWarps + w; C < n_coarse_cells; C += gridDim.x * kProlongWarps) {
    if (lane < 27) cv[w][lane] = __ldg(xc + __ldg(ctab + (int64_t)C * 27 + lane));
    __syncwarp();
    const int s = __ldg(owner_ptr + C), e = __ldg(owner_ptr + C + 1);
    for (int i = s + lane; i < e; i += 32) {
      const int n = __ldg(owner_node + i);
      const int oa = __ldg(owner_code + i);
      const int o = oa / 27, a = oa - 27 * o;
      const int px = 2 * (o & 1) + a % 3;
      const int py = 2 * ((o >> 1) & 1) + (a / 3) % 3;
      const int pz = 2 * (o >> 2) + a / 9;
      int ix[3], iy[3], iz[3];
      float wx[3], wy[3], wz[3];
      const int nx = stencil_1d(px, ix, wx);
      const int ny = stencil_1d(py, iy, wy);
      const int nz = stencil_1d(pz, iz, wz);
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int kz = 0; kz < nz; ++kz)
        for (int ky = 0; ky < ny; ++ky) {
          const float wyz = wy[ky] * wz[kz];
          for (int kx = 0; kx < nx; ++kx) {
            const float wgt = wx[kx] * wyz;
            const float4 v = cv[w][ix[kx] + 3 * iy[ky] + 9 * iz[kz]];
            acc.x = fmaf(wgt, v.x, acc.x);
            acc.y = fmaf(wgt, v.y, acc.y);
            acc.z = fmaf(wgt, v.z, acc.z);
            acc.w = fmaf(wgt, v.w, acc.w);
          }
        }
      if (bc_code) {
        const uint8_t code = bc_code[n];
        if (code == 1) {
          acc.y = acc.z = acc.w = 0.f;
        } else if (code == 2) {
          acc.y = bc_values[3 * (int64_t)n];
          acc.z = bc_values[3 * (int64_t)n + 1];
          acc.w = bc_values[3 * (int64_t)n + 2];
        }
      }
      xf[n] = acc;
    }
    __syncwarp();
  }
}

int32_t launch_prolongate(const dnnmg_prolong_t* P, const float* x_coarse, float* x_fine,
                          const dnnmg_dirichlet_t* bc, cudaStream_t s) {
  DNNMG_REQUIRE(P && x_coarse && x_fine, DNNMG_ERR_ARG, "prolongate: null argument");
  DNNMG_REQUIRE(P->coarse_cell_nodes && P->fine_src, DNNMG_ERR_ARG, "prolongate: null table");
  DNNMG_REQUIRE(((uintptr_t)x_coarse & 15) == 0 && ((uintptr_t)x_fine & 15) == 0, DNNMG_ERR_ARG,
                "prolongate: vectors must be 16-byte aligned");
  const uint8_t* code = nullptr;
  const float* vals = nullptr;
  if (bc) {
    DNNMG_REQUIRE(bc->n_nodes == P->n_fine_nodes, DNNMG_ERR_ARG,
                  "prolongate: Dirichlet data length %d does not match the fine level (%d nodes)",
                  bc->n_nodes, P->n_fine_nodes);
    code = bc->bc_code;
    vals = bc->bc_values;
  }
  if (P->n_fine_nodes == 0) return DNNMG_OK;
  if (P->owner_ptr && P->owner_node && P->owner_code) {
    const int blocks = grid_for((P->n_coarse_cells + kProlongWarps - 1) / kProlongWarps, 1, 8);
    prolongate_owner_kernel<<<blocks, 32 * kProlongWarps, 0, s>>>(
        P->n_coarse_cells, P->coarse_cell_nodes, P->owner_ptr, P->owner_node, P->owner_code,
        reinterpret_cast<const float4*>(x_coarse), reinterpret_cast<float4*>(x_fine), code, vals);
    DNNMG_CHECK_LAUNCH("prolongate_owner_kernel");
    return DNNMG_OK;
  }
  prolongate_kernel<<<grid_for(P->n_fine_nodes, 256), 256, 0, s>>>(
      P->n_fine_nodes, P->coarse_cell_nodes, P->fine_src,
      reinterpret_cast<const float4*>(x_coarse), reinterpret_cast<float4*>(x_fine), code, vals);
  DNNMG_CHECK_LAUNCH("prolongate_kernel");
  return DNNMG_OK;
}

int32_t launch_dirichlet(const dnnmg_dirichlet_t* bc, float* x, cudaStream_t s) {
  DNNMG_REQUIRE(bc && x && bc->bc_code, DNNMG_ERR_ARG, "apply_dirichlet: null argument");
  if (bc->n_nodes == 0) return DNNMG_OK;
  dirichlet_kernel<<<grid_for(bc->n_nodes, 256), 256, 0, s>>>(
      bc->n_nodes, bc->bc_code, bc->bc_values, reinterpret_cast<float4*>(x));
  DNNMG_CHECK_LAUNCH("dirichlet_kernel");
  return DNNMG_OK;
}

}  // namespace dnnmg
