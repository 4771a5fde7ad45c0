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
#include <cstdlib>

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

// v3: one warp per parent cell C, separable.  The 27 coarse values of C are staged in
// shared memory (prefetched one cell ahead), interpolated to the 5 x 5 x 5 lattice of the
// refined cell in three 1-D stages (x: 45 values and y: 75 in shared memory, z only at the
// owned nodes; an odd lattice position takes the 3-tap quarter-point stencil, an even one
// copies), writing the fine nodes whose first-appearance parent is C (owner list, CSR by C).
constexpr int kProlongWarps = 8;

__device__ __forceinline__ float4 lerp3(int p, const float4& a, const float4& b, const float4& c) {
  // p = 1: (3/8, 3/4, -1/8); p = 3: (-1/8, 3/4, 3/8) -- dyadic, as the 1-D Q2 basis at 1/4, 3/4
  const float w0 = p == 1 ? 0.375f : -0.125f, w2 = p == 1 ? -0.125f : 0.375f;
  float4 r;
  r.x = fmaf(w2, c.x, fmaf(0.75f, b.x, w0 * a.x));
  r.y = fmaf(w2, c.y, fmaf(0.75f, b.y, w0 * a.y));
  r.z = fmaf(w2, c.z, fmaf(0.75f, b.z, w0 * a.z));
  r.w = fmaf(w2, c.w, fmaf(0.75f, b.w, w0 * a.w));
  return r;
}

__global__ void __launch_bounds__(32 * kProlongWarps) prolongate_owner_kernel(
    int n_coarse_cells, const int32_t* __restrict__ ctab, const int32_t* __restrict__ owner_ptr,
    const int32_t* __restrict__ owner_node, const uint8_t* __restrict__ owner_code,
    const float4* __restrict__ xc, float4* __restrict__ xf, const uint8_t* __restrict__ bc_code,
    const float* __restrict__ bc_values, const uint8_t* __restrict__ bc_owner) {
  __shared__ float4 sm[kProlongWarps][27 + 45 + 75];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* cv = sm[w];        // [iz][iy][ix]
  float4* X1 = cv + 27;      // [iz][iy][px]
  float4* X2 = X1 + 45;      // [iz][py][px]
  const int stride = gridDim.x * kProlongWarps;
  int C = blockIdx.x * kProlongWarps + w;
  constexpr int kMaxOwned = 96;  // owned fine nodes per parent cell: <= 64 + faces (checked on host)
  float4 nxt = make_float4(0.f, 0.f, 0.f, 0.f);
  int s_nxt = 0, e_nxt = 0;
  if (C < n_coarse_cells) {
    if (lane < 27) nxt = __ldg(xc + __ldg(ctab + (int64_t)C * 27 + lane));
    s_nxt = __ldg(owner_ptr + C);
    e_nxt = __ldg(owner_ptr + C + 1);
  }
  for (; C < n_coarse_cells; C += stride) {
    if (lane < 27) cv[lane] = nxt;
    const int s = s_nxt, e = e_nxt;
    // this cell's owned nodes, their lattice codes and Dirichlet codes: loads in flight
    // under the interpolation stages
    int nn[kMaxOwned / 32], cc[kMaxOwned / 32], bb[kMaxOwned / 32];
#pragma unroll
    for (int k = 0; k < kMaxOwned / 32; ++k) {
      const int i = s + lane + 32 * k;
      nn[k] = i < e ? __ldg(owner_node + i) : -1;
      cc[k] = i < e ? __ldg(owner_code + i) : 0;
    }
    // Dirichlet codes: in owner order (coalesced, with the owner-list loads) when given, else
    // gathered per owned node (a dependent load)
#pragma unroll
    for (int k = 0; k < kMaxOwned / 32; ++k) {
      const int i = s + lane + 32 * k;
      bb[k] = bc_owner ? (i < e ? __ldg(bc_owner + i) : 0)
                       : ((bc_code && nn[k] >= 0) ? bc_code[nn[k]] : 0);
    }
    if (C + stride < n_coarse_cells) {
      if (lane < 27) nxt = __ldg(xc + __ldg(ctab + (int64_t)(C + stride) * 27 + lane));
      s_nxt = __ldg(owner_ptr + C + stride);
      e_nxt = __ldg(owner_ptr + C + stride + 1);
    }
    __syncwarp();
    // x stage: 45 = 9 lines x 5 positions
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int l = lane + 32 * r;
      if (l < 45) {
        const int line = l / 5, px = l - 5 * line;
        const float4* c = cv + 3 * line;
        X1[l] = (px & 1) ? lerp3(px, c[0], c[1], c[2]) : c[px >> 1];
      }
    }
    __syncwarp();
    // y stage: 75 = 3 iz x 5 py x 5 px
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int l = lane + 32 * r;
      if (l < 75) {
        const int iz = l / 25, py = (l / 5) % 5, px = l % 5;
        const float4* c = X1 + 15 * iz + px;  // [iy] stride 5
        X2[l] = (py & 1) ? lerp3(py, c[0], c[5], c[10]) : c[5 * (py >> 1)];
      }
    }
    __syncwarp();
    // z stage: only at the owned nodes (about half of the 5 x 5 x 5 lattice), from X2
#pragma unroll
    for (int k = 0; k < kMaxOwned / 32; ++k) {
      const int n = nn[k];
      if (n >= 0) {
        const int oa = cc[k];
        const int o = oa / 27, a = oa - 27 * o;
        const int px = 2 * (o & 1) + a % 3;
        const int py = 2 * ((o >> 1) & 1) + (a / 3) % 3;
        const int pz = 2 * (o >> 2) + a / 9;
        const float4* c = X2 + 5 * py + px;   // [iz] stride 25
        float4 acc = (pz & 1) ? lerp3(pz, c[0], c[25], c[50]) : c[25 * (pz >> 1)];
        if (bb[k] == 1) {
          acc.y = acc.z = acc.w = 0.f;
        } else if (bb[k] == 2) {
          acc.y = bc_values[3 * (int64_t)n];
          acc.z = bc_values[3 * (int64_t)n + 1];
          acc.w = bc_values[3 * (int64_t)n + 2];
        }
        xf[n] = acc;
      }
    }
    for (int i = s + kMaxOwned + lane; i < e; i += 32) {  // (never taken for box meshes)
      const int n = __ldg(owner_node + i);
      const int oa = __ldg(owner_code + i);
      const int o = oa / 27, a = oa - 27 * o;
      const int px = 2 * (o & 1) + a % 3;
      const int py = 2 * ((o >> 1) & 1) + (a / 3) % 3;
      const int pz = 2 * (o >> 2) + a / 9;
      const float4* c = X2 + 5 * py + px;
      float4 acc = (pz & 1) ? lerp3(pz, c[0], c[25], c[50]) : c[25 * (pz >> 1)];
      if (bc_code) {
        const uint8_t code = bc_owner ? __ldg(bc_owner + i) : bc_code[n];
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

// v4: lattice form.  One warp per parent cell C; every interpolation stage is a set of whole
// 1-D lines held in registers by one lane each (x: 9 lines, y: 15, z: the 25 columns of the
// 5 x 5 x 5 lattice of the refined cell), so a line costs 3 shared loads and 2 three-tap
// interpolations with compile-time weights, the lanes' roles are the same for every cell, and
// a stage stores only its new (odd-position) values: the next stage reads an even position
// from the array it came from through a per-lane base pointer.  The column lanes write their
// five results straight to global memory: lat[C][25 pz + 5 py + px] is the fine node at that
// lattice position when C is its first-appearance parent, else -1; with PACKED the node's
// Dirichlet code sits in bits 29-30 (dnnmg_dirichlet_t.lat_node_bc).  K1 is bound by the L1
// data pipe (ncu: 80-90 % l1tex, issue 45-63 %): v3 (owner lists, per-node index decoding, all
// positions stored by every stage) took 54 us at config 3, staging the finished lattice in
// shared memory for an owner-ordered (coalesced) write-out 52 us, this form 45 us and less.
__device__ __forceinline__ float4 lerp_lo(const float4& a, const float4& b, const float4& c) {
  float4 r;  // quarter point 1/4: (3/8, 3/4, -1/8), same operation order as lerp3
  r.x = fmaf(-0.125f, c.x, fmaf(0.75f, b.x, 0.375f * a.x));
  r.y = fmaf(-0.125f, c.y, fmaf(0.75f, b.y, 0.375f * a.y));
  r.z = fmaf(-0.125f, c.z, fmaf(0.75f, b.z, 0.375f * a.z));
  r.w = fmaf(-0.125f, c.w, fmaf(0.75f, b.w, 0.375f * a.w));
  return r;
}
__device__ __forceinline__ float4 lerp_hi(const float4& a, const float4& b, const float4& c) {
  float4 r;  // 3/4: (-1/8, 3/4, 3/8)
  r.x = fmaf(0.375f, c.x, fmaf(0.75f, b.x, -0.125f * a.x));
  r.y = fmaf(0.375f, c.y, fmaf(0.75f, b.y, -0.125f * a.y));
  r.z = fmaf(0.375f, c.z, fmaf(0.75f, b.z, -0.125f * a.z));
  r.w = fmaf(0.375f, c.w, fmaf(0.75f, b.w, -0.125f * a.w));
  return r;
}

template <bool PACKED>
__global__ void __launch_bounds__(32 * kProlongWarps) prolongate_lattice_kernel(
    int n_coarse_cells, const int32_t* __restrict__ ctab, const int32_t* __restrict__ lat,
    const float4* __restrict__ xc, float4* __restrict__ xf, const uint8_t* __restrict__ bc_code,
    const float* __restrict__ bc_values) {
  // cv[iz][iy][ix] 27 | X1[iz][iy][k] 18 (px = 2k+1) | X2[iz][k][px] 30 (py = 2k+1)
  __shared__ float4 sm[kProlongWarps][27 + 18 + 30];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* cv = sm[w];
  float4* X1 = cv + 27;
  float4* X2 = X1 + 18;
  // x line (iz, iy) = lane < 9
  const float4* xs = cv + 3 * lane;
  float4* xd = X1 + 2 * lane;
  // y line (iz, px) = lane < 15: even px reads cv (stride 3), odd px reads X1 (stride 2)
  const int y_iz = lane / 5, y_px = lane % 5;
  const float4* ys = (y_px & 1) ? X1 + 6 * y_iz + (y_px >> 1) : cv + 9 * y_iz + (y_px >> 1);
  const int y_st = (y_px & 1) ? 2 : 3;
  float4* yd = X2 + 10 * y_iz + y_px;  // [k] stride 5
  // z column (py, px) = lane < 25: [iz] from X2 (odd py), X1 (even py, odd px) or cv
  const int z_py = lane / 5, z_px = lane % 5;
  const float4* zs = (z_py & 1)   ? X2 + 5 * (z_py >> 1) + z_px
                     : (z_px & 1) ? X1 + 2 * (z_py >> 1) + (z_px >> 1)
                                  : cv + 3 * (z_py >> 1) + (z_px >> 1);
  const int z_st = (z_py & 1) ? 10 : (z_px & 1) ? 6 : 9;
  const int stride = gridDim.x * kProlongWarps;
  int C = blockIdx.x * kProlongWarps + w;
  float4 nxt = make_float4(0.f, 0.f, 0.f, 0.f);
  int id_nxt[5] = {-1, -1, -1, -1, -1};
  if (C < n_coarse_cells) {
    if (lane < 27) nxt = __ldg(xc + __ldg(ctab + (int64_t)C * 27 + lane));
    if (lane < 25) {
#pragma unroll
      for (int pz = 0; pz < 5; ++pz) id_nxt[pz] = __ldg(lat + (int64_t)C * 125 + 25 * pz + lane);
    }
  }
  for (; C < n_coarse_cells; C += stride) {
    if (lane < 27) cv[lane] = nxt;
    int id[5];
#pragma unroll
    for (int pz = 0; pz < 5; ++pz) id[pz] = id_nxt[pz];
    if (C + stride < n_coarse_cells) {  // next cell's loads in flight under this cell's stages
      if (lane < 27) nxt = __ldg(xc + __ldg(ctab + (int64_t)(C + stride) * 27 + lane));
      if (lane < 25) {
#pragma unroll
        for (int pz = 0; pz < 5; ++pz)
          id_nxt[pz] = __ldg(lat + (int64_t)(C + stride) * 125 + 25 * pz + lane);
      }
    }
    __syncwarp();
    if (lane < 9) {
      const float4 a = xs[0], b = xs[1], c = xs[2];
      xd[0] = lerp_lo(a, b, c);
      xd[1] = lerp_hi(a, b, c);
    }
    __syncwarp();
    if (lane < 15) {
      const float4 a = ys[0], b = ys[y_st], c = ys[2 * y_st];
      yd[0] = lerp_lo(a, b, c);
      yd[5] = lerp_hi(a, b, c);
    }
    __syncwarp();
    if (lane < 25) {
      const float4 a = zs[0], b = zs[z_st], c = zs[2 * z_st];
      float4 v[5];
      v[0] = a;
      v[1] = lerp_lo(a, b, c);
      v[2] = b;
      v[3] = lerp_hi(a, b, c);
      v[4] = c;
#pragma unroll
      for (int pz = 0; pz < 5; ++pz) {
        if (id[pz] >= 0) {
          const int n = PACKED ? (id[pz] & 0x1fffffff) : id[pz];
          const int code = PACKED ? (id[pz] >> 29) : (bc_code ? (int)bc_code[n] : 0);
          float4 acc = v[pz];
          if (code == 1) {
            acc.y = acc.z = acc.w = 0.f;
          } else if (code == 2) {
            acc.y = bc_values[3 * (int64_t)n];
            acc.z = bc_values[3 * (int64_t)n + 1];
            acc.w = bc_values[3 * (int64_t)n + 2];
          }
          xf[n] = acc;
        }
      }
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
  const uint8_t* owner_code = nullptr;
  const float* vals = nullptr;
  if (bc) {
    DNNMG_REQUIRE(bc->n_nodes == P->n_fine_nodes, DNNMG_ERR_ARG,
                  "prolongate: Dirichlet data length %d does not match the fine level (%d nodes)",
                  bc->n_nodes, P->n_fine_nodes);
    code = bc->bc_code;
    vals = bc->bc_values;
    owner_code = bc->bc_code_owner;
  }
  if (P->n_fine_nodes == 0) return DNNMG_OK;
  static const bool no_lattice = getenv("DNNMG_K1_OWNER") != nullptr;
  if (P->lat_node && !no_lattice) {
    const int blocks = grid_for((P->n_coarse_cells + kProlongWarps - 1) / kProlongWarps, 1, 4);
    const float4* xc = reinterpret_cast<const float4*>(x_coarse);
    float4* xf = reinterpret_cast<float4*>(x_fine);
    if (bc && bc->lat_node_bc)
      prolongate_lattice_kernel<true><<<blocks, 32 * kProlongWarps, 0, s>>>(
          P->n_coarse_cells, P->coarse_cell_nodes, bc->lat_node_bc, xc, xf, nullptr, vals);
    else
      prolongate_lattice_kernel<false><<<blocks, 32 * kProlongWarps, 0, s>>>(
          P->n_coarse_cells, P->coarse_cell_nodes, P->lat_node, xc, xf, code, vals);
    DNNMG_CHECK_LAUNCH("prolongate_lattice_kernel");
    return DNNMG_OK;
  }
  if (P->owner_ptr && P->owner_node && P->owner_code) {
    const int blocks = grid_for((P->n_coarse_cells + kProlongWarps - 1) / kProlongWarps, 1, 4);
    prolongate_owner_kernel<<<blocks, 32 * kProlongWarps, 0, s>>>(
        P->n_coarse_cells, P->coarse_cell_nodes, P->owner_ptr, P->owner_node, P->owner_code,
        reinterpret_cast<const float4*>(x_coarse), reinterpret_cast<float4*>(x_fine), code, vals,
        owner_code);
    DNNMG_CHECK_LAUNCH("prolongate_owner_kernel");
    return DNNMG_OK;
  }
  prolongate_kernel<<<grid_for(P->n_fine_nodes, 256), 256, 0, s>>>(
      P->n_fine_nodes, P->coarse_cell_nodes, P->fine_src,
      reinterpret_cast<const float4*>(x_coarse), reinterpret_cast<float4*>(x_fine), code, vals);
  DNNMG_CHECK_LAUNCH("prolongate_kernel");
  return DNNMG_OK;
}

// K6: b_coarse[m] = sum_{i in row m, ascending fine node} w_i * b_fine[fine_i] (P^T b)
__global__ void __launch_bounds__(256) restrict_kernel(int n_coarse, const int32_t* __restrict__ ptr,
                                                       const int32_t* __restrict__ fine,
                                                       const float* __restrict__ w,
                                                       const float4* __restrict__ bf,
                                                       float4* __restrict__ bc) {
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < n_coarse; m += gridDim.x * blockDim.x) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const int s = __ldg(ptr + m), e = __ldg(ptr + m + 1);
    for (int i = s; i < e; ++i) {
      const float wi = __ldg(w + i);
      const float4 v = __ldg(bf + __ldg(fine + i));
      acc.x = fmaf(wi, v.x, acc.x);
      acc.y = fmaf(wi, v.y, acc.y);
      acc.z = fmaf(wi, v.z, acc.z);
      acc.w = fmaf(wi, v.w, acc.w);
    }
    bc[m] = acc;
  }
}

// K6 owner-computes form: one warp per coarse (parent) cell scatters the b values of its
// owned fine nodes onto the 5 x 5 x 5 lattice of the refined cell and applies the transpose
// of the separable prolongation stencil (z: 125 -> 75, y: 75 -> 45, x: 45 -> 27), giving the
// cell's 27 partial sums of P^T b; a node sum over the coarse node -> (cell, a) CSR
// (ascending cell) completes them.
__device__ __forceinline__ float4 tlerp(const float4& a0, const float4& a1, const float4& a2,
                                        const float4& a3, const float4& a4, int i) {
  // sum_p phi_i(p/4) a_p: p even copies the node, p odd the quarter-point weights
  float4 r;
  if (i == 0) {
    r.x = fmaf(-0.125f, a3.x, fmaf(0.375f, a1.x, a0.x));
    r.y = fmaf(-0.125f, a3.y, fmaf(0.375f, a1.y, a0.y));
    r.z = fmaf(-0.125f, a3.z, fmaf(0.375f, a1.z, a0.z));
    r.w = fmaf(-0.125f, a3.w, fmaf(0.375f, a1.w, a0.w));
  } else if (i == 1) {
    r.x = fmaf(0.75f, a3.x, fmaf(0.75f, a1.x, a2.x));
    r.y = fmaf(0.75f, a3.y, fmaf(0.75f, a1.y, a2.y));
    r.z = fmaf(0.75f, a3.z, fmaf(0.75f, a1.z, a2.z));
    r.w = fmaf(0.75f, a3.w, fmaf(0.75f, a1.w, a2.w));
  } else {
    r.x = fmaf(0.375f, a3.x, fmaf(-0.125f, a1.x, a4.x));
    r.y = fmaf(0.375f, a3.y, fmaf(-0.125f, a1.y, a4.y));
    r.z = fmaf(0.375f, a3.z, fmaf(-0.125f, a1.z, a4.z));
    r.w = fmaf(0.375f, a3.w, fmaf(-0.125f, a1.w, a4.w));
  }
  return r;
}

__global__ void __launch_bounds__(32 * kProlongWarps) restrict_owner_kernel(
    int n_cells, const int32_t* __restrict__ owner_ptr, const int32_t* __restrict__ owner_node,
    const uint8_t* __restrict__ owner_code, const float4* __restrict__ bf,
    float4* __restrict__ scratch) {
  __shared__ float4 sm[kProlongWarps][125 + 75 + 45];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4* X3 = sm[w];        // [pz][py][px]
  float4* X2 = X3 + 125;     // [iz][py][px]
  float4* X1 = X2 + 75;      // [iz][iy][px]
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int C = blockIdx.x * kProlongWarps + w; C < n_cells; C += gridDim.x * kProlongWarps) {
    for (int l = lane; l < 125; l += 32) X3[l] = zero;
    __syncwarp();
    const int s = __ldg(owner_ptr + C), e = __ldg(owner_ptr + C + 1);
    for (int i = s + lane; i < e; i += 32) {
      const int oa = __ldg(owner_code + i);
      const int o = oa / 27, a = oa - 27 * o;
      const int px = 2 * (o & 1) + a % 3;
      const int py = 2 * ((o >> 1) & 1) + (a / 3) % 3;
      const int pz = 2 * (o >> 2) + a / 9;
      X3[25 * pz + 5 * py + px] = __ldg(bf + __ldg(owner_node + i));
    }
    __syncwarp();
    for (int l = lane; l < 75; l += 32) {          // z: [iz][py][px]
      const int iz = l / 25, yx = l % 25;
      const float4* c = X3 + yx;
      X2[l] = tlerp(c[0], c[25], c[50], c[75], c[100], iz);
    }
    __syncwarp();
    for (int l = lane; l < 45; l += 32) {          // y: [iz][iy][px]
      const int iz = l / 15, iy = (l / 5) % 3, px = l % 5;
      const float4* c = X2 + 25 * iz + px;
      X1[l] = tlerp(c[0], c[5], c[10], c[15], c[20], iy);
    }
    __syncwarp();
    if (lane < 27) {                               // x: [iz][iy][ix]
      const int line = lane / 3, ix = lane % 3;
      const float4* c = X1 + 5 * line;
      scratch[(int64_t)C * 27 + lane] = tlerp(c[0], c[1], c[2], c[3], c[4], ix);
    }
    __syncwarp();
  }
}

int32_t launch_node_sum(int n_nodes, const int32_t* ptr, const int32_t* idx, const float* elem,
                        float* out, cudaStream_t s);

int32_t launch_restrict(const dnnmg_restrict_t* R, const float* bf, float* bc, cudaStream_t s) {
  DNNMG_REQUIRE(R && bf && bc, DNNMG_ERR_ARG, "restrict: null argument");
  DNNMG_REQUIRE(((uintptr_t)bf & 15) == 0 && ((uintptr_t)bc & 15) == 0, DNNMG_ERR_ARG,
                "restrict: vectors must be 16-byte aligned");
  if (R->n_coarse_nodes == 0) return DNNMG_OK;
  if (R->owner_ptr && R->owner_node && R->owner_code && R->node_cell_ptr && R->node_cell_idx &&
      R->cell_scratch && R->n_coarse_cells > 0) {
    const int blocks = grid_for((R->n_coarse_cells + kProlongWarps - 1) / kProlongWarps, 1, 4);
    restrict_owner_kernel<<<blocks, 32 * kProlongWarps, 0, s>>>(
        R->n_coarse_cells, R->owner_ptr, R->owner_node, R->owner_code,
        reinterpret_cast<const float4*>(bf), reinterpret_cast<float4*>(R->cell_scratch));
    DNNMG_CHECK_LAUNCH("restrict_owner_kernel");
    return launch_node_sum(R->n_coarse_nodes, R->node_cell_ptr, R->node_cell_idx, R->cell_scratch,
                           bc, s);
  }
  DNNMG_REQUIRE(R->ptr && R->fine && R->w, DNNMG_ERR_ARG, "restrict: null table");
  restrict_kernel<<<grid_for(R->n_coarse_nodes, 256), 256, 0, s>>>(
      R->n_coarse_nodes, R->ptr, R->fine, R->w, reinterpret_cast<const float4*>(bf),
      reinterpret_cast<float4*>(bc));
  DNNMG_CHECK_LAUNCH("restrict_kernel");
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
