// Cell-based Vanka smoother of the coarse-level multigrid.
//
// Reference: msolve.VankaData / vanka_smooth (msolve.py:51-89).  Per cell the dense
// (d+1) 3^d = 108 saddle-point block of the level Jacobian is gathered from the CSR
// values through the assembler's pattern positions (assembly.py:110-126, flat_pos) and
// inverted once (float64, Gauss-Jordan with partial pivoting; a singular block is
// retried with a 1e-12 diagonal shift and flagged, as the reference does).  A sweep is
//
//   r  = b - J x                      (CSR SpMV, one warp per row)
//   dl = inv[c] r[dofs[c]]            (batched 108 x 108 matvec, one CTA per cell)
//   x += damping * weight * bincount(dofs, dl)   (owner-computes per dof, ascending
//                                                  (cell, local dof): bincount's order)
//
// All cells read the sweep-start iterate (Jacobi coupling).  No float atomics.
#include "common.cuh"

namespace dnnmg {

constexpr int kVankaThreads = 256;

// ---- setup: gather + invert (one CTA per cell, block in shared memory) -------------
__global__ void __launch_bounds__(kVankaThreads) vanka_invert_kernel(
    int n_cells, int ndl, const double* __restrict__ data, const int64_t* __restrict__ flat_pos,
    double* __restrict__ inv, int32_t* __restrict__ flags) {
  extern __shared__ double smem_v[];
  double* A = smem_v;                       // [ndl][ndl] row-major, inverted in place
  double* colk = A + ndl * ndl;             // column k before the elimination step
  int* perm = reinterpret_cast<int*>(colk + ndl);  // row swaps of the pivoting
  __shared__ double s_pval[32];
  __shared__ int s_pidx[32];
  __shared__ int s_piv;
  __shared__ int s_fail;
  const int nn = ndl * ndl;
  for (int c = blockIdx.x; c < n_cells; c += gridDim.x) {
    int used = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
      used = attempt;
      const int64_t base = (int64_t)c * nn;
      for (int e = threadIdx.x; e < nn; e += blockDim.x) {
        double v = data[flat_pos[base + e]];
        if (attempt == 1 && (e / ndl) == (e % ndl)) v += 1e-12;
        A[e] = v;
      }
      if (threadIdx.x == 0) s_fail = 0;
      __syncthreads();
      // in-place Gauss-Jordan with row pivoting: after step k, A holds the inverse of the
      // processed part; row swaps are undone as column swaps at the end
      for (int k = 0; k < ndl; ++k) {
        // pivot search over rows k..ndl-1 of column k (largest magnitude, lowest index)
        double best = -1.0;
        int bi = k;
        for (int i = k + threadIdx.x; i < ndl; i += blockDim.x) {
          const double a = fabs(A[i * ndl + k]);
          if (a > best) { best = a; bi = i; }
        }
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_down_sync(0xffffffffu, best, o);
          const int oi = __shfl_down_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (lane == 0) { s_pval[wid] = best; s_pidx[wid] = bi; }
        __syncthreads();
        if (threadIdx.x == 0) {
          double b = s_pval[0];
          int i = s_pidx[0];
          for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (s_pval[w] > b || (s_pval[w] == b && s_pidx[w] < i)) { b = s_pval[w]; i = s_pidx[w]; }
          s_piv = i;
          perm[k] = i;
          if (!(b > 0.0)) s_fail = 1;
        }
        __syncthreads();
        if (s_fail) break;
        const int p = s_piv;
        if (p != k)
          for (int j = threadIdx.x; j < ndl; j += blockDim.x) {
            const double t = A[k * ndl + j];
            A[k * ndl + j] = A[p * ndl + j];
            A[p * ndl + j] = t;
          }
        __syncthreads();
        const double piv = A[k * ndl + k];
        const double ip = 1.0 / piv;
        __syncthreads();
        for (int j = threadIdx.x; j < ndl; j += blockDim.x) {
          A[k * ndl + j] = (j == k) ? ip : A[k * ndl + j] * ip;
          colk[j] = A[j * ndl + k];
        }
        __syncthreads();
        // eliminate column k from every other row: A[i][j] -= A[i][k] * A[k][j], A[i][k] = -A[i][k]/piv
        for (int e = threadIdx.x; e < nn; e += blockDim.x) {
          const int i = e / ndl, j = e - i * ndl;
          if (i == k) continue;
          const double f = colk[i];
          if (j == k) A[e] = -f * ip;
          else A[e] = fma(-f, A[k * ndl + j], A[e]);
        }
        __syncthreads();
      }
      if (!s_fail) break;
      __syncthreads();
    }
    // 0: regular, 1: regularised by the 1e-12 shift (the reference's flagged cells), 2: singular
    if (threadIdx.x == 0 && flags) flags[c] = s_fail ? 2 : used;
    __syncthreads();
    // undo the row swaps as column swaps, last swap first
    for (int k = ndl - 1; k >= 0; --k) {
      const int p = perm[k];
      if (p != k)
        for (int i = threadIdx.x; i < ndl; i += blockDim.x) {
          const double t = A[i * ndl + k];
          A[i * ndl + k] = A[i * ndl + p];
          A[i * ndl + p] = t;
        }
      __syncthreads();
    }
    // stored transposed (column j of the inverse is contiguous): the apply kernel's
    // thread-per-row loads are then coalesced
    double* out = inv + (int64_t)c * nn;
    for (int e = threadIdx.x; e < nn; e += blockDim.x) {
      const int j = e / ndl, i = e - j * ndl;
      out[e] = A[i * ndl + j];
    }
    __syncthreads();
  }
}

// ---- sweep kernels -----------------------------------------------------------------
// r = b - J x, one warp per row, fixed lane-strided order + butterfly reduction
__global__ void __launch_bounds__(256) csr_residual_kernel(int n, const int32_t* __restrict__ ptr,
                                                           const int32_t* __restrict__ idx,
                                                           const double* __restrict__ val,
                                                           const double* __restrict__ x,
                                                           const double* __restrict__ b,
                                                           double* __restrict__ r) {
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < n; row += warps) {
    double s = 0.0;
    for (int k = ptr[row] + lane; k < ptr[row + 1]; k += 32) s = fma(val[k], x[idx[k]], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) r[row] = b[row] - s;
  }
}

// dl[c] = inv[c] * r[dofs[c]]; one CTA of kApplyThreads per cell, thread i = output row i,
// reading the transposed inverse column by column (coalesced), r[dofs] staged in SMEM
constexpr int kApplyThreads = 128;
__global__ void __launch_bounds__(kApplyThreads) vanka_apply_kernel(
    int n_cells, int ndl, const int32_t* __restrict__ dofs, const double* __restrict__ invT,
    const double* __restrict__ r, double* __restrict__ dl) {
  extern __shared__ double rl[];
  for (int c = blockIdx.x; c < n_cells; c += gridDim.x) {
    for (int i = threadIdx.x; i < ndl; i += blockDim.x) rl[i] = r[dofs[(int64_t)c * ndl + i]];
    __syncthreads();
    const double* M = invT + (int64_t)c * ndl * ndl;
    for (int i = threadIdx.x; i < ndl; i += blockDim.x) {
      double s0 = 0.0, s1 = 0.0;
      int j = 0;
      for (; j + 1 < ndl; j += 2) {
        s0 = fma(__ldg(M + (int64_t)j * ndl + i), rl[j], s0);
        s1 = fma(__ldg(M + (int64_t)(j + 1) * ndl + i), rl[j + 1], s1);
      }
      if (j < ndl) s0 = fma(__ldg(M + (int64_t)j * ndl + i), rl[j], s0);
      dl[(int64_t)c * ndl + i] = s0 + s1;
    }
    __syncthreads();
  }
}

// x[d] += damping * weight[d] * sum over (c, i) with dofs[c][i] == d, ascending (c, i)
__global__ void __launch_bounds__(256) vanka_update_kernel(int n_dofs, const int32_t* __restrict__ ptr,
                                                           const int32_t* __restrict__ idx,
                                                           const double* __restrict__ dl,
                                                           const double* __restrict__ weight,
                                                           double damping, double* __restrict__ x) {
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < n_dofs; d += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = ptr[d]; k < ptr[d + 1]; ++k) s += dl[idx[k]];
    x[d] = x[d] + damping * (weight[d] * s);
  }
}

}  // namespace dnnmg

extern "C" int32_t dnnmg_vanka_setup(int32_t n_cells, int32_t ndl, const double* csr_data,
                                     const int64_t* flat_pos, double* inv, int32_t* flags,
                                     dnnmg_stream_t s) {
  using namespace dnnmg;
  DNNMG_REQUIRE(n_cells >= 0 && ndl > 0 && ndl <= 128, DNNMG_ERR_ARG,
                "vanka_setup: bad block size %d", ndl);
  DNNMG_REQUIRE(n_cells == 0 || (csr_data && flat_pos && inv), DNNMG_ERR_ARG,
                "vanka_setup: null argument");
  if (n_cells == 0) return DNNMG_OK;
  const size_t smem = sizeof(double) * (ndl * ndl + ndl) + sizeof(int) * ndl;
  static uint64_t configured = 0;
  if (first_use_on_device(configured)) {
    cudaFuncSetAttribute(vanka_invert_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(double) * (128 * 128 + 128) + sizeof(int) * 128));
  }
  const int grid = n_cells < 2 * kSMs ? n_cells : 2 * kSMs;
  vanka_invert_kernel<<<grid, kVankaThreads, smem, as_stream(s)>>>(n_cells, ndl, csr_data,
                                                                   flat_pos, inv, flags);
  DNNMG_CHECK_LAUNCH("vanka_invert_kernel");
  return DNNMG_OK;
}

extern "C" int32_t dnnmg_vanka_smooth(const dnnmg_vanka_t* V, const dnnmg_csr_t* J,
                                      const double* b, double* x, int32_t sweeps, double damping,
                                      double* r, double* dl, dnnmg_stream_t s) {
  using namespace dnnmg;
  DNNMG_REQUIRE(V && J && b && x && r && dl && V->cell_dofs && V->inv && V->weight &&
                    V->dof_cell_ptr && V->dof_cell_idx && J->indptr && J->indices && J->data,
                DNNMG_ERR_ARG, "vanka_smooth: null argument");
  DNNMG_REQUIRE(J->n_rows == V->n_dofs, DNNMG_ERR_ARG,
                "vanka_smooth: length of the Jacobian (%d) and the Vanka data (%d) differ",
                J->n_rows, V->n_dofs);
  cudaStream_t st = as_stream(s);
  for (int it = 0; it < sweeps; ++it) {
    csr_residual_kernel<<<grid_for((int64_t)J->n_rows * 32, 256, 16), 256, 0, st>>>(
        J->n_rows, J->indptr, J->indices, J->data, x, b, r);
    DNNMG_CHECK_LAUNCH("csr_residual_kernel");
    if (V->n_cells > 0) {
      const int grid = V->n_cells < 16 * kSMs ? V->n_cells : 16 * kSMs;
      vanka_apply_kernel<<<grid, kApplyThreads, sizeof(double) * V->ndl, st>>>(
          V->n_cells, V->ndl, V->cell_dofs, V->inv, r, dl);
      DNNMG_CHECK_LAUNCH("vanka_apply_kernel");
    }
    vanka_update_kernel<<<grid_for(V->n_dofs, 256), 256, 0, st>>>(
        V->n_dofs, V->dof_cell_ptr, V->dof_cell_idx, dl, V->weight, damping, x);
    DNNMG_CHECK_LAUNCH("vanka_update_kernel");
  }
  return DNNMG_OK;
}
