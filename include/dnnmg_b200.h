/*
 * dnnmg_b200.h — C ABI of the B200-native DNN-MG fine-level correction step.
 *
 * The reference (dnnmg, arXiv 2307.14837, pure Python/numpy) exposes this hot
 * path only as Python functions; there is no FFI in the reference.  Each entry
 * point below replaces one of those functions and is what a ctypes/cffi binding
 * of the reference would bind:
 *
 *   dnnmg_prolongate        space.prolongate            space.py:177-185 (+ apply_dirichlet 245-255)
 *   dnnmg_apply_dirichlet   space.apply_dirichlet       space.py:245-255
 *   dnnmg_restrict          space.restrict_rhs          space.py:188-196 (P^T, Alg. 1 line 9)
 *   dnnmg_stab              Assembler.stab              assembly.py:169-178, 55-59
 *   dnnmg_residual          Assembler.assemble_residual assembly.py:261-267 (apply_operator 212-240)
 *   dnnmg_rhs_next          Assembler.assemble_rhs_next assembly.py:242-259
 *   dnnmg_gather            patch_ops.assemble_network_input  patch_ops.py:49-53 (local_restrict 23-29)
 *   dnnmg_local_restrict    patch_ops.local_restrict    patch_ops.py:23-29
 *   dnnmg_global_extend     patch_ops.global_extend     patch_ops.py:32-38
 *   dnnmg_mlp_forward       net.forward (eval mode)     net.py:124-164
 *   dnnmg_scatter_update    predict_correction scatter + x~ + scale*d
 *                                                       patch_ops.py:64-76, driver.py:268
 *   dnnmg_correction_step   TimeLoop._step_hybrid lines 251-268 (K1..K5 fused sequence)
 *   dnnmg_halo_*, dnnmg_nccl_*  x-slab decomposition of the same step (no reference
 *                           counterpart: the reference is single-process); the
 *                           interface sums reproduce assembly.py:180-184 / patch_ops.py:32-38
 *                           across ranks in the same (global) order
 *
 * Conventions (all match the reference):
 *   - dof vectors are node-major, component-minor: dof = 4*node + comp,
 *     comp 0 = pressure, 1..3 = velocity (space.py:3-7).  Device vectors are
 *     float32, 16-byte aligned, so a node is one float4.
 *   - index tables are int32, row-major, exactly the reference's numbering.
 *   - every pointer inside the structs and every array argument is a DEVICE
 *     pointer unless stated otherwise; calls are asynchronous on `stream`
 *     (a cudaStream_t passed as void*), never allocate, never synchronise,
 *     and are CUDA-graph capturable.
 *   - return value: DNNMG_OK or an error code; dnnmg_status_string() maps it
 *     to text.  Shape errors use the reference's ValueError wording
 *     ("length", "architecture", "width").
 */
#ifndef DNNMG_B200_H
#define DNNMG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* dnnmg_stream_t; /* cudaStream_t */

enum {
  DNNMG_OK = 0,
  DNNMG_ERR_ARG = 1,         /* invalid argument / shape ("length", "width") */
  DNNMG_ERR_CUDA = 2,        /* a CUDA launch or runtime call failed */
  DNNMG_ERR_UNSUPPORTED = 3, /* configuration not supported by this build */
  DNNMG_ERR_ARCH = 4         /* model architecture does not match the patch layout */
};

enum { DNNMG_ACT_RELU = 0, DNNMG_ACT_TANH = 1 };

enum {
  DNNMG_PREC_FP32 = 0,   /* SIMT fp32 FFMA (any width) */
  DNNMG_PREC_BF16 = 1,   /* tcgen05 kind::f16, bf16 operands, fp32 accumulate in TMEM */
  DNNMG_PREC_TF32X3 = 2, /* tcgen05 kind::tf32, 3-pass split (hi*hi + hi*lo + lo*hi), fp32 accuracy */
  DNNMG_PREC_F16X3 = 3,  /* tcgen05 kind::f16, fp16 3-pass split of power-of-two scaled weights,
                            fp32 accuracy at twice the tf32 rate; needs |activations| < 65504,
                            so only tanh models are accepted (relu: DNNMG_ERR_UNSUPPORTED,
                            use TF32X3) */
  DNNMG_PREC_FP8 = 4     /* tcgen05 kind::f8f6f4, e4m3 operands (weights scaled by a power of
                            two per layer), fp32 accumulate; report-only accuracy (~1e-1) */
};

/* Q2 embedding level l -> l+1 (space.py:117-165).  Each fine node n takes the
 * coarse shape values of the first (octant o, child-local node a, parent cell C)
 * that reaches it; fine_src[n] = C*216 + o*27 + a. */
typedef struct {
  int32_t n_fine_nodes;
  int32_t n_coarse_cells;
  const int32_t* coarse_cell_nodes; /* [n_coarse_cells][27] level-l Q2 node table */
  const int32_t* fine_src;          /* [n_fine_nodes] */
  /* optional owner lists (the same information grouped by parent cell): the fine
   * nodes whose first-appearance parent is C are owner_node[owner_ptr[C]..owner_ptr[C+1])
   * with local code o*27 + a in owner_code; when present K1 stages each parent's 27
   * coarse values once per cell instead of gathering them per fine node */
  const int32_t* owner_ptr;         /* [n_coarse_cells+1] or NULL */
  const int32_t* owner_node;        /* [n_fine_nodes] */
  const uint8_t* owner_code;        /* [n_fine_nodes] */
  /* optional lattice form of the owner lists (takes precedence in K1): lat_node[C][25 pz +
   * 5 py + px] = the fine node at position (px, py, pz) of the 5 x 5 x 5 lattice of the refined
   * cell C when C is its first-appearance parent, else -1.  K1 then interpolates whole 1-D
   * lines per lane with no per-node index decoding */
  const int32_t* lat_node;          /* [n_coarse_cells][125] or NULL */
} dnnmg_prolong_t;

/* Restriction level l+1 -> l of a dual (RHS) vector: b_coarse = P^T b_fine
 * (space.py:188-196), the transpose of the K1 stencil as a coarse-node CSR whose rows
 * list the fine nodes in ascending order with their dyadic weights.  Owner-computes on
 * coarse nodes: deterministic, no atomics. */
typedef struct {
  int32_t n_coarse_nodes;
  int32_t n_fine_nodes;
  const int32_t* ptr;   /* [n_coarse_nodes+1] */
  const int32_t* fine;  /* [nnz] */
  const float* w;       /* [nnz] */
  /* optional owner-computes form (all set, or all NULL): per coarse cell, the transpose of
   * K1's separable stencil applied to the fine nodes whose first-appearance parent it is
   * (owner lists as in dnnmg_prolong_t) gives 27 partial sums into cell_scratch, which are
   * then summed per coarse node over its incident (cell, local node) entries in ascending
   * cell order.  Deterministic; streams b_fine once instead of gathering it per P entry. */
  int32_t n_coarse_cells;
  const int32_t* coarse_cell_nodes; /* [n_coarse_cells][27] (unused by the kernels; layout ref) */
  const int32_t* owner_ptr;         /* [n_coarse_cells+1] */
  const int32_t* owner_node;        /* [n_fine_nodes] */
  const uint8_t* owner_code;        /* [n_fine_nodes]: o*27 + a */
  const int32_t* node_cell_ptr;     /* [n_coarse_nodes+1] CSR coarse node -> cell*27 + a */
  const int32_t* node_cell_idx;
  float* cell_scratch;              /* [n_coarse_cells][27][4] device scratch */
} dnnmg_restrict_t;

/* Dirichlet data of one level (space.py:245-255): bc_code[n] = 0 untouched,
 * 1 velocity := 0 (no-slip), 2 velocity := bc_values[n]. */
typedef struct {
  int32_t n_nodes;
  const uint8_t* bc_code;  /* [n_nodes] */
  const float* bc_values;  /* [n_nodes][3] or NULL when no code 2 is present */
  const uint8_t* bc_code_owner;  /* optional [n_nodes]: bc_code in the owner order of the
                                    prolongation it is applied with (dnnmg_prolong_t.owner_node),
                                    read coalesced instead of gathered per owned node; NULL:
                                    gathered */
  const int32_t* lat_node_bc;    /* optional [n_coarse_cells][125]: the lat_node table of the
                                    prolongation this data is applied with, each owned entry
                                    carrying bc_code[node] in bits 29-30 (node ids < 2^29), so
                                    that K1's lattice form needs no Dirichlet-code load; NULL:
                                    bc_code is gathered per node */
} dnnmg_dirichlet_t;

/* One fine level for assembly (assembly.py:65-108). */
typedef struct {
  int32_t n_nodes;
  int32_t n_cells;
  const int32_t* cell_nodes;     /* [n_cells][27] (space.cell_nodes) */
  const double* coords;          /* [n_nodes][3] node coordinates (float64: geometry is
                                    formed from cell-relative differences in fp64) */
  const float* h_T;              /* [n_cells] cell diameters (assembly.py:100-103) */
  const int32_t* node_cell_ptr;  /* [n_nodes+1] CSR node -> incident (cell*27 + a), */
  const int32_t* node_cell_idx;  /*   cells ascending (= the reference bincount order) */
  const uint8_t* dof_mask;       /* [n_nodes] bit c set <=> dof 4n+c constrained; NULL = none */
  const float* geo_q;            /* per-mesh geometry cache from dnnmg_level_geometry
                                    ([n_cells][10][64]: J^-1 row-major, w) or NULL: K2 then
                                    recomputes the isoparametric geometry every call */
  const int32_t* node_order;     /* [n_nodes] permutation: the node sum visits node_order[i]
                                    at position i (NULL = ascending ids).  Any order gives the
                                    same bits (each node's sum is ordered by its CSR row); the
                                    build passes nodes by descending first incident cell, so
                                    the element vectors written last (still in L2) are read
                                    first and every node is visited next to its cells */
  /* optional tensor-core element kernel (all set, or tc_const NULL = the SIMT kernel): */
  const void* tc_const;          /* constant operand image, dnnmg_k2tc_constants_bytes() bytes,
                                    written once by dnnmg_k2tc_constants */
  const float* tc_geo;           /* dnnmg_level_geometry_tc output */
  int32_t tc_geo_affine;         /* its layout: 0 = per point, 1 = per-cell affine record,
                                    2 = the same for axis-aligned cells (J^-1 diagonal) */
  /* optional, with node_order: the CSR rows stored in visiting order (row i = the row of node
     node_order[i]: entries visit_ptr[i] .. visit_ptr[i+1] of visit_idx), so the node sum reads
     its row bounds without first resolving the node id (one dependent load fewer) */
  const int32_t* visit_ptr;      /* [n_nodes+1] */
  const int32_t* visit_idx;
  /* optional, for a level whose cells are all axis-aligned boxes (an unjittered box mesh):
     the per-cell record of dnnmg_level_geometry_box, [n_cells][4] = (1/hx, 1/hy, 1/hz, det J).
     J^-1 is then diagonal and constant over a cell, and K2's element kernel takes its box form
     (no per-point geometry, no products with the zero off-diagonal entries); it takes
     precedence over geo_q.  Set it only when dnnmg_level_geometry_box reported 0 bad cells. */
  const float* geo_box;
} dnnmg_level_t;

typedef struct {
  float nu, k, alpha0, delta0;
  int32_t convection;  /* 1: with convection (reference default) */
} dnnmg_phys_t;

/* PatchSet (mesh.py:501-558).  For J=1 the node->patch CSR equals the
 * node->cell CSR of the fine level because patch p == fine cell p. */
typedef struct {
  int32_t n_patches;
  int32_t nodes_per_patch;        /* 27 (J=1) or 125 (J=2) */
  int32_t n_geo;                  /* 24 */
  int32_t n_nodes;                /* fine-level scalar nodes */
  const int32_t* node_table;      /* [n_patches][nodes_per_patch] */
  const float* geom;              /* [n_patches][n_geo] */
  const int32_t* node_patch_ptr;  /* [n_nodes+1] CSR node -> (patch*npp + slot), ascending patch */
  const int32_t* node_patch_idx;
  /* optional (all NULL/0 = absent): distinct nodes of every 128-patch tile of the fused
   * tensor-core gather.  Tile t's distinct nodes are tile_nodes[t*tile_cap ..
   * t*tile_cap + tile_count[t]) in ascending id; tile_slot[p*npp + s] is the position of
   * node_table[p][s] in its tile's list.  With these, the MLP kernel stages each tile's
   * distinct x~/r rows in shared memory one tile ahead (cp.async from a dedicated warp)
   * instead of gathering every (patch, slot) from global memory at the tile boundary. */
  int32_t tile_cap;               /* row stride of tile_nodes (>= max tile_count) */
  const int32_t* tile_nodes;      /* [n_tiles][tile_cap], n_tiles = ceil(n_patches/128) */
  const int32_t* tile_count;      /* [n_tiles] */
  const uint16_t* tile_slot;      /* [n_tiles*128][npp] (rows past n_patches: any valid slot) */
  const int32_t* node_order;      /* [n_nodes] visiting order of the scatter (K5), as
                                     dnnmg_level_t.node_order; NULL = ascending ids */
  const int32_t* visit_ptr;       /* optional, with node_order: the node -> (patch, slot) CSR */
  const int32_t* visit_idx;       /*   rows in visiting order, as dnnmg_level_t.visit_ptr */
} dnnmg_patchset_t;

#define DNNMG_MAX_LAYERS 16

/* Eval-mode MlpModel (net.py:54-159): depth hidden layers + linear head.
 * bn_scale = gamma/sqrt(running_var+eps), bn_shift = beta - running_mean*bn_scale. */
typedef struct {
  int32_t n_in, n_hidden, depth, n_out;
  int32_t activation;                    /* DNNMG_ACT_* */
  int32_t precision;                     /* DNNMG_PREC_* */
  const float* W[DNNMG_MAX_LAYERS];      /* W[i]: [dims[i]][dims[i+1]] row-major, i = 0..depth */
  const float* bn_scale;                 /* [depth][n_hidden] */
  const float* bn_shift;                 /* [depth][n_hidden] */
  const float* in_mean;                  /* [n_in] */
  const float* in_std;                   /* [n_in] */
  void* packed;                          /* tensor-core weight image (dnnmg_mlp_pack), or NULL */
} dnnmg_mlp_t;

/* ---- versioning / errors -------------------------------------------------- */
int32_t dnnmg_version(void);
const char* dnnmg_status_string(int32_t status);
const char* dnnmg_last_error(void);   /* detail of the last failing call (host string) */

/* ---- K1: prolongation + Dirichlet ------------------------------------------- */
int32_t dnnmg_prolongate(const dnnmg_prolong_t* P, const float* x_coarse, float* x_fine,
                         const dnnmg_dirichlet_t* bc /* nullable */, dnnmg_stream_t stream);
int32_t dnnmg_apply_dirichlet(const dnnmg_dirichlet_t* bc, float* x, dnnmg_stream_t stream);
/* restriction (next row #1, Alg. 1 line 9): b_coarse = P^T b_fine, node-major float4 */
int32_t dnnmg_restrict(const dnnmg_restrict_t* R, const float* b_fine, float* b_coarse,
                       dnnmg_stream_t stream);

/* ---- K2: stabilisation, residual, next RHS ---------------------------------- */
/* geometry cache of a level (constant mesh): geo_out = [n_cells][10][64] float32, i.e.
 * 2,560 bytes per cell; set lv->geo_q = geo_out to let K2 skip the geometry work */
int32_t dnnmg_level_geometry(const dnnmg_level_t* lv, float* geo_out, dnnmg_stream_t stream);
/* box record of a level (see dnnmg_level_t.geo_box): box_out = [n_cells][4] float32 (16-byte
 * aligned); *n_bad_dev (device int32, nullable) receives the number of cells that are not
 * axis-aligned boxes with their 27 nodes on the tri-quadratic lattice (tolerance 1e-12 of the
 * cell size, fp64) -- use the record only when it is 0. */
int32_t dnnmg_level_geometry_box(const dnnmg_level_t* lv, float* box_out, int32_t* n_bad_dev,
                                 dnnmg_stream_t stream);
/* Tensor-core K2 (element vectors as tcgen05 GEMMs, SURVEY App. C "K2 v2"): the constant
 * operand image (Q2 basis / gradient / projected-gradient tables at the Gauss points, fp16
 * hi/lo, 160 KB, device buffer 128-byte aligned) and the geometry in the kernel's layout:
 * affine != 0 (every cell's isoparametric map affine, e.g. an unjittered box) -> per-cell
 * record [10][n_cells] (J^-1 row-major, det J); affine == 0 -> the per-point cache re-laid
 * out by 128-cell tiles [n_tiles][10][64][128], then the cells' volumes [n_tiles*128] (the
 * reference mass applied exactly on the CUDA cores).  Needs lv->geo_q (dnnmg_level_geometry).
 * out: dnnmg_level_geometry_tc_floats(lv, affine) floats. */
int64_t dnnmg_k2tc_constants_bytes(void);
int32_t dnnmg_k2tc_constants(void* img, dnnmg_stream_t stream);
int64_t dnnmg_level_geometry_tc_floats(const dnnmg_level_t* lv, int32_t affine);
int32_t dnnmg_level_geometry_tc(const dnnmg_level_t* lv, float* out, int32_t affine,
                                dnnmg_stream_t stream);
int32_t dnnmg_stab(const dnnmg_level_t* lv, const float* x, const dnnmg_phys_t* ph,
                   float* alpha_T, float* delta_T, dnnmg_stream_t stream);
/* r = b_prev - A_h(x); rows with dof_mask bits set are zeroed when apply_mask != 0.
 * alpha_T/delta_T may be NULL: then they are evaluated at x inside the kernel
 * (exactly Assembler.stab(x) as the hybrid step does, driver.py:255).
 * elem_scratch: [n_cells][27][4] floats. */
int32_t dnnmg_residual(const dnnmg_level_t* lv, const float* x, const float* b_prev,
                       const float* alpha_T, const float* delta_T, const dnnmg_phys_t* ph,
                       float* elem_scratch, float* r, int32_t apply_mask, dnnmg_stream_t stream);
/* A_h(x) itself (Assembler.apply_operator, assembly.py:212-234). */
int32_t dnnmg_apply_operator(const dnnmg_level_t* lv, const float* x, const float* alpha_T,
                             const float* delta_T, const dnnmg_phys_t* ph,
                             float* elem_scratch, float* out, dnnmg_stream_t stream);
/* next-step RHS with f = None (assembly.py:242-259). */
int32_t dnnmg_rhs_next(const dnnmg_level_t* lv, const float* x, const dnnmg_phys_t* ph,
                       float* elem_scratch, float* b, dnnmg_stream_t stream);

/* ---- K3: patch gather --------------------------------------------------------- */
/* X[p] = [x rows | r rows | geom] : [n_patches][8*npp + n_geo] fp32 */
int32_t dnnmg_gather(const dnnmg_patchset_t* ps, const float* x, const float* r, float* X,
                     dnnmg_stream_t stream);
/* rows[p] = x[dof_table[p]] : [n_patches][4*npp] */
int32_t dnnmg_local_restrict(const dnnmg_patchset_t* ps, const float* x, float* rows,
                             dnnmg_stream_t stream);
/* out = mu * bincount(dof_table, rows)  (all 4 components) */
int32_t dnnmg_global_extend(const dnnmg_patchset_t* ps, const float* rows, float* out,
                            dnnmg_stream_t stream);

/* ---- K4: patch MLP --------------------------------------------------------------- */
int32_t dnnmg_mlp_packed_bytes(const dnnmg_mlp_t* m, int64_t* bytes);
int32_t dnnmg_mlp_pack(const dnnmg_mlp_t* m, void* packed, dnnmg_stream_t stream);
int32_t dnnmg_mlp_forward(const dnnmg_mlp_t* m, const float* X, int64_t n_rows, float* Y,
                          dnnmg_stream_t stream);
/* Widths the fused per-tile kernel does not hold on chip (tensor-core modes with
 * n_hidden != 256, n_in > 256 or n_out > 256; n_hidden % 32 == 0) run layer by layer
 * (one tcgen05 GEMM per layer with the BN/activation/skip epilogue fused, activations in
 * HBM in the split canonical operand layout), which needs a caller-owned device workspace
 * of dnnmg_mlp_workspace_bytes(m, n_rows) bytes (0: none needed). */
int32_t dnnmg_mlp_workspace_bytes(const dnnmg_mlp_t* m, int64_t n_rows, int64_t* bytes);
int32_t dnnmg_mlp_forward_ws(const dnnmg_mlp_t* m, const float* X, int64_t n_rows, float* Y,
                             void* workspace, int64_t workspace_bytes, dnnmg_stream_t stream);

/* K3 fused into K4 (tensor-core modes, 8*npp + n_geo <= 256): the network input rows
 * [x~ | r | geometry] are gathered straight into the layer-0 operand; X is never stored. */
int32_t dnnmg_mlp_forward_patches(const dnnmg_mlp_t* m, const dnnmg_patchset_t* ps, const float* x,
                                  const float* r, float* Y, dnnmg_stream_t stream);
/* The same for every tensor-core width: the fused kernel when it applies, else the layered
 * kernel with the layer-0 operand gathered from x~, r and the geometry (workspace as for
 * dnnmg_mlp_forward_ws). */
int32_t dnnmg_mlp_forward_patches_ws(const dnnmg_mlp_t* m, const dnnmg_patchset_t* ps,
                                     const float* x, const float* r, float* Y, void* workspace,
                                     int64_t workspace_bytes, dnnmg_stream_t stream);

/* Which layer-0 source dnnmg_mlp_forward_patches uses for (m, ps): 1 = direct gather of
 * every (patch, slot) at the tile boundary, 2 = staged gather of each tile's distinct nodes
 * (needs ps->tile_* and enough shared memory), -1 = no tensor-core model.  Host only. */
int32_t dnnmg_mlp_gather_mode(const dnnmg_mlp_t* m, const dnnmg_patchset_t* ps);
/* ---- K5: averaging scatter + correction update ---------------------------------------- */
/* d = mu * bincount(velocity rows Y); d[mask] = 0; pressure 0; x_corr = x_tilde + scale*d.
 * Y: [n_patches][3*npp].  x_tilde/x_corr may be NULL (then only d is written). */
int32_t dnnmg_scatter_update(const dnnmg_patchset_t* ps, const float* Y, const uint8_t* dof_mask,
                             const float* x_tilde, float scale, float* d, float* x_corr,
                             dnnmg_stream_t stream);

/* ---- training data -------------------------------------------------
 * rows[p] = [x~ rows | r rows | geometry | targets] as float64, the dataset-shard row of
 * driver.export_training_data (driver.py:317-383, io.write_dataset io.py:219-287):
 * features as assemble_network_input (patch_ops.py:49-53), targets as patch_targets
 * (patch_ops.py:79-82), i.e. (v_ref - x~) at the velocity slots.  r NULL: zero residual
 * block; v_ref NULL: zero targets; x_ref (float64, nullable) replaces x~ in the target
 * difference.  rows: [n_patches][8*npp + n_geo + 3*npp]. */
int32_t dnnmg_dataset_rows(const dnnmg_patchset_t* ps, const float* x_tilde, const float* r,
                           const double* v_ref, const double* x_ref, double* rows,
                           dnnmg_stream_t stream);
/* Per-column statistics of a float64 row block [n][w] for the dataset sidecar: stats =
 * [sum | centred sum of squares M2 | min | max], each [w]; deterministic (fixed-order
 * two-pass partials combined pairwise).
 * scratch: dnnmg_column_stats_scratch(w) doubles (device). */
int32_t dnnmg_column_stats_scratch(int32_t w);
/* Ideal correction of oracle_loop_features (driver.py:418-424): x_corr = x~ + d with
 * d = v_ref - x~ at free velocity dofs; pressure and constrained dofs (dof_mask bits) keep
 * x~.  Per node float4 x~ / x_corr, float64 v_ref [4*n_nodes]. */
int32_t dnnmg_ideal_update(int32_t n_nodes, const float* x_tilde, const double* v_ref,
                           const uint8_t* dof_mask, float* x_corr, dnnmg_stream_t stream);
int32_t dnnmg_column_stats(const double* rows, int64_t n, int32_t w, double* scratch,
                           double* stats, dnnmg_stream_t stream);
/* ---- coarse-level Vanka smoother (msolve.py:51-89) -----------------
 * A level Jacobian in CSR (float64, the reference's assemble_jacobian output) and the
 * prefactored cell blocks of VankaData. */
typedef struct {
  int32_t n_rows;
  const int32_t* indptr;   /* [n_rows+1] */
  const int32_t* indices;  /* [nnz] */
  const double* data;      /* [nnz] */
} dnnmg_csr_t;
typedef struct {
  int32_t n_cells, ndl, n_dofs;  /* ndl = (d+1) 3^d = 108 */
  const int32_t* cell_dofs;      /* [n_cells][ndl] (Assembler.cell_dofs) */
  const int32_t* dof_cell_ptr;   /* [n_dofs+1] CSR dof -> (cell*ndl + i), ascending: the */
  const int32_t* dof_cell_idx;   /*   order of np.bincount over cell_dofs */
  const double* weight;          /* [n_dofs] 1 / multiplicity */
  const double* inv;             /* [n_cells][ndl][ndl] inverted blocks, TRANSPOSED (column j of
                                    the inverse contiguous), as written by dnnmg_vanka_setup */
} dnnmg_vanka_t;
/* inv[c] = transpose of (J.data[flat_pos[c*ndl*ndl ...]] as an ndl x ndl block)^-1, float64
 * (Gauss-Jordan, partial pivoting); a singular block is retried with a 1e-12 diagonal
 * shift: flags[c] = 0 regular, 1 shifted (the reference's `flagged`), 2 singular. */
int32_t dnnmg_vanka_setup(int32_t n_cells, int32_t ndl, const double* csr_data,
                          const int64_t* flat_pos, double* inv, int32_t* flags,
                          dnnmg_stream_t stream);
/* `sweeps` Jacobi-coupled Vanka sweeps on x in place (msolve.vanka_smooth):
 * r = b - J x; dl = inv r[dofs]; x += damping * weight * bincount(dofs, dl).
 * Scratch: r [n_dofs], dl [n_cells*ndl] (float64, device). */
int32_t dnnmg_vanka_smooth(const dnnmg_vanka_t* V, const dnnmg_csr_t* J, const double* b,
                           double* x, int32_t sweeps, double damping, double* r, double* dl,
                           dnnmg_stream_t stream);
/* ---- whole correction step (driver.py:251-268) ------------------------------------------ */
typedef struct {
  float* x_tilde;   /* [4*n_fine] */
  float* r;         /* [4*n_fine] */
  float* elem;      /* [n_cells*27*4] */
  float* X;         /* [n_patches][n_in] */
  float* Y;         /* [n_patches][n_out] */
  float* d;         /* [4*n_fine] */
  float* x_mid;     /* [4*n_mid] intermediate level for J = 2, else NULL */
  void* mlp_ws;     /* dnnmg_mlp_workspace_bytes(m, n_patches) bytes, or NULL when 0 */
  int64_t mlp_ws_bytes; /* size of mlp_ws: a smaller buffer than the rows need is an error */
  void* b_ready;    /* optional cudaEvent_t: b_prev may still be in flight (e.g. its H2D copy);
                       the step waits for it on its stream right before its first read of b_prev
                       (the residual's node sum), so prolongation and the element kernel overlap
                       the copy.  NULL: b_prev is ready.  Not for use inside stream capture. */
} dnnmg_step_buffers_t;

/* prolongations: J entries (levels L..L+J-1); bc: Dirichlet data of the fine level. */
int32_t dnnmg_correction_step(const dnnmg_prolong_t* P, int32_t J, const dnnmg_dirichlet_t* bc,
                              const dnnmg_level_t* fine, const dnnmg_phys_t* ph,
                              const dnnmg_patchset_t* ps, const dnnmg_mlp_t* m,
                              const float* x_coarse, const float* b_prev, float scale,
                              const dnnmg_step_buffers_t* buf, float* x_corr,
                              dnnmg_stream_t stream);

/* ---- x-slab halo (interface) operations, SURVEY §8(e) -------------------------------------
 * The single-domain step sums, per node, element vectors in ascending GLOBAL cell id
 * (assembly.py:180-184) and patch predictions in ascending GLOBAL patch id
 * (patch_ops.py:32-38).  Along a slab interface those orders interleave the two sides, so
 * each rank sends its raw per-(cell, local node) element rows / per-(patch, slot) velocity
 * predictions of the interface nodes, and both ranks sum the union in the global order of a
 * merge plan: interface values are bitwise equal on both sides and to the single domain.
 * All buffers are float4 rows. */
typedef struct {
  int32_t n_nodes;           /* interface nodes of this side */
  const int32_t* nodes;      /* [n_nodes] local node ids, in the order both ranks agree on */
  int32_t n_send;            /* entries this rank sends (= entries it receives) */
  const int32_t* send;       /* [n_send] local entries (cell*27 + a, or patch*npp + slot):
                                nodes in order, each node's entries by ascending global id */
  const int32_t* merge_ptr;  /* [n_nodes+1] */
  const int32_t* merge_src;  /* [merge_ptr[n_nodes]] a node's entries by ascending global id:
                                >= 0 local entry, < 0 entry -(1+q) of the received message */
} dnnmg_halo_plan_t;

/* One rank's interfaces: side 0 = left neighbour (rank-1), side 1 = right (rank+1). */
typedef struct {
  int32_t peer[2];                 /* neighbour rank per side, -1 = no neighbour */
  dnnmg_halo_plan_t cells[2];      /* element-vector plans of the fine level */
  dnnmg_halo_plan_t patches[2];    /* (patch, slot) plans */
  float* send[2];                  /* [max n_send][4] device message buffers per side */
  float* recv[2];
} dnnmg_slab_t;

/* sendbuf[j] = rows[h->send[j]] (float4 rows, e.g. the element scratch of dnnmg_residual) */
int32_t dnnmg_halo_pack_rows(const dnnmg_halo_plan_t* h, const float* rows, float* sendbuf,
                             dnnmg_stream_t stream);
/* sendbuf[j] = (Y velocity triple of entry h->send[j] = patch*npp + slot, 0) */
int32_t dnnmg_halo_pack_patch_rows(const dnnmg_halo_plan_t* h, const dnnmg_patchset_t* ps,
                                   const float* Y, float* sendbuf, dnnmg_stream_t stream);
/* out[node] = b[node] - (merged sum) (b NULL: the sum itself, e.g. the next RHS); masked dofs
 * -> 0 (mask nullable) */
int32_t dnnmg_halo_merge_rows(const dnnmg_halo_plan_t* h, const float* rows, const float* recvbuf,
                              const float* b, const uint8_t* mask, float* out,
                              dnnmg_stream_t stream);
/* d[node] = mu * (merged sum of the velocity predictions), mu = 1/(incident patches on both
 * sides); masked dofs -> 0; x_corr = x~ + scale*d (x_corr nullable) */
int32_t dnnmg_halo_merge_scatter(const dnnmg_halo_plan_t* h, const dnnmg_patchset_t* ps,
                                 const float* Y, const float* recvbuf, const uint8_t* mask,
                                 const float* x_tilde, float scale, float* d, float* x_corr,
                                 dnnmg_stream_t stream);

/* NCCL (the library binds the libnccl.so.2 already loaded in the process, else dlopens it).
 * comm is an ncclComm_t.  Bootstrap: rank 0 calls dnnmg_nccl_unique_id (128 bytes), the id is
 * broadcast out of band (torch.distributed store), every rank calls dnnmg_nccl_comm_init. */
int32_t dnnmg_nccl_available(void);
int32_t dnnmg_nccl_unique_id(void* id_out /* 128 bytes */);
int32_t dnnmg_nccl_comm_init(const void* id, int32_t nranks, int32_t rank, void** comm);
int32_t dnnmg_nccl_comm_count(void* comm, int32_t* count);
int32_t dnnmg_nccl_comm_destroy(void* comm);
/* grouped ncclSend/ncclRecv of count[side] float4 rows with peer[side] (< 0: none) on stream */
int32_t dnnmg_halo_exchange(void* comm, const int32_t peer[2], const float* const send[2],
                            float* const recv[2], const int64_t count[2], dnnmg_stream_t stream);
/* exchange (a), between the residual and the MLP: pack the interface element vectors,
 * exchange with both neighbours, write the merged r = b_prev - A at the interface nodes
 * (b_prev NULL: the merged sum, for the next-step RHS) */
int32_t dnnmg_halo_pre(const dnnmg_slab_t* sl, void* comm, const float* elem_scratch,
                       const float* b_prev, const uint8_t* dof_mask, float* r,
                       dnnmg_stream_t stream);
/* exchange (b), after the MLP: pack the interface patch predictions, exchange, write the merged
 * d and x_corr at the interface nodes */
int32_t dnnmg_halo_post(const dnnmg_slab_t* sl, void* comm, const dnnmg_patchset_t* ps,
                        const float* Y, const uint8_t* dof_mask, const float* x_tilde, float scale,
                        float* d, float* x_corr, dnnmg_stream_t stream);

/* Number of kernels dnnmg_correction_step launches for this configuration. */
int32_t dnnmg_correction_step_launches(int32_t J, const dnnmg_mlp_t* m);

#ifdef __cplusplus
}
#endif
#endif /* DNNMG_B200_H */
