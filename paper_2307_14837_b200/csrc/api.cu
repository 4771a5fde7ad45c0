// extern "C" entry points of libdnnmg_b200.so (declared in include/dnnmg_b200.h).
#include <cstdarg>
#include <cstring>
#include "common.cuh"

namespace dnnmg {

static thread_local char g_last_error[512] = "";

int32_t set_error(int32_t status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return status;
}

int32_t launch_prolongate(const dnnmg_prolong_t*, const float*, float*, const dnnmg_dirichlet_t*,
                          cudaStream_t);
int32_t launch_dirichlet(const dnnmg_dirichlet_t*, float*, cudaStream_t);
int32_t launch_restrict(const dnnmg_restrict_t*, const float*, float*, cudaStream_t);
int32_t launch_level_geometry(const dnnmg_level_t*, float*, cudaStream_t);
int64_t k2tc_constant_bytes();
int32_t launch_k2tc_constants(void*, cudaStream_t);
int32_t launch_level_geometry_box(const dnnmg_level_t*, float*, int32_t*, cudaStream_t);
int32_t launch_k2tc_geometry(const dnnmg_level_t*, float*, int32_t, cudaStream_t);
int32_t launch_stab(const dnnmg_level_t*, const float*, const dnnmg_phys_t*, float*, float*,
                    cudaStream_t);
int32_t launch_residual(const dnnmg_level_t*, const float*, const float*, const float*,
                        const float*, const dnnmg_phys_t*, float*, float*, int, int, cudaStream_t,
                        cudaEvent_t b_ready = nullptr);
int32_t launch_gather(const dnnmg_patchset_t*, const float*, const float*, float*, cudaStream_t);
int32_t launch_restrict(const dnnmg_patchset_t*, const float*, float*, cudaStream_t);
int32_t launch_extend(const dnnmg_patchset_t*, const float*, float*, cudaStream_t);
int32_t launch_scatter_update(const dnnmg_patchset_t*, const float*, const uint8_t*, const float*,
                              float, float*, float*, cudaStream_t);
int32_t launch_mlp_simt(const dnnmg_mlp_t*, const float*, int64_t, float*, cudaStream_t);
int32_t mlp_tc_supported(const dnnmg_mlp_t*);
int32_t mlp_tc_packed_bytes(const dnnmg_mlp_t*, int64_t*);
int32_t launch_mlp_tc_pack(const dnnmg_mlp_t*, void*, cudaStream_t);
int32_t launch_mlp_tc(const dnnmg_mlp_t*, const float*, int64_t, float*, cudaStream_t);
int32_t launch_mlp_tc_gather(const dnnmg_mlp_t*, const dnnmg_patchset_t*, const float*,
                             const float*, float*, cudaStream_t);
int32_t mlp_tc_gather_mode(const dnnmg_mlp_t*, const dnnmg_patchset_t*);
int32_t mlp_layered_supported(const dnnmg_mlp_t*);
int32_t mlp_layered_packed_bytes(const dnnmg_mlp_t*, int64_t*);
int32_t mlp_layered_workspace_bytes(const dnnmg_mlp_t*, int64_t, int64_t*);
int32_t launch_mlp_layered_pack(const dnnmg_mlp_t*, void*, cudaStream_t);
int32_t launch_mlp_layered(const dnnmg_mlp_t*, const float*, int64_t, float*, void*, int64_t,
                           cudaStream_t);
int32_t launch_mlp_layered_patches(const dnnmg_mlp_t*, const dnnmg_patchset_t*, const float*,
                                   const float*, float*, void*, int64_t, cudaStream_t);

static int32_t check_mlp(const dnnmg_mlp_t* m) {
  DNNMG_REQUIRE(m, DNNMG_ERR_ARG, "mlp: null model");
  DNNMG_REQUIRE(m->depth >= 1 && m->depth < DNNMG_MAX_LAYERS, DNNMG_ERR_UNSUPPORTED,
                "mlp: depth %d outside [1, %d)", m->depth, DNNMG_MAX_LAYERS);
  DNNMG_REQUIRE(m->n_in > 0 && m->n_hidden > 0 && m->n_out > 0, DNNMG_ERR_ARG,
                "mlp: non-positive width");
  for (int i = 0; i <= m->depth; ++i)
    DNNMG_REQUIRE(m->W[i], DNNMG_ERR_ARG, "mlp: W[%d] is NULL", i);
  DNNMG_REQUIRE(m->bn_scale && m->bn_shift && m->in_mean && m->in_std, DNNMG_ERR_ARG,
                "mlp: missing normalisation vectors");
  // f16x3 splits the hidden activations into fp16 hi/lo parts: only a bounded activation
  // (tanh: |h| <= depth with the skips) keeps them inside the fp16 range; relu hidden
  // states are unbounded (net.py:57, the reference's default) and need tf32x3
  DNNMG_REQUIRE(m->precision != DNNMG_PREC_F16X3 || m->activation == DNNMG_ACT_TANH,
                DNNMG_ERR_UNSUPPORTED,
                "mlp: f16x3 needs a bounded activation (tanh); use tf32x3 for relu models");
  return DNNMG_OK;
}

}  // namespace dnnmg

using namespace dnnmg;

extern "C" {

int32_t dnnmg_version(void) { return 100; }

const char* dnnmg_status_string(int32_t status) {
  switch (status) {
    case DNNMG_OK: return "ok";
    case DNNMG_ERR_ARG: return "invalid argument";
    case DNNMG_ERR_CUDA: return "CUDA error";
    case DNNMG_ERR_UNSUPPORTED: return "unsupported configuration";
    case DNNMG_ERR_ARCH: return "model architecture does not match the patch layout";
    default: return "unknown status";
  }
}

const char* dnnmg_last_error(void) { return g_last_error; }

int32_t dnnmg_prolongate(const dnnmg_prolong_t* P, const float* xc, float* xf,
                         const dnnmg_dirichlet_t* bc, dnnmg_stream_t s) {
  return launch_prolongate(P, xc, xf, bc, as_stream(s));
}

int32_t dnnmg_apply_dirichlet(const dnnmg_dirichlet_t* bc, float* x, dnnmg_stream_t s) {
  return launch_dirichlet(bc, x, as_stream(s));
}

int32_t dnnmg_restrict(const dnnmg_restrict_t* R, const float* bf, float* bc, dnnmg_stream_t s) {
  return launch_restrict(R, bf, bc, as_stream(s));
}

int32_t dnnmg_level_geometry(const dnnmg_level_t* lv, float* geo, dnnmg_stream_t s) {
  return launch_level_geometry(lv, geo, as_stream(s));
}

int32_t dnnmg_level_geometry_box(const dnnmg_level_t* lv, float* box, int32_t* n_bad,
                                 dnnmg_stream_t s) {
  return launch_level_geometry_box(lv, box, n_bad, as_stream(s));
}

int64_t dnnmg_k2tc_constants_bytes(void) { return k2tc_constant_bytes(); }

int32_t dnnmg_k2tc_constants(void* img, dnnmg_stream_t s) {
  return launch_k2tc_constants(img, as_stream(s));
}

int64_t dnnmg_level_geometry_tc_floats(const dnnmg_level_t* lv, int32_t affine) {
  if (!lv || lv->n_cells <= 0) return 0;
  const int64_t n_tiles = (lv->n_cells + 127) / 128;
  return affine ? 10LL * lv->n_cells : n_tiles * 641 * 128;
}

int32_t dnnmg_level_geometry_tc(const dnnmg_level_t* lv, float* out, int32_t affine,
                                dnnmg_stream_t s) {
  return launch_k2tc_geometry(lv, out, affine, as_stream(s));
}

int32_t dnnmg_stab(const dnnmg_level_t* lv, const float* x, const dnnmg_phys_t* ph, float* aT,
                   float* dT, dnnmg_stream_t s) {
  return launch_stab(lv, x, ph, aT, dT, as_stream(s));
}

int32_t dnnmg_residual(const dnnmg_level_t* lv, const float* x, const float* b, const float* aT,
                       const float* dT, const dnnmg_phys_t* ph, float* elem, float* r,
                       int32_t apply_mask, dnnmg_stream_t s) {
  return launch_residual(lv, x, b, aT, dT, ph, elem, r, apply_mask, 1, as_stream(s));
}

int32_t dnnmg_apply_operator(const dnnmg_level_t* lv, const float* x, const float* aT,
                             const float* dT, const dnnmg_phys_t* ph, float* elem, float* out,
                             dnnmg_stream_t s) {
  return launch_residual(lv, x, nullptr, aT, dT, ph, elem, out, 0, 0, as_stream(s));
}

int32_t dnnmg_rhs_next(const dnnmg_level_t* lv, const float* x, const dnnmg_phys_t* ph,
                       float* elem, float* b, dnnmg_stream_t s) {
  return launch_residual(lv, x, nullptr, nullptr, nullptr, ph, elem, b, 0, 2, as_stream(s));
}

int32_t dnnmg_gather(const dnnmg_patchset_t* ps, const float* x, const float* r, float* X,
                     dnnmg_stream_t s) {
  return launch_gather(ps, x, r, X, as_stream(s));
}

int32_t dnnmg_local_restrict(const dnnmg_patchset_t* ps, const float* x, float* rows,
                             dnnmg_stream_t s) {
  return launch_restrict(ps, x, rows, as_stream(s));
}

int32_t dnnmg_global_extend(const dnnmg_patchset_t* ps, const float* rows, float* out,
                            dnnmg_stream_t s) {
  return launch_extend(ps, rows, out, as_stream(s));
}

int32_t dnnmg_mlp_packed_bytes(const dnnmg_mlp_t* m, int64_t* bytes) {
  int32_t st = check_mlp(m);
  if (st) return st;
  DNNMG_REQUIRE(bytes, DNNMG_ERR_ARG, "mlp_packed_bytes: null output");
  if (m->precision == DNNMG_PREC_FP32) {
    *bytes = 0;
    return DNNMG_OK;
  }
  if (mlp_tc_supported(m)) return mlp_tc_packed_bytes(m, bytes);
  DNNMG_REQUIRE(mlp_layered_supported(m), DNNMG_ERR_UNSUPPORTED,
                "mlp: tensor-core modes need n_hidden %% 32 == 0");
  return mlp_layered_packed_bytes(m, bytes);
}

int32_t dnnmg_mlp_pack(const dnnmg_mlp_t* m, void* packed, dnnmg_stream_t s) {
  int32_t st = check_mlp(m);
  if (st) return st;
  if (m->precision == DNNMG_PREC_FP32) return DNNMG_OK;
  DNNMG_REQUIRE(packed, DNNMG_ERR_ARG, "mlp_pack: null buffer");
  if (mlp_tc_supported(m)) return launch_mlp_tc_pack(m, packed, as_stream(s));
  return launch_mlp_layered_pack(m, packed, as_stream(s));
}

int32_t dnnmg_mlp_workspace_bytes(const dnnmg_mlp_t* m, int64_t n_rows, int64_t* bytes) {
  int32_t st = check_mlp(m);
  if (st) return st;
  DNNMG_REQUIRE(bytes && n_rows >= 0, DNNMG_ERR_ARG, "mlp_workspace_bytes: bad argument");
  *bytes = 0;
  if (m->precision == DNNMG_PREC_FP32 || mlp_tc_supported(m)) return DNNMG_OK;
  DNNMG_REQUIRE(mlp_layered_supported(m), DNNMG_ERR_UNSUPPORTED,
                "mlp: tensor-core modes need n_hidden %% 32 == 0");
  return mlp_layered_workspace_bytes(m, n_rows, bytes);
}

int32_t dnnmg_mlp_forward_ws(const dnnmg_mlp_t* m, const float* X, int64_t n_rows, float* Y,
                             void* workspace, int64_t ws_bytes, dnnmg_stream_t s) {
  int32_t st = check_mlp(m);
  if (st) return st;
  DNNMG_REQUIRE(n_rows >= 0, DNNMG_ERR_ARG, "mlp_forward: negative row count");
  if (n_rows == 0) return DNNMG_OK;   // an empty batch: nothing to read or write
  DNNMG_REQUIRE(X && Y, DNNMG_ERR_ARG, "mlp_forward: null argument");
  if (m->precision == DNNMG_PREC_FP32) return launch_mlp_simt(m, X, n_rows, Y, as_stream(s));
  DNNMG_REQUIRE(m->packed, DNNMG_ERR_ARG, "mlp_forward: tensor-core mode needs packed weights");
  if (mlp_tc_supported(m)) return launch_mlp_tc(m, X, n_rows, Y, as_stream(s));
  return launch_mlp_layered(m, X, n_rows, Y, workspace, ws_bytes, as_stream(s));
}

int32_t dnnmg_mlp_forward(const dnnmg_mlp_t* m, const float* X, int64_t n_rows, float* Y,
                          dnnmg_stream_t s) {
  int32_t st = check_mlp(m);
  if (st) return st;
  DNNMG_REQUIRE(n_rows >= 0, DNNMG_ERR_ARG, "mlp_forward: negative row count");
  if (n_rows == 0) return DNNMG_OK;   // an empty batch: nothing to read or write
  DNNMG_REQUIRE(X && Y, DNNMG_ERR_ARG, "mlp_forward: null argument");
  if (m->precision == DNNMG_PREC_FP32) return launch_mlp_simt(m, X, n_rows, Y, as_stream(s));
  DNNMG_REQUIRE(m->packed, DNNMG_ERR_ARG, "mlp_forward: tensor-core mode needs packed weights");
  DNNMG_REQUIRE(mlp_tc_supported(m), DNNMG_ERR_UNSUPPORTED,
                "mlp_forward: this width runs on the layered tensor-core kernel, which needs a "
                "workspace: use dnnmg_mlp_forward_ws");
  return launch_mlp_tc(m, X, n_rows, Y, as_stream(s));
}

static bool fused_gather(const dnnmg_mlp_t* m, const dnnmg_patchset_t* ps);
static bool layered_gather(const dnnmg_mlp_t* m);

int32_t dnnmg_mlp_forward_patches_ws(const dnnmg_mlp_t* m, const dnnmg_patchset_t* ps,
                                     const float* x, const float* r, float* Y, void* workspace,
                                     int64_t ws_bytes, dnnmg_stream_t s) {
  int32_t st = check_mlp(m);
  if (st) return st;
  DNNMG_REQUIRE(ps && ps->node_table && ps->geom && x && r && Y, DNNMG_ERR_ARG,
                "mlp_forward_patches: null argument");
  if (fused_gather(m, ps)) return dnnmg_mlp_forward_patches(m, ps, x, r, Y, s);
  DNNMG_REQUIRE(layered_gather(m), DNNMG_ERR_UNSUPPORTED,
                "mlp_forward_patches: needs a packed tensor-core model");
  DNNMG_REQUIRE(m->n_out == 3 * ps->nodes_per_patch, DNNMG_ERR_ARCH,
                "model architecture (%d outputs) does not match the patch layout (%d)", m->n_out,
                3 * ps->nodes_per_patch);
  if (ps->n_patches == 0) return DNNMG_OK;
  return launch_mlp_layered_patches(m, ps, x, r, Y, workspace, ws_bytes, as_stream(s));
}

int32_t dnnmg_mlp_forward_patches(const dnnmg_mlp_t* m, const dnnmg_patchset_t* ps, const float* x,
                                  const float* r, float* Y, dnnmg_stream_t s) {
  int32_t st = check_mlp(m);
  if (st) return st;
  DNNMG_REQUIRE(ps && ps->node_table && ps->geom && x && r && Y, DNNMG_ERR_ARG,
                "mlp_forward_patches: null argument");
  DNNMG_REQUIRE(m->n_in == 8 * ps->nodes_per_patch + ps->n_geo && m->n_out == 3 * ps->nodes_per_patch,
                DNNMG_ERR_ARCH, "model architecture (%d -> %d) does not match the patch layout (%d -> %d)",
                m->n_in, m->n_out, 8 * ps->nodes_per_patch + ps->n_geo, 3 * ps->nodes_per_patch);
  DNNMG_REQUIRE(m->precision != DNNMG_PREC_FP32 && mlp_tc_supported(m) && m->packed,
                DNNMG_ERR_UNSUPPORTED, "mlp_forward_patches: needs a packed tensor-core model");
  if (ps->n_patches == 0) return DNNMG_OK;
  return launch_mlp_tc_gather(m, ps, x, r, Y, as_stream(s));
}

int32_t dnnmg_mlp_gather_mode(const dnnmg_mlp_t* m, const dnnmg_patchset_t* ps) {
  if (!m || !ps || !m->packed || m->precision == DNNMG_PREC_FP32 || !mlp_tc_supported(m)) return -1;
  return mlp_tc_gather_mode(m, ps);
}

int32_t dnnmg_scatter_update(const dnnmg_patchset_t* ps, const float* Y, const uint8_t* mask,
                             const float* xt, float scale, float* d, float* xc, dnnmg_stream_t s) {
  return launch_scatter_update(ps, Y, mask, xt, scale, d, xc, as_stream(s));
}

static bool fused_gather(const dnnmg_mlp_t* m, const dnnmg_patchset_t* ps) {
  return m->precision != DNNMG_PREC_FP32 && mlp_tc_supported(m) && m->n_hidden == 256 && m->packed &&
         (ps == nullptr || (ps->n_geo % 4 == 0 && 8 * ps->nodes_per_patch + ps->n_geo <= 256));
}

static bool layered_gather(const dnnmg_mlp_t* m) {
  return m->precision != DNNMG_PREC_FP32 && !mlp_tc_supported(m) && mlp_layered_supported(m) &&
         m->packed;
}

int32_t dnnmg_correction_step_launches(int32_t J, const dnnmg_mlp_t* m) {
  // J prolongations + element + node-sum + MLP stage + scatter; the MLP stage is one fused
  // kernel, or (layered) epilogue affine + gathered layer-0 operand + one GEMM per layer,
  // or (fp32 SIMT) gather + MLP
  if (fused_gather(m, nullptr)) return J + 4;
  if (layered_gather(m)) return J + 3 + 2 + m->depth + 1;
  return J + 5;
}

int32_t dnnmg_correction_step(const dnnmg_prolong_t* P, int32_t J, const dnnmg_dirichlet_t* bc,
                              const dnnmg_level_t* fine, const dnnmg_phys_t* ph,
                              const dnnmg_patchset_t* ps, const dnnmg_mlp_t* m,
                              const float* x_coarse, const float* b_prev, float scale,
                              const dnnmg_step_buffers_t* buf, float* x_corr, dnnmg_stream_t s) {
  DNNMG_REQUIRE(P && fine && ph && ps && m && buf && x_coarse && b_prev && x_corr, DNNMG_ERR_ARG,
                "correction_step: null argument");
  DNNMG_REQUIRE(J == 1 || J == 2, DNNMG_ERR_ARG, "correction_step: unsupported patch depth J=%d", J);
  DNNMG_REQUIRE(J == 1 || buf->x_mid, DNNMG_ERR_ARG, "correction_step: J=2 needs x_mid");
  const int npp = ps->nodes_per_patch;
  DNNMG_REQUIRE(m->n_in == 8 * npp + ps->n_geo && m->n_out == 3 * npp, DNNMG_ERR_ARCH,
                "model architecture (%d -> %d) does not match the patch layout (%d -> %d)",
                m->n_in, m->n_out, 8 * npp + ps->n_geo, 3 * npp);
  cudaStream_t st = as_stream(s);
  int32_t rc;
  // (1) prolongate to L+J, (2) re-impose Dirichlet data on the fine level (driver.py:251-253)
  if (J == 1) {
    rc = launch_prolongate(&P[0], x_coarse, buf->x_tilde, bc, st);
  } else {
    rc = launch_prolongate(&P[0], x_coarse, buf->x_mid, nullptr, st);
    if (!rc) rc = launch_prolongate(&P[1], buf->x_mid, buf->x_tilde, bc, st);
  }
  if (rc) return rc;
  // (3) stab at x~ + residual against the carried RHS, masked (driver.py:255-258)
  rc = launch_residual(fine, buf->x_tilde, b_prev, nullptr, nullptr, ph, buf->elem, buf->r, 1, 1,
                       st, reinterpret_cast<cudaEvent_t>(buf->b_ready));
  if (rc) return rc;
  // (4) patch features, network, averaging scatter, update (driver.py:263-268)
  if (fused_gather(m, ps)) {
    rc = launch_mlp_tc_gather(m, ps, buf->x_tilde, buf->r, buf->Y, st);
  } else if (layered_gather(m)) {
    rc = launch_mlp_layered_patches(m, ps, buf->x_tilde, buf->r, buf->Y, buf->mlp_ws,
                                    buf->mlp_ws_bytes, st);
  } else {
    rc = launch_gather(ps, buf->x_tilde, buf->r, buf->X, st);
    if (!rc) rc = dnnmg_mlp_forward_ws(m, buf->X, ps->n_patches, buf->Y, buf->mlp_ws,
                                       buf->mlp_ws_bytes, s);
  }
  if (rc) return rc;
  return launch_scatter_update(ps, buf->Y, fine->dof_mask, buf->x_tilde, scale, buf->d, x_corr, st);
}

}  // extern "C"
