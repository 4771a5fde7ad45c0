// K4 fast path: tcgen05 / TMEM patch MLP (placeholder until the kernel lands).
#include "common.cuh"

namespace dnnmg {
int32_t mlp_tc_supported(const dnnmg_mlp_t*) { return 0; }
int32_t mlp_tc_packed_bytes(const dnnmg_mlp_t*, int64_t* b) { *b = 0; return DNNMG_ERR_UNSUPPORTED; }
int32_t launch_mlp_tc_pack(const dnnmg_mlp_t*, void*, cudaStream_t) { return DNNMG_ERR_UNSUPPORTED; }
int32_t launch_mlp_tc(const dnnmg_mlp_t*, const float*, int64_t, float*, cudaStream_t) {
  return DNNMG_ERR_UNSUPPORTED;
}
}  // namespace dnnmg
