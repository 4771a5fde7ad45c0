// Slab-interface (halo) kernels of the x-slab domain decomposition and the
// NCCL exchange that connects them.
//
// Each rank owns a contiguous x-range of level-0 cells and everything refined from them.
// Fine nodes on an interface plane are incident to cells and patches of both neighbouring
// slabs.  The single-domain step sums, per node, the element vectors of its incident cells
// in ascending GLOBAL cell id (assembly.py:180-184, np.bincount over cell_dofs) and the
// patch predictions of its incident patches in ascending GLOBAL patch id (patch_ops.py:32-38).
// Along an interface those orders interleave the two sides (cells are numbered k, then i,
// then j; children 8c+o), so a partial sum per side cannot reproduce them.  Instead each
// rank sends its raw per-(cell, local node) element vectors and per-(patch, slot) velocity
// predictions of the interface nodes, and both ranks sum the union in the global order
// described by a merge plan (built on the host, slab.py).  The interface values are then
// bitwise equal on both ranks AND to the single-domain step.
//
// A plan (dnnmg_halo_plan_t) per side and quantity:
//   nodes[i]                    interface node i (local id), order agreed by both ranks
//   send[j]                     local entry j of this rank's message (element row cell*27+a,
//                               or patch*npp+slot), nodes in order, ascending global id
//   merge_src[merge_ptr[i]..]   the node's entries in ascending global cell / patch id:
//                               >= 0 a local entry, < 0 entry -(1+q) of the received message
#include <dlfcn.h>
#include <cstring>
#include <nccl.h>

#include "common.cuh"

namespace dnnmg {

__global__ void __launch_bounds__(256) halo_pack_rows_kernel(int n, const int32_t* __restrict__ send,
                                                             const float4* __restrict__ src,
                                                             float4* __restrict__ out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    out[j] = __ldg(src + __ldg(send + j));
}

__global__ void __launch_bounds__(256) halo_pack_patch_kernel(int n, const int32_t* __restrict__ send,
                                                              int npp, const float* __restrict__ Y,
                                                              float4* __restrict__ out) {
  const int n_out = 3 * npp;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const int ps = __ldg(send + j);
    const int p = ps / npp;
    const float* y = Y + (int64_t)p * n_out + 3 * (ps - p * npp);
    out[j] = make_float4(__ldg(y), __ldg(y + 1), __ldg(y + 2), 0.f);
  }
}

// out[node] = b - sum (or the sum itself when b is NULL), summed exactly as node_sum_kernel
// (0 + v_0 + v_1 + ..., per component) over the merged entries; masked dofs -> 0
__global__ void __launch_bounds__(256) halo_merge_rows_kernel(
    int n, const int32_t* __restrict__ nodes, const int32_t* __restrict__ mptr,
    const int32_t* __restrict__ msrc, const float4* __restrict__ elem,
    const float4* __restrict__ recv, const float4* __restrict__ b,
    const uint8_t* __restrict__ mask, float4* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int node = __ldg(nodes + i);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = __ldg(mptr + i), e = __ldg(mptr + i + 1); j < e; ++j) {
      const int s = __ldg(msrc + j);
      const float4 v = s >= 0 ? __ldg(elem + s) : __ldg(recv + (-1 - s));
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    float4 r;
    if (b) {
      const float4 bb = __ldg(b + node);
      r = make_float4(bb.x - acc.x, bb.y - acc.y, bb.z - acc.z, bb.w - acc.w);
    } else {
      r = make_float4(1.0f * acc.x, 1.0f * acc.y, 1.0f * acc.z, 1.0f * acc.w);
    }
    if (mask) {
      const uint8_t m = mask[node];
      if (m & 1) r.x = 0.f;
      if (m & 2) r.y = 0.f;
      if (m & 4) r.z = 0.f;
      if (m & 8) r.w = 0.f;
    }
    out[node] = r;
  }
}

// d = mu * (merged sum of the velocity predictions), mu = 1/(number of incident patches on
// both sides), exactly as scatter_update_kernel; mask; x_corr = x~ + scale*d
__global__ void __launch_bounds__(256) halo_merge_scatter_kernel(
    int n, const int32_t* __restrict__ nodes, const int32_t* __restrict__ mptr,
    const int32_t* __restrict__ msrc, int npp, const float* __restrict__ Y,
    const float4* __restrict__ recv, const uint8_t* __restrict__ mask,
    const float4* __restrict__ xt, float scale, float4* __restrict__ d, float4* __restrict__ xc) {
  const int n_out = 3 * npp;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int node = __ldg(nodes + i);
    const int s0 = __ldg(mptr + i), e0 = __ldg(mptr + i + 1);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f;
    for (int j = s0; j < e0; ++j) {
      const int s = __ldg(msrc + j);
      float y0, y1, y2;
      if (s >= 0) {
        const int p = s / npp;
        const float* y = Y + (int64_t)p * n_out + 3 * (s - p * npp);
        y0 = __ldg(y);
        y1 = __ldg(y + 1);
        y2 = __ldg(y + 2);
      } else {
        const float4 v = __ldg(recv + (-1 - s));
        y0 = v.x;
        y1 = v.y;
        y2 = v.z;
      }
      a0 += y0;
      a1 += y1;
      a2 += y2;
    }
    const float mu = e0 > s0 ? 1.0f / (float)(e0 - s0) : 0.f;
    float4 dv = make_float4(0.f, mu * a0, mu * a1, mu * a2);
    const uint8_t m = mask ? mask[node] : 0;
    if (m & 2) dv.y = 0.f;
    if (m & 4) dv.z = 0.f;
    if (m & 8) dv.w = 0.f;
    if (d) d[node] = dv;
    if (xc) {
      const float4 x = __ldg(xt + node);
      xc[node] = make_float4(x.x, fmaf(scale, dv.y, x.y), fmaf(scale, dv.z, x.z),
                             fmaf(scale, dv.w, x.w));
    }
  }
}

static int32_t check_plan(const dnnmg_halo_plan_t* h, const char* who) {
  DNNMG_REQUIRE(h && h->n_nodes >= 0 && h->n_send >= 0, DNNMG_ERR_ARG, "%s: bad plan", who);
  DNNMG_REQUIRE(h->n_nodes == 0 || (h->nodes && h->merge_ptr && h->merge_src), DNNMG_ERR_ARG,
                "%s: incomplete plan", who);
  DNNMG_REQUIRE(h->n_send == 0 || h->send, DNNMG_ERR_ARG, "%s: plan without send list", who);
  return DNNMG_OK;
}

// ---- NCCL, resolved at run time -------------------------------------------------------------
// The library does not link libnccl: it binds the NCCL already loaded into the process (the
// one torch.distributed uses) or, failing that, dlopens libnccl.so.2, so a single NCCL serves
// the process.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
#define DNNMG_NCCL_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
  DNNMG_NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
  DNNMG_NCCL_SYM(CommInitRank, "ncclCommInitRank");
  DNNMG_NCCL_SYM(CommDestroy, "ncclCommDestroy");
  DNNMG_NCCL_SYM(CommCount, "ncclCommCount");
  DNNMG_NCCL_SYM(GroupStart, "ncclGroupStart");
  DNNMG_NCCL_SYM(GroupEnd, "ncclGroupEnd");
  DNNMG_NCCL_SYM(Send, "ncclSend");
  DNNMG_NCCL_SYM(Recv, "ncclRecv");
  DNNMG_NCCL_SYM(GetErrorString, "ncclGetErrorString");
#undef DNNMG_NCCL_SYM
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.CommCount &&
           api.GroupStart && api.GroupEnd && api.Send && api.Recv && api.GetErrorString;
  return api;
}

#define DNNMG_NCCL(call, what)                                                               \
  do {                                                                                       \
    ncclResult_t _r = (call);                                                                \
    if (_r != ncclSuccess)                                                                   \
      return ::dnnmg::set_error(DNNMG_ERR_CUDA, "%s: %s", what, nccl().GetErrorString(_r)); \
  } while (0)

}  // namespace dnnmg

using namespace dnnmg;

extern "C" {

int32_t dnnmg_halo_pack_rows(const dnnmg_halo_plan_t* h, const float* rows, float* sendbuf,
                             dnnmg_stream_t s) {
  int32_t st = check_plan(h, "halo_pack_rows");
  if (st) return st;
  if (h->n_send == 0) return DNNMG_OK;
  DNNMG_REQUIRE(rows && sendbuf, DNNMG_ERR_ARG, "halo_pack_rows: null argument");
  halo_pack_rows_kernel<<<grid_for(h->n_send, 256), 256, 0, as_stream(s)>>>(
      h->n_send, h->send, reinterpret_cast<const float4*>(rows), reinterpret_cast<float4*>(sendbuf));
  DNNMG_CHECK_LAUNCH("halo_pack_rows_kernel");
  return DNNMG_OK;
}

int32_t dnnmg_halo_pack_patch_rows(const dnnmg_halo_plan_t* h, const dnnmg_patchset_t* ps,
                                   const float* Y, float* sendbuf, dnnmg_stream_t s) {
  int32_t st = check_plan(h, "halo_pack_patch_rows");
  if (st) return st;
  DNNMG_REQUIRE(ps && ps->nodes_per_patch > 0, DNNMG_ERR_ARG, "halo_pack_patch_rows: no patch set");
  if (h->n_send == 0) return DNNMG_OK;
  DNNMG_REQUIRE(Y && sendbuf, DNNMG_ERR_ARG, "halo_pack_patch_rows: null argument");
  halo_pack_patch_kernel<<<grid_for(h->n_send, 256), 256, 0, as_stream(s)>>>(
      h->n_send, h->send, ps->nodes_per_patch, Y, reinterpret_cast<float4*>(sendbuf));
  DNNMG_CHECK_LAUNCH("halo_pack_patch_kernel");
  return DNNMG_OK;
}

int32_t dnnmg_halo_merge_rows(const dnnmg_halo_plan_t* h, const float* rows, const float* recvbuf,
                              const float* b, const uint8_t* mask, float* out, dnnmg_stream_t s) {
  int32_t st = check_plan(h, "halo_merge_rows");
  if (st) return st;
  if (h->n_nodes == 0) return DNNMG_OK;
  DNNMG_REQUIRE(rows && out && (recvbuf || h->n_send == 0), DNNMG_ERR_ARG,
                "halo_merge_rows: null argument");
  halo_merge_rows_kernel<<<grid_for(h->n_nodes, 256), 256, 0, as_stream(s)>>>(
      h->n_nodes, h->nodes, h->merge_ptr, h->merge_src, reinterpret_cast<const float4*>(rows),
      reinterpret_cast<const float4*>(recvbuf), reinterpret_cast<const float4*>(b), mask,
      reinterpret_cast<float4*>(out));
  DNNMG_CHECK_LAUNCH("halo_merge_rows_kernel");
  return DNNMG_OK;
}

int32_t dnnmg_halo_merge_scatter(const dnnmg_halo_plan_t* h, const dnnmg_patchset_t* ps,
                                 const float* Y, const float* recvbuf, const uint8_t* mask,
                                 const float* x_tilde, float scale, float* d, float* x_corr,
                                 dnnmg_stream_t s) {
  int32_t st = check_plan(h, "halo_merge_scatter");
  if (st) return st;
  DNNMG_REQUIRE(ps && ps->nodes_per_patch > 0, DNNMG_ERR_ARG, "halo_merge_scatter: no patch set");
  if (h->n_nodes == 0) return DNNMG_OK;
  DNNMG_REQUIRE(Y && (recvbuf || h->n_send == 0), DNNMG_ERR_ARG, "halo_merge_scatter: null argument");
  DNNMG_REQUIRE(!x_corr || x_tilde, DNNMG_ERR_ARG, "halo_merge_scatter: x_corr needs x_tilde");
  halo_merge_scatter_kernel<<<grid_for(h->n_nodes, 256), 256, 0, as_stream(s)>>>(
      h->n_nodes, h->nodes, h->merge_ptr, h->merge_src, ps->nodes_per_patch, Y,
      reinterpret_cast<const float4*>(recvbuf), mask, reinterpret_cast<const float4*>(x_tilde),
      scale, reinterpret_cast<float4*>(d), reinterpret_cast<float4*>(x_corr));
  DNNMG_CHECK_LAUNCH("halo_merge_scatter_kernel");
  return DNNMG_OK;
}

// ---- NCCL communicator and the neighbour exchange -------------------------------------------

int32_t dnnmg_nccl_available(void) { return nccl().ok ? 1 : 0; }

int32_t dnnmg_nccl_unique_id(void* id_out) {
  DNNMG_REQUIRE(id_out, DNNMG_ERR_ARG, "nccl_unique_id: null output");
  DNNMG_REQUIRE(nccl().ok, DNNMG_ERR_UNSUPPORTED, "nccl_unique_id: libnccl.so.2 not found");
  ncclUniqueId id;
  DNNMG_NCCL(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  memcpy(id_out, &id, sizeof(id));
  return DNNMG_OK;
}

int32_t dnnmg_nccl_comm_init(const void* id, int32_t nranks, int32_t rank, void** comm) {
  DNNMG_REQUIRE(id && comm && nranks > 0 && rank >= 0 && rank < nranks, DNNMG_ERR_ARG,
                "nccl_comm_init: bad argument");
  DNNMG_REQUIRE(nccl().ok, DNNMG_ERR_UNSUPPORTED, "nccl_comm_init: libnccl.so.2 not found");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  DNNMG_NCCL(nccl().CommInitRank(&c, nranks, uid, rank), "ncclCommInitRank");
  *comm = c;
  return DNNMG_OK;
}

int32_t dnnmg_nccl_comm_count(void* comm, int32_t* count) {
  DNNMG_REQUIRE(comm && count && nccl().ok, DNNMG_ERR_ARG, "nccl_comm_count: bad argument");
  int n = 0;
  DNNMG_NCCL(nccl().CommCount(static_cast<ncclComm_t>(comm), &n), "ncclCommCount");
  *count = n;
  return DNNMG_OK;
}

int32_t dnnmg_nccl_comm_destroy(void* comm) {
  if (!comm) return DNNMG_OK;
  DNNMG_REQUIRE(nccl().ok, DNNMG_ERR_UNSUPPORTED, "nccl_comm_destroy: libnccl.so.2 not found");
  DNNMG_NCCL(nccl().CommDestroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  return DNNMG_OK;
}

// One grouped exchange with both x-neighbours on `stream` (graph-capturable): side 0 = left
// (rank-1), side 1 = right (rank+1); count[side] float4 rows each way (0 / peer < 0: none).
int32_t dnnmg_halo_exchange(void* comm, const int32_t peer[2], const float* const send[2],
                            float* const recv[2], const int64_t count[2], dnnmg_stream_t s) {
  DNNMG_REQUIRE(comm && peer && send && recv && count, DNNMG_ERR_ARG, "halo_exchange: null argument");
  DNNMG_REQUIRE(nccl().ok, DNNMG_ERR_UNSUPPORTED, "halo_exchange: libnccl.so.2 not found");
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  cudaStream_t st = as_stream(s);
  DNNMG_NCCL(nccl().GroupStart(), "ncclGroupStart");
  for (int side = 0; side < 2; ++side) {
    if (peer[side] < 0 || count[side] == 0) continue;
    const size_t n = 4 * (size_t)count[side];
    ncclResult_t r = nccl().Send(send[side], n, ncclFloat32, peer[side], c, st);
    if (r == ncclSuccess) r = nccl().Recv(recv[side], n, ncclFloat32, peer[side], c, st);
    if (r != ncclSuccess) {
      nccl().GroupEnd();
      return set_error(DNNMG_ERR_CUDA, "halo_exchange: %s", nccl().GetErrorString(r));
    }
  }
  DNNMG_NCCL(nccl().GroupEnd(), "ncclGroupEnd");
  return DNNMG_OK;
}

// (a) before the MLP: pack the interface element vectors, exchange, merged residual rows
int32_t dnnmg_halo_pre(const dnnmg_slab_t* sl, void* comm, const float* elem, const float* b_prev,
                       const uint8_t* mask, float* r, dnnmg_stream_t s) {
  DNNMG_REQUIRE(sl && elem && r, DNNMG_ERR_ARG, "halo_pre: null argument");
  int32_t st;
  const float* send[2] = {sl->send[0], sl->send[1]};
  float* recv[2] = {sl->recv[0], sl->recv[1]};
  int64_t count[2];
  for (int side = 0; side < 2; ++side) {
    count[side] = sl->peer[side] >= 0 ? sl->cells[side].n_send : 0;
    if (count[side] && (st = dnnmg_halo_pack_rows(&sl->cells[side], elem, sl->send[side], s))) return st;
  }
  if (count[0] || count[1]) {
    DNNMG_REQUIRE(comm, DNNMG_ERR_ARG, "halo_pre: interfaces need a communicator");
    if ((st = dnnmg_halo_exchange(comm, sl->peer, send, recv, count, s))) return st;
  }
  for (int side = 0; side < 2; ++side)
    if (sl->peer[side] >= 0 &&
        (st = dnnmg_halo_merge_rows(&sl->cells[side], elem, sl->recv[side], b_prev, mask, r, s)))
      return st;
  return DNNMG_OK;
}

// (b) after the MLP: pack the interface patch predictions, exchange, merged scatter + update
int32_t dnnmg_halo_post(const dnnmg_slab_t* sl, void* comm, const dnnmg_patchset_t* ps,
                        const float* Y, const uint8_t* mask, const float* x_tilde, float scale,
                        float* d, float* x_corr, dnnmg_stream_t s) {
  DNNMG_REQUIRE(sl && ps && Y, DNNMG_ERR_ARG, "halo_post: null argument");
  int32_t st;
  const float* send[2] = {sl->send[0], sl->send[1]};
  float* recv[2] = {sl->recv[0], sl->recv[1]};
  int64_t count[2];
  for (int side = 0; side < 2; ++side) {
    count[side] = sl->peer[side] >= 0 ? sl->patches[side].n_send : 0;
    if (count[side] &&
        (st = dnnmg_halo_pack_patch_rows(&sl->patches[side], ps, Y, sl->send[side], s)))
      return st;
  }
  if (count[0] || count[1]) {
    DNNMG_REQUIRE(comm, DNNMG_ERR_ARG, "halo_post: interfaces need a communicator");
    if ((st = dnnmg_halo_exchange(comm, sl->peer, send, recv, count, s))) return st;
  }
  for (int side = 0; side < 2; ++side)
    if (sl->peer[side] >= 0 &&
        (st = dnnmg_halo_merge_scatter(&sl->patches[side], ps, Y, sl->recv[side], mask, x_tilde,
                                       scale, d, x_corr, s)))
      return st;
  return DNNMG_OK;
}

}  // extern "C"
