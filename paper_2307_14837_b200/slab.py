"""x-slab domain decomposition of the fine-level correction step.

The reference is single-process; this is the multi-GPU form of the same
step.  Rank r owns the level-0 cells with x-index in [a_r, b_r) and everything refined
from them: its coarse state, fine cells and patches.  Fine nodes on a slab interface plane
are incident to cells and patches of both neighbours.  Two exchanges per step complete
their values:

  (a) between the residual and the MLP: the raw element vectors of every interface
      (cell, local node) -> both ranks form r = b - A at the interface nodes;
  (b) after the MLP: the raw velocity predictions of every interface (patch, slot) ->
      both ranks form d = mu * sum and x_corr at the interface nodes.

The single-domain step sums each node's contributions in ascending GLOBAL cell id
(assembly.py:180-184) and ascending GLOBAL patch id (patch_ops.py:32-38); along an
interface those orders interleave the two sides (level-0 cells are numbered k, i, j;
children 8c+o).  A merge plan per side (``halo_plan``) lists each interface node's local
and received entries in that global order, so the interface values are bitwise equal on
both ranks and to the single-domain step.  The plans are built from lattice positions
alone: the neighbour's cells at an interface node are the mirror images of this rank's
across the plane, so no rank needs the global mesh or any setup communication.  Messages
at config 3: 64 x 64 interface fine cells x 9 face nodes = 36,864 float4 rows (590 KB) per
direction for (a), the same count for (b).

``SlabPartition`` is host-only (numpy): the local hierarchy with GLOBAL boundary tags, the
interface node lists, the merge plans, the global pressure pin.  ``SlabStep`` runs the local
kernels and the halo kernels through the C ABI.  Exchangers:
``NcclComm`` (the library's own NCCL communicator: send/recv to rank +-1 grouped on the
compute stream, dnnmg_halo_pre/post, graph-capturable), ``TorchDistExchanger``
(torch.distributed point-to-point; gloo stages through host memory) and
``InProcessExchanger`` (several slabs driven by one process, for single-GPU verification).
"""

import ctypes

import numpy as np

from . import mesh as meshmod, synthetic
from .space import FeSpace, no_slip

SIDES = ("left", "right")


def slab_ranges(n_x, world):
    """Contiguous level-0 x-ranges [a_r, b_r) of nearly equal size."""
    if n_x < world:
        raise ValueError(f"cannot split {n_x} x-cells over {world} ranks")
    edges = [(r * n_x) // world for r in range(world + 1)]
    return [(edges[r], edges[r + 1]) for r in range(world)]


def global_level0_vertices(lo, hi, n_cells, jitter_seed=None):
    """Level-0 vertices of the global box (x fastest), jittered as the single-domain build
    would be (synthetic.jitter_vertices draws per global interior vertex id)."""
    h = meshmod.build_template_mesh("box", extent_lo=lo, extent_hi=hi, n_cells=n_cells)
    V = h.levels[0].vertices
    if jitter_seed is not None:
        synthetic.jitter_vertices(V, n_cells, lo, hi, jitter_seed)
    return V


def global_is_box(V, n_cells, rtol=1e-13):
    """True when the global level-0 vertices (x fastest) form an axis-aligned tensor grid:
    every refined level then consists of axis-aligned boxes on every rank, and K2 may take its
    box form on all of them (as the single domain does)."""
    nx, ny, nz = (int(v) for v in n_cells)
    X = np.asarray(V, dtype=float).reshape(nz + 1, ny + 1, nx + 1, 3)
    tol = rtol * max(float(np.abs(X).max()), 1.0)
    return bool(np.abs(X[..., 0] - X[0, 0, :, 0][None, None, :]).max() <= tol
                and np.abs(X[..., 1] - X[0, :, 0, 1][None, :, None]).max() <= tol
                and np.abs(X[..., 2] - X[:, 0, 0, 2][:, None, None]).max() <= tol)


def global_cell_ids(lat, level, n0):
    """Global cell id of level-`level` cells with lattice index lat (n, 3) in a box of
    n0 = (NX, NY, NZ) level-0 cells: level-0 cells are numbered k, then i, j fastest
    (mesh.py:343-350), children 8c + o with o = ox + 2 oy + 4 oz (mesh.py:233-241)."""
    lat = np.asarray(lat, dtype=np.int64)
    cx, cy, cz = lat[:, 0], lat[:, 1], lat[:, 2]
    g = (cz >> level) * (n0[0] * n0[1]) + (cx >> level) * n0[1] + (cy >> level)
    for t in range(level - 1, -1, -1):
        g = 8 * g + ((cx >> t) & 1) + 2 * ((cy >> t) & 1) + 4 * ((cz >> t) & 1)
    return g


def cell_lattice(level_obj):
    """Global lattice index (n_cells, 3) of a (sub-box) level's cells."""
    return level_obj.lattice[level_obj.cells[:, 0]] + level_obj._offset


def halo_plan(nodes, csr_ptr, csr_idx, width, cell_lat, level, n0, plane):
    """Merge plan of one side for one quantity.

    nodes: interface node ids (agreed order); csr_ptr/csr_idx: node -> entries
    (cell*width + slot) of this rank; cell_lat: global lattice index of the local cells
    at `level`; plane: x cell index of the interface (cells with cx < plane lie left of it).
    Returns dict(nodes, send, merge_ptr, merge_src, counts, own_ids, remote_ids)."""
    nodes = np.asarray(nodes, dtype=np.int64)
    ptr = np.asarray(csr_ptr, dtype=np.int64)
    counts = ptr[nodes + 1] - ptr[nodes]
    total = int(counts.sum())
    node_of = np.repeat(np.arange(nodes.size), counts)
    off = np.zeros(nodes.size + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    ent = np.asarray(csr_idx, dtype=np.int64)[np.repeat(ptr[nodes], counts)
                                              + np.arange(total) - np.repeat(off[:-1], counts)]
    lat = cell_lat[ent // width]
    g_own = global_cell_ids(lat, level, n0)
    mir = lat.copy()
    mir[:, 0] = 2 * plane - 1 - mir[:, 0]
    g_rem = global_cell_ids(mir, level, n0)
    o_own = np.lexsort((g_own, node_of))
    o_rem = np.lexsort((g_rem, node_of))
    send = ent[o_own]
    # received entry q (the neighbour's message: nodes in order, its own ascending ids) is
    # the mirror of this rank's entry o_rem[q]
    ids = np.concatenate([g_own[o_own], g_rem[o_rem]])
    src = np.concatenate([send, -1 - np.arange(total)])
    row = np.concatenate([node_of[o_own], node_of[o_rem]])
    o = np.lexsort((ids, row))
    if np.any(np.diff(ids[o])[np.diff(row[o]) == 0] == 0):
        raise RuntimeError("halo plan: a global id appears on both sides of an interface")
    mptr = np.zeros(nodes.size + 1, dtype=np.int64)
    np.cumsum(2 * counts, out=mptr[1:])
    return dict(nodes=nodes, send=send, merge_ptr=mptr, merge_src=src[o], counts=counts,
                own_ids=g_own[o_own], remote_ids=g_rem[o_rem])


class SlabPartition:
    """One rank's part of an (L, J) patch split of a global box."""

    def __init__(self, lo, hi, n_cells, L, J, world, rank, jitter_seed=None, channel_tags=False,
                 bc_tags=(meshmod.WALL,)):
        self.world, self.rank, self.L, self.J = world, rank, L, J
        self.n0 = tuple(int(v) for v in n_cells)
        self.n_cells_global = self.n0
        self.a, self.b = slab_ranges(self.n0[0], world)[rank]
        V0 = global_level0_vertices(lo, hi, n_cells, jitter_seed)
        self.global_box = global_is_box(V0, n_cells)
        self.h = meshmod.build_subbox(V0, n_cells, (self.a, self.b), lo, hi, channel_tags)
        for _ in range(L + J):
            meshmod.refine_uniform(self.h)
        fl = L + J
        self.space = FeSpace(self.h, fl)
        self.patchset = meshmod.build_patches(self.h, L, J)
        # global lattice positions (doubled grid of each level) of the local Q2 nodes
        self.fine_pos = self._global_pos(fl)
        self.coarse_pos = self._global_pos(L)
        self.peer = {"left": rank - 1 if rank > 0 else -1,
                     "right": rank + 1 if rank < world - 1 else -1}
        self.iface, self.cell_plans, self.patch_plans = {}, {}, {}
        from .device import node_csr
        cptr, cidx = node_csr(self.space.cell_nodes)
        pptr, pidx = node_csr(self.patchset.node_table)
        lat_f = cell_lattice(self.h.levels[fl])
        lat_p = cell_lattice(self.h.levels[L + 1])       # patch p == level-(L+1) cell p
        for side, xcell in (("left", self.a), ("right", self.b)):
            if self.peer[side] < 0:
                continue
            xplane = 2 * xcell * 2 ** fl
            nodes = np.nonzero(self.fine_pos[:, 0] == xplane)[0]
            order = np.lexsort((self.fine_pos[nodes, 1], self.fine_pos[nodes, 2]))
            nodes = nodes[order]
            self.iface[side] = nodes
            self.cell_plans[side] = halo_plan(nodes, cptr, cidx, 27, lat_f, fl, self.n0,
                                              xcell * 2 ** fl)
            self.patch_plans[side] = halo_plan(nodes, pptr, pidx, self.patchset.nodes_per_patch,
                                               lat_p, L + 1, self.n0, xcell * 2 ** (L + 1))
        # constrained dofs: Dirichlet velocity (global tags) + the global pressure pin at
        # global node 0 = lattice (0,0,0) when the global box has no outflow (driver.py:56-65)
        self.mask = self.space.dirichlet_mask(bc_tags)
        if not channel_tags:
            origin = np.nonzero(np.all(self.fine_pos == 0, axis=1))[0]
            if origin.size:
                self.mask[4 * origin[0]] = True

    def _global_pos(self, level):
        lat = self.h._node_cache[level][2]          # local doubled-grid positions
        off = np.array([2 * self.a * 2 ** level, 0, 0], dtype=np.int64)
        return lat + off

    def global_fine_cells(self):
        """Global ids of the local fine cells (ascending: local order == global order)."""
        fl = self.L + self.J
        return global_cell_ids(cell_lattice(self.h.levels[fl]), fl, self.n0)

    def global_patches(self):
        return global_cell_ids(cell_lattice(self.h.levels[self.L + 1]), self.L + 1, self.n0)

    @property
    def n_patches(self):
        return len(self.patchset)


def global_index(global_h, level):
    """Map doubled-grid position key -> global node id of `level` of a global hierarchy."""
    global_h.scalar_nodes(level)
    lat = global_h._node_cache[level][2]
    ext = lat.max(axis=0) + 1
    keys = lat[:, 0] + ext[0] * (lat[:, 1] + ext[1] * lat[:, 2])
    lut = np.full(int(keys.max()) + 1, -1, dtype=np.int64)
    lut[keys] = np.arange(lat.shape[0])
    return lambda pos: lut[pos[:, 0] + ext[0] * (pos[:, 1] + ext[1] * pos[:, 2])]


# ---- exchangers -----------------------------------------------------------------------------

class TorchDistExchanger:
    """Neighbour exchange with torch.distributed point-to-point.  With the gloo backend the
    device messages are staged through host memory (CPU tests, or several ranks sharing one
    GPU); with NCCL they go device to device."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.host = dist.get_backend(group) == "gloo"

    def exchange(self, sends):
        """sends: {"left": tensor, "right": tensor} -> the neighbours' matching tensors."""
        import torch
        dist = self.dist
        recvs, ops, back = {}, [], {}
        for side, peer in (("left", self.rank - 1), ("right", self.rank + 1)):
            if side in sends:
                t = sends[side].contiguous()
                if self.host and t.is_cuda:
                    back[side] = t.device
                    t = t.cpu()
                recvs[side] = torch.empty_like(t)
                ops.append(dist.P2POp(dist.isend, t, peer, self.group))
                ops.append(dist.P2POp(dist.irecv, recvs[side], peer, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return {s: (v.to(back[s]) if s in back else v) for s, v in recvs.items()}


class InProcessExchanger:
    """Hands the interface buffers of neighbouring slabs to each other inside one process
    (slab r's "right" message is slab r+1's "left" one)."""

    @staticmethod
    def exchange_all(all_sends):
        out = [dict() for _ in all_sends]
        for r, sends in enumerate(all_sends):
            if "right" in sends:
                out[r + 1]["left"] = sends["right"].clone()
            if "left" in sends:
                out[r - 1]["right"] = sends["left"].clone()
        return out


class NcclComm:
    """The library's own NCCL communicator (dnnmg_nccl_comm_init).  Rank 0's unique id is
    broadcast through the torch.distributed store; the halo exchanges are then grouped
    ncclSend/ncclRecv with rank +-1 issued by the library on the compute stream
    (dnnmg_halo_pre / dnnmg_halo_post), capturable in a CUDA graph."""

    def __init__(self, rank, world, store=None, key="dnnmg_nccl_id"):
        from . import _lib
        self._lib = _lib
        if not _lib.load().dnnmg_nccl_available():
            raise RuntimeError("libnccl.so.2 is not available to libdnnmg_b200")
        self.rank, self.world = rank, world
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            _lib.call("dnnmg_nccl_unique_id", uid)
        if world > 1:
            if store is None:
                import torch.distributed as dist
                store = dist.distributed_c10d._get_default_store()
            if rank == 0:
                store.set(key, uid.raw)
            else:
                uid = ctypes.create_string_buffer(bytes(store.get(key)), 128)
        self.comm = ctypes.c_void_p()
        _lib.call("dnnmg_nccl_comm_init", uid, world, rank, ctypes.byref(self.comm))

    def count(self):
        n = ctypes.c_int32(0)
        self._lib.call("dnnmg_nccl_comm_count", self.comm, ctypes.byref(n))
        return n.value

    def close(self):
        if self.comm:
            self._lib.call("dnnmg_nccl_comm_destroy", self.comm)
            self.comm = ctypes.c_void_p()


# ---- the distributed step on the GPU ------------------------------------------------------------

class SlabStep:
    """CorrectionStep of one slab plus the two interface exchanges (merged in global order)."""

    def __init__(self, part, model, nu, k, bcs=None, alpha0=0.02, delta0=0.1, scale=1.0,
                 precision="fp32", t=0.0):
        import torch
        from . import _lib, device as dv
        from .step import CorrectionStep
        self._lib, self.dv, self.torch = _lib, dv, torch
        self.part = part
        bcs = bcs if bcs is not None else {meshmod.WALL: no_slip}
        self.step = CorrectionStep(part.h, part.L, part.J, model, nu, k, bcs=bcs, alpha0=alpha0,
                                   delta0=delta0, scale=scale, precision=precision,
                                   patchset=part.patchset, t=t, mask=part.mask,
                                   # one element-kernel form on every rank (bitwise equal to the
                                   # single domain): the box form only for an unjittered box
                                   k2_box=None if getattr(part, "global_box", True) else False)
        dev = dv.device()
        self._keep = []

        def plan_struct(p):
            if p is None:
                return _lib.HaloPlan(0, None, 0, None, None, None)
            arrs = [dv.upload(p[k], np.int32) for k in ("nodes", "send", "merge_ptr", "merge_src")]
            self._keep.extend(arrs)
            return _lib.HaloPlan(int(p["nodes"].size), dv.ptr(arrs[0]), int(p["send"].size),
                                 dv.ptr(arrs[1]), dv.ptr(arrs[2]), dv.ptr(arrs[3]))
        self.plans = {s: (plan_struct(part.cell_plans.get(s)), plan_struct(part.patch_plans.get(s)))
                      for s in SIDES}
        self.sendbuf, self.recvbuf = {}, {}
        for s in SIDES:
            if part.peer[s] < 0:
                continue
            n = max(self.plans[s][0].n_send, self.plans[s][1].n_send)
            self.sendbuf[s] = torch.zeros((n, 4), dtype=torch.float32, device=dev)
            self.recvbuf[s] = torch.zeros((n, 4), dtype=torch.float32, device=dev)
        self.struct = _lib.Slab((ctypes.c_int32 * 2)(part.peer["left"], part.peer["right"]),
                                (_lib.HaloPlan * 2)(self.plans["left"][0], self.plans["right"][0]),
                                (_lib.HaloPlan * 2)(self.plans["left"][1], self.plans["right"][1]),
                                (ctypes.c_void_p * 2)(*[self.sendbuf[s].data_ptr()
                                                        if s in self.sendbuf else None
                                                        for s in SIDES]),
                                (ctypes.c_void_p * 2)(*[self.recvbuf[s].data_ptr()
                                                        if s in self.recvbuf else None
                                                        for s in SIDES]))
        self.idx = {s: torch.as_tensor(n.astype(np.int64), device=dev) for s, n in part.iface.items()}

    def _sends(self, which):
        return {s: self.sendbuf[s][:self.plans[s][which].n_send] for s in self.sendbuf}

    def _land(self, recv, which):
        for s, t in recv.items():
            self.recvbuf[s][:self.plans[s][which].n_send].copy_(t)

    # ---- staged form: the exchange is the caller's (host exchangers, tests) ----
    def stage_residual(self, x_coarse, b_prev):
        """K1 + K2 locally, then this rank's interface element vectors (messages of (a))."""
        st, lib, dv = self.step, self._lib, self.dv
        s = dv.stream_handle()
        st.embed_into(x_coarse, st.x_tilde)
        lib.call("dnnmg_residual", ctypes.byref(st.lv), dv.ptr(st.x_tilde), dv.ptr(b_prev), None,
                 None, ctypes.byref(st.phys), dv.ptr(st.elem), dv.ptr(st.r), 1, s)
        for side in self.sendbuf:
            lib.call("dnnmg_halo_pack_rows", ctypes.byref(self.plans[side][0]), dv.ptr(st.elem),
                     dv.ptr(self.sendbuf[side]), s)
        self._b = b_prev
        return self._sends(0)

    def stage_predict(self, recv):
        """Merged interface residual, then K3, K4, K5 locally and this rank's interface patch
        predictions (messages of (b))."""
        st, lib, dv = self.step, self._lib, self.dv
        s = dv.stream_handle()
        self._land(recv, 0)
        for side in self.sendbuf:
            lib.call("dnnmg_halo_merge_rows", ctypes.byref(self.plans[side][0]), dv.ptr(st.elem),
                     dv.ptr(self.recvbuf[side]), dv.ptr(self._b), dv.ptr(st.mask_bits),
                     dv.ptr(st.r), s)
        st.predict_rows(s)
        lib.call("dnnmg_scatter_update", ctypes.byref(st.ps.struct), dv.ptr(st.Y),
                 dv.ptr(st.mask_bits), dv.ptr(st.x_tilde), ctypes.c_float(st.scale), dv.ptr(st.d),
                 dv.ptr(st.x_corr), s)
        for side in self.sendbuf:
            lib.call("dnnmg_halo_pack_patch_rows", ctypes.byref(self.plans[side][1]),
                     ctypes.byref(st.ps.struct), dv.ptr(st.Y), dv.ptr(self.sendbuf[side]), s)
        return self._sends(1)

    def stage_finish(self, recv):
        st, lib, dv = self.step, self._lib, self.dv
        s = dv.stream_handle()
        self._land(recv, 1)
        for side in self.sendbuf:
            lib.call("dnnmg_halo_merge_scatter", ctypes.byref(self.plans[side][1]),
                     ctypes.byref(st.ps.struct), dv.ptr(st.Y), dv.ptr(self.recvbuf[side]),
                     dv.ptr(st.mask_bits), dv.ptr(st.x_tilde), ctypes.c_float(st.scale),
                     dv.ptr(st.d), dv.ptr(st.x_corr), s)
        return st.x_corr

    # ---- fused form over the library's NCCL communicator ----
    def run(self, x_coarse, b_prev, exchanger, x_corr=None):
        """One distributed correction step.  exchanger: NcclComm (exchanges issued by the
        library on the current stream, no host synchronisation) or a host exchanger."""
        if not isinstance(exchanger, NcclComm):
            a = self.stage_residual(x_coarse, b_prev)
            b = self.stage_predict(exchanger.exchange(a))
            out = self.stage_finish(exchanger.exchange(b))
            if x_corr is not None:
                x_corr.copy_(out)
                return x_corr
            return out
        st, lib, dv = self.step, self._lib, self.dv
        out = st.x_corr if x_corr is None else x_corr
        s = dv.stream_handle()
        st.embed_into(x_coarse, st.x_tilde)
        lib.call("dnnmg_residual", ctypes.byref(st.lv), dv.ptr(st.x_tilde), dv.ptr(b_prev), None,
                 None, ctypes.byref(st.phys), dv.ptr(st.elem), dv.ptr(st.r), 1, s)
        lib.call("dnnmg_halo_pre", ctypes.byref(self.struct), exchanger.comm, dv.ptr(st.elem),
                 dv.ptr(b_prev), dv.ptr(st.mask_bits), dv.ptr(st.r), s)
        st.predict_rows(s)
        lib.call("dnnmg_scatter_update", ctypes.byref(st.ps.struct), dv.ptr(st.Y),
                 dv.ptr(st.mask_bits), dv.ptr(st.x_tilde), ctypes.c_float(st.scale), dv.ptr(st.d),
                 dv.ptr(out), s)
        lib.call("dnnmg_halo_post", ctypes.byref(self.struct), exchanger.comm,
                 ctypes.byref(st.ps.struct), dv.ptr(st.Y), dv.ptr(st.mask_bits),
                 dv.ptr(st.x_tilde), ctypes.c_float(st.scale), dv.ptr(st.d), dv.ptr(out), s)
        return out

    def stage_rhs(self, x, out=None):
        """Next-step fine RHS locally, then this rank's interface element vectors."""
        lib, dv, st = self._lib, self.dv, self.step
        self._rhs = st.rhs_next(x, out)
        s = dv.stream_handle()
        for side in self.sendbuf:
            lib.call("dnnmg_halo_pack_rows", ctypes.byref(self.plans[side][0]), dv.ptr(st.elem),
                     dv.ptr(self.sendbuf[side]), s)
        return self._sends(0)

    def finish_rhs(self, recv):
        lib, dv, st = self._lib, self.dv, self.step
        s = dv.stream_handle()
        self._land(recv, 0)
        for side in self.sendbuf:
            lib.call("dnnmg_halo_merge_rows", ctypes.byref(self.plans[side][0]), dv.ptr(st.elem),
                     dv.ptr(self.recvbuf[side]), None, None, dv.ptr(self._rhs), s)
        return self._rhs

    def rhs_next(self, x, exchanger, out=None):
        """Next-step fine RHS with the interface rows merged in global cell order."""
        lib, dv, st = self._lib, self.dv, self.step
        if isinstance(exchanger, NcclComm):
            out = st.rhs_next(x, out)
            lib.call("dnnmg_halo_pre", ctypes.byref(self.struct), exchanger.comm, dv.ptr(st.elem),
                     None, None, dv.ptr(out), dv.stream_handle())
            return out
        sends = self.stage_rhs(x, out)
        return self.finish_rhs(exchanger.exchange(sends) if sends else {})
