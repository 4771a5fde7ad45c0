"""x-slab domain decomposition of the fine-level correction step.

The reference is single-process; this is the multi-GPU form of
the same step.  Rank r owns the level-0 cells with x-index in [a_r, b_r) and
everything refined from them: its coarse state, fine cells and patches.  Fine
nodes on a slab interface plane belong to both neighbours.  Two exchanges per
step complete the interface values:

  (a) partial operator A_h(x~) at interface nodes (each side sums its own cells)
      -> both sides form r = b - (A_left + A_right) and re-apply the mask;
  (b) raw patch sums and patch counts at interface nodes
      -> both sides form d = (S_left + S_right) / (n_left + n_right).

Sums are taken left partial first on both ranks, so interface values are
bitwise identical on the two sides.  Messages are ~0.5 MB per direction at
config 3 (4,225 interface nodes x 16 B x 2), latency-bound over NVLink.

``SlabPartition`` is host-only (numpy): the local hierarchy with GLOBAL boundary
tags, the interface node lists ordered identically on both sides, the global
pressure pin.  ``SlabStep`` runs the local kernels through the C ABI and calls
an exchanger between the stages: ``TorchDistExchanger`` (torch.distributed P2P,
NCCL on GPUs / gloo on CPU) or ``InProcessExchanger`` (several slabs driven by
one process on one GPU, stage by stage, for single-GPU verification).
"""

import ctypes

import numpy as np

from . import mesh as meshmod, synthetic
from .space import FeSpace, no_slip


def slab_ranges(n_x, world):
    """Contiguous level-0 x-ranges [a_r, b_r) of nearly equal size."""
    if n_x < world:
        raise ValueError(f"cannot split {n_x} x-cells over {world} ranks")
    edges = [(r * n_x) // world for r in range(world + 1)]
    return [(edges[r], edges[r + 1]) for r in range(world)]


def global_level0_vertices(lo, hi, n_cells, jitter_seed=None):
    """Level-0 vertices of the global box (x fastest), jittered as the
    single-domain build would be (synthetic.jitter_vertices)."""
    h = meshmod.build_template_mesh("box", extent_lo=lo, extent_hi=hi, n_cells=n_cells)
    V = h.levels[0].vertices
    if jitter_seed is not None:
        synthetic.jitter_vertices(V, n_cells, lo, hi, jitter_seed)
    return V


class SlabPartition:
    """One rank's part of an (L, J) patch split of a global box."""

    def __init__(self, lo, hi, n_cells, L, J, world, rank, jitter_seed=None, channel_tags=False,
                 bc_tags=(meshmod.WALL,)):
        self.world, self.rank, self.L, self.J = world, rank, L, J
        self.n_cells_global = tuple(int(v) for v in n_cells)
        self.a, self.b = slab_ranges(self.n_cells_global[0], world)[rank]
        V0 = global_level0_vertices(lo, hi, n_cells, jitter_seed)
        self.h = meshmod.build_subbox(V0, n_cells, (self.a, self.b), lo, hi, channel_tags)
        for _ in range(L + J):
            meshmod.refine_uniform(self.h)
        fl = L + J
        self.space = FeSpace(self.h, fl)
        self.patchset = meshmod.build_patches(self.h, L, J)
        # global lattice positions (doubled grid of each level) of the local Q2 nodes
        self.fine_pos = self._global_pos(fl)
        self.coarse_pos = self._global_pos(L)
        xmax = 2 * self.b * 2 ** fl
        xmin = 2 * self.a * 2 ** fl
        self.iface = {}
        for side, xplane, present in (("left", xmin, rank > 0), ("right", xmax, rank < world - 1)):
            if not present:
                continue
            nodes = np.nonzero(self.fine_pos[:, 0] == xplane)[0]
            order = np.lexsort((self.fine_pos[nodes, 1], self.fine_pos[nodes, 2]))
            self.iface[side] = nodes[order]
        # constrained dofs: Dirichlet velocity (global tags) + the global pressure pin
        # at global node 0 = lattice (0,0,0) when the global box has no outflow (driver.py:56-65)
        self.mask = self.space.dirichlet_mask(bc_tags)
        if not channel_tags:
            origin = np.nonzero(np.all(self.fine_pos == 0, axis=1))[0]
            if origin.size:
                self.mask[4 * origin[0]] = True

    def _global_pos(self, level):
        lat = self.h._node_cache[level][2]          # local doubled-grid positions
        off = np.array([2 * self.a * 2 ** level, 0, 0], dtype=np.int64)
        return lat + off

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
    """Neighbour exchange with torch.distributed point-to-point (NCCL or gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def exchange(self, sends):
        """sends: {"left": tensor, "right": tensor} -> the neighbours' matching tensors."""
        import torch
        dist = self.dist
        recvs, ops = {}, []
        for side, peer in (("left", self.rank - 1), ("right", self.rank + 1)):
            if side in sends:
                recvs[side] = torch.empty_like(sends[side])
                ops.append(dist.P2POp(dist.isend, sends[side].contiguous(), peer, self.group))
                ops.append(dist.P2POp(dist.irecv, recvs[side], peer, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return recvs


class InProcessExchanger:
    """Hands the interface buffers of neighbouring slabs to each other inside one
    process (slab r's "right" message is slab r+1's "left" one)."""

    @staticmethod
    def exchange_all(all_sends):
        out = [dict() for _ in all_sends]
        for r, sends in enumerate(all_sends):
            if "right" in sends:
                out[r + 1]["left"] = sends["right"].clone()
            if "left" in sends:
                out[r - 1]["right"] = sends["left"].clone()
        return out


# ---- the distributed step on the GPU ------------------------------------------------------------

class SlabStep:
    """CorrectionStep of one slab plus the two interface exchanges."""

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
                                   patchset=part.patchset, t=t, mask=part.mask)
        dev = dv.device()
        self.idx = {s: torch.as_tensor(n.astype(np.int32), device=dev) for s, n in part.iface.items()}
        self.own = {s: torch.empty((n.size, 4), dtype=torch.float32, device=dev)
                    for s, n in part.iface.items()}

    # own_is_left: at my right interface I am the left owner
    @staticmethod
    def _left_owner(side):
        return 1 if side == "right" else 0

    def stage_residual(self, x_coarse, b_prev):
        """K1 + K2 locally, then this rank's partial operator at interface nodes."""
        st, lib, dv = self.step, self._lib, self.dv
        s = dv.stream_handle()
        st.embed_into(x_coarse, st.x_tilde)
        lib.call("dnnmg_residual", ctypes.byref(st.lv), dv.ptr(st.x_tilde), dv.ptr(b_prev), None,
                 None, ctypes.byref(st.phys), dv.ptr(st.elem), dv.ptr(st.r), 1, s)
        for side, idx in self.idx.items():
            lib.call("dnnmg_halo_operator", ctypes.byref(st.lv), dv.ptr(st.elem), dv.ptr(idx),
                     idx.numel(), dv.ptr(self.own[side]), s)
        self._b = b_prev
        return dict(self.own)

    def stage_predict(self, recv_operator):
        """Interface residual from both partials, then K3, K4, K5 locally and this
        rank's raw patch sums at interface nodes."""
        st, lib, dv = self.step, self._lib, self.dv
        s = dv.stream_handle()
        for side, idx in self.idx.items():
            lib.call("dnnmg_halo_residual", dv.ptr(idx), idx.numel(), dv.ptr(self._b),
                     dv.ptr(self.own[side]), dv.ptr(recv_operator[side]), self._left_owner(side),
                     dv.ptr(st.mask_bits), dv.ptr(st.r), s)
        st.predict_rows(s)
        lib.call("dnnmg_scatter_update", ctypes.byref(st.ps.struct), dv.ptr(st.Y),
                 dv.ptr(st.mask_bits), dv.ptr(st.x_tilde), ctypes.c_float(st.scale), dv.ptr(st.d),
                 dv.ptr(st.x_corr), s)
        for side, idx in self.idx.items():
            lib.call("dnnmg_halo_scatter_sums", ctypes.byref(st.ps.struct), dv.ptr(st.Y),
                     dv.ptr(idx), idx.numel(), dv.ptr(self.own[side]), s)
        return dict(self.own)

    def stage_finish(self, recv_sums):
        st, lib, dv = self.step, self._lib, self.dv
        s = dv.stream_handle()
        for side, idx in self.idx.items():
            lib.call("dnnmg_halo_scatter_apply", dv.ptr(idx), idx.numel(), dv.ptr(self.own[side]),
                     dv.ptr(recv_sums[side]), self._left_owner(side), dv.ptr(st.mask_bits),
                     dv.ptr(st.x_tilde), ctypes.c_float(st.scale), dv.ptr(st.d), dv.ptr(st.x_corr), s)
        return st.x_corr

    def run(self, x_coarse, b_prev, exchanger):
        """One distributed correction step with a TorchDistExchanger."""
        a = self.stage_residual(x_coarse, b_prev)
        b = self.stage_predict(exchanger.exchange(a))
        return self.stage_finish(exchanger.exchange(b))

    def rhs_next(self, x, exchanger, out=None):
        """Next-step fine RHS with the interface partial sums completed."""
        lib, dv, st = self._lib, self.dv, self.step
        out = st.rhs_next(x, out)
        s = dv.stream_handle()
        lv = st.level.struct()
        for side, idx in self.idx.items():
            lib.call("dnnmg_halo_operator", ctypes.byref(lv), dv.ptr(st.elem), dv.ptr(idx),
                     idx.numel(), dv.ptr(self.own[side]), s)
        recv = exchanger.exchange(dict(self.own))
        for side, idx in self.idx.items():
            lib.call("dnnmg_halo_sum", dv.ptr(idx), idx.numel(), dv.ptr(self.own[side]),
                     dv.ptr(recv[side]), self._left_owner(side), dv.ptr(out), s)
        return out
