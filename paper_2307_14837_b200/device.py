"""Device-resident index tables and the thin calls into libdnnmg_b200.

PyTorch is used only as plumbing here: CUDA memory, the current stream and
host<->device copies.  Every arithmetic operation on the correction path is a
kernel of libdnnmg_b200.so called through its C ABI (``_lib``); there is no
PyTorch or numpy fallback, and a missing library or GPU raises.

Tables are uploaded once per host object (hierarchy level, PatchSet, model)
and cached on that object, so repeated API calls only move the vectors.
"""

import ctypes
import os

import numpy as np
import torch

from . import _lib

ALPHA0, DELTA0 = 0.02, 0.1


def device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2307_14837_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def nbytes(t):
    return 0 if t is None else int(t.numel() * t.element_size())


def f32(x):
    """numpy / torch -> contiguous float32 CUDA tensor."""
    dev = device()
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(dev)


def upload(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).to(device())


def upload_opt(a, dtype=np.int32):
    return None if a is None else upload(a, dtype)


def like_input(t, ref):
    """Return a device result in the caller's convention: numpy float64 for numpy
    inputs (the reference's dtype), the CUDA tensor otherwise."""
    if isinstance(ref, torch.Tensor):
        return t
    return t.double().cpu().numpy()


def _cache(obj, key):
    store = obj.__dict__.setdefault("_b200_device", {})
    return store, key


def node_csr(table):
    """CSR node -> flat (row*width + slot) entries, rows ascending per node."""
    flat = np.asarray(table, dtype=np.int64).reshape(-1)
    order = np.argsort(flat, kind="stable")
    counts = np.bincount(flat, minlength=int(flat.max()) + 1 if flat.size else 0)
    ptr_ = np.zeros(counts.size + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr_[1:])
    return ptr_, order


def visit_order(ptr_, idx):
    """Visiting order of the owner-computes node passes (K2's node sum, K5): nodes by
    descending first incident row (their lowest cell / patch), ties by descending id.
    Each node then meets the element vectors / Y rows of its own cells together (the
    vertex nodes, numbered first, no longer sweep all of them at kernel start), and the
    rows the producing kernel wrote last, still in L2, are read first.  Any order gives
    the same bits.  DNNMG_NODE_ORDER=ascending|forward selects ids / ascending first row
    (diagnostic A/B)."""
    mode = os.environ.get("DNNMG_NODE_ORDER", "")
    if mode == "ascending":
        return None
    ptr_ = np.asarray(ptr_, dtype=np.int64)
    n = ptr_.size - 1
    idx = np.asarray(idx)
    first = np.full(n, -1, dtype=np.int64)
    has = ptr_[1:] > ptr_[:-1]
    first[has] = idx[ptr_[:-1][has]]
    order = np.lexsort((np.arange(n), first))
    return order if mode == "forward" else order[::-1].copy()


def visit_csr(ptr_, idx, order):
    """The CSR rows in visiting order (row i = the row of node order[i]), or (None, None)
    without an order."""
    if order is None:
        return None, None
    ptr_ = np.asarray(ptr_, dtype=np.int64)
    counts = (ptr_[1:] - ptr_[:-1])[order]
    vptr = np.zeros(order.size + 1, dtype=np.int64)
    np.cumsum(counts, out=vptr[1:])
    src = np.repeat(ptr_[:-1][order] - vptr[:-1], counts) + np.arange(vptr[-1])
    return vptr, np.asarray(idx)[src]


TILE_ROWS = 128  # patches per tensor-core MLP tile (kTcM in csrc/mlp_tc.cu)


def tile_tables(table, rows=TILE_ROWS):
    """Distinct nodes of every `rows`-patch tile of a node table, for the staged fused
    gather of the MLP kernel: (cap, nodes [n_tiles][cap] int32 ascending, count [n_tiles],
    slot [n_tiles*rows][npp] uint16 with nodes[t][slot[p][s]] == table[p][s]).  Rows past
    the last patch repeat the last row.  Returns None when a tile has more than 65535
    distinct nodes (not representable in uint16)."""
    table = np.asarray(table, dtype=np.int64)
    n, npp = table.shape
    if n == 0:
        return None
    T = (n + rows - 1) // rows
    pad = T * rows - n
    a = np.concatenate([table, np.repeat(table[-1:], pad, 0)]) if pad else table
    a = a.reshape(T, rows * npp)
    order = np.argsort(a, axis=1, kind="stable")
    srt = np.take_along_axis(a, order, 1)
    first = np.ones(srt.shape, dtype=bool)
    first[:, 1:] = srt[:, 1:] != srt[:, :-1]
    rank = np.cumsum(first, axis=1) - 1
    count = rank[:, -1] + 1
    if count.max() > 65535:
        return None
    cap = int((count.max() + 7) // 8 * 8)
    nodes = np.zeros((T, cap), dtype=np.int32)
    ti, pos = np.nonzero(first)
    nodes[ti, rank[ti, pos]] = srt[ti, pos]
    nodes[:, :] = np.where(np.arange(cap)[None, :] < count[:, None], nodes, nodes[:, :1])
    slot = np.empty_like(rank)
    np.put_along_axis(slot, order, rank, 1)
    return cap, nodes, count.astype(np.int32), slot.reshape(T * rows, npp).astype(np.uint16)


def dof_mask_bits(mask, n_nodes):
    """bool dof mask -> per-node bit field (bit c <=> dof 4n+c constrained)."""
    if mask is None:
        return None
    m = np.asarray(mask, dtype=bool).reshape(n_nodes, 4)
    return (m.astype(np.uint8) * np.array([1, 2, 4, 8], dtype=np.uint8)).sum(1).astype(np.uint8)


def cell_diameters(vertices, cells, chunk=1 << 16):
    """h_T = largest distance between two cell corners (assembly.py:99-103)."""
    out = np.empty(cells.shape[0])
    for s in range(0, cells.shape[0], chunk):
        C = vertices[cells[s:s + chunk]]
        d2 = ((C[:, :, None, :] - C[:, None, :, :]) ** 2).sum(-1)
        out[s:s + chunk] = np.sqrt(d2.max(axis=(1, 2)))
    return out


def lattice_table(src, n_coarse_cells):
    """lat[C][25 pz + 5 py + px] = fine node whose first-appearance parent is C and whose
    position in C's refined 5 x 5 x 5 lattice is (px, py, pz) (src = C*216 + o*27 + a: child
    octant o, local Q2 node a; space.py:117-165), else -1."""
    src = np.asarray(src, dtype=np.int64)
    C, oa = src // 216, src % 216
    o, a = oa // 27, oa % 27
    px = 2 * (o & 1) + a % 3
    py = 2 * ((o >> 1) & 1) + (a // 3) % 3
    pz = 2 * (o >> 2) + a // 9
    lat = np.full((n_coarse_cells, 125), -1, dtype=np.int64)
    lat[C, 25 * pz + 5 * py + px] = np.arange(src.size)
    return lat


class DeviceProlong:
    """K1 tables for level -> level+1."""

    def __init__(self, hierarchy, level):
        from .space import prolongation_source
        _, ctab = hierarchy.scalar_nodes(level)
        src = prolongation_source(hierarchy, level)
        self.ctab = upload(ctab, np.int32)
        self.src = upload(src, np.int32)
        self.n_fine = int(src.size)
        self.n_coarse_nodes = int(hierarchy.scalar_nodes(level)[0].shape[0])
        # owner lists: fine nodes grouped by their first-appearance parent cell
        parent = src // 216
        order = np.argsort(parent, kind="stable")
        counts = np.bincount(parent, minlength=ctab.shape[0])
        optr = np.zeros(ctab.shape[0] + 1, dtype=np.int64)
        np.cumsum(counts, out=optr[1:])
        self.owner_ptr = upload(optr, np.int32)
        self.owner_order = order                      # host copy (owner-ordered bc codes)
        self.owner_node = upload(order, np.int32)
        self.owner_code = upload(src[order] % 216, np.uint8)
        # lattice form: the owned fine node at every position of each parent's 5 x 5 x 5 lattice
        self.lat_host = lattice_table(src, int(ctab.shape[0]))
        self.lat_node = upload(self.lat_host, np.int32)
        self.struct = _lib.Prolong(self.n_fine, int(ctab.shape[0]), ptr(self.ctab), ptr(self.src),
                                   ptr(self.owner_ptr), ptr(self.owner_node), ptr(self.owner_code),
                                   ptr(self.lat_node))

    def lattice_with_codes(self, code):
        """lat_node with the Dirichlet code of every owned node in bits 29-30
        (dnnmg_dirichlet_t.lat_node_bc), or None when the node ids do not leave room."""
        if self.n_fine >= 1 << 29:
            return None
        lat = self.lat_host
        out = lat.copy()
        own = lat >= 0
        out[own] = lat[own] | (np.asarray(code, dtype=np.int64)[lat[own]] << 29)
        return out.astype(np.int32)

    @staticmethod
    def get(hierarchy, level):
        store, key = _cache(hierarchy, ("prolong", level))
        if key not in store:
            store[key] = DeviceProlong(hierarchy, level)
        return store[key]


class DeviceRestrict:
    """K6 tables for level+1 -> level: P^T as a coarse-node CSR (rows ascending fine node).
    The cell scratch is shared per (hierarchy, level): restrictions of one level are
    ordered on the caller's current stream."""

    def __init__(self, hierarchy, level):
        from .space import prolongation_matrix
        PT = prolongation_matrix(hierarchy, level).T.tocsr()
        PT.sort_indices()
        self.n_coarse, self.n_fine = int(PT.shape[0]), int(PT.shape[1])
        self.ptr = upload(PT.indptr, np.int32)
        self.fine = upload(PT.indices, np.int32)
        self.w = upload(PT.data, np.float32)   # dyadic weights: exact in fp32
        # owner-computes form: K1's owner lists plus the coarse node -> (cell, a) CSR
        # (env DNNMG_RESTRICT_CSR=1 keeps the P^T CSR form)
        P = DeviceProlong.get(hierarchy, level)
        ctab = hierarchy.scalar_nodes(level)[1]
        cp, ci = node_csr(ctab)
        self.cell_ptr = upload(cp, np.int32)
        self.cell_idx = upload(ci, np.int32)
        self.n_cells = int(ctab.shape[0])
        self.scratch = torch.empty(self.n_cells * 27 * 4, dtype=torch.float32, device=device())
        own = not os.environ.get("DNNMG_RESTRICT_CSR")
        self.struct = _lib.Restrict(self.n_coarse, self.n_fine, ptr(self.ptr), ptr(self.fine),
                                    ptr(self.w), self.n_cells if own else 0, ptr(P.ctab),
                                    ptr(P.owner_ptr) if own else None, ptr(P.owner_node),
                                    ptr(P.owner_code), ptr(self.cell_ptr), ptr(self.cell_idx),
                                    ptr(self.scratch))

    @staticmethod
    def get(hierarchy, level):
        store, key = _cache(hierarchy, ("restrict", level))
        if key not in store:
            store[key] = DeviceRestrict(hierarchy, level)
        return store[key]


def restrict_vector(hierarchy, b, level_fine, levels_down=1):
    """b_coarse = (P^T)^levels_down b on the device (space.py:188-196)."""
    v = f32(b)
    lvl = level_fine
    for _ in range(levels_down):
        R = DeviceRestrict.get(hierarchy, lvl - 1)
        if v.numel() != 4 * R.n_fine:
            raise ValueError(f"vector length {v.numel()} does not match level {lvl} "
                             f"({4 * R.n_fine} dofs)")
        out = torch.empty(4 * R.n_coarse, dtype=torch.float32, device=v.device)
        _lib.call("dnnmg_restrict", ctypes.byref(R.struct), ptr(v), ptr(out), stream_handle())
        v = out
        lvl -= 1
    return like_input(v, b)


_K2TC_CONST = {}


def k2tc_constants():
    """The tensor-core K2 constant operand image (one per device, written once)."""
    dev = torch.cuda.current_device()
    if dev not in _K2TC_CONST:
        n = int(_lib.load().dnnmg_k2tc_constants_bytes())
        buf = torch.empty(n, dtype=torch.uint8, device=device())
        _lib.call("dnnmg_k2tc_constants", ptr(buf), stream_handle())
        _K2TC_CONST[dev] = buf
    return _K2TC_CONST[dev]


def geometry_kind(vertices, cells, rtol=1e-10, chunk=1 << 18):
    """2 when every hexahedron is an axis-aligned box, 1 when every one is a parallelepiped
    (x fastest corner order) -- their isoparametric maps are affine (the Q2 nodes of this mesh
    code sit at the trilinear points), J is constant over the Gauss points and, for 2,
    diagonal -- else 0 (e.g. a jittered mesh)."""
    V = np.asarray(vertices, dtype=float)
    C = np.asarray(cells)
    kind = 2
    for s in range(0, C.shape[0], chunk):
        X = V[C[s:s + chunk]]
        h = np.abs(X[:, 7] - X[:, 0]).max(axis=1, keepdims=True) + 1e-300
        for axis, (e, pairs) in enumerate(((1, ((3, 2), (5, 4), (7, 6))), (2, ((3, 1), (6, 4), (7, 5))),
                                           (4, ((5, 1), (6, 2), (7, 3))))):
            d0 = X[:, e] - X[:, 0]
            for a, b in pairs:
                if np.any(np.abs(X[:, a] - X[:, b] - d0) > rtol * h):
                    return 0
            off = np.delete(d0, axis, axis=1)
            if np.any(off != 0.0):
                kind = 1
    return kind


def k2_tensor_cores(geo_kind):
    """Element kernel of K2 for a level.  The tensor-core one (csrc/residual_tc.cu) is opt-in
    (DNNMG_K2=tc, affine or per-point geometry): at config 3 it runs at parity with the SIMT
    kernel (1.00 vs 0.96 ms; per-point geometry 1.19 ms) with a ~2.5x larger (in-gate)
    residual error, so the SIMT kernel stays the default (K2)."""
    return os.environ.get("DNNMG_K2", "") == "tc"


class DeviceLevel:
    """K2 tables of one level: cell nodes, fp64 coordinates, h_T, node->cell CSR."""

    def __init__(self, space):
        h = space.hierarchy
        lvl = h.levels[space.level]
        self.n_nodes = int(space.n_nodes)
        self.n_cells = int(space.cell_nodes.shape[0])
        self.cell_nodes = upload(space.cell_nodes, np.int32)
        self.coords = upload(space.nodes, np.float64)
        self.h_T_host = cell_diameters(lvl.vertices, lvl.cells)
        self.h_T = upload(self.h_T_host, np.float32)
        p, idx = node_csr(space.cell_nodes)
        self.csr_ptr = upload(p, np.int32)
        self.csr_idx = upload(idx, np.int32)
        order = visit_order(p, idx)
        self.order = upload_opt(order)
        vp, vi = visit_csr(p, idx, order)
        self.vptr, self.vidx = upload_opt(vp), upload_opt(vi)
        self.elem = None
        self.geo_kind = geometry_kind(lvl.vertices, lvl.cells)
        self.affine = self.geo_kind > 0
        self.tc_geo = None

    def struct(self, dof_mask=None, geometry=False, tc=None, box=None):
        """geometry: with the per-mesh geometry -- the per-cell box record when every cell is an
        axis-aligned box (box=False forces the per-point cache), else the per-point cache.
        tc: use the tensor-core element kernel (default: with the geometry cache present,
        k2_tensor_cores)."""
        tc = geometry and k2_tensor_cores(self.geo_kind) if tc is None else tc
        box = self.geometry_box() if (geometry and not tc and box is not False) else None
        lv = _lib.Level(self.n_nodes, self.n_cells, ptr(self.cell_nodes), ptr(self.coords),
                        ptr(self.h_T), ptr(self.csr_ptr), ptr(self.csr_idx), ptr(dof_mask),
                        ptr(self.geometry()) if ((geometry and box is None) or tc) else None,
                        ptr(self.order), None, None, 0, ptr(self.vptr), ptr(self.vidx),
                        ptr(box))
        if tc:
            lv.tc_const = ptr(k2tc_constants())
            lv.tc_geo = ptr(self.geometry_tc())
            lv.tc_geo_affine = int(self.geo_kind)
        return lv

    def geometry_tc(self):
        """The geometry in the tensor-core kernel's layout: per-cell affine records for an
        affine mesh, else the per-point cache by 128-cell tiles."""
        if self.tc_geo is None:
            lv = _lib.Level(self.n_nodes, self.n_cells, ptr(self.cell_nodes), ptr(self.coords),
                            ptr(self.h_T), ptr(self.csr_ptr), ptr(self.csr_idx), None,
                            ptr(self.geometry()), None, None, None, 0)
            n = int(_lib.load().dnnmg_level_geometry_tc_floats(ctypes.byref(lv), int(self.affine)))
            self.tc_geo = torch.empty(max(n, 4), dtype=torch.float32, device=device())
            _lib.call("dnnmg_level_geometry_tc", ctypes.byref(lv), ptr(self.tc_geo),
                      int(self.affine), stream_handle())
        return self.tc_geo

    def geometry(self):
        """Per-mesh cache of J^-1 and w at every (cell, Gauss point) (2,560 B per cell),
        computed once in fp64 on the device (the reference's GeometryCache)."""
        if getattr(self, "geo_q", None) is None:
            self.geo_q = torch.empty(self.n_cells * 640, dtype=torch.float32, device=device())
            _lib.call("dnnmg_level_geometry", ctypes.byref(self.struct()), ptr(self.geo_q),
                      stream_handle())
        return self.geo_q

    def geometry_box(self):
        """Per-cell (1/hx, 1/hy, 1/hz, det J) when every cell of the level is an axis-aligned
        box with its Q2 nodes on the tri-quadratic lattice (checked on the device in fp64), else
        None.  K2 then takes its box form: J^-1 diagonal and constant over a cell."""
        if not hasattr(self, "geo_box"):
            self.geo_box = None
            if self.n_cells:
                rec = torch.empty(self.n_cells * 4, dtype=torch.float32, device=device())
                bad = torch.zeros(1, dtype=torch.int32, device=device())
                lv = _lib.Level(self.n_nodes, self.n_cells, ptr(self.cell_nodes), ptr(self.coords),
                                ptr(self.h_T), ptr(self.csr_ptr), ptr(self.csr_idx))
                _lib.call("dnnmg_level_geometry_box", ctypes.byref(lv), ptr(rec), ptr(bad),
                          stream_handle())
                if int(bad.item()) == 0:
                    self.geo_box = rec
        return self.geo_box

    def scratch(self):
        """Element-vector scratch shared by the reference-API calls on this level
        (assembly.Assembler), which are stream-ordered on the caller's current stream;
        CorrectionStep owns its own."""
        if self.elem is None:
            self.elem = torch.empty(self.n_cells * 27 * 4, dtype=torch.float32, device=device())
        return self.elem

    @staticmethod
    def get(space):
        store, key = _cache(space.hierarchy, ("level", space.level))
        if key not in store:
            store[key] = DeviceLevel(space)
        return store[key]


class DevicePatchSet:
    """K3/K5 tables: node table, geometry rows, node->(patch, slot) CSR."""

    def __init__(self, ps):
        self.n_patches = int(ps.node_table.shape[0])
        self.npp = int(ps.nodes_per_patch)
        self.n_geo = int(ps.n_geo)
        self.n_nodes = int(ps.mu.shape[0] // 4)
        self.node_table = upload(ps.node_table, np.int32)
        self.geom = upload(ps.geom_table, np.float32)
        p, idx = node_csr(ps.node_table)
        if p.size - 1 != self.n_nodes:
            raise RuntimeError("patch union does not cover the fine level")
        self.csr_ptr = upload(p, np.int32)
        self.csr_idx = upload(idx, np.int32)
        order = visit_order(p, idx)
        self.order = upload_opt(order)
        vp, vi = visit_csr(p, idx, order)
        self.vptr, self.vidx = upload_opt(vp), upload_opt(vi)
        tt = tile_tables(ps.node_table)
        self.tile_cap = 0
        self.tile_nodes = self.tile_count = self.tile_slot = None
        if tt is not None:
            self.tile_cap = tt[0]
            self.tile_nodes = upload(tt[1], np.int32)
            self.tile_count = upload(tt[2], np.int32)
            # uint16 has no torch dtype on every build: ship the raw bytes as int16
            self.tile_slot = upload(tt[3].view(np.int16), np.int16)
        self.struct = _lib.PatchSet(self.n_patches, self.npp, self.n_geo, self.n_nodes,
                                    ptr(self.node_table), ptr(self.geom), ptr(self.csr_ptr),
                                    ptr(self.csr_idx), self.tile_cap, ptr(self.tile_nodes),
                                    ptr(self.tile_count), ptr(self.tile_slot),
                                    ptr(self.order), ptr(self.vptr), ptr(self.vidx))

    @staticmethod
    def get(ps):
        store, key = _cache(ps, "patchset")
        if key not in store:
            store[key] = DevicePatchSet(ps)
        return store[key]


def tc_fused_supported(arch):
    """Widths of the fused per-tile tensor-core kernel (csrc/mlp_tc.cu, mlp_tc_supported);
    other widths run on the layer-major kernel (csrc/mlp_layer.cu)."""
    return arch.n_hidden in (128, 256) and arch.n_in <= 256 and arch.n_out <= arch.n_hidden


class DeviceModel:
    """Eval-mode MlpModel on the device (net.py:54-159), BN folded to scale/shift."""

    def __init__(self, model, precision="fp32"):
        from .net import effective_precision
        arch = model.arch
        self.arch = arch
        # f16x3 needs bounded activations: relu models fall back to tf32x3 (net.py docstring)
        self.requested_precision = precision
        precision = effective_precision(model.activation, precision)
        if precision != self.requested_precision:
            import warnings
            warnings.warn(f"precision {self.requested_precision} needs a bounded activation; "
                          f"the {model.activation} model runs in {precision}", stacklevel=2)
        self.precision = precision
        self.W = [f32(np.asarray(w, dtype=np.float64)) for w in model.W]
        scale, shift = [], []
        for i in range(arch.depth):
            s = np.asarray(model.gamma[i], float) / np.sqrt(np.asarray(model.running_var[i], float)
                                                            + model.bn_eps)
            scale.append(s)
            shift.append(np.asarray(model.beta[i], float) - np.asarray(model.running_mean[i], float) * s)
        self.scale = f32(np.concatenate(scale))
        self.shift = f32(np.concatenate(shift))
        self.in_mean = f32(np.asarray(model.input_mean, float))
        self.in_std = f32(np.asarray(model.input_std, float))
        Ws = (ctypes.c_void_p * _lib.MAX_LAYERS)(*([w.data_ptr() for w in self.W]
                                                  + [0] * (_lib.MAX_LAYERS - len(self.W))))
        act = _lib.ACT_TANH if model.activation == "tanh" else _lib.ACT_RELU
        self.struct = _lib.Mlp(arch.n_in, arch.n_hidden, arch.depth, arch.n_out, act,
                               _lib.PRECISIONS[precision], Ws, ptr(self.scale), ptr(self.shift),
                               ptr(self.in_mean), ptr(self.in_std), None)
        self.packed = None
        if precision != "fp32":
            nbytes = ctypes.c_int64(0)
            _lib.call("dnnmg_mlp_packed_bytes", ctypes.byref(self.struct), ctypes.byref(nbytes))
            self.packed = torch.empty(max(int(nbytes.value), 16), dtype=torch.uint8, device=device())
            self.struct.packed = ptr(self.packed)
            _lib.call("dnnmg_mlp_pack", ctypes.byref(self.struct), ptr(self.packed), stream_handle())

        self._ws = None

    def workspace_bytes(self, n_rows):
        """Bytes of the layered tensor-core kernel's workspace for n_rows (0: not needed)."""
        nbytes = ctypes.c_int64(0)
        _lib.call("dnnmg_mlp_workspace_bytes", ctypes.byref(self.struct), int(n_rows),
                  ctypes.byref(nbytes))
        return int(nbytes.value)

    def workspace(self, n_rows):
        """The model's shared workspace for the drop-in net.forward calls (stream-ordered on
        the caller's current stream; None when not needed), grown on demand and kept.
        CorrectionStep allocates its own (new_workspace)."""
        n = self.workspace_bytes(n_rows)
        if n == 0:
            return None
        if self._ws is None or self._ws.numel() < n:
            self._ws = torch.empty(n, dtype=torch.uint8, device=device())
        return self._ws

    def new_workspace(self, n_rows):
        """A workspace owned by the caller (None when not needed)."""
        n = self.workspace_bytes(n_rows)
        return None if n == 0 else torch.empty(n, dtype=torch.uint8, device=device())

    def forward(self, X, n_rows, Y):
        ws = self.workspace(n_rows)
        _lib.call("dnnmg_mlp_forward_ws", ctypes.byref(self.struct), ptr(X), int(n_rows), ptr(Y),
                  ptr(ws), nbytes(ws), stream_handle())


def dirichlet_codes(space, t, bcs):
    """(bc_code uint8 [n], bc_values float32 [n,3] or None) of apply_dirichlet at t."""
    code = np.zeros(space.n_nodes, dtype=np.uint8)
    vals = None
    for tag, fn in bcs.items():
        nodes = space.nodes_with_tag(tag)
        if nodes.size == 0 or fn is None:
            continue
        v = np.asarray(fn(t, space.nodes[nodes]), dtype=float).reshape(nodes.size, 3)
        if not np.any(v):
            code[nodes] = 1
        else:
            if vals is None:
                vals = np.zeros((space.n_nodes, 3), dtype=np.float32)
            code[nodes] = 2
            vals[nodes] = v
    return code, vals


class DeviceDirichlet:
    def __init__(self, space, t, bcs):
        code, vals = dirichlet_codes(space, t, bcs)
        self.code = upload(code, np.uint8)
        self.vals = None if vals is None else upload(vals, np.float32)
        self.struct = _lib.Dirichlet(int(space.n_nodes), ptr(self.code), ptr(self.vals))


# ---- reference-API operations -----------------------------------------------------------

def prolongate_state(hierarchy, x, levels_up=1):
    from .space import StateVector
    v = f32(x.values)
    lvl = x.level
    for _ in range(levels_up):
        P = DeviceProlong.get(hierarchy, lvl)
        if v.numel() != 4 * P.n_coarse_nodes:
            raise ValueError(f"vector length {v.numel()} does not match level {lvl} "
                             f"({4 * P.n_coarse_nodes} dofs)")
        out = torch.empty(4 * P.n_fine, dtype=torch.float32, device=v.device)
        _lib.call("dnnmg_prolongate", ctypes.byref(P.struct), ptr(v), ptr(out), None,
                  stream_handle())
        v = out
        lvl += 1
    return StateVector(lvl, like_input(v, x.values), x.time)


def apply_dirichlet_state(space, x, t, bcs):
    bc = DeviceDirichlet(space, t, bcs)
    if isinstance(x.values, torch.Tensor) and x.values.is_cuda and x.values.dtype == torch.float32 \
            and x.values.is_contiguous():
        _lib.call("dnnmg_apply_dirichlet", ctypes.byref(bc.struct), ptr(x.values), stream_handle())
        return x
    v = f32(x.values)
    _lib.call("dnnmg_apply_dirichlet", ctypes.byref(bc.struct), ptr(v), stream_handle())
    touched = torch.nonzero(bc.code).reshape(-1)
    rows = v.reshape(-1, 4)[touched]
    if isinstance(x.values, np.ndarray):
        # only the constrained rows change; untouched entries keep their float64 values
        x.values.reshape(-1, 4)[touched.cpu().numpy()] = rows.double().cpu().numpy()
    else:
        x.values.reshape(-1, 4)[touched.to(x.values.device)] = rows.to(x.values.dtype)
    return x
