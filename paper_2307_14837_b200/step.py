"""The fused fine-level correction step on device-resident data.

``CorrectionStep`` is the production form of ``driver.TimeLoop._step_hybrid``
lines 251-268 (prolongate -> Dirichlet -> stab -> residual -> gather -> MLP ->
scatter-average -> x~ + scale*d): all tables, weights and work buffers live in
HBM, one call issues the whole K1..K5 sequence through the single C-ABI entry
``dnnmg_correction_step`` on the current stream (no host synchronisation, no
allocation), and the sequence can be captured into a CUDA graph.
"""

import ctypes

import numpy as np
import torch

from . import _lib, device as dv, mesh as meshmod
from .patch_ops import check_model, input_width, output_width
from .space import FeSpace, no_slip


def constrained_mask(space, bcs):
    """Dirichlet velocity dofs plus the pressure pin at dof 0 when there is no
    outflow boundary (driver.py:56-65)."""
    m = space.dirichlet_mask(tuple(bcs.keys()))
    if not space.has_outflow:
        m[0] = True
    return m


class CorrectionStep:
    def __init__(self, hierarchy, L, J, model, nu, k, bcs=None, alpha0=0.02, delta0=0.1,
                 scale=1.0, precision="fp32", patchset=None, t=0.0, mask=None, k2_box=None):
        """k2_box: None = K2's box form whenever the fine level is axis-aligned (checked on the
        device); False = never (the slab decomposition passes it for a jittered global mesh so
        that every rank runs the same element-kernel form as the single domain)."""
        self.hierarchy, self.L, self.J = hierarchy, L, J
        self.k2_box = k2_box
        self.bcs = bcs if bcs is not None else {meshmod.WALL: no_slip}
        self.scale = float(scale)
        self.nu, self.k = nu, k
        self.space = FeSpace(hierarchy, L + J)
        self.coarse_ndof = 4 * hierarchy.scalar_nodes(L)[0].shape[0]
        self.prolongs = [dv.DeviceProlong.get(hierarchy, l) for l in range(L, L + J)]
        self.P = (_lib.Prolong * J)(*[p.struct for p in self.prolongs])
        self.level = dv.DeviceLevel.get(self.space)
        self.mask = constrained_mask(self.space, self.bcs) if mask is None else np.asarray(mask)
        self.mask_bits = dv.upload(dv.dof_mask_bits(self.mask, self.space.n_nodes), np.uint8)
        # K2 reads J^-1 and w from the per-mesh geometry cache (the mesh is fixed in time)
        self.lv = self.level.struct(self.mask_bits, geometry=True, box=self.k2_box)
        self.patchset = patchset if patchset is not None else meshmod.build_patches(hierarchy, L, J)
        self.ps = dv.DevicePatchSet.get(self.patchset)
        self.precision = precision
        # model=None: embedding and next-step RHS only (a hybrid loop before its first
        # correction, driver.py:261); run() then raises
        self.model = None
        self.fused_gather = False
        if model is not None:
            check_model(model, self.patchset)
            self.model = dv.DeviceModel(model, precision)
            precision = self.precision = self.model.precision   # relu: f16x3 -> tf32x3
            a = model.arch
            # K3 fused into K4 when the tensor-core MLP can stage the rows itself
            self.fused_gather = (precision not in ("fp32", "fp8") and a.n_hidden == 256 and a.n_in <= 256
                                 and a.n_out <= 256 and self.patchset.n_geo % 4 == 0)
        self.phys = _lib.Phys(float(nu), float(k), float(alpha0), float(delta0), 1)
        dev = dv.device()
        nf = self.space.n_nodes
        f = torch.float32
        self.x_tilde = torch.empty(4 * nf, dtype=f, device=dev)
        self.r = torch.empty(4 * nf, dtype=f, device=dev)
        self.d = torch.empty(4 * nf, dtype=f, device=dev)
        self.x_corr = torch.empty(4 * nf, dtype=f, device=dev)
        # element-vector scratch owned by this step (not the level's shared one), so steps on
        # the same level can run on different streams
        self.elem = torch.empty(self.level.n_cells * 27 * 4, dtype=f, device=dev)
        # layered tensor-core MLP (widths the fused kernel does not hold): the gather is fused
        # into its layer-0 operand; width 128 runs the fused kernel on stored X rows
        self.layered = (model is not None and precision != "fp32"
                        and (precision == "fp8" or not dv.tc_fused_supported(model.arch)))
        # X is only materialised when the gather is not fused into the MLP
        n_x = 0 if (self.fused_gather or self.layered or model is None) else self.ps.n_patches
        self.X = torch.empty((n_x, input_width(self.patchset)), dtype=f, device=dev)
        self.Y = torch.empty((self.ps.n_patches if model is not None else 0,
                              output_width(self.patchset)), dtype=f, device=dev)
        self.x_mid = (torch.empty(4 * self.prolongs[0].n_fine, dtype=f, device=dev)
                      if J == 2 else None)
        # its own MLP workspace (not the model's shared one): steps sharing a model can run
        # on different streams
        self.mlp_ws = self.model.new_workspace(self.ps.n_patches) if self.layered else None
        self.buf = _lib.StepBuffers(dv.ptr(self.x_tilde), dv.ptr(self.r), dv.ptr(self.elem),
                                    dv.ptr(self.X), dv.ptr(self.Y), dv.ptr(self.d),
                                    dv.ptr(self.x_mid), dv.ptr(self.mlp_ws), dv.nbytes(self.mlp_ws))
        self._t = None
        self.set_time(t)
        self.graph = None

    # Dirichlet data are re-evaluated only when they depend on t
    def set_time(self, t):
        code, vals = dv.dirichlet_codes(self.space, t, self.bcs)
        if self._t is not None and vals is None and self._static:
            return
        self._static = vals is None
        old = getattr(self, "bc", None)
        if (old is not None and vals is not None and old.vals is not None
                and old.vals.numel() == vals.size):
            # in place: a captured graph keeps reading the same buffers
            old.code.copy_(dv.upload(code, np.uint8))
            old.vals.copy_(dv.upload(vals, np.float32))
            if not np.array_equal(self._code_host, code):  # (codes normally do not depend on t)
                self._code_host = np.array(code, dtype=np.uint8)
                old.code_owner.copy_(dv.upload(self._code_host[self.prolongs[-1].owner_order], np.uint8))
                if old.lat_bc is not None:
                    old.lat_bc.copy_(dv.upload(self.prolongs[-1].lattice_with_codes(code), np.int32))
            self._t = t
            return
        self.graph = None  # new buffers: a graph captured earlier would read stale ones
        self.bc = dv.DeviceDirichlet.__new__(dv.DeviceDirichlet)
        self.bc.code = dv.upload(code, np.uint8)
        self._code_host = np.array(code, dtype=np.uint8)
        # the codes in the owner order of the last prolongation (K1 reads them coalesced)
        self.bc.code_owner = dv.upload(np.asarray(code, np.uint8)[self.prolongs[-1].owner_order], np.uint8)
        self.bc.vals = None if vals is None else dv.upload(vals, np.float32)
        # ... and packed into the lattice table of that prolongation (no code load at all)
        lat = self.prolongs[-1].lattice_with_codes(code)
        self.bc.lat_bc = None if lat is None else dv.upload(lat, np.int32)
        self.bc.struct = _lib.Dirichlet(self.space.n_nodes, dv.ptr(self.bc.code), dv.ptr(self.bc.vals),
                                        dv.ptr(self.bc.code_owner), dv.ptr(self.bc.lat_bc))
        self._t = t

    @property
    def n_patches(self):
        return self.ps.n_patches

    def twin(self):
        """A second workspace for the same problem: shares every device table and the
        packed model, owns its work buffers, so two steps can be in flight on two
        streams (HostPipeline(lanes=2))."""
        import copy
        t = copy.copy(self)
        dev = self.x_tilde.device
        f = torch.float32
        t.x_tilde = torch.empty_like(self.x_tilde)
        t.r = torch.empty_like(self.r)
        t.d = torch.empty_like(self.d)
        t.x_corr = torch.empty_like(self.x_corr)
        t.elem = torch.empty_like(self.elem)
        t.X = torch.empty_like(self.X)
        t.Y = torch.empty_like(self.Y)
        t.x_mid = None if self.x_mid is None else torch.empty_like(self.x_mid)
        t.mlp_ws = None if self.mlp_ws is None else torch.empty_like(self.mlp_ws)
        t.buf = _lib.StepBuffers(dv.ptr(t.x_tilde), dv.ptr(t.r), dv.ptr(t.elem), dv.ptr(t.X),
                                 dv.ptr(t.Y), dv.ptr(t.d), dv.ptr(t.x_mid), dv.ptr(t.mlp_ws),
                                 dv.nbytes(t.mlp_ws))
        if self.bc.vals is not None:
            # time-dependent Dirichlet data are updated in place by set_time: own a copy
            bc = dv.DeviceDirichlet.__new__(dv.DeviceDirichlet)
            bc.code, bc.vals = self.bc.code.clone(), self.bc.vals.clone()
            bc.code_owner = self.bc.code_owner
            bc.lat_bc = self.bc.lat_bc
            bc.struct = _lib.Dirichlet(self.space.n_nodes, dv.ptr(bc.code), dv.ptr(bc.vals),
                                       dv.ptr(bc.code_owner), dv.ptr(bc.lat_bc))
            t.bc = bc
        t.graph = None
        return t

    @property
    def launches(self):
        return int(_lib.load().dnnmg_correction_step_launches(self.J, ctypes.byref(self.model.struct)))

    def run(self, x_coarse, b_prev, x_corr=None):
        """Issue one correction step; all arguments are fp32 CUDA tensors."""
        out = self.x_corr if x_corr is None else x_corr
        if self.model is None:
            raise ValueError("correction step without a model: use embed_into() / rhs_next()")
        if x_coarse.numel() != self.coarse_ndof or b_prev.numel() != self.x_tilde.numel():
            raise ValueError("vector length does not match the coarse / fine level")
        _lib.call("dnnmg_correction_step", self.P, self.J, ctypes.byref(self.bc.struct),
                  ctypes.byref(self.lv), ctypes.byref(self.phys), ctypes.byref(self.ps.struct),
                  ctypes.byref(self.model.struct), dv.ptr(x_coarse), dv.ptr(b_prev),
                  ctypes.c_float(self.scale), ctypes.byref(self.buf), dv.ptr(out),
                  dv.stream_handle())
        return out

    __call__ = run

    def run_staged(self, x_coarse, b_prev, x_corr=None, events=None):
        """The same kernel sequence as run(), issued stage by stage through the
        per-kernel C-ABI entries so that CUDA events can bracket each stage
        (events: list of J+5 torch.cuda.Event, recorded on the current stream)."""
        out = self.x_corr if x_corr is None else x_corr
        s = dv.stream_handle()
        e = iter(events) if events is not None else None

        def mark():
            if e is not None:
                next(e).record()
        mark()
        cur = x_coarse
        for i, P in enumerate(self.prolongs):
            dst = self.x_tilde if i == self.J - 1 else self.x_mid
            bc = ctypes.byref(self.bc.struct) if i == self.J - 1 else None
            _lib.call("dnnmg_prolongate", ctypes.byref(P.struct), dv.ptr(cur), dv.ptr(dst), bc, s)
            cur = dst
            mark()
        _lib.call("dnnmg_residual", ctypes.byref(self.lv), dv.ptr(self.x_tilde), dv.ptr(b_prev),
                  None, None, ctypes.byref(self.phys), dv.ptr(self.elem), dv.ptr(self.r), 1, s)
        mark()
        self.predict_rows(s)
        mark()
        _lib.call("dnnmg_scatter_update", ctypes.byref(self.ps.struct), dv.ptr(self.Y),
                  dv.ptr(self.mask_bits), dv.ptr(self.x_tilde), ctypes.c_float(self.scale),
                  dv.ptr(self.d), dv.ptr(out), s)
        mark()
        return out

    def predict_rows(self, s):
        """Y = network(patch rows of x~, r): fused gather+MLP or gather then MLP."""
        if self.fused_gather or self.layered:
            _lib.call("dnnmg_mlp_forward_patches_ws", ctypes.byref(self.model.struct),
                      ctypes.byref(self.ps.struct), dv.ptr(self.x_tilde), dv.ptr(self.r),
                      dv.ptr(self.Y), dv.ptr(self.mlp_ws), dv.nbytes(self.mlp_ws), s)
            return
        _lib.call("dnnmg_gather", ctypes.byref(self.ps.struct), dv.ptr(self.x_tilde),
                  dv.ptr(self.r), dv.ptr(self.X), s)
        _lib.call("dnnmg_mlp_forward_ws", ctypes.byref(self.model.struct), dv.ptr(self.X),
                  self.ps.n_patches, dv.ptr(self.Y), dv.ptr(self.mlp_ws), dv.nbytes(self.mlp_ws), s)

    def stage_names(self):
        """Labels of the stages run_staged() brackets with events."""
        mid = ["K3K4_gather_mlp"] if (self.fused_gather or self.layered) else ["K3_gather+K4_mlp"]
        return ["K1_prolong"] * self.J + ["K2_residual"] + mid + ["K5_scatter"]

    def capture(self, x_coarse, b_prev):
        """Capture run(x_coarse, b_prev) into a CUDA graph (inputs are fixed buffers)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.run(x_coarse, b_prev)            # warm-up outside capture
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.run(x_coarse, b_prev)
        self.graph = g
        return g

    def residual_into(self, x_tilde, b_prev, r):
        """r = b_prev - A_h(x~) with stab at x~ and the mask (assembly.py:261-267), K2."""
        _lib.call("dnnmg_residual", ctypes.byref(self.lv), dv.ptr(x_tilde), dv.ptr(b_prev), None,
                  None, ctypes.byref(self.phys), dv.ptr(self.elem), dv.ptr(r), 1,
                  dv.stream_handle())
        return r

    def rhs_next(self, x, out=None):
        """Next-step fine RHS from a (corrected) fine state (assembly.py:242-259)."""
        out = torch.empty_like(self.x_tilde) if out is None else out
        lv = self.level.struct(geometry=True, box=self.k2_box)
        _lib.call("dnnmg_rhs_next", ctypes.byref(lv), dv.ptr(x), ctypes.byref(self.phys),
                  dv.ptr(self.elem), dv.ptr(out), dv.stream_handle())
        return out

    def embed_into(self, x_coarse, dst):
        """Prolongate (J levels) + Dirichlet into dst without allocation."""
        s = dv.stream_handle()
        cur = x_coarse
        for i, P in enumerate(self.prolongs):
            last = i == self.J - 1
            out = dst if last else self.x_mid
            bc = ctypes.byref(self.bc.struct) if last else None
            _lib.call("dnnmg_prolongate", ctypes.byref(P.struct), dv.ptr(cur), dv.ptr(out), bc, s)
            cur = out
        return dst

    def embed(self, x_coarse, t=None):
        """Prolongate + Dirichlet only (driver.embed_state, driver.py:611-619); t, when
        given, becomes the step's Dirichlet time (set_time)."""
        if t is not None and t != self._t:
            self.set_time(t)
        cur = dv.f32(x_coarse)
        for i, P in enumerate(self.prolongs):
            out = torch.empty(4 * P.n_fine, dtype=torch.float32, device=cur.device)
            bc = ctypes.byref(self.bc.struct) if i == self.J - 1 else None
            _lib.call("dnnmg_prolongate", ctypes.byref(P.struct), dv.ptr(cur), dv.ptr(out), bc,
                      dv.stream_handle())
            cur = out
        return cur


class HostPipeline:
    """Independent correction steps whose inputs and results live in pinned HOST
    memory, streamed through one CorrectionStep: the H2D copy of step i+1, the
    kernels of step i and the D2H copy of step i-1 run concurrently on three CUDA
    streams (two copy engines + compute) with double-buffered device inputs and
    outputs.  Each submit() enqueues one full step (copy in, K1..K5, copy out)
    and returns immediately; join() makes the caller's stream wait for all of it.

    This is the serving form of the step: with ~145 MB of host traffic per step
    at config 3, serialising copies and kernels would make the PCIe transfers,
    not the kernels, the step time."""

    def __init__(self, step, depth=2, lanes=1):
        """lanes = 2 runs consecutive steps on two compute streams with two workspaces
        (CorrectionStep.twin), so one step's memory-bound tail kernels can overlap the
        next step's head."""
        if lanes not in (1, 2) or depth % lanes:
            raise ValueError("lanes must be 1 or 2 and divide depth")
        self.step = step
        self.depth = depth
        self.steps = [step] + [step.twin() for _ in range(lanes - 1)]
        dev = step.x_tilde.device
        f = torch.float32
        self.dx = [torch.empty(step.coarse_ndof, dtype=f, device=dev) for _ in range(depth)]
        self.db = [torch.empty_like(step.x_tilde) for _ in range(depth)]
        self.dout = [torch.empty_like(step.x_tilde) for _ in range(depth)]
        self.s_in = torch.cuda.Stream(device=dev)
        self.s_runs = [torch.cuda.Stream(device=dev) for _ in range(lanes)]
        self.s_out = torch.cuda.Stream(device=dev)
        self.split = self.db[0].numel() * 4 >= (4 << 20)   # fine RHS >= 4 MB
        self.ev_x = [torch.cuda.Event() for _ in range(depth)]
        self.ev_in = [torch.cuda.Event() for _ in range(depth)]
        self.ev_run = [torch.cuda.Event() for _ in range(depth)]
        self.ev_out = [torch.cuda.Event() for _ in range(depth)]
        self.i = 0
        self._used = [False] * depth

    def begin(self):
        """Order the pipeline after everything already queued on the current stream."""
        cur = torch.cuda.current_stream()
        for s in [self.s_in, self.s_out] + self.s_runs:
            s.wait_stream(cur)

    def submit(self, x_host, b_host, out_host):
        k = self.i % self.depth
        with torch.cuda.stream(self.s_in):
            if self._used[k]:
                self.s_in.wait_event(self.ev_run[k])      # step i-depth has consumed dx/db[k]
            # a large fine RHS (68 MB at config 3) is copied after the coarse state, and the
            # step waits for it only right before the residual's node sum
            # (dnnmg_step_buffers_t.b_ready): prolongation and the element kernel overlap it.
            # (Small steps skip the split: the extra event costs more than it hides.)
            self.dx[k].copy_(x_host, non_blocking=True)
            if self.split:
                self.ev_x[k].record()
            self.db[k].copy_(b_host, non_blocking=True)
            self.ev_in[k].record()
        lane = self.i % len(self.steps)
        s_run = self.s_runs[lane]
        step = self.steps[lane]
        with torch.cuda.stream(s_run):
            s_run.wait_event(self.ev_x[k] if self.split else self.ev_in[k])
            if self._used[k]:
                s_run.wait_event(self.ev_out[k])          # dout[k] has been copied out
            if self.split:
                step.buf.b_ready = self.ev_in[k].cuda_event
            try:
                step.run(self.dx[k], self.db[k], self.dout[k])
            finally:
                step.buf.b_ready = None
            self.ev_run[k].record()
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(self.ev_run[k])
            out_host.copy_(self.dout[k], non_blocking=True)
            self.ev_out[k].record()
        self._used[k] = True
        self.i += 1

    def join(self):
        cur = torch.cuda.current_stream()
        for s in [self.s_in, self.s_out] + self.s_runs:
            cur.wait_stream(s)
