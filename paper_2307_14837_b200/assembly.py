"""Stabilised Crank-Nicolson Navier-Stokes residual on one fine level (drop-in for
the correction-path part of the reference ``dnnmg.assembly``).

``Assembler(space)`` uploads the level's tables once; ``stab``,
``assemble_residual``, ``apply_operator`` and ``assemble_rhs_next`` run kernel
K2 of libdnnmg_b200 (matrix-free, sum-factorised, fp32, deterministic node
sums).  Reference: assembly.py:38-108 (StabParams, stab_params, geometry
cache), 169-178 (stab), 212-234 (apply_operator), 242-259 (rhs_next),
261-267 (assemble_residual).  The Jacobian and the coarse solver are outside
the correction step.
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, device as dv


@dataclass
class StabParams:
    """Local projection stabilisation weights (assembly.py:38-52)."""
    alpha0: float = 0.02
    delta0: float = 0.1
    alpha_T: object = field(default=None)
    delta_T: object = field(default=None)

    @property
    def has_delta(self):
        if self.delta_T is None:
            return False
        d = self.delta_T
        return bool((d != 0).any()) if isinstance(d, torch.Tensor) else bool(np.any(d != 0.0))


def stab_params(h_T, vmax, nu, k, alpha0=0.02, delta0=0.1):
    """Host formula alpha0/den, delta0/den (assembly.py:55-59); used for scalars/tests."""
    h_T = np.asarray(h_T, dtype=float)
    den = nu / h_T ** 2 + np.asarray(vmax, dtype=float) / h_T + 1.0 / k
    return alpha0 / den, delta0 / den


class Assembler:
    """Per-level assembly context on the GPU (assembly.py:62-108)."""

    def __init__(self, space, n_gauss=4):
        if n_gauss != 4:
            raise NotImplementedError("the kernels implement the reference's 4-point rule")
        if space.dim != 3:
            raise NotImplementedError("only 3-D hexahedral levels are supported")
        self.space = space
        self.dim, self.ncomp = 3, 4
        self.nloc, self.ndl, self.nq = 27, 108, 64
        self.n_cells = space.cell_nodes.shape[0]
        self.dev = dv.DeviceLevel.get(space)
        self.h_T = self.dev.h_T_host
        self._mask_cache = (None, None)

    @property
    def cell_dofs(self):
        cn = self.space.cell_nodes
        return (4 * cn[:, :, None] + np.arange(4)[None, None, :]).reshape(self.n_cells, -1)

    def _vec(self, v, what="vector"):
        t = dv.f32(v)
        if t.numel() != self.space.ndof:
            raise ValueError(f"{what} length {t.numel()} does not match the level "
                             f"({self.space.ndof} dofs)")
        return t

    def _mask_bits(self, mask):
        if mask is None:
            return None
        if self._mask_cache[0] is mask:
            return self._mask_cache[1]
        m = mask.cpu().numpy() if isinstance(mask, torch.Tensor) else mask
        bits = dv.upload(dv.dof_mask_bits(m, self.space.n_nodes), np.uint8)
        self._mask_cache = (mask, bits)
        return bits

    @staticmethod
    def _phys(k, nu, alpha0, delta0, convection):
        return _lib.Phys(float(nu), float(k), float(alpha0), float(delta0), int(bool(convection)))

    def _stab_ptrs(self, stab):
        if stab is None or stab.alpha_T is None:
            return None, None, (stab.alpha0 if stab else dv.ALPHA0), (stab.delta0 if stab else dv.DELTA0)
        aT = dv.f32(stab.alpha_T)
        dT = dv.f32(stab.delta_T) if stab.delta_T is not None else torch.zeros_like(aT)
        return aT, dT, stab.alpha0, stab.delta0

    def stab(self, prev_values, nu, k, alpha0=0.02, delta0=0.1):
        """alpha_T, delta_T frozen at prev_values (assembly.py:169-178)."""
        x = self._vec(prev_values)
        aT = torch.empty(self.n_cells, dtype=torch.float32, device=x.device)
        dT = torch.empty_like(aT)
        lv = self.dev.struct()
        ph = self._phys(k, nu, alpha0, delta0, True)
        _lib.call("dnnmg_stab", ctypes.byref(lv), dv.ptr(x), ctypes.byref(ph), dv.ptr(aT),
                  dv.ptr(dT), dv.stream_handle())
        return StabParams(alpha0, delta0, dv.like_input(aT, prev_values),
                          dv.like_input(dT, prev_values))

    def apply_operator(self, x_values, k, nu, stab, convection=True):
        """A_h(x) as a dual vector (assembly.py:212-234)."""
        x = self._vec(x_values)
        aT, dT, a0, d0 = self._stab_ptrs(stab)
        out = torch.empty_like(x)
        lv = self.dev.struct()
        ph = self._phys(k, nu, a0, d0, convection)
        _lib.call("dnnmg_apply_operator", ctypes.byref(lv), dv.ptr(x), dv.ptr(aT), dv.ptr(dT),
                  ctypes.byref(ph), dv.ptr(self.dev.scratch()), dv.ptr(out), dv.stream_handle())
        return dv.like_input(out, x_values)

    def assemble_residual(self, x_values, b_prev, k, nu, stab, mask=None, convection=True):
        """r = b_prev - A_h(x); constrained rows zeroed (assembly.py:261-267)."""
        x = self._vec(x_values)
        b = self._vec(b_prev, "right-hand side")
        aT, dT, a0, d0 = self._stab_ptrs(stab)
        bits = self._mask_bits(mask)
        r = torch.empty_like(x)
        lv = self.dev.struct(bits)
        ph = self._phys(k, nu, a0, d0, convection)
        _lib.call("dnnmg_residual", ctypes.byref(lv), dv.ptr(x), dv.ptr(b), dv.ptr(aT), dv.ptr(dT),
                  ctypes.byref(ph), dv.ptr(self.dev.scratch()), dv.ptr(r), int(bits is not None),
                  dv.stream_handle())
        return dv.like_input(r, x_values)

    def assemble_rhs_next(self, x_values, f_old, f_new, k, nu, convection=True):
        """Next-step RHS from the (corrected) state, f = None (assembly.py:242-259)."""
        if f_old is not None or f_new is not None:
            raise NotImplementedError("volume forces are not part of the correction path")
        x = self._vec(x_values)
        out = torch.empty_like(x)
        lv = self.dev.struct()
        ph = self._phys(k, nu, 0.0, 0.0, convection)
        _lib.call("dnnmg_rhs_next", ctypes.byref(lv), dv.ptr(x), ctypes.byref(ph),
                  dv.ptr(self.dev.scratch()), dv.ptr(out), dv.stream_handle())
        return dv.like_input(out, x_values)
