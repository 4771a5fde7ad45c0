"""Patch restriction/extension and the network prediction pipeline (drop-in for
the reference ``dnnmg.patch_ops``, patch_ops.py:1-82).

Gather (K3), network (K4) and the valence-averaging scatter (K5) run on the GPU;
error messages match the reference ("length", "architecture", "eval").
"""

import ctypes

import numpy as np
import torch

from . import _lib, device as dv
from .net import resolve_precision


def velocity_slots(patchset):
    base = np.arange(patchset.nodes_per_patch) * patchset.ncomp
    return (base[:, None] + np.arange(1, patchset.ncomp)[None, :]).reshape(-1)


def input_width(patchset):
    return 2 * patchset.ndof_patch + patchset.n_geo


def output_width(patchset):
    return (patchset.ncomp - 1) * patchset.nodes_per_patch


def _fine_vec(x, patchset):
    n = x.shape[0] if not isinstance(x, torch.Tensor) else x.numel()
    if n != patchset.mu.shape[0]:
        raise ValueError(f"vector length {n} does not match the "
                         f"fine level ({patchset.mu.shape[0]} dofs)")
    return dv.f32(x)


def local_restrict(x, patchset):
    """Rows of patch-local values x[dof_table] (patch_ops.py:23-29)."""
    xd = _fine_vec(x, patchset)
    ps = dv.DevicePatchSet.get(patchset)
    rows = torch.empty((ps.n_patches, 4 * ps.npp), dtype=torch.float32, device=xd.device)
    _lib.call("dnnmg_local_restrict", ctypes.byref(ps.struct), dv.ptr(xd), dv.ptr(rows),
              dv.stream_handle())
    return dv.like_input(rows, x)


def global_extend(rows, patchset, mu=None):
    """mu * bincount(dof_table, rows) (patch_ops.py:32-38)."""
    ps = dv.DevicePatchSet.get(patchset)
    rd = dv.f32(rows)
    if rd.numel() != ps.n_patches * 4 * ps.npp:
        raise ValueError(f"rows length {rd.numel()} does not match the patch set "
                         f"({ps.n_patches} x {4 * ps.npp})")
    out = torch.empty(4 * ps.n_nodes, dtype=torch.float32, device=rd.device)
    _lib.call("dnnmg_global_extend", ctypes.byref(ps.struct), dv.ptr(rd), dv.ptr(out),
              dv.stream_handle())
    if mu is not None and mu is not patchset.mu:
        # a caller-supplied scaling replaces the stored reciprocal valence
        out = out * (dv.f32(mu) * dv.f32(np.asarray(patchset.valence, dtype=float)))
    return dv.like_input(out, rows)


def assemble_network_input(x_tilde, r, patchset):
    """Per-patch feature rows [state | residual | geometry] (patch_ops.py:49-53)."""
    xd = _fine_vec(x_tilde, patchset)
    rd = _fine_vec(r, patchset)
    ps = dv.DevicePatchSet.get(patchset)
    X = torch.empty((ps.n_patches, 8 * ps.npp + ps.n_geo), dtype=torch.float32, device=xd.device)
    _lib.call("dnnmg_gather", ctypes.byref(ps.struct), dv.ptr(xd), dv.ptr(rd), dv.ptr(X),
              dv.stream_handle())
    return dv.like_input(X, x_tilde)


def check_model(model, patchset):
    if model.mode != "eval":
        raise ValueError("predict_correction requires an eval-mode model")
    n_in, n_out = input_width(patchset), output_width(patchset)
    if model.arch.n_in != n_in or model.arch.n_out != n_out:
        raise ValueError(f"model architecture ({model.arch.n_in} -> {model.arch.n_out}) does "
                         f"not match the patch layout ({n_in} -> {n_out})")


def predict_correction(model, x_tilde, r, patchset, dirichlet_mask=None, precision=None):
    """Global velocity defect predicted patchwise; pressure block zero
    (patch_ops.py:56-76)."""
    check_model(model, patchset)
    xd = _fine_vec(x_tilde, patchset)
    rd = _fine_vec(r, patchset)
    ps = dv.DevicePatchSet.get(patchset)
    X = torch.empty((ps.n_patches, 8 * ps.npp + ps.n_geo), dtype=torch.float32, device=xd.device)
    _lib.call("dnnmg_gather", ctypes.byref(ps.struct), dv.ptr(xd), dv.ptr(rd), dv.ptr(X),
              dv.stream_handle())
    dm = dv.DeviceModel(model, resolve_precision(precision))
    Y = torch.empty((ps.n_patches, 3 * ps.npp), dtype=torch.float32, device=xd.device)
    dm.forward(X, ps.n_patches, Y)
    bits = None
    if dirichlet_mask is not None:
        m = dirichlet_mask.cpu().numpy() if isinstance(dirichlet_mask, torch.Tensor) else dirichlet_mask
        bits = dv.upload(dv.dof_mask_bits(m, ps.n_nodes), np.uint8)
    d = torch.empty(4 * ps.n_nodes, dtype=torch.float32, device=xd.device)
    _lib.call("dnnmg_scatter_update", ctypes.byref(ps.struct), dv.ptr(Y), dv.ptr(bits), None,
              ctypes.c_float(0.0), dv.ptr(d), None, dv.stream_handle())
    return dv.like_input(d, x_tilde)


def patch_targets(v_ref, x_tilde, patchset):
    """Training targets: fine-minus-prolongated velocity per patch (patch_ops.py:79-82)."""
    diff = dv.f32(v_ref) - dv.f32(x_tilde)
    rows = local_restrict(diff, patchset)
    out = rows[:, torch.as_tensor(velocity_slots(patchset), device=rows.device)]
    return dv.like_input(out, x_tilde)
