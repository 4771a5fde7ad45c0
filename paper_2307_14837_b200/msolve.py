"""Cell-based Vanka smoother of the coarse-level multigrid on the GPU.

Drop-in for the reference's ``msolve.VankaData`` / ``msolve.vanka_smooth``
(msolve.py:51-89), which the reference multigrid V-cycle (``MgPreconditioner.vcycle``,
msolve.py:101-137) calls 2 x 6 times per level and cycle — the dominant cost of a DNN-MG
run.  The Jacobian is still assembled by the caller (the reference's
``Assembler.assemble_jacobian`` on the host); here the 108 x 108 cell blocks are gathered
and inverted on the device once per Jacobian (``dnnmg_vanka_setup``, float64), and every
sweep — CSR residual, batched block solve, ordered per-dof accumulation, damped update —
runs as kernels (``dnnmg_vanka_smooth``).  Arrays: numpy float64 in -> numpy float64 out
(one H2D of x, b and one D2H of x per call), or float64 CUDA tensors in place.

    import dnnmg.msolve as ms, paper_2307_14837_b200.msolve as gms
    ms.VankaData, ms.vanka_smooth = gms.VankaData, gms.vanka_smooth   # reference MG on the GPU
"""

import ctypes

import numpy as np
import torch

from . import _lib, device as dv


def _i32(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dv.device())


def _f64(a):
    return torch.from_numpy(np.array(a, dtype=np.float64)).to(dv.device())


class DeviceCsr:
    """A scipy CSR matrix uploaded once (float64 values, int32 indices)."""

    def __init__(self, J):
        self.n = int(J.shape[0])
        self.indptr = _i32(J.indptr)
        self.indices = _i32(J.indices)
        self.data = _f64(J.data)
        self.struct = _lib.Csr(self.n, dv.ptr(self.indptr), dv.ptr(self.indices), dv.ptr(self.data))

    @staticmethod
    def get(J):
        """Cached on the matrix object (a Jacobian is reused across many smoothing calls)."""
        d = getattr(J, "_b200_csr", None)
        if d is None or d.data.numel() != J.data.size:
            d = DeviceCsr(J)
            try:
                J._b200_csr = d
            except AttributeError:
                pass
        return d


class VankaData:
    """Cell-local blocks of a level Jacobian, inverted on the device (msolve.py:51-74).

    ``asm`` is an assembler with ``n_cells``, ``ndl``, ``cell_dofs``, ``flat_pos`` and
    ``space.ndof`` (the reference ``Assembler``); ``J`` the level Jacobian (scipy CSR with the
    assembler's sorted pattern).  Same attributes as the reference: ``dofs``, ``weight``,
    ``flagged`` (cells regularised by the 1e-12 diagonal shift), ``ndof``; ``inv`` is the
    device tensor [n_cells, ndl, ndl]."""

    def __init__(self, asm, J):
        nc, ndl = int(asm.n_cells), int(asm.ndl)
        self.dofs = np.asarray(asm.cell_dofs)
        self.ndof = int(asm.space.ndof)
        counts = np.bincount(self.dofs.reshape(-1), minlength=self.ndof)
        self.weight = 1.0 / counts
        self.n_cells, self.ndl = nc, ndl
        self.csr = DeviceCsr.get(J)
        flat = torch.from_numpy(np.ascontiguousarray(asm.flat_pos, dtype=np.int64)).to(dv.device())
        # the device keeps the inverses transposed (coalesced block solves); .inv is the
        # reference's [n_cells, ndl, ndl] view
        self._invT = torch.empty((nc, ndl, ndl), dtype=torch.float64, device=dv.device())
        self.inv = self._invT.transpose(1, 2)
        flags = torch.zeros(max(nc, 1), dtype=torch.int32, device=dv.device())
        _lib.call("dnnmg_vanka_setup", nc, ndl, dv.ptr(self.csr.data), dv.ptr(flat),
                  dv.ptr(self._invT), dv.ptr(flags), dv.stream_handle())
        f = flags[:nc].cpu().numpy()
        if np.any(f == 2):
            raise np.linalg.LinAlgError("Singular matrix")
        self.flagged = [int(c) for c in np.nonzero(f == 1)[0]]
        flat_d = self.dofs.reshape(-1).astype(np.int64)
        order = np.argsort(flat_d, kind="stable")      # ascending (cell, i) per dof
        ptr = np.zeros(self.ndof + 1, dtype=np.int64)
        np.cumsum(counts, out=ptr[1:])
        self._dofs_d = _i32(self.dofs)
        self._ptr = _i32(ptr)
        self._idx = _i32(order)
        self._w = _f64(self.weight)
        self.struct = _lib.Vanka(nc, ndl, self.ndof, dv.ptr(self._dofs_d), dv.ptr(self._ptr),
                                 dv.ptr(self._idx), dv.ptr(self._w), dv.ptr(self._invT))
        self._r = torch.empty(self.ndof, dtype=torch.float64, device=dv.device())
        self._dl = torch.empty(max(nc * ndl, 1), dtype=torch.float64, device=dv.device())


def vanka_smooth(J, vanka, x, b, sweeps, damping):
    """Jacobi-coupled cell-Vanka sweeps; all cells read the sweep-start iterate
    (msolve.py:77-89).  numpy in -> new numpy array out (the reference returns a new x);
    float64 CUDA tensors -> x updated in place and returned."""
    csr = DeviceCsr.get(J) if not isinstance(J, DeviceCsr) else J
    if csr.n != vanka.ndof:
        raise ValueError(f"Jacobian length {csr.n} does not match the Vanka data ({vanka.ndof})")
    on_device = isinstance(x, torch.Tensor)
    xd = x if on_device else _f64(x)
    bd = b if isinstance(b, torch.Tensor) else _f64(b)
    if xd.dtype != torch.float64 or bd.dtype != torch.float64:
        raise ValueError("vanka_smooth works in float64")
    _lib.call("dnnmg_vanka_smooth", ctypes.byref(vanka.struct), ctypes.byref(csr.struct),
              dv.ptr(bd), dv.ptr(xd), int(sweeps), ctypes.c_double(float(damping)),
              dv.ptr(vanka._r), dv.ptr(vanka._dl), dv.stream_handle())
    return xd if on_device else xd.cpu().numpy()
