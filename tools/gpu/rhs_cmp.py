"""Tensor-core vs SIMT K2 in RHS form on the dataset test's channel mesh, per recorded state."""
import sys, os, ctypes
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch
from paper_2307_14837_b200 import _lib, device as dv, mesh as meshmod, space as spmod, synthetic, io as iomod
LO, HI, NC = (0, 0, -0.205), (1.0, 0.41, 0.205), (2, 1, 1)
h = meshmod.build_template_mesh("box", extent_lo=LO, extent_hi=HI, n_cells=NC, channel_tags=True)
synthetic.jitter_vertices(h.levels[0].vertices, NC, LO, HI, 21)
meshmod.refine_uniform(h)
s = spmod.FeSpace(h, 1); lvl = dv.DeviceLevel.get(s)
print("geo_kind", lvl.geo_kind, "cells", lvl.n_cells)
ft = iomod.Trajectory("tests/golden/dataset/fine.dmgt")
ph = _lib.Phys(1e-3, 0.02, 0.02, 0.1, 1)
def rel(a, b): return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
for i in range(ft.n_records):
    vals = ft.record(i)[2]
    x = dv.f32(np.asarray(vals))
    outs = {}
    for tc in (False, True):
        lv = lvl.struct(None, geometry=True, tc=tc)
        elem = torch.empty(lvl.n_cells * 108, device="cuda"); o = torch.empty_like(x)
        _lib.call("dnnmg_rhs_next", ctypes.byref(lv), dv.ptr(x), ctypes.byref(ph), dv.ptr(elem), dv.ptr(o), dv.stream_handle())
        torch.cuda.synchronize(); outs[tc] = o.double().cpu().numpy()
    v = np.asarray(vals).reshape(-1, 4)
    rb = {tc: spmod.restrict_rhs(h, dv.f32(outs[tc]), 1, 1).double().cpu().numpy() for tc in outs}
    print(i, "fine rel tc vs simt %.2e" % rel(outs[True], outs[False]),
          "restricted %.2e" % rel(rb[True], rb[False]), "norms fine %.3e coarse %.3e" % (np.linalg.norm(outs[False]), np.linalg.norm(rb[False])))
