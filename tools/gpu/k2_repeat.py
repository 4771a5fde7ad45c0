"""Determinism of the tensor-core K2 at config-3 size: 5 launches on the same inputs must give
identical bits (and match the SIMT kernel to fp32 rounding)."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2307_14837_b200 import _lib, device as dv, mesh as meshmod, space as spmod, synthetic
n_cells = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "64x32x32").split("x"))
h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1), n_cells=n_cells)
if len(sys.argv) > 2:
    synthetic.jitter_vertices(h.levels[0].vertices, n_cells, (0, 0, 0), (1, 1, 1), 5)
meshmod.refine_uniform(h)
s = spmod.FeSpace(h, 1)
lvl = dv.DeviceLevel.get(s)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(4 * s.n_nodes, device="cuda", generator=g)
b = torch.randn(4 * s.n_nodes, device="cuda", generator=g) * 1e-3
ph = _lib.Phys(1e-3, 5e-3, 0.02, 0.1, 1)
elem = torch.empty(lvl.n_cells * 108, device="cuda")
outs = []
for tc in (True, True, True, True, True, False):
    lv = lvl.struct(None, geometry=True, tc=tc)
    r = torch.empty_like(x)
    _lib.call("dnnmg_residual", ctypes.byref(lv), dv.ptr(x), dv.ptr(b), None, None, ctypes.byref(ph),
              dv.ptr(elem), dv.ptr(r), 0, dv.stream_handle())
    torch.cuda.synchronize()
    outs.append(r.clone())
same = all(torch.equal(outs[0], o) for o in outs[1:5])
d = (outs[0].double() - outs[5].double()).norm() / outs[5].double().norm()
print("tc repeat bitwise:", same, " rel diff tc vs simt %.2e" % d.item())
