"""CTA-0 timeline of the tensor-core K2 (DNNMG_K2TC_TRACE; needs a library built with
`make EXTRA=-DDNNMG_K2TC_DIAG_BUILD`): per stage the MMA lane's and
compute warps 0 / 15's stamps (cycles from the first MMA stamp), printed by the library
to stderr.   python tools/gpu/k2_trace.py [64x32x32]"""
import ctypes, os, sys
os.environ["DNNMG_K2TC_TRACE"] = "1"
sys.path.insert(0, ".")
import torch
from paper_2307_14837_b200 import _lib, device as dv, mesh as meshmod, space as spmod
n_cells = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "64x32x32").split("x"))
h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1), n_cells=n_cells)
meshmod.refine_uniform(h)
s = spmod.FeSpace(h, 1)
lvl = dv.DeviceLevel.get(s)
x = torch.randn(4 * s.n_nodes, device="cuda"); b = torch.randn_like(x) * 1e-3
ph = _lib.Phys(1e-3, 5e-3, 0.02, 0.1, 1)
elem = torch.empty(lvl.n_cells * 108, device="cuda"); r = torch.empty_like(x)
lv = lvl.struct(None, geometry=True, tc=True)
for _ in range(2):
    _lib.call("dnnmg_residual", ctypes.byref(lv), dv.ptr(x), dv.ptr(b), None, None, ctypes.byref(ph),
              dv.ptr(elem), dv.ptr(r), 0, dv.stream_handle())
torch.cuda.synchronize()
