import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, ctypes, torch
from conftest import GOLDEN_CASES
from golden_util import load_golden, product_hierarchy
from paper_2307_14837_b200 import _lib, device as dv, space as spmod
def rel(a,b): return np.linalg.norm(a-b)/max(np.linalg.norm(b),1e-300)
for name in GOLDEN_CASES:
    g = load_golden(name); h = product_hierarchy(g)
    lvl = dv.DeviceLevel.get(spmod.FeSpace(h, int(g["L"]) + int(g["J"])))
    out = {}
    for tc in (False, True):
        bits = dv.upload(dv.dof_mask_bits(g["mask"], lvl.n_nodes), np.uint8)
        lv = lvl.struct(bits, geometry=True, tc=tc)
        ph = _lib.Phys(float(g["nu"]), float(g["k"]), float(g["alpha0"]), float(g["delta0"]), 1)
        elem = torch.empty(lvl.n_cells * 108, dtype=torch.float32, device="cuda")
        x, b = dv.f32(g["x_tilde"]), dv.f32(g["b_prev"]); r = torch.empty_like(x)
        _lib.call("dnnmg_residual", ctypes.byref(lv), dv.ptr(x), dv.ptr(b), None, None, ctypes.byref(ph), dv.ptr(elem), dv.ptr(r), 1, dv.stream_handle())
        torch.cuda.synchronize(); out[tc] = r.double().cpu().numpy()
    print(name, "simt %.2e  tc %.2e" % (rel(out[False], g["r"]), rel(out[True], g["r"])))
