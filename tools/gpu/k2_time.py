"""Time K2 (element kernel + node sum, dnnmg_residual) on a box: tensor-core vs SIMT element
kernel, CUDA events, same inputs; prints ms per call and the relative difference.
    python tools/gpu/k2_time.py 64x32x32 [jitter]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2307_14837_b200 import _lib, device as dv, mesh as meshmod, space as spmod, synthetic

n_cells = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "64x32x32").split("x"))
jit = len(sys.argv) > 2
h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1), n_cells=n_cells)
if jit:
    synthetic.jitter_vertices(h.levels[0].vertices, n_cells, (0, 0, 0), (1, 1, 1), 5)
meshmod.refine_uniform(h)
s = spmod.FeSpace(h, 1)
lvl = dv.DeviceLevel.get(s)
rng = np.random.default_rng(0)
x = torch.tensor(rng.standard_normal(4 * s.n_nodes), dtype=torch.float32, device="cuda")
b = torch.tensor(rng.standard_normal(4 * s.n_nodes) * 1e-3, dtype=torch.float32, device="cuda")
ph = _lib.Phys(1e-3, 5e-3, 0.02, 0.1, 1)
elem = torch.empty(lvl.n_cells * 108, dtype=torch.float32, device="cuda")
res = {}
for tc in (False, True):
    lv = lvl.struct(None, geometry=True, tc=tc)
    r = torch.empty_like(x)
    call = lambda: _lib.call("dnnmg_residual", ctypes.byref(lv), dv.ptr(x), dv.ptr(b), None, None,
                             ctypes.byref(ph), dv.ptr(elem), dv.ptr(r), 0, dv.stream_handle())
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        call()
    e1.record()
    torch.cuda.synchronize()
    res[tc] = (e0.elapsed_time(e1) / n, r.double().cpu().numpy())
    print(("tc  " if tc else "simt"), f"{res[tc][0]:.4f} ms", "affine" if lvl.affine else "per-point")
d = np.linalg.norm(res[True][1] - res[False][1]) / np.linalg.norm(res[False][1])
print("rel diff tc vs simt", d)
