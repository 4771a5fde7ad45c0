"""Where the tensor-core and SIMT K2 (RHS form) differ on the dataset test's loop states
(the reference's recorded coarse solves, ideal correction) -- diagnostic."""
import sys, os, ctypes; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch
import test_gpu_dataset as T
from paper_2307_14837_b200 import driver, io as iomod, mesh as meshmod, _lib, device as dv
pr = T.Problem()
ft = iomod.Trajectory(os.path.join(T.DS, "fine.dmgt"))
m = driver._FineMachinery(pr, 0, 1, meshmod.build_patches(pr.hierarchy, 0, 1))
lvl = m.step.level
def rel(a, b): return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
for i in range(len(pr.solves["t"])):
    t = pr.solves["t"][i]; n = int(round(t / pr.k))
    xt = m.embed(pr.solves["x"][i], t)
    x_corr = m.ideal_update(xt, ft.values(n))
    outs = {}
    for tc in (False, True):
        lv = lvl.struct(None, geometry=True, tc=tc)
        elem = torch.empty(lvl.n_cells * 108, device="cuda"); o = torch.empty_like(x_corr)
        _lib.call("dnnmg_rhs_next", ctypes.byref(lv), dv.ptr(x_corr), ctypes.byref(m.step.phys), dv.ptr(elem), dv.ptr(o), dv.stream_handle())
        torch.cuda.synchronize(); outs[tc] = (o.double().cpu().numpy(), elem.double().cpu().numpy().reshape(-1, 27, 4))
    d = np.abs(outs[True][1] - outs[False][1]).max(axis=(1, 2))
    xv = x_corr.double().cpu().numpy().reshape(-1, 4)
    print(i, n, "rel %.2e" % rel(outs[True][0], outs[False][0]), "cell max diff", np.round(d, 5)[:16], "|v|max %.2f" % np.abs(xv[:, 1:]).max())
# per-cell max |scaled coefficient| of the tensor-core kernel (DNNMG_K2TC_CMAX; needs a library
# built with `make EXTRA=-DDNNMG_K2TC_DIAG_BUILD`)
cm = torch.zeros(lvl.n_cells, dtype=torch.int32, device="cuda")
os.environ["DNNMG_K2TC_CMAX"] = str(cm.data_ptr())
lv = lvl.struct(None, geometry=True, tc=True)
elem = torch.empty(lvl.n_cells * 108, device="cuda"); o = torch.empty_like(x_corr)
_lib.call("dnnmg_rhs_next", ctypes.byref(lv), dv.ptr(x_corr), ctypes.byref(m.step.phys), dv.ptr(elem), dv.ptr(o), dv.stream_handle())
torch.cuda.synchronize()
print("max |scaled coef| per cell (target ~2^8):", np.round(cm.cpu().numpy().view(np.float32), 4))
cm.zero_()
x = dv.f32(ft.values(n))
_lib.call("dnnmg_rhs_next", ctypes.byref(lv), dv.ptr(x), ctypes.byref(m.step.phys), dv.ptr(elem), dv.ptr(o), dv.stream_handle())
torch.cuda.synchronize()
print("on v_ref:", np.round(cm.cpu().numpy().view(np.float32), 4))
