"""The fused patch gather inside the tensor-core MLP (K3 into K4) against the
stand-alone gather + MLP, at sizes where every CTA runs several 128-patch tiles
and the last tile is partial.

The three layer-0 sources of the kernel — stored X rows, the direct per-(patch,
slot) gather and the staged gather of each tile's distinct nodes — feed the same
values through the same arithmetic, so their outputs must be bitwise equal; the
stored-X path is itself pinned against the float64 oracle MLP in
test_gpu_parity.py.  The gathered rows follow patch_ops.assemble_network_input
(patch_ops.py:49-53).
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_14837_b200 import _lib, device as dv, mesh as meshmod, net  # noqa: E402


def _patchset(n_cells, jitter):
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1),
                                    n_cells=n_cells)
    if jitter:
        lv = h.levels[0]
        rng = np.random.default_rng(3)
        inner = np.all((lv.vertices > 1e-9) & (lv.vertices < 1 - 1e-9), axis=1)
        lv.vertices[inner] += rng.uniform(-0.05, 0.05, (inner.sum(), 3)) / max(n_cells)
    meshmod.refine_uniform(h)
    return meshmod.build_patches(h, 0, 1)


def _model(seed, act="tanh", bn=False):
    rng = np.random.default_rng(seed)
    m = net.MlpModel(net.Architecture(240, 256, 3, 81), activation=act, seed=seed)
    dims = [240, 256, 256, 256, 81]
    m.W = [rng.uniform(-1, 1, (a, b)) * np.sqrt(6.0 / (a + b)) for a, b in zip(dims[:-1], dims[1:])]
    if bn:
        m.gamma = [rng.uniform(0.5, 1.5, 256) for _ in range(3)]
        m.beta = [rng.normal(0, 0.1, 256) for _ in range(3)]
        m.running_mean = [rng.normal(0, 0.2, 256) for _ in range(3)]
        m.running_var = [rng.uniform(0.5, 2.0, 256) for _ in range(3)]
        m.set_input_norm(rng.normal(0, 0.3, 240), rng.uniform(0.5, 2.0, 240))
    m.eval()
    return m


def _without_tiles(st):
    s = _lib.PatchSet()
    ctypes.memmove(ctypes.addressof(s), ctypes.addressof(st), ctypes.sizeof(st))
    s.tile_cap, s.tile_nodes, s.tile_count, s.tile_slot = 0, None, None, None
    return s


@pytest.mark.parametrize("precision", ["f16x3", "tf32x3", "bf16"])
@pytest.mark.parametrize("n_cells,jitter,bn", [((30, 20, 9), False, False),
                                               ((12, 11, 7), True, True)])
def test_fused_gather_modes_bitwise(precision, n_cells, jitter, bn):
    ps = _patchset(n_cells, jitter)
    dps = dv.DevicePatchSet.get(ps)
    assert dps.tile_cap > 0
    n = dps.n_patches
    rng = np.random.default_rng(n)
    x = torch.tensor(rng.standard_normal((dps.n_nodes, 4)), dtype=torch.float32, device="cuda")
    r = torch.tensor(rng.standard_normal((dps.n_nodes, 4)) * 1e-2, dtype=torch.float32, device="cuda")
    m = dv.DeviceModel(_model(n, "tanh" if precision != "tf32x3" or not bn else "relu", bn), precision)
    s = dv.stream_handle()
    Y = {k: torch.full((n, 81), float("nan"), device="cuda") for k in ("x", "direct", "staged")}
    X = torch.empty((n, 240), device="cuda")
    _lib.call("dnnmg_gather", ctypes.byref(dps.struct), dv.ptr(x), dv.ptr(r), dv.ptr(X), s)
    _lib.call("dnnmg_mlp_forward", ctypes.byref(m.struct), dv.ptr(X), n, dv.ptr(Y["x"]), s)
    _lib.call("dnnmg_mlp_forward_patches", ctypes.byref(m.struct), ctypes.byref(dps.struct),
              dv.ptr(x), dv.ptr(r), dv.ptr(Y["staged"]), s)
    mode = _lib.load().dnnmg_mlp_gather_mode(ctypes.byref(m.struct), ctypes.byref(dps.struct))
    assert mode == (1 if precision == "tf32x3" else 2), mode  # tf32x3 rings leave no room
    direct = _without_tiles(dps.struct)
    assert _lib.load().dnnmg_mlp_gather_mode(ctypes.byref(m.struct), ctypes.byref(direct)) == 1
    _lib.call("dnnmg_mlp_forward_patches", ctypes.byref(m.struct), ctypes.byref(direct),
              dv.ptr(x), dv.ptr(r), dv.ptr(Y["direct"]), s)
    torch.cuda.synchronize()
    assert torch.isfinite(Y["x"]).all()
    assert torch.equal(Y["direct"], Y["x"])
    assert torch.equal(Y["staged"], Y["x"])

