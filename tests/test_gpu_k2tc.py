"""The tensor-core K2 element kernel (csrc/residual_tc.cu: the forward and backward
constant-matrix contractions as tcgen05 GEMMs in the 3-pass fp16 split) against the
reference's golden residual and next-step RHS (assembly.py:212-267), and against the SIMT
element kernel, on every golden case: affine cells (config 0: per-cell geometry record),
jittered / J = 2 / coarse L = 1 / channel cells (per-point geometry), partial 128-cell
tiles, stab evaluated in the kernel or supplied."""
import ctypes

import numpy as np
import pytest

from conftest import GOLDEN_CASES
from golden_util import load_golden, product_hierarchy

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_14837_b200 import _lib, device as dv, space as spmod  # noqa: E402


def rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module", params=GOLDEN_CASES)
def case(request):
    g = load_golden(request.param)
    h = product_hierarchy(g)
    s = spmod.FeSpace(h, int(g["L"]) + int(g["J"]))
    return request.param, g, dv.DeviceLevel.get(s)


def run(level, g, tc, mode, stab_given):
    bits = dv.upload(dv.dof_mask_bits(g["mask"], level.n_nodes), np.uint8)
    lv = level.struct(bits if mode == "residual" else None, geometry=True, tc=tc)
    ph = _lib.Phys(float(g["nu"]), float(g["k"]), float(g["alpha0"]), float(g["delta0"]), 1)
    elem = torch.empty(level.n_cells * 108, dtype=torch.float32, device="cuda")
    s = dv.stream_handle()
    if mode == "residual":
        x, b = dv.f32(g["x_tilde"]), dv.f32(g["b_prev"])
        out = torch.empty_like(x)
        aT = dv.f32(g["alpha_T"]) if stab_given else None
        dT = dv.f32(g["delta_T"]) if stab_given else None
        _lib.call("dnnmg_residual", ctypes.byref(lv), dv.ptr(x), dv.ptr(b), dv.ptr(aT), dv.ptr(dT),
                  ctypes.byref(ph), dv.ptr(elem), dv.ptr(out), 1, s)
    else:
        x = dv.f32(g["x_corr"])
        out = torch.empty_like(x)
        _lib.call("dnnmg_rhs_next", ctypes.byref(lv), dv.ptr(x), ctypes.byref(ph), dv.ptr(elem),
                  dv.ptr(out), s)
    torch.cuda.synchronize()
    return out.double().cpu().numpy(), elem.double().cpu().numpy()


@pytest.mark.parametrize("stab_given", [False, True])
def test_k2tc_residual(case, stab_given):
    name, g, level = case
    r_tc, e_tc = run(level, g, True, "residual", stab_given)
    r_simt, e_simt = run(level, g, False, "residual", stab_given)
    assert rel(r_tc, g["r"]) < 2e-5, (name, rel(r_tc, g["r"]), rel(r_simt, g["r"]))
    assert rel(e_tc, e_simt) < 1e-5, (name, rel(e_tc, e_simt))
    assert np.all(r_tc[g["mask"]] == 0.0)


def test_k2tc_rhs_next(case):
    name, g, level = case
    b_tc, e_tc = run(level, g, True, "rhs", False)
    b_simt, _ = run(level, g, False, "rhs", False)
    assert rel(b_tc, g["b_next"]) < 2e-6, (name, rel(b_tc, g["b_next"]), rel(b_simt, g["b_next"]))


def test_k2tc_layout_choice():
    """config 0 (unjittered box) takes the per-cell affine record, a jittered mesh the
    per-point one."""
    for name, want in (("cfg0", True), ("jit", False)):
        g = load_golden(name)
        h = product_hierarchy(g)
        lvl = dv.DeviceLevel.get(spmod.FeSpace(h, int(g["L"]) + int(g["J"])))
        assert lvl.affine == want, name


@pytest.mark.parametrize("jitter", [False, True])
def test_k2tc_multi_tile(jitter):
    """Several 128-cell tiles per CTA (the next tile's nodes are prefetched during the stages,
    the previous tile's element vectors leave during the next tile's first stages) on a
    16x16x16 box (32,768 fine cells, 256 tiles on at most 148 CTAs): the tensor-core element
    kernel matches the SIMT one to fp32 rounding and repeats bit for bit."""
    from paper_2307_14837_b200 import mesh as meshmod, synthetic
    n = (16, 16, 16)
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1), n_cells=n)
    if jitter:
        synthetic.jitter_vertices(h.levels[0].vertices, n, (0, 0, 0), (1, 1, 1), 5)
    meshmod.refine_uniform(h)
    space = spmod.FeSpace(h, 1)
    level = dv.DeviceLevel.get(space)
    assert level.n_cells // 128 > 148
    gen = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(4 * space.n_nodes, device="cuda", generator=gen)
    b = torch.randn(4 * space.n_nodes, device="cuda", generator=gen) * 1e-3
    ph = _lib.Phys(1e-3, 5e-3, 0.02, 0.1, 1)
    elem = torch.empty(level.n_cells * 108, dtype=torch.float32, device="cuda")
    out = []
    for tc in (True, True, False):
        lv = level.struct(None, geometry=True, tc=tc)
        r = torch.empty_like(x)
        _lib.call("dnnmg_residual", ctypes.byref(lv), dv.ptr(x), dv.ptr(b), None, None,
                  ctypes.byref(ph), dv.ptr(elem), dv.ptr(r), 0, dv.stream_handle())
        torch.cuda.synchronize()
        out.append(r.double().cpu().numpy())
    assert np.array_equal(out[0], out[1])
    assert rel(out[0], out[2]) < 1e-6, rel(out[0], out[2])
