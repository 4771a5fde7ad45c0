"""GPU parity: every kernel of the correction path against the reference's own
golden output (tests/golden, produced by running dnnmg) and the reference's
property tests, through the product's drop-in API and the C ABI.

Tolerances (relative L2 against the float64 reference):
  index maps / gathers: exact (fp32 rounding of the same values)
  x~ (prolongation, dyadic weights): 1e-7
  r (residual, fp32 with cancellation b - A): 2e-5
  Y, d, x_corr in fp32 mode: 1e-5 (north-star gate)
"""
import copy

import numpy as np
import pytest

from conftest import GOLDEN_CASES
from golden_util import load_golden, product_hierarchy, product_model, product_bcs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_14837_b200 import mesh as meshmod, space as spmod, patch_ops, net  # noqa: E402
from paper_2307_14837_b200.assembly import Assembler, StabParams  # noqa: E402
from paper_2307_14837_b200.step import CorrectionStep, constrained_mask  # noqa: E402


def rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module", params=GOLDEN_CASES)
def case(request):
    g = load_golden(request.param)
    h = product_hierarchy(g)
    L, J = int(g["L"]), int(g["J"])
    s = spmod.FeSpace(h, L + J)
    ps = meshmod.build_patches(h, L, J)
    return request.param, g, h, s, ps


def test_prolongate_and_dirichlet(case):
    name, g, h, s, ps = case
    L, J = int(g["L"]), int(g["J"])
    xt = spmod.prolongate(h, spmod.StateVector(L, g["x_coarse"].copy()), J)
    assert xt.level == L + J
    spmod.apply_dirichlet(s, xt, float(g["t"]), product_bcs(g))
    assert rel(xt.values, g["x_tilde"]) < 1e-7


def test_prolongation_forms_bitwise(case):
    """K1's table forms: the owner-list kernel and the lattice kernel (lat_node) write the same
    bits, with the Dirichlet codes gathered, in owner order, or packed into the lattice table
    (dnnmg_dirichlet_t.lat_node_bc); the per-fine-node kernel (fine_src only: products of the
    three 1-D weights in one sum) agrees to fp32 rounding; every fine node is written exactly
    once."""
    import ctypes
    from paper_2307_14837_b200 import _lib, device as dv
    name, g, h, s, ps = case
    L, J = int(g["L"]), int(g["J"])
    P = dv.DeviceProlong.get(h, L + J - 1)
    assert np.array_equal(np.sort(P.lat_host[P.lat_host >= 0]), np.arange(P.n_fine))
    rng = np.random.default_rng(11)
    xc = torch.tensor(rng.standard_normal(4 * P.n_coarse_nodes), dtype=torch.float32, device="cuda")
    code, vals = dv.dirichlet_codes(s, float(g["t"]), product_bcs(g))
    dcode = dv.upload(code, np.uint8)
    dvals = None if vals is None else dv.upload(vals, np.float32)
    downer = dv.upload(np.asarray(code, np.uint8)[P.owner_order], np.uint8)
    dlat = dv.upload(P.lattice_with_codes(code), np.int32)
    n_f, n_c = P.n_fine, P.lat_host.shape[0]
    base = (dv.ptr(P.ctab), dv.ptr(P.src))
    owner = (dv.ptr(P.owner_ptr), dv.ptr(P.owner_node), dv.ptr(P.owner_code))
    forms = {"owner": _lib.Prolong(n_f, n_c, *base, *owner),
             "lattice": _lib.Prolong(n_f, n_c, *base, *owner, dv.ptr(P.lat_node)),
             "node": _lib.Prolong(n_f, n_c, *base)}
    bcs = {"none": None,
           "gathered": _lib.Dirichlet(n_f, dv.ptr(dcode), dv.ptr(dvals)),
           "owner": _lib.Dirichlet(n_f, dv.ptr(dcode), dv.ptr(dvals), dv.ptr(downer)),
           "packed": _lib.Dirichlet(n_f, dv.ptr(dcode), dv.ptr(dvals), dv.ptr(downer), dv.ptr(dlat))}
    ref = {}
    for fname, F in forms.items():
        for bname, B in bcs.items():
            out = torch.full((4 * n_f,), float("nan"), dtype=torch.float32, device="cuda")
            _lib.call("dnnmg_prolongate", ctypes.byref(F), dv.ptr(xc), dv.ptr(out),
                      None if B is None else ctypes.byref(B), dv.stream_handle())
            torch.cuda.synchronize()
            assert not torch.isnan(out).any(), (fname, bname)
            key = "none" if bname == "none" else "bc"
            if key not in ref:
                ref[key] = out
            if fname == "node":
                assert rel(out.cpu().numpy(), ref[key].cpu().numpy()) < 1e-6, (fname, bname)
            else:
                assert torch.equal(out, ref[key]), (fname, bname)


def test_stab(case):
    name, g, h, s, ps = case
    st = Assembler(s).stab(g["x_tilde"], float(g["nu"]), float(g["k"]))
    assert rel(st.alpha_T, g["alpha_T"]) < 1e-6
    assert rel(st.delta_T, g["delta_T"]) < 1e-6


def test_residual(case):
    name, g, h, s, ps = case
    asm = Assembler(s)
    st = StabParams(float(g["alpha0"]), float(g["delta0"]), g["alpha_T"], g["delta_T"])
    r = asm.assemble_residual(g["x_tilde"], g["b_prev"], float(g["k"]), float(g["nu"]), st,
                              mask=g["mask"])
    assert rel(r, g["r"]) < 2e-5, rel(r, g["r"])
    assert np.all(r[g["mask"]] == 0.0)
    # stab evaluated inside the kernel (alpha_T = None) gives the same residual
    r2 = asm.assemble_residual(g["x_tilde"], g["b_prev"], float(g["k"]), float(g["nu"]),
                               StabParams(), mask=g["mask"])
    assert rel(r2, g["r"]) < 2e-5


def test_rhs_next(case):
    name, g, h, s, ps = case
    b = Assembler(s).assemble_rhs_next(g["x_corr"], None, None, float(g["k"]), float(g["nu"]))
    assert rel(b, g["b_next"]) < 2e-6, rel(b, g["b_next"])


def test_network_input_exact(case):
    name, g, h, s, ps = case
    X = patch_ops.assemble_network_input(g["x_tilde"], g["r"], ps)
    assert np.array_equal(X, g["X"].astype(np.float32).astype(np.float64))


def test_forward_fp32(case):
    name, g, h, s, ps = case
    Y = net.forward(product_model(g), g["X"], precision="fp32")
    assert rel(Y, g["Y"]) < 1e-5, rel(Y, g["Y"])


def test_predict_correction_fp32(case):
    name, g, h, s, ps = case
    d = patch_ops.predict_correction(product_model(g), g["x_tilde"], g["r"], ps,
                                     dirichlet_mask=g["mask"], precision="fp32")
    assert rel(d, g["d"]) < 1e-5, rel(d, g["d"])
    assert np.all(d.reshape(-1, 4)[:, 0] == 0.0)
    assert np.all(d[g["mask"]] == 0.0)


def test_fused_step_fp32(case):
    name, g, h, s, ps = case
    L, J = int(g["L"]), int(g["J"])
    step = CorrectionStep(h, L, J, product_model(g), float(g["nu"]), float(g["k"]),
                          bcs=product_bcs(g), scale=float(g["scale"]), precision="fp32",
                          patchset=ps, t=float(g["t"]))
    xc = torch.tensor(g["x_coarse"], dtype=torch.float32, device="cuda")
    b = torch.tensor(g["b_prev"], dtype=torch.float32, device="cuda")
    out = step(xc, b).double().cpu().numpy()
    torch.cuda.synchronize()
    assert rel(step.x_tilde.cpu().numpy(), g["x_tilde"]) < 1e-7
    assert rel(step.r.cpu().numpy(), g["r"]) < 2e-5
    assert rel(step.d.cpu().numpy(), g["d"]) < 1e-5
    assert rel(out, g["x_corr"]) < 1e-5
    # deterministic: a second run is bitwise identical
    out2 = step(xc, b).double().cpu().numpy()
    assert np.array_equal(out, out2)


# ---- reference property tests (test_patch_ops.py) on the GPU -------------------------

@pytest.fixture(scope="module")
def ps3():
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1), n_cells=(3, 2, 2))
    meshmod.refine_uniform(h)
    return meshmod.build_patches(h, 0, 1)


def test_local_restrict_is_pure_gather(ps3):
    n = ps3.mu.shape[0]
    rows = patch_ops.local_restrict(np.arange(n, dtype=float), ps3)
    assert np.array_equal(rows, ps3.dof_table.astype(float))
    assert np.all(patch_ops.local_restrict(np.full(n, 3.25), ps3) == 3.25)
    with pytest.raises(ValueError, match="length"):
        patch_ops.local_restrict(np.zeros(n + 1), ps3)


def test_extend_restrict_identity(ps3):
    x = np.random.default_rng(3).standard_normal(ps3.mu.shape[0]).astype(np.float32)
    back = patch_ops.global_extend(patch_ops.local_restrict(x, ps3), ps3)
    assert np.abs(back - x).max() < 1e-6


def test_shared_dof_average(ps3):
    dof = int(np.nonzero(1.0 / ps3.mu >= 2)[0][0])
    owners = np.nonzero((ps3.dof_table == dof).any(axis=1))[0]
    rows = np.zeros((len(ps3), ps3.ndof_patch))
    slot = np.nonzero(ps3.dof_table[owners[0]] == dof)[0][0]
    rows[owners[0], slot] = 5.0
    out = patch_ops.global_extend(rows, ps3)
    assert out[dof] == pytest.approx(5.0 / owners.size, rel=1e-7)


def _model(ps, seed, hidden=12, depth=2):
    return net.MlpModel(net.Architecture(patch_ops.input_width(ps), hidden, depth,
                                         patch_ops.output_width(ps)), seed=seed).eval()


def test_zero_weight_model_zero_defect(ps3):
    m = net.zero_weights(_model(ps3, 0))
    rng = np.random.default_rng(1)
    n = ps3.mu.shape[0]
    d = patch_ops.predict_correction(m, rng.standard_normal(n), rng.standard_normal(n), ps3)
    assert np.all(d == 0.0)


def test_permutation_invariance(ps3):
    m = _model(ps3, 3)
    rng = np.random.default_rng(2)
    n = ps3.mu.shape[0]
    xt, r = rng.standard_normal(n), rng.standard_normal(n)
    d1 = patch_ops.predict_correction(m, xt, r, ps3)
    assert np.abs(d1).max() > 0 and np.all(d1.reshape(-1, 4)[:, 0] == 0.0)
    perm = rng.permutation(len(ps3))
    sh = copy.copy(ps3)
    sh.__dict__ = {k: v for k, v in ps3.__dict__.items() if k != "_b200_device"}
    sh.dof_table = ps3.dof_table[perm]
    sh.node_table = ps3.node_table[perm]
    sh.geom_table = ps3.geom_table[perm]
    d2 = patch_ops.predict_correction(m, xt, r, sh)
    assert np.abs(d1 - d2).max() < 1e-5 * np.abs(d1).max()


def test_model_patch_mismatch_rejected(ps3):
    n = ps3.mu.shape[0]
    bad = net.MlpModel(net.Architecture(10, 8, 2, 4), seed=0).eval()
    with pytest.raises(ValueError, match="architecture"):
        patch_ops.predict_correction(bad, np.zeros(n), np.zeros(n), ps3)
    tr = _model(ps3, 0).train()
    with pytest.raises(ValueError, match="eval"):
        patch_ops.predict_correction(tr, np.zeros(n), np.zeros(n), ps3)


def test_zero_state_zero_residual(ps3):
    """test_assembly.py:31-37 on the GPU."""
    h = ps3.hierarchy
    s = spmod.FeSpace(h, 1)
    asm = Assembler(s)
    x = np.zeros(s.ndof)
    st = asm.stab(x, 1e-2, 0.1)
    r = asm.assemble_residual(x, np.zeros_like(x), 0.1, 1e-2, st, mask=s.dirichlet_mask())
    assert np.all(r == 0.0)


# ---- tensor-core MLP modes (tcgen05): fp32-accurate 3xTF32 and bf16 ----------------------

TC_TOL = {"tf32x3": 1e-5, "f16x3": 1e-5, "bf16": 2e-2}


@pytest.mark.parametrize("precision", ["tf32x3", "f16x3", "bf16"])
def test_forward_tc_cfg0(precision):
    g = load_golden("cfg0")
    Y = net.forward(product_model(g), g["X"], precision=precision)
    assert rel(Y, g["Y"]) < TC_TOL[precision], rel(Y, g["Y"])


@pytest.mark.parametrize("precision", ["tf32x3", "f16x3", "bf16"])
def test_predict_correction_tc_cfg0(precision):
    g = load_golden("cfg0")
    h = product_hierarchy(g)
    ps = meshmod.build_patches(h, 0, 1)
    d = patch_ops.predict_correction(product_model(g), g["x_tilde"], g["r"], ps,
                                     dirichlet_mask=g["mask"], precision=precision)
    assert rel(d, g["d"]) < TC_TOL[precision], rel(d, g["d"])


@pytest.mark.parametrize("precision", ["tf32x3", "f16x3", "bf16"])
def test_fused_step_tc_cfg0(precision):
    g = load_golden("cfg0")
    h = product_hierarchy(g)
    step = CorrectionStep(h, 0, 1, product_model(g), float(g["nu"]), float(g["k"]),
                          precision=precision, t=float(g["t"]))
    xc = torch.tensor(g["x_coarse"], dtype=torch.float32, device="cuda")
    b = torch.tensor(g["b_prev"], dtype=torch.float32, device="cuda")
    step(xc, b)
    torch.cuda.synchronize()
    assert rel(step.d.cpu().numpy(), g["d"]) < TC_TOL[precision]


@pytest.mark.parametrize("precision", ["tf32x3", "f16x3", "bf16"])
@pytest.mark.parametrize("shape", [(240, 3, 81, "tanh", 1000, False), (174, 3, 81, "tanh", 4097, False),
                                   (240, 4, 81, "relu", 300, True), (256, 1, 200, "tanh", 129, True)])
def test_forward_tc_random(precision, shape):
    """Random rows (ragged tile counts), BN stats, input norm, relu/tanh; the
    float64 oracle MLP (net.py:124-159) is the reference."""
    from oracle import dnnmg_oracle as orc
    n_in, depth, n_out, act, rows, bn = shape
    rng = np.random.default_rng(n_in + rows)
    m = net.MlpModel(net.Architecture(n_in, 256, depth, n_out), activation=act, seed=rows)
    dims = [n_in] + [256] * depth + [n_out]
    m.W = [(rng.uniform(-1, 1, (a, b)) * np.sqrt(6.0 / (a + b))).astype(np.float32).astype(float)
           for a, b in zip(dims[:-1], dims[1:])]
    if bn:
        m.gamma = [rng.uniform(0.5, 1.5, 256) for _ in range(depth)]
        m.beta = [rng.normal(0, 0.1, 256) for _ in range(depth)]
        m.running_mean = [rng.normal(0, 0.2, 256) for _ in range(depth)]
        m.running_var = [rng.uniform(0.5, 2.0, 256) for _ in range(depth)]
        m.set_input_norm(rng.normal(0, 0.3, n_in), rng.uniform(0.5, 2.0, n_in))
    m.eval()
    X = rng.standard_normal((rows, n_in)).astype(np.float32).astype(float)
    ref = orc.mlp_forward(orc.Mlp(m.W, act, m.gamma, m.beta, m.running_mean, m.running_var,
                                  m.input_mean, m.input_std), X)
    Y = net.forward(m, X, precision=precision)
    assert rel(Y, ref) < TC_TOL[precision], rel(Y, ref)
    Y32 = net.forward(m, X, precision="fp32")
    assert rel(Y32, ref) < 1e-5


def test_tc_rejects_unsupported_width():
    """Hidden widths that are not a multiple of 32 have no tensor-core path (the layered
    kernel tiles N in 32-column groups); widths like 128 run layer by layer."""
    m = net.MlpModel(net.Architecture(240, 100, 3, 81), activation="tanh").eval()
    with pytest.raises(NotImplementedError):
        net.forward(m, np.zeros((4, 240)), precision="bf16")
    m = net.MlpModel(net.Architecture(240, 128, 3, 81), activation="tanh").eval()
    assert np.isfinite(net.forward(m, np.zeros((4, 240)), precision="bf16")).all()


@pytest.mark.parametrize("lanes", [1, 2])
@pytest.mark.parametrize("precision", ["fp32", "f16x3"])
def test_host_pipeline_matches_run(precision, lanes):
    """step.HostPipeline (H2D / kernels / D2H overlapped on three streams,
    double-buffered) returns exactly what CorrectionStep.run returns per step."""
    from paper_2307_14837_b200.step import HostPipeline
    g = load_golden("cfg0")
    h = product_hierarchy(g)
    step = CorrectionStep(h, 0, 1, product_model(g), float(g["nu"]), float(g["k"]),
                          precision=precision, t=float(g["t"]))
    rng = np.random.default_rng(5)
    ins = []
    for i in range(5):
        xc = (g["x_coarse"] * (1.0 + 0.1 * i) + 0.01 * rng.standard_normal(g["x_coarse"].shape))
        b = g["b_prev"] * (1.0 - 0.05 * i)
        ins.append((torch.tensor(xc, dtype=torch.float32).pin_memory(),
                    torch.tensor(b, dtype=torch.float32).pin_memory()))
    ref = []
    for xc, b in ins:
        ref.append(step(xc.cuda(), b.cuda()).cpu().clone())
    outs = [torch.empty_like(ref[0]).pin_memory() for _ in ins]
    pipe = HostPipeline(step, lanes=lanes)
    pipe.begin()
    for (xc, b), o in zip(ins, outs):
        pipe.submit(xc, b, o)
    pipe.join()
    torch.cuda.synchronize()
    for o, r in zip(outs, ref):
        assert torch.equal(o, r)


@pytest.mark.parametrize("wscale", [1e-6, 1.0, 3e3])
def test_f16x3_weight_scaling(wscale):
    """f16x3 keeps fp32-level accuracy for tiny and large weights: each GEMM's weights
    are rescaled by an exact power of two at pack time (mlp_tc.cu pack_scale_kernel)
    and the inverse is folded into the BN scale / head output."""
    from oracle import dnnmg_oracle as orc
    rng = np.random.default_rng(11)
    n_in, depth, n_out, rows = 240, 3, 81, 777
    m = net.MlpModel(net.Architecture(n_in, 256, depth, n_out), activation="tanh", seed=3)
    dims = [n_in] + [256] * depth + [n_out]
    m.W = [rng.uniform(-1, 1, (a, b)) * np.sqrt(6.0 / (a + b)) * wscale for a, b in zip(dims[:-1], dims[1:])]
    # keep the pre-activations O(1): BN scale undoes the weight scale of the hidden layers
    m.gamma = [np.full(256, 1.0 / wscale) for _ in range(depth)]
    m.beta = [rng.normal(0, 0.1, 256) for _ in range(depth)]
    m.running_mean = [np.zeros(256) for _ in range(depth)]
    m.running_var = [np.ones(256) - m.bn_eps for _ in range(depth)]
    m.eval()
    X = rng.standard_normal((rows, n_in))
    ref = orc.mlp_forward(orc.Mlp(m.W, "tanh", m.gamma, m.beta, m.running_mean, m.running_var,
                                  m.input_mean, m.input_std), X)
    Y = net.forward(m, X, precision="f16x3")
    assert rel(Y, ref) < 1e-5, rel(Y, ref)


# ---- restriction P^T (next row #1, space.py:188-196) ---------------------------------------

def _golden_P(g, i):
    import scipy.sparse as sp
    ind = g[f"P{i}_indptr"]
    nf = ind.size - 1
    nc = int(g[f"P{i}_indices"].max()) + 1 if g[f"P{i}_indices"].size else 0
    return sp.csr_matrix((g[f"P{i}_data"], g[f"P{i}_indices"], ind), shape=(nf, nc))


@pytest.mark.parametrize("name", ["cfg0", "jit", "j2", "lvl1"])
def test_restrict_rhs_is_Pt(name):
    """restrict_rhs(b, L+J, J) == (P^T)^J b with the reference's own P (golden CSR)."""
    import scipy.sparse as sp
    g = load_golden(name)
    h = product_hierarchy(g)
    L, J = int(g["L"]), int(g["J"])
    ref = g["b_next"].astype(float)
    for i in reversed(range(L, L + J)):
        P = _golden_P(g, i)
        ref = sp.kron(P, sp.identity(4, format="csr"), format="csr").T @ ref
    got = spmod.restrict_rhs(h, g["b_next"], L + J, J)
    assert got.shape == ref.shape
    assert rel(got, ref) < 1e-6, rel(got, ref)
    assert np.all(spmod.restrict_rhs(h, np.zeros_like(g["b_next"]), L + J, J) == 0.0)


def test_restrict_transpose_pairing():
    """test_space.py:52-59 on the GPU: b . (P x) == (P^T b) . x."""
    g = load_golden("jit")
    h = product_hierarchy(g)
    rng = np.random.default_rng(3)
    nc = 4 * h.scalar_nodes(0)[0].shape[0]
    nf = 4 * h.scalar_nodes(1)[0].shape[0]
    x = rng.standard_normal(nc)
    b = rng.standard_normal(nf)
    Px = spmod.prolongate(h, spmod.StateVector(0, x, 0.0)).values
    Ptb = spmod.restrict_rhs(h, b, 1, 1)
    lhs, rhs = b @ Px, Ptb @ x
    assert abs(lhs - rhs) < 1e-5 * (np.abs(b) @ np.abs(Px) + 1.0), (lhs, rhs)


@pytest.mark.parametrize("name", ["cfg0", "jit", "chan"])
def test_geometry_cache_matches_recomputed(name):
    """K2 with the per-mesh geometry cache (J^-1, w per Gauss point, fp64 setup) gives the
    same residual as the path that recomputes the isoparametric geometry per call, and
    both match the reference."""
    import ctypes
    from paper_2307_14837_b200 import _lib, device as dv
    g = load_golden(name)
    h = product_hierarchy(g)
    L, J = int(g["L"]), int(g["J"])
    s = spmod.FeSpace(h, L + J)
    lvl = dv.DeviceLevel.get(s)
    mask = dv.upload(dv.dof_mask_bits(g["mask"], s.n_nodes), np.uint8)
    xt = torch.tensor(g["x_tilde"], dtype=torch.float32, device="cuda")
    b = torch.tensor(g["b_prev"], dtype=torch.float32, device="cuda")
    ph = _lib.Phys(float(g["nu"]), float(g["k"]), float(g["alpha0"]), float(g["delta0"]), 1)
    out = []
    for geo in (False, True):
        lv = lvl.struct(mask, geometry=geo, box=False)
        r = torch.empty_like(xt)
        _lib.call("dnnmg_residual", ctypes.byref(lv), dv.ptr(xt), dv.ptr(b), None, None,
                  ctypes.byref(ph), dv.ptr(lvl.scratch()), dv.ptr(r), 1, dv.stream_handle())
        torch.cuda.synchronize()
        out.append(r.cpu().numpy().astype(float))
    assert rel(out[1], out[0]) < 1e-5, rel(out[1], out[0])
    # the cached geometry is formed in fp64: at least as close to the reference
    assert rel(out[1], g["r"]) < 2e-5, rel(out[1], g["r"])
    assert rel(out[1], g["r"]) <= 1.2 * rel(out[0], g["r"]) + 1e-9


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_box_geometry_matches_cached(name):
    """K2's box form (levels of axis-aligned cells: per-cell (1/hx, 1/hy, 1/hz, det J), no
    products with the zero off-diagonal entries of J^-1) against the per-point geometry cache
    on the same level, residual and next-step RHS; a jittered level must not get the record."""
    import ctypes
    from paper_2307_14837_b200 import _lib, device as dv
    g = load_golden(name)
    h = product_hierarchy(g)
    L, J = int(g["L"]), int(g["J"])
    s = spmod.FeSpace(h, L + J)
    lvl = dv.DeviceLevel.get(s)
    box = lvl.geometry_box()
    # the device check (27 nodes of every cell on the box lattice, fp64) on any level
    rec = torch.empty(max(lvl.n_cells, 1) * 4, dtype=torch.float32, device="cuda")
    bad = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    _lib.call("dnnmg_level_geometry_box", ctypes.byref(lvl.struct()), dv.ptr(rec), dv.ptr(bad),
              dv.stream_handle())
    if box is None:
        assert int(bad.item()) > 0, (name, lvl.geo_kind, int(bad.item()))
        assert not lvl.struct(None, geometry=True).geo_box
        return
    assert int(bad.item()) == 0
    assert name != "jit"
    X = np.asarray(s.nodes)[np.asarray(s.cell_nodes)]
    hx = X[:, 2, 0] - X[:, 0, 0]
    assert np.allclose(rec.cpu().numpy().reshape(-1, 4)[:, 0], 1.0 / hx, rtol=1e-6)
    mask = dv.upload(dv.dof_mask_bits(g["mask"], s.n_nodes), np.uint8)
    xt = torch.tensor(g["x_tilde"], dtype=torch.float32, device="cuda")
    b = torch.tensor(g["b_prev"], dtype=torch.float32, device="cuda")
    ph = _lib.Phys(float(g["nu"]), float(g["k"]), float(g["alpha0"]), float(g["delta0"]), 1)
    res, rhs = [], []
    for use_box in (False, True):
        lv = lvl.struct(mask, geometry=True, tc=False, box=use_box)
        assert bool(lv.geo_box) == use_box and bool(lv.geo_q) == (not use_box)
        r = torch.empty_like(xt)
        _lib.call("dnnmg_residual", ctypes.byref(lv), dv.ptr(xt), dv.ptr(b), None, None,
                  ctypes.byref(ph), dv.ptr(lvl.scratch()), dv.ptr(r), 1, dv.stream_handle())
        bn = torch.empty_like(xt)
        _lib.call("dnnmg_rhs_next", ctypes.byref(lv), dv.ptr(xt), ctypes.byref(ph),
                  dv.ptr(lvl.scratch()), dv.ptr(bn), dv.stream_handle())
        torch.cuda.synchronize()
        res.append(r.cpu().numpy().astype(float))
        rhs.append(bn.cpu().numpy().astype(float))
    assert rel(res[1], res[0]) < 2e-6, rel(res[1], res[0])
    assert rel(rhs[1], rhs[0]) < 1e-6, rel(rhs[1], rhs[0])
    assert rel(res[1], g["r"]) < 2e-5, rel(res[1], g["r"])


@pytest.mark.parametrize("name", ["cfg0", "jit", "j2", "lvl1", "chan"])
def test_restrict_owner_form_matches_csr_form(name):
    """K6 owner-computes form (transpose of K1's per-cell stencil + ordered node sum) against
    the P^T CSR form on the same vector: equal to fp32 rounding."""
    import ctypes
    from paper_2307_14837_b200 import _lib, device as dv
    g = load_golden(name)
    h = product_hierarchy(g)
    L, J = int(g["L"]), int(g["J"])
    R = dv.DeviceRestrict.get(h, L + J - 1)
    b = torch.tensor(np.random.default_rng(7).standard_normal(4 * R.n_fine), dtype=torch.float32,
                     device="cuda")
    outs = []
    for owner in (True, False):
        st = _lib.Restrict()
        ctypes.memmove(ctypes.addressof(st), ctypes.addressof(R.struct), ctypes.sizeof(st))
        if not owner:
            st.owner_ptr = None
        out = torch.empty(4 * R.n_coarse, dtype=torch.float32, device="cuda")
        _lib.call("dnnmg_restrict", ctypes.byref(st), dv.ptr(b), dv.ptr(out), dv.stream_handle())
        outs.append(out.double().cpu().numpy())
    assert R.struct.owner_ptr is not None
    assert rel(outs[0], outs[1]) < 1e-6, rel(outs[0], outs[1])
