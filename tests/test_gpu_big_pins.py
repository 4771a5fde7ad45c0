"""GPU parity at BASELINE config-2 and config-3 scale against the reference's own run
(tests/golden/cfg{2,3}_pin.npz: 16,384 sampled dofs per vector plus every full vector's
per-component norms; made by tests/golden/make_big.py on the reference's chunked
Assembler).

config 2: 65,536 patches of 5x5x5 nodes (J = 2), 1,024 -> 512x3 -> 375 (layered MLP);
config 3: 524,288 patches (J = 1), 240 -> 256x3 -> 81 (fused MLP), the bench workload.

Everything runs on the GPU as the time loop does: x^0 embedded at t = 0, the carried
fine RHS b_prev = rhs_next(x^0_fine) in fp32, then one correction step at t = dt.
Tolerances (relative L2 on the sampled dofs, and relative error of every norm), the
north-star gates of test_gpu_parity.py: x~ 1e-7, b_prev 2e-6, r 2e-5, d and x_corr 1e-5
(2e-2 for bf16), b_next 2e-6 + the d gate; the reference's sampled network-input rows X
through the product's MLP against its Y at the same gates.  Measured on B200
(tools/gpu/pin_errors.py, profiles/r1_parity_pins.txt): config 3 f16x3 d 2.0e-6, config 2
f16x3 d 3.8e-6.
"""
import os

import numpy as np
import pytest

from golden_util import load_golden, sampled_rel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_14837_b200 import mesh as meshmod, net, space as spmod, synthetic  # noqa: E402
from paper_2307_14837_b200.net import Architecture, MlpModel  # noqa: E402
from paper_2307_14837_b200.step import CorrectionStep  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
TOL_D = {"fp32": 1e-5, "tf32x3": 1e-5, "f16x3": 1e-5, "bf16": 2e-2}
_CACHE = {}


def problem(name):
    if name in _CACHE:
        return _CACHE[name]
    if not os.path.exists(os.path.join(HERE, "golden", f"{name}_pin.npz")):
        pytest.skip(f"{name}_pin.npz not generated")
    pin = load_golden(f"{name}_pin")
    cfg = synthetic.CONFIGS[name]
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1),
                                    n_cells=cfg["n_cells"])
    if cfg["jitter"]:
        synthetic.jitter_vertices(h.levels[0].vertices, cfg["n_cells"], (0, 0, 0), (1, 1, 1),
                                  cfg["seed"] + 1)
    for _ in range(cfg["J"]):
        meshmod.refine_uniform(h)
    ps = meshmod.build_patches(h, 0, cfg["J"])
    dims = [int(pin["n_in"])] + [cfg["hidden"]] * cfg["depth"] + [int(pin["n_out"])]
    m = MlpModel(Architecture(dims[0], cfg["hidden"], cfg["depth"], dims[-1]), activation="tanh")
    m.W = [w.astype(np.float64) for w in synthetic.xavier_weights(dims, cfg["seed"] + 7)]
    m.eval()
    modes = synthetic.fourier_modes(cfg["seed"])
    xyz = spmod.FeSpace(h, 0).nodes
    x0 = synthetic.coarse_state(xyz, modes, cfg["seed"], 0, 0.0, cfg["nu"])
    x1 = synthetic.coarse_state(xyz, modes, cfg["seed"], 1, cfg["dt"], cfg["nu"])
    assert np.isclose(np.linalg.norm(x1), float(pin["x_coarse_norm"]), rtol=1e-15)
    _CACHE[name] = dict(cfg=cfg, h=h, ps=ps, model=m, x0=x0, x1=x1, pin=pin)
    return _CACHE[name]


def check(name, v, pin, tol):
    e, en = sampled_rel(v.double().cpu().numpy(), pin, name)
    assert e < tol and en < tol, (name, e, en)


@pytest.mark.parametrize("name,precision", [("cfg2", "f16x3"), ("cfg2", "bf16"),
                                            ("cfg3", "f16x3"), ("cfg3", "fp32")])
def test_big_config_step(name, precision):
    c = problem(name)
    cfg, pin = c["cfg"], c["pin"]
    step = CorrectionStep(c["h"], 0, cfg["J"], c["model"], cfg["nu"], cfg["dt"],
                          precision=precision, patchset=c["ps"], t=0.0)
    assert step.n_patches == int(pin["n_patches"])
    assert step.x_tilde.numel() == int(pin["ndof"])
    b = step.rhs_next(step.embed(torch.tensor(c["x0"], dtype=torch.float32, device="cuda")))
    check("b_prev", b, pin, 2e-6)
    step.set_time(cfg["dt"])
    out = step(torch.tensor(c["x1"], dtype=torch.float32, device="cuda"), b)
    torch.cuda.synchronize()
    check("x_tilde", step.x_tilde, pin, 1e-7)
    check("r", step.r, pin, 2e-5)
    check("d", step.d, pin, TOL_D[precision])
    check("x_corr", out, pin, TOL_D[precision])
    if precision != "bf16":
        check("b_next", step.rhs_next(out), pin, 2e-6 + TOL_D[precision])
    # the product's OWN gathered network-input rows (dnnmg_gather over its index tables) at
    # the reference's sampled patches: the geometry block bit-exact, the x~ / r blocks at the
    # x~ / r gates (a wrong node map would show O(1) errors)
    from paper_2307_14837_b200 import patch_ops
    X = patch_ops.assemble_network_input(step.x_tilde, step.r, c["ps"])
    rows = torch.as_tensor(pin["rows"].astype(np.int64), device="cuda")
    Xs = X[rows].cpu().numpy()
    nd = 4 * c["ps"].nodes_per_patch
    assert np.array_equal(Xs[:, 2 * nd:], pin["X"][:, 2 * nd:])
    ex = np.linalg.norm(Xs[:, :nd] - pin["X"][:, :nd]) / np.linalg.norm(pin["X"][:, :nd])
    er = np.linalg.norm(Xs[:, nd:2 * nd] - pin["X"][:, nd:2 * nd]) / np.linalg.norm(
        pin["X"][:, nd:2 * nd])
    assert ex < 1e-7 and er < 2e-5, (ex, er)
    del X
    # the reference's own network input rows through the product's MLP
    Y = net.forward(c["model"], pin["X"].astype(np.float64), precision=precision)
    assert np.linalg.norm(Y - pin["Y"]) / np.linalg.norm(pin["Y"]) < TOL_D[precision]
