"""GPU parity at BASELINE config-1 scale (8,192 patches, jittered Q2 cells, 240 -> 256x3
-> 81 tanh, dt = 0.005) against the reference's own run (tests/golden/cfg1_pin.npz:
16,384 sampled dofs per vector plus every full vector's per-component norms; made by
tests/golden/make_cfg1.py).  Inputs are the same seeded coarse state and the carried
fine RHS b_prev in float64 (the oracle, itself pinned to the reference at this size by
test_oracle_cfg1.py), rounded to fp32 as in the cfg0 golden tests.

Tolerances (relative L2 on the sampled dofs, and relative error of every norm), the
same gates as test_gpu_parity.py: x~ 1e-7, r 2e-5, d and x_corr 1e-5 for fp32 / tf32x3
/ f16x3, 2e-2 for bf16; next RHS 2e-6.
"""
import numpy as np
import pytest

from golden_util import cfg1_case, sampled_rel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_14837_b200 import mesh as meshmod, synthetic  # noqa: E402
from paper_2307_14837_b200.net import Architecture, MlpModel  # noqa: E402
from paper_2307_14837_b200.step import CorrectionStep  # noqa: E402

TOL_D = {"fp32": 1e-5, "tf32x3": 1e-5, "f16x3": 1e-5, "bf16": 2e-2}


@pytest.fixture(scope="module")
def c1():
    c = cfg1_case()
    cfg = c["cfg"]
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1),
                                    n_cells=cfg["n_cells"])
    synthetic.jitter_vertices(h.levels[0].vertices, cfg["n_cells"], (0, 0, 0), (1, 1, 1),
                              cfg["seed"] + 1)
    meshmod.refine_uniform(h)
    c["h"] = h
    c["ps"] = meshmod.build_patches(h, 0, 1)
    W = c["W"]
    m = MlpModel(Architecture(W[0].shape[0], W[0].shape[1], len(W) - 1, W[-1].shape[1]),
                 activation="tanh")
    m.W = W
    c["model"] = m.eval()
    return c


def make_step(c1, precision):
    cfg = c1["cfg"]
    return CorrectionStep(c1["h"], 0, 1, c1["model"], cfg["nu"], cfg["dt"], precision=precision,
                          patchset=c1["ps"], t=cfg["dt"])


def check(name, v, pin, tol):
    e, en = sampled_rel(v.double().cpu().numpy(), pin, name)
    assert e < tol and en < tol, (name, e, en)


@pytest.mark.parametrize("precision", ["fp32", "tf32x3", "f16x3", "bf16"])
def test_cfg1_step(c1, precision):
    pin = c1["pin"]
    step = make_step(c1, precision)
    assert step.n_patches == 8192
    xc = torch.tensor(c1["x1"], dtype=torch.float32, device="cuda")
    b = torch.tensor(c1["b_prev"], dtype=torch.float32, device="cuda")
    out = step(xc, b)
    torch.cuda.synchronize()
    check("x_tilde", step.x_tilde, pin, 1e-7)
    check("r", step.r, pin, 2e-5)
    check("d", step.d, pin, TOL_D[precision])
    check("x_corr", out, pin, TOL_D[precision])
    if precision != "bf16":
        check("b_next", step.rhs_next(out), pin, 2e-6 + TOL_D[precision])
    # deterministic: a second run is bitwise identical
    assert torch.equal(out, step(xc, b))


def test_cfg1_carried_rhs_on_gpu(c1):
    """b_prev made on the GPU (embed x^0 at t = 0, then rhs_next) as the time loop does,
    and the step fed with it: the whole config-1 step without any float64 input."""
    pin = c1["pin"]
    step = make_step(c1, "f16x3")
    x0 = torch.tensor(c1["x0"], dtype=torch.float32, device="cuda")
    b = step.rhs_next(step.embed(x0, t=0.0))
    check("b_prev", b, pin, 2e-6)
    step.set_time(c1["cfg"]["dt"])
    out = step(torch.tensor(c1["x1"], dtype=torch.float32, device="cuda"), b)
    check("r", step.r, pin, 2e-5)
    check("x_corr", out, pin, 1e-5)
