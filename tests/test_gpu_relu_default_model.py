"""The reference's DEFAULT network through the correction step at BASELINE config-1 scale:
Architecture(240, 64, 8, 81) with relu (config.py:69-71; MlpModel default activation,
net.py:39-57), trained-style BN statistics and input normalisation.

Relu hidden states are unbounded, so the fp16 hi/lo split of f16x3 is not safe for them:
requesting f16x3 runs the model in tf32x3 (net.effective_precision; the C ABI rejects
f16x3 + relu with DNNMG_ERR_UNSUPPORTED), and d must still meet the fp32 gate (1e-5)
against the float64 oracle (itself pinned to the reference at this size by
tests/test_oracle_cfg1.py)."""
import warnings

import numpy as np
import pytest

from golden_util import cfg1_case

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import dnnmg_oracle as orc  # noqa: E402
from paper_2307_14837_b200 import mesh as meshmod, synthetic  # noqa: E402
from paper_2307_14837_b200.net import Architecture, MlpModel  # noqa: E402
from paper_2307_14837_b200.step import CorrectionStep  # noqa: E402


def rel(a, b):
    return np.linalg.norm(np.asarray(a, float) - b) / np.linalg.norm(b)


def default_model(seed=71):
    """Reference defaults (hidden 64, depth 8, relu, He-uniform init) with trained-style
    BN statistics and input normalisation; weights rounded to fp32 values."""
    m = MlpModel(Architecture(240, 64, 8, 81), activation="relu", seed=seed)
    m.W = [w.astype(np.float32).astype(np.float64) for w in m.W]
    rng = np.random.default_rng(seed + 1)
    H, depth = 64, 8
    m.gamma = [rng.uniform(0.5, 1.5, H) for _ in range(depth)]
    m.beta = [rng.normal(0, 0.1, H) for _ in range(depth)]
    m.running_mean = [rng.normal(0, 0.2, H) for _ in range(depth)]
    m.running_var = [rng.uniform(0.5, 2.0, H) for _ in range(depth)]
    m.set_input_norm(rng.normal(0, 0.3, 240), rng.uniform(0.05, 2.0, 240))
    return m.eval()


def test_default_relu_model_cfg1():
    c = cfg1_case()
    cfg, ctx = c["cfg"], c["ctx"]
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1),
                                    n_cells=cfg["n_cells"])
    synthetic.jitter_vertices(h.levels[0].vertices, cfg["n_cells"], (0, 0, 0), (1, 1, 1),
                              cfg["seed"] + 1)
    meshmod.refine_uniform(h)
    m = default_model()
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        step = CorrectionStep(h, 0, 1, m, cfg["nu"], cfg["dt"], precision="f16x3",
                              t=cfg["dt"])
    assert step.model.requested_precision == "f16x3"
    assert step.precision == step.model.precision == "tf32x3"
    assert any("bounded activation" in str(x.message) for x in w)
    assert step.layered       # hidden 64: the layer-major tcgen05 kernel
    xc = torch.tensor(c["x1"], dtype=torch.float32, device="cuda")
    b = torch.tensor(c["b_prev"], dtype=torch.float32, device="cuda")
    out = step(xc, b)
    torch.cuda.synchronize()
    om = orc.Mlp(m.W, "relu", m.gamma, m.beta, m.running_mean, m.running_var, m.input_mean,
                 m.input_std)
    x1 = c["x1"].astype(np.float32).astype(np.float64)
    bp = c["b_prev"].astype(np.float32).astype(np.float64)
    ref = orc.correction_step(x1, bp, ctx, om, cfg["dt"], cfg["nu"], cfg["dt"])
    # the hidden states do leave the tanh range: relu with 8 skips grows them
    hid = np.abs(orc.mlp_forward(orc.Mlp(m.W[:-1] + [np.eye(64)], "relu", m.gamma, m.beta,
                                         m.running_mean, m.running_var, m.input_mean,
                                         m.input_std), ref["X"][:512])).max()
    assert hid > 8.0, hid
    assert rel(step.d.double().cpu().numpy(), ref["d"]) < 1e-5
    assert rel(out.double().cpu().numpy(), ref["x_corr"]) < 1e-5
