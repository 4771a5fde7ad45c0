"""The oracle at BASELINE config-1 scale (8,192 patches, jittered, 240 -> 256x3 -> 81)
against the reference's own run (tests/golden/cfg1_pin.npz: sampled dofs and full-vector
norms, made by tests/golden/make_cfg1.py).  ~5 s on one core."""
import numpy as np
import pytest

from oracle import dnnmg_oracle as orc
from golden_util import cfg1_case, sampled_rel


@pytest.fixture(scope="module")
def c1():
    return cfg1_case()


def test_cfg1_sizes(c1):
    pin, ctx = c1["pin"], c1["ctx"]
    assert int(pin["n_patches"]) == ctx["dof_table"].shape[0] == 8192
    assert int(pin["ndof"]) == ctx["coords"].shape[0] * 4
    assert int(pin["n_masked"]) == int(ctx["mask"].sum())
    assert np.isclose(np.linalg.norm(c1["x1"]), float(pin["x_coarse_norm"]), rtol=1e-15)
    assert np.isclose(np.linalg.norm(c1["x0"]), float(pin["x0_coarse_norm"]), rtol=1e-15)


def test_cfg1_oracle_step_matches_reference(c1):
    pin, ctx, cfg = c1["pin"], c1["ctx"], c1["cfg"]
    e, en = sampled_rel(c1["b_prev"], pin, "b_prev")
    assert e < 1e-14 and en < 1e-14
    model = orc.Mlp(c1["W"], activation="tanh")
    out = orc.correction_step(c1["x1"], c1["b_prev"], ctx, model, cfg["dt"], cfg["nu"], cfg["dt"])
    for name, tol in (("x_tilde", 1e-15), ("r", 1e-12), ("d", 1e-12), ("x_corr", 1e-12)):
        e, en = sampled_rel(out[name], pin, name)
        assert e < tol and en < tol, (name, e, en)
    rows = pin["rows"]
    assert np.array_equal(out["X"][rows].astype(np.float32), pin["X"])
    assert np.linalg.norm(out["Y"][rows] - pin["Y"]) / np.linalg.norm(pin["Y"]) < 1e-12
    assert np.allclose(out["alpha_T"][pin["cells"]], pin["alpha_T"], rtol=1e-14, atol=0)
    assert np.allclose(out["delta_T"][pin["cells"]], pin["delta_T"], rtol=1e-14, atol=0)
    b = orc.rhs_next(out["x_corr"], ctx["coords"], ctx["table"], cfg["dt"], cfg["nu"])
    e, en = sampled_rel(b, pin, "b_next")
    assert e < 1e-13 and en < 1e-13
