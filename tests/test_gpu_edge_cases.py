"""Edge cases on the GPU path: empty batches and empty windows, a single row, ragged tile
counts, and the error behaviour the reference's tests pin (ValueError wording)."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_14837_b200 import driver, io as iomod, net, patch_ops, mesh as meshmod  # noqa: E402


def _model(n_in, H, n_out, seed=0):
    m = net.MlpModel(net.Architecture(n_in, H, 3, n_out), activation="tanh", seed=seed)
    m.eval()
    return m


@pytest.mark.parametrize("precision", ["fp32", "f16x3", "tf32x3", "bf16", "fp8"])
@pytest.mark.parametrize("H", [128, 256, 512])
def test_mlp_empty_and_single_row(precision, H):
    if precision == "fp8" and H % 64:
        pytest.skip("fp8 widths are multiples of 64")
    m = _model(174, H, 81, seed=H)
    Y0 = net.forward(m, np.zeros((0, 174)), precision=precision)
    assert Y0.shape == (0, 81)
    x = np.random.default_rng(1).standard_normal((1, 174))
    y1 = net.forward(m, x, precision=precision)
    y2 = net.forward(m, np.repeat(x, 300, axis=0), precision=precision)[-1:]
    assert y1.shape == (1, 81) and np.isfinite(y1).all()
    # a row's result does not depend on where in a (ragged) batch it sits
    assert np.array_equal(y1, y2)


def test_mlp_width_errors():
    m = _model(174, 128, 81)
    with pytest.raises(ValueError, match="width"):
        net.forward(m, np.zeros((4, 170)), precision="f16x3")


def test_predict_correction_length_error():
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1), n_cells=(2, 1, 1))
    meshmod.refine_uniform(h)
    ps = meshmod.build_patches(h, 0, 1)
    m = _model(patch_ops.input_width(ps), 32, patch_ops.output_width(ps))
    n = ps.mu.shape[0]
    with pytest.raises(ValueError, match="length"):
        patch_ops.predict_correction(m, np.zeros(n + 4), np.zeros(n), ps, precision="f16x3")


def test_export_with_an_empty_window(tmp_path):
    """A validation window that contains no step gives an empty set: no shards, zero
    rows and widths, zero statistics — as io.write_dataset does for rows == 0."""
    from test_gpu_dataset import Problem, DS
    pr = Problem()
    ct = iomod.Trajectory(os.path.join(DS, "coarse.dmgt"))
    ft = iomod.Trajectory(os.path.join(DS, "fine.dmgt"))
    path = driver.export_training_data(pr, 0, 1, ct, ft, (0.02, 0.06), (5.0, 6.0), tmp_path)
    meta = json.loads(path.read_text())
    v = meta["sets"]["val"]
    assert v["rows"] == 0 and v["shards"] == [] and v["n_features"] == 0
    assert all(x == 0.0 for st in v["component_stats"].values() for x in st.values())
    X, T, _ = iomod.load_dataset(path, "val")
    assert X.shape[0] == 0 and T.shape[0] == 0
    assert meta["sets"]["train"]["rows"] == 2 * 16


def test_graph_replay_follows_time_dependent_dirichlet():
    """set_time with a ramped inflow updates the Dirichlet data in place, so a captured
    CUDA graph replays at the new time; a twin keeps its own copy."""
    from paper_2307_14837_b200 import space as spmod
    from paper_2307_14837_b200.step import CorrectionStep
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, -0.205), extent_hi=(1.0, 0.41, 0.205),
                                    n_cells=(3, 2, 2), channel_tags=True)
    meshmod.refine_uniform(h)
    bcs = {meshmod.INFLOW: spmod.inflow_profile(3, 1.0, 0.41), meshmod.WALL: spmod.no_slip}
    ps = meshmod.build_patches(h, 0, 1)
    m = _model(patch_ops.input_width(ps), 256, patch_ops.output_width(ps), seed=3)
    step = CorrectionStep(h, 0, 1, m, 1e-3, 0.01, bcs=bcs, precision="f16x3", patchset=ps, t=0.05)
    rng = np.random.default_rng(0)
    nc = spmod.FeSpace(h, 0).n_nodes
    xc = torch.tensor(rng.standard_normal(4 * nc), dtype=torch.float32, device="cuda")
    b = torch.tensor(rng.standard_normal(4 * step.space.n_nodes) * 1e-2, dtype=torch.float32,
                     device="cuda")
    twin = step.twin()
    g = step.capture(xc, b)
    step.set_time(0.4)
    g.replay()
    torch.cuda.synchronize()
    got = step.x_corr.clone()
    fresh = CorrectionStep(h, 0, 1, m, 1e-3, 0.01, bcs=bcs, precision="f16x3", patchset=ps, t=0.4)
    want = fresh(xc, b)
    assert torch.equal(got, want)
    # the twin still runs at t = 0.05
    at05 = CorrectionStep(h, 0, 1, m, 1e-3, 0.01, bcs=bcs, precision="f16x3", patchset=ps, t=0.05)
    assert torch.equal(twin(xc, b), at05(xc, b))
    assert not torch.equal(got, at05(xc, b))
