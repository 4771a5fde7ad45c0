"""Training-data export on the GPU against the dataset the
REFERENCE's ``driver.export_training_data`` wrote from the same trajectories
(tests/golden/dataset, made by tests/golden/make_dataset.py).

Shard names, headers and row counts must match exactly (the byte layout of
io.write_dataset, io.py:219-266); feature and target rows match the float64 reference
within the fp32 tolerances of the correction path (x~ dyadic prolongation ~1e-7,
residual ~1e-5); the loop pass replays the reference's recorded coarse Newton solves
(the coarse solver is out of scope) and checks the coarse RHS it is handed; the
self-consistency export has exactly zero targets and zero residual rows.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_14837_b200 import driver, io as iomod, mesh as meshmod, space as spmod, synthetic  # noqa: E402
from paper_2307_14837_b200.step import constrained_mask  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
DS = os.path.join(HERE, "golden", "dataset")
LO, HI, NC = (0, 0, -0.205), (1.0, 0.41, 0.205), (2, 1, 1)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


class Problem:
    """Duck-typed NsProblem; solve_step replays the reference's recorded coarse solves."""

    def __init__(self):
        h = meshmod.build_template_mesh("box", extent_lo=LO, extent_hi=HI, n_cells=NC,
                                        channel_tags=True)
        synthetic.jitter_vertices(h.levels[0].vertices, NC, LO, HI, 21)
        meshmod.refine_uniform(h)
        self.hierarchy = h
        self.nu, self.k = 1e-3, 0.02
        self.bcs = {meshmod.INFLOW: spmod.inflow_profile(3, 1.5, 0.41), meshmod.WALL: spmod.no_slip}
        self.alpha0, self.delta0 = 0.02, 0.1
        self.f = None
        self.convection = True
        self.reimpose_fine_dirichlet = True
        with np.load(os.path.join(DS, "solves.npz")) as z:
            self.solves = {k: z[k] for k in z.files}
        self.i = 0
        self.b_err = []

    def space(self, level):
        return spmod.FeSpace(self.hierarchy, level)

    def mask(self, level):
        return constrained_mask(self.space(level), self.bcs)

    def solve_step(self, level, x_prev, b, t, solver=None):
        i = self.i
        self.i += 1
        assert abs(t - self.solves["t"][i]) < 1e-12
        self.b_err.append(rel(np.asarray(b), self.solves["b"][i]))
        return spmod.StateVector(level, self.solves["x"][i].copy(), t), None, solver


@pytest.mark.parametrize("which", ["loop", "self"])
def test_export_matches_reference(tmp_path, which):
    pr = Problem()
    ct = iomod.Trajectory(os.path.join(DS, "coarse.dmgt" if which == "loop" else "fine.dmgt"))
    ft = iomod.Trajectory(os.path.join(DS, "fine.dmgt"))
    path = driver.export_training_data(pr, 0, 1, ct, ft, (0.02, 0.06), (0.06, 0.1), tmp_path,
                                       shard_bytes=30000, loop_pass=(which == "loop"))
    mine = json.loads(path.read_text())
    ref_path = os.path.join(DS, which, "dataset.json")
    theirs = json.loads(open(ref_path).read())
    assert mine["layout"] == theirs["layout"]
    if which == "loop":
        assert pr.i == len(pr.solves["t"]) and max(pr.b_err) < 1e-5, pr.b_err
    for name in ("train", "val"):
        a, b = mine["sets"][name], theirs["sets"][name]
        assert a["shards"] == b["shards"]
        assert (a["rows"], a["n_features"], a["n_targets"]) == (b["rows"], b["n_features"], b["n_targets"])
        for shard in a["shards"]:       # headers identical (40 bytes)
            assert (tmp_path / shard).read_bytes()[:40] == open(os.path.join(DS, which, shard), "rb").read(40)
        X, T, _ = iomod.load_dataset(path, name)
        Xr, Tr, _ = iomod.load_dataset(ref_path, name)
        nd = mine["layout"]["n_dof_patch"]
        assert rel(X[:, :nd], Xr[:, :nd]) < 1e-6                    # state rows
        assert rel(X[:, 2 * nd:], Xr[:, 2 * nd:]) < 1e-6            # geometry rows
        if which == "self":
            assert np.all(X[:, nd:2 * nd] == 0.0) and np.all(T == 0.0) and np.all(Tr == 0.0)
        else:
            assert rel(X[:, nd:2 * nd], Xr[:, nd:2 * nd]) < 2e-5    # residual rows
            assert rel(T, Tr) < 1e-5, rel(T, Tr)                    # targets
        np.testing.assert_allclose(a["feature_mean"], b["feature_mean"], rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(a["feature_std"], b["feature_std"], rtol=1e-5, atol=1e-6)
        for c, st in b["component_stats"].items():
            for k, v in st.items():
                assert a["component_stats"][c][k] == pytest.approx(v, rel=1e-5, abs=1e-6)


def test_replay_features_matches_time_loop_machinery():
    """replay_features = embed + residual against a carried RHS (driver.py:294-314)."""
    pr = Problem()
    ct = iomod.Trajectory(os.path.join(DS, "coarse.dmgt"))
    xp = driver.embed_state(pr, 0, 1, ct.values(2), 2 * pr.k)
    from paper_2307_14837_b200.assembly import Assembler
    asm = Assembler(pr.space(1))
    b_prev = asm.assemble_rhs_next(xp, None, None, pr.k, pr.nu)
    xt, r = driver.replay_features(pr, 0, 1, ct.values(3), b_prev, 3 * pr.k)
    xt2 = driver.embed_state(pr, 0, 1, ct.values(3), 3 * pr.k)
    assert np.array_equal(xt, xt2)
    stab = asm.stab(xt, pr.nu, pr.k)
    r2 = asm.assemble_residual(xt, b_prev, pr.k, pr.nu, stab, mask=pr.mask(1))
    assert rel(r, r2) < 1e-5       # stab fused into K2 vs the separate stab kernel
