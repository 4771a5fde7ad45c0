"""The hybrid time loop with the fine level on the GPU against the REFERENCE's own
``driver.TimeLoop`` trajectory (tests/golden/timeloop.npz, made by
tests/golden/make_timeloop.py in the build container).

The coarse Newton/GMRES/multigrid solve is the caller's (out of scope): a replay
problem hands the loop the reference's coarse solutions x^n and records the coarse
right-hand sides the loop passes to it.  Everything the loop carries on the fine level
is the product's: Dirichlet re-imposition at t_n (time-dependent inflow ramp),
residual against the carried fine RHS, the network correction (gated by
correction_start, damped by correction_scale), the next fine RHS and its restriction
(driver.py:201-280).  Tolerances are relative L2 against the float64 reference; the
fine RHS is carried in fp32 across steps, so errors accumulate slightly.
"""
import numpy as np
import pytest

from golden_util import load_golden, product_model

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_14837_b200 import driver, mesh as meshmod, space as spmod, synthetic  # noqa: E402
from paper_2307_14837_b200.step import constrained_mask  # noqa: E402


def rel(a, b):
    a = a.double().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, float)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


class ReplayProblem:
    """Duck-typed NsProblem whose coarse solve replays the reference's solutions."""

    def __init__(self, g):
        n_cells = tuple(int(v) for v in g["n_cells"])
        h = meshmod.build_template_mesh("box", extent_lo=g["lo"], extent_hi=g["hi"],
                                        n_cells=n_cells, channel_tags=True)
        synthetic.jitter_vertices(h.levels[0].vertices, n_cells, g["lo"], g["hi"], int(g["jitter"]))
        for _ in range(int(g["L"]) + int(g["J"])):
            meshmod.refine_uniform(h)
        self.hierarchy = h
        self.nu, self.k = float(g["nu"]), float(g["k"])
        self.bcs = {meshmod.INFLOW: spmod.inflow_profile(3, float(g["vbar"]), 0.41),
                    meshmod.WALL: spmod.no_slip}
        self.alpha0, self.delta0 = float(g["alpha0"]), float(g["delta0"])
        self.f = None
        self.convection = True
        self.reimpose_fine_dirichlet = True
        self.g = g
        self.received_b = []
        self._spaces = {}

    def space(self, level):
        if level not in self._spaces:
            self._spaces[level] = spmod.FeSpace(self.hierarchy, level)
        return self._spaces[level]

    def mask(self, level):
        return constrained_mask(self.space(level), self.bcs)

    def solve_step(self, level, x_prev, b, t, solver=None):
        n = len(self.received_b) + 1
        self.received_b.append(np.array(b))
        assert abs(t - float(self.g[f"t_{n}"])) < 1e-12
        x = spmod.StateVector(level, self.g[f"x_{n}"].copy(), t)
        return x, None, solver


@pytest.fixture(scope="module")
def g():
    return load_golden("timeloop")


@pytest.mark.parametrize("precision", ["fp32", "f16x3", "tf32x3"])
def test_timeloop_matches_reference(g, precision):
    pr = ReplayProblem(g)
    model = product_model(g)
    loop = driver.TimeLoop(pr, int(g["L"]), J=int(g["J"]), model=model,
                           correction_scale=float(g["scale"]), correction_start=float(g["start"]),
                           precision=precision)
    st = loop.state
    assert rel(st.x.values, g["x_0"]) < 1e-14
    assert rel(st.x_fine.values, g["x_fine_0"]) < 1e-6
    assert rel(st.b_next_fine, g["b_next_fine_0"]) < 1e-5
    assert rel(st.b_next, g["b_next_0"]) < 1e-5
    steps = int(g["steps"])
    for n in range(1, steps + 1):
        st = loop.step()
        assert st.n == n and abs(st.t - float(g[f"t_{n}"])) < 1e-12
        # the coarse RHS the loop handed to the solver is the reference's b_next^{n-1}
        assert rel(pr.received_b[-1], g[f"b_next_{n - 1}"]) < 1e-5, n
        e_x = rel(st.x_fine.values, g[f"x_fine_{n}"])
        e_bf = rel(st.b_next_fine, g[f"b_next_fine_{n}"])
        e_b = rel(st.b_next, g[f"b_next_{n}"])
        assert e_x < 1e-5 and e_bf < 2e-5 and e_b < 2e-5, (n, e_x, e_bf, e_b)
    # corrections started at t >= correction_start only
    assert loop.net_evals == sum(float(g[f"t_{n}"]) >= float(g["start"]) - 1e-12
                                 for n in range(1, steps + 1))
    assert [s.n for s in loop.step_log] == list(range(1, steps + 1))


def test_timeloop_without_model_is_zero_correction(g):
    pr = ReplayProblem(g)
    loop = driver.TimeLoop(pr, int(g["L"]), J=int(g["J"]), model=None)
    st = loop.step()
    xt = loop.fine.embed(st.x.values)
    assert torch.equal(st.x_fine.values, xt)
    assert loop.net_evals == 0


def test_timeloop_rejects_unsupported(g):
    pr = ReplayProblem(g)
    with pytest.raises(NotImplementedError):
        driver.TimeLoop(pr, 0, J=0)
    pr.f = lambda t, pts: np.zeros((pts.shape[0], 3))
    with pytest.raises(NotImplementedError):
        driver.TimeLoop(pr, 0, J=1)


class ResumeReplay(ReplayProblem):
    """Replays the reference's coarse solutions of a resumed run."""

    def __init__(self, g, r, name):
        super().__init__(g)
        self.r, self.name = r, name

    def solve_step(self, level, x_prev, b, t, solver=None):
        n = len(self.received_b) + 1
        self.received_b.append(np.array(b))
        assert abs(t - float(self.r[f"{self.name}_t_{n}"])) < 1e-12
        return spmod.StateVector(level, self.r[f"{self.name}_x_{n}"].copy(), t), None, solver


@pytest.mark.parametrize("name", ["hybrid", "mg"])
def test_resume_from_reference_checkpoint(g, name):
    """driver.resume_loop on a checkpoint the reference wrote mid-run (hybrid, and pure-MG
    resumed as hybrid with the fine RHS rebuilt on the device) continues like the
    reference's own resumed loop (driver.py:453-480)."""
    import os
    r = load_golden("timeloop_resume")
    pr = ResumeReplay(g, r, name)
    ck = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", f"timeloop_{name}.dmgc")
    loop = driver.resume_loop(pr, ck, model=product_model(g), J=int(g["J"]), precision="f16x3",
                              correction_scale=float(g["scale"]), correction_start=float(g["start"]))
    assert rel(loop.state.b_next_fine, r[f"{name}_b_next_fine_0"]) < 1e-5
    # the coarse RHS the first resumed solve receives (for 'mg': the restriction of the
    # rebuilt fine RHS, driver.py:476-478)
    assert rel(loop.state.b_next, r[f"{name}_b_next_0"]) < 2e-5
    for n in (1, 2):
        st = loop.step()
        assert rel(pr.received_b[n - 1], r[f"{name}_b_next_{n - 1}"]) < 2e-5, n
        assert rel(st.x_fine.values, r[f"{name}_x_fine_{n}"]) < 1e-5, n
        assert rel(st.b_next_fine, r[f"{name}_b_next_fine_{n}"]) < 2e-5, n
        assert rel(st.b_next, r[f"{name}_b_next_{n}"]) < 2e-5, n
    # checkpoint_state of the resumed loop round-trips through the reference format
    n, t, arrays, meta = driver.checkpoint_state(loop)
    assert n == 4 and meta["J"] == int(g["J"]) and "b_next_fine" in arrays
