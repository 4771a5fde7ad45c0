"""Cell-Vanka smoother on the GPU against the REFERENCE's own
VankaData / vanka_smooth (tests/golden/vanka.npz, made by make_vanka.py): the Jacobian
of a jittered channel box assembled by the reference (convection, LPS stabilisation),
its 108 x 108 cell blocks inverted on the device, 4 damped sweeps
(msolve.py:51-89).  Float64 throughout: inverses and sweeps agree to ~1e-12."""
import numpy as np
import pytest
import scipy.sparse as sp

from golden_util import load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_14837_b200 import msolve  # noqa: E402


class Asm:
    """The reference Assembler attributes VankaData reads."""

    def __init__(self, g):
        self.cell_dofs = g["cell_dofs"]
        self.n_cells, self.ndl = self.cell_dofs.shape
        self.flat_pos = g["flat_pos"]

        class S:
            ndof = int(g["ndof"])
        self.space = S()


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b)


@pytest.fixture(scope="module")
def g():
    return load_golden("vanka")


def jac(g, data=None):
    n = int(g["ndof"])
    return sp.csr_matrix((g["data"] if data is None else data, g["indices"], g["indptr"]), shape=(n, n))


def test_vanka_matches_reference(g):
    J = jac(g)
    V = msolve.VankaData(Asm(g), J)
    assert V.flagged == [] and len(g["flagged"]) == 0
    assert np.array_equal(V.weight, g["weight"])
    assert rel(V.inv[0].cpu().numpy(), g["inv0"]) < 1e-11
    blocks = g["data"][g["flat_pos"]].reshape(V.n_cells, V.ndl, V.ndl)
    eye = np.eye(V.ndl)
    for c in range(V.n_cells):
        assert np.abs(V.inv[c].cpu().numpy() @ blocks[c] - eye).max() < 1e-9
    x4 = msolve.vanka_smooth(J, V, g["x0"].copy(), g["b"], 4, 0.7)
    assert rel(x4, g["x4"]) < 1e-11, rel(x4, g["x4"])
    # device form: in place on float64 CUDA tensors, same result
    xd = torch.tensor(g["x0"], dtype=torch.float64, device="cuda")
    bd = torch.tensor(g["b"], dtype=torch.float64, device="cuda")
    out = msolve.vanka_smooth(J, V, xd, bd, 4, 0.7)
    assert out is xd and np.array_equal(xd.cpu().numpy(), x4)


def test_vanka_one_sweep_is_the_reference_formula(g):
    J = jac(g)
    V = msolve.VankaData(Asm(g), J)
    x0, b = g["x0"], g["b"]
    r = b - J @ x0
    inv = V.inv.cpu().numpy()
    dl = np.einsum("cij,cj->ci", inv, r[V.dofs])
    upd = np.bincount(V.dofs.reshape(-1), weights=dl.reshape(-1), minlength=V.ndof)
    ref = x0 + 0.7 * (V.weight * upd)
    assert rel(msolve.vanka_smooth(J, V, x0.copy(), b, 1, 0.7), ref) < 1e-13


def test_singular_block_is_shifted_and_flagged(g):
    data = g["data"].copy()
    fp = g["flat_pos"].reshape(-1, 108 * 108)
    data[fp[1]] = 0.0                               # cell 1's block (and the entries it shares)
    J = jac(g, data)
    V = msolve.VankaData(Asm(g), J)
    blocks = data[g["flat_pos"]].reshape(V.n_cells, V.ndl, V.ndl)
    flagged = []
    for c in range(V.n_cells):                      # the reference's fallback (msolve.py:62-72)
        try:
            ref = np.linalg.inv(blocks[c])
        except np.linalg.LinAlgError:
            ref = np.linalg.inv(blocks[c] + 1e-12 * np.eye(V.ndl))
            flagged.append(c)
        assert rel(V.inv[c].cpu().numpy(), ref) < 1e-9
    assert V.flagged == flagged == [1]


def test_length_mismatch_rejected(g):
    J = jac(g)
    V = msolve.VankaData(Asm(g), J)
    with pytest.raises(ValueError, match="length"):
        msolve.vanka_smooth(sp.identity(10, format="csr"), V, np.zeros(10), np.zeros(10), 1, 0.7)
