"""Drop-in check: the product consumes objects that only carry the reference's
public attributes (dnnmg MeshLevel / MeshHierarchy / PatchSet / MlpModel,
mesh.py:60-220, 501-564; net.py:32-70), not this package's own classes.

``RefLevel`` / ``RefHierarchy`` / ``RefModel`` below expose exactly the
reference's attribute names (``dim, vertices, cells, parent_of,
boundary_faces, n_cells``; ``dim, levels, scalar_nodes(level), top``;
``arch, W, gamma, beta, running_mean, running_var, bn_eps, input_mean,
input_std, activation, mode``) and nothing else.  The reference package itself
cannot be imported on the GPU box, so the objects are filled from a golden
case; the host-side index maps are compared on CPU and the full correction
step on the GPU.
"""
import numpy as np
import pytest

from golden_util import load_golden, product_hierarchy, product_model


class RefLevel:
    def __init__(self, lvl):
        self.dim = 3
        self.vertices = np.array(lvl.vertices, dtype=float)
        self.cells = np.array(lvl.cells, dtype=np.int64)
        self.parent_of = None
        self.boundary_faces = [tuple(int(v) for v in f) for f in np.asarray(lvl.boundary_faces)]

    @property
    def n_cells(self):
        return self.cells.shape[0]


class RefHierarchy:
    """Reference-shaped hierarchy: levels + scalar_nodes(level) + top."""

    def __init__(self, h):
        self.dim = 3
        self.levels = [RefLevel(lvl) for lvl in h.levels]
        self._nodes = [tuple(np.array(a) for a in h.scalar_nodes(l)) for l in range(len(h.levels))]

    def scalar_nodes(self, level):
        return self._nodes[level]

    @property
    def top(self):
        return len(self.levels) - 1


class RefModel:
    def __init__(self, m):
        self.arch = m.arch
        self.W = [np.array(w) for w in m.W]
        self.gamma = [np.array(v) for v in m.gamma]
        self.beta = [np.array(v) for v in m.beta]
        self.running_mean = [np.array(v) for v in m.running_mean]
        self.running_var = [np.array(v) for v in m.running_var]
        self.bn_eps = m.bn_eps
        self.input_mean = np.array(m.input_mean)
        self.input_std = np.array(m.input_std)
        self.activation = m.activation
        self.mode = "eval"


@pytest.mark.parametrize("case", ["cfg0", "chan"])
def test_host_maps_from_reference_shaped_objects(case):
    from paper_2307_14837_b200 import mesh as meshmod, space as spmod
    g = load_golden(case)
    h = product_hierarchy(g)
    rh = RefHierarchy(h)
    L, J = int(g["L"]), int(g["J"])
    s_ref, s_own = spmod.FeSpace(rh, L + J), spmod.FeSpace(h, L + J)
    assert np.array_equal(s_ref.nodes, s_own.nodes)
    assert np.array_equal(s_ref.node_tags, s_own.node_tags)
    assert np.array_equal(s_ref.dirichlet_mask(), s_own.dirichlet_mask())
    for l in range(L, L + J):
        assert np.array_equal(spmod.prolongation_source(rh, l), spmod.prolongation_source(h, l))
    p_ref, p_own = meshmod.build_patches(rh, L, J), meshmod.build_patches(h, L, J)
    assert np.array_equal(p_ref.node_table, p_own.node_table)
    assert np.array_equal(p_ref.dof_table, g["dof_table"])
    assert np.array_equal(p_ref.mu, p_own.mu)
    assert np.allclose(p_ref.geom_table, p_own.geom_table, rtol=0, atol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["cfg0", "jit"])
def test_step_from_reference_shaped_objects(case):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2307_14837_b200.step import CorrectionStep
    g = load_golden(case)
    rh = RefHierarchy(product_hierarchy(g))
    model = RefModel(product_model(g))
    L, J = int(g["L"]), int(g["J"])
    step = CorrectionStep(rh, L, J, model, float(g["nu"]), float(g["k"]), t=float(g["t"]))
    xc = torch.tensor(g["x_coarse"], dtype=torch.float32, device="cuda")
    b = torch.tensor(g["b_prev"], dtype=torch.float32, device="cuda")
    step(xc, b)
    torch.cuda.synchronize()
    d = step.d.cpu().numpy().astype(float)
    assert np.linalg.norm(d - g["d"]) / np.linalg.norm(g["d"]) < 1e-5
