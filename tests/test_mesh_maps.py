"""CPU tests of the product's host-side index maps (bit-exact vs the reference's
golden output) and the reference's mesh/patch property tests (test_mesh.py,
test_patch_ops.py, test_space.py) restated for the product mesh module."""
import numpy as np
import pytest

from golden_util import load_golden, product_hierarchy
from paper_2307_14837_b200 import mesh as meshmod, space as spmod
from paper_2307_14837_b200.step import constrained_mask
from conftest import GOLDEN_CASES


@pytest.fixture(scope="module", params=GOLDEN_CASES)
def case(request):
    g = load_golden(request.param)
    return request.param, g, product_hierarchy(g)


def test_numbering_bit_exact(case):
    name, g, h = case
    L, J = int(g["L"]), int(g["J"])
    coords, table = h.scalar_nodes(L + J)
    assert np.array_equal(table, g["cell_nodes"])
    assert np.array_equal(coords, g["fine_coords"])
    assert np.array_equal(h.scalar_nodes(L)[0], g["coarse_coords"])


def test_patch_tables_bit_exact(case):
    name, g, h = case
    ps = meshmod.build_patches(h, int(g["L"]), int(g["J"]))
    assert np.array_equal(ps.dof_table, g["dof_table"])
    assert np.array_equal(ps.node_table, g["node_table"])
    assert np.array_equal(ps.valence, g["valence"])
    assert np.array_equal(ps.mu, g["mu"])
    assert np.abs(ps.geom_table - g["geom"]).max() < 1e-14


def test_tags_and_mask_bit_exact(case):
    name, g, h = case
    s = spmod.FeSpace(h, int(g["L"]) + int(g["J"]))
    assert np.array_equal(s.node_tags, g["node_tags"])
    bcs = {meshmod.INFLOW: None, meshmod.WALL: None} if int(g["channel"]) else {meshmod.WALL: None}
    assert np.array_equal(constrained_mask(s, bcs), g["mask"])


def test_prolongation_bit_exact(case):
    name, g, h = case
    L, J = int(g["L"]), int(g["J"])
    for l in range(L, L + J):
        P = spmod.prolongation_matrix(h, l)
        assert np.array_equal(P.indptr, g[f"P{l}_indptr"])
        assert np.array_equal(P.indices, g[f"P{l}_indices"])
        assert np.array_equal(P.data, g[f"P{l}_data"])


def test_dof_counts_per_patch():
    """N_dof^P in {108, 500} for 3-D (test_mesh.py:116-122)."""
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1), n_cells=(1, 1, 1))
    meshmod.refine_uniform(h)
    meshmod.refine_uniform(h)
    assert meshmod.build_patches(h, 0, 1).ndof_patch == 108
    assert meshmod.build_patches(h, 0, 2).ndof_patch == 500
    with pytest.raises(ValueError, match="J"):
        meshmod.build_patches(h, 0, 3)
    with pytest.raises(ValueError):
        meshmod.build_patches(h, 1, 2)


def test_patches_partition_fine_cells():
    """Fine cells of all patches form a partition (test_mesh.py:125-131)."""
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(2, 1, 1), n_cells=(2, 1, 1))
    for _ in range(2):
        meshmod.refine_uniform(h)
    ps = meshmod.build_patches(h, 0, 2)
    cells = np.concatenate([p.fine_cells for p in ps])
    assert np.array_equal(np.sort(cells), np.arange(h.levels[2].n_cells))
    # local_to_global is injective per patch (test_mesh.py:134-136)
    assert all(np.unique(p.local_to_global).size == p.local_to_global.size for p in ps)


def test_unit_cube_features():
    """Edges 1, diagonals sqrt(3), angles pi/2 (test_mesh.py:144-150)."""
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1), n_cells=(1, 1, 1))
    f = meshmod.geometry_features_of_cells(h.levels[0], np.array([0]))[0]
    assert np.allclose(f[:12], 1.0) and np.allclose(f[12:16], np.sqrt(3.0))
    assert np.allclose(f[16:], np.pi / 2)


def test_valence_counts_integer():
    """1/mu is the integer patch-membership count (test_patch_ops.py:42-49)."""
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1), n_cells=(3, 2, 2))
    meshmod.refine_uniform(h)
    ps = meshmod.build_patches(h, 0, 1)
    inv = 1.0 / ps.mu
    assert np.all(inv == np.round(inv))
    counts = np.zeros_like(ps.mu)
    for p in ps.patches:
        counts[p.local_to_global] += 1.0
    assert np.array_equal(counts, inv)
    assert set(np.unique(inv).tolist()) <= {1.0, 2.0, 4.0, 8.0}


def test_nodes_nested():
    """Q2 nodes of level l lead the numbering of level l+1 (test_space.py:20-24)."""
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1), n_cells=(2, 1, 1))
    for _ in range(2):
        meshmod.refine_uniform(h)
    for l in (0, 1):
        c0, _ = h.scalar_nodes(l)
        c1, _ = h.scalar_nodes(l + 1)
        assert np.array_equal(c1[:c0.shape[0]], c0)


def test_prolongation_reproduces_quadratics():
    """The Q2 embedding is exact: the nodal values of a global Q2 polynomial are
    mapped to its fine nodal values (test_space.py:25-41, any size)."""
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 2, 1), n_cells=(3, 2, 2))
    meshmod.refine_uniform(h)
    P = spmod.prolongation_matrix(h, 0)
    f = lambda x: 1 + x[:, 0] - 2 * x[:, 1] ** 2 + x[:, 0] * x[:, 2] + 0.5 * x[:, 2] ** 2
    c0, _ = h.scalar_nodes(0)
    c1, _ = h.scalar_nodes(1)
    assert np.abs(P @ f(c0) - f(c1)).max() < 1e-12
    assert np.abs(P @ np.ones(c0.shape[0]) - 1.0).max() < 1e-14


def test_non_box_templates_rejected():
    with pytest.raises(NotImplementedError):
        meshmod.build_template_mesh("channel_cylinder_3d")


def test_tile_tables_cover_node_table():
    """Per-tile distinct-node tables of the staged fused gather (device.tile_tables):
    nodes[t][slot[p][s]] == node_table[p][s], lists ascending and duplicate-free."""
    from paper_2307_14837_b200 import device as dv
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1),
                                    n_cells=(5, 4, 3))
    meshmod.refine_uniform(h)
    nt = np.asarray(meshmod.build_patches(h, 0, 1).node_table)
    cap, nodes, count, slot = dv.tile_tables(nt)
    assert count.size == (nt.shape[0] + 127) // 128 and cap >= count.max()
    for t in range(count.size):
        rows = nt[128 * t:128 * (t + 1)]
        assert np.array_equal(nodes[t][slot[128 * t:128 * t + len(rows)].astype(np.int64)], rows)
        assert np.all(np.diff(nodes[t][:count[t]]) > 0)
        assert count[t] == np.unique(rows).size


def test_lattice_table_reproduces_prolongation(case):
    """K1's lattice table (device.lattice_table: the owned fine node at every position of each
    parent cell's 5 x 5 x 5 lattice) against the prolongation matrix that is pinned bit-exact
    above: the tensor product of the 1-D quarter-point stencils at a node's lattice position, on
    its parent's 27 nodes, is exactly that node's row of P; every fine node is owned once."""
    from paper_2307_14837_b200 import device as dv
    name, g, h = case
    L, J = int(g["L"]), int(g["J"])
    w1 = {0: {0: 1.0}, 1: {0: 0.375, 1: 0.75, 2: -0.125}, 2: {1: 1.0},
          3: {0: -0.125, 1: 0.75, 2: 0.375}, 4: {2: 1.0}}
    for l in range(L, L + J):
        P = spmod.prolongation_matrix(h, l).tocsr()
        ctab = h.scalar_nodes(l)[1]
        src = spmod.prolongation_source(h, l)
        lat = dv.lattice_table(src, ctab.shape[0])
        assert lat.shape == (ctab.shape[0], 125)
        owned = lat[lat >= 0]
        assert np.array_equal(np.sort(owned), np.arange(P.shape[0]))
        rng = np.random.default_rng(5)
        cells = rng.choice(ctab.shape[0], size=min(40, ctab.shape[0]), replace=False)
        for C in cells:
            for pos in np.nonzero(lat[C] >= 0)[0]:
                n = lat[C, pos]
                px, py, pz = pos % 5, (pos // 5) % 5, pos // 25
                row = {}
                for iz, wz in w1[pz].items():
                    for iy, wy in w1[py].items():
                        for ix, wx in w1[px].items():
                            m = ctab[C, 9 * iz + 3 * iy + ix]
                            row[m] = row.get(m, 0.0) + wx * wy * wz
                ref = dict(zip(P.indices[P.indptr[n]:P.indptr[n + 1]],
                               P.data[P.indptr[n]:P.indptr[n + 1]]))
                assert row == ref, (l, C, pos, n)
