"""Bit-exact index maps at FULL BASELINE scale (configs 1, 2 and 3): the product's vectorised
mesh numbering, PatchSet tables, geometry features, constrained-dof mask and prolongation
matrix must hash byte-identically to the reference's own tables
(tests/golden/table_hashes.json, written by tests/golden/make_table_hashes.py from the
reference: mesh.py:162-216, 501-558; space.py:117-165; driver.py:56-65)."""
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

from paper_2307_14837_b200 import mesh as meshmod, synthetic  # noqa: E402
from paper_2307_14837_b200.space import FeSpace, prolongation_matrix, no_slip  # noqa: E402

HASHES = json.load(open(os.path.join(HERE, "golden", "table_hashes.json")))


def _digest():
    # the generator's canonical byte form, without importing the reference
    import hashlib

    def digest(a, kind):
        dt = np.int64 if kind == "i" else (np.float64 if kind == "f" else np.bool_)
        b = np.ascontiguousarray(np.asarray(a), dtype=dt)
        return hashlib.sha256(b.tobytes()).hexdigest() + f":{b.shape}"
    return digest


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_full_size_tables_hash_like_the_reference(name):
    if name not in HASHES:
        pytest.skip(f"no reference hashes for {name}")
    from paper_2307_14837_b200.step import constrained_mask
    digest = _digest()
    c = synthetic.CONFIGS[name]
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1),
                                    n_cells=c["n_cells"])
    if c["jitter"]:
        synthetic.jitter_vertices(h.levels[0].vertices, c["n_cells"], (0, 0, 0), (1, 1, 1),
                                  c["seed"] + 1)
    for _ in range(c["J"]):
        meshmod.refine_uniform(h)
    fl = c["J"]
    ps = meshmod.build_patches(h, 0, c["J"])
    fc, ft = h.scalar_nodes(fl)
    cc, _ = h.scalar_nodes(0)
    P = prolongation_matrix(h, 0).tocsr()
    mask = constrained_mask(FeSpace(h, fl), {meshmod.WALL: no_slip})
    got = {
        "fine_coords": digest(fc, "f"), "cell_nodes": digest(ft, "i"),
        "coarse_coords": digest(cc, "f"),
        "dof_table": digest(ps.dof_table, "i"), "node_table": digest(ps.node_table, "i"),
        "valence": digest(ps.valence, "i"), "mu": digest(ps.mu, "f"),
        "geom_table": digest(ps.geom_table, "f"), "mask": digest(mask, "b"),
        "P_indptr": digest(P.indptr, "i"), "P_indices": digest(P.indices, "i"),
        "P_data": digest(P.data, "f"),
    }
    want = HASHES[name]
    assert len(ps) == want["n_patches"]
    bad = [k for k in got if got[k] != want[k]]
    assert not bad, bad
