"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  Index maps must be bit-exact; float results
agree to ~1e-12 relative (different but equivalent summation orders)."""
import numpy as np
import pytest

from oracle import dnnmg_oracle as orc
from golden_util import oracle_context, oracle_bcs, oracle_model


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def ctx_cache():
    return {}


def _ctx(golden, cache):
    name, g = golden
    if name not in cache:
        cache[name] = oracle_context(g)
    return cache[name]


def test_index_maps_bit_exact(golden, ctx_cache):
    name, g = golden
    c = _ctx(golden, ctx_cache)
    assert np.array_equal(c["table"], g["cell_nodes"])
    assert np.array_equal(c["coords"], g["fine_coords"])
    assert np.array_equal(c["coarse_coords"], g["coarse_coords"])
    assert np.array_equal(c["tags"], g["node_tags"])
    assert np.array_equal(c["mask"], g["mask"])
    assert np.array_equal(c["dof_table"], g["dof_table"])
    assert np.array_equal(c["node_table"], g["node_table"])
    assert np.array_equal(c["valence"], g["valence"])
    assert np.array_equal(c["mu"], g["mu"])
    assert np.allclose(c["geom"], g["geom"], rtol=1e-14, atol=1e-15)
    assert np.array_equal(c["h_T"], g["h_T"])
    L = int(g["L"])
    for i, (indptr, indices, data) in enumerate(c["P"]):
        l = L + i
        assert np.array_equal(indptr, g[f"P{l}_indptr"])
        assert np.array_equal(indices, g[f"P{l}_indices"])
        assert np.array_equal(data, g[f"P{l}_data"])


def test_correction_step_matches_reference(golden, ctx_cache):
    name, g = golden
    c = _ctx(golden, ctx_cache)
    out = orc.correction_step(g["x_coarse"], g["b_prev"], c, oracle_model(g), float(g["t"]),
                              float(g["nu"]), float(g["k"]), float(g["alpha0"]),
                              float(g["delta0"]), float(g["scale"]), bcs=oracle_bcs(g))
    assert rel(out["x_tilde"], g["x_tilde"]) < 1e-14
    assert rel(out["alpha_T"], g["alpha_T"]) < 1e-14
    assert rel(out["delta_T"], g["delta_T"]) < 1e-14
    assert rel(out["r"], g["r"]) < 1e-11
    assert rel(out["X"], g["X"]) < 1e-11
    assert rel(out["Y"], g["Y"]) < 1e-10
    assert rel(out["d"], g["d"]) < 1e-10
    assert rel(out["x_corr"], g["x_corr"]) < 1e-11
    # zeroed rows / pressure block as the reference
    assert np.all(out["r"][g["mask"]] == 0.0)
    assert np.all(out["d"].reshape(-1, 4)[:, 0] == 0.0)


def test_rhs_next_matches_reference(golden, ctx_cache):
    name, g = golden
    c = _ctx(golden, ctx_cache)
    b = orc.rhs_next(g["x_corr"], c["coords"], c["table"], float(g["k"]), float(g["nu"]))
    assert rel(b, g["b_next"]) < 1e-12


def test_stab_golden_value():
    """assembly.py:55-59 pinned by test_assembly.py:15-21 (alpha_T = 1.480933e-4)."""
    h_T, vmax, nu, k = 0.1, 1.0, 5e-4, 0.008
    den = nu / h_T ** 2 + vmax / h_T + 1.0 / k
    assert 0.02 / den == pytest.approx(1.480933e-4, rel=1e-6)
