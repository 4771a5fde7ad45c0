"""SHA-256 fingerprints of the REFERENCE's index maps at full BASELINE scale (configs 1-3).

The reference builds configs 2 and 3 (4,276,737 fine Q2 nodes) in ~6 min each
(SURVEY.md §8(c)); the tables themselves (hundreds of MB) cannot be committed, so this
script stores, per config, the SHA-256 of each table in a canonical byte form (C order,
int64 for indices, float64 for reals):

  fine Q2 node coordinates and cell_nodes of level L+J (mesh.py:162-216),
  coarse (level L) Q2 node coordinates,
  PatchSet dof_table, node_table, valence, mu and geom_table (mesh.py:501-558),
  the constrained-dof mask of NsProblem (driver.py:56-65),
  the prolongation matrix P level L -> L+1 as CSR (space.py:117-165).

tests/test_table_hashes.py rebuilds the same tables with the product's vectorised
mesh code and asserts byte-identical hashes: bit-exact index maps at full size.

    python tests/golden/make_table_hashes.py      # ~15 min, rewrites table_hashes.json
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as mg  # noqa: E402  (sets up sys.path for dnnmg and the product)
from dnnmg import mesh as meshmod, space as spmod, driver  # noqa: E402
from paper_2307_14837_b200 import synthetic  # noqa: E402


def digest(a, kind):
    dt = np.int64 if kind == "i" else (np.float64 if kind == "f" else np.bool_)
    b = np.ascontiguousarray(np.asarray(a), dtype=dt)
    return hashlib.sha256(b.tobytes()).hexdigest() + f":{b.shape}"


def tables(h, ps, L, J, mask, P):
    fl = L + J
    fc, ft = h.scalar_nodes(fl)
    cc, _ = h.scalar_nodes(L)
    P = P.tocsr()
    return {
        "fine_coords": digest(fc, "f"), "cell_nodes": digest(ft, "i"),
        "coarse_coords": digest(cc, "f"),
        "dof_table": digest(ps.dof_table, "i"), "node_table": digest(ps.node_table, "i"),
        "valence": digest(ps.valence, "i"), "mu": digest(ps.mu, "f"),
        "geom_table": digest(ps.geom_table, "f"), "mask": digest(mask, "b"),
        "P_indptr": digest(P.indptr, "i"), "P_indices": digest(P.indices, "i"),
        "P_data": digest(P.data, "f"),
    }


def main(names):
    path = os.path.join(HERE, "table_hashes.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for name in names:
        t0 = time.time()
        c = synthetic.CONFIGS[name]
        case = dict(lo=(0, 0, 0), hi=(1, 1, 1), n_cells=c["n_cells"], L=0, J=c["J"],
                    jitter=c["seed"] + 1 if c["jitter"] else None, channel=False)
        h = mg.build(case)
        pr = driver.NsProblem(h, nu=c["nu"], k=c["dt"], bcs=mg.bcs_of(case))
        ps = meshmod.build_patches(h, 0, c["J"])
        mask = pr.mask(c["J"])
        P = spmod.prolongation_matrix(h, 0)
        out[name] = tables(h, ps, 0, c["J"], mask, P)
        out[name]["n_patches"] = len(ps)
        print(name, len(ps), "patches", f"{time.time() - t0:.0f} s", flush=True)
        json.dump(out, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg1", "cfg2", "cfg3"])
