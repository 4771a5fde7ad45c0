"""Host-side x-slab merge plans (slab.halo_plan), CPU only: the interface sums of the
distributed step must follow the single-domain summation order exactly — ascending
GLOBAL cell id per node for the element vectors (assembly.py:180-184) and ascending
GLOBAL patch id for the patch predictions (patch_ops.py:32-38).

For boxes split into 2 and 3 slabs (J = 1 and 2, L = 0 and 1, jittered) this checks that
  * the global cell / patch ids computed from lattice positions are the global
    hierarchy's own numbering (local order == global order, so interior node sums keep
    the global order as they are),
  * the neighbour's message as this rank predicts it (mirrored ids, per node ascending)
    is exactly what the neighbour sends (its own ids, per node ascending),
  * each interface node's merged entry list, mapped to global ids, is its row of the
    global node -> (cell, local node) / (patch, slot) CSR.
"""
import numpy as np
import pytest

from paper_2307_14837_b200 import mesh as meshmod, synthetic
from paper_2307_14837_b200.device import node_csr
from paper_2307_14837_b200.slab import SlabPartition, global_index

LO, HI = (0.0, 0.0, 0.0), (1.0, 0.5, 0.75)


def global_hierarchy(n_cells, L, J, jit):
    gh = meshmod.build_template_mesh("box", extent_lo=LO, extent_hi=HI, n_cells=n_cells)
    synthetic.jitter_vertices(gh.levels[0].vertices, n_cells, LO, HI, jit)
    for _ in range(L + J):
        meshmod.refine_uniform(gh)
    return gh


def entry_ids(part, plan, width, gid_of_local):
    """Global (cell|patch) id of every merged entry of a plan, per node."""
    rows = []
    remote = plan["remote_ids"]
    for i in range(plan["nodes"].size):
        src = plan["merge_src"][plan["merge_ptr"][i]:plan["merge_ptr"][i + 1]]
        rows.append([int(gid_of_local[s // width]) if s >= 0 else int(remote[-1 - s])
                     for s in src])
    return rows


@pytest.mark.parametrize("n_cells,L,J,world", [((4, 2, 3), 0, 1, 2), ((6, 2, 2), 0, 1, 3),
                                               ((4, 2, 2), 0, 2, 2), ((4, 2, 2), 1, 1, 2)])
def test_merge_plans_follow_global_order(n_cells, L, J, world):
    jit = 11
    gh = global_hierarchy(n_cells, L, J, jit)
    fl = L + J
    g_fine = global_index(gh, fl)
    gtab = gh.scalar_nodes(fl)[1]
    gps = meshmod.build_patches(gh, L, J)
    gc_ptr, gc_idx = node_csr(gtab)
    gp_ptr, gp_idx = node_csr(gps.node_table)
    parts = [SlabPartition(LO, HI, n_cells, L, J, world, r, jitter_seed=jit) for r in range(world)]
    total_cells = 0
    for p in parts:
        gcell = p.global_fine_cells()
        gpatch = p.global_patches()
        total_cells += gcell.size
        # local ids map monotonically onto the global numbering, and the cell tables agree
        assert np.all(np.diff(gcell) > 0) and np.all(np.diff(gpatch) > 0)
        fid = g_fine(p.fine_pos)
        assert np.array_equal(fid[p.space.cell_nodes], gtab[gcell])
        assert np.array_equal(fid[p.patchset.node_table], gps.node_table[gpatch])
        assert np.array_equal(p.space.nodes, gh.scalar_nodes(fl)[0][fid])
        for side in p.iface:
            for plan, width, gid, ptr_, idx_ in (
                    (p.cell_plans[side], 27, gcell, gc_ptr, gc_idx),
                    (p.patch_plans[side], p.patchset.nodes_per_patch, gpatch, gp_ptr, gp_idx)):
                rows = entry_ids(p, plan, width, gid)
                for i, node in enumerate(plan["nodes"]):
                    gn = fid[node]
                    want = [int(e) // width for e in idx_[ptr_[gn]:ptr_[gn + 1]]]
                    assert rows[i] == want, (side, i)
    assert total_cells == gtab.shape[0]
    # the message each rank expects is the one its neighbour sends
    for r in range(world - 1):
        for which in ("cell_plans", "patch_plans"):
            mine = getattr(parts[r], which)["right"]
            theirs = getattr(parts[r + 1], which)["left"]
            assert np.array_equal(mine["counts"], theirs["counts"])
            assert np.array_equal(mine["remote_ids"], theirs["own_ids"])
            assert np.array_equal(theirs["remote_ids"], mine["own_ids"])
            assert np.array_equal(parts[r].fine_pos[mine["nodes"]],
                                  parts[r + 1].fine_pos[theirs["nodes"]])


def test_global_box_predicate():
    """Every rank decides from the global level-0 vertices whether K2 may take its box form, so
    that all ranks run the element-kernel form of the single domain."""
    from paper_2307_14837_b200 import slab
    lo, hi = (0.0, 0.0, 0.0), (1.0, 0.5, 0.5)
    assert slab.global_is_box(slab.global_level0_vertices(lo, hi, (4, 3, 2), None), (4, 3, 2))
    assert not slab.global_is_box(slab.global_level0_vertices(lo, hi, (8, 2, 2), 31), (8, 2, 2))
    # one cell across y and z: no interior vertex, nothing is jittered
    assert slab.global_is_box(slab.global_level0_vertices(lo, hi, (8, 1, 1), 31), (8, 1, 1))
    for world in (1, 2):
        for rank in range(world):
            p = slab.SlabPartition(lo, hi, (4, 2, 2), 0, 1, world, rank, jitter_seed=7)
            assert p.global_box is False
            p = slab.SlabPartition(lo, hi, (4, 2, 2), 0, 1, world, rank)
            assert p.global_box is True
