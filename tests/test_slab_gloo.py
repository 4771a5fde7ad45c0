"""Multi-rank x-slab decomposition on CPU: 2 (and 3) processes over torch.distributed
gloo.  Each rank builds its SlabPartition (local hierarchy with global boundary
tags, interface node lists and merge plans, global pressure pin), computes its local
part of the correction step with the float64 oracle, exchanges the raw interface element
rows and patch predictions with TorchDistExchanger, and merges them in the plans' global
order exactly as the halo kernels do.  The assembled global d must
equal the single-domain oracle result, and both sides of an interface must hold
identical values."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASE = dict(lo=(0.0, 0.0, 0.0), hi=(1.0, 0.5, 0.5), n_cells=(4, 2, 2), L=0, J=1, jitter=21,
            nu=1e-3, k=0.005, seed=7, hidden=16)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _global_problem():
    sys.path.insert(0, REPO)
    from oracle import dnnmg_oracle as orc
    from paper_2307_14837_b200 import synthetic
    c = CASE

    def jf(V):
        synthetic.jitter_vertices(V, c["n_cells"], c["lo"], c["hi"], c["jitter"])
    ctx = orc.build_context(c["lo"], c["hi"], c["n_cells"], c["L"], c["J"], jitter_fn=jf)
    npp = ctx["dof_table"].shape[1] // 4
    dims = [8 * npp + 24, c["hidden"], c["hidden"], 3 * npp]
    model = orc.Mlp(synthetic.xavier_weights(dims, c["seed"]), activation="tanh")
    modes = synthetic.fourier_modes(c["seed"])
    x0 = synthetic.coarse_state(ctx["coarse_coords"], modes, c["seed"], 0, 0.0, c["nu"])
    xf0 = orc.prolongate_state(ctx["P"], x0)
    orc.impose_dirichlet(xf0, ctx["tags"], ctx["coords"], 0.0, {orc.WALL: orc.no_slip})
    b = orc.rhs_next(xf0, ctx["coords"], ctx["table"], c["k"], c["nu"])
    x1 = synthetic.coarse_state(ctx["coarse_coords"], modes, c["seed"], 1, c["k"], c["nu"])
    ref = orc.correction_step(x1, b, ctx, model, c["k"], c["nu"], c["k"])
    return ctx, model, x1, b, ref


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, REPO)
        from oracle import dnnmg_oracle as orc
        from paper_2307_14837_b200 import space as spmod, mesh as meshmod
        from paper_2307_14837_b200.slab import SlabPartition, TorchDistExchanger
        c = CASE
        ctx, model, x1, b, ref = _global_problem()
        # global doubled-lattice position -> global node id (oracle numbering == reference)
        gh = meshmod.build_template_mesh("box", extent_lo=c["lo"], extent_hi=c["hi"],
                                         n_cells=c["n_cells"])
        from paper_2307_14837_b200 import synthetic
        synthetic.jitter_vertices(gh.levels[0].vertices, c["n_cells"], c["lo"], c["hi"], c["jitter"])
        for _ in range(c["L"] + c["J"]):
            meshmod.refine_uniform(gh)
        from paper_2307_14837_b200.slab import global_index
        g_fine = global_index(gh, c["L"] + c["J"])
        g_coarse = global_index(gh, c["L"])
        part = SlabPartition(c["lo"], c["hi"], c["n_cells"], c["L"], c["J"], world, rank,
                             jitter_seed=c["jitter"])
        ex = TorchDistExchanger()
        fid = g_fine(part.fine_pos)
        cid = g_coarse(part.coarse_pos)
        # coordinates of the local mesh equal the global ones bit-for-bit
        assert np.array_equal(part.space.nodes, ctx["coords"][fid])
        # ---- local part of the step, float64 oracle arithmetic ----
        xl = x1.reshape(-1, 4)[cid].reshape(-1)
        P = spmod.prolongation_matrix(part.h, c["L"])
        csr = (P.indptr, P.indices, P.data)
        xt = orc.prolongate_state([csr], xl)
        orc.impose_dirichlet(xt, part.space.node_tags, part.space.nodes, c["k"], {orc.WALL: orc.no_slip})
        table = part.space.cell_nodes
        lvl = part.h.levels[c["L"] + c["J"]]
        h_T = orc.cell_diameters(orc.Level(lvl.vertices, lvl.cells))
        aT, dT = orc.stab_weights(xt, table, h_T, c["nu"], c["k"])
        geom = orc.GeometryCache(part.space.nodes, table)
        A = np.zeros(xt.size)
        for sl, g in geom.chunks:
            cont, mom = orc.element_vectors(xt, g, table[sl], c["k"], c["nu"], aT[sl], dT[sl])
            A += orc.assemble(table[sl], cont, mom, xt.size)
        # element rows (cell*27 + a) -> exchange (a) of the interface rows in plan order,
        # merged per node in ascending global cell id (halo_merge_rows_kernel)
        cont, mom = orc.element_vectors(xt, geom.chunks[0][1], table, c["k"], c["nu"], aT, dT) \
            if len(geom.chunks) == 1 else (None, None)
        assert cont is not None
        elem = np.concatenate([cont[:, :, None], mom], axis=2).reshape(-1, 4)
        sends = {s: torch.tensor(elem[pl["send"]]) for s, pl in part.cell_plans.items()}
        recv = ex.exchange(sends)
        A4 = A.reshape(-1, 4)
        for s, pl in part.cell_plans.items():
            rv = recv[s].numpy()
            for i, node in enumerate(pl["nodes"]):
                acc = np.zeros(4)
                for src in pl["merge_src"][pl["merge_ptr"][i]:pl["merge_ptr"][i + 1]]:
                    acc = acc + (elem[src] if src >= 0 else rv[-1 - src])
                A4[node] = acc
        bl = b.reshape(-1, 4)[fid].reshape(-1)
        r = bl - A
        r[part.mask] = 0.0
        ps = part.patchset
        X = orc.network_input(xt, r, ps.dof_table, ps.geom_table)
        Y = orc.mlp_forward(model, X)
        rows = np.zeros(ps.dof_table.shape)
        npp = ps.nodes_per_patch
        vel = (np.arange(npp)[:, None] * 4 + np.arange(1, 4)[None, :]).ravel()
        rows[:, vel] = Y
        S = np.bincount(ps.dof_table.ravel(), weights=rows.ravel(), minlength=xt.size).reshape(-1, 4)
        cnt = np.bincount(ps.node_table.ravel(), minlength=xt.size // 4).astype(float)
        d = (S / cnt[:, None])
        # exchange (b): the interface (patch, slot) predictions, merged in ascending global
        # patch id with the global valence (halo_merge_scatter_kernel)
        Yr = Y.reshape(-1, 3)
        sends = {s: torch.tensor(Yr[pl["send"]]) for s, pl in part.patch_plans.items()}
        recv = ex.exchange(sends)
        for s, pl in part.patch_plans.items():
            rv = recv[s].numpy()
            for i, node in enumerate(pl["nodes"]):
                src_i = pl["merge_src"][pl["merge_ptr"][i]:pl["merge_ptr"][i + 1]]
                acc = np.zeros(3)
                for src in src_i:
                    acc = acc + (Yr[src] if src >= 0 else rv[-1 - src])
                d[node, 1:] = acc / len(src_i)
        d[:, 0] = 0.0
        d = d.reshape(-1)
        d[part.mask] = 0.0
        err_r = np.abs(r - ref["r"].reshape(-1, 4)[fid].reshape(-1)).max() / np.abs(ref["r"]).max()
        err_d = np.abs(d - ref["d"].reshape(-1, 4)[fid].reshape(-1)).max() / np.abs(ref["d"]).max()
        iface_d = {s: d.reshape(-1, 4)[n].copy() for s, n in part.iface.items()}
        out_q.put((rank, err_r, err_d, iface_d, part.n_patches, len(part.iface)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_decomposition_gloo(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time
    results = {}
    deadline = time.time() + 300
    while len(results) < world:
        try:
            rank, err_r, err_d, iface_d, n_p, n_if = q.get(timeout=2)
            results[rank] = (err_r, err_d, iface_d, n_p, n_if)
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            if dead or time.time() > deadline:
                for p in procs:
                    p.kill()
                pytest.fail(f"slab worker failed (exit codes {[p.exitcode for p in procs]})")
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    total_patches = sum(v[3] for v in results.values())
    assert total_patches == 8 * int(np.prod(CASE["n_cells"]))
    for rank, (err_r, err_d, iface_d, n_p, n_if) in results.items():
        assert err_r < 1e-12, (rank, err_r)
        assert err_d < 1e-12, (rank, err_d)
        assert n_if == (1 if rank in (0, world - 1) else 2)
    for r in range(world - 1):  # both sides of every interface hold identical values
        assert np.array_equal(results[r][2]["right"], results[r + 1][2]["left"])
