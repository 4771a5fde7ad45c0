"""Generate the config-2 / config-3-scale golden pins by running the REFERENCE ``dnnmg``.

At 524,288 fine cells the reference's ``Assembler`` needs ~400 GB unchunked
(SURVEY.md §8(c)), so the assembly runs on the chunked-Assembler oracle: the
reference's own ``Assembler`` constructed on a space view holding a slice of the
cells, ``assemble_rhs_next`` / ``stab`` + ``apply_operator`` per chunk, summed
(the dual vectors are sums over cells, assembly.py:180-184).  Mesh, PatchSet,
prolongation, network input, forward and predict_correction run unchunked, exactly
as make_golden.py does (driver.py:251-271).  Stored as in make_cfg1.py: sampled
dofs of every vector, per-component full norms, sampled patch rows of X and Y.

    python tests/golden/make_big.py cfg2      # ~15 min, 4 workers, ~30 GB peak
    python tests/golden/make_big.py cfg3
    python tests/golden/trim_pin.py cfg2 96        # fixture size: 96 X/Y rows kept
    python tests/golden/trim_pin.py cfg3 96
    python tests/golden/make_big.py cfg1 _chunked   # check: equals cfg1_pin.npz (unchunked)
"""

import os
import sys
import time
import types
from multiprocessing import get_context

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as mg  # noqa: E402  (sets up sys.path for dnnmg and the product)
from dnnmg import mesh as meshmod, space as spmod, patch_ops, driver, net  # noqa: E402
from dnnmg.assembly import Assembler  # noqa: E402
from paper_2307_14837_b200 import synthetic  # noqa: E402

N_DOF_SAMPLES = 16384
N_ROW_SAMPLES = 256
N_CELL_SAMPLES = 1024
CHUNK = int(os.environ.get("DNNMG_GOLDEN_CHUNK", 8192))
WORKERS = 4

_G = {}  # inherited by the forked workers


def chunk_view(space, lo, hi):
    lvl = space.hierarchy.levels[space.level]
    view_lvl = types.SimpleNamespace(vertices=lvl.vertices, cells=lvl.cells[lo:hi])
    levels = {space.level: view_lvl}
    return types.SimpleNamespace(dim=space.dim, n_comp=space.n_comp, nodes=space.nodes,
                                 cell_nodes=space.cell_nodes[lo:hi], n_nodes=space.n_nodes,
                                 ndof=space.ndof, level=space.level,
                                 hierarchy=types.SimpleNamespace(levels=levels))


def _pass1(bounds):
    lo, hi = bounds
    g = _G
    asm = Assembler(chunk_view(g["space"], lo, hi))
    b = asm.assemble_rhs_next(g["xf0"], None, None, g["k"], g["nu"])
    st = asm.stab(g["xt"], g["nu"], g["k"], g["alpha0"], g["delta0"])
    a = asm.apply_operator(g["xt"], g["k"], g["nu"], st)
    return lo, b, a, st.alpha_T, st.delta_T


def _pass2(bounds):
    lo, hi = bounds
    g = _G
    asm = Assembler(chunk_view(g["space"], lo, hi))
    return asm.assemble_rhs_next(g["x_corr"], None, None, g["k"], g["nu"])


def case_of(name):
    c = synthetic.CONFIGS[name]
    return dict(lo=(0, 0, 0), hi=(1, 1, 1), n_cells=c["n_cells"], L=0, J=c["J"],
                jitter=c["seed"] + 1 if c["jitter"] else None, hidden=c["hidden"],
                depth=c["depth"], act="tanh", dt=c["dt"], nu=c["nu"], seed=c["seed"],
                channel=False, scale=1.0, bn=False)


def comp_norms(v):
    return np.linalg.norm(v.reshape(-1, 4), axis=0)


def main(name, suffix=""):
    t0 = time.time()
    case = case_of(name)
    h = mg.build(case)
    L, J = case["L"], case["J"]
    fl = L + J
    nu, k = case["nu"], case["dt"]
    bcs = mg.bcs_of(case)
    pr = driver.NsProblem(h, nu=nu, k=k, bcs=bcs)
    ps = meshmod.build_patches(h, L, J)
    print("mesh + patches", time.time() - t0, flush=True)
    n_in, n_out = patch_ops.input_width(ps), patch_ops.output_width(ps)
    model = mg.make_model(case, n_in, n_out)
    sL, sF = pr.space(L), pr.space(fl)
    modes = synthetic.fourier_modes(case["seed"])
    x0 = synthetic.coarse_state(sL.nodes, modes, case["seed"], 0, 0.0, nu)
    x1 = synthetic.coarse_state(sL.nodes, modes, case["seed"], 1, k, nu)
    xf0 = driver.embed_state(pr, L, J, x0, 0.0)
    t = k
    xt = spmod.prolongate(h, spmod.StateVector(L, x1.copy(), 0.0), J)
    spmod.apply_dirichlet(sF, xt, t, bcs)
    mask = pr.mask(fl)
    nc = sF.cell_nodes.shape[0]
    bounds = [(lo, min(lo + CHUNK, nc)) for lo in range(0, nc, CHUNK)]
    _G.update(space=sF, xf0=xf0, xt=xt.values, k=k, nu=nu, alpha0=pr.alpha0,
              delta0=pr.delta0)
    b_prev = np.zeros(sF.ndof)
    Ax = np.zeros(sF.ndof)
    alpha_T = np.zeros(nc)
    delta_T = np.zeros(nc)
    with get_context("fork").Pool(WORKERS) as pool:
        for lo, b, a, aT, dT in pool.imap_unordered(_pass1, bounds):
            b_prev += b
            Ax += a
            alpha_T[lo:lo + aT.size] = aT
            delta_T[lo:lo + dT.size] = dT
    print("pass 1", time.time() - t0, flush=True)
    r = b_prev - Ax
    r[mask] = 0.0
    X = patch_ops.assemble_network_input(xt.values, r, ps)
    Y = net.forward(model, X)
    d = patch_ops.predict_correction(model, xt.values, r, ps, dirichlet_mask=mask)
    x_corr = xt.values + case["scale"] * d
    _G.update(x_corr=x_corr)
    b_next = np.zeros(sF.ndof)
    with get_context("fork").Pool(WORKERS) as pool:
        for b in pool.imap_unordered(_pass2, bounds):
            b_next += b
    print("pass 2", time.time() - t0, flush=True)

    rng = np.random.default_rng(20260101)
    ndof = xt.values.size
    dofs = np.sort(rng.choice(ndof, N_DOF_SAMPLES, replace=False))
    rows = np.sort(rng.choice(len(ps), N_ROW_SAMPLES, replace=False))
    cells = np.sort(rng.choice(nc, N_CELL_SAMPLES, replace=False))
    vecs = dict(x_tilde=xt.values, b_prev=b_prev, r=r, d=d, x_corr=x_corr, b_next=b_next)
    out = dict(n_patches=len(ps), ndof=ndof, n_in=n_in, n_out=n_out, dofs=dofs, rows=rows,
               cells=cells, x_coarse_norm=np.linalg.norm(x1), x0_coarse_norm=np.linalg.norm(x0),
               X=X[rows].astype(np.float32), Y=Y[rows], alpha_T=alpha_T[cells],
               delta_T=delta_T[cells], n_masked=int(mask.sum()), chunk=CHUNK)
    for vname, v in vecs.items():
        out[vname] = v[dofs]
        out[vname + "_norms"] = comp_norms(v)
    np.savez_compressed(os.path.join(HERE, f"{name}_pin{suffix}.npz"), **out)
    print(name, "patches", len(ps), "ndof", ndof, "|r|", np.linalg.norm(r), "|d|",
          np.linalg.norm(d), "total", time.time() - t0)


if __name__ == "__main__":
    main(sys.argv[1], *sys.argv[2:3])
