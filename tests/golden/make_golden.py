"""Generate golden vectors by running the REFERENCE ``dnnmg`` package itself.

Runs only in the build container, where ``/root/reference/pkg/src`` is
importable (it does not exist on the GPU box; the tests only read the committed
``*.npz``).  For every case it builds the reference mesh hierarchy, space,
assembler, patch set and an eval-mode ``MlpModel``, feeds the seeded synthetic
inputs of ``paper_2307_14837_b200.synthetic`` (identical values to the ones
the oracle and the GPU path see), and records every intermediate of one hybrid
correction step exactly as ``driver.TimeLoop._step_hybrid`` (driver.py:251-268)
computes it, plus the next-step RHS (driver.py:269-271) and all index maps.

    python tests/golden/make_golden.py            # rewrites tests/golden/*.npz
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from dnnmg import mesh as meshmod, space as spmod, patch_ops, driver  # noqa: E402
from dnnmg.net import Architecture, MlpModel  # noqa: E402

from paper_2307_14837_b200 import synthetic  # noqa: E402

CASES = {
    # BASELINE config 0 exactly: 128 patches, 240->256x3->81 tanh
    "cfg0": dict(lo=(0, 0, 0), hi=(1, 1, 1), n_cells=(4, 2, 2), L=0, J=1, jitter=None,
                 hidden=256, depth=3, act="tanh", dt=0.01, nu=1e-3, seed=100,
                 channel=False, scale=1.0, bn=False),
    # jittered (non-affine Q2 cells), config-1 style
    "jit": dict(lo=(0, 0, 0), hi=(1, 1, 1), n_cells=(3, 2, 2), L=0, J=1, jitter=11,
                hidden=32, depth=3, act="tanh", dt=0.005, nu=1e-3, seed=101,
                channel=False, scale=1.0, bn=False),
    # J = 2 patches (125 nodes, 1024 -> H -> 375), config-2 style
    "j2": dict(lo=(0, 0, 0), hi=(1, 0.5, 0.5), n_cells=(2, 1, 1), L=0, J=2, jitter=12,
               hidden=32, depth=3, act="tanh", dt=0.005, nu=1e-3, seed=102,
               channel=False, scale=1.0, bn=False),
    # coarse level L = 1 (multi-level numbering), relu, trained-style BN + input norm
    "lvl1": dict(lo=(0, 0, 0), hi=(1, 1, 1), n_cells=(2, 1, 1), L=1, J=1, jitter=13,
                 hidden=48, depth=4, act="relu", dt=0.005, nu=2e-3, seed=103,
                 channel=False, scale=0.7, bn=True),
    # channel tags: inflow profile (non-zero Dirichlet data), outflow (no pressure pin)
    "chan": dict(lo=(0, 0, -0.205), hi=(1.0, 0.41, 0.205), n_cells=(3, 2, 2), L=0, J=1,
                 jitter=None, hidden=32, depth=2, act="tanh", dt=0.01, nu=1e-3, seed=104,
                 channel=True, scale=1.0, bn=True),
}


def build(case):
    h = meshmod.build_template_mesh("box", extent_lo=case["lo"], extent_hi=case["hi"],
                                    n_cells=case["n_cells"], channel_tags=case["channel"])
    if case["jitter"] is not None:
        synthetic.jitter_vertices(h.levels[0].vertices, case["n_cells"], case["lo"],
                                  case["hi"], case["jitter"])
    for _ in range(case["L"] + case["J"]):
        meshmod.refine_uniform(h)
    return h


def bcs_of(case):
    if case["channel"]:
        return {meshmod.INFLOW: spmod.inflow_profile(3, 1.0, 0.41), meshmod.WALL: spmod.no_slip}
    return {meshmod.WALL: spmod.no_slip}


def make_model(case, n_in, n_out):
    dims = [n_in] + [case["hidden"]] * case["depth"] + [n_out]
    model = MlpModel(Architecture(n_in, case["hidden"], case["depth"], n_out),
                     activation=case["act"])
    model.W = synthetic.xavier_weights(dims, case["seed"] + 7)
    if case["bn"]:
        rng = np.random.default_rng(case["seed"] + 9)
        H = case["hidden"]
        model.gamma = [rng.uniform(0.5, 1.5, H) for _ in range(case["depth"])]
        model.beta = [rng.normal(0, 0.1, H) for _ in range(case["depth"])]
        model.running_mean = [rng.normal(0, 0.2, H) for _ in range(case["depth"])]
        model.running_var = [rng.uniform(0.5, 2.0, H) for _ in range(case["depth"])]
        model.set_input_norm(rng.normal(0, 0.3, n_in), rng.uniform(0.5, 2.0, n_in))
    return model.eval()


def run_case(name, case):
    h = build(case)
    L, J = case["L"], case["J"]
    fl = L + J
    nu, k = case["nu"], case["dt"]
    bcs = bcs_of(case)
    pr = driver.NsProblem(h, nu=nu, k=k, bcs=bcs)
    ps = meshmod.build_patches(h, L, J)
    model = make_model(case, patch_ops.input_width(ps), patch_ops.output_width(ps))
    sL = pr.space(L)
    modes = synthetic.fourier_modes(case["seed"])
    x0 = synthetic.coarse_state(sL.nodes, modes, case["seed"], 0, 0.0, nu)
    x1 = synthetic.coarse_state(sL.nodes, modes, case["seed"], 1, k, nu)
    # carried fine RHS of the initial state (driver.py:211-219)
    xf0 = driver.embed_state(pr, L, J, x0, 0.0)
    b_prev = pr.asm(fl).assemble_rhs_next(xf0, None, None, k, nu)
    # one hybrid correction step (driver.py:251-271)
    t = k
    xt = spmod.prolongate(h, spmod.StateVector(L, x1.copy(), 0.0), J)
    spmod.apply_dirichlet(pr.space(fl), xt, t, bcs)
    asm = pr.asm(fl)
    stab = asm.stab(xt.values, nu, k, pr.alpha0, pr.delta0)
    r = asm.assemble_residual(xt.values, b_prev, k, nu, stab, mask=pr.mask(fl))
    X = patch_ops.assemble_network_input(xt.values, r, ps)
    from dnnmg import net
    Y = net.forward(model, X)
    d = patch_ops.predict_correction(model, xt.values, r, ps, dirichlet_mask=pr.mask(fl))
    x_corr = xt.values + case["scale"] * d
    b_next = asm.assemble_rhs_next(x_corr, None, None, k, nu)
    out = dict(
        n_cells=np.array(case["n_cells"]), lo=np.array(case["lo"], float),
        hi=np.array(case["hi"], float), L=L, J=J,
        jitter=-1 if case["jitter"] is None else case["jitter"],
        channel=int(case["channel"]), nu=nu, k=k, t=t, scale=case["scale"],
        alpha0=pr.alpha0, delta0=pr.delta0, act=case["act"],
        x_coarse=x1, x0_coarse=x0, b_prev=b_prev,
        coarse_coords=sL.nodes, fine_coords=pr.space(fl).nodes,
        cell_nodes=pr.space(fl).cell_nodes, node_tags=pr.space(fl).node_tags,
        mask=pr.mask(fl), h_T=asm.h_T,
        dof_table=ps.dof_table, node_table=ps.node_table, valence=ps.valence,
        mu=ps.mu, geom=ps.geom_table,
        x_tilde=xt.values, alpha_T=stab.alpha_T, delta_T=stab.delta_T, r=r, X=X, Y=Y,
        d=d, x_corr=x_corr, b_next=b_next,
        n_layers=len(model.W),
    )
    for l in range(L, fl):
        P = spmod.prolongation_matrix(h, l)
        out[f"P{l}_indptr"], out[f"P{l}_indices"], out[f"P{l}_data"] = P.indptr, P.indices, P.data
    for i, W in enumerate(model.W):
        out[f"W{i}"] = W.astype(np.float32)
    for i in range(case["depth"]):
        out[f"gamma{i}"] = model.gamma[i]
        out[f"beta{i}"] = model.beta[i]
        out[f"rmean{i}"] = model.running_mean[i]
        out[f"rvar{i}"] = model.running_var[i]
    out["input_mean"], out["input_std"] = model.input_mean, model.input_std
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "patches", len(ps), "fine nodes", pr.space(fl).n_nodes,
          "|d|", np.linalg.norm(d), "|r|", np.linalg.norm(r))


if __name__ == "__main__":
    for name, case in CASES.items():
        run_case(name, case)
