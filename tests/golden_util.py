"""Rebuild the oracle context / model of a golden case (test helper)."""
import numpy as np

from oracle import dnnmg_oracle as orc
from paper_2307_14837_b200 import synthetic


def oracle_context(g):
    n_cells = tuple(int(v) for v in g["n_cells"])
    lo, hi = g["lo"], g["hi"]
    jit = int(g["jitter"])
    jf = None
    if jit >= 0:
        def jf(verts):
            synthetic.jitter_vertices(verts, n_cells, lo, hi, jit)
    channel = bool(int(g["channel"]))
    bc_tags = (orc.INFLOW, orc.WALL) if channel else (orc.WALL,)
    return orc.build_context(lo, hi, n_cells, int(g["L"]), int(g["J"]), jitter_fn=jf,
                             channel_tags=channel, bc_tags=bc_tags)


def oracle_bcs(g):
    if int(g["channel"]):
        return {orc.INFLOW: orc.parabolic_inflow(1.0, 0.41), orc.WALL: orc.no_slip}
    return {orc.WALL: orc.no_slip}


def oracle_model(g):
    n = int(g["n_layers"])
    depth = n - 1
    W = [g[f"W{i}"].astype(np.float64) for i in range(n)]
    return orc.Mlp(W, activation=str(g["act"]),
                   gamma=[g[f"gamma{i}"] for i in range(depth)],
                   beta=[g[f"beta{i}"] for i in range(depth)],
                   running_mean=[g[f"rmean{i}"] for i in range(depth)],
                   running_var=[g[f"rvar{i}"] for i in range(depth)],
                   input_mean=g["input_mean"], input_std=g["input_std"])


def load_golden(name):
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", f"{name}.npz")
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


def product_hierarchy(g):
    """Build the same (jittered) hierarchy with the product's mesh module."""
    from paper_2307_14837_b200 import mesh
    n_cells = tuple(int(v) for v in g["n_cells"])
    h = mesh.build_template_mesh("box", extent_lo=g["lo"], extent_hi=g["hi"], n_cells=n_cells,
                                 channel_tags=bool(int(g["channel"])))
    if int(g["jitter"]) >= 0:
        synthetic.jitter_vertices(h.levels[0].vertices, n_cells, g["lo"], g["hi"], int(g["jitter"]))
    for _ in range(int(g["L"]) + int(g["J"])):
        mesh.refine_uniform(h)
    return h


def product_model(g):
    """The golden case's eval-mode model as this package's MlpModel."""
    from paper_2307_14837_b200.net import Architecture, MlpModel
    n = int(g["n_layers"])
    depth = n - 1
    W = [g[f"W{i}"].astype(np.float64) for i in range(n)]
    m = MlpModel(Architecture(W[0].shape[0], W[0].shape[1], depth, W[-1].shape[1]),
                 activation=str(g["act"]))
    m.W = W
    m.gamma = [g[f"gamma{i}"] for i in range(depth)]
    m.beta = [g[f"beta{i}"] for i in range(depth)]
    m.running_mean = [g[f"rmean{i}"] for i in range(depth)]
    m.running_var = [g[f"rvar{i}"] for i in range(depth)]
    m.input_mean, m.input_std = g["input_mean"], g["input_std"]
    return m.eval()


def product_bcs(g):
    from paper_2307_14837_b200 import mesh, space
    if int(g["channel"]):
        return {mesh.INFLOW: space.inflow_profile(3, 1.0, 0.41), mesh.WALL: space.no_slip}
    return {mesh.WALL: space.no_slip}


def cfg1_case():
    """BASELINE config 1 rebuilt with the oracle: context, coarse states x^0 / x^1, the
    carried fine RHS b_prev (rhs_next of the embedded x^0, float64), the Xavier weights
    and the reference's pin (tests/golden/make_cfg1.py)."""
    from paper_2307_14837_b200 import synthetic
    c = synthetic.CONFIGS["cfg1"]

    def jf(verts):
        synthetic.jitter_vertices(verts, c["n_cells"], (0, 0, 0), (1, 1, 1), c["seed"] + 1)
    ctx = orc.build_context((0, 0, 0), (1, 1, 1), c["n_cells"], 0, c["J"], jitter_fn=jf)
    modes = synthetic.fourier_modes(c["seed"])
    x0 = synthetic.coarse_state(ctx["coarse_coords"], modes, c["seed"], 0, 0.0, c["nu"])
    x1 = synthetic.coarse_state(ctx["coarse_coords"], modes, c["seed"], 1, c["dt"], c["nu"])
    xf0 = orc.prolongate_state(ctx["P"], x0)
    orc.impose_dirichlet(xf0, ctx["tags"], ctx["coords"], 0.0, {orc.WALL: orc.no_slip})
    b_prev = orc.rhs_next(xf0, ctx["coords"], ctx["table"], c["dt"], c["nu"])
    pin = load_golden("cfg1_pin")
    dims = [int(pin["n_in"])] + [c["hidden"]] * c["depth"] + [int(pin["n_out"])]
    W = [w.astype(np.float64) for w in synthetic.xavier_weights(dims, c["seed"] + 7)]
    return dict(cfg=c, ctx=ctx, x0=x0, x1=x1, b_prev=b_prev, W=W, pin=pin)


def sampled_rel(v, pin, name):
    """Relative L2 error of v on the pin's sampled dofs, and the worst per-component
    relative error of v's full-vector norms."""
    s = np.asarray(v, dtype=float)
    ref = pin[name]
    e = np.linalg.norm(s[pin["dofs"]] - ref) / max(np.linalg.norm(ref), 1e-300)
    n = np.linalg.norm(s.reshape(-1, 4), axis=0)
    rn = pin[name + "_norms"]
    en = np.max(np.abs(n - rn) / np.maximum(rn, 1e-300) * (rn > 0))
    return e, en
