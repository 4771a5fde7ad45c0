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
