"""Generate the config-1-scale golden pin by running the REFERENCE ``dnnmg`` package.

BASELINE config 1 (8,192 patches: level 0 = 16x8x8 Q2 cells, jittered, J = 1,
240 -> 256x3 -> 81 tanh, dt = 0.005, nu = 1e-3) is too large to commit as full
vectors (283,140 dofs per vector), so this script runs the reference's hybrid
correction step exactly as make_golden.py does (driver.py:251-271) and stores

* every full vector's L2 norm, per component (p, u, v, w),
* 16,384 seeded-random dof samples of x~, b_prev, r, d, x_corr, b_next,
* 256 seeded-random patch rows of X (fp32, exact) and Y, 1,024 cells of alpha_T / delta_T,

with the same seeded inputs bench.py's config 1 builds (synthetic.CONFIGS["cfg1"]).
The GPU test (tests/test_gpu_cfg1.py) rebuilds the problem with the product,
runs one correction step and compares against the samples and the norms.
Runs only in the build container (needs /root/reference; ~1 min, 6.5 GB RSS).

    python tests/golden/make_cfg1.py            # rewrites tests/golden/cfg1_pin.npz
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as mg  # noqa: E402  (sets up sys.path for dnnmg and the product)
from dnnmg import mesh as meshmod, space as spmod, patch_ops, driver, net  # noqa: E402
from paper_2307_14837_b200 import synthetic  # noqa: E402

N_DOF_SAMPLES = 16384
N_ROW_SAMPLES = 256
N_CELL_SAMPLES = 1024


def case_of_cfg1():
    c = synthetic.CONFIGS["cfg1"]
    return dict(lo=(0, 0, 0), hi=(1, 1, 1), n_cells=c["n_cells"], L=0, J=c["J"],
                jitter=c["seed"] + 1 if c["jitter"] else None, hidden=c["hidden"],
                depth=c["depth"], act="tanh", dt=c["dt"], nu=c["nu"], seed=c["seed"],
                channel=False, scale=1.0, bn=False)


def comp_norms(v):
    return np.linalg.norm(v.reshape(-1, 4), axis=0)


def main():
    case = case_of_cfg1()
    h = mg.build(case)
    L, J = case["L"], case["J"]
    fl = L + J
    nu, k = case["nu"], case["dt"]
    bcs = mg.bcs_of(case)
    pr = driver.NsProblem(h, nu=nu, k=k, bcs=bcs)
    ps = meshmod.build_patches(h, L, J)
    n_in, n_out = patch_ops.input_width(ps), patch_ops.output_width(ps)
    model = mg.make_model(case, n_in, n_out)
    sL = pr.space(L)
    modes = synthetic.fourier_modes(case["seed"])
    x0 = synthetic.coarse_state(sL.nodes, modes, case["seed"], 0, 0.0, nu)
    x1 = synthetic.coarse_state(sL.nodes, modes, case["seed"], 1, k, nu)
    xf0 = driver.embed_state(pr, L, J, x0, 0.0)
    asm = pr.asm(fl)
    b_prev = asm.assemble_rhs_next(xf0, None, None, k, nu)
    t = k
    xt = spmod.prolongate(h, spmod.StateVector(L, x1.copy(), 0.0), J)
    spmod.apply_dirichlet(pr.space(fl), xt, t, bcs)
    stab = asm.stab(xt.values, nu, k, pr.alpha0, pr.delta0)
    r = asm.assemble_residual(xt.values, b_prev, k, nu, stab, mask=pr.mask(fl))
    X = patch_ops.assemble_network_input(xt.values, r, ps)
    Y = net.forward(model, X)
    d = patch_ops.predict_correction(model, xt.values, r, ps, dirichlet_mask=pr.mask(fl))
    x_corr = xt.values + case["scale"] * d
    b_next = asm.assemble_rhs_next(x_corr, None, None, k, nu)

    rng = np.random.default_rng(20260101)
    ndof = xt.values.size
    dofs = np.sort(rng.choice(ndof, N_DOF_SAMPLES, replace=False))
    rows = np.sort(rng.choice(len(ps), N_ROW_SAMPLES, replace=False))
    cells = np.sort(rng.choice(asm.n_cells, N_CELL_SAMPLES, replace=False))
    vecs = dict(x_tilde=xt.values, b_prev=b_prev, r=r, d=d, x_corr=x_corr, b_next=b_next)
    out = dict(n_patches=len(ps), ndof=ndof, n_in=n_in, n_out=n_out, dofs=dofs, rows=rows,
               cells=cells, x_coarse_norm=np.linalg.norm(x1), x0_coarse_norm=np.linalg.norm(x0),
               X=X[rows].astype(np.float32), Y=Y[rows], alpha_T=stab.alpha_T[cells],
               delta_T=stab.delta_T[cells],
               n_masked=int(pr.mask(fl).sum()))
    for name, v in vecs.items():
        out[name] = v[dofs]
        out[name + "_norms"] = comp_norms(v)
    np.savez_compressed(os.path.join(HERE, "cfg1_pin.npz"), **out)
    print("cfg1 patches", len(ps), "ndof", ndof, "|r|", np.linalg.norm(r), "|d|",
          np.linalg.norm(d))


if __name__ == "__main__":
    main()
