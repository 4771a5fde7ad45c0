"""Golden trajectory of the REFERENCE hybrid time loop (driver.TimeLoop, driver.py:170-280).

Runs only in the build container (``/root/reference/pkg/src`` importable).  A small
channel problem (parabolic inflow ramp, no-slip walls, outflow) is stepped by the
reference's own ``TimeLoop`` in hybrid mode (L = 0, J = 1) with a trained-style model
(tanh, BN statistics, input normalisation), a damped correction and a delayed
correction start.  For the initial state and every step the file records what the
loop carries: the coarse solution x^n (the output of the coarse Newton solve),
the corrected fine state x_fine^n, the fine RHS b_next_fine^n and its restriction
b_next^n.  The GPU test replays the coarse solutions through the product's
``driver.TimeLoop`` and compares everything it carries, step by step.

    python tests/golden/make_timeloop.py          # rewrites tests/golden/timeloop.npz
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

CASE = dict(lo=(0, 0, -0.205), hi=(1.0, 0.41, 0.205), n_cells=(3, 2, 2), L=0, J=1,
            hidden=256, depth=3, act="tanh", dt=0.02, nu=1e-3, seed=105, scale=0.5,
            start=0.04, steps=4, vbar=1.5)


def main():
    c = CASE
    h = meshmod.build_template_mesh("box", extent_lo=c["lo"], extent_hi=c["hi"],
                                    n_cells=c["n_cells"], channel_tags=True)
    synthetic.jitter_vertices(h.levels[0].vertices, c["n_cells"], c["lo"], c["hi"], 17)
    for _ in range(c["L"] + c["J"]):
        meshmod.refine_uniform(h)
    bcs = {meshmod.INFLOW: spmod.inflow_profile(3, c["vbar"], 0.41), meshmod.WALL: spmod.no_slip}
    pr = driver.NsProblem(h, nu=c["nu"], k=c["dt"], bcs=bcs)
    ps = meshmod.build_patches(h, c["L"], c["J"])
    n_in, n_out = patch_ops.input_width(ps), patch_ops.output_width(ps)
    dims = [n_in] + [c["hidden"]] * c["depth"] + [n_out]
    model = MlpModel(Architecture(n_in, c["hidden"], c["depth"], n_out), activation=c["act"])
    model.W = synthetic.xavier_weights(dims, c["seed"] + 7)
    assert all(np.array_equal(W, W.astype(np.float32)) for W in model.W)
    rng = np.random.default_rng(c["seed"] + 9)
    H = c["hidden"]
    model.gamma = [rng.uniform(0.5, 1.5, H) for _ in range(c["depth"])]
    model.beta = [rng.normal(0, 0.1, H) for _ in range(c["depth"])]
    model.running_mean = [rng.normal(0, 0.2, H) for _ in range(c["depth"])]
    model.running_var = [rng.uniform(0.5, 2.0, H) for _ in range(c["depth"])]
    model.set_input_norm(rng.normal(0, 0.3, n_in), rng.uniform(0.5, 2.0, n_in))
    model.eval()

    loop = driver.TimeLoop(pr, c["L"], J=c["J"], model=model, correction_scale=c["scale"],
                           correction_start=c["start"])
    st = loop.state
    out = dict(n_cells=np.array(c["n_cells"]), lo=np.array(c["lo"], float),
               hi=np.array(c["hi"], float), L=c["L"], J=c["J"], jitter=17, nu=c["nu"],
               k=c["dt"], scale=c["scale"], start=c["start"], steps=c["steps"], vbar=c["vbar"],
               act=c["act"], alpha0=pr.alpha0, delta0=pr.delta0,
               x_0=st.x.values.copy(), x_fine_0=st.x_fine.values.copy(),
               b_next_0=st.b_next.copy(), b_next_fine_0=st.b_next_fine.copy())
    for n in range(1, c["steps"] + 1):
        st = loop.step()
        out[f"t_{n}"] = st.t
        out[f"x_{n}"] = st.x.values.copy()
        out[f"x_fine_{n}"] = st.x_fine.values.copy()
        out[f"b_next_{n}"] = st.b_next.copy()
        out[f"b_next_fine_{n}"] = st.b_next_fine.copy()
        print(n, st.t, "|x|", np.linalg.norm(st.x.values), "|x_fine|",
              np.linalg.norm(st.x_fine.values), "|b_fine|", np.linalg.norm(st.b_next_fine),
              "net evals", loop.net_evals)
    for i, W in enumerate(model.W):
        out[f"W{i}"] = W.astype(np.float32)   # xavier_weights are fp32 values: lossless
    for i in range(c["depth"]):
        out[f"gamma{i}"] = model.gamma[i]
        out[f"beta{i}"] = model.beta[i]
        out[f"rmean{i}"] = model.running_mean[i]
        out[f"rvar{i}"] = model.running_var[i]
    out["input_mean"], out["input_std"] = model.input_mean, model.input_std
    out["n_layers"] = len(model.W)
    np.savez_compressed(os.path.join(HERE, "timeloop.npz"), **out)
    checkpoints(pr, model)


def checkpoints(pr, model):
    """Reference checkpoints for resume tests (driver.checkpoint_state / resume_loop,
    driver.py:442-480): a hybrid loop saved after step 2 and resumed for 2 steps, and a
    pure-MG loop (J = 0) saved after step 2 and resumed as a hybrid loop."""
    from dnnmg import io as iomod
    c = CASE
    out = {}
    hyb = driver.TimeLoop(pr, c["L"], J=c["J"], model=model, correction_scale=c["scale"],
                          correction_start=c["start"])
    hyb.run(2)
    iomod.save_checkpoint(os.path.join(HERE, "timeloop_hybrid.dmgc"), *driver.checkpoint_state(hyb))
    mg = driver.TimeLoop(pr, c["L"], J=0)
    mg.run(2)
    iomod.save_checkpoint(os.path.join(HERE, "timeloop_mg.dmgc"), *driver.checkpoint_state(mg))
    for name in ("hybrid", "mg"):
        loop = driver.resume_loop(pr, os.path.join(HERE, f"timeloop_{name}.dmgc"), model=model,
                                  J=c["J"])
        loop.correction_scale, loop.correction_start = c["scale"], c["start"]
        out[f"{name}_b_next_fine_0"] = loop.state.b_next_fine.copy()
        out[f"{name}_b_next_0"] = loop.state.b_next.copy()   # RHS of the first resumed solve
        for n in (1, 2):
            st = loop.step()
            out[f"{name}_t_{n}"] = st.t
            out[f"{name}_x_{n}"] = st.x.values.copy()
            out[f"{name}_x_fine_{n}"] = st.x_fine.values.copy()
            out[f"{name}_b_next_fine_{n}"] = st.b_next_fine.copy()
            out[f"{name}_b_next_{n}"] = st.b_next.copy()
    np.savez_compressed(os.path.join(HERE, "timeloop_resume.npz"), **out)


if __name__ == "__main__":
    main()
