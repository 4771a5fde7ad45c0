"""Golden training dataset written by the REFERENCE ``driver.export_training_data``
(driver.py:317-383) and ``io.write_dataset`` (io.py:219-266).

Runs only in the build container (``/root/reference/pkg/src`` importable).  Two synthetic
"DMGT" trajectories of a small channel problem (L = 0, J = 1, 16 patches) are written with
the reference's TrajectoryWriter: the coarse run holds the seeded Fourier field at the
level-0 nodes, the fine run the same field at the level-1 nodes (so targets are the Q2
interpolation defect).  The reference then exports (a) train/val windows with the
ideal-correction loop pass — its coarse Newton solves are recorded so the GPU test can
replay them — and (b) the self-consistency case (fine run as its own coarse run).  Small
shards exercise the shard splitting.

    python tests/golden/make_dataset.py           # rewrites tests/golden/dataset/
"""

import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from dnnmg import mesh as meshmod, space as spmod, driver, io as iomod  # noqa: E402

from paper_2307_14837_b200 import synthetic  # noqa: E402

CASE = dict(lo=(0, 0, -0.205), hi=(1.0, 0.41, 0.205), n_cells=(2, 1, 1), jitter=21, L=0, J=1,
            dt=0.02, nu=1e-3, seed=106, vbar=1.5, n_steps=6, t_train=(0.02, 0.06),
            t_val=(0.06, 0.1), shard_bytes=30000)
OUT = os.path.join(HERE, "dataset")


def build(c):
    h = meshmod.build_template_mesh("box", extent_lo=c["lo"], extent_hi=c["hi"],
                                    n_cells=c["n_cells"], channel_tags=True)
    synthetic.jitter_vertices(h.levels[0].vertices, c["n_cells"], c["lo"], c["hi"], c["jitter"])
    for _ in range(c["L"] + c["J"]):
        meshmod.refine_uniform(h)
    return h


def main():
    c = CASE
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    h = build(c)
    bcs = {meshmod.INFLOW: spmod.inflow_profile(3, c["vbar"], 0.41), meshmod.WALL: spmod.no_slip}
    pr = driver.NsProblem(h, nu=c["nu"], k=c["dt"], bcs=bcs)
    modes = synthetic.fourier_modes(c["seed"])
    for lvl, name in ((c["L"], "coarse"), (c["L"] + c["J"], "fine")):
        s = pr.space(lvl)
        w = iomod.TrajectoryWriter(os.path.join(OUT, f"{name}.dmgt"), lvl, s.ndof, c["dt"])
        for n in range(c["n_steps"] + 1):
            w.append(n, n * c["dt"], synthetic.coarse_state(s.nodes, modes, c["seed"], n,
                                                            n * c["dt"], c["nu"]))
        w.close()
    ct = iomod.Trajectory(os.path.join(OUT, "coarse.dmgt"))
    ft = iomod.Trajectory(os.path.join(OUT, "fine.dmgt"))
    solves = []
    orig = pr.solve_step

    def recording_solve(level, x_prev, b, t, solver=None):
        x, stats, solver = orig(level, x_prev, b, t, solver=solver)
        solves.append((t, np.array(b), x.values.copy()))
        return x, stats, solver
    pr.solve_step = recording_solve
    driver.export_training_data(pr, c["L"], c["J"], ct, ft, c["t_train"], c["t_val"],
                                os.path.join(OUT, "loop"), shard_bytes=c["shard_bytes"],
                                loop_pass=True)
    driver.export_training_data(pr, c["L"], c["J"], ft, ft, c["t_train"], c["t_val"],
                                os.path.join(OUT, "self"), shard_bytes=c["shard_bytes"])
    np.savez_compressed(os.path.join(OUT, "solves.npz"),
                        t=np.array([s[0] for s in solves]),
                        b=np.stack([s[1] for s in solves]), x=np.stack([s[2] for s in solves]))
    print("solves", len(solves), "files", sorted(os.listdir(os.path.join(OUT, "loop"))))


if __name__ == "__main__":
    main()
