"""BASELINE.md §2's full-size CPU baseline: the REFERENCE's own correction step at config 3
(524,288 patches, 4,276,737 fine nodes) on this host, float64.

The unchunked reference Assembler needs ~400 GB at this size, so the
residual runs on the chunked-Assembler oracle: the reference's own `Assembler` built on a
space view holding 8,192 cells at a time; per chunk only `stab` + `apply_operator` are
timed (chunk construction -- the geometry cache -- is setup and excluded), each chunk once
with the BLAS pool at all host cores and once at one core.  Prolongation + Dirichlet
(`embed_state`), the gather, the network and the scatter (`predict_correction`) run
unchunked and are timed the same way.  Output: one JSON line (patches/s per thread
setting, stage breakdown), also written to gpurun_out/cpu_reference_cfg3.json.

    python tools/cpu_reference_cfg3.py [cfg3]     # ~30 min, ~16 GB peak RSS

Needs the reference installed in baseline/_ref (bench.py --impl reference does the same on
a 16x8x8 sample within the driver's time budget).
"""

import json
import os
import sys
import time
import types

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "baseline", "_ref"))

from threadpoolctl import threadpool_limits  # noqa: E402

from dnnmg import driver, mesh as meshmod, net, patch_ops, space as spmod  # noqa: E402
from dnnmg.assembly import Assembler  # noqa: E402
from paper_2307_14837_b200 import synthetic  # noqa: E402

CHUNK = 8192


def chunk_view(space, lo, hi):
    lvl = space.hierarchy.levels[space.level]
    view_lvl = types.SimpleNamespace(vertices=lvl.vertices, cells=lvl.cells[lo:hi])
    return types.SimpleNamespace(dim=space.dim, n_comp=space.n_comp, nodes=space.nodes,
                                 cell_nodes=space.cell_nodes[lo:hi], n_nodes=space.n_nodes,
                                 ndof=space.ndof, level=space.level,
                                 hierarchy=types.SimpleNamespace(levels={space.level: view_lvl}))


def timed(fn, threads):
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        out = fn()
        return out, time.perf_counter() - t0


def main(name="cfg3"):
    t_start = time.time()
    cores = os.cpu_count()
    c = synthetic.CONFIGS[name]
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1),
                                    n_cells=c["n_cells"])
    if c["jitter"]:
        synthetic.jitter_vertices(h.levels[0].vertices, c["n_cells"], (0, 0, 0), (1, 1, 1),
                                  c["seed"] + 1)
    for _ in range(c["J"]):
        meshmod.refine_uniform(h)
    L, J = 0, c["J"]
    fl = L + J
    nu, k = c["nu"], c["dt"]
    pr = driver.NsProblem(h, nu=nu, k=k, bcs={meshmod.WALL: spmod.no_slip})
    ps = meshmod.build_patches(h, L, J)
    n_in, n_out = patch_ops.input_width(ps), patch_ops.output_width(ps)
    model = net.MlpModel(net.Architecture(n_in, c["hidden"], c["depth"], n_out), activation="tanh")
    model.W = synthetic.xavier_weights([n_in] + [c["hidden"]] * c["depth"] + [n_out], c["seed"] + 7)
    model.eval()
    sL, sF = pr.space(L), pr.space(fl)
    mask = pr.mask(fl)
    modes = synthetic.fourier_modes(c["seed"])
    x1 = synthetic.coarse_state(sL.nodes, modes, c["seed"], 1, k, nu)
    b_prev = np.zeros(sF.ndof)    # the RHS's value does not change the work
    setup_s = time.time() - t_start
    print(f"setup (mesh, PatchSet) {setup_s:.0f} s", flush=True)
    res = {}
    driver.embed_state(pr, L, J, x1, k)          # builds and caches P (setup)
    for threads in (cores, 1):
        xt, t_embed = timed(lambda: driver.embed_state(pr, L, J, x1, k), threads)
        res.setdefault(threads, {})["embed_state_s"] = t_embed
    nc = sF.cell_nodes.shape[0]
    A = np.zeros(sF.ndof)
    t_asm = {cores: 0.0, 1: 0.0}
    t_build = 0.0
    for lo in range(0, nc, CHUNK):
        t0 = time.perf_counter()
        asm = Assembler(chunk_view(sF, lo, min(lo + CHUNK, nc)))      # setup: excluded
        t_build += time.perf_counter() - t0
        for threads in (cores, 1):
            def work():
                st = asm.stab(xt, nu, k, pr.alpha0, pr.delta0)
                return asm.apply_operator(xt, k, nu, st)
            a, dt = timed(work, threads)
            t_asm[threads] += dt
        A += a
        del asm
        if (lo // CHUNK) % 8 == 0:
            print(f"chunk {lo // CHUNK}/{nc // CHUNK}: build {t_build:.0f} s, stab+apply "
                  f"{t_asm[cores]:.1f} s ({cores} thr) / {t_asm[1]:.1f} s (1 thr)", flush=True)
    r = b_prev - A
    r[mask] = 0.0
    for threads in (cores, 1):
        d, t_pred = timed(lambda: patch_ops.predict_correction(model, xt, r, ps,
                                                               dirichlet_mask=mask), threads)
        _, t_upd = timed(lambda: xt + d, threads)
        res[threads].update(stab_apply_operator_s=t_asm[threads], predict_correction_s=t_pred,
                            update_s=t_upd)
        res[threads]["step_s"] = sum(v for key, v in res[threads].items() if key.endswith("_s"))
        res[threads]["patches_per_s"] = len(ps) / res[threads]["step_s"]
    line = {"metric": "patches/s, reference CPU correction step (chunked residual)",
            "workload": name, "patches": len(ps), "fine_nodes": sF.n_nodes, "cores": cores,
            "all_cores": res[cores], "one_core": res[1], "chunk_cells": CHUNK,
            "excluded_setup_s": {"mesh_patchset": setup_s, "chunk_geometry": t_build},
            "wall_s": time.time() - t_start,
            "note": "BASELINE.md §2: the reference's own functions in float64; per chunk only "
                    "stab + apply_operator timed; BLAS threads via threadpoolctl"}
    print(json.dumps(line), flush=True)
    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    with open(os.path.join(REPO, "gpurun_out", f"cpu_reference_{name}.json"), "w") as f:
        json.dump(line, f, indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:2])
