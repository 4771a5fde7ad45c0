"""Golden Vanka smoothing by the REFERENCE (msolve.VankaData / vanka_smooth, msolve.py:51-89).

Runs only in the build container.  A jittered 3x1x1 channel box (level 0, 3 cells, 252
dofs) with its Jacobian assembled by the reference at a seeded state (convection,
LPS stabilisation; unmasked, so the cell blocks are well conditioned), the reference's Vanka
blocks, and 4 damped sweeps from a seeded iterate.

    python tests/golden/make_vanka.py             # rewrites tests/golden/vanka.npz
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from dnnmg import mesh as meshmod, space as spmod, driver, msolve  # noqa: E402

from paper_2307_14837_b200 import synthetic  # noqa: E402

LO, HI, NC = (0, 0, -0.205), (1.0, 0.41, 0.205), (3, 1, 1)


def main():
    h = meshmod.build_template_mesh("box", extent_lo=LO, extent_hi=HI, n_cells=NC, channel_tags=True)
    synthetic.jitter_vertices(h.levels[0].vertices, NC, LO, HI, 31)
    bcs = {meshmod.INFLOW: spmod.inflow_profile(3, 1.5, 0.41), meshmod.WALL: spmod.no_slip}
    pr = driver.NsProblem(h, nu=1e-3, k=0.02, bcs=bcs)
    s = pr.space(0)
    asm = pr.asm(0)
    rng = np.random.default_rng(41)
    xs = synthetic.coarse_state(s.nodes, synthetic.fourier_modes(41), 41, 1, pr.k, pr.nu)
    stab = asm.stab(xs, pr.nu, pr.k, pr.alpha0, pr.delta0)
    # the full (unmasked) Jacobian: on a 3-cell box the Dirichlet-condensed blocks are
    # near-singular (cond ~1e20), which would make any two inverses incomparable
    J = asm.assemble_jacobian(xs, pr.k, pr.nu, stab, mask=None)
    V = msolve.VankaData(asm, J)
    # a consistent system b = J x* (smoothing reduces the error), seeded start
    b = J @ (xs + 0.1 * rng.standard_normal(s.ndof))
    x0 = xs.copy()
    x4 = msolve.vanka_smooth(J, V, x0.copy(), b, 4, 0.7)
    np.savez_compressed(os.path.join(HERE, "vanka.npz"), indptr=J.indptr, indices=J.indices,
                        data=J.data, flat_pos=asm.flat_pos, cell_dofs=asm.cell_dofs,
                        ndof=s.ndof, x0=x0, b=b, x4=x4, weight=V.weight,
                        inv0=V.inv[0], flagged=np.array(V.flagged, dtype=np.int64))
    blocks = J.data[asm.flat_pos].reshape(asm.n_cells, asm.ndl, asm.ndl)
    print("cond", [f"{np.linalg.cond(B):.2e}" for B in blocks])
    print("ndof", s.ndof, "nnz", J.nnz, "cells", asm.n_cells, "|x4-x0|", np.linalg.norm(x4 - x0),
          "|b-Jx0|", np.linalg.norm(b - J @ x0), "|b-Jx4|", np.linalg.norm(b - J @ x4))


if __name__ == "__main__":
    main()
