"""Hybrid DNN-MG time loop with the fine level on the GPU (driver.TimeLoop, driver.py:170-280).

Drop-in for the reference's ``TimeLoop`` in hybrid mode (J >= 1): the coarse implicit
solve stays with the caller's problem object (the reference ``NsProblem`` and its
Newton / GMRES / multigrid solver on the host, out of scope here), everything on the
fine level runs as sm_100a kernels through the C ABI:

    step n (driver.py:245-280)                          here
    x = problem.solve_step(L, x, b_next, t)             caller (host)
    x~ = prolongate(x); apply_dirichlet(x~, t)          K1   (CorrectionStep.embed_into / run)
    stab, r = b_next_fine - A_h(x~)                     K2
    d = predict_correction(model, x~, r)                K3/K4/K5 (fused step)
    x_corr = x~ + scale d   (t >= correction_start)
    b_next_fine = assemble_rhs_next(x_corr)             K2, RHS form (dnnmg_rhs_next)
    b_next = restrict_rhs(b_next_fine)                  K6   (dnnmg_restrict), copied to host

The carried fine RHS ``b_next_fine`` and the corrected fine state stay in HBM (fp32)
between steps; only the coarse vectors cross PCIe (x in, b_next out), which is what a
host-side coarse solver needs.  The problem object is duck-typed on the attributes the
reference loop uses: ``hierarchy, nu, k, bcs, alpha0, delta0, f, convection,
reimpose_fine_dirichlet, space(level), mask(level), solve_step(level, x, b, t,
solver=None)``.
"""

import time as _time
from dataclasses import dataclass

import numpy as np
import torch

from . import device as dv, mesh as meshmod, space as spmod
from .step import CorrectionStep


@dataclass
class TimeLoopState:
    """driver.TimeLoopState (driver.py:144-153); x_fine.values and b_next_fine are
    fp32 CUDA tensors, x / b_next the host (float64) coarse vectors of the solver."""
    n: int
    t: float
    x: object
    b_next: np.ndarray
    x_fine: object = None
    b_next_fine: object = None
    prev_x: object = None
    prev_x_fine: object = None


@dataclass
class StepStats:
    """driver.StepStats (driver.py:156-166)."""
    n: int = 0
    t: float = 0.0
    newton_iterations: int = 0
    gmres_iterations: int = 0
    jacobian_builds: int = 0
    wall_time: float = 0.0
    net_time: float = 0.0
    net_evals: int = 0


class TimeLoop:
    """Sequential hybrid time loop over (L, L+J); see the module docstring.

    correction_start delays the network corrections (before it the step is the
    zero-correction step, driver.py:261); correction_scale damps the defect."""

    def __init__(self, problem, level, J=0, model=None, initial=None, correction_scale=1.0,
                 correction_start=0.0, precision="fp32"):
        if J < 1:
            raise NotImplementedError("pure multigrid runs (J = 0) have no fine-level "
                                      "correction; use the coarse solver's own loop")
        if getattr(problem, "f", None) is not None:
            raise NotImplementedError("volume forces on the fine level are not supported "
                                      "(the correction path uses f = None)")
        if not getattr(problem, "convection", True):
            raise NotImplementedError("the Stokes form (convection=False) is not supported")
        if not getattr(problem, "reimpose_fine_dirichlet", True):
            raise NotImplementedError("reimpose_fine_dirichlet=False is not supported")
        self.problem = problem
        self.level = level
        self.J = J
        self.model = model
        self.correction_scale = correction_scale
        self.correction_start = correction_start
        fl = level + J
        self.patchset = meshmod.build_patches(problem.hierarchy, level, J)
        self.fine = CorrectionStep(problem.hierarchy, level, J, model, problem.nu, problem.k,
                                   bcs=problem.bcs, alpha0=problem.alpha0,
                                   delta0=problem.delta0, scale=correction_scale,
                                   precision=precision, patchset=self.patchset,
                                   mask=np.asarray(problem.mask(fl)))
        self.solver = None
        self.net_evals = 0
        self.state = self._initial_state(initial)
        self.step_log = []

    @property
    def fine_level(self):
        return self.level + self.J

    def _restrict(self, bf):
        b = spmod.restrict_rhs(self.problem.hierarchy, bf, self.fine_level, self.J)
        return b.double().cpu().numpy()

    def _initial_state(self, initial):
        """driver.py:201-219: coarse initial state with Dirichlet data at t = 0, its
        embedding on level L+J and the first carried right-hand sides."""
        pr = self.problem
        s = pr.space(self.level)
        x0 = s.zero_state()
        if initial is not None:
            vals = initial(0.0, s.nodes)
            x0.values.reshape(s.n_nodes, s.n_comp)[:, 1:] = vals
        _coarse_dirichlet(s, x0, 0.0, pr.bcs)
        self.fine.set_time(0.0)
        xf = self.fine.embed_into(dv.f32(x0.values), torch.empty_like(self.fine.x_tilde))
        bf = self.fine.rhs_next(xf)
        fl = self.fine_level
        return TimeLoopState(0, 0.0, x0, self._restrict(bf),
                             x_fine=spmod.StateVector(fl, xf, 0.0), b_next_fine=bf)

    def step(self):
        t0 = _time.perf_counter()
        stats = self._step_hybrid()
        stats.wall_time = _time.perf_counter() - t0
        self.step_log.append(stats)
        return self.state

    def _step_hybrid(self):
        pr, st, L = self.problem, self.state, self.level
        fl = self.fine_level
        t_next = round(st.t / pr.k + 1) * pr.k
        x, nstats, self.solver = pr.solve_step(L, st.x, st.b_next, t_next, solver=self.solver)
        self.fine.set_time(t_next)
        xc = dv.f32(x.values)
        x_corr = torch.empty_like(self.fine.x_tilde)
        net_time = 0.0
        if self.model is not None and t_next >= self.correction_start - 1e-12:
            tn = _time.perf_counter()
            self.fine.run(xc, st.b_next_fine, x_corr)   # K1..K5 (residual against b_next_fine)
            torch.cuda.current_stream().synchronize()
            net_time = _time.perf_counter() - tn
            self.net_evals += 1
        else:
            self.fine.embed_into(xc, x_corr)             # zero correction: x_corr = x~
        bf = self.fine.rhs_next(x_corr)
        b = self._restrict(bf)
        self.state = TimeLoopState(st.n + 1, t_next, x, b,
                                   x_fine=spmod.StateVector(fl, x_corr, t_next),
                                   b_next_fine=bf, prev_x=st.x, prev_x_fine=st.x_fine)
        return StepStats(st.n + 1, t_next, _stat(nstats, "iterations"),
                         _stat(nstats, "gmres_iterations"), _stat(nstats, "jacobian_builds"),
                         net_time=net_time, net_evals=1 if self.model is not None else 0)

    def run(self, n_steps, callback=None):
        for _ in range(n_steps):
            self.step()
            if callback is not None:
                callback(self)
        return self.state


def _stat(obj, name):
    return int(getattr(obj, name, 0) or 0)


def _coarse_dirichlet(space, x, t, bcs):
    """Dirichlet data on the coarse (host) state, exactly space.apply_dirichlet
    (space.py:245-255): every node carries one tag (precedence resolved when tagging)."""
    v = x.values.reshape(space.n_nodes, space.n_comp)
    for tag, fn in bcs.items():
        idx = space.nodes_with_tag(tag)
        if len(idx) == 0 or fn is None:
            continue
        v[idx, 1:] = fn(t, space.nodes[idx])
    x.time = t
    return x
