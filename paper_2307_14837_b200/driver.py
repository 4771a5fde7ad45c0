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


# -- training data on the GPU (driver.py:286-431) -------------------

def steps_in_interval(interval, k, n_max):
    """Step indices n in 1..n_max with lo < n k <= hi (driver.py:286-291)."""
    lo, hi = interval
    eps = 1e-9 * k
    return [n for n in range(1, n_max + 1) if lo + eps < n * k <= hi + eps]


class _FineMachinery:
    """Device workspace of the replayed hybrid machinery on level L+J: embedding with
    Dirichlet data at t (K1), next RHS (K2 RHS form), residual (K2), dataset rows, column
    statistics, ideal correction.  Vectors are fp32 CUDA tensors, trajectory values
    float64 on the device."""

    def __init__(self, problem, L, J, patchset):
        if getattr(problem, "f", None) is not None:
            raise NotImplementedError("volume forces on the fine level are not supported")
        if not getattr(problem, "reimpose_fine_dirichlet", True):
            raise NotImplementedError("reimpose_fine_dirichlet=False is not supported")
        self.pr, self.L, self.J = problem, L, J
        fl = L + J
        self.step = CorrectionStep(problem.hierarchy, L, J, None, problem.nu, problem.k,
                                   bcs=problem.bcs, alpha0=problem.alpha0,
                                   delta0=problem.delta0, patchset=patchset,
                                   mask=np.asarray(problem.mask(fl)))
        self.ps = self.step.ps
        self.w = 11 * self.ps.npp + self.ps.n_geo
        self.nf = 8 * self.ps.npp + self.ps.n_geo
        dev = self.step.x_tilde.device
        self.rows = torch.empty((self.ps.n_patches, self.w), dtype=torch.float64, device=dev)
        lib = _lib()
        self.scratch = torch.empty(int(lib.dnnmg_column_stats_scratch(self.w)),
                                   dtype=torch.float64, device=dev)
        self.stats = torch.empty((4, self.w), dtype=torch.float64, device=dev)

    def embed(self, values, t, out=None):
        self.step.set_time(t)
        out = torch.empty_like(self.step.x_tilde) if out is None else out
        return self.step.embed_into(dv.f32(values), out)

    def rhs(self, x):
        return self.step.rhs_next(x)

    def residual(self, xt, b):
        return self.step.residual_into(xt, b, torch.empty_like(xt))

    def make_rows(self, xt, r, v_ref=None, x_ref=None):
        """Feature + target rows [n_patches][w] (float64) and their column statistics."""
        import ctypes
        s = dv.stream_handle()
        vr = None if v_ref is None else _f64(v_ref)
        xr = None if x_ref is None else _f64(x_ref)
        lib_call("dnnmg_dataset_rows", ctypes.byref(self.ps.struct), dv.ptr(xt), dv.ptr(r),
                 dv.ptr(vr), dv.ptr(xr), dv.ptr(self.rows), s)
        lib_call("dnnmg_column_stats", dv.ptr(self.rows), ctypes.c_int64(self.ps.n_patches),
                 self.w, dv.ptr(self.scratch), dv.ptr(self.stats), s)
        return self.rows.cpu().numpy(), self.stats.cpu().numpy()

    def ideal_update(self, xt, v_ref):
        import ctypes
        out = torch.empty_like(xt)
        lib_call("dnnmg_ideal_update", ctypes.c_int32(xt.numel() // 4), dv.ptr(xt),
                 dv.ptr(_f64(v_ref)), dv.ptr(self.step.mask_bits), dv.ptr(out),
                 dv.stream_handle())
        return out

    def restrict(self, bf):
        return spmod.restrict_rhs(self.pr.hierarchy, bf, self.L + self.J, self.J)


def _lib():
    from . import _lib as lib
    return lib.load()


def lib_call(name, *args):
    from . import _lib as lib
    lib.call(name, *args)


def _f64(v):
    if isinstance(v, torch.Tensor):
        return v.to(device=dv.device(), dtype=torch.float64).contiguous()
    return torch.from_numpy(np.array(v, dtype=np.float64)).to(dv.device())


def embed_state(problem, L, J, values, t):
    """Prolongate coarse values to L+J and re-impose the boundary data at t (driver.py:611-619),
    on the GPU; numpy in -> float64 numpy out."""
    m = _FineMachinery(problem, L, J, meshmod.build_patches(problem.hierarchy, L, J))
    return dv.like_input(m.embed(values, t), values)


def replay_features(problem, L, J, coarse_values, b_fine, t):
    """One step of the hybrid machinery without a model: (x~, r) (driver.py:294-314)."""
    m = _FineMachinery(problem, L, J, meshmod.build_patches(problem.hierarchy, L, J))
    xt = m.embed(coarse_values, t)
    r = m.residual(xt, dv.f32(b_fine))
    return dv.like_input(xt, coarse_values), dv.like_input(r, coarse_values)


def _loop_rows(m, coarse_traj, fine_traj, n_start, interval, emit):
    """oracle_loop_features (driver.py:386-431) on the device: the hybrid loop under the
    ideal correction from the coarse state at n_start; emit(n, rows, stats) per step."""
    pr, L, J = m.pr, m.L, m.J
    x = spmod.StateVector(L, np.array(coarse_traj.values(n_start), dtype=float), n_start * pr.k)
    xf = m.embed(x.values, x.time)
    bf = m.rhs(xf)
    b = m.restrict(bf).double().cpu().numpy()
    solver = None
    n = n_start
    eps = 1e-9 * pr.k
    while (n + 1) * pr.k <= interval[1] + eps and n + 1 <= fine_traj.n_steps:
        n += 1
        t = n * pr.k
        x, _, solver = pr.solve_step(L, x, b, t, solver=solver)
        xt = m.embed(x.values, t)
        r = m.residual(xt, bf)
        v = fine_traj.values(n)
        rows, stats = m.make_rows(xt, r, v_ref=v)
        emit(n, rows, stats)
        x_corr = m.ideal_update(xt, v)
        bf = m.rhs(x_corr)
        b = m.restrict(bf).double().cpu().numpy()


def oracle_loop_features(problem, L, J, coarse_traj, fine_traj, n_start, interval, patchset):
    """(n, features, targets) per step of the ideal-correction loop (driver.py:386-431)."""
    m = _FineMachinery(problem, L, J, patchset)
    out = []
    _loop_rows(m, coarse_traj, fine_traj, n_start, interval,
               lambda n, rows, st: out.append((n, rows[:, :m.nf].copy(), rows[:, m.nf:].copy())))
    return out


def export_training_data(problem, L, J, coarse_traj, fine_traj, t_train, t_val, out_dir,
                         shard_bytes=256 * 2 ** 20, loop_pass=False):
    """The (features, targets) dataset of a coarse and a fine run (driver.py:317-383), built
    on the GPU and streamed into the reference's shard format (io.write_dataset).

    Per step n in the half-open windows: x~ = embed(coarse^n), b = rhs(embed(coarse^{n-1})),
    r = b - A_h(x~) (K1, K2); the row block [x~ | r | geometry | fine^n - x~] is formed by
    ``dnnmg_dataset_rows`` and its column statistics by ``dnnmg_column_stats``.  With
    loop_pass the ideal-correction loop's rows are appended (the coarse solves are the
    problem's own, as in the reference)."""
    from . import io as iomod
    pr = problem
    if abs(coarse_traj.k - fine_traj.k) > 1e-14:
        raise ValueError("runs do not share the time step size")
    fl = L + J
    if fine_traj.level != fl:
        raise ValueError(f"fine run level {fine_traj.level} incompatible with L={L}, J={J}")
    same_level = coarse_traj.level == fl
    if not same_level and coarse_traj.level != L:
        raise ValueError(f"coarse run level {coarse_traj.level} != L={L}")
    patchset = meshmod.build_patches(pr.hierarchy, L, J)
    n_max = min(coarse_traj.n_steps, fine_traj.n_steps)
    windows = (("train", t_train), ("val", t_val))
    steps = {name: steps_in_interval(iv, pr.k, n_max) for name, iv in windows}
    loop_steps = []
    n_lo = None
    if loop_pass and not same_level:
        lo, hi = min(t_train[0], t_val[0]), max(t_train[1], t_val[1])
        n_lo = steps_in_interval((lo, hi), pr.k, n_max)[0]
        eps = 1e-9 * pr.k
        n = n_lo - 1
        while (n + 1) * pr.k <= hi + eps and n + 1 <= fine_traj.n_steps:
            n += 1
            loop_steps.append(n)
    m = _FineMachinery(pr, L, J, patchset)
    n_p = m.ps.n_patches
    writer = iomod.DatasetWriter(out_dir, patchset)
    loop_in = {name: [n for n in loop_steps if n in set(steps_in_interval(iv, pr.k, n_max))]
               for name, iv in windows}
    for name, _ in windows:
        writer.begin_set(name, n_p * (len(steps[name]) + len(loop_in[name])), m.nf,
                         3 * m.ps.npp, shard_bytes)
    for name, _ in windows:
        for n in steps[name]:
            xc = coarse_traj.values(n)
            v = fine_traj.values(n)
            if same_level:
                xt = dv.f32(xc)
                rows, stats = m.make_rows(xt, None, v_ref=v, x_ref=xc)
            else:
                xp = m.embed(coarse_traj.values(n - 1), (n - 1) * pr.k)
                b_prev = m.rhs(xp)
                xt = m.embed(xc, n * pr.k)
                r = m.residual(xt, b_prev)
                rows, stats = m.make_rows(xt, r, v_ref=v)
            writer.add_rows(name, rows, stats)
    if loop_steps:
        def emit(n, rows, stats):
            for name, _ in windows:
                if n in loop_in[name]:
                    writer.add_rows(name, rows, stats)
        _loop_rows(m, coarse_traj, fine_traj, n_lo - 1, (None, max(t_train[1], t_val[1])), emit)
    return writer.finish()


# -- checkpoint / resume (driver.py:442-480) --------------------------------------------

def checkpoint_state(loop):
    """Arrays + meta needed to resume a loop exactly (driver.py:442-450); the fine state
    and the carried fine RHS come back from the device."""
    st = loop.state
    arrays = {"x": st.x.values, "b_next": st.b_next}
    if st.x_fine is not None:
        arrays["x_fine"] = st.x_fine.values
        arrays["b_next_fine"] = st.b_next_fine
    meta = {"level": loop.level, "J": loop.J, "n": st.n, "t": st.t}
    return st.n, st.t, arrays, meta


def resume_loop(problem, ckpt_path, model=None, J=None, precision="fp32", **kw):
    """TimeLoop continued from a "DMGC" checkpoint (driver.py:453-480).  A pure-MG checkpoint
    (J = 0) resumes as a hybrid loop when J is given: the fine RHS history is rebuilt from
    the embedded coarse state on the device, as a zero-correction hybrid run would carry."""
    from . import io as iomod
    step, t, arrays, meta = iomod.load_checkpoint(ckpt_path)
    J = J if J is not None else meta["J"]
    to_hybrid = J > 0 and meta["J"] == 0
    loop = TimeLoop(problem, meta["level"], J, model=model, precision=precision, **kw)
    L, fl = meta["level"], meta["level"] + J
    x = spmod.StateVector(L, arrays["x"].copy(), t)
    st = TimeLoopState(step, t, x, arrays["b_next"].copy())
    if "x_fine" in arrays:
        st.x_fine = spmod.StateVector(fl, dv.f32(arrays["x_fine"]), t)
        st.b_next_fine = dv.f32(arrays["b_next_fine"])
    elif to_hybrid:
        loop.fine.set_time(t)
        xf = loop.fine.embed_into(dv.f32(x.values), torch.empty_like(loop.fine.x_tilde))
        st.x_fine = spmod.StateVector(fl, xf, t)
        st.b_next_fine = loop.fine.rhs_next(xf)
        # the coarse RHS of the first resumed solve is the restriction of the rebuilt fine
        # RHS, not the pure-MG checkpoint's own b_next (driver.py:476-478)
        st.b_next = loop._restrict(st.b_next_fine)
    loop.state = st
    return loop
