#!/usr/bin/env python
"""Benchmark of the DNN-MG fine-level correction step (BASELINE.json metric:
"patches/sec for DNN-MG correction step (1/2/4/8 B200) and % of roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3]
                    [--precision fp32|bf16|tf32x3|f16x3] [--impl ours|reference]
                    [--no-e2e] [--no-cpu-baseline] [--no-aux]
    python bench.py --mlp-sweep        # BASELINE config 4: isolated patch-MLP sweep

Workload (default): BASELINE config 3 under the SURVEY §0.1 mapping — unit box,
level L = 64x32x32 cells, J = 1: 524,288 patches, 4,276,737 fine Q2 nodes,
MLP 240 -> 256x3 -> 81 tanh, seeded synthetic Fourier inputs, fp32 arithmetic
(the MLP in the fp32-accurate f16x3 tensor-core mode).

A timed step is one full correction (driver.py:251-268): prolongate (K1) ->
Dirichlet -> stab + residual (K2) -> patch gather (K3) -> patch MLP (K4) ->
averaging scatter + update (K5), inputs resident in HBM.  The timed steps
cycle over 4 distinct (x_L^n, b_prev^n) pairs (308 MB > 126 MB L2, and every
kernel streams >L2-sized arrays), so no step reads its inputs from L2.
`e2e` repeats the measurement through the public API with pinned HOST
buffers: x_L and b_prev copied H2D and x_corr copied D2H inside every step,
pipelined by step.HostPipeline (copies of neighbouring steps overlap the
kernels of the current one).

`aux` times the rows around the step (next-step RHS, restriction, training-data
rows + statistics, Vanka sweeps); they are not part of `value`.

--impl reference times the reference ITSELF (the unmodified package installed in
baseline/_ref, float64 numpy, all host threads and one) on a bounded sample of the same
workload.
Multi-GPU (torchrun): the x-slab decomposition (slab.py) of the config-3 box, strong
scaling, NCCL P2P halo exchange twice per step, timed on the device, max over ranks.
"""

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "patches/sec for DNN-MG correction step (1/2/4/8 B200) and % of roofline"
UNIT = "patches/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--precision", default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", default="16x8x8", help="coarse box of the CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--pipe-depth", type=int, default=2,
                    help="device input/output buffers of the e2e host pipeline")
    ap.add_argument("--no-aux", action="store_true", help="skip the next-row aux timings")
    ap.add_argument("--mlp-sweep", action="store_true",
                    help="BASELINE config 4: isolated patch-MLP sweep (one JSON line)")
    ap.add_argument("--sweep-batches", default="1024,16384,262144,4194304")
    ap.add_argument("--force-slabs", action="store_true",
                    help="run the multi-GPU x-slab path even on one GPU (code-path check)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def default_precision(cfg_name):
    """fp32-accuracy mode: every kernel in fp32, the MLP on tcgen05 with the
    3-pass fp16 split of scaled weights (f16x3: d within 1e-5 of the float64
    reference, tests/test_gpu_parity.py; tanh keeps activations in fp16 range).
    Width 256 (configs 0, 1, 3) runs the fused per-tile kernel, config 2
    (1024 -> 512x3 -> 375) the layer-major kernel."""
    return "f16x3"


# ---------------------------------------------------------------------------
# CPU oracle (reference port) timing — the only place bench.py runs oracle/
# ---------------------------------------------------------------------------

def cpu_oracle_rate(cfg, sample, steps, warmup):
    """Time the float64 oracle correction step on a bounded sample box."""
    from oracle import dnnmg_oracle as orc
    from paper_2307_14837_b200 import synthetic
    n_cells = tuple(int(v) for v in sample.split("x"))
    L, J = 0, cfg["J"]
    ctx = orc.build_context((0, 0, 0), (1, 1, 1), n_cells, L, J, cache_geometry=True)
    n_p = ctx["dof_table"].shape[0]
    npp = ctx["dof_table"].shape[1] // 4
    dims = [8 * npp + 24] + [cfg["hidden"]] * cfg["depth"] + [3 * npp]
    model = orc.Mlp(synthetic.xavier_weights(dims, cfg["seed"] + 7), activation="tanh")
    modes = synthetic.fourier_modes(cfg["seed"])
    nu, k = cfg["nu"], cfg["dt"]
    x0 = synthetic.coarse_state(ctx["coarse_coords"], modes, cfg["seed"], 0, 0.0, nu)
    xf0 = orc.prolongate_state(ctx["P"], x0)
    orc.impose_dirichlet(xf0, ctx["tags"], ctx["coords"], 0.0, {orc.WALL: orc.no_slip})
    b = orc.rhs_next(xf0, ctx["coords"], ctx["table"], k, nu, cache=ctx["geometry"])
    xs = [synthetic.coarse_state(ctx["coarse_coords"], modes, cfg["seed"], n, n * k, nu)
          for n in (1, 2)]
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        orc.correction_step(xs[i % 2], b, ctx, model, k * (1 + i % 2), nu, k)
        if i >= warmup:
            times.append(time.perf_counter() - t0)
    t = float(np.median(times))
    return n_p / t, n_p, t


REF_DIR = os.path.join(REPO, "baseline", "_ref")


def import_reference():
    """The UNMODIFIED reference package `dnnmg`, pip-installed into baseline/_ref (DESIGN.md
    §6 records the install).  Returns the module namespace or raises."""
    if not os.path.isdir(os.path.join(REF_DIR, "dnnmg")):
        raise RuntimeError("baseline/_ref/dnnmg is not installed")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import dnnmg  # noqa: F401
    from dnnmg import driver, mesh, net, patch_ops, space
    return dict(driver=driver, mesh=mesh, net=net, patch_ops=patch_ops, space=space)


class ReferenceStep:
    """One correction step of the reference's own code path (driver.py:251-268, BASELINE.md
    §2): embed_state (prolongate + Dirichlet) -> Assembler.stab -> assemble_residual ->
    patch_ops.predict_correction (gather, net.forward, bincount scatter) -> x~ + d, float64,
    on a bounded sample box with the config's per-patch work (same J, MLP, inputs)."""

    def __init__(self, cfg, sample):
        from paper_2307_14837_b200 import synthetic
        R = import_reference()
        self.R = R
        n_cells = tuple(int(v) for v in sample.split("x"))
        h = R["mesh"].build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1),
                                          n_cells=n_cells)
        if cfg["jitter"]:
            synthetic.jitter_vertices(h.levels[0].vertices, n_cells, (0, 0, 0), (1, 1, 1),
                                      cfg["seed"] + 1)
        for _ in range(cfg["J"]):
            R["mesh"].refine_uniform(h)
        self.L, self.J = 0, cfg["J"]
        self.nu, self.k = cfg["nu"], cfg["dt"]
        self.pr = R["driver"].NsProblem(h, nu=self.nu, k=self.k,
                                        bcs={R["mesh"].WALL: R["space"].no_slip})
        self.ps = R["mesh"].build_patches(h, self.L, self.J)
        n_in, n_out = R["patch_ops"].input_width(self.ps), R["patch_ops"].output_width(self.ps)
        self.model = R["net"].MlpModel(R["net"].Architecture(n_in, cfg["hidden"], cfg["depth"],
                                                             n_out), activation="tanh")
        self.model.W = synthetic.xavier_weights([n_in] + [cfg["hidden"]] * cfg["depth"] + [n_out],
                                                cfg["seed"] + 7)
        self.model.eval()
        fl = self.L + self.J
        self.asm = self.pr.asm(fl)           # the reference's Assembler (geometry cache: setup)
        self.mask = self.pr.mask(fl)
        modes = synthetic.fourier_modes(cfg["seed"])
        nodes = self.pr.space(self.L).nodes
        x0 = synthetic.coarse_state(nodes, modes, cfg["seed"], 0, 0.0, self.nu)
        xf0 = R["driver"].embed_state(self.pr, self.L, self.J, x0, 0.0)
        self.b = self.asm.assemble_rhs_next(xf0, None, None, self.k, self.nu)
        self.xs = [synthetic.coarse_state(nodes, modes, cfg["seed"], n, n * self.k, self.nu)
                   for n in (1, 2)]
        self.n_patches = len(self.ps)

    def __call__(self, i):
        R, pr = self.R, self.pr
        t = (1 + i % 2) * self.k
        xt = R["driver"].embed_state(pr, self.L, self.J, self.xs[i % 2], t)
        stab = self.asm.stab(xt, self.nu, self.k, pr.alpha0, pr.delta0)
        r = self.asm.assemble_residual(xt, self.b, self.k, self.nu, stab, mask=self.mask)
        d = R["patch_ops"].predict_correction(self.model, xt, r, self.ps, dirichlet_mask=self.mask)
        return xt + d


def reference_rate(step, steps, warmup, threads):
    """Mean patches/s of `steps` reference steps after `warmup`, with the BLAS pool limited to
    `threads` (threadpoolctl: OPENBLAS_NUM_THREADS at run time)."""
    from threadpoolctl import threadpool_limits
    with threadpool_limits(limits=threads):
        for i in range(warmup):
            step(i)
        t0 = time.perf_counter()
        for i in range(steps):
            step(i)
        dt = (time.perf_counter() - t0) / max(steps, 1)
    return step.n_patches / dt, dt


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the step (baseline/_ref,
    float64 numpy/scipy) on this host, all cores and one core, rank 0 only."""
    from paper_2307_14837_b200 import synthetic
    if rank != 0:
        return
    cfg = synthetic.CONFIGS[args.config]
    cores = os.cpu_count()
    try:
        t_setup = time.perf_counter()
        step = ReferenceStep(cfg, args.cpu_sample)
        t_setup = time.perf_counter() - t_setup
    except Exception as exc:
        print(json.dumps({"impl": "reference", "unavailable": f"reference import/setup failed: "
                          f"{str(exc)[:160]}"}), flush=True)
        return
    rate, t = reference_rate(step, args.steps, args.warmup, cores)
    rate1, t1 = reference_rate(step, max(1, args.steps // 4), min(args.warmup, 1), 1)
    sample = (f"{step.n_patches} patches ({args.cpu_sample} coarse box, J={cfg['J']}, "
              f"{cfg['hidden']}x{cfg['depth']} tanh MLP) of {args.config}: the reference's "
              f"embed_state -> stab -> assemble_residual -> predict_correction -> x~+d, float64; "
              f"mean of {args.steps} steps after {args.warmup} warm-up ({t:.3f} s/step); "
              f"setup (Assembler geometry cache, PatchSet) {t_setup:.1f} s excluded")
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "sample": args.cpu_sample},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "reference",
                         "threads": cores, "sample": sample,
                         "threads_1": {"value": rate1, "unit": UNIT, "cores": 1,
                                       "s_per_step": t1,
                                       "steps": max(1, args.steps // 4)}},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    REASONS = {
        0x0000000000000004: "sw_power_cap", 0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown", 0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown", 0x0000000000000002: "applications_clocks_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass
        self._stop = threading.Event()

    def _loop(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                bits = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for b, name in self.REASONS.items():
                    if bits & b:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def load_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def build_workload(cfg_name, precision, device_index):
    import torch
    from paper_2307_14837_b200 import mesh as meshmod, synthetic
    from paper_2307_14837_b200.net import Architecture, MlpModel
    from paper_2307_14837_b200.patch_ops import input_width, output_width
    from paper_2307_14837_b200.step import CorrectionStep
    cfg = synthetic.CONFIGS[cfg_name]
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1),
                                    n_cells=cfg["n_cells"])
    if cfg["jitter"]:
        synthetic.jitter_vertices(h.levels[0].vertices, cfg["n_cells"], (0, 0, 0), (1, 1, 1),
                                  cfg["seed"] + 1)
    for _ in range(cfg["J"]):
        meshmod.refine_uniform(h)
    ps = meshmod.build_patches(h, 0, cfg["J"])
    n_in, n_out = input_width(ps), output_width(ps)
    model = MlpModel(Architecture(n_in, cfg["hidden"], cfg["depth"], n_out), activation="tanh")
    model.W = synthetic.xavier_weights([n_in] + [cfg["hidden"]] * cfg["depth"] + [n_out],
                                       cfg["seed"] + 7)
    model.eval()
    nu, k = cfg["nu"], cfg["dt"]
    step = CorrectionStep(h, 0, cfg["J"], model, nu, k, precision=precision, patchset=ps)
    # seeded coarse states at t_n on the GPU (float64 Fourier sum, rounded to fp32)
    K, A, B = synthetic.fourier_modes(cfg["seed"])
    dev = torch.device("cuda", device_index)
    coarse_xyz = torch.tensor(h.scalar_nodes(0)[0], dtype=torch.float64, device=dev)
    kk = torch.tensor(2 * np.pi * K, dtype=torch.float64, device=dev)
    At = torch.tensor(A, dtype=torch.float64, device=dev)
    Bt = torch.tensor(B, dtype=torch.float64, device=dev)

    def coarse_state(n):
        t = n * k
        decay = torch.exp(-nu * (kk ** 2).sum(1) * t)
        x = torch.empty((coarse_xyz.shape[0], 4), dtype=torch.float64, device=dev)
        for s in range(0, coarse_xyz.shape[0], 1 << 16):
            ph = coarse_xyz[s:s + (1 << 16)] @ kk.T
            x[s:s + (1 << 16), 1:] = torch.cos(ph) @ (At * decay[:, None]) + \
                torch.sin(ph) @ (Bt * decay[:, None])
        x[:, 0] = torch.from_numpy(np.random.default_rng(cfg["seed"] + 1000 + n)
                                   .normal(0.0, 0.1, coarse_xyz.shape[0])).to(dev)
        return x.reshape(-1).float().contiguous()

    # carried fine RHS through the real recurrence: b^1 = rhs(embed(x^0)), b^{n+1} = rhs(x_corr^n)
    b = step.rhs_next(step.embed(coarse_state(0)))
    pairs = []
    for n in range(1, 5):
        xl = coarse_state(n)
        pairs.append((xl, b.clone()))
        xc = step(xl, b)
        b = step.rhs_next(xc)
    torch.cuda.synchronize()
    return step, pairs, cfg, h


def algorithmic_units(step, cfg):
    """Per-launch algorithmic bytes / flops of each kernel."""
    nf = step.space.n_nodes
    nl = step.coarse_ndof // 4
    npch = step.n_patches
    npp = step.ps.npp
    n_in, H, d, n_out = 8 * npp + 24, cfg["hidden"], cfg["depth"], 3 * npp
    return {
        "K1_prolong": {"bytes": 16 * nl + 16 * nf},
        "K2_residual": {"bytes": 72 * nf, "flops_ref_formulation": 213078 * step.level.n_cells},
        "K3_gather": {"bytes": 32 * nf + 96 * npch + 4 * n_in * npch},
        "K4_mlp": {"flops": 2 * (n_in * H + (d - 1) * H * H + H * n_out) * npch},
        "K3K4_gather_mlp": {"flops": 2 * (n_in * H + (d - 1) * H * H + H * n_out) * npch},
        "K5_scatter": {"bytes": 4 * n_out * npch + 48 * nf},
    }


def build_slab_workload(cfg_name, precision, device_index, world, rank, comm):
    """Strong scaling: the config's global box (config 3: 64x32x32 level-0 cells, 524,288
    patches) cut into `world` x-slabs; rank r owns slab r.  The coarse states are the global
    seeded fields at this slab's coarse nodes (pressure drawn per GLOBAL coarse node), the
    carried fine RHS follows the distributed recurrence b^{n+1} = rhs(x_corr^n) with merged
    interface rows."""
    import torch
    from paper_2307_14837_b200 import mesh as meshmod, synthetic
    from paper_2307_14837_b200.net import Architecture, MlpModel
    from paper_2307_14837_b200.slab import SlabPartition, SlabStep, global_index
    cfg = synthetic.CONFIGS[cfg_name]
    nc = tuple(cfg["n_cells"])
    jit = (cfg["seed"] + 1) if cfg["jitter"] else None
    part = SlabPartition((0, 0, 0), (1, 1, 1), nc, 0, cfg["J"], world, rank, jitter_seed=jit)
    npp = part.patchset.nodes_per_patch
    n_in, n_out = 8 * npp + 24, 3 * npp
    model = MlpModel(Architecture(n_in, cfg["hidden"], cfg["depth"], n_out), activation="tanh")
    model.W = synthetic.xavier_weights([n_in] + [cfg["hidden"]] * cfg["depth"] + [n_out],
                                       cfg["seed"] + 7)
    model.eval()
    nu, k = cfg["nu"], cfg["dt"]
    slab = SlabStep(part, model, nu, k, precision=precision)
    # global coarse node ids of this slab's coarse nodes (level-0 numbering of the global box)
    g0 = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1), n_cells=nc)
    n_glob = g0.scalar_nodes(0)[0].shape[0]
    cid = global_index(g0, 0)(part.coarse_pos)
    K, A, B = synthetic.fourier_modes(cfg["seed"])
    dev = torch.device("cuda", device_index)
    xyz = torch.tensor(part.h.scalar_nodes(0)[0], dtype=torch.float64, device=dev)
    kk = torch.tensor(2 * np.pi * K, dtype=torch.float64, device=dev)
    At = torch.tensor(A, dtype=torch.float64, device=dev)
    Bt = torch.tensor(B, dtype=torch.float64, device=dev)

    def coarse(n):
        t = n * k
        decay = torch.exp(-nu * (kk ** 2).sum(1) * t)
        x = torch.empty((xyz.shape[0], 4), dtype=torch.float64, device=dev)
        for s0 in range(0, xyz.shape[0], 1 << 16):
            ph = xyz[s0:s0 + (1 << 16)] @ kk.T
            x[s0:s0 + (1 << 16), 1:] = torch.cos(ph) @ (At * decay[:, None]) + \
                torch.sin(ph) @ (Bt * decay[:, None])
        p = np.random.default_rng(cfg["seed"] + 1000 + n).normal(0.0, 0.1, n_glob)[cid]
        x[:, 0] = torch.from_numpy(p).to(dev)
        return x.reshape(-1).float().contiguous()

    b = slab.rhs_next(slab.step.embed(coarse(0)), comm)
    pairs = []
    for n in range(1, 5):
        xl = coarse(n)
        pairs.append((xl, b.clone()))
        xc = slab.run(xl, b, comm)
        b = slab.rhs_next(xc, comm).clone()
    torch.cuda.synchronize()
    return slab, pairs, cfg


def slab_staged(slab, comm, x_coarse, b_prev, events):
    """slab.run with CUDA events between the stages (same kernels, same stream)."""
    import ctypes
    from paper_2307_14837_b200 import _lib, device as dvm
    st = slab.step
    s = dvm.stream_handle()
    e = iter(events)
    next(e).record()
    st.embed_into(x_coarse, st.x_tilde)
    next(e).record()
    _lib.call("dnnmg_residual", ctypes.byref(st.lv), dvm.ptr(st.x_tilde), dvm.ptr(b_prev), None,
              None, ctypes.byref(st.phys), dvm.ptr(st.elem), dvm.ptr(st.r), 1, s)
    next(e).record()
    _lib.call("dnnmg_halo_pre", ctypes.byref(slab.struct), comm.comm, dvm.ptr(st.elem),
              dvm.ptr(b_prev), dvm.ptr(st.mask_bits), dvm.ptr(st.r), s)
    next(e).record()
    st.predict_rows(s)
    next(e).record()
    _lib.call("dnnmg_scatter_update", ctypes.byref(st.ps.struct), dvm.ptr(st.Y),
              dvm.ptr(st.mask_bits), dvm.ptr(st.x_tilde), ctypes.c_float(st.scale), dvm.ptr(st.d),
              dvm.ptr(st.x_corr), s)
    next(e).record()
    _lib.call("dnnmg_halo_post", ctypes.byref(slab.struct), comm.comm, ctypes.byref(st.ps.struct),
              dvm.ptr(st.Y), dvm.ptr(st.mask_bits), dvm.ptr(st.x_tilde), ctypes.c_float(st.scale),
              dvm.ptr(st.d), dvm.ptr(st.x_corr), s)
    next(e).record()


SLAB_STAGES = ["K1_prolong", "K2_residual", "halo_a", "K3K4_gather_mlp", "K5_scatter", "halo_b"]


def run_slabs(args, rank, world, local):
    """x-slab decomposition of config 3 (strong scaling) over the library's own NCCL
    communicator: one rank per GPU under torchrun, or one process with --force-slabs."""
    import torch
    import torch.distributed as tdist
    from paper_2307_14837_b200.slab import NcclComm
    torch.cuda.set_device(local)
    tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = NcclComm(rank, world)
    assert comm.count() == world
    precision = args.precision or default_precision(args.config)
    slab, pairs, cfg = build_slab_workload(args.config, precision, local, world, rank, comm)
    st = slab.step
    S = len(pairs)

    def barrier():
        tdist.barrier()
        torch.cuda.synchronize()

    for i in range(args.warmup):
        slab.run(*pairs[i % S], comm)
    barrier()
    # per-stage events inside a first timed pass
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(SLAB_STAGES) + 1)]
    kern_ms = np.zeros(len(SLAB_STAGES))
    for i in range(args.steps):
        slab_staged(slab, comm, *pairs[i % S], ev)
        ev[-1].synchronize()
        kern_ms += np.array([ev[j].elapsed_time(ev[j + 1]) for j in range(len(SLAB_STAGES))])
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    with sampler:
        e0.record()
        for i in range(args.steps):
            slab.run(*pairs[i % S], comm)
        e1.record()
        barrier()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms = float(t.item())
    tot = torch.tensor([slab.part.n_patches], dtype=torch.float64, device="cuda")
    tdist.all_reduce(tot)
    n_total = int(tot.item())
    e2e = None
    if not args.no_e2e:
        # the same distributed steps with every rank's x_L / b_prev copied from pinned host
        # memory and its x_corr copied back inside each step, pipelined as step.HostPipeline:
        # H2D of step i+1 | kernels + halo exchanges of step i | D2H of step i-1
        hx = [p[0].cpu().pin_memory() for p in pairs]
        hb = [p[1].cpu().pin_memory() for p in pairs]
        hout = [torch.empty(st.x_corr.numel(), dtype=torch.float32).pin_memory() for _ in range(2)]
        dx = [torch.empty_like(pairs[0][0]) for _ in range(2)]
        db = [torch.empty_like(pairs[0][1]) for _ in range(2)]
        dout = [torch.empty_like(st.x_corr) for _ in range(2)]
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_run = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        used = [False, False]
        comp = torch.cuda.current_stream()
        barrier()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record()
        s_in.wait_stream(comp)
        s_out.wait_stream(comp)
        for i in range(args.steps):
            k = i % 2
            with torch.cuda.stream(s_in):
                if used[k]:
                    s_in.wait_event(ev_run[k])
                dx[k].copy_(hx[i % S], non_blocking=True)
                db[k].copy_(hb[i % S], non_blocking=True)
                ev_in[k].record()
            comp.wait_event(ev_in[k])
            if used[k]:
                comp.wait_event(ev_out[k])
            slab.run(dx[k], db[k], comm, x_corr=dout[k])
            ev_run[k].record()
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_run[k])
                hout[k].copy_(dout[k], non_blocking=True)
                ev_out[k].record()
            used[k] = True
        comp.wait_stream(s_in)
        comp.wait_stream(s_out)
        h1.record()
        barrier()
        te = torch.tensor([h0.elapsed_time(h1)], dtype=torch.float64, device="cuda")
        tdist.all_reduce(te, op=tdist.ReduceOp.MAX)
        byts = torch.tensor([(dx[0].numel() + db[0].numel()) * 4, hout[0].numel() * 4],
                            dtype=torch.float64, device="cuda")
        tdist.all_reduce(byts)
        e2e = {"value": n_total * args.steps / (float(te.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(byts[0].item()), "d2h_bytes_per_step": int(byts[1].item()),
               "overlap": "H2D(i+1) | kernels + halo exchanges(i) | D2H(i-1) on 3 streams"}
    if rank == 0:
        avg = kern_ms / args.steps
        per_kernel = {nm: {"ms": float(avg[j]), "share": float(avg[j] / avg.sum())}
                      for j, nm in enumerate(SLAB_STAGES)}
        units = algorithmic_units(st, cfg)
        peaks, peak_kind = load_peaks()
        for nm, entry in per_kernel.items():
            u = units.get(nm, {})
            if "bytes" in u:
                entry["GB/s"] = u["bytes"] / (entry["ms"] / 1e3) / 1e9
                entry["hbm_frac"] = entry["GB/s"] / peaks["hbm_gbs"]
            if "flops" in u:
                entry["TFLOP/s"] = u["flops"] / (entry["ms"] / 1e3) / 1e12
        roof = roofline_of(per_kernel, units, precision, peaks, peak_kind, st.level.n_cells,
                           "box" if st.level.geometry_box() is not None else "general")
        cpu = None if args.no_cpu_baseline else cpu_baseline_entry(cfg, args)
        line = {
            "metric": METRIC, "value": n_total * args.steps / (ms / 1e3), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32" if precision in ("fp32", "tf32x3", "f16x3")
            else f"f32 (MLP {precision})", "data": "synthetic",
            "config": {"workload": args.config, "patches": n_total,
                       "patches_rank0": slab.part.n_patches, "J": cfg["J"],
                       "coarse_cells": int(np.prod(cfg["n_cells"])), "precision": precision,
                       "parallelism": f"x-slab decomposition x{world} (strong scaling of the "
                       f"{args.config} box), NCCL send/recv halo exchange (2 per step) inside "
                       "libdnnmg_b200, interface sums merged in global order (bitwise equal "
                       "to 1 GPU)",
                       "l2": "inputs > L2 (4 cycled input pairs, every kernel streams >L2-sized "
                             "arrays)"},
            "e2e": e2e,
            "gpu_launches": int((st.launches + 4 * sum(p >= 0 for p in slab.part.peer.values()))
                                * args.steps),
            "roofline": roof, "kernels": per_kernel, "cpu_baseline": cpu,
            "clocks": sampler.summary(), "nccl_ranks": comm.count(),
        }
        print(json.dumps(line), flush=True)
    comm.close()
    tdist.destroy_process_group()


def dataset_aux(step, steps, barrier):
    """Next row #3: training-data rows of the step's x~ and r (dnnmg_dataset_rows, float64
    [x~ | r | geometry | targets] per patch) and their column statistics, config 3."""
    import ctypes
    import torch
    from paper_2307_14837_b200 import _lib, device as dvm
    ps = step.ps
    w = 11 * ps.npp + ps.n_geo
    rows = torch.empty((ps.n_patches, w), dtype=torch.float64, device="cuda")
    v_ref = torch.randn(step.x_tilde.numel(), dtype=torch.float64, device="cuda")
    lib = _lib.load()
    scratch = torch.empty(int(lib.dnnmg_column_stats_scratch(w)), dtype=torch.float64, device="cuda")
    stats = torch.empty((4, w), dtype=torch.float64, device="cuda")
    s = dvm.stream_handle()

    def rows_call():
        _lib.call("dnnmg_dataset_rows", ctypes.byref(ps.struct), dvm.ptr(step.x_tilde),
                  dvm.ptr(step.r), dvm.ptr(v_ref), None, dvm.ptr(rows), s)

    def stats_call():
        _lib.call("dnnmg_column_stats", dvm.ptr(rows), ctypes.c_int64(ps.n_patches), w,
                  dvm.ptr(scratch), dvm.ptr(stats), s)
    rows_call()
    stats_call()
    barrier()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    for _ in range(steps):
        rows_call()
    e[1].record()
    for _ in range(steps):
        stats_call()
    e[2].record()
    barrier()
    t_rows = e[0].elapsed_time(e[1]) / steps
    t_stats = e[1].elapsed_time(e[2]) / steps
    npp = ps.npp
    # algorithmic bytes per patch: node indices, x~ and r float4 rows, geometry, the three
    # float64 velocity comps of v_ref per node, and the float64 row written
    per_patch = 4 * npp + 2 * 16 * npp + 4 * ps.n_geo + 24 * npp + 8 * w
    byts = per_patch * ps.n_patches
    return {"rows_ms": t_rows, "rows_GB/s": byts / (t_rows / 1e3) / 1e9,
            "stats_ms": t_stats, "stats_GB/s": 8 * w * ps.n_patches / (t_stats / 1e3) / 1e9,
            "rows": ps.n_patches, "row_bytes": 8 * w,
            "note": "driver.export_training_data per step: row block + sidecar statistics"}


def vanka_aux(step, steps, barrier, n_cells=(16, 8, 8)):
    """Next row #4: cell-Vanka smoothing on a config-1-sized level (1,024 cells, 38,148 dofs,
    Q2/Q2 block pattern of Assembler._init_sparsity, synthetic diagonally dominant values):
    block inversion once, then sweeps (msolve.vanka_smooth)."""
    import scipy.sparse as spm
    import torch
    from paper_2307_14837_b200 import mesh as meshmod, msolve
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1),
                                    n_cells=n_cells)
    cn = h.scalar_nodes(0)[1]
    nc, ndof = cn.shape[0], 4 * h.scalar_nodes(0)[0].shape[0]
    dofs = (4 * cn[:, :, None] + np.arange(4)).reshape(nc, -1).astype(np.int64)
    ndl = dofs.shape[1]
    rows = np.repeat(dofs, ndl, axis=1).reshape(-1)
    cols = np.tile(dofs, (1, ndl)).reshape(-1)
    pat = spm.coo_matrix((np.ones(rows.size), (rows, cols)), shape=(ndof, ndof)).tocsr()
    pat.sort_indices()
    keys = np.repeat(np.arange(ndof, dtype=np.int64), np.diff(pat.indptr)) * ndof + pat.indices
    flat_pos = np.searchsorted(keys, rows * ndof + cols)
    rng = np.random.default_rng(5)
    data = rng.standard_normal(pat.nnz)
    data[np.searchsorted(keys, np.arange(ndof, dtype=np.int64) * (ndof + 1))] += 2.0 * ndl
    J = spm.csr_matrix((data, pat.indices, pat.indptr), shape=(ndof, ndof))

    class Asm:
        pass
    asm = Asm()
    asm.n_cells, asm.ndl, asm.cell_dofs, asm.flat_pos = nc, ndl, dofs, flat_pos

    class Space:
        pass
    asm.space = Space()
    asm.space.ndof = ndof
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    V = msolve.VankaData(asm, J)
    t1.record()
    torch.cuda.synchronize()
    x = torch.zeros(ndof, dtype=torch.float64, device="cuda")
    b = torch.tensor(rng.standard_normal(ndof), dtype=torch.float64, device="cuda")
    msolve.vanka_smooth(J, V, x, b, 2, 0.7)
    sweeps = 12 * max(1, steps // 4)
    barrier()
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record()
    msolve.vanka_smooth(J, V, x, b, sweeps, 0.7)
    s1.record()
    barrier()
    t_sweep = s0.elapsed_time(s1) / sweeps
    # per sweep: the inverse blocks (float64), the CSR matrix (value + column), the iterate
    # gathers and the per-dof accumulation
    byts = nc * ndl * ndl * 8 + J.nnz * 12 + ndof * 8 * 6 + nc * ndl * 16
    return {"cells": nc, "dofs": ndof, "nnz": int(J.nnz), "setup_ms": t0.elapsed_time(t1),
            "sweep_ms": t_sweep, "sweep_GB/s": byts / (t_sweep / 1e3) / 1e9,
            "note": "msolve.VankaData + vanka_smooth on a synthetic config-1-level Jacobian"}


# executed FP32 work of K2's element kernel per fine cell and lane, from its SASS mix at
# config 3 (ncu smsp__sass_thread_inst_executed_op_{ffma,fmul,fadd}_pred_on / 32 / cells,
# profiles/r1_kernels_cfg3_ncu.txt): FFMA 659.7, FMUL 271.8, FADD 85.4
# (general form, per-point geometry cache); the box form of axis-aligned levels (config 3,
# profiles/r2_kernels_cfg3_ncu.txt): FFMA 551.7, FMUL 273.9, FADD 85.4
DRAM_TRAFFIC_FILE = "r2_dram_traffic.json"   # newest ncu DRAM capture (per round)
K2_EXEC_FLOP_PER_CELL = {"general": 32 * (2 * 659.7 + 271.8 + 85.4),
                         "box": 32 * (2 * 551.7 + 273.9 + 85.4)}


def fp32_nominal_tflops(peaks):
    """FP32 SIMT peak: 148 SMs x 128 lanes x 2 FLOP x the max SM clock of MEASURED_PEAKS."""
    return 148 * 128 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12


def roofline_of(per_kernel, units, precision, peaks, peak_kind, n_cells=None, k2_form="general"):
    """`roofline` of the dominant stage (largest event time) and the K2 FP32 roofline."""
    names = [n for n in per_kernel if n in units or n.startswith("K3K4")]
    dom = max(names, key=lambda n: per_kernel[n]["ms"])
    du = units.get(dom, units["K4_mlp"])
    if "flops" in du:
        ach = du["flops"] / (per_kernel[dom]["ms"] / 1e3) / 1e12
        peak = {"bf16": peaks["bf16_tflops_sustained"],
                "f16x3": peaks["bf16_tflops_sustained"] / 3.0,
                "tf32x3": peaks["bf16_tflops_sustained"] / 2.0 / 3.0}.get(
                    precision, peaks["bf16_tflops_sustained"] / 2.0)
        roof = {"kernel": dom, "bound": "tensor", "achieved": ach, "peak": peak,
                "unit": "TFLOP/s", "frac": ach / peak, "traffic": None,
                "peak_source": f"{peak_kind} bf16 sustained"
                + {"bf16": "", "f16x3": " / 3 passes (fp16 rate = bf16 rate)",
                   "tf32x3": " / 2 (tf32 rate) / 3 passes"}.get(precision, " / 2")}
    else:
        ach = du["bytes"] / (per_kernel[dom]["ms"] / 1e3) / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": ach / peaks["hbm_gbs"], "traffic": None,
                "peak_source": f"{peak_kind} hbm copy"}
    # K2 is FP32-issue-bound, not HBM-bound: its executed FP32 work against the nominal FP32
    # SIMT peak at the max SM clock (no micro-benchmark number)
    if "K2_residual" in per_kernel and n_cells:
        pk = fp32_nominal_tflops(peaks)
        ach2 = K2_EXEC_FLOP_PER_CELL[k2_form] * n_cells / (per_kernel["K2_residual"]["ms"] / 1e3) / 1e12
        per_kernel["K2_residual"]["fp32_roofline"] = {
            "bound": "fp32 issue", "achieved": ach2, "peak": pk, "unit": "TFLOP/s",
            "frac": ach2 / pk,
            "peak_source": "nominal FP32: 148 SMs x 128 lanes x 2 x sm_max_mhz (MEASURED_PEAKS)",
            "element_kernel_form": k2_form,
            "flop_source": "executed FFMA/FMUL/FADD per cell from the element kernel's SASS mix"}
    # DRAM traffic per launch of each stage from the committed ncu capture
    try:
        with open(os.path.join(REPO, "profiles", DRAM_TRAFFIC_FILE)) as f:
            traffic = json.load(f)
    except Exception:
        traffic = {}
    if isinstance(traffic.get(dom), (int, float)):
        roof["traffic"] = traffic[dom]
        roof["traffic_source"] = f"profiles/{DRAM_TRAFFIC_FILE} (ncu --set full, per launch)"
    for nm, entry in per_kernel.items():
        if isinstance(traffic.get(nm), (int, float)):
            entry["dram_bytes_ncu"] = traffic[nm]
    return roof


def cpu_baseline_entry(cfg, args):
    """The reference's own CPU path (baseline/_ref) on this host on a bounded sample (rank 0,
    N = 1 line); the float64 oracle port when the reference is not installed."""
    cores = os.cpu_count()
    try:
        step = ReferenceStep(cfg, args.cpu_sample)
    except Exception as exc:
        rate, n_s, t_s = cpu_oracle_rate(cfg, args.cpu_sample, 2, 1)
        return {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                "sample": f"{n_s} patches ({args.cpu_sample} coarse box, J={cfg['J']}), float64 "
                          f"numpy oracle, median of 2 steps ({t_s:.2f} s/step); reference "
                          f"unavailable: {str(exc)[:80]}"}
    rate, t = reference_rate(step, 3, 1, cores)
    rate1, t1 = reference_rate(step, 2, 0, 1)
    return {"value": rate, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"{step.n_patches} patches ({args.cpu_sample} coarse box, J={cfg['J']}) "
                      f"through the reference's embed_state -> stab -> assemble_residual -> "
                      f"predict_correction, float64, mean of 3 steps ({t:.2f} s/step), all "
                      f"{cores} host threads",
            "threads_1": {"value": rate1, "unit": UNIT, "cores": 1, "s_per_step": t1}}


def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as tdist
    if world > 1 or args.force_slabs:
        if world == 1:   # single-process check of the distributed code path
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29555")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        return run_slabs(args, rank, world, local)
    torch.cuda.set_device(local)
    precision = args.precision or default_precision(args.config)
    step, pairs, cfg, h = build_workload(args.config, precision, local)
    n_p = step.n_patches
    S = len(pairs)

    def barrier():
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()

    # ---- per-kernel events inside the timed region (same stream) ----
    names = step.stage_names()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
    kern_ms = np.zeros(len(names))

    for i in range(args.warmup):
        step.run_staged(*pairs[i % S])
    barrier()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    with sampler:
        t_start.record()
        for i in range(args.steps):
            step.run_staged(*pairs[i % S], events=ev)
            # read this step's per-kernel durations lazily (events are reused next step)
            ev[-1].synchronize()
            kern_ms += np.array([ev[j].elapsed_time(ev[j + 1]) for j in range(len(names))])
        t_end.record()
        barrier()
    ms = t_start.elapsed_time(t_end)
    # device-timed fused path without per-kernel events (graph-free, same kernels)
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for i in range(args.steps):
        step(*pairs[i % S])
    f1.record()
    barrier()
    ms_fused = f0.elapsed_time(f1)
    # Alg. 1 lines 8-9 around the step (not part of `value`): next-step fine RHS from the
    # corrected state (K2 in RHS form + node sum) and its restriction to the coarse level (K6)
    aux = {}
    try:
        from paper_2307_14837_b200 import device as dvm
        xc_out = step(*pairs[0])
        b_next = step.rhs_next(xc_out)
        dvm.restrict_vector(h, b_next, step.L + step.J, step.J)   # builds the K6 tables
        barrier()
        a0, a1, a2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a0.record()
        for _ in range(args.steps):
            step.rhs_next(xc_out, b_next)
        a1.record()
        for _ in range(args.steps):
            dvm.restrict_vector(h, b_next, step.L + step.J, step.J)
        a2.record()
        barrier()
        aux = {"rhs_next_ms": a0.elapsed_time(a1) / args.steps,
               "restrict_ms": a1.elapsed_time(a2) / args.steps,
               "note": "Alg. 1 lines 8-9 (next-step RHS, P^T restriction); outside the timed step"}
    except Exception as exc:  # pragma: no cover - auxiliary numbers only
        aux = {"error": str(exc)[:200]}
    # the same step replayed from CUDA graphs (one per input pair): removes launch gaps,
    # which dominate for the small configs
    graphs = []
    for xl, bp in pairs:
        out = torch.empty_like(step.x_corr)
        g = torch.cuda.CUDAGraph()
        s_cap = torch.cuda.Stream()
        s_cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s_cap):
            step(xl, bp, out)
        torch.cuda.current_stream().wait_stream(s_cap)
        with torch.cuda.graph(g):
            step(xl, bp, out)
        graphs.append(g)
    for i in range(args.warmup):
        graphs[i % S].replay()
    barrier()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record()
    for i in range(args.steps):
        graphs[i % S].replay()
    g1.record()
    barrier()
    ms_graph = g0.elapsed_time(g1)
    ms_dev = min(ms, ms_fused, ms_graph)
    t = torch.tensor([ms_dev], dtype=torch.float64, device="cuda")
    if world > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * n_p * args.steps / (ms_max / 1e3)

    # ---- e2e through the public step API with pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        from paper_2307_14837_b200.step import HostPipeline
        hx = [p[0].cpu().pin_memory() for p in pairs]
        hb = [p[1].cpu().pin_memory() for p in pairs]
        hout = [torch.empty(step.x_corr.numel(), dtype=torch.float32).pin_memory()
                for _ in range(S)]
        pipe = HostPipeline(step, depth=args.pipe_depth)
        pipe.begin()
        for i in range(max(args.warmup, 2)):
            pipe.submit(hx[i % S], hb[i % S], hout[i % S])
        pipe.join()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pipe.begin()
        for i in range(args.steps):
            pipe.submit(hx[i % S], hb[i % S], hout[i % S])
        pipe.join()
        e1.record()
        barrier()
        dx, db = pipe.dx[0], pipe.db[0]
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        if world > 1:
            tdist.all_reduce(te, op=tdist.ReduceOp.MAX)
        e2e = {"value": world * n_p * args.steps / (float(te.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(dx.numel() * 4 + db.numel() * 4),
               "d2h_bytes_per_step": int(hout[0].numel() * 4),
               "overlap": "H2D(i+1) | kernels(i) | D2H(i-1) on 3 streams (step.HostPipeline)"}

    # the rows around the step (training-data rows + statistics, Vanka sweeps): after the e2e
    # measurement -- their host-side setup (scipy / BLAS worker threads) otherwise competes with
    # the thread that enqueues the pipelined copies (e2e 269 M instead of 295 M patches/s)
    if not args.no_aux:
        for key, fn in (("dataset_rows", dataset_aux), ("vanka", vanka_aux)):
            try:
                aux[key] = fn(step, args.steps, barrier)
            except Exception as exc:  # pragma: no cover - auxiliary numbers only
                aux[key] = {"error": str(exc)[:200]}
    if rank != 0:
        if world > 1:
            tdist.destroy_process_group()
        return
    # ---- roofline of the dominant kernel ----
    peaks, peak_kind = load_peaks()
    units = algorithmic_units(step, cfg)
    avg = kern_ms / args.steps
    share = avg / avg.sum()
    per_kernel = {}
    for j, nm in enumerate(names):
        u = units.get(nm, units.get("K4_mlp"))
        entry = {"ms": float(avg[j]), "share": float(share[j])}
        if "bytes" in u:
            entry["GB/s"] = u["bytes"] / (avg[j] / 1e3) / 1e9
            entry["hbm_frac"] = entry["GB/s"] / peaks["hbm_gbs"]
        if "flops" in u:
            entry["TFLOP/s"] = u["flops"] / (avg[j] / 1e3) / 1e12
        if "flops_ref_formulation" in u:
            entry["ref_formulation_TFLOP/s"] = u["flops_ref_formulation"] / (avg[j] / 1e3) / 1e12
        per_kernel[nm] = entry
    roof = roofline_of(per_kernel, units, precision, peaks, peak_kind, step.level.n_cells,
                       "box" if step.level.geometry_box() is not None else "general")
    cpu = None if args.no_cpu_baseline else cpu_baseline_entry(cfg, args)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "f32" if precision in ("fp32", "tf32x3", "f16x3") else f"f32 (MLP {precision})",
        "data": "synthetic",
        "config": {"workload": args.config, "patches": n_p, "fine_nodes": step.space.n_nodes,
                   "coarse_cells": int(np.prod(cfg["n_cells"])), "J": cfg["J"],
                   "mlp": f"{8 * step.ps.npp + 24}->{cfg['hidden']}x{cfg['depth']}->{3 * step.ps.npp} tanh",
                   "precision": precision, "l2": "inputs > L2 (4 cycled input pairs, 308 MB)",
                   "parallelism": "single GPU"},
        "e2e": e2e,
        "gpu_launches": int(step.launches * args.steps),
        "roofline": roof,
        "kernels": per_kernel,
        "ms_per_step_fused": ms_fused / args.steps, "ms_per_step_staged": ms / args.steps,
        "ms_per_step_graph": ms_graph / args.steps,
        "aux": aux,
        "cpu_baseline": cpu,
        "clocks": sampler.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        tdist.destroy_process_group()


def run_mlp_sweep(args):
    """BASELINE config 4: isolated patch-MLP throughput, 174 -> H x3 -> 81 tanh, Xavier
    weights, N(0,1) inputs resident in HBM, for H in {128, 256, 512, 1024}, batches
    2^10 .. 2^22 rows and the tensor-core modes (fp32-accurate f16x3 / tf32x3, bf16).
    H = 128 and 256 run the fused per-tile kernel, 512 and 1024 the layer-major kernel.
    One JSON line: rows/s, TFLOP/s of the reference FLOPs and the fraction of the mode's
    tensor peak per point (CUDA events, median-free mean of K launches after W warm-ups)."""
    import torch
    from paper_2307_14837_b200 import device as dvm, synthetic
    from paper_2307_14837_b200.net import Architecture, MlpModel
    peaks, peak_kind = load_peaks()
    modes = (args.precision,) if args.precision else ("f16x3", "tf32x3", "bf16", "fp8")
    hs = (128, 256, 512, 1024)
    batches = tuple(int(b) for b in args.sweep_batches.split(","))
    out = []
    for H in hs:
        dims = [174, H, H, H, 81]
        model = MlpModel(Architecture(174, H, 3, 81), activation="tanh")
        model.W = synthetic.xavier_weights(dims, 4 + H)
        model.eval()
        flop = 2 * sum(a * b for a, b in zip(dims[:-1], dims[1:]))
        for mode in modes:
            dm = dvm.DeviceModel(model, mode)
            for B in batches:
                X = torch.randn((B, 174), device="cuda")
                Y = torch.empty((B, 81), device="cuda")
                dm.workspace(B)
                for _ in range(max(args.warmup, 3)):
                    dm.forward(X, B, Y)
                reps = max(3, min(args.steps, int(2 ** 22 // B) + 3))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(reps):
                    dm.forward(X, B, Y)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
                tf = flop * B / (ms / 1e3) / 1e12
                peak = {"bf16": peaks["bf16_tflops_sustained"],
                        "f16x3": peaks["bf16_tflops_sustained"] / 3.0,
                        "tf32x3": peaks["bf16_tflops_sustained"] / 6.0,
                        "fp8": 2.0 * peaks["bf16_tflops_sustained"]}[mode]
                out.append({"H": H, "mode": mode, "batch": B, "ms": ms, "rows/s": B / (ms / 1e3),
                            "TFLOP/s": tf, "frac": tf / peak,
                            "kernel": ("fused" if dvm.tc_fused_supported(model.arch) and mode != "fp8"
                                       else "layered")})
                del X, Y
            del dm
    line = {"metric": "patch-MLP rows/s and TFLOP/s (BASELINE config 4)", "n_gpus": 1,
            "data": "synthetic", "dtype": "fp32 accumulate",
            "config": {"workload": "cfg4", "mlp": "174 -> H x3 -> 81 tanh", "H": list(hs),
                       "batches": list(batches), "modes": list(modes)},
            "peak_source": f"{peak_kind} bf16 sustained; f16x3 = /3, tf32x3 = /6, fp8 = x2",
            "points": out}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.mlp_sweep:
        run_mlp_sweep(args)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
