"""The x-slab step across a REAL process boundary: 2 and 3 processes, each driving its slab's
CUDA kernels (K1..K5 and the halo pack / merge kernels) on the one leased GPU, exchanging
the interface messages with torch.distributed over gloo (staged through host memory; NCCL
refuses two ranks on one device).  The assembled r, d, x_corr and next-step RHS must be
bitwise equal to the single-domain GPU step.  No rank's kernels wait on another's: the
exchanges are host-synchronous."""
import os
import queue
import socket
import sys
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, precision, out_q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, REPO)
        sys.path.insert(0, os.path.join(REPO, "tests"))
        import test_slab_gpu as T
        from paper_2307_14837_b200.slab import SlabPartition, SlabStep, TorchDistExchanger
        torch.cuda.set_device(0)
        gh = T.meshmod.build_template_mesh("box", extent_lo=T.LO, extent_hi=T.HI,
                                           n_cells=T.CASES[1]["nc"])
        T.synthetic.jitter_vertices(gh.levels[0].vertices, T.CASES[1]["nc"], T.LO, T.HI, T.JIT)
        T.meshmod.refine_uniform(gh)
        g_fine, g_coarse = T.global_index(gh, 1), T.global_index(gh, 0)
        part = SlabPartition(T.LO, T.HI, T.CASES[1]["nc"], 0, 1, world, rank, jitter_seed=T.JIT)
        ex = TorchDistExchanger()
        assert ex.host
        slab = SlabStep(part, T.model_for(1), T.NU, T.K, precision=precision, t=T.K)
        modes = T.synthetic.fourier_modes(5)
        cid = g_coarse(part.coarse_pos)
        xyz = gh.scalar_nodes(0)[0]
        # the coarse states of the global box (as the single-domain run draws them: pressure
        # per global coarse node), restricted to this slab's coarse nodes
        x0, x1 = (torch.tensor(T.synthetic.coarse_state(xyz, modes, 5, n, n * T.K, T.NU)
                               .reshape(-1, 4)[cid].reshape(-1), dtype=torch.float32,
                               device="cuda") for n in (0, 1))
        slab.step.set_time(0.0)
        b = slab.rhs_next(slab.step.embed(x0), ex).clone()
        slab.step.set_time(T.K)
        out = slab.run(x1, b, ex).clone()
        b_next = slab.rhs_next(out, ex).clone()
        torch.cuda.synchronize()
        fid = g_fine(part.fine_pos)
        out_q.put((rank, fid, b.cpu().numpy(), slab.step.r.cpu().numpy(),
                   slab.step.d.cpu().numpy(), out.cpu().numpy(), b_next.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,precision", [(2, "f16x3"), (3, "fp32")])
def test_slab_processes_bitwise_equal_single_domain(world, precision):
    import test_slab_gpu as T
    import torch.multiprocessing as mp
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, precision, q)) for r in range(world)]
    for p in procs:
        p.start()
    results, deadline = {}, time.time() + 600
    while len(results) < world:
        try:
            item = q.get(timeout=2)
            results[item[0]] = item[1:]
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs) or time.time() > deadline:
                for p in procs:
                    p.kill()
                pytest.fail(f"slab worker failed (exit codes {[p.exitcode for p in procs]})")
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = T.single_domain(1, precision)
    for name, j in (("b", 1), ("r", 2), ("d", 3), ("x_corr", 4), ("b_next", 5)):
        full = np.full(ref[name].numel(), np.nan, dtype=np.float32).reshape(-1, 4)
        for rank, res in results.items():
            full[res[0]] = res[j].reshape(-1, 4)
        assert np.array_equal(full.reshape(-1), ref[name].cpu().numpy()), name
