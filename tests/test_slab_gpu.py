"""x-slab decomposition on one GPU: N slabs driven stage by stage in one process
(InProcessExchanger) through the real halo kernels of the C ABI.  The
assembled d must match the single-domain GPU step and the float64 oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_14837_b200 import mesh as meshmod, synthetic, net  # noqa: E402
from paper_2307_14837_b200.slab import (SlabPartition, SlabStep, InProcessExchanger,  # noqa: E402
                                        global_index)
from paper_2307_14837_b200.step import CorrectionStep  # noqa: E402

LO, HI, NC, JIT = (0.0, 0.0, 0.0), (1.0, 0.5, 0.5), (6, 2, 2), 31
NU, K = 1e-3, 0.005


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.fixture(scope="module")
def problem():
    gh = meshmod.build_template_mesh("box", extent_lo=LO, extent_hi=HI, n_cells=NC)
    synthetic.jitter_vertices(gh.levels[0].vertices, NC, LO, HI, JIT)
    meshmod.refine_uniform(gh)
    ps = meshmod.build_patches(gh, 0, 1)
    m = net.MlpModel(net.Architecture(240, 256, 3, 81), activation="tanh")
    m.W = synthetic.xavier_weights([240, 256, 256, 256, 81], 5)
    m.eval()
    modes = synthetic.fourier_modes(5)
    x1 = synthetic.coarse_state(gh.scalar_nodes(0)[0], modes, 5, 1, K, NU)
    step = CorrectionStep(gh, 0, 1, m, NU, K, precision="fp32", patchset=ps, t=K)
    xc = torch.tensor(x1, dtype=torch.float32, device="cuda")
    b = step.rhs_next(step.embed(torch.tensor(synthetic.coarse_state(
        gh.scalar_nodes(0)[0], modes, 5, 0, 0.0, NU), dtype=torch.float32, device="cuda")))
    step(xc, b)
    torch.cuda.synchronize()
    return gh, m, x1, b.clone(), step.d.double().cpu().numpy(), step.x_corr.double().cpu().numpy()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("precision", ["fp32", "tf32x3", "f16x3"])
def test_inprocess_slabs_match_single_domain(problem, world, precision):
    gh, m, x1, b, d_ref, xc_ref = problem
    g_fine, g_coarse = global_index(gh, 1), global_index(gh, 0)
    parts = [SlabPartition(LO, HI, NC, 0, 1, world, r, jitter_seed=JIT) for r in range(world)]
    steps = [SlabStep(p, m, NU, K, precision=precision, t=K) for p in parts]
    xs, bs, fids = [], [], []
    b4 = b.view(-1, 4)
    for p in parts:
        cid = torch.as_tensor(g_coarse(p.coarse_pos), device="cuda")
        fid = g_fine(p.fine_pos)
        fids.append(fid)
        xs.append(torch.tensor(x1, dtype=torch.float32, device="cuda").view(-1, 4)[cid].reshape(-1).contiguous())
        bs.append(b4[torch.as_tensor(fid, device="cuda")].reshape(-1).contiguous())
    a = [s.stage_residual(x, bb) for s, x, bb in zip(steps, xs, bs)]
    recv = InProcessExchanger.exchange_all(a)
    sums = [s.stage_predict(rv) for s, rv in zip(steps, recv)]
    recv = InProcessExchanger.exchange_all(sums)
    outs = [s.stage_finish(rv) for s, rv in zip(steps, recv)]
    torch.cuda.synchronize()
    d = np.zeros_like(d_ref).reshape(-1, 4)
    xc = np.zeros_like(xc_ref).reshape(-1, 4)
    for s, fid, o in zip(steps, fids, outs):
        d[fid] = s.step.d.double().cpu().numpy().reshape(-1, 4)
        xc[fid] = o.double().cpu().numpy().reshape(-1, 4)
    tol = 1e-5 if precision in ("tf32x3", "f16x3") else 1e-6
    assert rel(d.reshape(-1), d_ref) < tol
    assert rel(xc.reshape(-1), xc_ref) < tol
    for r in range(world - 1):  # both sides of every interface hold identical values
        L = steps[r].step.d.view(-1, 4)[steps[r].idx["right"].long()]
        R = steps[r + 1].step.d.view(-1, 4)[steps[r + 1].idx["left"].long()]
        assert torch.equal(L, R)
