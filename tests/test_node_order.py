"""Visiting order of the owner-computes node passes (K2's node sum, K5's scatter):
`device.visit_order` is a permutation by descending first incident row, and the
correction step gives the same bits in every order (each node's own sum stays in its
CSR row's ascending order, the reference's bincount order)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2307_14837_b200 import device as dv  # noqa: E402


def test_visit_order_is_descending_first_row(monkeypatch):
    monkeypatch.delenv("DNNMG_NODE_ORDER", raising=False)
    rng = np.random.default_rng(3)
    table = np.stack([rng.permutation(40)[:6] for _ in range(30)])
    ptr, idx = dv.node_csr(table)
    order = dv.visit_order(ptr, idx)
    n = ptr.size - 1
    assert sorted(order.tolist()) == list(range(n))
    first = [idx[ptr[i]] if ptr[i + 1] > ptr[i] else -1 for i in range(n)]
    keys = [(first[i], i) for i in order]
    assert keys == sorted(keys, reverse=True)
    monkeypatch.setenv("DNNMG_NODE_ORDER", "forward")
    assert np.array_equal(dv.visit_order(ptr, idx), order[::-1])
    monkeypatch.setenv("DNNMG_NODE_ORDER", "ascending")
    assert dv.visit_order(ptr, idx) is None


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
def test_step_bits_independent_of_visit_order(monkeypatch):
    from paper_2307_14837_b200 import mesh as meshmod, synthetic
    from paper_2307_14837_b200.net import Architecture, MlpModel
    from paper_2307_14837_b200.step import CorrectionStep

    dims = [240, 256, 256, 256, 81]
    W = synthetic.xavier_weights(dims, 11)
    model = MlpModel(Architecture(240, 256, 3, 81), activation="tanh")
    model.W = [w.copy() for w in W]
    model.eval()
    rng = np.random.default_rng(5)
    outs = []
    for mode in ("ascending", "forward", ""):
        monkeypatch.setenv("DNNMG_NODE_ORDER", mode)
        h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1),
                                        n_cells=(6, 4, 3))
        meshmod.refine_uniform(h)
        step = CorrectionStep(h, 0, 1, model, 1e-3, 0.01, precision="f16x3", t=0.01)
        if not outs:
            nL = h.scalar_nodes(0)[0].shape[0]
            nf = h.scalar_nodes(1)[0].shape[0]
            x = torch.tensor(rng.standard_normal(4 * nL), dtype=torch.float32, device="cuda")
            b = torch.tensor(1e-3 * rng.standard_normal(4 * nf), dtype=torch.float32,
                             device="cuda")
        out = step(x, b)
        torch.cuda.synchronize()
        outs.append((out.clone(), step.d.clone()))
    for o, d in outs[1:]:
        assert torch.equal(o, outs[0][0]) and torch.equal(d, outs[0][1])
