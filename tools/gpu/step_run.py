"""Short driver for ncu captures: a few fused correction steps on a coarse box
(default 32x16x16, J=1, 65,536 patches), f16x3 MLP, synthetic inputs."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2307_14837_b200 import mesh as meshmod, synthetic
from paper_2307_14837_b200.net import Architecture, MlpModel
from paper_2307_14837_b200.step import CorrectionStep

n_cells = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "32x16x16").split("x"))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
h = meshmod.build_template_mesh("box", extent_lo=(0, 0, 0), extent_hi=(1, 1, 1), n_cells=n_cells)
meshmod.refine_uniform(h)
model = MlpModel(Architecture(240, 256, 3, 81), activation="tanh")
model.W = synthetic.xavier_weights([240, 256, 256, 256, 81], 7)
model.eval()
step = CorrectionStep(h, 0, 1, model, 1e-3, 5e-3, precision="f16x3", t=5e-3)
rng = np.random.default_rng(0)
xc = torch.tensor(rng.standard_normal(step.coarse_ndof) * 0.5, dtype=torch.float32, device="cuda")
b = torch.tensor(rng.standard_normal(4 * step.space.n_nodes) * 1e-4, dtype=torch.float32, device="cuda")
for _ in range(steps):
    out = step(xc, b)
torch.cuda.synchronize()
print("ok", step.n_patches, float(out.abs().sum()))
