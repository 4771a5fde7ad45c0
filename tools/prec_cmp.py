"""Relative L2 error of the MLP output against the float64 oracle per precision mode
(a diagnostic script run on the GPU box: python tools/prec_cmp.py)."""
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2307_14837_b200 import net
from oracle import dnnmg_oracle as orc
for n_in, depth, act, rows in [(240, 3, "tanh", 4096), (174, 3, "tanh", 4097), (240, 4, "relu", 2000)]:
    rng = np.random.default_rng(n_in + rows)
    m = net.MlpModel(net.Architecture(n_in, 256, depth, 81), activation=act, seed=rows)
    m.eval()
    X = rng.standard_normal((rows, n_in))
    ref = orc.mlp_forward(orc.Mlp(m.W, act, m.gamma, m.beta, m.running_mean, m.running_var, m.input_mean, m.input_std), X)
    out = []
    for p in ["fp32", "tf32x3", "f16x3", "bf16", "fp8"]:
        Y = net.forward(m, X, precision=p)
        out.append(f"{p}={np.linalg.norm(Y-ref)/np.linalg.norm(ref):.2e}")
    print(n_in, depth, act, " ".join(out))
