"""Writes tests/golden/model_small.dnmg with the REFERENCE's own save_model (run in the
build container, where /root/reference exists) plus the arrays it holds, so that the
product's DNMG reader is pinned against a file the reference produced."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from dnnmg import net as rnet  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
arch = rnet.Architecture(40, 16, 3, 9)
m = rnet.MlpModel(arch, activation="tanh", seed=5)
rng = np.random.default_rng(9)
for i in range(arch.depth):
    m.gamma[i] = rng.uniform(0.5, 1.5, 16)
    m.beta[i] = rng.normal(0, 0.1, 16)
    m.running_mean[i] = rng.normal(0, 0.2, 16)
    m.running_var[i] = rng.uniform(0.5, 2.0, 16)
m.set_input_norm(rng.normal(0, 0.3, 40), rng.uniform(0.5, 2.0, 40))
rnet.save_model(m, os.path.join(HERE, "model_small.dnmg"))
arrays = {"input_mean": m.input_mean, "input_std": m.input_std}
for i, W in enumerate(m.W):
    arrays[f"W{i}"] = W
for i in range(arch.depth):
    arrays[f"gamma{i}"], arrays[f"beta{i}"] = m.gamma[i], m.beta[i]
    arrays[f"rmean{i}"], arrays[f"rvar{i}"] = m.running_mean[i], m.running_var[i]
np.savez_compressed(os.path.join(HERE, "model_small.npz"), **arrays)
print("wrote model_small.dnmg / model_small.npz")
