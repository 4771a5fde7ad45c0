"""Patch network: architecture, eval-mode state and the GPU forward (drop-in for
the reference ``dnnmg.net`` on the correction path, net.py:27-164).

    f_1(x) = act(BN_1(W_1 x)),  f_i(x) = act(BN_i(W_i x)) + x,  f_L(x) = W_L x

with no biases and input standardisation first.  ``forward`` in eval mode runs
kernel K4 of libdnnmg_b200; training (train-mode BN, backward, AdamW) is outside
the correction step.
"""

from dataclasses import dataclass

import numpy as np

ACTIVATIONS = ("relu", "tanh")


@dataclass(frozen=True)
class Architecture:
    n_in: int
    n_hidden: int
    depth: int
    n_out: int


def param_count(arch):
    a = arch
    return (a.n_in * a.n_hidden + (a.depth - 1) * a.n_hidden ** 2 + a.n_hidden * a.n_out
            + 2 * a.depth * a.n_hidden)


class MlpModel:
    """Weights, batch-norm state and input normalisation (net.py:54-112).

    Initialisation follows the reference: He-uniform hidden weights
    U(+-sqrt(6/fan_in)), head U(+-0.01)/sqrt(H), from default_rng(seed).
    """

    def __init__(self, arch, activation="relu", seed=0, bn_eps=1e-5, bn_momentum=0.1):
        if activation not in ACTIVATIONS:
            raise ValueError(f"unknown activation '{activation}'")
        self.arch = arch
        self.activation = activation
        self.bn_eps = bn_eps
        self.bn_momentum = bn_momentum
        self.mode = "train"
        rng = np.random.default_rng(seed)
        dims = [arch.n_in] + [arch.n_hidden] * arch.depth
        self.W = [rng.uniform(-np.sqrt(6.0 / dims[i]), np.sqrt(6.0 / dims[i]), (dims[i], dims[i + 1]))
                  for i in range(arch.depth)]
        self.W.append(rng.uniform(-0.01, 0.01, (arch.n_hidden, arch.n_out)) / np.sqrt(arch.n_hidden))
        H = arch.n_hidden
        self.gamma = [np.ones(H) for _ in range(arch.depth)]
        self.beta = [np.zeros(H) for _ in range(arch.depth)]
        self.running_mean = [np.zeros(H) for _ in range(arch.depth)]
        self.running_var = [np.ones(H) for _ in range(arch.depth)]
        self.input_mean = np.zeros(arch.n_in)
        self.input_std = np.ones(arch.n_in)

    def train(self):
        self.mode = "train"
        return self

    def eval(self):
        self.mode = "eval"
        return self

    def set_input_norm(self, mean, std):
        mean = np.asarray(mean, dtype=float).copy()
        std = np.asarray(std, dtype=float).copy()
        floor = 1e-8 * np.maximum(1.0, np.abs(mean))
        std[std < floor] = 1.0
        self.input_mean = mean
        self.input_std = std

    def parameters(self):
        for i, W in enumerate(self.W):
            yield ("W", i, W)
        for i in range(self.arch.depth):
            yield ("gamma", i, self.gamma[i])
            yield ("beta", i, self.beta[i])

    def copy(self):
        import copy
        return copy.deepcopy(self)

    def n_parameters(self):
        return param_count(self.arch)


def zero_weights(model):
    for W in model.W:
        W[:] = 0.0
    return model


def resolve_precision(precision=None):
    import os
    p = precision or os.environ.get("DNNMG_B200_PRECISION", "fp32")
    if p not in ("fp32", "bf16", "tf32x3", "f16x3"):
        raise ValueError(f"unknown precision '{p}' (fp32 | bf16 | tf32x3 | f16x3)")
    return p


def forward(model, X, precision=None):
    """Eval-mode network output for a batch on the GPU (net.py:162-164)."""
    import torch
    from . import device as dv
    if model.mode != "eval":
        raise NotImplementedError("train-mode forward (batch statistics) is outside the "
                                  "correction path; call model.eval()")
    Xd = dv.f32(X)
    if Xd.dim() != 2 or Xd.shape[1] != model.arch.n_in:
        raise ValueError(f"batch width {tuple(Xd.shape)} does not match n_in={model.arch.n_in}")
    dm = dv.DeviceModel(model, resolve_precision(precision))
    Y = torch.empty((Xd.shape[0], model.arch.n_out), dtype=torch.float32, device=Xd.device)
    dm.forward(Xd, Xd.shape[0], Y)
    return dv.like_input(Y, X)
