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
    if p not in ("fp32", "bf16", "tf32x3", "f16x3", "fp8"):
        raise ValueError(f"unknown precision '{p}' (fp32 | bf16 | tf32x3 | f16x3 | fp8)")
    return p


def effective_precision(activation, precision):
    """The tensor-core mode a model actually runs in.  f16x3 splits the hidden activations
    into fp16 hi/lo parts, which is exact to fp32 accuracy only while |h| < 65504: tanh
    bounds the hidden states (|h| <= depth with the skips), relu -- the reference's default
    activation (net.py:57, config.py:69-71) -- does not.  Relu models therefore run in
    tf32x3 (same fp32 accuracy, fp32 exponent range, half the f16x3 rate); the library
    rejects f16x3 + relu outright (DNNMG_ERR_UNSUPPORTED)."""
    if precision == "f16x3" and activation != "tanh":
        return "tf32x3"
    return precision


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


# -- "DNMG" model file (net.py:337-392): trained weights for the correction path ----------
#
# Little-endian layout: b"DNMG", u32 version (= 1), u32 n_in, n_hidden, depth, n_out,
# u32 len(activation), the activation name, f64 bn_eps, f64 bn_momentum, then float64
# arrays: input_mean[n_in], input_std[n_in], W_0..W_depth (row-major, fan_in x fan_out),
# and per hidden layer gamma, beta, running_mean, running_var [n_hidden].

_DNMG_MAGIC = b"DNMG"
_DNMG_VERSION = 1


def _dnmg_shapes(arch):
    dims = [arch.n_in] + [arch.n_hidden] * arch.depth + [arch.n_out]
    shapes = [("input_mean", None, (arch.n_in,)), ("input_std", None, (arch.n_in,))]
    shapes += [("W", i, (dims[i], dims[i + 1])) for i in range(arch.depth + 1)]
    for i in range(arch.depth):
        shapes += [(name, i, (arch.n_hidden,)) for name in ("gamma", "beta", "running_mean",
                                                            "running_var")]
    return shapes


def load_model(path):
    """Read a DNMG model file into an eval-mode MlpModel."""
    raw = open(path, "rb").read()
    if raw[:4] != _DNMG_MAGIC:
        raise ValueError(f"not a model file: bad magic {raw[:4]!r}")
    head = np.frombuffer(raw, dtype="<u4", count=6, offset=4)
    if int(head[0]) != _DNMG_VERSION:
        raise ValueError(f"unsupported model file version {int(head[0])}")
    n_in, n_hidden, depth, n_out, tag_len = (int(v) for v in head[1:])
    off = 28
    activation = raw[off:off + tag_len].decode()
    off += tag_len
    bn_eps, bn_momentum = (float(v) for v in np.frombuffer(raw, dtype="<f8", count=2, offset=off))
    off += 16
    arch = Architecture(n_in, n_hidden, depth, n_out)
    model = MlpModel(arch, activation=activation, bn_eps=bn_eps, bn_momentum=bn_momentum)
    for name, i, shape in _dnmg_shapes(arch):
        n = int(np.prod(shape))
        if off + 8 * n > len(raw):
            raise ValueError("model file truncated")
        arr = np.frombuffer(raw, dtype="<f8", count=n, offset=off).reshape(shape).astype(np.float64)
        off += 8 * n
        if i is None:
            setattr(model, name, arr)
        else:
            getattr(model, name)[i] = arr
    return model.eval()


def save_model(model, path):
    """Write a DNMG model file (the reference's format, readable by its load_model)."""
    a = model.arch
    tag = model.activation.encode()
    parts = [_DNMG_MAGIC,
             np.array([_DNMG_VERSION, a.n_in, a.n_hidden, a.depth, a.n_out, len(tag)],
                      dtype="<u4").tobytes(),
             tag, np.array([model.bn_eps, model.bn_momentum], dtype="<f8").tobytes()]
    for name, i, shape in _dnmg_shapes(a):
        arr = getattr(model, name) if i is None else getattr(model, name)[i]
        arr = np.asarray(arr, dtype="<f8")
        if arr.shape != shape:
            raise ValueError(f"{name}[{i}] has shape {arr.shape}, expected {shape}")
        parts.append(np.ascontiguousarray(arr).tobytes())
    with open(path, "wb") as f:
        f.write(b"".join(parts))
