"""Seeded synthetic inputs for the correction-step workloads.

The reference measures on the 3-D channel benchmark whose meshes and dataset are
not available here; these seeded fields stand in for the coarse Newton-MG output
with the shapes, sizes and value scales of BASELINE.json's configs:

* coarse velocity: divergence-free random Fourier field
  v(x,t) = sum_k [A_k cos(2 pi k.x) + B_k sin(2 pi k.x)] exp(-nu (2 pi |k|)^2 t),
  k in {0..7}^3 \\ {0}, A_k, B_k ~ N(0,1)/|k|^2 projected onto k-perp;
* pressure: N(0, 0.1^2) per node, redrawn per step;
* interior level-0 vertices jittered by U(+-0.1 h0) (config 1/2);
* weights: Xavier-uniform U(+-sqrt(6/(fan_in+fan_out))) per layer.

Everything is generated in float64 with numpy and rounded to float32 so that the
GPU path and the CPU oracle see identical values.
"""

import numpy as np

N_MODES_1D = 8


def fourier_modes(seed):
    """(K (511,3) int, A (511,3), B (511,3)) for seed; lexicographic k, kx slowest."""
    rng = np.random.default_rng(seed)
    g = np.arange(N_MODES_1D)
    K = np.stack(np.meshgrid(g, g, g, indexing="ij"), axis=-1).reshape(-1, 3)[1:]
    k2 = (K.astype(float) ** 2).sum(1)
    khat = K / np.sqrt(k2)[:, None]
    A = rng.standard_normal((K.shape[0], 3)) / k2[:, None]
    B = rng.standard_normal((K.shape[0], 3)) / k2[:, None]
    A -= (A * khat).sum(1, keepdims=True) * khat
    B -= (B * khat).sum(1, keepdims=True) * khat
    return K, A, B


def fourier_velocity(points, modes, t, nu, chunk=1 << 14):
    """Evaluate the Fourier velocity field at points (n,3) and time t -> (n,3) f64."""
    K, A, B = modes
    kk = 2.0 * np.pi * K.astype(float)
    decay = np.exp(-nu * (kk ** 2).sum(1) * t)
    Ad = A * decay[:, None]
    Bd = B * decay[:, None]
    pts = np.asarray(points, dtype=float)
    out = np.empty((pts.shape[0], 3))
    for s in range(0, pts.shape[0], chunk):
        ph = pts[s:s + chunk] @ kk.T
        out[s:s + chunk] = np.cos(ph) @ Ad + np.sin(ph) @ Bd
    return out


def coarse_state(points, modes, seed, step, t, nu):
    """Node-major (p, vx, vy, vz) coarse dof vector, fp32-rounded, returned as f64."""
    n = points.shape[0]
    x = np.empty((n, 4))
    x[:, 1:] = fourier_velocity(points, modes, t, nu)
    x[:, 0] = np.random.default_rng(seed + 1000 + step).normal(0.0, 0.1, n)
    return x.reshape(-1).astype(np.float32).astype(np.float64)


def jitter_vertices(vertices, n_cells, extent_lo, extent_hi, seed, amp=0.1):
    """Jitter interior vertices of a level-0 box in place (vertex-id order)."""
    lo = np.asarray(extent_lo, dtype=float)
    hi = np.asarray(extent_hi, dtype=float)
    h0 = (hi - lo) / np.asarray(n_cells, dtype=float)
    tol = 1e-9 * max(float(np.max(hi - lo)), 1.0)
    interior = np.all((vertices > lo + tol) & (vertices < hi - tol), axis=1)
    idx = np.nonzero(interior)[0]
    rng = np.random.default_rng(seed)
    vertices[idx] += rng.uniform(-amp, amp, (idx.size, 3)) * h0
    return vertices


def xavier_weights(dims, seed, dtype=np.float32):
    """Xavier-uniform matrices (dims[i], dims[i+1]), rounded to dtype, returned f64."""
    rng = np.random.default_rng(seed)
    out = []
    for fi, fo in zip(dims[:-1], dims[1:]):
        lim = np.sqrt(6.0 / (fi + fo))
        out.append(rng.uniform(-lim, lim, (fi, fo)).astype(dtype).astype(np.float64))
    return out


# BASELINE.json configs under the SURVEY.md §0.1 mapping
CONFIGS = {
    "cfg0": dict(n_cells=(4, 2, 2), J=1, jitter=False, hidden=256, depth=3,
                 steps=1, dt=0.01, nu=1e-3, seed=100),
    "cfg1": dict(n_cells=(16, 8, 8), J=1, jitter=True, hidden=256, depth=3,
                 steps=10, dt=0.005, nu=1e-3, seed=101),
    "cfg2": dict(n_cells=(32, 16, 16), J=2, jitter=True, hidden=512, depth=3,
                 steps=5, dt=0.005, nu=1e-3, seed=102),
    "cfg3": dict(n_cells=(64, 32, 32), J=1, jitter=False, hidden=256, depth=3,
                 steps=10, dt=0.005, nu=1e-3, seed=103),
}
