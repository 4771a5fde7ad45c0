"""Q2 reference element on [0,1]^3 (host-side constants; elements.py:1-118).

Local node numbering is lexicographic with x fastest; the Gauss rule is the
4-point tensor rule on [0,1]^3, q = qx + 4 qy + 16 qz.  The CUDA kernels use the
same 1-D factors (csrc/residual.cu); these host versions build the
prolongation stencils and serve the API.
"""

import numpy as np

q2_nodes_1d = np.array([0.0, 0.5, 1.0])


def N_LOC(dim):
    return 3 ** dim


def lattice(dim, n=3):
    f = np.arange(n ** dim)
    return np.stack([(f // n ** k) % n for k in range(dim)], axis=1).astype(np.int64)


def _phi1d(x):
    x = np.asarray(x, dtype=float)
    return np.stack([2.0 * (x - 0.5) * (x - 1.0), 4.0 * x * (1.0 - x), 2.0 * x * (x - 0.5)], -1)


def _dphi1d(x):
    x = np.asarray(x, dtype=float)
    return np.stack([4.0 * x - 3.0, 4.0 - 8.0 * x, 4.0 * x - 1.0], -1)


def shape_q2(points, dim=3):
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    idx = lattice(dim)
    out = np.ones((pts.shape[0], idx.shape[0]))
    for k in range(dim):
        out *= _phi1d(pts[:, k])[:, idx[:, k]]
    return out


def grad_q2(points, dim=3):
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    idx = lattice(dim)
    out = np.empty((pts.shape[0], idx.shape[0], dim))
    for comp in range(dim):
        g = np.ones((pts.shape[0], idx.shape[0]))
        for k in range(dim):
            g *= (_dphi1d if k == comp else _phi1d)(pts[:, k])[:, idx[:, k]]
        out[:, :, comp] = g
    return out


def gauss_rule(dim, n=4):
    x, w = np.polynomial.legendre.leggauss(n)
    x, w = 0.5 * (x + 1.0), 0.5 * w
    idx = lattice(dim, n)
    pts = np.stack([x[idx[:, k]] for k in range(dim)], axis=1)
    wts = np.prod(np.stack([w[idx[:, k]] for k in range(dim)], axis=1), axis=1)
    return pts, wts


def q1_embedding_matrix(dim=3):
    idx = lattice(dim)
    verts = np.nonzero(np.all((idx == 0) | (idx == 2), axis=1))[0]
    coord = idx / 2.0
    PI = np.zeros((idx.shape[0], idx.shape[0]))
    for v in verts:
        xv = idx[v] / 2.0
        PI[:, v] = np.prod(xv * coord + (1.0 - xv) * (1.0 - coord), axis=1)
    return PI
