"""Equal-order Q2 spaces, Dirichlet data and the Q2 prolongation (drop-in for
the reference ``dnnmg.space``, space.py:33-255).

State vectors are node-major, component-minor: dof = 4*node + comp, comp 0 the
pressure (space.py:3-7).  ``prolongate`` and ``apply_dirichlet`` run on the GPU
through libdnnmg_b200 (kernel K1); host-side work here is only the one-time
construction of the index tables they use.
"""

from dataclasses import dataclass

import numpy as np

from . import mesh as meshmod
from .mesh import LAT2, LAT3

__all__ = ["FeSpace", "StateVector", "prolongate", "prolongation_source",
           "prolongation_matrix", "full_prolongation", "apply_dirichlet", "ramp",
           "inflow_profile", "no_slip", "benchmark_bcs", "inject", "restrict_rhs"]


def _face_nodes():
    return [np.nonzero(LAT3[:, f // 2] == 2 * (f % 2))[0] for f in range(6)]


class FeSpace:
    """Q2 scalar nodes of one level with 4 components per node (space.py:33-85).

    Accepts this package's MeshHierarchy or any object with the reference's
    ``scalar_nodes`` / ``levels[l].boundary_faces`` interface.
    """

    def __init__(self, hierarchy, level):
        self.hierarchy = hierarchy
        self.level = level
        self.dim = hierarchy.dim
        if self.dim != 3:
            raise NotImplementedError("only 3-D hexahedral spaces are supported")
        self.n_comp = 4
        coords, table = hierarchy.scalar_nodes(level)
        self.nodes = coords
        self.cell_nodes = table
        self.n_nodes = coords.shape[0]
        self.ndof = 4 * self.n_nodes
        self._tag_nodes()

    def _tag_nodes(self):
        """Per-node tag; later tags win: OUTFLOW < INFLOW < WALL < OBSTACLE (space.py:48-61)."""
        faces = np.asarray(self.hierarchy.levels[self.level].boundary_faces, dtype=np.int64)
        faces = faces.reshape(-1, 3)
        fn = np.stack(_face_nodes())                       # (6, 9)
        tags = np.zeros(self.n_nodes, dtype=np.int64)
        for t in (meshmod.OUTFLOW, meshmod.INFLOW, meshmod.WALL, meshmod.OBSTACLE):
            sel = faces[faces[:, 2] == t]
            if sel.size:
                tags[self.cell_nodes[sel[:, 0][:, None], fn[sel[:, 1]]].reshape(-1)] = t
        self.node_tags = tags
        self.has_outflow = bool(np.any(tags == meshmod.OUTFLOW))

    def nodes_with_tag(self, tag):
        return np.nonzero(self.node_tags == tag)[0]

    def velocity_dofs(self, nodes):
        return (4 * np.asarray(nodes)[:, None] + np.arange(1, 4)[None, :]).reshape(-1)

    def dirichlet_mask(self, tags=(meshmod.INFLOW, meshmod.WALL, meshmod.OBSTACLE)):
        mask = np.zeros(self.ndof, dtype=bool)
        for t in tags:
            nodes = self.nodes_with_tag(t)
            if nodes.size:
                mask[self.velocity_dofs(nodes)] = True
        return mask

    def zero_state(self, time=0.0):
        return StateVector(self.level, np.zeros(self.ndof), time)

    def split(self, values):
        m = values.reshape(self.n_nodes, self.n_comp)
        return m[:, 0], m[:, 1:]


@dataclass
class StateVector:
    level: int
    values: object          # numpy float64 (reference-compatible) or torch CUDA float32
    time: float = 0.0

    def copy(self):
        return StateVector(self.level, self.values.copy() if isinstance(self.values, np.ndarray)
                           else self.values.clone(), self.time)


# -- transfer tables ---------------------------------------------------------------

def _stencils():
    """Coarse Q2 shape values at the child-local nodes of each octant:
    (8, 27 child-local, 27 coarse) (space.py:136-141)."""
    from .elements import shape_q2
    return np.stack([shape_q2((LAT2[o][None, :] + LAT3 / 2.0) / 2.0) for o in range(8)])


def prolongation_source(hierarchy, level):
    """For every scalar node of level+1: the first (octant, child-local node,
    parent cell) reaching it, packed as C*216 + o*27 + a (space.py:142-159)."""
    cache = hierarchy.__dict__.setdefault("_b200_prolong_src", {})
    if level not in cache:
        _, ctab = hierarchy.scalar_nodes(level)
        fcoords, ftab = hierarchy.scalar_nodes(level + 1)
        nc = ctab.shape[0]
        nodes = ftab.reshape(nc, 8, 27).transpose(1, 2, 0).reshape(-1)     # order (o, a, C)
        uniq, first = np.unique(nodes, return_index=True)
        if uniq.size != fcoords.shape[0]:
            raise RuntimeError("prolongation: fine nodes not reached by any parent")
        o = first // (27 * nc)
        a = (first // nc) % 27
        C = first % nc
        src = np.empty(fcoords.shape[0], dtype=np.int64)
        src[uniq] = C * 216 + o * 27 + a
        cache[level] = src
    return cache[level]


def prolongation_matrix(hierarchy, level):
    """Scalar prolongation level -> level+1 as scipy CSR (space.py:117-165)."""
    import scipy.sparse as sp
    cache = hierarchy.__dict__.setdefault("_b200_prolong_csr", {})
    if level not in cache:
        src = prolongation_source(hierarchy, level)
        _, ctab = hierarchy.scalar_nodes(level)
        sten = _stencils().reshape(216, 27)
        C, oa = src // 216, src % 216
        W = sten[oa]                                   # (nf, 27)
        cols = ctab[C]                                 # (nf, 27)
        nzr, nzc = np.nonzero(np.abs(W) > 1e-14)
        P = sp.csr_matrix((W[nzr, nzc], (nzr, cols[nzr, nzc])),
                          shape=(src.size, hierarchy.scalar_nodes(level)[0].shape[0]))
        P.sum_duplicates()
        cache[level] = P
    return cache[level]


def full_prolongation(hierarchy, level, n_comp=4):
    import scipy.sparse as sp
    return sp.kron(prolongation_matrix(hierarchy, level), sp.identity(n_comp, format="csr"),
                   format="csr")


def prolongate(hierarchy, x, levels_up=1):
    """Embed a state levels_up levels finer on the GPU (space.py:177-185)."""
    from . import device
    return device.prolongate_state(hierarchy, x, levels_up)


def inject(space_coarse, x_fine):
    """Pointwise restriction: coarse nodes lead the numbering (space.py:199-202)."""
    return StateVector(space_coarse.level, x_fine.values[:space_coarse.ndof].copy(), x_fine.time)


def restrict_rhs(hierarchy, b, level_fine, levels_down=1):
    """P^T restriction of a dual vector on the GPU (space.py:188-196, Alg. 1 line 9)."""
    from . import device
    return device.restrict_vector(hierarchy, b, level_fine, levels_down)


# -- Dirichlet data ---------------------------------------------------------------------

def ramp(t):
    return 0.5 - 0.5 * np.cos(5 * np.pi * t) if t <= 0.2 else 1.0


def inflow_profile(dim, vbar, H):
    """Parabolic inflow with smooth startup (space.py:212-231)."""
    if dim != 3:
        raise NotImplementedError("only the 3-D profile is supported")

    def profile(t, pts):
        y, z = pts[:, 1], pts[:, 2]
        out = np.zeros((pts.shape[0], 3))
        out[:, 0] = ramp(t) * 1.125 * vbar * y * (H - y) * (H ** 2 - z ** 2) / ((H / 2) ** 2 * H ** 2)
        return out
    return profile


def no_slip(t, pts):
    return np.zeros((pts.shape[0], pts.shape[1]))


def benchmark_bcs(dim, vbar, H):
    return {meshmod.INFLOW: inflow_profile(dim, vbar, H), meshmod.WALL: no_slip,
            meshmod.OBSTACLE: no_slip}


def apply_dirichlet(space, x, t, bcs):
    """Impose the tagged velocity boundary values at time t, in place (space.py:245-255)."""
    from . import device
    device.apply_dirichlet_state(space, x, t, bcs)
    x.time = t
    return x
