"""Hexahedral box hierarchies, Q2 node numbering, patches and geometry features.

Drop-in mirror of the reference ``dnnmg.mesh`` API for the correction path
(mesh.py:60-246, 452-611): ``build_template_mesh("box", ...)``,
``refine_uniform``, ``MeshHierarchy.scalar_nodes``, ``build_patches`` /
``PatchSet`` and ``geometry_features_of_cells``.  The numbering is bit-exact
with the reference (tests/test_mesh_maps.py checks it against the oracle, which
is pinned by the reference's own output), but computed without per-node Python
loops: every level carries the integer lattice position of its vertices, so a
Q2 node is identified by its position on the doubled lattice, and "first
appearance in (cell, local node) order" becomes one ``np.unique`` over the
flattened (cell, node) keys.  Config 3 (524,288 fine cells) numbers in seconds
instead of the reference's ~5 minutes.

Only the box template is implemented; the channel/obstacle templates are out
of scope for the correction step.
"""

import numpy as np

INFLOW, OUTFLOW, WALL, OBSTACLE = 1, 2, 3, 4
TAG_NAMES = {INFLOW: "inflow", OUTFLOW: "outflow", WALL: "wall", OBSTACLE: "obstacle"}

FACES_3D = ((0, 2, 4, 6), (1, 3, 5, 7), (0, 1, 4, 5), (2, 3, 6, 7), (0, 1, 2, 3), (4, 5, 6, 7))
EDGES_3D = ((0, 1), (2, 3), (4, 5), (6, 7), (0, 2), (1, 3), (4, 6), (5, 7),
            (0, 4), (1, 5), (2, 6), (3, 7))
DIAGONALS_3D = ((0, 7), (1, 6), (2, 5), (3, 4))

LAT3 = np.stack([np.arange(27) % 3, (np.arange(27) // 3) % 3, np.arange(27) // 9], axis=1)
LAT2 = np.stack([np.arange(8) % 2, (np.arange(8) // 2) % 2, np.arange(8) // 4], axis=1)
VERTEX_LOCAL = np.array([0, 2, 6, 8, 18, 20, 24, 26])        # corner k <-> local Q2 node
NONVERTEX_LOCAL = np.array([a for a in range(27) if a not in set(VERTEX_LOCAL.tolist())])


def _parent_corners(a):
    """Local corner numbers whose mean defines local Q2 node a, in the
    reference's enumeration (free axes, first free axis fastest; mesh.py:192-198)."""
    free = np.nonzero(LAT3[a] == 1)[0]
    out = []
    for m in range(2 ** free.size):
        p = LAT3[a].copy()
        for t, axis in enumerate(free):
            p[axis] = 2 * ((m >> t) & 1)
        out.append(int(p[0] // 2 + 2 * (p[1] // 2) + 4 * (p[2] // 2)))
    return out


PARENTS = [_parent_corners(a) for a in range(27)]


class MeshLevel:
    """Vertices, 8-corner cells (tensor order, x fastest) and refinement parent."""

    def __init__(self, dim, vertices, cells, parent_of=None, lattice=None):
        self.dim = dim
        self.vertices = np.asarray(vertices, dtype=float)
        self.cells = np.asarray(cells, dtype=np.int64)
        self.parent_of = parent_of
        self.lattice = lattice            # (n_vertices, 3) integer grid positions
        self._boundary_faces = None
        self._extent = None      # (global grid size at this level, channel tags)
        self._offset = 0         # lattice offset of this (sub-)box inside the global box

    @property
    def n_cells(self):
        return self.cells.shape[0]

    @property
    def n_vertices(self):
        return self.vertices.shape[0]

    @property
    def boundary_faces(self):
        """(cell, local face, tag) rows sorted by (cell, face) (mesh.py:118-151)."""
        if self._boundary_faces is None:
            self._boundary_faces = _box_boundary_faces(self)
        return self._boundary_faces

    @boundary_faces.setter
    def boundary_faces(self, value):
        self._boundary_faces = value

    def cell_volumes(self):
        """Volumes of the trilinear cells by 2-point Gauss (mesh.py:76-93)."""
        x, w = np.polynomial.legendre.leggauss(2)
        x, w = 0.5 * (x + 1.0), 0.5 * w
        pts = x[LAT2]
        wts = w[LAT2[:, 0]] * w[LAT2[:, 1]] * w[LAT2[:, 2]]
        ders = np.ones((8, 8, 3))
        for comp in range(3):
            for k in range(3):
                xk = LAT2[:, k][None, :]
                if k == comp:
                    ders[:, :, comp] *= 2 * xk - 1.0
                else:
                    ders[:, :, comp] *= xk * pts[:, k][:, None] + (1 - xk) * (1 - pts[:, k][:, None])
        X = self.vertices[self.cells]
        J = np.einsum('qaj,cai->cqij', ders, X)
        return np.linalg.det(J) @ wts


def _box_boundary_faces(lvl):
    ext, channel = lvl._extent
    base = lvl.lattice[lvl.cells[:, 0]] + lvl._offset
    rows = []
    for f in range(6):
        axis, side = f // 2, f % 2
        on = (base[:, axis] == 0) if side == 0 else (base[:, axis] + 1 == ext[axis])
        cells = np.nonzero(on)[0]
        tag = WALL
        if channel and axis == 0:
            tag = INFLOW if side == 0 else OUTFLOW
        rows.append(np.stack([cells, np.full(cells.size, f), np.full(cells.size, tag)], axis=1))
    faces = np.concatenate(rows, axis=0)
    order = np.lexsort((faces[:, 1], faces[:, 0]))
    return faces[order]


class MeshHierarchy:
    """Nested box levels 0..top (mesh.py:96-220)."""

    def __init__(self, level0, extent_lo, extent_hi, obstacles=(), channel_tags=True):
        self.dim = level0.dim
        self.levels = [level0]
        self.extent_lo = np.asarray(extent_lo, dtype=float)
        self.extent_hi = np.asarray(extent_hi, dtype=float)
        self.obstacles = list(obstacles)
        self.channel_tags = channel_tags
        self._node_cache = {}
        self._grid = np.asarray(level0.lattice.max(axis=0))
        if level0._extent is None:
            level0._extent = (self._grid, channel_tags)
        self._check_orientation(level0)

    def _check_orientation(self, lvl):
        vols = lvl.cell_volumes()
        if np.any(vols <= 0):
            bad = int(np.argmin(vols))
            raise ValueError(f"cell {bad} has non-positive Jacobian (volume {vols[bad]:.3e})")

    @property
    def top(self):
        return len(self.levels) - 1

    def scalar_nodes(self, level):
        """(coords (n, 3), cell_nodes (nc, 27)) of level (mesh.py:162-216)."""
        if level in self._node_cache:
            return self._node_cache[level][:2]
        lvl = self.levels[level]
        C = lvl.cells
        nc, nv = C.shape[0], lvl.n_vertices
        base = lvl.lattice[C[:, 0]]
        ext = 2 * lvl.lattice.max(axis=0) + 1
        table = np.empty((nc, 27), dtype=np.int64)
        table[:, VERTEX_LOCAL] = C
        pos = 2 * base[:, None, :] + LAT3[NONVERTEX_LOCAL][None, :, :]     # (nc, 19, 3)
        keys = (pos[..., 0] + ext[0] * (pos[..., 1] + ext[1] * pos[..., 2])).reshape(-1)
        uniq, first, inv = np.unique(keys, return_index=True, return_inverse=True)
        order = np.argsort(first, kind="stable")
        rank = np.empty(order.size, dtype=np.int64)
        rank[order] = np.arange(order.size)
        table[:, NONVERTEX_LOCAL] = (nv + rank[inv]).reshape(nc, NONVERTEX_LOCAL.size)
        # coordinates: mean of the parent corners of the first-appearance cell
        f_sorted = first[order]
        c_of = f_sorted // NONVERTEX_LOCAL.size
        a_of = NONVERTEX_LOCAL[f_sorted % NONVERTEX_LOCAL.size]
        new_xyz = np.empty((order.size, 3))
        new_lat = np.empty((order.size, 3), dtype=np.int64)
        V = lvl.vertices
        for a in NONVERTEX_LOCAL:
            sel = np.nonzero(a_of == a)[0]
            if sel.size == 0:
                continue
            par = C[c_of[sel]][:, PARENTS[a]]
            acc = V[par[:, 0]].copy()
            for j in range(1, par.shape[1]):
                acc = acc + V[par[:, j]]
            new_xyz[sel] = acc / par.shape[1]
            new_lat[sel] = 2 * base[c_of[sel]] + LAT3[a]
        coords = np.concatenate([V, new_xyz], axis=0)
        lattice = np.concatenate([2 * lvl.lattice, new_lat], axis=0)
        self._node_cache[level] = (coords, table, lattice)
        return coords, table


def refine_uniform(h):
    """Append one uniformly refined level (mesh.py:223-246)."""
    lvl = h.levels[-1]
    level = len(h.levels) - 1
    coords, table = h.scalar_nodes(level)
    lattice = h._node_cache[level][2]
    nc = lvl.n_cells
    cells = np.empty((8 * nc, 8), dtype=np.int64)
    lat3 = {tuple(v): a for a, v in enumerate(LAT3)}
    for o in range(8):
        cols = [lat3[tuple(LAT2[o] + d)] for d in LAT2]
        cells[o::8] = table[:, cols]
    parent = np.repeat(np.arange(nc), 8)
    new = MeshLevel(3, coords, cells, parent_of=parent, lattice=lattice)
    new._extent = (2 * lvl._extent[0], h.channel_tags)
    new._offset = 2 * lvl._offset
    h._check_orientation(new)
    h.levels.append(new)
    return h


def build_template_mesh(geometry, **params):
    """Level-0 mesh of a template (mesh.py:452-487); only "box" is supported."""
    if geometry != "box":
        raise NotImplementedError(f"template '{geometry}' is outside the correction-step scope")
    lo = np.asarray(params.get("extent_lo", (0.0, 0.0, 0.0)), dtype=float)
    hi = np.asarray(params.get("extent_hi", (1.0, 1.0, 1.0)), dtype=float)
    if lo.size != 3:
        raise NotImplementedError("only 3-D boxes are supported")
    n = [int(v) for v in params.get("n_cells", (1, 1, 1))]
    axes = [np.linspace(lo[k], hi[k], n[k] + 1) for k in range(3)]
    nx, ny, nz = n[0] + 1, n[1] + 1, n[2] + 1
    kk, jj, ii = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    lattice = np.stack([ii.ravel(), jj.ravel(), kk.ravel()], axis=1).astype(np.int64)
    verts = np.stack([axes[0][lattice[:, 0]], axes[1][lattice[:, 1]], axes[2][lattice[:, 2]]], axis=1)
    # cells ordered (k, i, j), j fastest; corners in tensor order (mesh.py:343-350, 394-398)
    k, i, j = np.meshgrid(np.arange(n[2]), np.arange(n[0]), np.arange(n[1]), indexing="ij")
    k, i, j = k.ravel(), i.ravel(), j.ravel()
    v0 = i + nx * (j + ny * k)
    bot = np.stack([v0, v0 + 1, v0 + nx, v0 + nx + 1], axis=1)
    cells = np.concatenate([bot, bot + nx * ny], axis=1)
    lvl = MeshLevel(3, verts, cells, lattice=lattice)
    return MeshHierarchy(lvl, lo, hi, (), params.get("channel_tags", False))


def build_subbox(vertices_global, n_cells_global, x_range, lo, hi, channel_tags=False):
    """Level-0 hierarchy of the x-slab [x_range[0], x_range[1]) of a global box whose
    (possibly jittered) level-0 vertices are `vertices_global` (x-fastest order).
    Boundary tags are those of the GLOBAL box: slab-interface faces are interior."""
    n = [int(v) for v in n_cells_global]
    a, b = int(x_range[0]), int(x_range[1])
    nxg = n[0] + 1
    nx, ny, nz = b - a + 1, n[1] + 1, n[2] + 1
    kk, jj, ii = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    lattice = np.stack([ii.ravel(), jj.ravel(), kk.ravel()], axis=1).astype(np.int64)
    gid = (lattice[:, 0] + a) + nxg * (lattice[:, 1] + ny * lattice[:, 2])
    verts = np.asarray(vertices_global, dtype=float)[gid]
    k, i, j = np.meshgrid(np.arange(n[2]), np.arange(b - a), np.arange(n[1]), indexing="ij")
    k, i, j = k.ravel(), i.ravel(), j.ravel()
    v0 = i + nx * (j + ny * k)
    bot = np.stack([v0, v0 + 1, v0 + nx, v0 + nx + 1], axis=1)
    cells = np.concatenate([bot, bot + nx * ny], axis=1)
    lvl = MeshLevel(3, verts, cells, lattice=lattice)
    lvl._extent = (np.asarray(n, dtype=np.int64), channel_tags)
    lvl._offset = np.array([a, 0, 0], dtype=np.int64)
    return MeshHierarchy(lvl, lo, hi, (), channel_tags)


# -- patches -------------------------------------------------------------------

class Patch:
    """One patch view (mesh.py:492-498)."""

    def __init__(self, coarse_cell, fine_cells, local_to_global, scalar_nodes, geometry):
        self.coarse_cell = coarse_cell
        self.fine_cells = fine_cells
        self.local_to_global = local_to_global
        self.scalar_nodes = scalar_nodes
        self.geometry = geometry


class PatchSet:
    """All patches of an (L, J) split plus the valence scaling (mesh.py:501-564)."""

    def __init__(self, hierarchy, L, J):
        if J not in (1, 2):
            raise ValueError(f"unsupported patch depth J={J}; need 1 or 2")
        if L + J > hierarchy.top:
            raise ValueError("mesh hierarchy lacks the fine level L+J")
        self.hierarchy = hierarchy
        self.L, self.J = L, J
        self.dim = 3
        self.ncomp = 4
        width = 3 if J == 1 else 5
        self.nodes_per_patch = width ** 3
        self.ndof_patch = 4 * self.nodes_per_patch
        coarse = hierarchy.levels[L]
        fcoords, ftab = hierarchy.scalar_nodes(L + J)
        n_patch = coarse.n_cells * 8
        if J == 1:
            node_table = np.ascontiguousarray(ftab[:n_patch])
        else:
            # grid position 2*g + a (g grandchild octant, a local node), flattened x fastest
            g_of = np.empty(125, dtype=np.int64)
            a_of = np.empty(125, dtype=np.int64)
            for g in range(8):
                for a in range(27):
                    p = 2 * LAT2[g] + LAT3[a]
                    s = p[0] + 5 * (p[1] + 5 * p[2])
                    g_of[s], a_of[s] = g, a
            rows = 8 * np.arange(n_patch)[:, None] + g_of[None, :]
            node_table = ftab[rows, a_of[None, :]]
        self.node_table = node_table
        self.dof_table = (4 * node_table[:, :, None] + np.arange(4)).reshape(n_patch, -1)
        n_fine = 4 * fcoords.shape[0]
        counts = np.bincount(self.dof_table.reshape(-1), minlength=n_fine)
        if np.any(counts == 0):
            raise RuntimeError("patch union does not cover the fine level")
        self.valence = counts
        self.mu = 1.0 / counts
        geo = geometry_features_of_cells(coarse, np.arange(coarse.n_cells))
        self.geom_table = np.repeat(geo, 8, axis=0)
        self.n_geo = self.geom_table.shape[1]
        self._patches = None

    def __len__(self):
        return self.node_table.shape[0]

    @property
    def patches(self):
        if self._patches is None:
            J = self.J
            self._patches = [
                Patch(p // 8, np.array([p]) if J == 1 else 8 * p + np.arange(8),
                      self.dof_table[p], self.node_table[p], self.geom_table[p])
                for p in range(len(self))]
        return self._patches

    def __iter__(self):
        return iter(self.patches)


def build_patches(hierarchy, L, J):
    return PatchSet(hierarchy, L, J)


def _angles_at_vertices(X):
    out = np.empty((X.shape[0], 8))
    incident = [[] for _ in range(8)]
    for (a, b) in EDGES_3D:
        incident[a].append((a, b))
        incident[b].append((b, a))
    for v in range(8):
        vecs = [X[:, b] - X[:, a] for (a, b) in incident[v]]
        angs = []
        for i in range(len(vecs)):
            for j in range(i + 1, len(vecs)):
                num = np.sum(vecs[i] * vecs[j], axis=1)
                den = np.linalg.norm(vecs[i], axis=1) * np.linalg.norm(vecs[j], axis=1)
                angs.append(np.arccos(np.clip(num / den, -1.0, 1.0)))
        out[:, v] = np.mean(angs, axis=0)
    return out


def geometry_features_of_cells(level, cell_ids):
    """12 edge lengths, 4 diagonals, 8 mean vertex angles per cell (mesh.py:594-611)."""
    X = level.vertices[level.cells[cell_ids]]
    el = np.stack([np.linalg.norm(X[:, b] - X[:, a], axis=1) for (a, b) in EDGES_3D], axis=1)
    if np.any(el <= 0):
        raise ValueError("degenerate cell: zero-length edge")
    dl = np.stack([np.linalg.norm(X[:, b] - X[:, a], axis=1) for (a, b) in DIAGONALS_3D], axis=1)
    return np.concatenate([el, dl, _angles_at_vertices(X)], axis=1)


def n_geo(dim):
    return 10 if dim == 2 else 24
