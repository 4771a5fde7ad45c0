"""CPU ORACLE for the DNN-MG fine-level correction step — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The product path (``paper_2307_14837_b200``)
never imports anything under ``oracle/`` and fails loudly when its CUDA library
is missing.

It is a float64 numpy restatement of the reference package ``dnnmg``
(arXiv 2307.14837, ``/root/reference/pkg/src/dnnmg``) for exactly the hot path
``driver.TimeLoop._step_hybrid`` lines 251-268: prolongation, Dirichlet
re-imposition, stabilisation weights, residual assembly, patch gather, patch
MLP (eval mode) and the valence-averaging scatter, plus the index maps they
rely on (box template numbering, Q2 node numbering, refinement, PatchSet) and
the next-step RHS (assembly.py:242-259).  Every function cites the reference
lines it restates.

Pinning: ``tests/golden/*.npz`` were produced by running the reference itself
(``tests/golden/make_golden.py``, in the build container where
``/root/reference`` is importable); ``tests/test_oracle_golden.py`` checks this
restatement against them (index maps bit-exact, floats to ~1e-12).
"""

import numpy as np

# boundary tags (mesh.py:19)
INFLOW, OUTFLOW, WALL, OBSTACLE = 1, 2, 3, 4

# local cell corner / face / edge conventions, tensor order x fastest (mesh.py:26-34)
CORNER_FACES = ((0, 2, 4, 6), (1, 3, 5, 7), (0, 1, 4, 5), (2, 3, 6, 7), (0, 1, 2, 3), (4, 5, 6, 7))
CELL_EDGES = ((0, 1), (2, 3), (4, 5), (6, 7), (0, 2), (1, 3), (4, 6), (5, 7),
              (0, 4), (1, 5), (2, 6), (3, 7))
CELL_DIAGS = ((0, 7), (1, 6), (2, 5), (3, 4))


# ----------------------------------------------------------------------------
# reference element (elements.py)
# ----------------------------------------------------------------------------

def multi_index(n):
    """(n^3, 3) lattice indices, x fastest (elements.py:25-31)."""
    f = np.arange(n ** 3)
    return np.stack([f % n, (f // n) % n, f // (n * n)], axis=1)


def basis_1d(x):
    """Q2 basis on nodes {0, 1/2, 1} (elements.py:34-39)."""
    x = np.asarray(x, dtype=float)
    return np.stack([2.0 * (x - 0.5) * (x - 1.0), 4.0 * x * (1.0 - x), 2.0 * x * (x - 0.5)], -1)


def dbasis_1d(x):
    """Derivatives of basis_1d (elements.py:42-46)."""
    x = np.asarray(x, dtype=float)
    return np.stack([4.0 * x - 3.0, 4.0 - 8.0 * x, 4.0 * x - 1.0], -1)


def q2_shape(pts):
    """Q2 shape values (npts, 27) (elements.py:49-60)."""
    pts = np.atleast_2d(np.asarray(pts, dtype=float))
    ix = multi_index(3)
    out = np.ones((pts.shape[0], 27))
    for k in range(3):
        out *= basis_1d(pts[:, k])[:, ix[:, k]]
    return out


def q2_grad(pts):
    """Q2 reference gradients (npts, 27, 3) (elements.py:63-76)."""
    pts = np.atleast_2d(np.asarray(pts, dtype=float))
    ix = multi_index(3)
    v = [basis_1d(pts[:, k])[:, ix[:, k]] for k in range(3)]
    d = [dbasis_1d(pts[:, k])[:, ix[:, k]] for k in range(3)]
    out = np.empty((pts.shape[0], 27, 3))
    for c in range(3):
        g = np.ones((pts.shape[0], 27))
        for k in range(3):
            g = g * (d[k] if k == c else v[k])
        out[:, :, c] = g
    return out


def gauss_points(n=4):
    """Tensor Gauss-Legendre rule on [0,1]^3 (elements.py:79-93)."""
    x, w = np.polynomial.legendre.leggauss(n)
    x, w = 0.5 * (x + 1.0), 0.5 * w
    ix = multi_index(n)
    return x[ix], w[ix[:, 0]] * w[ix[:, 1]] * w[ix[:, 2]]


def q1_projector():
    """Q2 -> Q1 nodal interpolation matrix PI (27, 27) (elements.py:96-118)."""
    ix = multi_index(3)
    corner = np.all((ix == 0) | (ix == 2), axis=1)
    PI = np.zeros((27, 27))
    for b in range(27):
        pos = ix[b] / 2.0
        for v in np.nonzero(corner)[0]:
            s = ix[v] / 2.0
            PI[b, v] = np.prod(s * pos + (1.0 - s) * (1.0 - pos))
    return PI


# ----------------------------------------------------------------------------
# meshes (mesh.py)
# ----------------------------------------------------------------------------

class Level:
    """One mesh level: vertex coordinates and 8-corner cells (mesh.py:60-74)."""

    def __init__(self, verts, cells):
        self.verts = np.asarray(verts, dtype=float)
        self.cells = np.asarray(cells, dtype=np.int64)


def box_level0(lo, hi, n_cells):
    """Level-0 box: vertices x-fastest, cells ordered (k, i, j) with j fastest
    (mesh.py:300-305, 319-325, 343-350, 378-398)."""
    nx, ny, nz = (int(n) + 1 for n in n_cells)
    ax = [np.linspace(lo[d], hi[d], int(n_cells[d]) + 1) for d in range(3)]
    kk, jj, ii = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    verts = np.stack([ax[0][ii.ravel()], ax[1][jj.ravel()], ax[2][kk.ravel()]], axis=1)

    def vid(i, j, k):
        return i + nx * (j + ny * k)

    cells = []
    for k in range(nz - 1):
        for i in range(nx - 1):
            for j in range(ny - 1):
                bot = [vid(i, j, k), vid(i + 1, j, k), vid(i, j + 1, k), vid(i + 1, j + 1, k)]
                cells.append(bot + [v + nx * ny for v in bot])
    return Level(verts, np.asarray(cells, dtype=np.int64))


def q2_numbering(level):
    """Scalar Q2 node coordinates and (nc, 27) table (mesh.py:162-216).

    Vertices keep their ids; every edge/face/centre node gets the next id at its
    first appearance in (cell ascending, local node ascending) order.  Edge and
    face nodes are identified by their sorted parent corners, centres by cell.
    Coordinates are the mean of the parent corners summed in the reference's
    parent order (free axes enumerated x fastest).
    """
    ix = multi_index(3)
    corner_of = {tuple(2 * c): n for n, c in enumerate(multi_index(2))}
    # per local node: the local corner numbers of its parents in reference order
    parents = []
    for a in range(27):
        free = np.nonzero(ix[a] == 1)[0]
        plist = []
        # enumerate 2^len(free) replacements with the first free axis fastest
        for m in range(2 ** free.size):
            p = ix[a].copy()
            for t, axis in enumerate(free):
                p[axis] = 2 * ((m >> t) & 1)
            plist.append(corner_of[tuple(p)])
        parents.append((free.size, plist))
    nv = level.verts.shape[0]
    table = np.empty((level.cells.shape[0], 27), dtype=np.int64)
    seen = {}
    new_xyz = []
    for c, cv in enumerate(level.cells):
        for a in range(27):
            nfree, plist = parents[a]
            if nfree == 0:
                table[c, a] = cv[corner_of[tuple(ix[a])]]
                continue
            pv = cv[plist]
            key = ("c", c) if nfree == 3 else tuple(sorted(pv.tolist()))
            nid = seen.get(key)
            if nid is None:
                nid = nv + len(new_xyz)
                seen[key] = nid
                acc = level.verts[pv[0]].copy()
                for q in pv[1:]:
                    acc = acc + level.verts[q]
                new_xyz.append(acc / len(pv))
            table[c, a] = nid
    coords = np.concatenate([level.verts, np.asarray(new_xyz).reshape(-1, 3)], axis=0)
    return coords, table


def refine(level, coords, table):
    """Uniform refinement: child 8c+o in octant order, new vertices = Q2 nodes
    (mesh.py:223-246)."""
    ix3 = {tuple(v): a for a, v in enumerate(multi_index(3))}
    octs = multi_index(2)
    cells = np.empty((level.cells.shape[0] * 8, 8), dtype=np.int64)
    for o in range(8):
        cols = [ix3[tuple(octs[o] + d)] for d in octs]
        cells[o::8] = table[:, cols]
    return Level(coords.copy(), cells)


class Hierarchy:
    """Box hierarchy with cached Q2 numberings (mesh.py:96-216)."""

    def __init__(self, lo, hi, n_cells, channel_tags=False):
        self.lo = np.asarray(lo, dtype=float)
        self.hi = np.asarray(hi, dtype=float)
        self.channel_tags = channel_tags
        self.levels = [box_level0(lo, hi, n_cells)]
        self._q2 = {}

    def q2(self, l):
        if l not in self._q2:
            self._q2[l] = q2_numbering(self.levels[l])
        return self._q2[l]

    def refine(self):
        l = len(self.levels) - 1
        coords, table = self.q2(l)
        self.levels.append(refine(self.levels[l], coords, table))


def boundary_faces(level, lo, hi, channel_tags):
    """Faces owned by one cell with their tag, sorted (mesh.py:118-151)."""
    owner = {}
    for c, cv in enumerate(level.cells):
        for f, cf in enumerate(CORNER_FACES):
            key = tuple(sorted(cv[list(cf)].tolist()))
            owner[key] = None if key in owner else (c, f)
    tol = 1e-9 * max(float(np.max(hi - lo)), 1.0)
    out = []
    for key, own in owner.items():
        if own is None:
            continue
        x = level.verts[list(key)][:, 0]
        tag = WALL
        if channel_tags:
            if np.all(np.abs(x - lo[0]) < tol):
                tag = INFLOW
            elif np.all(np.abs(x - hi[0]) < tol):
                tag = OUTFLOW
        out.append((own[0], own[1], tag))
    out.sort()
    return out


def node_tags(h, l):
    """Per-node tag with precedence OUTFLOW < INFLOW < WALL < OBSTACLE
    (space.py:23-30, 48-61)."""
    _, table = h.q2(l)
    ix = multi_index(3)
    face_nodes = [np.nonzero(ix[:, f // 2] == 2 * (f % 2))[0] for f in range(6)]
    tags = np.zeros(table.max() + 1, dtype=np.int64)
    faces = boundary_faces(h.levels[l], h.lo, h.hi, h.channel_tags)
    for t in (OUTFLOW, INFLOW, WALL, OBSTACLE):
        nodes = [table[c][face_nodes[f]] for (c, f, tt) in faces if tt == t]
        if nodes:
            tags[np.concatenate(nodes)] = t
    return tags


def constrained_dofs(tags, bc_tags):
    """Dirichlet velocity dofs of the bc tags plus a pressure pin at dof 0 when
    no node is OUTFLOW (space.py:66-77, driver.py:56-65)."""
    mask = np.zeros(4 * tags.size, dtype=bool)
    for t in bc_tags:
        nodes = np.nonzero(tags == t)[0]
        for c in (1, 2, 3):
            mask[4 * nodes + c] = True
    if not np.any(tags == OUTFLOW):
        mask[0] = True
    return mask


def impose_dirichlet(x, tags, coords, t, bcs):
    """In-place velocity boundary values (space.py:245-255)."""
    m = x.reshape(-1, 4)
    for tag, fn in bcs.items():
        nodes = np.nonzero(tags == tag)[0]
        if nodes.size == 0 or fn is None:
            continue
        m[nodes, 1:] = fn(t, coords[nodes])
    return x


def no_slip(t, pts):
    return np.zeros((pts.shape[0], 3))


def parabolic_inflow(vbar, H):
    """3-D inflow profile (space.py:212-231, 3-D branch)."""
    def profile(t, pts):
        w = 0.5 - 0.5 * np.cos(5 * np.pi * t) if t <= 0.2 else 1.0
        y, z = pts[:, 1], pts[:, 2]
        out = np.zeros((pts.shape[0], 3))
        out[:, 0] = w * 1.125 * vbar * y * (H - y) * (H ** 2 - z ** 2) / ((H / 2) ** 2 * H ** 2)
        return out
    return profile


# ----------------------------------------------------------------------------
# patches and geometry features (mesh.py:501-611)
# ----------------------------------------------------------------------------

def vertex_angles(X):
    """Mean pairwise angle of the incident edge vectors per corner (mesh.py:574-591)."""
    out = np.empty((X.shape[0], 8))
    inc = [[] for _ in range(8)]
    for a, b in CELL_EDGES:
        inc[a].append((a, b))
        inc[b].append((b, a))
    for v in range(8):
        vec = [X[:, b] - X[:, a] for a, b in inc[v]]
        ang = []
        for i in range(len(vec)):
            for j in range(i + 1, len(vec)):
                cosv = np.sum(vec[i] * vec[j], axis=1) / (
                    np.linalg.norm(vec[i], axis=1) * np.linalg.norm(vec[j], axis=1))
                ang.append(np.arccos(np.clip(cosv, -1.0, 1.0)))
        out[:, v] = np.mean(ang, axis=0)
    return out


def cell_features(level, ids):
    """12 edges, 4 diagonals, 8 mean vertex angles (mesh.py:594-611)."""
    X = level.verts[level.cells[ids]]
    el = np.stack([np.linalg.norm(X[:, b] - X[:, a], axis=1) for a, b in CELL_EDGES], axis=1)
    dl = np.stack([np.linalg.norm(X[:, b] - X[:, a], axis=1) for a, b in CELL_DIAGS], axis=1)
    return np.concatenate([el, dl, vertex_angles(X)], axis=1)


def patch_tables(h, L, J):
    """dof_table, node_table, valence, mu, geom_table (mesh.py:501-558)."""
    if J not in (1, 2):
        raise ValueError(f"unsupported patch depth J={J}; need 1 or 2")
    _, ftab = h.q2(L + J)
    ncoarse = h.levels[L].cells.shape[0]
    ix3 = multi_index(3)
    octs = multi_index(2)
    rows = []
    for M in range(ncoarse):
        for o in range(8):
            ch = 8 * M + o
            if J == 1:
                rows.append(ftab[ch])
                continue
            grid = np.full((5, 5, 5), -1, dtype=np.int64)   # indexed [x, y, z]
            for g in range(8):
                gc = 8 * ch + g
                for a in range(27):
                    p = 2 * octs[g] + ix3[a]
                    grid[p[0], p[1], p[2]] = ftab[gc, a]
            rows.append(grid.transpose(2, 1, 0).reshape(-1))
    node_table = np.asarray(rows, dtype=np.int64)
    dof_table = (4 * node_table[:, :, None] + np.arange(4)).reshape(node_table.shape[0], -1)
    nfine = 4 * h.q2(L + J)[0].shape[0]
    valence = np.bincount(dof_table.ravel(), minlength=nfine)
    geom = cell_features(h.levels[L], np.repeat(np.arange(ncoarse), 8))
    return dof_table, node_table, valence, 1.0 / valence, geom


# ----------------------------------------------------------------------------
# transfer (space.py:117-185)
# ----------------------------------------------------------------------------

def prolongation_csr(h, l):
    """Scalar Q2 embedding level l -> l+1 as (indptr, indices, data), columns
    ascending per row (space.py:117-165): each fine node takes the coarse shape
    values of the first (octant, local node, parent cell) that reaches it."""
    _, ctab = h.q2(l)
    fcoords, ftab = h.q2(l + 1)
    nf = fcoords.shape[0]
    octs = multi_index(2)
    ix3 = multi_index(3)
    src = np.full((nf, 3), -1, dtype=np.int64)      # (octant, local node, parent cell)
    for o in range(8):
        child = ftab[o::8]
        for a in range(27):
            nodes, first = np.unique(child[:, a], return_index=True)
            fresh = src[nodes, 0] < 0
            src[nodes[fresh]] = np.stack([np.full(fresh.sum(), o), np.full(fresh.sum(), a),
                                          first[fresh]], axis=1)
    sten = [q2_shape((octs[o][None, :] + ix3 / 2.0) / 2.0) for o in range(8)]
    cols, vals, counts = [], [], np.empty(nf, dtype=np.int64)
    for n in range(nf):
        o, a, C = src[n]
        w = sten[o][a]
        nz = np.nonzero(np.abs(w) > 1e-14)[0]
        c = ctab[C, nz]
        order = np.argsort(c, kind="stable")
        cols.append(c[order])
        vals.append(w[nz][order])
        counts[n] = nz.size
    indptr = np.zeros(nf + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(counts)
    return indptr, np.concatenate(cols), np.concatenate(vals)


def prolongate_state(csrs, x):
    """kron(P, I4) applied per level (space.py:168-185)."""
    v = np.asarray(x, dtype=float).reshape(-1, 4)
    for csr in csrs:
        indptr, indices, data = csr
        rowid = np.repeat(np.arange(indptr.size - 1), np.diff(indptr))
        out = np.zeros((indptr.size - 1, 4))
        np.add.at(out, rowid, data[:, None] * v[indices])
        v = out
    return v.reshape(-1)


# ----------------------------------------------------------------------------
# assembly (assembly.py)
# ----------------------------------------------------------------------------

class Quadrature:
    """Constant tables: N (64,27), dN (64,27,3), weights (64,), PI (27,27)."""

    def __init__(self):
        pts, self.wq = gauss_points(4)
        self.N = q2_shape(pts)
        self.dN = q2_grad(pts)
        self.PI = q1_projector()


QUAD = Quadrature()


def _es(*a):
    return np.einsum(*a, optimize=True)


def cell_diameters(level):
    """h_T: largest distance between two corners (assembly.py:99-103)."""
    C = level.verts[level.cells]
    d2 = ((C[:, :, None, :] - C[:, None, :, :]) ** 2).sum(-1)
    return np.sqrt(d2.max(axis=(1, 2)))


def cell_geometry(coords, table):
    """Isoparametric Q2 geometry per (cell, Gauss point) (assembly.py:77-98):
    G (nc,64,27,3), w (nc,64), Gpi = G.PI, and the node-major flattened
    gradient tables Gt = G^(nc,27,64*3) and dGt = Gt - Gpi^ used by the
    batched matrix products."""
    Q = QUAD
    X = coords[table]
    J = np.einsum('qaj,cai->cqij', Q.dN, X, optimize=True)
    det = np.linalg.det(J)
    if np.any(det <= 0):
        raise ValueError("non-positive Jacobian in isoparametric map")
    Jinv = np.linalg.inv(J)
    nc = X.shape[0]
    G = np.ascontiguousarray(np.einsum('qaj,cqji->cqai', Q.dN, Jinv, optimize=True))
    Gpi = np.ascontiguousarray(np.einsum('cqbj,ba->cqaj', G, Q.PI, optimize=True))
    Gt = np.ascontiguousarray(G.transpose(0, 2, 1, 3)).reshape(nc, 27, 192)
    dGt = Gt - np.ascontiguousarray(Gpi.transpose(0, 2, 1, 3)).reshape(nc, 27, 192)
    return G, Q.wq[None, :] * det, Gpi, Gt, dGt


def _chunks(n, size):
    for s in range(0, n, size):
        yield slice(s, min(n, s + size))


class GeometryCache:
    """Per-level geometry tables computed once, in chunks, like the reference's
    Assembler.__init__ (assembly.py:65-108)."""

    def __init__(self, coords, table, chunk=4096):
        self.chunks = [(sl, cell_geometry(coords, table[sl]))
                       for sl in _chunks(table.shape[0], chunk)]


def stab_weights(x, table, h_T, nu, k, alpha0=0.02, delta0=0.1):
    """alpha_T, delta_T at x (assembly.py:55-59, 169-178)."""
    vh = x.reshape(-1, 4)[table][:, :, 1:]
    vmax = np.sqrt((vh ** 2).sum(-1)).max(axis=1)
    den = nu / h_T ** 2 + vmax / h_T + 1.0 / k
    return alpha0 / den, delta0 / den


def _at_q(loc):
    """(nc,27,m) nodal values -> (nc,m,64) values at the Gauss points."""
    return np.matmul(loc.transpose(0, 2, 1), QUAD.N.T)


def _grad_at_q(loc, Gt):
    """(nc,27,m) -> (nc,m,64,3) physical gradients."""
    nc, _, m = loc.shape
    return np.matmul(loc.transpose(0, 2, 1), Gt).reshape(nc, m, 64, 3)


def element_vectors(x, geom, table, k, nu, alpha_T, delta_T, convection=True):
    """Per-cell (cont (nc,27), mom (nc,27,3)) of A_h(x) (assembly.py:148-167, 212-240);
    geom = cell_geometry of these cells.  Index order: fields (nc, comp, q[, j])."""
    Q = QUAD
    G, w, Gpi, Gt, dGt = geom
    nc = table.shape[0]
    loc = x.reshape(-1, 4)[table]
    ph, vh = loc[:, :, :1], np.ascontiguousarray(loc[:, :, 1:])
    v = _at_q(vh)                                  # (nc,3,64)
    gv = _grad_at_q(vh, Gt)                        # (nc,3,64,3)  [c,i,q,j]
    p = _at_q(ph)[:, 0]                            # (nc,64)
    gp = _grad_at_q(ph, Gt)[:, 0]                  # (nc,64,3)
    gpp = gp - _grad_at_q(ph, dGt)[:, 0]           # Gpi part: Gt - dGt
    conv = np.einsum('cjq,ciqj->ciq', v, gv) if convection else np.zeros_like(v)
    div = gv[:, 0, :, 0] + gv[:, 1, :, 1] + gv[:, 2, :, 2]
    # momentum: mass/k + 1/2 convection (N test), 1/2 nu diffusion and pressure (G test)
    mom = np.matmul(w[:, None, :] * (v / k + 0.5 * conv), Q.N)                   # (nc,3,27)
    flux = 0.5 * nu * w[:, None, :, None] * gv                                  # [c,i,q,j]
    flux[:, 0, :, 0] -= w * p
    flux[:, 1, :, 1] -= w * p
    flux[:, 2, :, 2] -= w * p
    mom += np.matmul(Gt, flux.reshape(nc, 3, 192).transpose(0, 2, 1)).transpose(0, 2, 1)
    # continuity: (div v, xi) + alpha (grad(p - pi p), grad(xi - pi xi))
    cont = np.matmul(w * div, Q.N)
    y = (alpha_T[:, None, None] * w[:, :, None] * (gp - gpp)).reshape(nc, 192, 1)
    cont += np.matmul(dGt, y)[:, :, 0]
    use_delta = convection and delta_T is not None and np.any(delta_T != 0.0)
    if use_delta:
        pvh = np.matmul(Q.PI, vh)                                               # (nc,27,3)
        pv = _at_q(pvh)
        gpv = _grad_at_q(pvh, Gt)
        g = conv - np.einsum('cjq,ciqj->ciq', pv, gpv)
        S = np.matmul(G, v.transpose(0, 2, 1)[:, :, :, None])[..., 0] \
            - np.matmul(Gpi, pv.transpose(0, 2, 1)[:, :, :, None])[..., 0]        # (nc,64,27)
        mom += np.matmul(delta_T[:, None, None] * w[:, None, :] * g, S)
    return cont, mom.transpose(0, 2, 1)


def rhs_vectors(x, geom, table, k, nu, f_old=None, f_new=None, convection=True):
    """Per-cell momentum rows of the next-step RHS (assembly.py:242-259)."""
    Q = QUAD
    G, w, _, Gt, _ = geom
    nc = table.shape[0]
    vh = np.ascontiguousarray(x.reshape(-1, 4)[table][:, :, 1:])
    v = _at_q(vh)
    gv = _grad_at_q(vh, Gt)
    acc = v / k - (0.5 * np.einsum('cjq,ciqj->ciq', v, gv) if convection else 0.0)
    for fa in (f_old, f_new):
        if fa is not None:
            acc = acc + 0.5 * _at_q(np.ascontiguousarray(fa[table]))
    mom = np.matmul(w[:, None, :] * acc, Q.N)
    flux = (0.5 * nu * w[:, None, :, None] * gv).reshape(nc, 3, 192)
    mom -= np.matmul(Gt, flux.transpose(0, 2, 1)).transpose(0, 2, 1)
    return np.zeros((nc, 27)), mom.transpose(0, 2, 1)


def assemble(table, cont, mom, ndof):
    """Dual-vector accumulation in ascending cell order (assembly.py:180-184)."""
    loc = np.concatenate([cont[:, :, None], mom], axis=2).reshape(-1)
    dofs = (4 * table[:, :, None] + np.arange(4)).reshape(-1)
    return np.bincount(dofs, weights=loc, minlength=ndof)


def _geometry(coords, table, cache):
    return cache if cache is not None else GeometryCache(coords, table)


def residual(x, b_prev, coords, table, k, nu, alpha_T, delta_T, mask=None, cache=None):
    """r = b_prev - A_h(x), constrained rows zeroed (assembly.py:261-267)."""
    A = np.zeros(x.size)
    for sl, geom in _geometry(coords, table, cache).chunks:
        cont, mom = element_vectors(x, geom, table[sl], k, nu, alpha_T[sl], delta_T[sl])
        A += assemble(table[sl], cont, mom, x.size)
    r = b_prev - A
    if mask is not None:
        r[mask] = 0.0
    return r


def rhs_next(x, coords, table, k, nu, cache=None):
    """Next-step fine RHS with f = None (assembly.py:242-259)."""
    out = np.zeros(x.size)
    for sl, geom in _geometry(coords, table, cache).chunks:
        cont, mom = rhs_vectors(x, geom, table[sl], k, nu)
        out += assemble(table[sl], cont, mom, x.size)
    return out


# ----------------------------------------------------------------------------
# patch network and correction (net.py:124-159, patch_ops.py:16-76, driver.py:251-268)
# ----------------------------------------------------------------------------

class Mlp:
    """Eval-mode network state (net.py:54-112)."""

    def __init__(self, W, activation="tanh", gamma=None, beta=None, running_mean=None,
                 running_var=None, input_mean=None, input_std=None, bn_eps=1e-5):
        self.W = [np.asarray(w, dtype=float) for w in W]
        depth = len(W) - 1
        H = self.W[0].shape[1]
        self.activation = activation
        self.gamma = gamma if gamma is not None else [np.ones(H)] * depth
        self.beta = beta if beta is not None else [np.zeros(H)] * depth
        self.running_mean = running_mean if running_mean is not None else [np.zeros(H)] * depth
        self.running_var = running_var if running_var is not None else [np.ones(H)] * depth
        n_in = self.W[0].shape[0]
        self.input_mean = input_mean if input_mean is not None else np.zeros(n_in)
        self.input_std = input_std if input_std is not None else np.ones(n_in)
        self.bn_eps = bn_eps


def mlp_forward(m, X):
    """Eval forward: normalise input, BN-affine, activation, skip for i >= 1,
    linear head (net.py:124-159)."""
    act = np.tanh if m.activation == "tanh" else (lambda z: np.maximum(z, 0.0))
    h = (np.asarray(X, dtype=float) - m.input_mean) / m.input_std
    for i in range(len(m.W) - 1):
        z = h @ m.W[i]
        zhat = (z - m.running_mean[i]) * (1.0 / np.sqrt(m.running_var[i] + m.bn_eps))
        a = act(zhat * m.gamma[i] + m.beta[i])
        h = a + h if i >= 1 else a
    return h @ m.W[-1]


def network_input(x_tilde, r, dof_table, geom):
    """[x~ rows | r rows | geometry] (patch_ops.py:23-29, 49-53)."""
    return np.concatenate([x_tilde[dof_table], r[dof_table], geom], axis=1)


def scatter_average(Y, dof_table, mu, mask=None):
    """Velocity rows -> global defect by bincount, times mu, masked (patch_ops.py:16-20, 32-38, 64-76)."""
    npp = dof_table.shape[1] // 4
    rows = np.zeros(dof_table.shape)
    vel = (np.arange(npp)[:, None] * 4 + np.arange(1, 4)[None, :]).ravel()
    rows[:, vel] = Y
    d = mu * np.bincount(dof_table.ravel(), weights=rows.ravel(), minlength=mu.size)
    if mask is not None:
        d[mask] = 0.0
    return d


def correction_step(x_coarse, b_prev, ctx, model, t, nu, k, alpha0=0.02, delta0=0.1,
                    scale=1.0, bcs=None):
    """One fine-level correction (driver.py:251-268); returns a dict of every
    intermediate.  ctx holds the index maps built by ``build_context``."""
    bcs = bcs if bcs is not None else {WALL: no_slip}
    xt = prolongate_state(ctx["P"], x_coarse)
    impose_dirichlet(xt, ctx["tags"], ctx["coords"], t, bcs)
    aT, dT = stab_weights(xt, ctx["table"], ctx["h_T"], nu, k, alpha0, delta0)
    r = residual(xt, b_prev, ctx["coords"], ctx["table"], k, nu, aT, dT, ctx["mask"],
                 cache=ctx.get("geometry"))
    X = network_input(xt, r, ctx["dof_table"], ctx["geom"])
    Y = mlp_forward(model, X)
    d = scatter_average(Y, ctx["dof_table"], ctx["mu"], ctx["mask"])
    return dict(x_tilde=xt, alpha_T=aT, delta_T=dT, r=r, X=X, Y=Y, d=d, x_corr=xt + scale * d)


def build_context(lo, hi, n_cells, L, J, jitter_fn=None, channel_tags=False, bc_tags=(WALL,),
                  cache_geometry=False):
    """Hierarchy plus every index map the correction step needs; cache_geometry
    precomputes the per-level geometry once as the reference's Assembler does."""
    h = Hierarchy(lo, hi, n_cells, channel_tags)
    if jitter_fn is not None:
        jitter_fn(h.levels[0].verts)
    for _ in range(L + J):
        h.refine()
    coords, table = h.q2(L + J)
    tags = node_tags(h, L + J)
    dof_table, node_table, valence, mu, geom = patch_tables(h, L, J)
    return dict(h=h, coords=coords, table=table, tags=tags,
                mask=constrained_dofs(tags, bc_tags),
                P=[prolongation_csr(h, l) for l in range(L, L + J)],
                h_T=cell_diameters(h.levels[L + J]), dof_table=dof_table,
                node_table=node_table, valence=valence, mu=mu, geom=geom,
                coarse_coords=h.q2(L)[0],
                geometry=GeometryCache(coords, table) if cache_geometry else None)
