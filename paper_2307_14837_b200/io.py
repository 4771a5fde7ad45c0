"""Binary formats on the training-data path (reference io.py), host side.

* "DMGT" state trajectories (io.py:150-212): header <4sIIQd (magic, version, level,
  ndof, k), then records <Qd (step, t) + float64[ndof]; record 0 is the initial state.
* "DMGD" dataset shards + ``dataset.json`` sidecar (io.py:216-287): per shard a header
  <4sIIIIIIIQ (magic, version, n_features, n_targets, n_dof_patch, n_geo, dim, J, rows)
  followed by the row block [features | targets] as little-endian float64.

The writer here is a stream: row blocks arrive per time step straight from the GPU
(``dnnmg_dataset_rows``) together with their per-column statistics
(``dnnmg_column_stats``), and are cut into shards of exactly the reference's size and
order, so ``load_dataset`` of either implementation reads the other's output.
"""

import json
import struct
from pathlib import Path

import numpy as np

TRAJ_MAGIC, TRAJ_VERSION = b"DMGT", 1
DATA_MAGIC, DATA_VERSION = b"DMGD", 1
_TRAJ_HDR = struct.Struct("<4sIIQd")
_TRAJ_REC = struct.Struct("<Qd")
_DATA_HDR = struct.Struct("<4sIIIIIIIQ")
COMPONENTS = ("p", "v_x", "v_y", "v_z")


# -- trajectories ----------------------------------------------------------------------

class TrajectoryWriter:
    """Append-only (step, t, values) series; steps must be 0, 1, 2, ... (io.py:153-171)."""

    def __init__(self, path, level, ndof, k):
        self.path = Path(path)
        self.ndof = int(ndof)
        self.count = 0
        self.f = open(self.path, "wb")
        self.f.write(_TRAJ_HDR.pack(TRAJ_MAGIC, TRAJ_VERSION, int(level), self.ndof, float(k)))

    def append(self, step, t, values):
        if step != self.count:
            raise ValueError(f"trajectory steps must be contiguous (got {step}, "
                             f"expected {self.count})")
        v = np.ascontiguousarray(values, dtype="<f8")
        if v.size != self.ndof:
            raise ValueError(f"record length {v.size} != ndof {self.ndof}")
        self.f.write(_TRAJ_REC.pack(step, float(t)))
        self.f.write(v.tobytes())
        self.count += 1

    def close(self):
        self.f.close()


class Trajectory:
    """Memory-mapped reader (io.py:174-212)."""

    def __init__(self, path):
        self.path = Path(path)
        with open(self.path, "rb") as f:
            magic, version, level, ndof, k = _TRAJ_HDR.unpack(f.read(_TRAJ_HDR.size))
        if magic != TRAJ_MAGIC:
            raise ValueError(f"not a trajectory file: bad magic {magic!r}")
        if version != TRAJ_VERSION:
            raise ValueError(f"unsupported trajectory version {version}")
        self.level, self.ndof, self.k = level, ndof, k
        self._rec = _TRAJ_REC.size + 8 * ndof
        body = self.path.stat().st_size - _TRAJ_HDR.size
        if body % self._rec:
            raise ValueError("truncated trajectory file")
        self.n_records = body // self._rec
        self._mm = np.memmap(self.path, dtype="<u1", mode="r", offset=_TRAJ_HDR.size)

    @property
    def n_steps(self):
        return self.n_records - 1

    def record(self, i):
        off = i * self._rec
        step, t = _TRAJ_REC.unpack(self._mm[off:off + _TRAJ_REC.size].tobytes())
        vals = np.frombuffer(self._mm[off + _TRAJ_REC.size:off + self._rec].tobytes(), dtype="<f8")
        return step, t, vals

    def values(self, n):
        step, _, vals = self.record(n)
        if step != n:
            raise ValueError("non-contiguous trajectory")
        return vals

    def time(self, n):
        return self.record(n)[1]


# -- datasets ----------------------------------------------------------------------------

class ColumnStats:
    """Running per-column (sum, centred sum of squares M2, min, max) over row blocks,
    combined pairwise in block order (Chan et al.; deterministic, no E[x^2] - mean^2
    cancellation); the sidecar's mean / std / extrema derive from it."""

    def __init__(self, w):
        self.n = 0
        self.s = np.zeros(w)
        self.q = np.zeros(w)
        self.mn = np.full(w, np.inf)
        self.mx = np.full(w, -np.inf)

    def add(self, n, stats):
        """stats: [4][w] = sum | centred sum of squares | min | max of a block of n rows."""
        if n == 0:
            return
        if self.n:
            delta = stats[0] / n - self.s / self.n
            self.q = self.q + stats[1] + delta * delta * (self.n * n / (self.n + n))
        else:
            self.q = np.array(stats[1], dtype=float)
        self.n += n
        self.s += stats[0]
        self.mn = np.minimum(self.mn, stats[2])
        self.mx = np.maximum(self.mx, stats[3])

    def mean(self):
        return self.s / self.n

    def std(self):
        return np.sqrt(self.q / self.n)


class DatasetWriter:
    """Streamed "DMGD" shards and the ``dataset.json`` sidecar (io.py:219-266)."""

    def __init__(self, out_dir, patchset, dim=3):
        self.out = Path(out_dir)
        self.out.mkdir(parents=True, exist_ok=True)
        self.ps = patchset
        self.dim = dim
        self.sets = {}
        self.layout = {"n_dof_patch": int(patchset.ndof_patch), "n_geo": int(patchset.n_geo),
                       "dim": dim, "J": int(patchset.J), "L": int(patchset.L),
                       "feature_order": "state|residual|geometry"}

    def begin_set(self, name, rows, n_features, n_targets, shard_bytes):
        """Declare a set of `rows` rows (known in advance, so shard sizes are fixed)."""
        if rows == 0:
            n_features = n_targets = 0
        row_bytes = 8 * (n_features + n_targets)
        per = max(1, shard_bytes // max(row_bytes, 1))
        self.sets[name] = dict(rows=rows, nf=n_features, nt=n_targets, per=per, done=0,
                               shards=[], f=None, left=0,
                               stats=ColumnStats(n_features + n_targets))

    def add_rows(self, name, block, stats=None):
        """Append a float64 row block [k][nf+nt] (with its column statistics)."""
        st = self.sets[name]
        block = np.ascontiguousarray(block, dtype="<f8")
        k = block.shape[0]
        if st["done"] + k > st["rows"]:
            raise ValueError(f"set {name!r}: more rows than declared")
        if stats is not None:
            st["stats"].add(k, np.asarray(stats))
        i = 0
        while i < k:
            if st["left"] == 0:
                self._open_shard(name, st)
            take = min(st["left"], k - i)
            st["f"].write(block[i:i + take].tobytes())
            st["left"] -= take
            st["done"] += take
            i += take
            if st["left"] == 0:
                st["f"].close()
                st["f"] = None

    def _open_shard(self, name, st):
        s = len(st["shards"])
        n = min(st["per"], st["rows"] - st["done"])
        fname = f"{name}_{s:03d}.dmgd"
        f = open(self.out / fname, "wb")
        ps = self.ps
        f.write(_DATA_HDR.pack(DATA_MAGIC, DATA_VERSION, st["nf"], st["nt"], int(ps.ndof_patch),
                               int(ps.n_geo), self.dim, int(ps.J), n))
        st["shards"].append(fname)
        st["f"], st["left"] = f, n

    def finish(self):
        doc = {"layout": self.layout, "sets": {}}
        for name, st in self.sets.items():
            if st["done"] != st["rows"]:
                raise ValueError(f"set {name!r}: {st['done']} of {st['rows']} rows written")
            doc["sets"][name] = self._set_doc(st)
        path = self.out / "dataset.json"
        path.write_text(json.dumps(doc, indent=1))
        return path

    def _set_doc(self, st):
        rows, nf = st["rows"], st["nf"]
        cs = st["stats"]
        comp = {}
        ndof = int(self.ps.ndof_patch)
        nc = self.dim + 1
        for c, cname in enumerate(COMPONENTS[:nc]):
            if rows == 0:
                comp[cname] = {"max": 0.0, "mean": 0.0, "min": 0.0, "sigma": 0.0}
                continue
            cols = np.arange(c, ndof, nc)
            cnt = rows * cols.size
            mean = cs.s[cols].sum() / cnt
            # pooled over the component's columns: sum of M2 plus the between-column part
            cm = cs.s[cols] / rows
            var = (cs.q[cols].sum() + rows * ((cm - mean) ** 2).sum()) / cnt
            comp[cname] = {"max": float(cs.mx[cols].max()), "mean": float(mean),
                           "min": float(cs.mn[cols].min()), "sigma": float(np.sqrt(var))}
        return {"shards": st["shards"], "rows": int(rows), "n_features": int(nf),
                "n_targets": int(st["nt"]), "component_stats": comp,
                "feature_mean": cs.mean()[:nf].tolist() if rows else [],
                "feature_std": cs.std()[:nf].tolist() if rows else []}


def load_dataset(dataset_json, name):
    """(features, targets, sidecar) of one set, shards concatenated (io.py:269-287)."""
    meta = json.loads(Path(dataset_json).read_text())
    base = Path(dataset_json).parent
    X, T = [], []
    for shard in meta["sets"][name]["shards"]:
        with open(base / shard, "rb") as f:
            hdr = _DATA_HDR.unpack(f.read(_DATA_HDR.size))
            if hdr[0] != DATA_MAGIC:
                raise ValueError(f"not a dataset shard: bad magic {hdr[0]!r}")
            if hdr[1] != DATA_VERSION:
                raise ValueError(f"unsupported dataset version {hdr[1]}")
            nf, nt, rows = hdr[2], hdr[3], hdr[8]
            blk = np.frombuffer(f.read(8 * rows * (nf + nt)), dtype="<f8").reshape(rows, nf + nt)
        X.append(blk[:, :nf])
        T.append(blk[:, nf:])
    nf = meta["sets"][name]["n_features"]
    nt = meta["sets"][name]["n_targets"]
    Xc = np.concatenate(X) if X else np.zeros((0, nf))
    Tc = np.concatenate(T) if T else np.zeros((0, nt))
    return Xc, Tc, meta


# -- checkpoints -------------------------------------------------------------------------

_CKPT_MAGIC, _CKPT_VERSION = b"DMGC", 1
_CKPT_HDR = struct.Struct("<IQdI")   # version, step, t, meta length (after the magic)


def save_checkpoint(path, step, t, arrays, meta=None):
    """"DMGC" checkpoint (io.py:112-128): named float64 vectors plus a JSON meta; device
    tensors are copied to the host."""
    meta_b = json.dumps(meta or {}, sort_keys=True).encode()
    with open(path, "wb") as f:
        f.write(_CKPT_MAGIC)
        f.write(_CKPT_HDR.pack(_CKPT_VERSION, int(step), float(t), len(meta_b)))
        f.write(meta_b)
        f.write(struct.pack("<I", len(arrays)))
        for name, arr in arrays.items():
            if hasattr(arr, "detach"):
                arr = arr.detach().double().cpu().numpy()
            a = np.ascontiguousarray(arr, dtype="<f8").reshape(-1)
            nb = name.encode()
            f.write(struct.pack("<I", len(nb)))
            f.write(nb)
            f.write(struct.pack("<Q", a.size))
            f.write(a.tobytes())


def load_checkpoint(path):
    """(step, t, arrays, meta) of a "DMGC" file (io.py:131-147)."""
    with open(path, "rb") as f:
        magic = f.read(4)
        if magic != _CKPT_MAGIC:
            raise ValueError(f"not a checkpoint file: bad magic {magic!r}")
        version, step, t, metalen = _CKPT_HDR.unpack(f.read(_CKPT_HDR.size))
        if version != _CKPT_VERSION:
            raise ValueError(f"unsupported checkpoint version {version}")
        meta = json.loads(f.read(metalen).decode())
        (count,) = struct.unpack("<I", f.read(4))
        arrays = {}
        for _ in range(count):
            (nl,) = struct.unpack("<I", f.read(4))
            name = f.read(nl).decode()
            (size,) = struct.unpack("<Q", f.read(8))
            arrays[name] = np.frombuffer(f.read(8 * size), dtype="<f8").copy()
    return step, t, arrays, meta
