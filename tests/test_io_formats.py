"""Host-side file formats of the training-data path (reference io.py) against files
written by the REFERENCE itself (tests/golden/dataset, made by make_dataset.py):
"DMGT" trajectories are read back, and the streamed "DMGD" shard writer, fed the
reference's own rows, reproduces the reference's shards byte for byte and its
sidecar (io.py:150-287)."""
import json
import os

import numpy as np
import pytest

from paper_2307_14837_b200 import io as iomod, mesh as meshmod, synthetic

HERE = os.path.dirname(os.path.abspath(__file__))
DS = os.path.join(HERE, "golden", "dataset")


def _patchset():
    h = meshmod.build_template_mesh("box", extent_lo=(0, 0, -0.205), extent_hi=(1.0, 0.41, 0.205),
                                    n_cells=(2, 1, 1), channel_tags=True)
    synthetic.jitter_vertices(h.levels[0].vertices, (2, 1, 1), (0, 0, -0.205), (1.0, 0.41, 0.205), 21)
    meshmod.refine_uniform(h)
    return h, meshmod.build_patches(h, 0, 1)


def test_trajectory_reader_reads_reference_file():
    t = iomod.Trajectory(os.path.join(DS, "coarse.dmgt"))
    assert (t.level, t.n_steps, t.k) == (0, 6, 0.02)
    h, _ = _patchset()
    nodes = h.scalar_nodes(0)[0]
    modes = synthetic.fourier_modes(106)
    for n in (0, 3, 6):
        assert np.array_equal(t.values(n), synthetic.coarse_state(nodes, modes, 106, n, n * 0.02, 1e-3))
        assert t.time(n) == n * 0.02


def test_trajectory_roundtrip_and_errors(tmp_path):
    p = tmp_path / "a.dmgt"
    w = iomod.TrajectoryWriter(p, 2, 5, 0.1)
    for n in range(3):
        w.append(n, 0.1 * n, np.arange(5) + n)
    with pytest.raises(ValueError, match="contiguous"):
        w.append(5, 0.5, np.zeros(5))
    w.close()
    t = iomod.Trajectory(p)
    assert t.n_steps == 2 and np.array_equal(t.values(2), np.arange(5) + 2)
    with open(p, "ab") as f:
        f.write(b"xx")
    with pytest.raises(ValueError, match="truncated"):
        iomod.Trajectory(p)
    q = tmp_path / "b.dmgt"
    q.write_bytes(b"NOPE" + bytes(24))
    with pytest.raises(ValueError, match="magic"):
        iomod.Trajectory(q)


@pytest.mark.parametrize("which", ["loop", "self"])
def test_dataset_writer_reproduces_reference_shards(tmp_path, which):
    ref = os.path.join(DS, which, "dataset.json")
    meta = json.loads(open(ref).read())
    _, ps = _patchset()
    w = iomod.DatasetWriter(tmp_path, ps)
    blocks = {}
    for name in ("train", "val"):
        X, T, _ = iomod.load_dataset(ref, name)
        rows = np.concatenate([X, T], axis=1)
        blocks[name] = rows
        w.begin_set(name, rows.shape[0], X.shape[1], T.shape[1], 30000)
    for name, rows in blocks.items():
        for i in range(0, rows.shape[0], 16):      # one 16-patch block per step
            b = rows[i:i + 16]
            m2 = ((b - b.mean(0)) ** 2).sum(0)
            w.add_rows(name, b, np.stack([b.sum(0), m2, b.min(0), b.max(0)]))
    out = json.loads(w.finish().read_text())
    assert out["layout"] == meta["layout"]
    for name in ("train", "val"):
        mine, theirs = out["sets"][name], meta["sets"][name]
        assert mine["shards"] == theirs["shards"]
        for k in ("rows", "n_features", "n_targets"):
            assert mine[k] == theirs[k]
        for shard in mine["shards"]:
            assert (tmp_path / shard).read_bytes() == open(os.path.join(DS, which, shard), "rb").read()
        np.testing.assert_allclose(mine["feature_mean"], theirs["feature_mean"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(mine["feature_std"], theirs["feature_std"], rtol=1e-6, atol=1e-9)
        for c, st in theirs["component_stats"].items():
            for k, v in st.items():
                assert mine["component_stats"][c][k] == pytest.approx(v, rel=1e-7, abs=1e-10)


@pytest.mark.parametrize("name", ["hybrid", "mg"])
def test_checkpoint_roundtrip_is_byte_identical(tmp_path, name):
    """"DMGC" checkpoints written by the reference (driver.checkpoint_state +
    io.save_checkpoint, made by make_timeloop.py) read back and re-written byte for byte."""
    src = os.path.join(HERE, "golden", f"timeloop_{name}.dmgc")
    step, t, arrays, meta = iomod.load_checkpoint(src)
    assert step == 2 and abs(t - 0.04) < 1e-12 and meta["n"] == 2
    assert ("x_fine" in arrays) == (name == "hybrid")
    out = tmp_path / "c.dmgc"
    iomod.save_checkpoint(out, step, t, arrays, meta)
    assert out.read_bytes() == open(src, "rb").read()
    bad = tmp_path / "bad.dmgc"
    bad.write_bytes(b"NOPE" + bytes(24))
    with pytest.raises(ValueError, match="magic"):
        iomod.load_checkpoint(bad)
