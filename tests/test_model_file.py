"""DNMG model files (net.py:337-392): the product's reader against a
file written by the reference's own save_model (tests/golden/make_model_fixture.py),
a write/read round trip, and the reference's error messages."""
import os

import numpy as np
import pytest

from paper_2307_14837_b200 import net

HERE = os.path.dirname(os.path.abspath(__file__))


def test_reads_reference_written_file():
    m = net.load_model(os.path.join(HERE, "golden", "model_small.dnmg"))
    z = np.load(os.path.join(HERE, "golden", "model_small.npz"))
    assert m.mode == "eval" and m.activation == "tanh"
    assert (m.arch.n_in, m.arch.n_hidden, m.arch.depth, m.arch.n_out) == (40, 16, 3, 9)
    assert np.array_equal(m.input_mean, z["input_mean"])
    assert np.array_equal(m.input_std, z["input_std"])
    for i in range(4):
        assert np.array_equal(m.W[i], z[f"W{i}"])
    for i in range(3):
        assert np.array_equal(m.gamma[i], z[f"gamma{i}"])
        assert np.array_equal(m.beta[i], z[f"beta{i}"])
        assert np.array_equal(m.running_mean[i], z[f"rmean{i}"])
        assert np.array_equal(m.running_var[i], z[f"rvar{i}"])


def test_round_trip_is_byte_identical(tmp_path):
    src = os.path.join(HERE, "golden", "model_small.dnmg")
    m = net.load_model(src)
    out = tmp_path / "copy.dnmg"
    net.save_model(m, str(out))
    assert out.read_bytes() == open(src, "rb").read()


def test_rejects_bad_files(tmp_path):
    bad = tmp_path / "bad.dnmg"
    bad.write_bytes(b"XXXX" + bytes(40))
    with pytest.raises(ValueError, match="magic"):
        net.load_model(str(bad))
    raw = bytearray(open(os.path.join(HERE, "golden", "model_small.dnmg"), "rb").read())
    raw[4] = 7
    bad.write_bytes(bytes(raw))
    with pytest.raises(ValueError, match="version"):
        net.load_model(str(bad))
    bad.write_bytes(open(os.path.join(HERE, "golden", "model_small.dnmg"), "rb").read()[:200])
    with pytest.raises(ValueError, match="truncated"):
        net.load_model(str(bad))
