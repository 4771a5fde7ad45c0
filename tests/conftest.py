import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")
GOLDEN_CASES = ("cfg0", "jit", "j2", "lvl1", "chan")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session", params=GOLDEN_CASES)
def golden(request):
    return request.param, load_golden(request.param)


def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
