"""Print the measured errors of the GPU step against the reference's full-size pins
(tests/golden/cfg{1,2,3}_pin.npz) per precision — the numbers DESIGN.md §3 quotes.
Run on the GPU box: python tools/gpu/pin_errors.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_gpu_big_pins as big  # noqa: E402
from golden_util import sampled_rel  # noqa: E402
from paper_2307_14837_b200.step import CorrectionStep  # noqa: E402

for name, precs in (("cfg1", ("fp32", "f16x3", "tf32x3", "bf16")),
                    ("cfg2", ("f16x3", "tf32x3", "bf16")),
                    ("cfg3", ("fp32", "f16x3", "tf32x3", "bf16"))):
    try:
        c = big.problem(name)
    except BaseException as e:  # pytest.skip outside pytest
        print(name, "skipped:", e)
        continue
    cfg, pin = c["cfg"], c["pin"]
    for p in precs:
        step = CorrectionStep(c["h"], 0, cfg["J"], c["model"], cfg["nu"], cfg["dt"], precision=p,
                              patchset=c["ps"], t=0.0)
        b = step.rhs_next(step.embed(torch.tensor(c["x0"], dtype=torch.float32, device="cuda")))
        step.set_time(cfg["dt"])
        out = step(torch.tensor(c["x1"], dtype=torch.float32, device="cuda"), b)
        torch.cuda.synchronize()
        res = {"b_prev": b, "x_tilde": step.x_tilde, "r": step.r, "d": step.d, "x_corr": out,
               "b_next": step.rhs_next(out)}
        msg = " ".join(f"{k}={sampled_rel(v.double().cpu().numpy(), pin, k)[0]:.1e}"
                       for k, v in res.items())
        print(name, p, msg, flush=True)
