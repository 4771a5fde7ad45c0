"""Stand-alone MLP timing (config 4 style sweep point): python tools/perf_mlp.py ROWS PREC."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2307_14837_b200 import device as dv, net  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 524288
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16"
n_in = int(sys.argv[3]) if len(sys.argv) > 3 else 240
m = net.MlpModel(net.Architecture(n_in, 256, 3, 81), activation="tanh").eval()
dm = dv.DeviceModel(m, prec)
X = torch.randn(rows, n_in, device="cuda")
Y = torch.empty(rows, 81, device="cuda")
for _ in range(3):
    dm.forward(X, rows, Y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    dm.forward(X, rows, Y)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
fl = 2 * (n_in * 256 + 2 * 256 * 256 + 256 * 81) * rows
print(f"{prec} rows={rows} {ms:.3f} ms  {fl / ms / 1e9:.1f} TFLOP/s")
