"""Keep the first N sampled patch rows of a pin (X, Y, rows) to bound the fixture size:
python tests/golden/trim_pin.py cfg2 128"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
name, n = sys.argv[1], int(sys.argv[2])
path = os.path.join(HERE, f"{name}_pin.npz")
with np.load(path) as z:
    d = {k: z[k] for k in z.files}
for k in ("rows", "X", "Y"):
    d[k] = d[k][:n]
np.savez_compressed(path, **d)
