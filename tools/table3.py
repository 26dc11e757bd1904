"""Table 3-style map-size study: online training at weight
length 64 on square maps 16x16 ... 512x512 with the same data and number of
steps; prints kernel time per map and the ratio per doubling beside the
paper's (P5000) ratios.  python tools/table3.py [steps] [docs]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_09598_b200 import som  # noqa: E402
from synth import uniform_matrix  # noqa: E402

PAPER = {16: 34.25, 32: 32.81, 64: 33.37, 128: 38.40, 256: 111.03, 512: 431.38}   # P:304-305, seconds

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
X = uniform_matrix(n, 64, 64)
out = []
prev = None
for side in (16, 32, 64, 128, 256, 512):
    W0 = uniform_matrix(side * side, 64, side)
    with som.SOM(side, side, 64, 1) as m:
        m.set_weights(W0)
        m.train_online(X, epochs=(steps + n - 1) // n, alpha0=0.1, sigma0=side / 2.0, seed=1, t_end=min(steps, 200))
        m.set_weights(W0)
        m.train_online(X, epochs=(steps + n - 1) // n, alpha0=0.1, sigma0=side / 2.0, seed=1, t_end=steps)
        ms, units, _ = som.som_last_stats(m.h)
        g, k = som.som_last_train_config(m.h)
    row = {"map": f"{side}x{side}", "N": side * side, "steps": units, "ms": ms, "us_per_step": 1000.0 * ms / units,
           "ratio": None if prev is None else ms / prev, "grid": g, "kernel": k,
           "paper_s": PAPER[side], "paper_ratio": None if side == 16 else PAPER[side] / PAPER[side // 2]}
    prev = ms
    out.append(row)
    print(json.dumps(row), flush=True)
