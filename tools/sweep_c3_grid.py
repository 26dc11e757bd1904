"""c3 grid-size sweep for kernels 4 and 10: us/step over an early window
(full coverage) and a late window (sigma at its floor), from the same
weights (the late window starts from a snapshot at t = 450,000).

  python tools/sweep_c3_grid.py [steps=5000]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_09598_b200 import som  # noqa: E402
from synth import CONFIGS, bank_corpus  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
cfg = CONFIGS["c3"]
n, d = cfg["n"], cfg["d"]
C = bank_corpus(n, d, seed=301)
rp, ci, va = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))
m = som.SOM(cfg["rows"], cfg["cols"], d, cfg["topo"])
som.som_init_random_csr(m.h, rp, ci, va, n, 1301)
W0 = m.get_weights()
som.som_train_online_csr(m.h, rp, ci, va, n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, 0, 450000, None)
W450 = m.get_weights()
res = []
for tier in ("0", "1"):
    os.environ["SOM_TRAIN_TIER"] = tier
    for G in (148, 144, 136, 128, 120, 112, 96, 74):
        som.som_set_train_grid(m.h, G)
        row = {"tier": tier, "G": G}
        for name, W, t0 in (("early", W0, 0), ("late", W450, 450000)):
            m.set_weights(W)
            som.som_train_online_csr(m.h, rp, ci, va, n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, t0, t0 + steps,
                                     None)
            ms, units, _ = som.som_last_stats(m.h)
            g, k = som.som_last_train_config(m.h)
            row[name] = round(1000 * ms / units, 3)
            row["kernel"] = k
            row["grid"] = g
        print(json.dumps(row), flush=True)
        res.append(row)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/sweep_c3_grid.json", "w") as f:
    json.dump(res, f, indent=1)
