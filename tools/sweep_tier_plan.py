"""Kernel 10 storage plan sweep on c3: (shared-memory rows, ring chunks)
against us/step over an early window (every unit updated) from the same
weights.   python tools/sweep_tier_plan.py [steps=3000]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_09598_b200 import som  # noqa: E402
from synth import CONFIGS, bank_corpus  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
cfg = CONFIGS["c3"]
n, d = cfg["n"], cfg["d"]
C = bank_corpus(n, d, seed=301)
rp, ci, va = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))
m = som.SOM(cfg["rows"], cfg["cols"], d, cfg["topo"])
som.som_init_random_csr(m.h, rp, ci, va, n, 1301)
W0 = m.get_weights()
os.environ["SOM_TRAIN_TIER"] = "1"
os.environ["SOM_TIER_HANDOVER"] = "0"
res = []
for nsm, ring in ((3, 16), (3, 8), (4, 4), (4, 5), (4, 6), (2, 16), (1, 16), (0, 16), (3, 6)):
    os.environ["SOM_TIER_NSM"] = str(nsm)
    os.environ["SOM_TIER_RING"] = str(ring)
    m.set_weights(W0)
    try:
        som.som_train_online_csr(m.h, rp, ci, va, n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, 0, steps, None)
        ms, units, _ = som.som_last_stats(m.h)
        r = {"nsm": nsm, "ring": ring, "us_per_step": round(1000 * ms / units, 3),
             "kernel": som.som_last_train_config(m.h)[1]}
    except Exception as e:
        r = {"nsm": nsm, "ring": ring, "error": str(e)[:120]}
    print(json.dumps(r), flush=True)
    res.append(r)
