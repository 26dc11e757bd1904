"""c3 full schedule in segments, kernel 10 (train_tier.cu) vs kernel 4
(train_csr.cu): per-segment us/step and the BMU logs / final weights of the
two runs compared.

  python tools/prof_tier.py [segment=25000] [max_steps=0 (full T)]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_09598_b200 import som  # noqa: E402
from synth import CONFIGS, bank_corpus  # noqa: E402

seg = int(sys.argv[1]) if len(sys.argv) > 1 else 25000
max_steps = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = CONFIGS["c3"]
n, d = cfg["n"], cfg["d"]
T = cfg["epochs"] * n
T_run = min(T, max_steps) if max_steps else T
C = bank_corpus(n, d, seed=301)
rp, ci, va = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))


def run(tier):
    os.environ["SOM_TRAIN_TIER"] = tier
    m = som.SOM(cfg["rows"], cfg["cols"], d, cfg["topo"])
    som.som_init_random_csr(m.h, rp, ci, va, n, 1301)
    log = torch.empty(T_run, dtype=torch.int32, device="cuda")
    out = []
    for t0 in range(0, T_run, seg):
        t1 = min(T_run, t0 + seg)
        som.som_train_online_csr(m.h, rp, ci, va, n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, t0, t1, log[t0:t1])
        ms, _, _ = som.som_last_stats(m.h)
        g, k = som.som_last_train_config(m.h)
        out.append((t0, t1, ms, k))
    W = m.get_weights()
    m.close()
    return out, log.cpu().numpy(), W


res = {"steps": T_run, "segment": seg}
runs = {}
for tier in ("1", "0"):
    segs, log, W = run(tier)
    runs[tier] = (log, W)
    res[f"tier{tier}"] = {"total_s": sum(s[2] for s in segs) / 1000, "kernel": segs[0][3],
                          "us_per_step": [round(1000 * s[2] / (s[1] - s[0]), 3) for s in segs]}
    print(f"SOM_TRAIN_TIER={tier}: kernel {segs[0][3]}, total {res[f'tier{tier}']['total_s']:.3f} s", flush=True)
    print("  us/step per segment:", res[f"tier{tier}"]["us_per_step"], flush=True)
l1, W1 = runs["1"]
l0, W0 = runs["0"]
res["bmu_logs_equal"] = bool(np.array_equal(l1, l0))
res["first_diff"] = int(np.flatnonzero(l1 != l0)[0]) if not res["bmu_logs_equal"] else -1
res["w_max_abs_diff"] = float(np.abs(W1.astype(np.float64) - W0).max())
res["w_bit_identical"] = bool(np.array_equal(W1, W0))
print(json.dumps({k: v for k, v in res.items() if not k.startswith("tier")}))
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/prof_tier.json", "w") as f:
    json.dump(res, f, indent=1)
