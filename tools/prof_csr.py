"""Dense global-W training vs CSR training with the sparse distance path over
a full schedule, in segments: per-segment us/step, mean updated units, and a
BMU-log / weight comparison of the two runs.

  python tools/prof_csr.py [cfg=c3] [segment=20000] [max_steps=0 (full T)]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_09598_b200 import som  # noqa: E402
from synth import CONFIGS, bank_corpus  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c3"
seg = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
max_steps = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cfg = CONFIGS[cfg_name]
n, d, rows, cols, topo = cfg["n"], cfg["d"], cfg["rows"], cfg["cols"], cfg["topo"]
T = cfg["epochs"] * n
T_run = min(T, max_steps) if max_steps else T
C = bank_corpus(n, d, seed=301)
rp, ci, va = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))
Xd = torch.from_numpy(C.dense()).cuda()


def run(csr):
    m = som.SOM(rows, cols, d, topo)
    som.som_set_train_mode(m.h, 2)
    som.som_init_random(m.h, Xd, n, 1301)
    log = torch.empty(T_run, dtype=torch.int32, device="cuda")
    out = []
    for t0 in range(0, T_run, seg):
        t1 = min(T_run, t0 + seg)
        lg = log[t0:t1]
        if csr:
            som.som_train_online_csr(m.h, rp, ci, va, n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, t0, t1, lg)
        else:
            som.som_train_online(m.h, Xd, n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, t0, t1, lg)
        ms, _, _ = som.som_last_stats(m.h)
        g, k = som.som_last_train_config(m.h)
        out.append((t0, t1, ms, g, k))
    W = m.get_weights()
    m.close()
    return out, log.cpu().numpy(), W


dense, log_d, W_d = run(False)
sparse, log_s, W_s = run(True)
tot_d = sum(r[2] for r in dense)
tot_s = sum(r[2] for r in sparse)
rows_out = []
for a, b in zip(dense, sparse):
    rows_out.append({"t0": a[0], "t1": a[1], "dense_us": 1000 * a[2] / (a[1] - a[0]),
                     "csr_us": 1000 * b[2] / (b[1] - b[0]), "kernels": [a[4], b[4]], "grid": [a[3], b[3]]})
res = {"cfg": cfg_name, "steps": T_run, "T": T, "dense_s": tot_d / 1000, "csr_s": tot_s / 1000,
       "speedup": tot_d / tot_s, "bmu_logs_equal": bool(np.array_equal(log_d, log_s)),
       "first_diff": int(np.flatnonzero(log_d != log_s)[0]) if not np.array_equal(log_d, log_s) else -1,
       "w_max_abs_diff": float(np.abs(W_d.astype(np.float64) - W_s).max()), "segments": rows_out}
for r in rows_out:
    print(f"[{r['t0']:>7}, {r['t1']:>7})  dense {r['dense_us']:7.2f} us/step   csr {r['csr_us']:7.2f} us/step")
print(json.dumps({k: v for k, v in res.items() if k != "segments"}))
os.makedirs("gpurun_out", exist_ok=True)
with open(f"gpurun_out/prof_csr_{cfg_name}.json", "w") as f:
    json.dump(res, f, indent=1)
