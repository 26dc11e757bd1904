"""A/B of the in-GPU winner exchange: tagged all-gather (SOM_XCHG_ATOMIC=0)
vs atomic max + arrival counter (SOM_XCHG_ATOMIC=1) vs tagged slots read
once a relaxed arrival counter is complete (SOM_XCHG_ATOMIC=2), same training window,
BMU logs and final weights compared bit for bit.

  python tools/xchg_ab.py c2 [t0=0] [steps=50000] [grids=0] [reps=2]
  python tools/xchg_ab.py c3 [t0] [steps]          (CSR input, AUTO kernel)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_09598_b200 import som  # noqa: E402
from synth import CONFIGS, bank_corpus, init_rows  # noqa: E402

name = sys.argv[1]
t0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 50000
grids = [int(g) for g in sys.argv[4].split(",")] if len(sys.argv) > 4 else [0]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
cfg = dict(CONFIGS[name])
n, d = cfg["n"], cfg["d"]
csr = name in ("c3", "c4")
C = bank_corpus(n, d, seed=301 if csr else 1)
m = som.SOM(cfg["rows"], cfg["cols"], d, cfg["topo"])
if csr:
    rp, ci, va = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))
    som.som_init_random_csr(m.h, rp, ci, va, n, 1301)
    W0 = torch.empty(cfg["rows"] * cfg["cols"], d, device="cuda")
    som.som_get_weights(m.h, W0)
else:
    X = torch.from_numpy(C.dense()).cuda()
    W0 = torch.from_numpy(init_rows(C.dense(), cfg["rows"] * cfg["cols"], 1001)).cuda()


def run(atomic, G):
    os.environ["SOM_XCHG_ATOMIC"] = str(atomic)
    som.som_set_train_grid(m.h, G)
    best = 1e30
    for _ in range(reps):
        m.set_weights(W0)
        log = torch.empty(steps, dtype=torch.int32, device="cuda")
        if csr:
            som.som_train_online_csr(m.h, rp, ci, va, n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, t0, t0 + steps, log)
        else:
            som.som_train_online(m.h, X, n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, t0, t0 + steps, log)
        ms, units, _ = som.som_last_stats(m.h)
        best = min(best, ms)
    g, k = som.som_last_train_config(m.h)
    Wn = torch.empty_like(W0)
    som.som_get_weights(m.h, Wn)
    return best, g, k, log.cpu().numpy(), Wn


for G in grids:
    res = {}
    for atomic in (0, 1, 2, 0, 1, 2):
        ms, g, k, log, Wn = run(atomic, G)
        if atomic in res:
            res[atomic] = (min(ms, res[atomic][0]),) + res[atomic][1:]
        else:
            res[atomic] = (ms, g, k, log, Wn)
    same = all(np.array_equal(res[0][3], res[m][3]) and torch.equal(res[0][4], res[m][4]) for m in (1, 2))
    print(f"{name} [{t0}, {t0 + steps}) G={res[0][1]} kernel={res[0][2]}: all-gather "
          f"{1000 * res[0][0] / steps:.3f} us/step, atomic {1000 * res[1][0] / steps:.3f}, "
          f"count+slots {1000 * res[2][0] / steps:.3f}, identical={same}", flush=True)
