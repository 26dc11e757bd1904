"""One c3 training window with the library named by SOM_LIB (A/B of two builds
on one box): us/step, kernel, and hashes of the BMU log and the final weights
(equal hashes = bit-identical results).

  SOM_LIB=ab/libsom_X.so python tools/lib_ab.py [t0=0] [steps=3000] [reps=2]"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_09598_b200 import som  # noqa: E402
from synth import CONFIGS, bank_corpus  # noqa: E402

t0 = int(sys.argv[1]) if len(sys.argv) > 1 else 0
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = CONFIGS["c3"]
n, d = cfg["n"], cfg["d"]
C = bank_corpus(n, d, seed=301)
rp, ci, va = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))
m = som.SOM(cfg["rows"], cfg["cols"], d, cfg["topo"])
som.som_init_random_csr(m.h, rp, ci, va, n, 1301)
W0 = torch.empty(cfg["rows"] * cfg["cols"], d, device="cuda")
som.som_get_weights(m.h, W0)
best = 1e30
for _ in range(reps):
    m.set_weights(W0)
    log = torch.empty(steps, dtype=torch.int32, device="cuda")
    som.som_train_online_csr(m.h, rp, ci, va, n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, t0, t0 + steps, log)
    ms, _, _ = som.som_last_stats(m.h)
    best = min(best, ms)
g, k = som.som_last_train_config(m.h)
W = torch.empty_like(W0)
som.som_get_weights(m.h, W)
hl = hashlib.sha1(log.cpu().numpy().tobytes()).hexdigest()[:10]
hw = hashlib.sha1(W.cpu().numpy().tobytes()).hexdigest()[:10]
print(f"{os.path.basename(os.environ.get('SOM_LIB', 'libsom.so'))} c3 [{t0}, {t0 + steps}) kernel {k} G {g}: "
      f"{1000 * best / steps:.3f} us/step  log {hl}  W {hw}", flush=True)
