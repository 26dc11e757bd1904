"""One c3 training window for ncu / timing: init + [t0, t0 + steps) with the
kernel AUTO picks under the current environment (SOM_TRAIN_ONCHIP etc.).
A pre-window [0, t0) runs first when t0 > 0 (profile with --launch-skip).

  python tools/c3_window.py [t0=0] [steps=300] [csr=1]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_09598_b200 import som  # noqa: E402
from synth import CONFIGS, bank_corpus  # noqa: E402

t0 = int(sys.argv[1]) if len(sys.argv) > 1 else 0
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
csr = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cfg = CONFIGS["c3"]
n, d = cfg["n"], cfg["d"]
C = bank_corpus(n, d, seed=301)
rp, ci, va = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))
m = som.SOM(cfg["rows"], cfg["cols"], d, cfg["topo"])
som.som_init_random_csr(m.h, rp, ci, va, n, 1301)


def win(a, b):
    if csr:
        som.som_train_online_csr(m.h, rp, ci, va, n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, a, b, None)
    else:
        Xd = torch.from_numpy(C.dense()).cuda()
        som.som_train_online(m.h, Xd, n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, a, b, None)
    ms, units, _ = som.som_last_stats(m.h)
    g, k = som.som_last_train_config(m.h)
    return ms, g, k


if t0 > 0:
    win(0, t0)
ms, g, k = win(t0, t0 + steps)
print(f"c3 window [{t0}, {t0 + steps}): kernel {k} grid {g}: {1000 * ms / steps:.2f} us/step")
