"""c4-shaped training on one GPU (100x100 hex map, 20k terms, W = 800 MB in
HBM), for timing / ncu: python tools/prof_c4.py [steps] [csr 0/1] [docs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_09598_b200 import som  # noqa: E402
from synth import bank_corpus, init_rows  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
csr = len(sys.argv) > 2 and sys.argv[2] == "1"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4000
C = bank_corpus(n, 20000, seed=44)
X = torch.from_numpy(C.dense()).cuda()
W0 = torch.from_numpy((0.5 * init_rows(bank_corpus(10000, 20000, seed=45).dense(), 10000, 1)
                       + 0.5 * C.dense().mean(0)).astype(np.float32)).cuda()
rp, ci, va = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))
m = som.SOM(100, 100, 20000, 1)
for rep in range(2):
    m.set_weights(W0)
    if csr:
        som.som_train_online_csr(m.h, rp, ci, va, n, 2, 0.1, 50.0, None, 1, 0, steps, None)
    else:
        som.som_train_online(m.h, X, n, 2, 0.1, 50.0, None, 1, 0, steps, None)
    ms, units, _ = som.som_last_stats(m.h)
    g, k = som.som_last_train_config(m.h)
    gb = (4.0 * 10000 * 20000 * 2) / 1e9
    print(f"rep {rep}: kernel {k} G={g}: {units} steps in {ms:.3f} ms = {1000 * ms / units:.1f} us/step "
          f"(~{gb * units / ms:.0f} GB/s if every unit is updated)")
