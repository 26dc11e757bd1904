"""c4-shaped training window on one GPU (100 x 100 hex, 20,000 terms, W =
800 MB), CSR input, from the same weights: us/step and the kernel under the
current environment (SOM_DENSE_COVER: 0 = kernel 4, 1e-4 = kernel 3).
The schedule position is tau = t / T with T = 2 n.

  python tools/c4_window.py tau0 [steps=200] [n=4000]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_09598_b200 import som  # noqa: E402
from synth import bank_corpus, init_rows  # noqa: E402

tau0 = float(sys.argv[1])
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4000
C = bank_corpus(n, 20000, seed=44)
W0 = torch.from_numpy((0.5 * init_rows(bank_corpus(10000, 20000, seed=45).dense(), 10000, 1)
                       + 0.5 * C.dense().mean(0)).astype(np.float32)).cuda()
rp, ci, va = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))
m = som.SOM(100, 100, 20000, 1)
t0 = int(tau0 * 2 * n)
best = 1e30
for rep in range(2):
    m.set_weights(W0)
    som.som_train_online_csr(m.h, rp, ci, va, n, 2, 0.1, 50.0, None, 1, t0, t0 + steps, None)
    ms, units, _ = som.som_last_stats(m.h)
    best = min(best, ms)
g, k = som.som_last_train_config(m.h)
print(f"c4 tau {tau0:.3f} [{t0}, {t0 + steps}) kernel {k} G {g}: {1000 * best / steps:.1f} us/step", flush=True)
