"""Reproduce the sharded-test conditions step by step (one GPU, 2 ranks)."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1905_09598_b200 import som  # noqa: E402
from paper_1905_09598_b200.dist import ShardedSOM  # noqa: E402
from synth import bank_corpus, init_rows  # noqa: E402

variant = sys.argv[1]
P = 2
X = bank_corpus(300, 512, seed=41).dense()
W0 = init_rows(X, 144, 41)
ranks = [ShardedSOM(12, 12, 512, 1, r, P, device=0, defer_peers=True) for r in range(P)]
boxes = [s.mailbox_ptr() for s in ranks]
for s in ranks:
    s.set_peers(boxes)
    som.som_set_train_grid(s.h, 16)
    s.set_weights(W0)
ranges = [(0, 700), (700, 1200)] if "two" in variant else [(0, 700)]
bar = threading.Barrier(P)
res = [[] for _ in range(P)]


def work(r):
    for tb, te in ranges:
        log = None
        if "log" in variant:
            log = np.empty(te - tb, np.int32)
        if "log1" in variant and tb > 0:
            log = None
        if "log2" in variant and tb == 0:
            log = None
        if "dlog" in variant:
            import torch
            log = torch.empty(te - tb, dtype=torch.int32, device="cuda")
        if "bar" in variant:
            bar.wait()
        t0 = time.time()
        try:
            som.som_train_online(ranks[r].h, X, 300, 4, 0.1, 6.0, None, 5, tb, te, log)
            res[r].append(("ok", round(time.time() - t0, 4)))
        except Exception as e:
            res[r].append((str(e)[:40], round(time.time() - t0, 4)))
        if "bar" in variant:
            bar.wait()


th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
[t.start() for t in th]
[t.join() for t in th]
print(variant, res, flush=True)
