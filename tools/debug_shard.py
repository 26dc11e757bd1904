"""Do two same-device sharded ranks' training kernels overlap?  Prints kernel
start/end (globaltimer, from the phase trace) per rank."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_09598_b200 import som  # noqa: E402
from paper_1905_09598_b200.dist import ShardedSOM  # noqa: E402
from synth import bank_corpus, init_rows  # noqa: E402

print("concurrentKernels", torch.cuda.get_device_properties(0).multi_processor_count)
P, G = 2, int(sys.argv[1]) if len(sys.argv) > 1 else 4
X = bank_corpus(300, 512, seed=41).dense()
W0 = init_rows(X, 144, 41)
ranks = [ShardedSOM(12, 12, 512, 1, r, P, device=0, defer_peers=True) for r in range(P)]
boxes = [s.mailbox_ptr() for s in ranks]
print("mailboxes", [hex(b) for b in boxes])
trs = []
for s in ranks:
    s.set_peers(boxes)
    som.som_set_train_grid(s.h, G)
    som.som_set_train_mode(s.h, som.SOM_TRAIN_W_REGISTERS)
    s.set_weights(W0)
    tr = torch.zeros(148 * 50 * 8, dtype=torch.int64, device="cuda")
    som.som_set_trace(s.h, tr, 50)
    trs.append(tr)
res = [None] * P
t0 = time.time()


def work(r):
    try:
        som.som_train_online(ranks[r].h, X, 300, 4, 0.1, 6.0, None, 5, 0, int(sys.argv[2]) if len(sys.argv) > 2 else 50, None)
        res[r] = ("ok", time.time() - t0)
    except Exception as e:
        res[r] = (str(e), time.time() - t0)


th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
[t.start() for t in th]
[t.join() for t in th]
print(res)
for r in range(P):
    t = trs[r].view(148, 50, 8)[:G].cpu().numpy()
    print(f"rank {r}: first loop-top {t[:, 0, 0].min()} last {t[:, :, 0].max()} "
          f"steps traced {np.count_nonzero(t[0, :, 0])} winner-known t0 {t[0, 0, 4]}")
