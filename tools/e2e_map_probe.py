import time, sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_1905_09598_b200 import som
from synth import bank_corpus
n, d, N = 200000, 20000, 10000
C = bank_corpus(n, d, seed=501)
W = (0.5 * bank_corpus(N, d, seed=502).dense() + 0.5 / np.sqrt(d)).astype(np.float32)
m = som.SOM(100, 100, d, 1); m.set_weights(W)
drp, dci, dva = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))
hrp, hci, hva = (torch.from_numpy(a).pin_memory() for a in (C.indptr, C.indices, C.data))
db1 = torch.empty(n, dtype=torch.int32, device='cuda'); db2 = torch.empty_like(db1); dd1 = torch.empty(n, dtype=torch.float32, device='cuda')
hb1 = torch.empty(n, dtype=torch.int32).pin_memory(); hb2 = torch.empty_like(hb1).pin_memory(); hd1 = torch.empty(n, dtype=torch.float32).pin_memory()
for label, args in (("device in/out", (drp, dci, dva, n, db1, db2, dd1)), ("host in, device out", (hrp, hci, hva, n, db1, db2, dd1)),
                    ("device in, host out", (drp, dci, dva, n, hb1, hb2, hd1)), ("host in/out", (hrp, hci, hva, n, hb1, hb2, hd1))):
    for r in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        som.som_map_csr(m.h, *args)
        dt = time.perf_counter() - t0
        ms, _, _ = som.som_last_stats(m.h)
    print(f"{label}: wall {dt*1e3:.1f} ms, device {ms:.1f} ms")
