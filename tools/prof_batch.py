"""Batch SOM epochs on the c3 shape (for ncu / timing):
python tools/prof_batch.py [epochs] [docs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_09598_b200 import som  # noqa: E402
from synth import bank_corpus, init_rows  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
C = bank_corpus(n, 10000, seed=300)
W0 = torch.from_numpy(init_rows(C.dense()[:5000], 2500, 301)).cuda()
rp, ci, va = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))
with som.SOM(50, 50, 10000, 1) as m:
    m.set_weights(W0)
    som.som_train_batch_csr(m.h, rp, ci, va, n, E, 25.0, None, None)
    ms, units, launches = som.som_last_stats(m.h)
print(f"{E} epochs x {n} docs: {ms:.2f} ms ({ms / E:.2f} ms/epoch), {launches} launches")
