"""Run the tensor-core mapping on a c3-like CSR workload (for ncu / timing):
python tools/prof_map.py [docs] [units_side] [terms] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_09598_b200 import som  # noqa: E402
from synth import bank_corpus  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
side = int(sys.argv[2]) if len(sys.argv) > 2 else 50
d = int(sys.argv[3]) if len(sys.argv) > 3 else 10000
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
C = bank_corpus(n, d, seed=33)
W = (0.5 * bank_corpus(side * side, d, seed=34).dense() + 0.5 / np.sqrt(d)).astype(np.float32)
m = som.SOM(side, side, d, 1)
m.set_weights(W)
som.som_set_map_precision(m.h, som.SOM_MAP_3XTF32)
rp = torch.from_numpy(C.indptr).cuda()
ci = torch.from_numpy(C.indices).cuda()
va = torch.from_numpy(C.data).cuda()
b1 = torch.empty(n, dtype=torch.int32, device="cuda")
b2 = torch.empty(n, dtype=torch.int32, device="cuda")
d1 = torch.empty(n, dtype=torch.float32, device="cuda")
for r in range(reps):
    som.som_map_csr(m.h, rp, ci, va, n, b1, b2, d1)
    ms, units, launches = som.som_last_stats(m.h)
    nf = som.som_last_map_fallbacks(m.h)
    flop = 2.0 * n * side * side * d
    print(f"[fallbacks {nf}] rep {r}: {n} docs x {side * side} units x {d} terms: {ms:.3f} ms, {n / ms * 1e3:.0f} docs/s, "
          f"{flop / ms / 1e9:.1f} algorithmic TFLOP/s ({3 * flop / ms / 1e9:.1f} executed tf32), {launches} launches")
