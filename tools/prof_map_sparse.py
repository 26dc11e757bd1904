"""Time the exact sparse mapping (SOM_MAP_SPARSE_F64) on a c5-shaped CSR
sample for each unit-tile width (SOM_SPARSE_J = 1, 2, 4):
python tools/prof_map_sparse.py [docs] [units_side] [terms] [reps] [J...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_09598_b200 import som  # noqa: E402
from synth import bank_corpus  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
side = int(sys.argv[2]) if len(sys.argv) > 2 else 100
d = int(sys.argv[3]) if len(sys.argv) > 3 else 20000
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
cfgs = sys.argv[5:] or ["d4", "f2", "f4", "f8"]   # d = fp64 W^T, f = fp32; number = J (tile 64 J)
C = bank_corpus(n, d, seed=501)
W = (0.5 * bank_corpus(side * side, d, seed=502).dense() + 0.5 / np.sqrt(d)).astype(np.float32)
m = som.SOM(side, side, d, 1)
m.set_weights(W)
rp = torch.from_numpy(C.indptr).cuda()
ci = torch.from_numpy(C.indices).cuda()
va = torch.from_numpy(C.data).cuda()
b1 = torch.empty(n, dtype=torch.int32, device="cuda")
b2 = torch.empty(n, dtype=torch.int32, device="cuda")
d1 = torch.empty(n, dtype=torch.float32, device="cuda")
nnz = C.nnz
ref = None
for J in cfgs:
    os.environ["SOM_SPARSE_F32"] = "1" if J[0] == "f" else "0"
    os.environ["SOM_SPARSE_J"] = J[1:].split("/")[0]
    if "/" in J:
        os.environ["SOM_SPARSE_DPC"] = J.split("/")[1]
    som.som_set_map_precision(m.h, som.SOM_MAP_SPARSE_F64)
    for r in range(reps):
        som.som_map_csr(m.h, rp, ci, va, n, b1, b2, d1)
        ms, units, launches = som.som_last_stats(m.h)
        fma = float(nnz) * side * side
        print(f"J={J} rep {r}: {n} docs ({nnz / n:.1f} nnz) x {side * side} units x {d} terms: {ms:.3f} ms, "
              f"{n / ms * 1e3:.0f} docs/s, {fma / ms / 1e9:.2f} T fp64 FMA/s, "
              f"{(4 if J[0] == 'f' else 8) * fma / ms / 1e9:.1f} TB/s of W^T operands, {launches} launches", flush=True)
    out = (b1.cpu().numpy().copy(), d1.cpu().numpy().copy())
    if ref is None:
        ref = out
    else:
        print(f"  J={J} vs J={cfgs[0]}: bmu1 equal {np.array_equal(ref[0], out[0])}, d1 equal {np.array_equal(ref[1], out[1])}")
som.som_set_map_precision(m.h, som.SOM_MAP_3XTF32)
som.som_map_csr(m.h, rp, ci, va, n, b1, b2, d1)
ms, _, _ = som.som_last_stats(m.h)
tb1 = b1.cpu().numpy()
print(f"3xTF32 path: {ms:.3f} ms, {n / ms * 1e3:.0f} docs/s; bmu1 agreement with sparse fp64 {np.mean(tb1 == ref[0]):.6f}")
