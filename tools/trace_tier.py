"""Phase breakdown of kernel 10 (train_tier.cu) via som_set_trace.
python tools/trace_tier.py [t_begin=450000] [steps=2000] [tier=1]
Trains [0, t_begin) untraced, then traces `steps` steps (globaltimer ns)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_09598_b200 import som  # noqa: E402
from synth import CONFIGS, bank_corpus  # noqa: E402

tb = int(sys.argv[1]) if len(sys.argv) > 1 else 450000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
os.environ["SOM_TRAIN_TIER"] = sys.argv[3] if len(sys.argv) > 3 else "1"
cfg = dict(CONFIGS["c3"])
n, d = cfg["n"], cfg["d"]
C = bank_corpus(n, d, seed=301)
rp, ci, va = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))
m = som.SOM(cfg["rows"], cfg["cols"], d, cfg["topo"])
som.som_init_random_csr(m.h, rp, ci, va, n, 1301)
if tb > 0:
    som.som_train_online_csr(m.h, rp, ci, va, n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, 0, tb, None)
tr = torch.zeros(148 * steps * 8, dtype=torch.int64, device="cuda")
som.som_set_trace(m.h, tr, steps)
som.som_train_online_csr(m.h, rp, ci, va, n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, tb, tb + steps, None)
ms, units, _ = som.som_last_stats(m.h)
G, k = som.som_last_train_config(m.h)
t = tr.view(148, steps, 8)[:G].cpu().numpy().astype(np.float64)[:, 50:]
print(f"t=[{tb},{tb + steps}) G={G} kernel={k}: {1000 * ms / units:.3f} us/step (event)")
if k == 10:
    seg = [("top -> dense pass done", 0, 1), ("dense -> sparse sums done", 1, 2), ("sparse -> keys (barrier A)", 2, 3),
           ("keys -> winner (exchange)", 3, 4), ("A -> bitmap+cache (2')", 3, 5), ("cache -> onchip spec", 5, 6),
           ("onchip spec -> 2' done", 6, 7)]
else:
    seg = [(f"[{i}] -> [{i + 1}]", i, i + 1) for i in range(6)]
for name, i, j in seg:
    dd = t[:, :, j] - t[:, :, i]
    med = np.median(dd, axis=1)
    print(f"  {name:28s} median over CTAs {np.median(med):7.0f} ns  min {med.min():7.0f}  max {med.max():7.0f}"
          f"   per-step max over CTAs: median {np.median(dd.max(0)):7.0f}  p90 {np.percentile(dd.max(0), 90):7.0f}")
top = t[:, :, 0]
print(f"  loop-top spread per step: median {np.median(top.max(0) - top.min(0)):.0f} ns")
loop = np.diff(t[:, :, 0], axis=1)
print(f"  loop period median {np.median(loop):.0f} ns")
pub = t[:, :, 3]
print(f"  publish spread per step: median {np.median(pub.max(0) - pub.min(0)):.0f} ns")
