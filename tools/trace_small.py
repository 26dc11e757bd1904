"""Phase breakdown of the short-row training kernel (train_small.cu) via
som_set_trace on a Table 3 map: python tools/trace_small.py side [grid] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_09598_b200 import som  # noqa: E402
from synth import uniform_matrix  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 256
grid = int(sys.argv[2]) if len(sys.argv) > 2 else 0
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
X = torch.from_numpy(uniform_matrix(10000, 64, 64)).cuda()
W0 = torch.from_numpy(uniform_matrix(side * side, 64, side)).cuda()
m = som.SOM(side, side, 64, 1)
som.som_set_train_grid(m.h, grid)
tr = torch.zeros(148 * steps * 8, dtype=torch.int64, device="cuda")
som.som_set_trace(m.h, tr, steps)
m.set_weights(W0)
som.som_train_online(m.h, X, 10000, 2, 0.1, side / 2.0, None, 1, 0, steps, None)
ms, units, _ = som.som_last_stats(m.h)
G, k = som.som_last_train_config(m.h)
t = tr.view(148, steps, 8)[:G].cpu().numpy().astype(np.float64)[:, 100:]
print(f"{side}x{side} d=64 G={G} kernel={k}: {1000 * ms / units:.3f} us/step (event)")
names = {(0, 1): "fused pass", (1, 2): "barrier A", (2, 3): "CTA key+publish", (3, 4): "poll (exchange)",
         (2, 5): "tables+x64 (warps 1-15)", (4, 6): "winner -> barrier B", (0, 6): "whole step"}
for (i, j), nm in names.items():
    dd = np.median(t[:, :, j] - t[:, :, i], axis=1)
    print(f"  {nm:26s} median over CTAs {np.median(dd):7.0f} ns  min {dd.min():7.0f}  max {dd.max():7.0f}")
pub = t[:, :, 3]
top = t[:, :, 0]
win = t[:, :, 4]
print(f"  loop-top spread per step: median {np.median(top.max(0) - top.min(0)):.0f} ns")
print(f"  publish spread per step: median {np.median(pub.max(0) - pub.min(0)):.0f} ns, "
      f"p90 {np.percentile(pub.max(0) - pub.min(0), 90):.0f}")
print(f"  last publish -> first winner known: median {np.median(win.min(0) - pub.max(0)):.0f} ns")
late = np.bincount(np.argmax(pub, axis=0), minlength=G)
print("  most often last to publish:", [(int(c), int(late[c])) for c in np.argsort(-late)[:6]])
raw = tr.view(148, steps, 8)[0, 100:105].cpu().numpy()
print("  CTA 0 raw phases (ns from loop top):", [(r - r[0]).tolist() for r in raw[:2]])
