"""Phase breakdown of the CSR training kernel (train_csr.cu) via som_set_trace.
python tools/trace_csr.py [cfg=c3] [t_begin] [steps] [grid]
Trains [0, t_begin) untraced (to reach that point of the schedule), then
traces `steps` steps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_09598_b200 import som  # noqa: E402
from synth import CONFIGS, bank_corpus  # noqa: E402

cfg = dict(CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"])
tb = int(sys.argv[2]) if len(sys.argv) > 2 else 450000
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3000
grid = int(sys.argv[4]) if len(sys.argv) > 4 else 0
n, d = cfg["n"], cfg["d"]
C = bank_corpus(n, d, seed=301)
rp, ci, va = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))
Xd = torch.from_numpy(C.dense()).cuda()
m = som.SOM(cfg["rows"], cfg["cols"], d, cfg["topo"])
som.som_set_train_mode(m.h, 2)
som.som_set_train_grid(m.h, grid)
som.som_init_random(m.h, Xd, n, 1301)
if tb > 0:
    som.som_train_online_csr(m.h, rp, ci, va, n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, 0, tb, None)
tr = torch.zeros(148 * steps * 8, dtype=torch.int64, device="cuda")
som.som_set_trace(m.h, tr, steps)
som.som_train_online_csr(m.h, rp, ci, va, n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, tb, tb + steps, None)
ms, units, _ = som.som_last_stats(m.h)
G, k = som.som_last_train_config(m.h)
t = tr.view(148, steps, 8)[:G].cpu().numpy().astype(np.float64)[:, 100:]
names = ["dense pass", "keys", "exchange", "nbhd+ring issue", "wait barB", "scatter+C+x", "-"]
print(f"t=[{tb},{tb + steps}) G={G} kernel={k}: {1000 * ms / units:.3f} us/step (event)")
dd = np.diff(t, axis=2)
for i in range(6):
    med = np.median(dd[:, :, i], axis=1)
    print(f"  {names[i]:18s} median over CTAs {np.median(med):6.0f} ns  min {med.min():6.0f}  max {med.max():6.0f}")
loop = np.diff(t[:, :, 0], axis=1)
print(f"  loop period median {np.median(loop):.0f} ns")
pub = t[:, :, 2]
print(f"  publish spread per step: median {np.median(pub.max(0) - pub.min(0)):.0f} ns")
late = np.bincount(np.argmax(pub, axis=0), minlength=G)
print("  most often last to publish:", [(int(c), int(late[c])) for c in np.argsort(-late)[:6]])
last = np.argmax(pub, axis=0)
cols = np.arange(pub.shape[1])
print("  last publisher's phases (median over steps):")
for i in range(6):
    print(f"    {names[i]:18s} {np.median(dd[last, cols, i]):6.0f} ns   (max over CTAs, median over steps "
          f"{np.median(dd[:, :, i].max(0)):6.0f})")
top0 = t[:, :, 0]
print(f"  loop-top spread per step: median {np.median(top0.max(0) - top0.min(0)):.0f} ns; "
      f"last publisher's loop-top lag {np.median(top0[last, cols] - top0.min(0)):.0f} ns")
if k == 4:   # TMA kernel: slot 7 = neighbourhood lists done, before the ring issue
    for name, i, j in (("h + lists", 3, 7), ("ring issue", 7, 4)):
        dd7 = t[:, :, j] - t[:, :, i]
        print(f"  {name:18s} median over CTAs {np.median(np.median(dd7, axis=1)):6.0f}  "
              f"per-step max over CTAs: median {np.median(dd7.max(0)):6.0f}")
# CTAs that updated rows this step (dense pass > 600 ticks) vs the others
dp = t[:, :, 1] - t[:, :, 0]
upd = dp > 600
if upd.any():
    print(f"  steps x CTAs with a dense pass: {upd.mean() * 100:.1f} %")
    for i in range(6):
        dd6 = t[:, :, i + 1] - t[:, :, i]
        print(f"    {names[i]:18s} updating CTAs median {np.median(dd6[upd]):7.0f}   others {np.median(dd6[~upd]):7.0f}")
    if k == 4:
        for name, i, j in (("h + lists", 3, 7), ("ring issue", 7, 4)):
            dd7 = t[:, :, j] - t[:, :, i]
            print(f"    {name:18s} updating CTAs median {np.median(dd7[upd]):7.0f}   others {np.median(dd7[~upd]):7.0f}")
