"""Phase breakdown of the register-resident training kernel via som_set_trace.
python tools/trace_train.py c2 [grid] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_09598_b200 import som  # noqa: E402
from synth import CONFIGS, bank_corpus, init_rows  # noqa: E402

cfg = dict(CONFIGS[sys.argv[1]])
grid = int(sys.argv[2]) if len(sys.argv) > 2 else 0
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3000
tb = int(sys.argv[4]) if len(sys.argv) > 4 else 0
C = bank_corpus(cfg["n"], cfg["d"], seed=1)
X = torch.from_numpy(C.dense()).cuda()
W0 = torch.from_numpy(init_rows(C.dense(), cfg["rows"] * cfg["cols"], 1001)).cuda()
m = som.SOM(cfg["rows"], cfg["cols"], cfg["d"], cfg["topo"])
som.som_set_train_grid(m.h, grid)
tr = torch.zeros(148 * steps * 8, dtype=torch.int64, device="cuda")
som.som_set_trace(m.h, tr, steps)
m.set_weights(W0)
som.som_train_online(m.h, X, cfg["n"], cfg["epochs"], 0.1, cfg["sigma0"], None, 1, tb, tb + steps, None)
ms, units, _ = som.som_last_stats(m.h)
G, k = som.som_last_train_config(m.h)
t = tr.view(148, steps, 8)[:G].cpu().numpy().astype(np.float64)[:, 200:]
names = ["fused+reduce", "issue_x+barA", "w0 key", "publish+poll", "h compute", "x shift/read", "barB"]
if k == 6:   # train_spec.cu phases
    names = ["bounds+publish", "wait+h", "(pass end, thread 32)", "barA+totals", "-", "-", "-"]
print(f"{sys.argv[1]} t=[{tb},{tb + steps}) G={G} kernel={k}: {1000 * ms / units:.3f} us/step (event)")
d = np.diff(t, axis=2)                        # [G][steps][7]
for i in range(7):
    med = np.median(d[:, :, i], axis=1)       # per CTA
    print(f"  {names[i]:14s} median over CTAs {np.median(med):6.0f} ns  min {med.min():6.0f}  max {med.max():6.0f}")
if k == 6:
    ps = np.median(t[:, 1:, 3] - t[:, :-1, 4], axis=1)
    print(f"  pass (totals(t-1) -> thread 32 pass end): median {np.median(ps):.0f}  max {ps.max():.0f}")
pub = t[:, :, 3]                              # publish time per CTA per step
spread = pub.max(0) - pub.min(0)
late = np.argmax(pub, axis=0)
print(f"  publish spread per step: median {np.median(spread):.0f} ns, p90 {np.percentile(spread, 90):.0f}")
cnt = np.bincount(late, minlength=G)
top = np.argsort(-cnt)[:8]
print("  most often last to publish:", [(int(c), int(cnt[c])) for c in top])
arr_top = t[:, :, 0]                          # loop-top time per CTA
print(f"  loop-top spread per step: median {np.median(arr_top.max(0) - arr_top.min(0)):.0f} ns")
win = t[:, :, 4]
print(f"  winner-known spread: median {np.median(win.max(0) - win.min(0)):.0f} ns; "
      f"first-known minus last-publish: median {np.median(win.min(0) - pub.max(0)):.0f} ns")
sm = None
