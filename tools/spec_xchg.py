import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_1905_09598_b200 import som
from synth import CONFIGS, bank_corpus, init_rows
cfg = dict(CONFIGS["c2"]); steps = 3000; tb = int(sys.argv[1]) if len(sys.argv) > 1 else 250000
C = bank_corpus(cfg["n"], cfg["d"], seed=1)
X = torch.from_numpy(C.dense()).cuda()
W0 = torch.from_numpy(init_rows(C.dense(), cfg["rows"] * cfg["cols"], 1001)).cuda()
m = som.SOM(cfg["rows"], cfg["cols"], cfg["d"], cfg["topo"])
tr = torch.zeros(148 * steps * 8, dtype=torch.int64, device="cuda")
som.som_set_trace(m.h, tr, steps)
m.set_weights(W0)
som.som_train_online(m.h, X, cfg["n"], cfg["epochs"], 0.1, cfg["sigma0"], None, 1, tb, tb + steps, None)
G, k = som.som_last_train_config(m.h)
t = tr.view(148, steps, 8)[:G].cpu().numpy().astype(np.int64)[:, 200:]
t = t.astype(np.int64)
if k == 6:
    pub, known = t[:, :, 1], t[:, :, 2]
    print("kernel 6 (globaltimer ns)")
else:
    pub, known = t[:, :, 3], t[:, :, 4]
    print("kernel 2 (globaltimer ns)")
if k == 6:
    print(" poll iterations median", np.median(t[:, :, 4] - 0), "(raw)")
    first = t[:, :, 5]; det = t[:, :, 6]
    print(" publish -> first poll fail (own CTA) median", np.median(first - pub))
    print(" last publish -> first detection median", np.median(det.min(0) - pub.max(0)))
    print(" detection -> known (h) median", np.median(known - det))
per = np.diff(known.min(0))
print(" step period (ns) median", np.median(per))
print(" publish spread (max-min over CTAs) median", np.median(pub.max(0) - pub.min(0)))
print(" last publish -> first known median", np.median(known.min(0) - pub.max(0)))
print(" known spread median", np.median(known.max(0) - known.min(0)))
late = np.argmax(pub, axis=0)
cnt = np.bincount(late, minlength=G); top = np.argsort(-cnt)[:6]
print(" latest publisher:", [(int(c), int(cnt[c])) for c in top])
# which phase makes the latest publisher late: its known(t-1) vs others
kp = known[:, :-1]; pp = pub[:, 1:]
d = pp - kp   # known(t-1) -> publish(t) per CTA
print(" known(t-1)->publish(t) median per CTA: min %.0f med %.0f max %.0f" % tuple(np.percentile(np.median(d, axis=1), [0, 50, 100])))
