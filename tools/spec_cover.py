import os, sys
sys.path.insert(0, '/root/repo')
import torch
from paper_1905_09598_b200 import som
from synth import CONFIGS, bank_corpus, init_rows
cfg = dict(CONFIGS["c2"])
C = bank_corpus(cfg["n"], cfg["d"], seed=1)
X = torch.from_numpy(C.dense()).cuda()
W0 = torch.from_numpy(init_rows(C.dense(), 400, 1001)).cuda()
T = cfg["n"] * cfg["epochs"]
for cov in sys.argv[1:]:
    if cov == "k2": os.environ["SOM_TRAIN_SPEC"] = "0"
    else: os.environ.pop("SOM_TRAIN_SPEC", None); os.environ["SOM_SPEC_COVER"] = cov
    m = som.SOM(20, 20, 3000, 1)
    best = 1e9
    for _ in range(2):
        m.set_weights(W0)
        som.som_train_online(m.h, X, cfg["n"], cfg["epochs"], 0.1, cfg["sigma0"], None, 1, 0, T, None)
        ms, units, l = som.som_last_stats(m.h)
        best = min(best, ms)
    print(cov, f"{1000*best/T:.3f} us/step, launches {l}, kernel {som.som_last_train_config(m.h)[1]}", flush=True)
    m.close()
