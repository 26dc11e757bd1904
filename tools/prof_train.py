"""Run only the training kernel on a config (for ncu): python tools/prof_train.py c2 [epochs]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_09598_b200 import som  # noqa: E402
from synth import CONFIGS, bank_corpus, init_rows  # noqa: E402

cfg = dict(CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
limit = int(sys.argv[3]) if len(sys.argv) > 3 else -1
C = bank_corpus(cfg["n"], cfg["d"], seed=1)
X = torch.from_numpy(C.dense()).cuda()
W0 = torch.from_numpy(init_rows(C.dense(), cfg["rows"] * cfg["cols"], 1001)).cuda()
m = som.SOM(cfg["rows"], cfg["cols"], cfg["d"], cfg["topo"])
for rep in range(2):
    m.set_weights(W0)
    som.som_train_online(m.h, X, cfg["n"], epochs, 0.1, cfg["sigma0"], None, 1, 0, limit, None)
    ms, units, _ = som.som_last_stats(m.h)
    print(f"rep {rep}: {units} steps in {ms:.3f} ms = {1000 * ms / units:.3f} us/step")
