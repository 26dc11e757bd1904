"""us/step of kernel 2 (G auto) and kernel 6 (G = 100) over windows of the
c2 schedule, each window started from the same weights (the step cost
depends on t through the neighbourhood radius).
python tools/spec_windows.py [window]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_09598_b200 import som  # noqa: E402
from synth import CONFIGS, bank_corpus, init_rows  # noqa: E402

cfg = dict(CONFIGS["c2"])
win = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
C = bank_corpus(cfg["n"], cfg["d"], seed=1)
X = torch.from_numpy(C.dense()).cuda()
W0 = torch.from_numpy(init_rows(C.dense(), cfg["rows"] * cfg["cols"], 1001)).cuda()
T = cfg["n"] * cfg["epochs"]
for tb in range(0, T, 50000):
    row = []
    for spec, grid in (("0", 0), ("1", 100)):
        os.environ["SOM_TRAIN_SPEC"] = spec
        m = som.SOM(cfg["rows"], cfg["cols"], cfg["d"], cfg["topo"])
        som.som_set_train_grid(m.h, grid)
        best = 1e9
        for _ in range(2):
            m.set_weights(W0)
            som.som_train_online(m.h, X, cfg["n"], cfg["epochs"], 0.1, cfg["sigma0"], None, 1, tb, tb + win, None)
            ms, units, _ = som.som_last_stats(m.h)
            best = min(best, 1000 * ms / units)
        row.append(best)
        m.close()
    print(f"t in [{tb}, {tb + win}): kernel 2 {row[0]:.3f}  kernel 6 {row[1]:.3f} us/step", flush=True)
