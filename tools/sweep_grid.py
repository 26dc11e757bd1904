"""Sweep the training grid size on a config: python tools/sweep_grid.py c2 epochs G1,G2,..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1905_09598_b200 import som  # noqa: E402
from synth import CONFIGS, bank_corpus, init_rows  # noqa: E402

cfg = dict(CONFIGS[sys.argv[1]])
epochs = int(sys.argv[2])
grids = [int(g) for g in sys.argv[3].split(",")]
modes = [int(m) for m in sys.argv[4].split(",")] if len(sys.argv) > 4 else [0]
C = bank_corpus(cfg["n"], cfg["d"], seed=1)
X = torch.from_numpy(C.dense()).cuda()
W0 = torch.from_numpy(init_rows(C.dense(), cfg["rows"] * cfg["cols"], 1001)).cuda()
m = som.SOM(cfg["rows"], cfg["cols"], cfg["d"], cfg["topo"])
ref = None
for mode in modes:
    for G in grids:
        som.som_set_train_mode(m.h, mode)
        som.som_set_train_grid(m.h, G)
        print(f"-- mode {mode} grid {G}", flush=True)
        best, units = 1e30, 0
        for rep in range(2):
            m.set_weights(W0)
            try:
                som.som_train_online(m.h, X, cfg["n"], epochs, 0.1, cfg["sigma0"], None, 1, 0, -1, None)
            except som.SomError as e:
                print("   ", e)
                break
            ms, units, _ = som.som_last_stats(m.h)
            best = min(best, ms)
        if units == 0:
            continue
        g, k = som.som_last_train_config(m.h)
        Wn = torch.empty_like(W0)
        som.som_get_weights(m.h, Wn)
        same = "" if ref is None else ("same" if torch.equal(ref, Wn) else "DIFF")
        ref = Wn if ref is None else ref
        print(f"mode={mode} G={g} kernel={k}: {units} steps {best:.2f} ms = {1000 * best / units:.3f} us/step {same}",
              flush=True)
