"""A/B of the register-resident training kernels on a config: kernel 2
(train_reg.cu) vs kernel 6 (train_spec.cu, overlapped exchange).  Weights
and BMU logs must be identical; prints us/step and the fallback count.
python tools/spec_ab.py c2 [steps] [grid]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_09598_b200 import som  # noqa: E402
from synth import CONFIGS, bank_corpus, init_rows  # noqa: E402

cfg = dict(CONFIGS[sys.argv[1]])
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 0
grid = int(sys.argv[3]) if len(sys.argv) > 3 else 0
C = bank_corpus(cfg["n"], cfg["d"], seed=1)
X = torch.from_numpy(C.dense()).cuda()
W0 = torch.from_numpy(init_rows(C.dense(), cfg["rows"] * cfg["cols"], 1001)).cuda()
T = steps or cfg["n"] * cfg["epochs"]
res = {}
for spec in ("0", "1"):
    os.environ["SOM_TRAIN_SPEC"] = spec
    m = som.SOM(cfg["rows"], cfg["cols"], cfg["d"], cfg["topo"])
    som.som_set_train_grid(m.h, grid)
    out = []
    for rep in range(2):
        m.set_weights(W0)
        log = torch.empty(T, dtype=torch.int32, device="cuda")
        som.som_train_online(m.h, X, cfg["n"], cfg["epochs"], 0.1, cfg["sigma0"], None, 1, 0, T, log)
        ms, units, _ = som.som_last_stats(m.h)
        out.append(ms)
    G, k = som.som_last_train_config(m.h)
    fb = som.som_last_spec_fallbacks(m.h)
    res[spec] = (m.get_weights(), log.cpu().numpy())
    print(f"{sys.argv[1]} spec={spec} kernel={k} G={G}: {1000 * min(out) / T:.3f} us/step over {T} steps, "
          f"fallbacks {fb}", flush=True)
    m.close()
same_w = np.array_equal(res["0"][0], res["1"][0])
same_log = np.array_equal(res["0"][1], res["1"][1])
print(f"identical weights: {same_w}, identical BMU log: {same_log}")
if not same_log:
    i = int(np.argmax(res["0"][1] != res["1"][1]))
    print("first BMU mismatch at step", i, res["0"][1][i], res["1"][1][i])
