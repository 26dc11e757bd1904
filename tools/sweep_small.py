"""Short-row kernel grid sweep on a Table 3 map: python tools/sweep_small.py side G1,G2,... [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_09598_b200 import som  # noqa: E402
from synth import uniform_matrix  # noqa: E402

side = int(sys.argv[1])
grids = [int(g) for g in sys.argv[2].split(",")]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20000
X = uniform_matrix(10000, 64, 64)
W0 = uniform_matrix(side * side, 64, side)
for G in grids:
    with som.SOM(side, side, 64, 1) as m:
        som.som_set_train_grid(m.h, G)
        m.set_weights(W0)
        m.train_online(X, epochs=2, alpha0=0.1, sigma0=side / 2.0, seed=1, t_end=steps)
        ms, units, _ = som.som_last_stats(m.h)
        g, k = som.som_last_train_config(m.h)
    print(f"{side}x{side} G={g} kernel={k}: {1000 * ms / units:.3f} us/step", flush=True)
