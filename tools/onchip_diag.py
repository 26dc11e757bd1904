"""Kernel 9 (train_onchip.cu) vs kernel 4 (train_csr.cu) on the real c3 corpus:
from one weight snapshot at step t_a, run windows of K steps with each kernel
and compare BMU logs and weights bit for bit; report the differing units by
storage class (TMEM / shared-memory / streamed row) of kernel 9's placement.
Also times both kernels per segment of the schedule.

  python tools/onchip_diag.py [t_a=450000] [seg=25000]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_09598_b200 import som  # noqa: E402
from synth import CONFIGS, bank_corpus  # noqa: E402

t_a = int(sys.argv[1]) if len(sys.argv) > 1 else 450000
seg = int(sys.argv[2]) if len(sys.argv) > 2 else 25000
cfg = CONFIGS["c3"]
n, d, rows, cols, topo = cfg["n"], cfg["d"], cfg["rows"], cfg["cols"], cfg["topo"]
T = cfg["epochs"] * n
C = bank_corpus(n, d, seed=301)
rp, ci, va = (torch.from_numpy(a).cuda() for a in (C.indptr, C.indices, C.data))
N = rows * cols


def unit_tab(G, NL):
    """port of build_unit_tab (som_train_api.cu) for rank 0 of 1"""
    S = (NL + G - 1) // G
    best_alpha, best_len = cols % G, -1.0
    for al in range(1, G):
        mn = 1e300
        for di in range(0, min(rows, 65)):
            dj0 = ((-al * di) % G + G) % G
            for dj in (dj0, dj0 - G):
                if di == 0 and dj == 0:
                    continue
                if dj >= cols or -dj >= cols:
                    continue
                ln = di * di + dj * dj if topo == 0 else dj * dj + 0.75 * di * di
                mn = min(mn, ln)
        if mn > best_len:
            best_len, best_alpha = mn, al
    cnt = [0] * G
    where = {}
    for l in range(NL):
        i, j = divmod(l, cols)
        k = (best_alpha * i + j) % G
        while cnt[k] >= S:
            k = (k + 1) % G
        where[l] = (k, cnt[k])
        cnt[k] += 1
    return where


def set_kernel(k9):
    os.environ["SOM_TRAIN_ONCHIP"] = "1" if k9 else "0"


def train(m, t0, t1, log=None):
    som.som_train_online_csr(m.h, rp, ci, va, n, cfg["epochs"], 0.1, cfg["sigma0"], None, 1, t0, t1, log)
    ms, _, _ = som.som_last_stats(m.h)
    return ms, som.som_last_train_config(m.h)


out = {"t_a": t_a}
m = som.SOM(rows, cols, d, topo)
som.som_init_random_csr(m.h, rp, ci, va, n, 1301)
W0 = m.get_weights()

# per-segment timing of both kernels over the schedule (independent runs)
seg_rows = []
for k9 in (False, True):
    set_kernel(k9)
    m.set_weights(W0)
    for s0 in range(0, T, seg):
        ms, (g, k) = train(m, s0, min(T, s0 + seg))
        seg_rows.append({"kernel": k, "t0": s0, "us": 1000 * ms / (min(T, s0 + seg) - s0)})
        if k9 and s0 == 0:
            print(f"kernel {k} grid {g}: first segment {seg_rows[-1]['us']:.2f} us/step", flush=True)
    out[f"total_s_k{k}"] = sum(r["us"] * seg for r in seg_rows if r["kernel"] == k) / 1e6
for r in seg_rows:
    print(f"k{r['kernel']} [{r['t0']:>7}) {r['us']:7.2f} us/step")
out["segments"] = seg_rows

# snapshot at t_a with kernel 4
set_kernel(False)
m.set_weights(W0)
train(m, 0, t_a)
Wa = m.get_weights()
G = 148
where = unit_tab(G, N)
ntm, nsm = 5, 4   # train_onchip_plan at d = 10000, S = 17 (see DESIGN.md kernel 9)
res = []
for K in (1, 2, 3, 5, 10, 100):
    W = {}
    L = {}
    for k9 in (False, True):
        set_kernel(k9)
        m.set_weights(Wa)
        log = torch.empty(K, dtype=torch.int32, device="cuda")
        _, (g, k) = train(m, t_a, t_a + K, log)
        W[k9], L[k9] = m.get_weights(), log.cpu().numpy()
    diff = np.abs(W[True].astype(np.float64) - W[False]).max(axis=1)
    bad = np.flatnonzero(diff > 0)
    cls = {}
    for u in bad:
        b, s = where[int(u)]
        c = "tmem" if s < ntm else "smem" if s < ntm + nsm else "global"
        cls[c] = cls.get(c, 0) + 1
    r = {"K": K, "logs_equal": bool(np.array_equal(L[True], L[False])), "units_differing": int(bad.size),
         "max_abs": float(diff.max()), "by_class": cls,
         "bad_units_first": [(int(u), where[int(u)]) for u in bad[:12]],
         "last_bmus": L[False][-3:].tolist()}
    print(json.dumps(r), flush=True)
    res.append(r)
out["windows"] = res
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/onchip_diag.json", "w") as f:
    json.dump(out, f, indent=1)
