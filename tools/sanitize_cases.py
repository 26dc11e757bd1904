"""Tiny invocations of each training / mapping kernel for compute-sanitizer
(racecheck, synccheck, memcheck).  Host numpy buffers only (no torch), so
the sanitizer sees libsom's kernels alone.  Each case also checks its result
against the oracle (BMU log equal), so a run that "passes" the sanitizer
with a wrong answer is visible.

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py k2
  cases: k1 k2 k3 k4 k4x1 k4x2 k5 k6 k10 k10b k10w12 map_exact map_sparse map_tc map_tc2 metrics batch sharded2"""
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1905_09598_b200 import som  # noqa: E402
from synth import bank_corpus, init_rows  # noqa: E402

case = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40


def train_case(rows, cols, d, n, mode=som.SOM_TRAIN_AUTO, csr=False, env=None, grid=0, topo=1, expect=None):
    for k, v in (env or {}).items():
        os.environ[k] = v
    C = bank_corpus(n, d, seed=d + n)
    X = C.dense()
    W0 = init_rows(X, rows * cols, 5)
    sigma0 = max(rows, cols) / 2.0
    with som.SOM(rows, cols, d, topo) as m:
        som.som_set_train_mode(m.h, mode)
        if grid:
            som.som_set_train_grid(m.h, grid)
        m.set_weights(W0)
        log = np.empty(steps, np.int32)
        if csr:
            m.train_online_csr(C.indptr, C.indices, C.data, C.n, 2, alpha0=0.1, sigma0=sigma0, seed=3, t_end=steps,
                               bmu_log=log)
        else:
            m.train_online(X, 2, alpha0=0.1, sigma0=sigma0, seed=3, t_end=steps, bmu_log=log)
        g, k = som.som_last_train_config(m.h)
        W = m.get_weights()
    Wo, logo = oracle.train_online(W0, rows, cols, topo, X, 2, 0.1, sigma0, 3, t_end=steps)
    assert np.array_equal(log, logo), "BMU log differs from the oracle"
    assert np.abs(W.astype(np.float64) - Wo).max() <= 1e-4
    if expect is not None:
        assert k == expect, (k, expect)
    print(f"{case}: kernel {k} grid {g}, {steps} steps, BMU log = oracle, max|dW| "
          f"{np.abs(W.astype(np.float64) - Wo).max():.2g}")


def map_case(prec, csr):
    C = bank_corpus(300, 2048, seed=11)
    X = C.dense()
    W = init_rows(X, 16 * 16, 12)
    with som.SOM(16, 16, 2048, 1) as m:
        m.set_weights(W)
        m.set_map_precision(prec)
        b1, b2, d1 = m.map_csr(C.indptr, C.indices, C.data, C.n) if csr else m.map(X)
    ob1, ob2, od1, m12, m23 = oracle.map_docs(W, X, want_margins=True)
    ok = m12 > 1e-5
    assert np.array_equal(b1[ok], ob1[ok])
    print(f"{case}: {ok.sum()} margin docs, bmu1 = oracle")


if case == "k1":
    train_case(12, 12, 1000, 300, mode=som.SOM_TRAIN_W_SHARED, expect=1)
elif case == "k2":
    train_case(10, 10, 512, 200, mode=som.SOM_TRAIN_W_REGISTERS, expect=2)
elif case == "k3":
    train_case(16, 16, 2048, 300, mode=som.SOM_TRAIN_W_GLOBAL, env={"SOM_TRAIN_DENSE_CSR": "0"}, expect=3)
elif case == "k4":
    train_case(16, 16, 2048, 300, mode=som.SOM_TRAIN_W_GLOBAL, csr=True, expect=4)
elif case == "k5":
    train_case(16, 16, 64, 300, expect=5)
elif case == "k6":
    train_case(10, 10, 512, 200, mode=som.SOM_TRAIN_W_REGISTERS, env={"SOM_TRAIN_SPEC": "1"}, expect=6)
elif case == "k10":
    train_case(20, 20, 7600, 600, csr=True, expect=10, grid=20)
elif case == "k10b":
    train_case(20, 20, 6000, 600, csr=True, expect=10, grid=16)
elif case == "k4x1":   # kernel 4 with the atomic-max exchange (G = 100 >= 96)
    train_case(16, 16, 2048, 300, mode=som.SOM_TRAIN_W_GLOBAL, csr=True, expect=4, grid=100,
               env={"SOM_XCHG_ATOMIC": "1"})
elif case == "k4x2":   # kernel 4 with the counter-hinted all-gather (the default from 96 CTAs)
    train_case(16, 16, 2048, 300, mode=som.SOM_TRAIN_W_GLOBAL, csr=True, expect=4, grid=100)
elif case == "k10w12":   # kernel 10 with 12 data warps on a row 16 warps would take
    train_case(20, 20, 7600, 600, csr=True, expect=10, grid=20, env={"SOM_TIER_NDW": "12"})
elif case == "map_tc2":   # > 148 work items: CTAs alternate the two TMEM accumulator buffers
    C = bank_corpus(10240, 512, seed=15)
    X = C.dense()
    W = init_rows(X, 16 * 16, 16)
    with som.SOM(16, 16, 512, 1) as m:
        m.set_weights(W)
        m.set_map_precision(som.SOM_MAP_3XTF32)
        b1, b2, d1 = m.map(X)
    ob1, ob2, od1 = oracle.map_docs(W, X)
    assert np.array_equal(b1, ob1) and np.array_equal(b2, ob2)
    print(f"{case}: {C.n} docs, bmu1/bmu2 = oracle on every document")
elif case == "map_exact":
    map_case(som.SOM_MAP_EXACT_F64, False)
elif case == "map_sparse":
    map_case(som.SOM_MAP_SPARSE_F64, True)
elif case == "map_tc":
    map_case(som.SOM_MAP_3XTF32, False)
elif case == "metrics":
    C = bank_corpus(300, 512, seed=13)
    X = C.dense()
    W = init_rows(X, 100, 14)
    with som.SOM(10, 10, 512, 1) as m:
        m.set_weights(W)
        qe, te = m.errors(X)
        U = m.umatrix()
    assert abs(U - oracle.umatrix(W, 10, 10, 1)).max() <= 1e-5
    print(f"{case}: qe {qe:.6f} te {te:.4f}, U-matrix = oracle")
elif case == "batch":
    C = bank_corpus(300, 512, seed=15)
    X = C.dense()
    W0 = init_rows(X, 100, 16)
    with som.SOM(10, 10, 512, 1) as m:
        m.set_weights(W0)
        m.train_batch(X, 3, sigma0=5.0)
        W = m.get_weights()
    Wo, _ = oracle.train_batch(W0, 10, 10, 1, X, 3, 5.0)
    assert np.abs(W - Wo).max() <= 1e-5
    print(f"{case}: 3 batch epochs = oracle")
elif case == "sharded2":
    # two neuron shards on one device, each its own grid on its own thread,
    # exchanging winners through each other's mailboxes
    from paper_1905_09598_b200.dist import ShardedSOM
    C = bank_corpus(200, 512, seed=17)
    X = C.dense()
    W0 = init_rows(X, 100, 18)
    import torch
    Xd = torch.from_numpy(X).cuda()     # staged before any grid spins
    P = 2
    ranks = [ShardedSOM(10, 10, 512, 1, r, P, device=0, defer_peers=True) for r in range(P)]
    boxes = [s.mailbox_ptr() for s in ranks]
    logs = [np.empty(steps, np.int32) for _ in range(P)]
    for s in ranks:
        s.set_peers(boxes)
        som.som_set_train_grid(s.h, 4)
        s.set_weights(W0)

    def work(r):
        som.som_train_online(ranks[r].h, Xd, 200, 2, 0.1, 5.0, None, 3, 0, steps, logs[r])

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    _, logo = oracle.train_online(W0, 10, 10, 1, X, 2, 0.1, 5.0, 3, t_end=steps)
    assert all(np.array_equal(l, logo) for l in logs)
    print(f"{case}: P=2 on one device, both logs = oracle")
else:
    raise SystemExit(f"unknown case {case}")
