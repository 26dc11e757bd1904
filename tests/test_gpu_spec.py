"""Kernel 6 (train_spec.cu, opt-in with SOM_TRAIN_SPEC=1): the register-
resident training step with the winner exchange of step t overlapped with
the distance pass of step t+1 and certified speculative distances (DESIGN.md
R32).  Its BMU log and weights must equal the oracle's, and on a c2 prefix
long enough to take the exact fallback (near-ties) they must equal kernel
2's bit for bit."""
import math

import numpy as np
import pytest

import oracle
from synth import CONFIGS, bank_corpus, init_rows

pytestmark = pytest.mark.gpu


@pytest.fixture
def som(monkeypatch):
    from paper_1905_09598_b200 import som as s
    s.lib()
    monkeypatch.setenv("SOM_TRAIN_SPEC", "1")
    return s


def _train(som, rows, cols, topo, X, W0, epochs, alpha0, sigma0, seed, t_end=-1, grid=0, kind=0, cutoff=1e-4):
    n, d = X.shape
    with som.SOM(rows, cols, d, topo) as m:
        som.som_set_train_grid(m.h, grid)
        m.set_weights(W0)
        T = epochs * n if t_end < 0 else t_end
        log = np.full(T, -7, np.int32)
        m.train_online(X, epochs=epochs, alpha0=alpha0, sigma0=sigma0, seed=seed, kind=kind, cutoff=cutoff,
                       t_end=t_end, bmu_log=log)
        G, k = som.som_last_train_config(m.h)
        fb = som.som_last_spec_fallbacks(m.h)
        return m.get_weights(), log, k, fb


@pytest.mark.parametrize("rows,cols,topo,d,n,seed,grid", [
    (10, 10, 0, 500, 200, 1, 0),      # c1
    (10, 10, 1, 500, 200, 2, 16),     # hex, 7 units per CTA
    (7, 9, 0, 132, 150, 3, 32),       # ragged: 63 units over 32 CTAs, d4 = 33 chunks
    (12, 11, 1, 4000, 120, 4, 128),   # 132 units over 128 CTAs, three chunks per pass thread
])
def test_spec_matches_oracle(som, rows, cols, topo, d, n, seed, grid):
    C = bank_corpus(n, d, seed=seed)
    X = C.dense()
    W0 = init_rows(X, rows * cols, seed + 1000)
    W, log, k, fb = _train(som, rows, cols, topo, X, W0, 10, 0.1, max(rows, cols) / 2.0, seed, grid=grid)
    assert k == 6
    Wo, logo = oracle.train_online(W0, rows, cols, topo, X, 10, 0.1, max(rows, cols) / 2.0, seed, eps=1e-4)
    assert np.array_equal(log, logo), f"first BMU mismatch at step {np.flatnonzero(log != logo)[:1]}"
    assert np.abs(W.astype(np.float64) - Wo).max() <= 1e-4
    assert np.count_nonzero(W != Wo) <= W.size // 1000


def test_spec_no_cutoff_and_decay_kind(som):
    """eps = 0 (every unit updated every step) and the exponential schedule."""
    C = bank_corpus(200, 500, seed=7)
    X = C.dense()
    W0 = init_rows(X, 100, 1007)
    W, log, k, _ = _train(som, 10, 10, 0, X, W0, 5, 0.3, 5.0, 7, kind=1, cutoff=0.0)
    assert k == 6
    Wo, logo = oracle.train_online(W0, 10, 10, 0, X, 5, 0.3, 5.0, 7, kind=1, eps=0.0, k=math.log(100.0))
    assert np.array_equal(log, logo)
    assert np.abs(W.astype(np.float64) - Wo).max() <= 1e-4


def test_spec_c2_prefix_equals_register_kernel(som, monkeypatch):
    """c2 (20x20 hex, 5,000 x 3,000), first 50,000 steps: kernel 6 takes the
    exact fallback on near-ties (counted) and still gives kernel 2's BMU log
    and weights bit for bit."""
    cfg = dict(CONFIGS["c2"])
    C = bank_corpus(cfg["n"], cfg["d"], seed=1)
    X = C.dense()
    W0 = init_rows(X, cfg["rows"] * cfg["cols"], 1001)
    T = 50000
    W6, log6, k6, fb = _train(som, cfg["rows"], cfg["cols"], cfg["topo"], X, W0, cfg["epochs"], 0.1,
                              cfg["sigma0"], 1, t_end=T)
    monkeypatch.setenv("SOM_TRAIN_SPEC", "0")
    W2, log2, k2, _ = _train(som, cfg["rows"], cfg["cols"], cfg["topo"], X, W0, cfg["epochs"], 0.1,
                             cfg["sigma0"], 1, t_end=T)
    assert (k6, k2) == (6, 2)
    assert fb > 0
    assert np.array_equal(log6, log2)
    assert np.array_equal(W6, W2)
    print(f" [c2 prefix: {fb} of {T} steps took the exact fallback]", end="")


def test_hybrid_c2_full_schedule_equals_register_kernel(som, monkeypatch):
    """SOM_TRAIN_SPEC=2 (kernel id 7): kernel 6 while the neighbourhood covers
    >= 70 % of the map, then kernel 2, over the full c2 schedule (500,000
    steps): two launches, and the BMU log and weights of kernel 2 alone
    (which test_c2_full_schedule checks against the oracle) bit for bit."""
    cfg = dict(CONFIGS["c2"])
    C = bank_corpus(cfg["n"], cfg["d"], seed=1)
    X = C.dense()
    W0 = init_rows(X, cfg["rows"] * cfg["cols"], 1001)
    out = {}
    for mode in ("2", "0"):
        monkeypatch.setenv("SOM_TRAIN_SPEC", mode)
        with som.SOM(cfg["rows"], cfg["cols"], cfg["d"], cfg["topo"]) as m:
            m.set_weights(W0)
            log = np.full(cfg["n"] * cfg["epochs"], -7, np.int32)
            m.train_online(X, epochs=cfg["epochs"], alpha0=0.1, sigma0=cfg["sigma0"], seed=1, bmu_log=log)
            _, _, launches = som.som_last_stats(m.h)
            out[mode] = (m.get_weights(), log, som.som_last_train_config(m.h)[1], launches)
    assert out["2"][2:] == (7, 2) and out["0"][2:] == (2, 1)
    assert np.array_equal(out["2"][1], out["0"][1])
    assert np.array_equal(out["2"][0], out["0"][0])
