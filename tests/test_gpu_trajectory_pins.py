"""SURVEY §8.C trajectory pins at the configs' real shapes: the GPU BMU log
equals the oracle's and the weights agree (bar: BMU log identical, weights
within 1e-4 max-abs; observed bit-identical) over
  * c3: 50x50 hex, the real 50,000 x 10,000 corpus, the first 2,000 steps
    of the 10-epoch schedule (W = 100 MB, the streamed kernels);
  * c4: 100x100 hex, the real 200,000 x 20,000 corpus (CSR), the first 200
    steps of the 2-epoch schedule (W = 800 MB);
  * neuron sharding at P = 8 emulated on one device (8 handles, 8 grids,
    mailbox exchange) against P = 1 and the oracle."""
import numpy as np
import pytest

import oracle
from synth import CONFIGS, bank_corpus, init_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def som():
    from paper_1905_09598_b200 import som as s
    s.lib()
    return s


def _assert_same(W, log, Wo, logo):
    assert np.array_equal(log, logo), f"BMU log differs first at step {int(np.argmax(log != logo))}"
    assert np.abs(W - Wo).max() <= 1e-4
    return bool(np.array_equal(W, Wo))


@pytest.mark.parametrize("csr", [False, True])
def test_c3_real_corpus_2000_steps(som, csr):
    cfg = CONFIGS["c3"]
    C = bank_corpus(cfg["n"], cfg["d"], seed=1 + 300)
    N = cfg["rows"] * cfg["cols"]
    X = C.dense()
    W0 = init_rows(X, N, 1301)
    steps = 2000
    with som.SOM(cfg["rows"], cfg["cols"], cfg["d"], cfg["topo"]) as m:
        m.set_weights(W0)
        log = np.empty(steps, np.int32)
        if csr:
            m.train_online_csr(C.indptr, C.indices, C.data, C.n, cfg["epochs"], alpha0=0.1, sigma0=cfg["sigma0"],
                               seed=1, t_end=steps, bmu_log=log)
        else:
            m.train_online(X, epochs=cfg["epochs"], alpha0=0.1, sigma0=cfg["sigma0"], seed=1, t_end=steps,
                           bmu_log=log)
        kern = som.som_last_train_config(m.h)[1]
        W = m.get_weights()
    Wo, logo = oracle.train_online(W0, cfg["rows"], cfg["cols"], cfg["topo"], X, cfg["epochs"], 0.1, cfg["sigma0"],
                                   1, t_end=steps)
    bit = _assert_same(W, log, Wo, logo)
    print(f" [c3 2000 steps {'csr' if csr else 'dense'}: kernel {kern}, bit-identical W: {bit}]", end="")


def test_c4_real_corpus_200_steps(som):
    cfg = CONFIGS["c4"]
    C = bank_corpus(cfg["n"], cfg["d"], seed=1 + 400)
    N = cfg["rows"] * cfg["cols"]
    # the init rows: N distinct documents, densified one by one (no 16 GB dense copy)
    idx = np.sort(np.random.default_rng(1401).choice(C.n, N, replace=False))
    W0 = np.zeros((N, cfg["d"]), np.float32)
    for u, i in enumerate(idx):
        W0[u, C.indices[C.indptr[i]:C.indptr[i + 1]]] = C.data[C.indptr[i]:C.indptr[i + 1]]
    steps = 200
    with som.SOM(cfg["rows"], cfg["cols"], cfg["d"], cfg["topo"]) as m:
        m.set_weights(W0)
        log = np.empty(steps, np.int32)
        m.train_online_csr(C.indptr, C.indices, C.data, C.n, cfg["epochs"], alpha0=0.1, sigma0=cfg["sigma0"],
                           seed=1, t_end=steps, bmu_log=log)
        kern = som.som_last_train_config(m.h)[1]
        W = m.get_weights()
    Wo, logo = oracle.train_online_csr(W0, cfg["rows"], cfg["cols"], cfg["topo"], C.indptr, C.indices, C.data,
                                       cfg["epochs"], 0.1, cfg["sigma0"], 1, t_end=steps)
    bit = _assert_same(W, log, Wo, logo)
    print(f" [c4 200 steps csr: kernel {kern}, bit-identical W: {bit}]", end="")


def test_neuron_sharded_p8_identity(som):
    from test_gpu_sharded import _run_sharded
    C = bank_corpus(400, 512, seed=46)
    X = C.dense()
    W0 = init_rows(X, 16 * 16, 46)
    T = 3 * 400
    W, logs = _run_sharded(som, 8, 16, 16, 1, X, W0, 3, 8.0, 7, 8, [(0, 500), (500, T)])
    with som.SOM(16, 16, 512, 1) as m:
        m.set_weights(W0)
        ref_log = np.empty(T, np.int32)
        m.train_online(X, epochs=3, alpha0=0.1, sigma0=8.0, seed=7, bmu_log=ref_log)
        Wref = m.get_weights()
    for r in range(8):
        assert np.array_equal(logs[r], ref_log), f"rank {r} BMU log differs"
    assert np.array_equal(W, Wref)
    Wo, logo = oracle.train_online(W0, 16, 16, 1, X, 3, 0.1, 8.0, 7)
    _assert_same(W, ref_log, Wo, logo)
