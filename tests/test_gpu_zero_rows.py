"""All-zero rows ("retained but excluded from training sample draws",
S:218, "mean over nonzero rows"): the GPU draws only the
non-zero rows and scores only them, matching the oracle, on every training
kernel family; a corpus of zero rows only is SOM_EEMPTY."""
import numpy as np
import pytest

import oracle
from synth import bank_corpus, init_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def som():
    from paper_1905_09598_b200 import som as s
    s.lib()
    return s


def _with_zero_rows(n, d, seed, frac=0.2):
    C = bank_corpus(n, d, seed=seed)
    X = C.dense()
    rng = np.random.default_rng(seed)
    zero = rng.choice(n, int(frac * n), replace=False)
    X[zero] = 0.0
    rp, ci, va = C.indptr, C.indices, C.data.copy()
    for i in zero:                       # CSR twin: explicit zeros stay in the pattern
        va[rp[i]:rp[i + 1]] = 0.0
    return X, (rp, ci, va), np.sort(zero)


@pytest.mark.parametrize("rows,cols,d,mode", [(10, 10, 500, "auto"), (6, 7, 96, "small"), (20, 20, 3000, "glb"),
                                             (12, 12, 501, "auto")])
def test_training_skips_zero_rows(som, rows, cols, d, mode):
    n = 300
    X, _, zero = _with_zero_rows(n, d, 7)
    W0 = init_rows(X[np.setdiff1d(np.arange(n), zero)], rows * cols, 7)
    T = 3 * n
    with som.SOM(rows, cols, d, 1) as m:
        if mode == "glb":
            som.som_set_train_mode(m.h, som.SOM_TRAIN_W_GLOBAL)
        m.set_weights(W0)
        log = np.empty(T, np.int32)
        m.train_online(X, epochs=3, alpha0=0.1, sigma0=rows / 2, seed=3, bmu_log=log)
        W = m.get_weights()
        qe, te = m.errors(X)
    Wo, logo = oracle.train_online(W0, rows, cols, 1, X, 3, 0.1, rows / 2, 3)
    assert np.array_equal(log, logo)
    assert np.abs(W - Wo).max() <= 1e-4
    assert abs(qe - oracle.qerror(Wo, X)) <= 1e-6
    assert te == oracle.topographic_error(Wo, rows, cols, 1, X)


def test_csr_training_and_errors_skip_zero_rows(som):
    """c3-like rows through the CSR kernels (sparse distance path), zero rows
    holding explicit 0.0 entries."""
    n, d = 2000, 10000
    X, (rp, ci, va), zero = _with_zero_rows(n, d, 8, frac=0.1)
    W0 = init_rows(X[np.setdiff1d(np.arange(n), zero)], 2500, 8)
    steps = 120
    with som.SOM(50, 50, d, 1) as m:
        m.set_weights(W0)
        log = np.empty(steps, np.int32)
        m.train_online_csr(rp, ci, va, n, 10, alpha0=0.1, sigma0=25.0, seed=4, t_end=steps, bmu_log=log)
        W = m.get_weights()
        qe, te = m.errors_csr(rp, ci, va, n)
    Wo, logo = oracle.train_online_csr(W0, 50, 50, 1, rp, ci, va, 10, 0.1, 25.0, 4, t_end=steps)
    assert np.array_equal(log, logo)
    assert np.abs(W - Wo).max() <= 1e-4
    assert abs(qe - oracle.qerror(Wo, X)) <= 1e-6
    assert te == oracle.topographic_error(Wo, 50, 50, 1, X)


def test_all_zero_rows_is_empty(som):
    with som.SOM(3, 3, 16, 1) as m:
        with pytest.raises(som.SomError) as e:
            m.train_online(np.zeros((5, 16), np.float32), epochs=1, sigma0=1.5)
        assert e.value.status == som.SOM_EEMPTY
        with pytest.raises(som.SomError) as e:
            m.errors(np.zeros((5, 16), np.float32))
        assert e.value.status == som.SOM_EEMPTY
        b1, _, _ = m.map(np.zeros((5, 16), np.float32))     # mapping still assigns every row
        assert np.all(b1 == 0)
